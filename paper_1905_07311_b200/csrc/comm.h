#pragma once
#include <cstring>
#include "common.cuh"

namespace rt {
void nccl_unique_id(void *out128);
Comm *comm_create(const void *id128, int rank, int nranks);
void comm_destroy(Comm *c);
void allreduce_sum_f64(Ctx &ctx, double *buf, size_t n);
void allreduce_sum(Ctx &ctx, void *buf, size_t n, bool f64);
void allgather_f64(Ctx &ctx, const double *send, double *recv, size_t n);
// integer collectives (exact): sums of int64 words, maxima of uint64 words, gathers
void allreduce_i64_sum(Ctx &ctx, void *buf, size_t n);
void allreduce_u64_max(Ctx &ctx, void *buf, size_t n);
void allgather_i64(Ctx &ctx, const void *send, void *recv, size_t n);
void allgather_bytes(Ctx &ctx, const void *send, void *recv, size_t bytes);
}  // namespace rt
