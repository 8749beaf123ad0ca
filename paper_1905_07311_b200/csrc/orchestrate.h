// Host orchestration of the algorithms (sequencing only; arithmetic is in the kernels).
#pragma once
#include <functional>
#include "kernels.h"

namespace rt {

struct DenseIn {
  const void *ptr = nullptr;
  DT dt = DT::F32;
  int d = 0;
  int64_t gdims[kMaxModes] = {0};  // global dims
  int64_t ldims[kMaxModes] = {0};  // local dims (last mode = shard extent)
  bool sharded = false;
  int64_t offset = 0;              // shard offset along the last mode
  DevBuf<unsigned char> owned;     // device copy of a host input
};

void prepare_dense(Ctx &c, const rtucker_dense_desc *X, DenseIn &in);
void check_order(const int32_t *order, int d, int32_t *out, const int64_t *dims, bool sharded);
void rank_caps(const int64_t *dims, int d, int n, int64_t r, int p, bool strict, int &ell, int &rr);
rtucker_result *new_result(int d);
void free_result(Ctx &c, rtucker_result *r);
void finish_result(Ctx &c, rtucker_result *r, uint32_t flags);
// Synchronises the context stream, reads and clears the device status word (StatusBit) and
// throws the matching error.
void check_status(Ctx &c);
// Fixed-rank entry (algo 0 = R-STHOSVD, 1 = R-HOSVD), with the RTUCKER_GRAPH replay path.
rtucker_result *run_fixed_rank(Ctx &c, int algo, const rtucker_dense_desc *X, const int64_t *ranks, int p,
                               uint64_t seed, const int32_t *order, uint32_t flags);
void destroy_graphs(Ctx &c);

// Global unfolding-column offset of this rank's slab for mode n < d-1 (the last mode is
// sharded): c_glob = c_loc + offset * prod_{k != n, k < d-1} dims_k.
inline int64_t col_offset_for(const DenseIn &in, const int64_t *cur, int n) {
  if (!in.sharded || n == in.d - 1) return 0;
  int64_t lm = 1;
  for (int k = 0; k < in.d - 1; ++k)
    if (k != n) lm *= cur[k];
  return lm * in.offset;
}

struct ResultGuard {  // frees a partially built result when an exception unwinds
  Ctx &c;
  rtucker_result *r;
  ~ResultGuard() {
    if (r) free_result(c, r);
  }
  rtucker_result *release() {
    rtucker_result *t = r;
    r = nullptr;
    return t;
  }
};

rtucker_result *run_sthosvd(Ctx &c, const rtucker_dense_desc *X, const int64_t *ranks, int p, uint64_t seed,
                            const int32_t *order, uint32_t flags);
rtucker_result *run_hosvd(Ctx &c, const rtucker_dense_desc *X, const int64_t *ranks, int p, uint64_t seed,
                          uint32_t flags);
rtucker_result *run_adaptive(Ctx &c, const rtucker_dense_desc *X, double tol, int block, const double *mode_tol,
                             const int32_t *order, uint64_t seed, uint32_t flags);
void debug_coo_sketch(Ctx &c, const rtucker_coo_desc *X, int mode, int ell, uint64_t seed, bool normals_f64,
                      double *Y);
rtucker_result *run_sparse_sthosvd(Ctx &c, const rtucker_coo_desc *X, const int64_t *ranks, int p,
                                   uint64_t seed, const int32_t *order, double eta, uint32_t flags);
double run_rel_error(Ctx &c, const rtucker_dense_desc *X, const rtucker_result *res);

}  // namespace rt
