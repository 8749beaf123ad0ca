// NCCL collectives for the sharded path: the library owns its own
// ncclComm_t, bootstrapped from a ncclUniqueId the caller broadcasts (the Python binding
// does it over torch.distributed).  NCCL is resolved at run time with dlopen so that the
// library does not pin an NCCL build: it binds to the libnccl.so.2 already loaded by the
// process (torch's) when there is one.
#include <dlfcn.h>
#include <nccl.h>

#include "comm.h"

namespace rt {

namespace {
struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi &api() {
  static NcclApi a;
  if (a.h) return a;
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char *n : names) {
    a.h = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (a.h) break;
  }
  if (!a.h)
    for (const char *n : names) {
      a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
  if (!a.h) return a;
  a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(a.h, "ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))dlsym(a.h, "ncclCommInitRank");
  a.CommDestroy = (decltype(a.CommDestroy))dlsym(a.h, "ncclCommDestroy");
  a.AllReduce = (decltype(a.AllReduce))dlsym(a.h, "ncclAllReduce");
  a.AllGather = (decltype(a.AllGather))dlsym(a.h, "ncclAllGather");
  a.GetErrorString = (decltype(a.GetErrorString))dlsym(a.h, "ncclGetErrorString");
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.AllGather;
  return a;
}

void check(ncclResult_t r, const char *what) {
  if (r != ncclSuccess) {
    std::string m = std::string(what) + ": " + (api().GetErrorString ? api().GetErrorString(r) : "nccl error");
    throw Error(RTUCKER_ENCCL, m);
  }
}
}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
};

void nccl_unique_id(void *out128) {
  NcclApi &a = api();
  if (!a.ok) throw Error(RTUCKER_ENCCL, "NCCL library not available");
  ncclUniqueId id;
  check(a.GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out128, &id, sizeof id);
}

Comm *comm_create(const void *id128, int rank, int nranks) {
  NcclApi &a = api();
  if (!a.ok) throw Error(RTUCKER_ENCCL, "NCCL library not available");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  Comm *c = new Comm;
  check(a.CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  return c;
}

void comm_destroy(Comm *c) {
  if (!c) return;
  if (c->comm && api().ok) api().CommDestroy(c->comm);
  delete c;
}

void allreduce_sum_f64(Ctx &ctx, double *buf, size_t n) {
  if (ctx.nranks <= 1 || n == 0) return;
  check(api().AllReduce(buf, buf, n, ncclFloat64, ncclSum, ctx.comm->comm, ctx.stream), "ncclAllReduce");
}

void allreduce_sum(Ctx &ctx, void *buf, size_t n, bool f64) {
  if (ctx.nranks <= 1 || n == 0) return;
  check(api().AllReduce(buf, buf, n, f64 ? ncclFloat64 : ncclFloat32, ncclSum, ctx.comm->comm,
                        ctx.stream),
        "ncclAllReduce");
}

void allgather_f64(Ctx &ctx, const double *send, double *recv, size_t n) {
  if (ctx.nranks <= 1) {
    if (send != recv)
      RT_CUDA(cudaMemcpyAsync(recv, send, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
    return;
  }
  check(api().AllGather(send, recv, n, ncclFloat64, ctx.comm->comm, ctx.stream), "ncclAllGather");
}

void allreduce_i64_sum(Ctx &ctx, void *buf, size_t n) {
  if (ctx.nranks <= 1 || n == 0) return;
  check(api().AllReduce(buf, buf, n, ncclInt64, ncclSum, ctx.comm->comm, ctx.stream), "ncclAllReduce(int64)");
}

void allreduce_u64_max(Ctx &ctx, void *buf, size_t n) {
  if (ctx.nranks <= 1 || n == 0) return;
  check(api().AllReduce(buf, buf, n, ncclUint64, ncclMax, ctx.comm->comm, ctx.stream), "ncclAllReduce(max)");
}

void allgather_i64(Ctx &ctx, const void *send, void *recv, size_t n) {
  if (ctx.nranks <= 1) {
    if (send != recv)
      RT_CUDA(cudaMemcpyAsync(recv, send, n * 8, cudaMemcpyDeviceToDevice, ctx.stream));
    return;
  }
  check(api().AllGather(send, recv, n, ncclInt64, ctx.comm->comm, ctx.stream), "ncclAllGather(int64)");
}

void allgather_bytes(Ctx &ctx, const void *send, void *recv, size_t bytes) {
  if (ctx.nranks <= 1) {
    if (send != recv) RT_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, ctx.stream));
    return;
  }
  check(api().AllGather(send, recv, bytes, ncclUint8, ctx.comm->comm, ctx.stream), "ncclAllGather(bytes)");
}

}  // namespace rt
