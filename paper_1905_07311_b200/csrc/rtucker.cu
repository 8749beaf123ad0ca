// librtucker: C ABI (include/rtucker.h) and the host orchestrator of the randomized
// Tucker algorithms.  Every arithmetic step runs in the kernels of sketch.cu, ttm.cu,
// linalg.cu, sparse.cu; this file only sequences them, validates arguments, manages
// workspace (stream-ordered allocations) and the collectives of the sharded path.
#include <cmath>
#include <cstring>
#include <algorithm>
#include <numeric>
#include <functional>
#include <mutex>
#include <vector>

#include "comm.h"
#include "kernels_extra.h"
#include "orchestrate.h"

using namespace rt;

struct rtucker_ctx {
  Ctx c;
};

namespace rt {

void set_smem_attr(const void *func, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void *, size_t>> done;  // largest size set per kernel
  std::lock_guard<std::mutex> lk(mu);
  for (auto &e : done)
    if (e.first == func) {
      if (e.second >= bytes) return;
      RT_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
      e.second = bytes;
      return;
    }
  RT_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done.emplace_back(func, bytes);
}

// Reads and clears the device status word (synchronising calls only).
void check_status(Ctx &c) {
  unsigned h = 0;
  RT_CUDA(cudaMemcpyAsync(&h, c.status, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  if (!h) return;
  RT_CUDA(cudaMemsetAsync(c.status, 0, sizeof(unsigned), c.stream));
  if (h & ST_SHARD_LAYOUT)
    throw Error(RTUCKER_EINVAL, "the shards of the ranks do not tile the last mode [0, I_d) (rank order)");
  if (h & ST_BAD_INDEX) throw Error(RTUCKER_EINVAL, "a COO index lies outside its mode's range");
  if (h & ST_SINGULAR_PQ) throw Error(RTUCKER_ENUMERIC, "SP-STHOSVD: singular P^T Q (fewer than l independent rows)");
  if (h & ST_EIG_NOT_CONVERGED)
    throw Error(RTUCKER_ENUMERIC, "a Jacobi eigensolve did not converge within its sweep cap");
}

// ---------------------------------------------------------------- argument checks --
static DT to_dt(rtucker_dtype t) {
  if (t == RTUCKER_F32) return DT::F32;
  if (t == RTUCKER_F64) return DT::F64;
  throw Error(RTUCKER_EINVAL, "dtype must be RTUCKER_F32 or RTUCKER_F64");
}

void prepare_dense(Ctx &c, const rtucker_dense_desc *X, DenseIn &in) {
  RT_REQUIRE(X != nullptr, "null tensor descriptor");
  if (X->d > kMaxModes) throw Error(RTUCKER_EUNSUPPORTED, "d > RTUCKER_MAX_MODES");
  RT_REQUIRE(X->d >= 1, "d must be >= 1");
  RT_REQUIRE(X->data != nullptr, "null tensor data");
  in.dt = to_dt(X->dtype);
  in.d = X->d;
  for (int k = 0; k < in.d; ++k) {
    RT_REQUIRE(X->dims[k] >= 1, "every dim must be >= 1");
    in.gdims[k] = X->dims[k];
    in.ldims[k] = X->dims[k];
  }
  // multi-rank contract (rtucker.h): every rank holds a non-empty slab of the last mode
  RT_REQUIRE(c.nranks == 1 || X->shard_extent >= 1,
             "multi-rank calls need a sharded input (shard_extent >= 1 on every rank, so I_d >= nranks)");
  in.sharded = X->shard_extent > 0 && (X->shard_extent != X->dims[in.d - 1] || c.nranks > 1 || c.loopback_sharding);
  in.offset = 0;
  if (X->shard_extent > 0) {
    RT_REQUIRE(X->shard_offset >= 0 && X->shard_offset + X->shard_extent <= X->dims[in.d - 1],
               "shard range outside the last mode");
    in.ldims[in.d - 1] = X->shard_extent;
    in.offset = X->shard_offset;
  }
  RT_REQUIRE(!in.sharded || c.nranks > 1 || (c.loopback_sharding && X->shard_extent == X->dims[in.d - 1]),
             "a partial shard needs a multi-rank context");
  const int64_t n = prod(in.ldims, in.d);
  if (X->memory == RTUCKER_HOST) {
    in.owned.alloc(c, n * dt_size(in.dt));
    RT_CUDA(cudaMemcpyAsync(in.owned.p, X->data, n * dt_size(in.dt), cudaMemcpyHostToDevice, c.stream));
    in.ptr = in.owned.p;
  } else {
    in.ptr = X->data;
  }
}

void check_order(const int32_t *order, int d, int32_t *out, const int64_t *dims, bool sharded) {
  if (order) {
    bool seen[kMaxModes] = {false};
    for (int k = 0; k < d; ++k) {
      RT_REQUIRE(order[k] >= 0 && order[k] < d && !seen[order[k]], "order is not a permutation");
      seen[order[k]] = true;
      out[k] = order[k];
    }
  } else {
    // process the largest modes first, ties by ascending index
    std::iota(out, out + d, 0);
    std::stable_sort(out, out + d, [&](int a, int b) { return dims[a] > dims[b]; });
    if (sharded) {  // sharded dense runs process the sharded last mode last
      std::stable_partition(out, out + d, [&](int a) { return a != d - 1; });
    }
  }
  RT_REQUIRE(!sharded || out[d - 1] == d - 1, "a sharded tensor must be processed with its last mode last");
}

// l_n = min(r_n + p, I_n, prod others) on the current dims (reading R5).
void rank_caps(const int64_t *dims, int d, int n, int64_t r, int p, bool strict, int &ell, int &rr) {
  int64_t others = 1;
  for (int k = 0; k < d; ++k)
    if (k != n) others *= dims[k];
  const int64_t cap = std::min<int64_t>(dims[n], others);
  int64_t e = r + p;
  if (e > cap) {
    RT_REQUIRE(!strict, "r_n + p exceeds min(I_n, prod_{k!=n} I_k) (RTUCKER_STRICT)");
    e = cap;
  }
  ell = (int)e;
  rr = (int)std::min<int64_t>(r, e);
}

// --------------------------------------------------------------------- result ------
// Result structs live in pinned memory (device-to-host scalar copies land in them
// asynchronously).  They are recycled through a process-wide free list: cudaMallocHost takes
// driver locks and stalled concurrent kernel launches when called once per call in a
// throughput loop; cudaFreeHost would synchronise the device.
std::mutex g_result_mu;
std::vector<rtucker_result *> g_result_free;
constexpr int kResultSlab = 64;

rtucker_result *new_result(int d) {
  rtucker_result *r = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_result_mu);
    if (!g_result_free.empty()) {
      r = g_result_free.back();
      g_result_free.pop_back();
    }
  }
  if (!r) {
    // the free list is empty: pin a slab of kResultSlab structs at once (a throughput loop that
    // keeps K results alive paid one cudaMallocHost per call beyond the recycled ones, up to
    // ~16 ms each under driver contention: 16.6 ms/step measured for a 3.9 ms step)
    rtucker_result *slab = nullptr;
    if (cudaMallocHost((void **)&slab, sizeof(rtucker_result) * kResultSlab) != cudaSuccess)
      throw Error(RTUCKER_ENOMEM, "cudaMallocHost(result slab)");
    r = slab;
    std::lock_guard<std::mutex> lk(g_result_mu);
    for (int i = kResultSlab - 1; i >= 1; --i) g_result_free.push_back(slab + i);
  }
  memset(r, 0, sizeof *r);
  r->d = d;
  r->dtype = RTUCKER_F64;
  r->memory = RTUCKER_DEVICE;
  return r;
}

static void free_result_struct(rtucker_result *r) {
  std::lock_guard<std::mutex> lk(g_result_mu);
  g_result_free.push_back(r);
}

void free_result(Ctx &c, rtucker_result *r) {
  if (!r) return;
  auto fr = [&](void *p) {
    if (!p) return;
    if (r->memory == RTUCKER_HOST) cudaFreeHost(p);
    else dev_free(c, p);
  };
  fr(r->core);
  for (int k = 0; k < kMaxModes; ++k) {
    fr(r->factors[k]);
    fr(r->core_idx[k]);
    fr(r->selection[k]);
  }
  fr(r->core_vals);
  // asynchronous copies into the struct must land before it is handed out again (cudaFreeHost,
  // used before, synchronised the whole device here)
  cudaStreamSynchronize(c.stream);
  std::lock_guard<std::mutex> lk(g_result_mu);
  g_result_free.push_back(r);
}

// Moves device result buffers to pinned host memory when RTUCKER_RESULT_HOST is set.
void finish_result(Ctx &c, rtucker_result *r, uint32_t flags) {
  if (!(flags & RTUCKER_RESULT_HOST)) return;
  auto mv = [&](void *&p, size_t bytes) {
    if (!p) return;
    void *h = nullptr;
    RT_CUDA(cudaMallocHost(&h, std::max<size_t>(bytes, 1)));
    RT_CUDA(cudaMemcpyAsync(h, p, bytes, cudaMemcpyDeviceToHost, c.stream));
    dev_free(c, p);
    p = h;
  };
  const size_t vs = r->dtype == RTUCKER_F64 ? 8 : 4;
  int64_t core_n = 1;
  for (int k = 0; k < r->d; ++k) core_n *= r->ranks[k];
  if (r->core) mv(r->core, core_n * vs);
  for (int k = 0; k < r->d; ++k) {
    if (r->factors[k]) mv(r->factors[k], (size_t)r->dims[k] * r->ranks[k] * 8);
    if (r->core_idx[k]) mv(*(void **)&r->core_idx[k], r->core_nnz * 4);
    if (r->selection[k]) mv(*(void **)&r->selection[k], r->ranks[k] * 8);
  }
  if (r->core_vals) mv(r->core_vals, r->core_nnz * vs);
  r->memory = RTUCKER_HOST;
  check_status(c);  // synchronises
}

// ------------------------------------------------------------- CUDA-graph plans ----
// RTUCKER_GRAPH for the fixed-rank calls (include/rtucker.h).  A plan is keyed by everything the
// enqueued work depends on; its template result points into the plan's arena (core, factors)
// and its `internal` field at the device residual block (2 d doubles: ||G||^2, residual per mode).
struct GraphPlan {
  std::vector<int64_t> key;
  cudaGraphExec_t exec = nullptr;
  char *arena = nullptr;
  size_t arena_size = 0;
  rtucker_result *tmpl = nullptr;
  uint64_t launches = 0;
};
struct GraphCache {
  std::vector<GraphPlan *> plans;
};

static std::vector<int64_t> plan_key(int algo, const rtucker_dense_desc *X, const int64_t *ranks, int p, uint64_t seed,
                                     const int32_t *order, uint32_t flags, const Ctx &c) {
  std::vector<int64_t> k = {algo, (int64_t)(uintptr_t)X->data, X->dtype, X->d, X->shard_offset, X->shard_extent,
                            X->memory, p, (int64_t)seed, (int64_t)(flags & ~RTUCKER_GRAPH), c.nranks,
                            c.loopback_sharding ? 1 : 0};
  for (int i = 0; i < X->d && i < kMaxModes; ++i) {
    k.push_back(X->dims[i]);
    k.push_back(ranks[i]);
    k.push_back(order ? order[i] : -1);
  }
  return k;
}

void destroy_graphs(Ctx &c) {
  auto *gc = (GraphCache *)c.graphs;
  if (!gc) return;
  for (GraphPlan *pl : gc->plans) {
    if (pl->exec) cudaGraphExecDestroy(pl->exec);
    if (pl->arena) cudaFree(pl->arena);
    if (pl->tmpl) {
      std::lock_guard<std::mutex> lk(g_result_mu);
      g_result_free.push_back(pl->tmpl);
    }
    delete pl;
  }
  delete gc;
  c.graphs = nullptr;
}

rtucker_result *run_fixed_rank(Ctx &c, int algo, const rtucker_dense_desc *X, const int64_t *ranks, int p,
                               uint64_t seed, const int32_t *order, uint32_t flags) {
  auto body = [&]() {
    return algo == 0 ? run_sthosvd(c, X, ranks, p, seed, order, flags) : run_hosvd(c, X, ranks, p, seed, flags);
  };
  if (!(flags & RTUCKER_GRAPH) || (flags & RTUCKER_RESULT_HOST) || c.profiling || !X || !ranks ||
      X->memory != RTUCKER_DEVICE || X->d < 1 || X->d > kMaxModes)
    return body();
  if (!c.graphs) c.graphs = new GraphCache;
  auto *gc = (GraphCache *)c.graphs;
  const std::vector<int64_t> key = plan_key(algo, X, ranks, p, seed, order, flags, c);
  GraphPlan *pl = nullptr;
  for (GraphPlan *q : gc->plans)
    if (q->key == key) pl = q;
  if (pl && !pl->exec) return body();  // capture failed earlier for this key
  if (!pl) {
    // 1. eager call (its result is returned) counting the workspace it allocates
    c.arena = Ctx::Arena{};
    c.arena.counting = true;
    rtucker_result *res = nullptr;
    try {
      res = body();
    } catch (...) {
      c.arena = Ctx::Arena{};
      throw;
    }
    const size_t need = c.arena.counted + (1 << 20);
    c.arena = Ctx::Arena{};
    // 2. capture the same call with the arena allocator
    auto *np = new GraphPlan;
    np->key = key;
    np->arena_size = need;
    cudaError_t e = cudaMalloc((void **)&np->arena, need);
    if (e != cudaSuccess) {  // no room for a plan: stay eager
      (void)cudaGetLastError();
      delete np;
      return res;
    }
    c.arena.base = np->arena;
    c.arena.size = need;
    c.arena.on = true;
    c.capturing = true;
    const uint64_t l0 = c.launches;
    cudaGraph_t g = nullptr;
    rtucker_result *tmpl = nullptr;
    try {
      RT_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed));
      tmpl = body();
      RT_CUDA(cudaStreamEndCapture(c.stream, &g));
      RT_CUDA(cudaGraphInstantiate(&np->exec, g, 0));
    } catch (const std::exception &ex) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(c.stream, &junk);
      if (junk) cudaGraphDestroy(junk);
      if (g) cudaGraphDestroy(g);
      c.capturing = false;
      c.arena = Ctx::Arena{};
      cudaFree(np->arena);
      np->arena = nullptr;
      (void)cudaGetLastError();
      // capture failed: the eager result stands; the key stays as an eager-only plan (no retry)
      fprintf(stderr, "[rtucker] RTUCKER_GRAPH: capture failed, calls with this key stay eager: %s\n", ex.what());
      gc->plans.push_back(np);
      return res;
    }
    cudaGraphDestroy(g);
    np->launches = c.launches - l0;
    c.launches = l0;
    c.capturing = false;
    c.arena = Ctx::Arena{};
    np->tmpl = tmpl;
    gc->plans.push_back(np);
    return res;
  }
  // 3. replay: one graph launch, then the outputs are copied into a fresh result
  RT_CUDA(cudaGraphLaunch(pl->exec, c.stream));
  c.launches += pl->launches;
  const rtucker_result *t = pl->tmpl;
  ResultGuard rg{c, new_result(t->d)};
  rtucker_result *r = rg.r;
  memcpy(r->dims, t->dims, sizeof r->dims);
  memcpy(r->ranks, t->ranks, sizeof r->ranks);
  memcpy(r->ell, t->ell, sizeof r->ell);
  memcpy(r->order, t->order, sizeof r->order);
  r->seed = t->seed;
  r->flags = flags;
  r->dtype = t->dtype;
  int64_t ncore = 1;
  for (int k = 0; k < t->d; ++k) ncore *= t->ranks[k];
  if (t->core) {
    r->core = dev_alloc(c, sizeof(double) * ncore);
    RT_CUDA(cudaMemcpyAsync(r->core, t->core, sizeof(double) * ncore, cudaMemcpyDeviceToDevice, c.stream));
  }
  for (int k = 0; k < t->d; ++k) {
    if (!t->factors[k]) continue;
    const size_t b = sizeof(double) * t->dims[k] * t->ranks[k];
    r->factors[k] = dev_alloc(c, b);
    RT_CUDA(cudaMemcpyAsync(r->factors[k], t->factors[k], b, cudaMemcpyDeviceToDevice, c.stream));
  }
  if (t->internal) {  // residual block: [||G||^2 at 2n, residual at 2n+1]
    const double *scal = (const double *)t->internal;
    for (int k = 0; k < t->d; ++k)
      RT_CUDA(cudaMemcpyAsync(&r->mode_residual_sq[k], scal + 2 * k + 1, sizeof(double), cudaMemcpyDeviceToHost,
                              c.stream));
    const int first = algo == 0 ? t->order[0] : 0;
    RT_CUDA(cudaMemcpyAsync(&r->norm_sq, scal + 2 * first, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  }
  return rg.release();
}

}  // namespace rt

// ======================================================================= C ABI ======
static rtucker_status guard(rtucker_ctx *ctx, const std::function<void()> &fn) {
  try {
    fn();
    if (ctx) ctx->c.last_error.clear();
    return RTUCKER_OK;
  } catch (const Error &e) {
    if (ctx) ctx->c.last_error = e.what();
    return e.code;
  } catch (const std::exception &e) {
    if (ctx) ctx->c.last_error = e.what();
    return RTUCKER_ECUDA;
  }
}

extern "C" {

const char *rtucker_version(void) { return "rtucker 0.1 (sm_100a)"; }

rtucker_status rtucker_memcpy(rtucker_ctx *ctx, void *dst, const void *src, size_t bytes, int kind) {
  if (!ctx || (!dst && bytes) || (!src && bytes) || kind < 0 || kind > 4) return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    if (bytes) RT_CUDA(cudaMemcpyAsync(dst, src, bytes, (cudaMemcpyKind)kind, ctx->c.stream));
  });
}

rtucker_status rtucker_sync(rtucker_ctx *ctx) {
  if (!ctx) return RTUCKER_EINVAL;
  return guard(ctx, [&] { check_status(ctx->c); });
}

rtucker_status rtucker_debug_loopback_sharding(rtucker_ctx *ctx, int enabled) {
  if (!ctx || ctx->c.nranks != 1) return RTUCKER_EINVAL;
  ctx->c.loopback_sharding = enabled != 0;
  return RTUCKER_OK;
}

rtucker_status rtucker_set_profiling(rtucker_ctx *ctx, int enabled) {
  if (!ctx) return RTUCKER_EINVAL;
  ctx->c.profiling = enabled != 0;
  return RTUCKER_OK;
}

rtucker_status rtucker_phase_times(rtucker_ctx *ctx, double *ms, int64_t *counts, int reset) {
  if (!ctx) return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    Ctx &c = ctx->c;
    RT_CUDA(cudaStreamSynchronize(c.stream));
    for (auto &e : c.events) {
      float t = 0.f;
      RT_CUDA(cudaEventElapsedTime(&t, e.a, e.b));
      c.phase_ms[e.slot] += t;
      c.phase_n[e.slot] += 1;
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    c.events.clear();
    if (ms) memcpy(ms, c.phase_ms, sizeof c.phase_ms);
    if (counts) memcpy(counts, c.phase_n, sizeof c.phase_n);
    if (reset) {
      memset(c.phase_ms, 0, sizeof c.phase_ms);
      memset(c.phase_n, 0, sizeof c.phase_n);
    }
  });
}

rtucker_status rtucker_ctx_create(int device, void *cuda_stream, const void *nccl_unique_id, int rank,
                                  int nranks, rtucker_alloc_fn alloc_fn, rtucker_free_fn free_fn,
                                  void *alloc_user, rtucker_ctx **out) {
  if (!out) return RTUCKER_EINVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return RTUCKER_EINVAL;
  if (nranks > 1 && !nccl_unique_id) return RTUCKER_EINVAL;
  if ((alloc_fn == nullptr) != (free_fn == nullptr)) return RTUCKER_EINVAL;
  rtucker_ctx *ctx = new rtucker_ctx;
  ctx->c.alloc_fn = alloc_fn;
  ctx->c.free_fn = free_fn;
  ctx->c.alloc_user = alloc_user;
  rtucker_status st = guard(ctx, [&] {
    RT_CUDA(cudaSetDevice(device));
    ctx->c.device = device;
    if (cuda_stream) {
      ctx->c.stream = (cudaStream_t)cuda_stream;
    } else {
      RT_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
      ctx->c.own_stream = true;
    }
    RT_CUDA(cudaDeviceGetAttribute(&ctx->c.num_sms, cudaDevAttrMultiProcessorCount, device));
    RT_CUDA(cudaStreamCreateWithFlags(&ctx->c.aux, cudaStreamNonBlocking));
    // library-owned stream-ordered pool (used when no allocation hooks are given); freed
    // workspace stays in it between calls (no re-mapping of the large B / shrunk-core
    // buffers on every decomposition).  The device's default pool is not modified.
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = device;
    RT_CUDA(cudaMemPoolCreate(&ctx->c.pool, &pp));
    uint64_t thr = UINT64_MAX;
    RT_CUDA(cudaMemPoolSetAttribute(ctx->c.pool, cudaMemPoolAttrReleaseThreshold, &thr));
    RT_CUDA(cudaMalloc((void **)&ctx->c.status, sizeof(unsigned)));
    RT_CUDA(cudaMemset(ctx->c.status, 0, sizeof(unsigned)));
    // pin the first slab of result structs now, outside any caller's timed or captured loop
    {
      std::unique_lock<std::mutex> lk(g_result_mu);
      const bool empty = g_result_free.empty();
      lk.unlock();
      if (empty) free_result_struct(new_result(0));
    }
    ctx->c.rank = rank;
    ctx->c.nranks = nranks;
    if (nranks > 1) ctx->c.comm = comm_create(nccl_unique_id, rank, nranks);
  });
  if (st != RTUCKER_OK) {
    if (ctx->c.status) cudaFree(ctx->c.status);
    if (ctx->c.pool) cudaMemPoolDestroy(ctx->c.pool);
    delete ctx;
    return st;
  }
  *out = ctx;
  return RTUCKER_OK;
}

void rtucker_ctx_destroy(rtucker_ctx *ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->c.stream);
  destroy_graphs(ctx->c);
  if (ctx->c.aux) {
    cudaStreamSynchronize(ctx->c.aux);
    cudaStreamDestroy(ctx->c.aux);
  }
  if (ctx->c.sk_flags) cudaFree(ctx->c.sk_flags);
  if (ctx->c.status) cudaFree(ctx->c.status);
  comm_destroy(ctx->c.comm);
  if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
  if (ctx->c.pool) {
    cudaDeviceSynchronize();
    cudaMemPoolDestroy(ctx->c.pool);
  }
  delete ctx;
}

rtucker_status rtucker_ctx_set_stream(rtucker_ctx *ctx, void *cuda_stream) {
  if (!ctx || !cuda_stream) return RTUCKER_EINVAL;
  if (ctx->c.own_stream) {
    cudaStreamSynchronize(ctx->c.stream);
    cudaStreamDestroy(ctx->c.stream);
    ctx->c.own_stream = false;
  }
  ctx->c.stream = (cudaStream_t)cuda_stream;
  return RTUCKER_OK;
}

const char *rtucker_last_error(const rtucker_ctx *ctx) {
  return ctx ? ctx->c.last_error.c_str() : "null context";
}

uint64_t rtucker_launch_count(const rtucker_ctx *ctx) { return ctx ? ctx->c.launches : 0; }

rtucker_status rtucker_nccl_unique_id(void *out128) {
  if (!out128) return RTUCKER_EINVAL;
  return guard(nullptr, [&] { nccl_unique_id(out128); });
}

rtucker_status rtucker_hosvd(rtucker_ctx *ctx, const rtucker_dense_desc *X, const int64_t *ranks,
                             int32_t p, uint64_t seed, uint32_t flags, rtucker_result **out) {
  if (!ctx || !out || !ranks) return RTUCKER_EINVAL;
  *out = nullptr;
  return guard(ctx, [&] { *out = run_fixed_rank(ctx->c, 1, X, ranks, p, seed, nullptr, flags); });
}

rtucker_status rtucker_sthosvd(rtucker_ctx *ctx, const rtucker_dense_desc *X, const int64_t *ranks,
                               int32_t p, uint64_t seed, const int32_t *order, uint32_t flags,
                               rtucker_result **out) {
  if (!ctx || !out || !ranks) return RTUCKER_EINVAL;
  *out = nullptr;
  return guard(ctx, [&] { *out = run_fixed_rank(ctx->c, 0, X, ranks, p, seed, order, flags); });
}

rtucker_status rtucker_adaptive(rtucker_ctx *ctx, const rtucker_dense_desc *X, double tol, int32_t block,
                                const double *mode_tol, const int32_t *order, uint64_t seed,
                                uint32_t flags, rtucker_result **out) {
  if (!ctx || !out) return RTUCKER_EINVAL;
  *out = nullptr;
  return guard(ctx, [&] { *out = run_adaptive(ctx->c, X, tol, block, mode_tol, order, seed, flags); });
}

rtucker_status rtucker_sparse_sthosvd(rtucker_ctx *ctx, const rtucker_coo_desc *X, const int64_t *ranks,
                                      int32_t p, uint64_t seed, const int32_t *order, double eta,
                                      uint32_t flags, rtucker_result **out) {
  if (!ctx || !out || !ranks) return RTUCKER_EINVAL;
  *out = nullptr;
  return guard(ctx, [&] { *out = run_sparse_sthosvd(ctx->c, X, ranks, p, seed, order, eta, flags); });
}

void rtucker_result_free(rtucker_ctx *ctx, rtucker_result *res) {
  if (!ctx || !res) return;
  free_result(ctx->c, res);
}

rtucker_status rtucker_rel_error(rtucker_ctx *ctx, const rtucker_dense_desc *X, const rtucker_result *res,
                                 double *out) {
  if (!ctx || !res || !out) return RTUCKER_EINVAL;
  return guard(ctx, [&] { *out = run_rel_error(ctx->c, X, res); });
}

rtucker_status rtucker_debug_sketch(rtucker_ctx *ctx, const rtucker_dense_desc *X, int32_t mode, int32_t ell,
                                    int64_t k0, uint64_t seed, uint32_t flags, double *Y_out) {
  if (!ctx || !Y_out) return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    DenseIn in;
    prepare_dense(ctx->c, X, in);
    RT_REQUIRE(mode >= 0 && mode < in.d, "mode out of range");
    RT_REQUIRE(ell >= 1 && k0 >= 0, "ell >= 1 and k0 >= 0 required");
    const bool f64 = in.dt == DT::F64 || (flags & RTUCKER_ACCUM_MASK) == RTUCKER_ACCUM_FP64;
    sketch_dense(ctx->c, in.ptr, in.dt, mode_view(in.ldims, in.d, mode), mode, ell, k0, seed,
                 col_offset_for(in, in.ldims, mode), f64, Y_out, nullptr);
  });
}

rtucker_status rtucker_debug_ttm(rtucker_ctx *ctx, const rtucker_dense_desc *X, int32_t mode, const double *A,
                                 int32_t J, uint32_t flags, double *out, double *gram) {
  if (!ctx || !A || J < 1 || (!out && !gram)) return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    DenseIn in;
    prepare_dense(ctx->c, X, in);
    RT_REQUIRE(mode >= 0 && mode < in.d, "mode out of range");
    const ModeView v = mode_view(in.ldims, in.d, mode);
    const uint32_t acc = flags & RTUCKER_ACCUM_MASK;
    const bool f64 = in.dt == DT::F64 || acc == RTUCKER_ACCUM_FP64;
    ttm_dense(ctx->c, in.ptr, in.dt, v, A, v.I, J, out, DT::F64, f64, gram);
  });
}

rtucker_status rtucker_debug_omega(rtucker_ctx *ctx, rtucker_dtype dtype, uint64_t seed, int32_t mode,
                                   const int64_t *cols, int64_t n, int32_t ell, int64_t k0, void *out) {
  if (!ctx || !cols || !out || n < 0 || ell < 1 || k0 < 0) return RTUCKER_EINVAL;
  return guard(ctx, [&] { omega_rows(ctx->c, to_dt(dtype), seed, mode, cols, n, ell, k0, out); });
}

rtucker_status rtucker_debug_philox(rtucker_ctx *ctx, const uint32_t *ctr, int64_t n, uint32_t key0,
                                    uint32_t key1, uint32_t *out) {
  if (!ctx || !ctr || !out || n < 0) return RTUCKER_EINVAL;
  return guard(ctx, [&] { philox_raw(ctx->c, ctr, n, key0, key1, out); });
}

rtucker_status rtucker_debug_qr(rtucker_ctx *ctx, int64_t m, int32_t n, const double *Y, double *Q) {
  if (!ctx || !Y || !Q || n < 1 || m < n) return RTUCKER_EINVAL;
  return guard(ctx, [&] { thin_qr(ctx->c, Y, m, n, Q); });
}

rtucker_status rtucker_debug_eig(rtucker_ctx *ctx, int32_t n, const double *A, double *w, double *V,
                                 int32_t *sweeps_out) {
  if (!ctx || !A || !w || !V || n < 1) return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    DevBuf<int> sw(ctx->c, 1);
    sym_eig(ctx->c, A, n, w, V, sw.p);
    int h = 0;
    RT_CUDA(cudaMemcpyAsync(&h, sw.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->c.stream));
    RT_CUDA(cudaStreamSynchronize(ctx->c.stream));
    if (sweeps_out) *sweeps_out = h;
  });
}

rtucker_status rtucker_debug_gram_eig(rtucker_ctx *ctx, int32_t n, const double *A, double *w, double *V,
                                      int32_t *sweeps_out) {
  if (!ctx || !A || !w || !V || n < 1) return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    DevBuf<int> sw(ctx->c, 1);
    gram_eig(ctx->c, A, n, w, V, sw.p, 1);
    int h = 0;
    RT_CUDA(cudaMemcpyAsync(&h, sw.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->c.stream));
    RT_CUDA(cudaStreamSynchronize(ctx->c.stream));
    if (sweeps_out) *sweeps_out = h;
  });
}

rtucker_status rtucker_debug_gram_eig_ex(rtucker_ctx *ctx, int32_t n, const double *A, double *w, double *V,
                                         int32_t *sweeps_out, int32_t rel_acc, int32_t r_need) {
  if (!ctx || !A || !w || !V || n < 1 || r_need < 1) return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    DevBuf<int> sw(ctx->c, 1);
    sw.zero();
    gram_eig(ctx->c, A, n, w, V, sw.p, r_need, rel_acc != 0);
    int h = 0;
    RT_CUDA(cudaMemcpyAsync(&h, sw.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->c.stream));
    RT_CUDA(cudaStreamSynchronize(ctx->c.stream));
    if (sweeps_out) *sweeps_out = h;
    check_status(ctx->c);
  });
}

rtucker_status rtucker_debug_gemm(rtucker_ctx *ctx, int transA, int transB, int64_t m, int64_t n, int64_t k,
                                  const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc) {
  if (!ctx || !A || !B || !C || m < 1 || n < 1 || k < 1) return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    gemm_f64_batched(ctx->c, transA != 0, transB != 0, A, lda, 0, B, ldb, 0, C, ldc, 0, m, n, k, 1);
  });
}

rtucker_status rtucker_debug_gram(rtucker_ctx *ctx, int64_t L, int64_t K, int64_t R, const double *B, double *C) {
  if (!ctx || !B || !C || L < 1 || K < 1 || R < 1) return RTUCKER_EINVAL;
  return guard(ctx, [&] { gram_f64(ctx->c, B, L, K, R, C); });
}

rtucker_status rtucker_debug_coo_sketch(rtucker_ctx *ctx, const rtucker_coo_desc *X, int32_t mode, int32_t ell,
                                        uint64_t seed, uint32_t flags, double *Y_out) {
  if (!ctx || !X || !Y_out || X->d < 1 || X->d > RTUCKER_MAX_MODES || mode < 0 || mode >= X->d || ell < 1 ||
      ell > 64 || X->nnz < 0 || (X->dtype != RTUCKER_F32 && X->dtype != RTUCKER_F64))
    return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    debug_coo_sketch(ctx->c, X, mode, ell, seed, (flags & RTUCKER_ACCUM_MASK) == RTUCKER_ACCUM_FP64, Y_out);
    check_status(ctx->c);
  });
}

rtucker_status rtucker_debug_srrqr(rtucker_ctx *ctx, int64_t m, int32_t l, const double *Q, double eta,
                                   int64_t *sel, double *A, int32_t *swaps_out) {
  if (!ctx || !Q || !sel || !A || l < 1 || m < l || !(eta >= 1.0)) return RTUCKER_EINVAL;
  return guard(ctx, [&] {
    DevBuf<int> sw(ctx->c, 1);
    srrqr(ctx->c, Q, m, l, eta, sel, A, sw.p);
    int h = 0;
    RT_CUDA(cudaMemcpyAsync(&h, sw.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->c.stream));
    check_status(ctx->c);
    if (swaps_out) *swaps_out = h;
  });
}

}  // extern "C"
