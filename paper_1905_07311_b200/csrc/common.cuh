// Shared host/device plumbing for librtucker (no method arithmetic here).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>
#include <stdexcept>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: no-ops unless a profiler is attached

#include "../../include/rtucker.h"

namespace rt {

constexpr int kMaxModes = RTUCKER_MAX_MODES;

// Error carried through the orchestrator as an exception and mapped to a status code
// at the C boundary.
struct Error : std::runtime_error {
  rtucker_status code;
  Error(rtucker_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define RT_REQUIRE(cond, msg)                                                          \
  do {                                                                                 \
    if (!(cond)) throw ::rt::Error(RTUCKER_EINVAL, std::string(msg));                  \
  } while (0)

#define RT_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      char b_[512];                                                                    \
      snprintf(b_, sizeof b_, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),  \
               __FILE__, __LINE__);                                                    \
      throw ::rt::Error(e_ == cudaErrorMemoryAllocation ? RTUCKER_ENOMEM : RTUCKER_ECUDA, \
                        b_);                                                           \
    }                                                                                  \
  } while (0)

// Experimental kernel variants and probes are selected by environment variables only in an
// experiments build (-DRTUCKER_EXPERIMENTS, e.g. RTUCKER_NVCC_EXTRA=-DRTUCKER_EXPERIMENTS);
// the shipped library ignores them and always runs the tested path.
#ifdef RTUCKER_EXPERIMENTS
#define RT_EXP_GETENV(name) getenv(name)
#else
#define RT_EXP_GETENV(name) ((const char *)nullptr)
#endif

struct Comm;  // comm.cpp

// Device status bits, set by kernels and reported at the next synchronisation point
// (rtucker_sync or any call that synchronises) as RTUCKER_ENUMERIC.
enum StatusBit : unsigned {
  ST_EIG_NOT_CONVERGED = 1u,   // a Jacobi eigensolve hit its sweep cap
  ST_SHARD_LAYOUT = 2u,        // the shards of a multi-rank call do not tile the last mode
  ST_SINGULAR_PQ = 4u,         // SP-STHOSVD: singular P^T Q (fewer than l independent rows)
  ST_BAD_INDEX = 8u,           // RTUCKER_DEBUG_CHECKS: a COO index out of range
};

// Phase timing (measurement only): CUDA events recorded on the context stream around
// each step of the path; resolved lazily by rtucker_phase_times().
enum Phase { PH_SKETCH = 0, PH_QR = 1, PH_BPASS = 2, PH_EIG = 3, PH_SHRINK = 4, PH_OTHER = 5, PH_COUNT = 6 };

struct PhaseEvent {
  int slot;  // phase * kMaxModes + position of the mode in the processing order
  cudaEvent_t a, b;
};

struct Ctx {
  // workspace and result allocations: the caller's hooks (e.g. torch's caching allocator)
  // when given, else a library-owned stream-ordered pool (the device's default pool is not
  // touched)
  rtucker_alloc_fn alloc_fn = nullptr;
  rtucker_free_fn free_fn = nullptr;
  void *alloc_user = nullptr;
  cudaMemPool_t pool = nullptr;
  unsigned *status = nullptr;       // device status word (StatusBit)
  // CUDA-graph mode of the fixed-rank calls (RTUCKER_GRAPH): while a call is captured, device
  // allocations come from a bump arena sized by a counting eager run, and frees are no-ops
  struct Arena {
    char *base = nullptr;
    size_t size = 0, off = 0, counted = 0;
    bool on = false, counting = false;
  } arena;
  bool capturing = false;
  void *graphs = nullptr;           // graph plan cache (rtucker.cu)
  cudaStream_t aux = nullptr;       // side stream for the small solves of R-HOSVD (overlap)
  bool deterministic = true;        // fixed-order reductions (RTUCKER_NONDETERMINISTIC clears)
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, nranks = 1;
  Comm *comm = nullptr;
  uint64_t launches = 0;
  int num_sms = 148;
  std::string last_error;
  bool profiling = false;
  bool loopback_sharding = false;  // debug: run the sharded path on one rank (full slab)
  std::vector<PhaseEvent> events;
  double phase_ms[PH_COUNT * kMaxModes] = {0};
  int64_t phase_n[PH_COUNT * kMaxModes] = {0};
  // stream-K hand-off flags (one per CTA of a persistent grid); a launch signals with its own
  // epoch value, so the flags never need resetting
  unsigned *sk_flags = nullptr;
  int sk_n = 0;
  unsigned sk_epoch = 0;
};

// RAII scope that records a start/stop event pair when profiling is on, and always an NVTX
// range ("sketch m2", ...) for timeline tools (nsys / ncu --nvtx); NVTX calls are no-ops
// without an attached tool.
inline const char *phase_name(int phase, int pos) {
  static const char *names[PH_COUNT][kMaxModes] = {
      {"sketch m1", "sketch m2", "sketch m3", "sketch m4", "sketch m5", "sketch m6", "sketch m7", "sketch m8"},
      {"qr m1", "qr m2", "qr m3", "qr m4", "qr m5", "qr m6", "qr m7", "qr m8"},
      {"bpass m1", "bpass m2", "bpass m3", "bpass m4", "bpass m5", "bpass m6", "bpass m7", "bpass m8"},
      {"eig m1", "eig m2", "eig m3", "eig m4", "eig m5", "eig m6", "eig m7", "eig m8"},
      {"shrink m1", "shrink m2", "shrink m3", "shrink m4", "shrink m5", "shrink m6", "shrink m7", "shrink m8"},
      {"other m1", "other m2", "other m3", "other m4", "other m5", "other m6", "other m7", "other m8"}};
  return names[phase][pos < 0 ? 0 : (pos < kMaxModes ? pos : kMaxModes - 1)];
}

struct PhaseScope {
  Ctx &c;
  PhaseEvent ev{};
  bool on, open = false, nvtx_open = false;
  int pos;
  PhaseScope(Ctx &ctx, int phase, int position) : c(ctx), on(ctx.profiling), pos(position) { start(phase); }
  void start(int phase) {
    nvtxRangePushA(phase_name(phase, pos));
    nvtx_open = true;
    if (!on) return;
    ev.slot = phase * kMaxModes + (pos < kMaxModes ? pos : kMaxModes - 1);
    cudaEventCreate(&ev.a);
    cudaEventCreate(&ev.b);
    cudaEventRecord(ev.a, c.stream);
    open = true;
  }
  void stop() {
    if (nvtx_open) {
      nvtxRangePop();
      nvtx_open = false;
    }
    if (!on || !open) return;
    cudaEventRecord(ev.b, c.stream);
    c.events.push_back(ev);
    open = false;
  }
  void next(int phase) {
    stop();
    start(phase);
  }
  ~PhaseScope() { stop(); }
};

// Stream-ordered device allocation on the context stream through the context's allocator.
inline void *dev_alloc(Ctx &c, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void *p = nullptr;
  const size_t aligned = (bytes + 255) & ~(size_t)255;
  if (c.arena.on) {
    if (c.arena.off + aligned > c.arena.size) throw Error(RTUCKER_ENOMEM, "graph arena exhausted");
    p = c.arena.base + c.arena.off;
    c.arena.off += aligned;
    return p;
  }
  if (c.arena.counting) c.arena.counted += aligned;
  if (c.alloc_fn) {
    p = c.alloc_fn(bytes, (void *)c.stream, c.alloc_user);
    if (!p) throw Error(RTUCKER_ENOMEM, "allocation hook returned NULL");
    return p;
  }
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, c.pool, c.stream);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    throw Error(e == cudaErrorMemoryAllocation ? RTUCKER_ENOMEM : RTUCKER_ECUDA,
                std::string("device allocation failed: ") + cudaGetErrorString(e));
  }
  return p;
}
inline void dev_free(Ctx &c, void *p) {
  if (!p) return;
  if (c.arena.base && (char *)p >= c.arena.base && (char *)p < c.arena.base + c.arena.size) return;
  if (c.free_fn) c.free_fn(p, (void *)c.stream, c.alloc_user);
  else cudaFreeAsync(p, c.stream);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size (host-side cache:
// the attribute call is not free and most kernels are launched with the same size every call).
void set_smem_attr(const void *func, size_t bytes);
template <typename F>
inline void smem_attr(F *func, size_t bytes) {
  set_smem_attr((const void *)func, bytes);
}

// Runs the enclosed work on another stream of the context (restores the main stream on exit).
struct OnStream {
  Ctx &c;
  cudaStream_t saved;
  OnStream(Ctx &ctx, cudaStream_t s) : c(ctx), saved(ctx.stream) { c.stream = s; }
  ~OnStream() { c.stream = saved; }
};
// Event recorded on `from`, waited on by `to` (fork / join; captured into graphs as edges).
inline void stream_dep(cudaStream_t from, cudaStream_t to) {
  cudaEvent_t e;
  RT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  RT_CUDA(cudaEventRecord(e, from));
  RT_CUDA(cudaStreamWaitEvent(to, e, 0));
  RT_CUDA(cudaEventDestroy(e));
}

// Count every library kernel launch (reported as gpu_launches by bench.py).
#define RT_LAUNCH(ctx, kern, grid, block, smem, ...)                                   \
  do {                                                                                 \
    kern<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);                      \
    (ctx).launches++;                                                                  \
    RT_CUDA(cudaGetLastError());                                                       \
  } while (0)

// Stream-ordered device buffer (cudaMallocAsync on the context stream).
template <typename T>
struct DevBuf {
  T *p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  Ctx *c = nullptr;
  DevBuf() = default;
  DevBuf(Ctx &ctx, size_t count) { alloc(ctx, count); }
  void alloc(Ctx &ctx, size_t count) {
    release();
    c = &ctx;
    s = ctx.stream;
    n = count;
    if (count) p = (T *)dev_alloc(ctx, count * sizeof(T));
  }
  void zero() {
    if (n) RT_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  T *release_ownership() {
    T *q = p;
    p = nullptr;
    n = 0;
    return q;
  }
  void release() {
    if (p) dev_free(*c, p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n), s(o.s), c(o.c) { o.p = nullptr; o.n = 0; }
  DevBuf &operator=(DevBuf &&o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; c = o.c; o.p = nullptr; o.n = 0; }
    return *this;
  }
};

inline int64_t prod(const int64_t *d, int n) {
  int64_t p = 1;
  for (int i = 0; i < n; ++i) p *= d[i];
  return p;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace rt
