/*
 * rtucker.h — C ABI of the B200-native randomized Tucker hot path.
 *
 * The library computes Tucker approximations X ~ [G; A_1, ..., A_d] (§2.1,
 * P:37) with the randomized algorithms of the paper:
 *   rtucker_hosvd          R-HOSVD, Alg 2
 *   rtucker_sthosvd        R-STHOSVD, Alg 3
 *   rtucker_adaptive       adaptive R-STHOSVD, Alg 5 [Alg 4 with a flag]
 *   rtucker_sparse_sthosvd SP-STHOSVD on a COO tensor, Alg 6
 * Each mode's factor comes from the randomized range finder of Alg 1:
 * Y = X_(n) Omega_n, Y = QR, B = Q^T X_(n), thin SVD of B, A_n = Q U_B(:,1:r_n).
 *
 * Conventions:
 *  - Modes and all indices are 0-based.  A dense tensor is stored first-mode-fastest:
 *    element (i_1..i_d) at i_1 + I_1*(i_2 + I_2*(...)).  Matrices are column-major.
 *  - The mode-n unfolding X_(n) has column index c = sum_{k!=n} i_k prod_{m<k,m!=n} I_m
 *    (lower modes fastest; eq. (kron)).
 *  - Omega_n[c, k] is generated on the fly by Philox4x32-10 with key = seed
 *    and counter (k>>2, n | v<<8, c_lo, c_hi) followed by Box-Muller (DESIGN reading
 *    R3); it is never stored and never read from HBM.  The same seed therefore gives
 *    the same Omega for any GPU count or block split.
 *  - Ranks: l_n = r_n + p is clamped to min(I_n, prod_{k!=n} I_k) on the current dims
 *    (Alg 2/3 requirement P:160; DESIGN reading R5) unless RTUCKER_STRICT.
 *
 * Memory and ownership:
 *  - Input descriptors are BORROWED and never modified.  Device inputs must stay alive
 *    until the work enqueued on the context stream has completed; host inputs
 *    (memory = RTUCKER_HOST) are copied to the device inside the call.
 *  - Device workspace and device results are allocated stream-ordered on the context
 *    stream through the context's allocator: the caller's rtucker_alloc_fn/rtucker_free_fn
 *    hooks when given to rtucker_ctx_create (the Python binding routes them to torch's
 *    caching allocator), else a memory pool owned by the library (created per context;
 *    the device's default pool and its attributes are not touched).
 *  - Results are owned by the library and released with rtucker_result_free(), which
 *    synchronises the context stream (asynchronous copies into the result struct must land
 *    before it is recycled).  With RTUCKER_RESULT_HOST the core/factors are host (pinned)
 *    memory, else device memory.
 *  - Calls enqueue work on the context stream.  The fixed-rank calls (rtucker_hosvd,
 *    rtucker_sthosvd) on device results do NOT synchronise: the device buffers are valid in
 *    stream order, and the host fields norm_sq / mode_residual_sq are filled by asynchronous
 *    copies, valid only after rtucker_sync() (or any synchronising call).  Every call that
 *    returns host metadata (realised ranks of the adaptive variant, nnz of the sparse
 *    variant, any RTUCKER_RESULT_HOST result) synchronises the stream before returning.
 *
 * Multi-GPU (one context per rank, NCCL communicator of the library): every rank calls the
 * same function with identical scalar arguments.  Dense inputs must be SHARDED along the
 * last mode on every rank (shard_extent >= 1, so I_d >= nranks), the shards of all ranks
 * tiling [0, I_d) in rank order; the sparse variant takes each rank's own nonzeros (a
 * partition of the tensor's nonzeros).  Results are replicated on every rank.
 *
 * Errors: every call returns an rtucker_status; rtucker_last_error() gives a message.
 *  Kernel-side conditions (a Jacobi eigensolve that did not converge within its sweep cap,
 *  shards that do not tile the last mode) are recorded in a device status word and
 *  returned as RTUCKER_ENUMERIC / RTUCKER_EINVAL by the next synchronising call.
 *  RTUCKER_EINVAL       invalid argument (d<1, dim<1, r_n not in [1, I_n], p<0, tol not in
 *                       (0,1), block<1, order not a permutation, eta<1, strict-cap
 *                       violation, SP cap r_n+p >= min(I_n, prod others), ...)
 *  RTUCKER_EUNSUPPORTED d > RTUCKER_MAX_MODES or a size this build does not handle
 *  RTUCKER_ENUMERIC     non-finite norm, singular P^T Q in SP-STHOSVD
 *  RTUCKER_ECUDA / RTUCKER_ENCCL / RTUCKER_ENOMEM   runtime failures
 */
#ifndef RTUCKER_H_
#define RTUCKER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTUCKER_MAX_MODES 8

typedef enum {
  RTUCKER_OK = 0,
  RTUCKER_EINVAL = 1,
  RTUCKER_ENOMEM = 2,
  RTUCKER_ENUMERIC = 3,
  RTUCKER_ECUDA = 4,
  RTUCKER_ENCCL = 5,
  RTUCKER_EUNSUPPORTED = 6
} rtucker_status;

typedef enum { RTUCKER_F32 = 0, RTUCKER_F64 = 1 } rtucker_dtype;
typedef enum { RTUCKER_DEVICE = 0, RTUCKER_HOST = 1 } rtucker_memory;

/* Flags (bitmask). */
#define RTUCKER_STRICT            (1u << 0)  /* error instead of clamping l_n */
/* Precision policy for fp32 data (fp64 data always computes in fp64).  Every policy
 * accumulates sums in fp64 (fp32 partial products are flushed into fp64 accumulators
 * every few dozen terms); norms, Grams, QR and eigensolves are fp64 throughout.
 *   AUTO    FP64 when max_n l_n <= 12, else HYBRID
 *   FP64    fp64 products; B and every shrunk intermediate stored in fp64
 *   FAST    fp32 (or 3xTF32 tensor-core) products; B and intermediates stored in fp32
 *   HYBRID  FAST products on the fp32 input, B and intermediates stored in fp64 (later
 *           passes therefore run in fp64) */
#define RTUCKER_ACCUM_AUTO        (0u << 1)
#define RTUCKER_ACCUM_FP64        (1u << 1)
#define RTUCKER_ACCUM_FAST        (2u << 1)
#define RTUCKER_ACCUM_HYBRID      (3u << 1)
#define RTUCKER_ACCUM_MASK        (3u << 1)
#define RTUCKER_ADAPT_NO_TRUNCATE (1u << 3)  /* adaptive: keep the block basis (no post-truncation) */
#define RTUCKER_ADAPT_HOSVD       (1u << 4)  /* adaptive: Alg 4 (modes independent) instead of Alg 5 */
#define RTUCKER_RESULT_HOST       (1u << 5)  /* copy core/factors to host memory */
#define RTUCKER_NO_CORE           (1u << 6)  /* R-HOSVD: factors only */
/* Determinism: every path uses fixed-order reductions and no floating-point
 * atomics, so reruns with the same inputs and GPU count are bit-identical.  The flag is
 * the default behaviour and is accepted for clarity. */
#define RTUCKER_DETERMINISTIC     (1u << 7)
/* Debug checks: index-range and finite-value checks of the inputs, and a stream
 * synchronisation with error check after every step (slow; for debugging). */
#define RTUCKER_DEBUG_CHECKS      (1u << 8)
/* rtucker_sparse_sthosvd: SP-HOSVD instead of SP-STHOSVD (the paper's first variant):
 * every mode is sketched and selected on X itself, and the core is X x_1 P_1^T ... x_d P_d^T,
 * one filter by all selections (order is ignored; nnz_history = [nnz(X), nnz(core)]). */
#define RTUCKER_SP_HOSVD          (1u << 9)
/* Fixed-rank calls (rtucker_hosvd / rtucker_sthosvd, device result): replay the whole call as one
 * CUDA graph.  The first call with a given (input pointer, shape, ranks, p, seed, order, flags)
 * runs eagerly, sizes a workspace arena and captures the call; later identical calls launch the
 * graph and copy core, factors and residuals into a fresh result (host enqueue ~ one graph launch
 * plus a few copies).  The context keeps the arena and the graph until it is destroyed.
 * Ignored with RTUCKER_RESULT_HOST or while phase profiling is on. */
#define RTUCKER_GRAPH             (1u << 10)
/* Randomized subspace iteration (the paper's remedy for slowly decaying spectra, P:550-553;
 * NEXT-3): RTUCKER_POWER(q), q = 0..15, adds q steps Z = orth(X_(n)^T Q), Q = orth(X_(n) Z)
 * after each range finder's QR in rtucker_hosvd / rtucker_sthosvd (unsharded inputs; two extra
 * passes over the mode's tensor per step). */
#define RTUCKER_POWER(q)          (((uint32_t)(q) & 15u) << 12)
#define RTUCKER_POWER_MASK        (15u << 12)
/* Deterministic comparators (NEXT-4; the paper's baselines of Table 6.2): with this
 * flag rtucker_hosvd / rtucker_sthosvd compute the deterministic HOSVD / STHOSVD
 * (P:74-92): the leading r_n eigenvectors of the full unfolding's Gram G_(n) G_(n)^T instead of
 * a sketch (p and seed are ignored; single GPU; fp64 products and intermediates). */
#define RTUCKER_EXACT_SVD         (1u << 16)

/* Dense tensor, first-mode-fastest.  When the tensor is sharded across ranks along its
 * LAST mode, dims[] are the GLOBAL dims and this rank holds the contiguous slab of
 * shard_extent last-mode indices starting at shard_offset; shard_extent = 0 means
 * unsharded. */
typedef struct {
  rtucker_dtype dtype;
  int32_t d;
  int64_t dims[RTUCKER_MAX_MODES];
  int64_t shard_offset, shard_extent;
  rtucker_memory memory;
  const void *data;
} rtucker_dense_desc;

/* Sparse COO tensor, structure of arrays, 0-based int32 indices, duplicates merged
 * (SPEC D3 / DESIGN §2).  nnz is the local count (nnz-partitioned across ranks). */
typedef struct {
  rtucker_dtype dtype;
  int32_t d;
  int64_t dims[RTUCKER_MAX_MODES];
  int64_t nnz;
  rtucker_memory memory;
  const int32_t *idx[RTUCKER_MAX_MODES];
  const void *vals;
} rtucker_coo_desc;

typedef struct rtucker_ctx rtucker_ctx; /* one per GPU / rank; not thread-safe */

/* Allocation hooks: alloc returns `bytes` of device memory usable in stream order on
 * `stream` (a cudaStream_t), or NULL on failure (-> RTUCKER_ENOMEM); free releases it in
 * stream order.  `user` is passed through. */
typedef void *(*rtucker_alloc_fn)(size_t bytes, void *stream, void *user);
typedef void (*rtucker_free_fn)(void *ptr, void *stream, void *user);

/* Result of a decomposition.  core / factors are fp64 (dtype field) for dense
 * algorithms; the SP core keeps the input value dtype (values copied exactly). */
typedef struct {
  int32_t d;
  int64_t dims[RTUCKER_MAX_MODES];   /* input dims */
  int64_t ranks[RTUCKER_MAX_MODES];  /* realised r_n (core dims; l_n for SP) */
  int64_t ell[RTUCKER_MAX_MODES];    /* sketch width used per mode (adaptive: columns drawn) */
  int32_t order[RTUCKER_MAX_MODES];  /* processing order used */
  uint64_t seed;
  uint32_t flags;
  rtucker_dtype dtype;               /* dtype of core/factors */
  rtucker_memory memory;             /* where core/factors live */
  void *core;                        /* dense r_1 x .. x r_d, first-mode-fastest */
  void *factors[RTUCKER_MAX_MODES];  /* A_n: dims[n] x ranks[n], column-major */
  double mode_residual_sq[RTUCKER_MAX_MODES]; /* ||G_prev||^2 - ||G_next||^2 per mode (host) */
  double norm_sq;                    /* ||X||_F^2 (host) */
  /* sparse results */
  int64_t core_nnz;
  int32_t *core_idx[RTUCKER_MAX_MODES]; /* (memory as above) 0-based in the core dims */
  void *core_vals;                      /* input value dtype */
  int64_t *selection[RTUCKER_MAX_MODES];/* sorted original indices S_n, length ranks[n] */
  int64_t nnz_history[RTUCKER_MAX_MODES + 1];
  int32_t swaps[RTUCKER_MAX_MODES];
  void *internal;                    /* library bookkeeping */
} rtucker_result;

/* Context.  device: CUDA ordinal.  cuda_stream: cudaStream_t to enqueue on (NULL =
 * a library-created stream).  nccl_unique_id: NULL for single-GPU, else the 128-byte
 * ncclUniqueId shared by all ranks (NCCL is loaded at run time).  alloc_fn / free_fn:
 * allocation hooks (both NULL = library-owned pool; both or neither must be given). */
rtucker_status rtucker_ctx_create(int device, void *cuda_stream, const void *nccl_unique_id,
                                  int rank, int nranks, rtucker_alloc_fn alloc_fn,
                                  rtucker_free_fn free_fn, void *alloc_user, rtucker_ctx **out);
void rtucker_ctx_destroy(rtucker_ctx *ctx);
rtucker_status rtucker_ctx_set_stream(rtucker_ctx *ctx, void *cuda_stream);
const char *rtucker_last_error(const rtucker_ctx *ctx);
/* Number of library kernels launched on this context since creation. */
uint64_t rtucker_launch_count(const rtucker_ctx *ctx);
/* Writes a fresh ncclUniqueId (128 bytes) for rank 0 to broadcast. */
rtucker_status rtucker_nccl_unique_id(void *out128);
const char *rtucker_version(void);

/* R-HOSVD, Alg 2.  ranks: d target ranks r_n; p >= 0 oversampling. */
rtucker_status rtucker_hosvd(rtucker_ctx *ctx, const rtucker_dense_desc *X, const int64_t *ranks,
                             int32_t p, uint64_t seed, uint32_t flags, rtucker_result **out);

/* R-STHOSVD, Alg 3.  order: permutation of 0..d-1 or NULL = decreasing
 * dims, ties by index.  Sharded inputs need order[d-1] == d-1. */
rtucker_status rtucker_sthosvd(rtucker_ctx *ctx, const rtucker_dense_desc *X, const int64_t *ranks,
                               int32_t p, uint64_t seed, const int32_t *order, uint32_t flags,
                               rtucker_result **out);

/* Adaptive R-STHOSVD, Alg 5, AdaptRangeFinder per DESIGN reading R8.
 * tol in (0,1); block >= 1; mode_tol: NULL = tol/sqrt(d) each, else d values
 * with sum eps_n^2 = tol^2 (eps_n = 0: mode not compressed).  Synchronises the stream. */
rtucker_status rtucker_adaptive(rtucker_ctx *ctx, const rtucker_dense_desc *X, double tol,
                                int32_t block, const double *mode_tol, const int32_t *order,
                                uint64_t seed, uint32_t flags, rtucker_result **out);

/* SP-STHOSVD, Alg 6.  Strict cap r_n + p < min(I_n, prod others);
 * eta >= 1 (2.0 in the paper).  Synchronises the stream. */
rtucker_status rtucker_sparse_sthosvd(rtucker_ctx *ctx, const rtucker_coo_desc *X,
                                      const int64_t *ranks, int32_t p, uint64_t seed,
                                      const int32_t *order, double eta, uint32_t flags,
                                      rtucker_result **out);

void rtucker_result_free(rtucker_ctx *ctx, rtucker_result *res);

/* Stream-ordered copy on the context stream (plumbing for bindings): kind as in
 * cudaMemcpyKind (0 H2H, 1 H2D, 2 D2H, 3 D2D, 4 default). */
rtucker_status rtucker_memcpy(rtucker_ctx *ctx, void *dst, const void *src, size_t bytes, int kind);
/* Blocks until all work enqueued on the context stream has completed; then reports (and
 * clears) the device status word: RTUCKER_ENUMERIC for a non-converged eigensolve,
 * RTUCKER_EINVAL for a shard layout that does not tile the last mode. */
rtucker_status rtucker_sync(rtucker_ctx *ctx);

/* Phase timing for measurement: when enabled, CUDA events are recorded on the context
 * stream around every step (0 sketch, 1 QR, 2 B-pass, 3 eig, 4 shrink/core, 5 other),
 * per position of the mode in the processing order.  rtucker_phase_times synchronises,
 * accumulates and returns ms[6*8] and counts[6*8] (slot = phase*8 + position); reset
 * clears them. */
rtucker_status rtucker_set_profiling(rtucker_ctx *ctx, int enabled);
rtucker_status rtucker_phase_times(rtucker_ctx *ctx, double *ms, int64_t *counts, int reset);

/* ---- measurement / debug exports (not part of the method) ---------------------- */

/* Single-rank loopback of the sharded dense path: with enabled != 0, a descriptor whose
 * shard covers the whole last mode (shard_offset 0, shard_extent = dims[d-1]) runs the
 * multi-rank code path (global column offsets, row-block gather of the last mode, B_d
 * reduction) with the collectives degenerating to local copies.  nranks must be 1. */
rtucker_status rtucker_debug_loopback_sharding(rtucker_ctx *ctx, int enabled);

/* ||X - X_hat||_F / ||X||_F for a dense result, computed on the device. */
rtucker_status rtucker_rel_error(rtucker_ctx *ctx, const rtucker_dense_desc *X,
                                 const rtucker_result *res, double *out);

/* Y = X_(mode) Omega_mode(:, k0:k0+ell) (Alg 1 line 1), fp64 I_mode x ell column-major,
 * written to Y_out (DEVICE pointer).  flags select the accumulation policy. */
rtucker_status rtucker_debug_sketch(rtucker_ctx *ctx, const rtucker_dense_desc *X, int32_t mode,
                                    int32_t ell, int64_t k0, uint64_t seed, uint32_t flags,
                                    double *Y_out);

/* B = A^T X_(mode) stored (L, J, R) in fp64 (out, DEVICE, may be NULL) and/or its Gram
 * B_(mode) B_(mode)^T (gram, J x J, DEVICE, may be NULL); A is I_mode x J fp64 column-major
 * (DEVICE).  The B-pass of Alg 1 line 3 with fp64 storage (HYBRID / FP64 products per
 * flags). */
rtucker_status rtucker_debug_ttm(rtucker_ctx *ctx, const rtucker_dense_desc *X, int32_t mode, const double *A,
                                 int32_t J, uint32_t flags, double *out, double *gram);

/* Omega rows: out[i + n*k] = Omega_mode[cols[i], k0 + k] for i < n, k < ell in `dtype`
 * precision (DEVICE pointers; cols int64). */
rtucker_status rtucker_debug_omega(rtucker_ctx *ctx, rtucker_dtype dtype, uint64_t seed,
                                   int32_t mode, const int64_t *cols, int64_t n, int32_t ell,
                                   int64_t k0, void *out);

/* Raw Philox4x32-10 words: out[4i..4i+3] = Philox(ctr[4i..4i+3], key) (DEVICE pointers). */
rtucker_status rtucker_debug_philox(rtucker_ctx *ctx, const uint32_t *ctr, int64_t n,
                                    uint32_t key0, uint32_t key1, uint32_t *out);

/* Householder thin QR of an m x n fp64 column-major matrix: Q (m x n) (DEVICE). */
rtucker_status rtucker_debug_qr(rtucker_ctx *ctx, int64_t m, int32_t n, const double *Y, double *Q);

/* Symmetric eigendecomposition of an n x n fp64 matrix: eigenvalues descending in w,
 * eigenvectors in V (column-major) (DEVICE). */
rtucker_status rtucker_debug_eig(rtucker_ctx *ctx, int32_t n, const double *A, double *w, double *V,
                                 int32_t *sweeps_out /* host, may be NULL */);

/* Eigenpairs of a symmetric positive semidefinite Gram (the hot-path eigensolver): pivoted
 * Cholesky + one-sided Jacobi on the factor.  Eigenvalues descending in w; eigenvectors in V
 * accurate to ~eps * sqrt(w_0 / w_k) (DEVICE pointers). */
rtucker_status rtucker_debug_gram_eig(rtucker_ctx *ctx, int32_t n, const double *A, double *w, double *V,
                                      int32_t *sweeps_out /* host, may be NULL */);

/* The same eigensolver as the hot path selects it for a Gram of fp32 data (rel_acc = 0) or fp64
 * data (rel_acc = 1), the wanted rank r_need deciding its fallback (Alg 1 line 4).  For
 * rel_acc = 0 and 32 < n <= 64 this is the mixed-precision solver (fp32 Jacobi on the pivoted
 * Cholesky factor, then fp64 Newton refinement on the tensor cores), eigenvectors to
 * ~eps w_0 / gap; *sweeps_out = fp32 sweeps + 1000 x refinement steps, or the fp64 Jacobi's
 * sweep count when the fallback ran (DEVICE pointers; EINVAL for n < 1 or r_need < 1). */
rtucker_status rtucker_debug_gram_eig_ex(rtucker_ctx *ctx, int32_t n, const double *A, double *w, double *V,
                                         int32_t *sweeps_out /* host, may be NULL */, int32_t rel_acc,
                                         int32_t r_need);

/* C (m x n) = op(A) op(B), fp64 column-major on the tensor cores (the library's GEMM for the
 * adaptive truncation and the eigensolver), DEVICE pointers; trans* != 0 transposes. */
rtucker_status rtucker_debug_gemm(rtucker_ctx *ctx, int transA, int transB, int64_t m, int64_t n, int64_t k,
                                  const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc);

/* Gram C (K x K) = B_(n) B_(n)^T of an fp64 tensor stored (L, K, R) (DEVICE pointers). */
rtucker_status rtucker_debug_gram(rtucker_ctx *ctx, int64_t L, int64_t K, int64_t R, const double *B, double *C);

/* Sparse sketch Y = X_(mode) Omega_mode(:, 0:ell) of a COO tensor (Alg 6 line 4), summed
 * in fixed point over the nonzeros (DESIGN reading R20), fp64 I_mode x ell column-major, written
 * to Y_out (DEVICE).  flags: RTUCKER_ACCUM_FP64 draws fp64 normals for fp32 values (fp64
 * values always use fp64 normals).  ell <= 64. */
rtucker_status rtucker_debug_coo_sketch(rtucker_ctx *ctx, const rtucker_coo_desc *X, int32_t mode, int32_t ell,
                                        uint64_t seed, uint32_t flags, double *Y_out);

/* Strong-RRQR row selection (DESIGN reading R9) of an m x l orthonormal fp64 Q:
 * sel (l, sorted ascending, DEVICE int64) and A = Q Q[sel,:]^{-1} (m x l, DEVICE). */
rtucker_status rtucker_debug_srrqr(rtucker_ctx *ctx, int64_t m, int32_t l, const double *Q,
                                   double eta, int64_t *sel, double *A, int32_t *swaps_out);

#ifdef __cplusplus
}
#endif
#endif /* RTUCKER_H_ */
