// Adaptive randomized Tucker: Alg 5 adaptive R-STHOSVD and, with
// RTUCKER_ADAPT_HOSVD, Alg 4 adaptive R-HOSVD.  The range finder
// AdaptRangeFinder is cited, not given, by the paper; this follows DESIGN
// reading R8, block by block:
//   E = ||G||^2;  k = 0
//   loop: stop if E <= tau^2 or k >= cap;  bb = min(b, cap - k)
//         W = G_(n) Omega(:, k:k+bb)            (sketch kernel, global column index k)
//         W <- (I - Q Q^T) W, twice              (fp64 tensor-core GEMMs)
//         stop ("floor") if ||W|| <= floor ||X|| (block discarded)
//         Q_i = qr(W);  B_i = Q_i^T G_(n) (+ Gram);  E -= ||B_i||^2;  k += bb
//   truncation (default): eigenpairs of B B^T, r = min{r : ||G||^2 - sum_{i<=r} s_i^2 <= tau^2},
//   A = Q U(:, 1:r) (signs per R4b), G <- U(:, 1:r)^T B.  ADAPT_NO_TRUNCATE keeps A = Q, G = B.
// tau_n = eps_n ||X||_F with eps_n = eps / sqrt(d) or the caller's mode_tol.
//
// Host synchronisation: ONE per block.  The floor test and the residual update are decided
// together after B_i: Q_i and B_i are formed speculatively and dropped when the projected
// block was below the floor (the only wasted pass is the final one of a floored mode).  The
// Ozaki B-pass's column maxima are computed once per mode (G does not change inside a mode).
//
// Multi-GPU: the dense input is sharded along its last mode, which is processed
// last.  Modes n < d: the block sketch W and ||B_i||^2 are allreduced (W is I_n x b), QR and the
// projections run redundantly, B stays sharded, the truncation Gram is allreduced and the
// shrink is local.  Mode d: W's rows are local and complete (placed and summed like the
// fixed-rank path), B_i = Q_i^T G_(d) sums over the sharded index and is allreduced
// (b x prod_{k<d} r_k per block: the known bandwidth limit of SURVEY §8(e)), and the core
// ends up replicated.
#include <cmath>
#include <cstring>
#include <vector>

#include "comm.h"
#include "kernels_extra.h"
#include "orchestrate.h"

namespace rt {

namespace {

__global__ void trace_kernel(const double *__restrict__ A, int n, int64_t lda, double *__restrict__ out) {
  __shared__ double s[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += A[i + lda * i];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    *out = t;
  }
}

// W (m x b) -= Q (m x k) T (k x b), column-major, one thread per output element.
__global__ void sub_gemm_kernel(double *__restrict__ W, int64_t m, int b, const double *__restrict__ Q, int k,
                                const double *__restrict__ T) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * b; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    double s = 0.0;
    for (int t = 0; t < k; ++t) s += Q[i + m * t] * T[t + (int64_t)k * j];
    W[e] -= s;
  }
}

struct ModeOut {
  double *A = nullptr;  // I x r (owned by the result)
  int r = 0;            // realised rank
  int k = 0;            // columns drawn
  DevBuf<unsigned char> G;  // new core (L, r, R) in dtype `gt` (unless uncompressed)
  DT gt = DT::F64;
  bool replaced = false;
  bool rows_replicated = false;  // mode d of a sharded input: the new core is replicated
};

// scal[slot] = trace(gram) (||B_i||^2), slot+1 = ||W||^2 (from W), fetched together
__global__ void block_stats_kernel(const double *__restrict__ gram, int bb, const double *__restrict__ W,
                                   int64_t nw, double *__restrict__ out) {
  __shared__ double s[32];
  double v = 0.0, t = 0.0;
  for (int i = threadIdx.x; i < bb; i += blockDim.x) t += gram[i + (int64_t)bb * i];
  for (int64_t e = threadIdx.x; e < nw; e += blockDim.x) v = fma(W[e], W[e], v);
  for (int o = 16; o; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s[threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double w = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) w += s[k];
    out[0] = t;
    out[1] = w;
  }
}

template <typename T>
T fetch(Ctx &c, const T *dev) {
  T h;
  RT_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  return h;
}

struct Shard {
  bool on = false;        // input sharded along the last mode
  bool rows = false;      // this mode is the sharded last mode (local rows of G_(n))
  int64_t col_offset = 0; // global unfolding-column offset of the local slab (modes n < d)
  int64_t row_offset = 0; // shard offset along the last mode (rows of Q for mode d)
  int64_t I_glob = 0;     // global I_n
  bool rel_acc = false;   // fp64 data: relative-accuracy eigensolver (gram_eig)
};

// AdaptRangeFinder on the mode-n unfolding of G (local dims cur, global dims gcur), threshold
// tau2 = tau^2.
ModeOut adapt_mode(Ctx &c, const void *G, DT gt, const int64_t *cur, const int64_t *gcur, int d, int n, double tau2,
                   int block, uint64_t seed, double floor_abs, bool mul_f64, DT store, bool truncate, bool want_core,
                   double *gnorm2_dev, bool fp32_data, const Shard &sh) {
  const ModeView v = mode_view(cur, d, n);
  const int64_t I = gcur[n];  // global rows of W and Q
  ModeOut out;
  // ||G||^2 (fp64), summed over the ranks
  sumsq(c, G, gt, v.L * v.I * v.R, gnorm2_dev);
  if (sh.on) allreduce_sum_f64(c, gnorm2_dev, 1);
  const double gn2 = fetch(c, gnorm2_dev);
  if (!std::isfinite(gn2)) throw Error(RTUCKER_ENUMERIC, "adaptive: non-finite norm");
  int64_t others = 1;
  for (int k2 = 0; k2 < d; ++k2)
    if (k2 != n) others *= gcur[k2];
  const int cap = (int)std::min<int64_t>(I, others);  // column cap on the global dims (reading R8)
  // Ozaki column maxima of the fp32 input: once per mode (G is fixed inside the mode)
  DevBuf<uint32_t> colmax;
  if (gt == DT::F32 && !mul_f64 && store == DT::F64 && v.L == 1 && !sh.rows && ozaki_bpass_enabled()) {
    colmax.alloc(c, (size_t)v.R);
    column_maxima(c, (const float *)G, v, colmax.p);
  }
  DevBuf<double> Q(c, (size_t)I * cap);
  DevBuf<unsigned char> Bfull(c, (size_t)v.L * cap * v.R * dt_size(store));
  DevBuf<double> scal(c, 4), T(c, (size_t)cap * block);
  double E = gn2;
  int k = 0;
  while (true) {
    if (E <= tau2 || k >= cap) break;
    const int bb = std::min(block, cap - k);
    DevBuf<double> W(c, (size_t)I * bb + 1);
    {
      PhaseScope ps(c, PH_SKETCH, n);
      if (!sh.rows) {
        sketch_dense(c, G, gt, v, n, bb, k, seed, sh.col_offset, mul_f64, W.p, nullptr, fp32_data);
        if (sh.on) allreduce_sum_f64(c, W.p, (size_t)I * bb);
      } else {
        DevBuf<double> wl(c, (size_t)v.I * bb), cov(c, (size_t)I * (bb + 1));
        cov.zero();
        sketch_dense(c, G, gt, v, n, bb, k, seed, 0, mul_f64, wl.p, nullptr, fp32_data);
        place_rows(c, wl.p, v.I, bb, sh.row_offset, I, cov.p, cov.p + (size_t)I * bb);
        allreduce_sum_f64(c, cov.p, cov.n);
        check_cover(c, cov.p + (size_t)I * bb, I);
        RT_CUDA(cudaMemcpyAsync(W.p, cov.p, sizeof(double) * I * bb, cudaMemcpyDeviceToDevice, c.stream));
      }
    }
    PhaseScope ps(c, PH_QR, n);
    if (k > 0) {  // W <- (I - Q Q^T) W, twice (re-orthogonalisation)
      for (int rep = 0; rep < 2; ++rep) {
        gemm_f64(c, true, Q.p, I, W.p, I, T.p, k, k, bb, I);                 // T = Q^T W
        gemm_f64(c, false, Q.p, I, T.p, k, W.p, I, I, bb, k, 1.0, -1.0);     // W -= Q T
      }
    }
    double *Qi = Q.p + (size_t)I * k;
    householder_qr(c, W.p, I, bb, Qi);  // the basis of Q is the core basis with ADAPT_NO_TRUNCATE
    ps.next(PH_BPASS);
    // B_i = Q_i^T G_(n) written into rows k..k+bb of B (L, cap, R) via a strided copy
    DevBuf<double> gram(c, (size_t)bb * bb);
    DevBuf<unsigned char> Bi(c, (size_t)v.L * bb * v.R * dt_size(store));
    if (!sh.rows) {
      ttm_dense(c, G, gt, v, Qi, I, bb, Bi.p, store, mul_f64, gram.p, colmax.p);
      if (sh.on) allreduce_sum_f64(c, gram.p, (size_t)bb * bb);
    } else {
      ttm_dense(c, G, gt, v, Qi + sh.row_offset, I, bb, Bi.p, store, mul_f64, nullptr);
      allreduce_sum(c, Bi.p, (size_t)v.L * bb * v.R, store == DT::F64);  // sum over the sharded index
      mode_gram(c, Bi.p, store, ModeView{v.L, bb, v.R}, gram.p);
    }
    RT_CUDA(cudaMemcpy2DAsync((unsigned char *)Bfull.p + (size_t)v.L * k * dt_size(store),
                              (size_t)v.L * cap * dt_size(store), Bi.p, (size_t)v.L * bb * dt_size(store),
                              (size_t)v.L * bb * dt_size(store), v.R, cudaMemcpyDeviceToDevice, c.stream));
    RT_LAUNCH(c, block_stats_kernel, 1, 256, 0, gram.p, bb, W.p, (int64_t)I * bb, scal.p);
    double st[2];
    RT_CUDA(cudaMemcpyAsync(st, scal.p, sizeof st, cudaMemcpyDeviceToHost, c.stream));
    RT_CUDA(cudaStreamSynchronize(c.stream));
    // W was the PROJECTED block before its QR (householder_qr leaves W unchanged): the floor
    // test (range exhausted) discards this block and stops
    if (std::sqrt(st[1]) <= floor_abs) break;
    E -= st[0];  // E -= ||B_i||^2 (exact identity for orthonormal Q)
    k += bb;
  }
  out.k = k;
  // compact B to (L, k, R)
  DevBuf<unsigned char> B(c, (size_t)v.L * std::max(k, 1) * v.R * dt_size(store));
  if (k > 0)
    RT_CUDA(cudaMemcpy2DAsync(B.p, (size_t)v.L * k * dt_size(store), Bfull.p, (size_t)v.L * cap * dt_size(store),
                              (size_t)v.L * k * dt_size(store), v.R, cudaMemcpyDeviceToDevice, c.stream));
  Bfull.release();
  const ModeView vb{v.L, k, v.R};
  out.rows_replicated = sh.rows;
  if (!truncate || k == 0) {
    out.r = k;
    out.A = (double *)dev_alloc(c, sizeof(double) * I * std::max(k, 1));
    if (k > 0) RT_CUDA(cudaMemcpyAsync(out.A, Q.p, sizeof(double) * I * k, cudaMemcpyDeviceToDevice, c.stream));
    out.G = std::move(B);
    out.gt = store;
    out.replaced = true;
    return out;
  }
  // ---- truncation: eigenpairs of B B^T (thin SVD of B), r from the cumulative spectrum
  PhaseScope ps(c, PH_EIG, n);
  DevBuf<double> gram(c, (size_t)k * k), w(c, k), U(c, (size_t)k * k);
  if (store == DT::F64 && k > 64) gram_f64(c, (const double *)B.p, v.L, k, v.R, gram.p);  // tensor cores
  else mode_gram(c, B.p, store, vb, gram.p);
  if (sh.on && !sh.rows) allreduce_sum_f64(c, gram.p, (size_t)k * k);
  gram_eig(c, gram.p, k, w.p, U.p, nullptr, k, sh.rel_acc);  // r not known yet: the whole spectrum
  std::vector<double> hw(k);
  RT_CUDA(cudaMemcpyAsync(hw.data(), w.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  int r = k;
  double cum = 0.0;
  for (int i = 0; i < k; ++i) {
    cum += hw[i];
    if (gn2 - cum <= tau2) {
      r = i + 1;
      break;
    }
  }
  out.r = r;
  out.A = (double *)dev_alloc(c, sizeof(double) * I * r);
  gemm_small(c, false, Q.p, I, U.p, k, out.A, I, I, r, k);
  canonical_signs(c, out.A, I, r, U.p, k, k);
  if (want_core) {
    ps.next(PH_SHRINK);
    out.G.alloc(c, (size_t)v.L * r * v.R * dt_size(store));
    if (store == DT::F64 && r > 64) {  // G <- U_r^T B as GEMMs on the fp64 tensor cores
      if (v.L == 1)
        gemm_f64(c, true, U.p, k, (const double *)B.p, k, (double *)out.G.p, r, r, v.R, k);
      else  // per r-slab: G_r (L x r) = B_r (L x k) U_r (k x r)
        gemm_f64_batched(c, false, false, (const double *)B.p, v.L, v.L * k, U.p, k, 0, (double *)out.G.p, v.L,
                         v.L * r, v.L, r, k, v.R);
    } else {
      ttm_dense(c, B.p, store, vb, U.p, k, r, out.G.p, store, mul_f64 || store == DT::F64, nullptr);
    }
    out.gt = store;
    out.replaced = true;
  }
  return out;
}

}  // namespace

rtucker_result *run_adaptive(Ctx &c, const rtucker_dense_desc *X, double tol, int block, const double *mode_tol,
                             const int32_t *order, uint64_t seed, uint32_t flags) {
  DenseIn in;
  prepare_dense(c, X, in);
  RT_REQUIRE(tol > 0.0 && tol < 1.0, "tol must lie in (0, 1)");
  RT_REQUIRE(block >= 1, "block must be >= 1");
  const int d = in.d;
  std::vector<double> eps(d, tol / std::sqrt((double)d));
  if (mode_tol) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      RT_REQUIRE(mode_tol[k] >= 0.0, "mode_tol must be >= 0");
      eps[k] = mode_tol[k];
      s += mode_tol[k] * mode_tol[k];
    }
    RT_REQUIRE(std::fabs(s - tol * tol) <= 1e-12 * std::max(1.0, tol * tol), "sum mode_tol^2 must equal tol^2");
  }
  const bool hosvd = flags & RTUCKER_ADAPT_HOSVD;
  const bool truncate = !(flags & RTUCKER_ADAPT_NO_TRUNCATE);
  int32_t ord[kMaxModes];
  check_order(hosvd ? nullptr : order, d, ord, in.gdims, in.sharded);
  if (hosvd)
    for (int k = 0; k < d; ++k) ord[k] = k;
  RT_REQUIRE(!in.sharded || eps[d - 1] > 0.0, "a sharded last mode must be compressed (mode_tol[d-1] > 0)");
  // precision: fp64 data -> fp64; fp32 data -> FP64 / FAST per flag, AUTO = HYBRID (fp32
  // products on the fp32 input, fp64 B and intermediates)
  const uint32_t acc = flags & RTUCKER_ACCUM_MASK;
  const bool f64 = in.dt == DT::F64 || acc == RTUCKER_ACCUM_FP64;
  const DT store = (in.dt == DT::F64 || acc != RTUCKER_ACCUM_FAST) ? DT::F64 : DT::F32;
  ResultGuard rg{c, new_result(d)};
  rtucker_result *res = rg.r;
  for (int k = 0; k < d; ++k) {
    res->dims[k] = in.gdims[k];
    res->order[k] = ord[k];
  }
  res->seed = seed;
  res->flags = flags;
  DevBuf<double> scal(c, 4);
  sumsq(c, in.ptr, in.dt, prod(in.ldims, d), scal.p);
  if (in.sharded) allreduce_sum_f64(c, scal.p, 1);
  const double nx2 = fetch(c, scal.p);
  if (!std::isfinite(nx2)) throw Error(RTUCKER_ENUMERIC, "adaptive: non-finite ||X||");
  RT_REQUIRE(nx2 > 0.0, "adaptive: ||X|| = 0");
  res->norm_sq = nx2;
  const double nx = std::sqrt(nx2);
  // range-exhaustion floor (reading R8): 1e-13 ||X|| for fp64 data, 1e-6 ||X|| for fp32 data
  const double floor_abs = (in.dt == DT::F64 ? 1e-13 : 1e-6) * nx;

  int64_t cur[kMaxModes], gcur[kMaxModes];
  memcpy(cur, in.ldims, sizeof cur);
  memcpy(gcur, in.gdims, sizeof gcur);
  const void *G = in.ptr;
  DT gt = in.dt;
  bool g_sharded = in.sharded;  // the current core still holds only this rank's slab
  DevBuf<unsigned char> gown;
  for (int jj = 0; jj < d; ++jj) {
    const int n = ord[jj];
    res->order[jj] = n;
    if (eps[n] == 0.0) {  // mode not compressed: A = I (reading R8)
      double *A = (double *)dev_alloc(c, sizeof(double) * gcur[n] * gcur[n]);
      std::vector<double> eye((size_t)gcur[n] * gcur[n], 0.0);
      for (int64_t i = 0; i < gcur[n]; ++i) eye[i + gcur[n] * i] = 1.0;
      RT_CUDA(cudaMemcpyAsync(A, eye.data(), sizeof(double) * eye.size(), cudaMemcpyHostToDevice, c.stream));
      RT_CUDA(cudaStreamSynchronize(c.stream));
      res->factors[n] = A;
      res->ranks[n] = gcur[n];
      res->ell[n] = gcur[n];
      continue;
    }
    const double tau2 = (eps[n] * nx) * (eps[n] * nx);
    const void *src = hosvd ? in.ptr : G;
    const DT st = hosvd ? in.dt : gt;
    const int64_t *dims = hosvd ? in.ldims : cur;
    const int64_t *gdims = hosvd ? in.gdims : gcur;
    const bool mulf = f64 || st == DT::F64;
    Shard sh;
    sh.on = in.sharded;
    sh.rows = in.sharded && n == d - 1;
    sh.row_offset = in.offset;
    sh.col_offset = (in.sharded && n != d - 1) ? col_offset_for(in, dims, n) : 0;
    sh.rel_acc = in.dt == DT::F64;
    ModeOut mo = adapt_mode(c, src, st, dims, gdims, d, n, tau2, block, seed, floor_abs, mulf, store, truncate,
                            !hosvd, scal.p + 1, in.dt == DT::F32 && !f64, sh);
    res->factors[n] = mo.A;
    res->ranks[n] = mo.r;
    res->ell[n] = mo.k;
    if (!hosvd) {
      const double before = fetch(c, scal.p + 1);  // ||G_prev||^2 (global) computed in adapt_mode
      cur[n] = mo.r;
      gcur[n] = mo.r;
      gown = std::move(mo.G);
      G = gown.p;
      gt = mo.gt;
      if (mo.rows_replicated) g_sharded = false;
      sumsq(c, G, gt, prod(cur, d), scal.p + 2);
      if (g_sharded) allreduce_sum_f64(c, scal.p + 2, 1);
      res->mode_residual_sq[n] = before - fetch(c, scal.p + 2);
    }
  }
  if (hosvd) {  // G = X x_1 A_1^T ... x_d A_d^T (Alg 4 line 5); mode d of a sharded input: partial + allreduce
    PhaseScope ps(c, PH_SHRINK, 0);
    memcpy(cur, in.ldims, sizeof cur);
    DevBuf<unsigned char> g0, g1;
    const void *Gc = in.ptr;
    DT gc = in.dt;
    for (int n = 0; n < d; ++n) {
      const ModeView v = mode_view(cur, d, n);
      const int rr = (int)res->ranks[n];
      const bool last_sharded = in.sharded && n == d - 1;
      DevBuf<unsigned char> &dst = (Gc == g0.p) ? g1 : g0;
      const DT ot = last_sharded ? DT::F64 : store;
      dst.alloc(c, (size_t)v.L * rr * v.R * dt_size(ot));
      const double *An = (const double *)res->factors[n] + (last_sharded ? in.offset : 0);
      ttm_dense(c, Gc, gc, v, An, in.gdims[n], rr, dst.p, ot, f64 || gc == DT::F64 || ot == DT::F64, nullptr);
      if (last_sharded) allreduce_sum_f64(c, (double *)dst.p, (size_t)v.L * rr * v.R);
      Gc = dst.p;
      gc = ot;
      cur[n] = rr;
    }
    gown = std::move(Gc == g0.p ? g0 : g1);
    G = gown.p;
    gt = gc;
  }
  const int64_t ncore = prod(cur, d);
  res->core = dev_alloc(c, sizeof(double) * std::max<int64_t>(ncore, 1));
  convert(c, G, gt, res->core, DT::F64, ncore);
  finish_result(c, res, flags);
  check_status(c);  // synchronises
  return rg.release();
}

}  // namespace rt
