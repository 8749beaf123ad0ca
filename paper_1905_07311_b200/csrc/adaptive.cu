// Adaptive randomized Tucker: Alg 5 adaptive R-STHOSVD and, with
// RTUCKER_ADAPT_HOSVD, Alg 4 adaptive R-HOSVD.  The range finder
// AdaptRangeFinder is cited, not given, by the paper; this follows DESIGN
// reading R8, block by block:
//   E = ||G||^2;  k = 0
//   loop: stop if E <= tau^2 or k >= cap;  bb = min(b, cap - k)
//         W = G_(n) Omega(:, k:k+bb)            (sketch kernel, global column index k)
//         W <- (I - Q Q^T) W, twice              (small fp64 GEMMs)
//         stop ("floor") if ||W|| <= floor ||X|| (block discarded)
//         Q_i = qr(W);  B_i = Q_i^T G_(n) (+ Gram);  E -= ||B_i||^2;  k += bb
//   truncation (default): eigenpairs of B B^T, r = min{r : ||G||^2 - sum_{i<=r} s_i^2 <= tau^2},
//   A = Q U(:, 1:r) (signs per R4b), G <- U(:, 1:r)^T B.  ADAPT_NO_TRUNCATE keeps A = Q, G = B.
// tau_n = eps_n ||X||_F with eps_n = eps / sqrt(d) or the caller's mode_tol.
// The stop decisions are data dependent, so every block synchronises the stream.
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
};

template <typename T>
T fetch(Ctx &c, const T *dev) {
  T h;
  RT_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  return h;
}

// AdaptRangeFinder on the mode-n unfolding of G (dims cur), threshold tau2 = tau^2.
ModeOut adapt_mode(Ctx &c, const void *G, DT gt, const int64_t *cur, int d, int n, double tau2, int block,
                   uint64_t seed, double floor_abs, bool mul_f64, DT store, bool truncate, bool want_core,
                   double *gnorm2_dev, bool fp32_data) {
  const ModeView v = mode_view(cur, d, n);
  const int64_t I = v.I;
  int64_t others = v.L * v.R;
  const int cap = (int)std::min<int64_t>(I, others);
  ModeOut out;
  // ||G||^2 (fp64)
  sumsq(c, G, gt, v.L * v.I * v.R, gnorm2_dev);
  const double gn2 = fetch(c, gnorm2_dev);
  if (!std::isfinite(gn2)) throw Error(RTUCKER_ENUMERIC, "adaptive: non-finite norm");
  DevBuf<double> Q(c, (size_t)I * cap);
  DevBuf<unsigned char> Bfull(c, (size_t)v.L * cap * v.R * dt_size(store));
  DevBuf<double> scal(c, 4);
  double E = gn2;
  int k = 0;
  while (true) {
    if (E <= tau2 || k >= cap) break;
    const int bb = std::min(block, cap - k);
    DevBuf<double> W(c, (size_t)I * bb);
    {
      PhaseScope ps(c, PH_SKETCH, n);
      sketch_dense(c, G, gt, v, n, bb, k, seed, 0, mul_f64, W.p, nullptr, fp32_data);
    }
    PhaseScope ps(c, PH_QR, n);
    if (k > 0) {  // W <- (I - Q Q^T) W, twice (re-orthogonalisation)
      DevBuf<double> T(c, (size_t)k * bb);
      for (int rep = 0; rep < 2; ++rep) {
        gemm_small(c, true, Q.p, I, W.p, I, T.p, k, k, bb, I);
        RT_LAUNCH(c, sub_gemm_kernel, std::max(1, std::min(1024, ceil_div(I * bb, 256))), 256, 0, W.p, I, bb, Q.p, k,
                  T.p);
      }
    }
    sumsq(c, W.p, DT::F64, I * bb, scal.p);
    const double wn = std::sqrt(fetch(c, scal.p));
    if (wn <= floor_abs) break;  // range exhausted: the block is discarded
    householder_qr(c, W.p, I, bb, Q.p + (size_t)I * k);  // the basis of Q is the core basis with ADAPT_NO_TRUNCATE
    ps.next(PH_BPASS);
    // B_i = Q_i^T G_(n) written into rows k..k+bb of B (L, cap, R) via a strided TTM
    DevBuf<double> gram(c, (size_t)bb * bb);
    DevBuf<unsigned char> Bi(c, (size_t)v.L * bb * v.R * dt_size(store));
    ttm_dense(c, G, gt, v, Q.p + (size_t)I * k, I, bb, Bi.p, store, mul_f64, gram.p);
    RT_CUDA(cudaMemcpy2DAsync((unsigned char *)Bfull.p + (size_t)v.L * k * dt_size(store),
                              (size_t)v.L * cap * dt_size(store), Bi.p, (size_t)v.L * bb * dt_size(store),
                              (size_t)v.L * bb * dt_size(store), v.R, cudaMemcpyDeviceToDevice, c.stream));
    RT_LAUNCH(c, trace_kernel, 1, 256, 0, gram.p, bb, bb, scal.p + 1);
    E -= fetch(c, scal.p + 1);  // E -= ||B_i||^2 (exact identity for orthonormal Q)
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
  mode_gram(c, B.p, store, vb, gram.p);
  sym_eig(c, gram.p, k, w.p, U.p);  // r not known yet: accurate tail needed
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
    ttm_dense(c, B.p, store, vb, U.p, k, r, out.G.p, store, mul_f64 || store == DT::F64, nullptr);
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
  if (in.sharded) throw Error(RTUCKER_EUNSUPPORTED, "rtucker_adaptive: sharded inputs are not supported yet");
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
  check_order(hosvd ? nullptr : order, d, ord, in.gdims, false);
  if (hosvd)
    for (int k = 0; k < d; ++k) ord[k] = k;
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
  const int64_t N = prod(in.gdims, d);
  sumsq(c, in.ptr, in.dt, N, scal.p);
  const double nx2 = fetch(c, scal.p);
  if (!std::isfinite(nx2)) throw Error(RTUCKER_ENUMERIC, "adaptive: non-finite ||X||");
  RT_REQUIRE(nx2 > 0.0, "adaptive: ||X|| = 0");
  res->norm_sq = nx2;
  const double nx = std::sqrt(nx2);
  // range-exhaustion floor (reading R8): 1e-13 ||X|| for fp64 data, 1e-6 ||X|| for fp32 data
  const double floor_abs = (in.dt == DT::F64 ? 1e-13 : 1e-6) * nx;

  int64_t cur[kMaxModes];
  memcpy(cur, in.gdims, sizeof cur);
  const void *G = in.ptr;
  DT gt = in.dt;
  DevBuf<unsigned char> gown;
  for (int jj = 0; jj < d; ++jj) {
    const int n = ord[jj];
    res->order[jj] = n;
    if (eps[n] == 0.0) {  // mode not compressed: A = I (reading R8)
      double *A = nullptr;
      A = (double *)dev_alloc(c, sizeof(double) * cur[n] * cur[n]);
      std::vector<double> eye((size_t)cur[n] * cur[n], 0.0);
      for (int64_t i = 0; i < cur[n]; ++i) eye[i + cur[n] * i] = 1.0;
      RT_CUDA(cudaMemcpyAsync(A, eye.data(), sizeof(double) * eye.size(), cudaMemcpyHostToDevice, c.stream));
      RT_CUDA(cudaStreamSynchronize(c.stream));
      res->factors[n] = A;
      res->ranks[n] = cur[n];
      res->ell[n] = cur[n];
      continue;
    }
    const double tau2 = (eps[n] * nx) * (eps[n] * nx);
    const void *src = hosvd ? in.ptr : G;
    const DT st = hosvd ? in.dt : gt;
    const int64_t *dims = hosvd ? in.gdims : cur;
    const bool mulf = f64 || st == DT::F64;
    ModeOut mo = adapt_mode(c, src, st, dims, d, n, tau2, block, seed, floor_abs, mulf, store, truncate, !hosvd,
                            scal.p + 1, in.dt == DT::F32 && !f64);
    res->factors[n] = mo.A;
    res->ranks[n] = mo.r;
    res->ell[n] = mo.k;
    if (!hosvd) {
      const double before = fetch(c, scal.p + 1);  // ||G_prev||^2 computed in adapt_mode
      cur[n] = mo.r;
      gown = std::move(mo.G);
      G = gown.p;
      gt = mo.gt;
      sumsq(c, G, gt, prod(cur, d), scal.p + 2);
      res->mode_residual_sq[n] = before - fetch(c, scal.p + 2);
    }
  }
  if (hosvd) {  // G = X x_1 A_1^T ... x_d A_d^T (Alg 4 line 5)
    PhaseScope ps(c, PH_SHRINK, 0);
    memcpy(cur, in.gdims, sizeof cur);
    DevBuf<unsigned char> g0, g1;
    const void *Gc = in.ptr;
    DT gc = in.dt;
    for (int n = 0; n < d; ++n) {
      const ModeView v = mode_view(cur, d, n);
      const int rr = (int)res->ranks[n];
      DevBuf<unsigned char> &dst = (Gc == g0.p) ? g1 : g0;
      dst.alloc(c, (size_t)v.L * rr * v.R * dt_size(store));
      ttm_dense(c, Gc, gc, v, (const double *)res->factors[n], in.gdims[n], rr, dst.p, store,
                f64 || gc == DT::F64 || store == DT::F64, nullptr);
      Gc = dst.p;
      gc = store;
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
  RT_CUDA(cudaStreamSynchronize(c.stream));
  return rg.release();
}

}  // namespace rt
