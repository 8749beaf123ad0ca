// Latency-critical small dense linear algebra (fp64) of the range finder.
//
//  householder_qr   thin QR of the sketch Y (I_n x l) (Alg 1 line 2), explicit Q.
//                   Householder (not CholeskyQR) because the sketches are numerically
//                   rank-deficient (SURVEY §7 hard part 2).  The rows are spread over a
//                   thread-block cluster (1..16 CTAs), each CTA keeping its row slab of W
//                   and Q in shared memory.  One cluster barrier per column: the norm of the
//                   pivot column x_j and all dots x_j^T w_c are reduced in the same exchange
//                   (DSMEM, fixed-order butterfly so every CTA derives the identical
//                   reflector), and v^T w_c = x_j^T w_c + (v_0 - alpha) w_c[j] follows.
//  sym_eig          eigenpairs of the l x l Gram B B^T (thin SVD of B, Alg 1 line 4)
//                   by one-sided (Hestenes) Jacobi on the Gram itself: each warp owns one
//                   column pair of the round-robin ordering, so a round needs a single CTA
//                   barrier.  Relative stopping test |g_pq| <= tol sqrt(g_pp g_qq).
//  canonical_signs  the sign convention of DESIGN reading R4b.
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace rt {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ cluster QR ------
// (nvcc 12.9 note: an earlier form of the local row index, (int)(j - r0) with int64 r0,
// was mis-evaluated in the second loop on sm_100a; all row arithmetic below is int.)
constexpr int kQRT = 512;  // threads per CTA
constexpr int kNW = kQRT / 32;
constexpr int kMaxN = 64;  // columns handled by the cluster kernel

// Sum over the cluster of slot `idx` of the message buffers: lane k reads CTA k's value,
// then a butterfly (identical order in every warp of every CTA => identical results).
__device__ __forceinline__ double cluster_sum(cg::cluster_group &cl, double *buf, int idx, int ncta, int lane) {
  double v = 0.0;
  for (int k = lane; k < ncta; k += 32) v += cl.map_shared_rank(buf, k)[idx];
  return warp_sum(v);
}

__global__ void __launch_bounds__(kQRT) qr_cluster_kernel(const double *__restrict__ Y, int64_t m, int n,
                                                          int rows, double *__restrict__ Q) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int ncta = (int)cl.num_blocks();
  const int me = (int)cl.block_rank();
  const int64_t r0 = (int64_t)me * rows;
  const int r0i = me * rows;  // < 2^31: the slabs fit in shared memory
  const int64_t left = m - r0;
  const int nloc = left <= 0 ? 0 : (left < rows ? (int)left : rows);
  double *W = sm;                        // rows x n (column-major, ld = rows)
  double *Qs = W + (size_t)rows * n;     // rows x n
  double *msg = Qs + (size_t)rows * n;   // [2][kMaxN][2]: (partial dot, row-j entry)
  double *beta = msg + 4 * kMaxN;        // [kMaxN]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int e = tid; e < rows * n; e += kQRT) {
    const int i = e % rows, c = e / rows;
    W[e] = (i < nloc) ? Y[r0 + i + m * c] : 0.0;
  }
  __syncthreads();
  int it = 0;  // barrier-separated iteration counter (message buffer parity)

  for (int j = 0; j < n; ++j, ++it) {
    double *buf = msg + (it & 1) * 2 * kMaxN;
    const int jl = j - r0i;                   // local index of row j (owner: 0 <= jl < nloc)
    const bool owner = jl >= 0 && jl < nloc;
    const int i0 = max(jl, 0);                // local rows with global index >= j
    // partial x_j^T w_c over local rows >= j (c = j gives ||x_j||^2) and w_c[j] (owner)
    for (int c = j + warp; c < n; c += kNW) {
      double d = 0.0;
      for (int i = i0 + lane; i < nloc; i += 32) d += W[i + rows * j] * W[i + rows * c];
      d = warp_sum(d);
      if (lane == 0) {
        buf[2 * c] = d;
        buf[2 * c + 1] = owner ? W[jl + rows * c] : 0.0;
      }
    }
    cl.sync();
    const double nrm2 = cluster_sum(cl, buf, 2 * j, ncta, lane);
    const double alpha = cluster_sum(cl, buf, 2 * j + 1, ncta, lane);
    const double nrm = sqrt(nrm2);
    double b = 0.0, v0 = 0.0;
    if (nrm > 0.0) {
      v0 = alpha + (alpha >= 0.0 ? nrm : -nrm);
      b = 1.0 / (nrm * (nrm + fabs(alpha)));
    }
    if (tid == 0) beta[j] = b;
    if (b != 0.0) {
      for (int c = j + 1 + warp; c < n; c += kNW) {
        const double D = cluster_sum(cl, buf, 2 * c, ncta, lane);
        const double R = cluster_sum(cl, buf, 2 * c + 1, ncta, lane);
        const double f = b * (D + (v0 - alpha) * R);   // beta * v^T w_c
        for (int i = i0 + lane; i < nloc; i += 32) {
          const double vi = (i == jl) ? v0 : W[i + rows * j];
          W[i + rows * c] -= f * vi;
        }
      }
    }
    __syncthreads();
    if (owner && tid == 0) W[jl + rows * j] = v0;  // store v in place (v_j = v0)
    __syncthreads();
  }

  // ---- Q = H_0 H_1 ... H_{n-1} [I_n; 0], accumulated backwards
  for (int e = tid; e < rows * n; e += kQRT) {
    const int i = e % rows, c = e / rows;
    Qs[e] = (r0 + i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = n - 1; j >= 0; --j) {
    const double b = beta[j];
    if (b == 0.0) continue;  // identical in every CTA
    double *buf = msg + (it & 1) * 2 * kMaxN;
    ++it;
    const int jl = j - r0i;
    const int i0 = max(jl, 0);
    for (int c = j + warp; c < n; c += kNW) {
      double d = 0.0;
      for (int i = i0 + lane; i < nloc; i += 32) d += W[i + rows * j] * Qs[i + rows * c];
      d = warp_sum(d);
      if (lane == 0) buf[2 * c] = d;
    }
    cl.sync();
    for (int c = j + warp; c < n; c += kNW) {
      const double f = b * cluster_sum(cl, buf, 2 * c, ncta, lane);
      for (int i = i0 + lane; i < nloc; i += 32) Qs[i + rows * c] -= f * W[i + rows * j];
    }
    __syncthreads();
  }
  cl.sync();  // no CTA leaves while others may still read its message buffers
  for (int e = tid; e < nloc * n; e += kQRT) {
    const int i = e % nloc, c = e / nloc;
    Q[r0 + i + m * c] = Qs[i + rows * c];
  }
}

// Fallback for tall sketches that do not fit the cluster's shared memory (sparse modes
// with I_n ~ 1e5): same reflectors, one CTA, W and Q in global memory.
constexpr int kQRG = 1024;
__global__ void __launch_bounds__(kQRG) qr_global_kernel(double *__restrict__ W, int64_t m, int n,
                                                         double *__restrict__ Q) {
  extern __shared__ double gsm[];
  double *sbeta = gsm, *sdot = gsm + n;
  __shared__ double sred[kQRG / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kQRG / 32;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int64_t i = j + tid; i < m; i += kQRG) { const double x = W[i + m * j]; s += x * x; }
    s = warp_sum(s);
    if (lane == 0) sred[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += sred[w];
      const double alpha = W[j + m * j], nrm = sqrt(t);
      if (nrm == 0.0) {
        sbeta[j] = 0.0;
      } else {
        W[j + m * j] = alpha + (alpha >= 0.0 ? nrm : -nrm);
        sbeta[j] = 1.0 / (nrm * (nrm + fabs(alpha)));
      }
    }
    __syncthreads();
    const double b = sbeta[j];
    if (b == 0.0) continue;
    for (int c = j + 1 + warp; c < n; c += nw) {
      double d = 0.0;
      for (int64_t i = j + lane; i < m; i += 32) d += W[i + m * j] * W[i + m * c];
      d = warp_sum(d);
      if (lane == 0) sdot[c] = d;
    }
    __syncthreads();
    for (int c = j + 1; c < n; ++c) {
      const double f = b * sdot[c];
      for (int64_t i = j + tid; i < m; i += kQRG) W[i + m * c] -= f * W[i + m * j];
    }
    __syncthreads();
  }
  for (int64_t e = tid; e < m * n; e += kQRG) Q[e] = ((e % m) == (e / m)) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = n - 1; j >= 0; --j) {
    const double b = sbeta[j];
    if (b == 0.0) continue;
    for (int c = j + warp; c < n; c += nw) {
      double d = 0.0;
      for (int64_t i = j + lane; i < m; i += 32) d += W[i + m * j] * Q[i + m * c];
      d = warp_sum(d);
      if (lane == 0) sdot[c] = d;
    }
    __syncthreads();
    for (int c = j; c < n; ++c) {
      const double f = b * sdot[c];
      for (int64_t i = j + tid; i < m; i += kQRG) Q[i + m * c] -= f * W[i + m * j];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- one-sided Jacobi eig -------
constexpr int kEigT = 1024;

// Pair k of round t of the round-robin tournament on np (even) indices.
__device__ __forceinline__ void rr_pair(int k, int t, int np, int &p, int &q) {
  auto pos = [&](int i) { return i == 0 ? 0 : ((i - 1 + t) % (np - 1)) + 1; };
  p = pos(k);
  q = pos(np - 1 - k);
  if (p > q) { const int s = p; p = q; q = s; }
}

// M <- M J, V <- V J on column pairs until the columns of M = G V are orthogonal; then
// G V = V diag(lambda) with lambda_k = v_k^T m_k.
__global__ void __launch_bounds__(kEigT) jacobi_kernel(const double *__restrict__ Ain, int n, double *__restrict__ w,
                                                       double *__restrict__ Vout, double *__restrict__ gws,
                                                       double tol, int max_sweeps, int *__restrict__ info) {
  extern __shared__ double esm[];
  const int np = n + (n & 1);
  double *M = gws ? gws : esm;                // np x np, column-major
  double *V = M + (size_t)np * np;
  double *lam = V + (size_t)np * np;          // np
  __shared__ int sconv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kEigT / 32;

  for (int e = tid; e < np * np; e += kEigT) {
    const int i = e % np, j = e / np;
    M[e] = (i < n && j < n) ? 0.5 * (Ain[i + n * j] + Ain[j + n * i]) : 0.0;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int npairs = np / 2;
  int sweeps = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) sconv = 1;
    __syncthreads();
    for (int t = 0; t < np - 1; ++t) {
      for (int k = warp; k < npairs; k += NW) {
        int p, q;
        rr_pair(k, t, np, p, q);
        double a = 0.0, b = 0.0, g = 0.0;
        for (int r = lane; r < np; r += 32) {
          const double mp = M[r + np * p], mq = M[r + np * q];
          a = fma(mp, mp, a);
          b = fma(mq, mq, b);
          g = fma(mp, mq, g);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        g = warp_sum(g);
        if (g == 0.0 || fabs(g) <= tol * sqrt(a * b)) continue;  // warp-uniform
        if (lane == 0) sconv = 0;
        const double zeta = (b - a) / (2.0 * g);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = rsqrt(1.0 + tt * tt), s = tt * c;
        for (int r = lane; r < np; r += 32) {
          const double mp = M[r + np * p], mq = M[r + np * q];
          M[r + np * p] = c * mp - s * mq;
          M[r + np * q] = s * mp + c * mq;
          const double vp = V[r + np * p], vq = V[r + np * q];
          V[r + np * p] = c * vp - s * vq;
          V[r + np * q] = s * vp + c * vq;
        }
      }
      __syncthreads();
    }
    sweeps = sweep + 1;
    const int done = sconv;
    __syncthreads();
    if (done) break;
  }
  if (tid == 0 && info) *info = sweeps;
  // lambda_k = v_k^T m_k
  for (int k = warp; k < np; k += NW) {
    double d = 0.0;
    for (int r = lane; r < np; r += 32) d = fma(V[r + np * k], M[r + np * k], d);
    d = warp_sum(d);
    if (lane == 0) lam[k] = d;
  }
  __syncthreads();
  // sort descending (ties by index), drop the padding index
  for (int i = tid; i < n; i += kEigT) {
    const double di = lam[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = lam[j];
      if (dj > di || (dj == di && j < i)) ++rank;
    }
    w[rank] = di;
    for (int r = 0; r < n; ++r) Vout[r + (int64_t)n * rank] = V[r + np * i];
  }
}

// One CTA per column k: argmax |A[:, k]| (first index on ties); flip A[:, k] and U[:, k]
// when that entry is negative (DESIGN reading R4b).
__global__ void canonical_signs_kernel(double *__restrict__ A, int64_t m, double *__restrict__ U, int64_t ldu,
                                       int ell) {
  const int k = blockIdx.x;
  double *a = A + m * k;
  double best = -1.0;
  int64_t bi = 0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double v = fabs(a[i]);
    if (v > best) { best = v; bi = i; }
  }
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  __shared__ double sgn;
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = sv[0];
    int64_t i0 = si[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sv[w] > b || (sv[w] == b && si[w] < i0)) { b = sv[w]; i0 = si[w]; }
    sgn = a[i0] < 0.0 ? -1.0 : 1.0;
  }
  __syncthreads();
  if (sgn > 0.0) return;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) a[i] = -a[i];
  if (U)
    for (int i = threadIdx.x; i < ell; i += blockDim.x) U[i + ldu * k] = -U[i + ldu * k];
}

}  // namespace

void canonical_signs(Ctx &c, double *A, int64_t m, int r, double *U, int64_t ldu, int ell) {
  RT_LAUNCH(c, canonical_signs_kernel, r, 256, 0, A, m, U, ldu, ell);
}

void householder_qr(Ctx &c, const double *Y, int64_t m, int n, double *Q) {
  RT_REQUIRE(m >= n && n >= 1, "qr: need m >= n >= 1");
  RT_REQUIRE(n <= 4096, "qr: more than 4096 columns is not supported");
  // smallest cluster whose row slabs fit in shared memory (RTUCKER_QR_NCTA forces a size,
  // for testing the multi-CTA path on small inputs)
  static const int forced = [] {
    const char *e = getenv("RTUCKER_QR_NCTA");
    return e ? atoi(e) : 0;
  }();
  for (int ncta : {1, 2, 4, 8, 16}) {
    if (n > kMaxN) break;
    if (forced > 0 && ncta != forced) continue;
    const int rows = (int)((m + ncta - 1) / ncta);
    const size_t smem = sizeof(double) * ((size_t)2 * rows * n + 5 * kMaxN);
    if (smem > 200 * 1024) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(kQRT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ncta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RT_CUDA(cudaFuncSetAttribute(qr_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (ncta > 8)
      RT_CUDA(cudaFuncSetAttribute(qr_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RT_CUDA(cudaLaunchKernelEx(&cfg, qr_cluster_kernel, Y, m, n, rows, Q));
    c.launches++;
    return;
  }
  DevBuf<double> W(c, (size_t)m * n);
  RT_CUDA(cudaMemcpyAsync(W.p, Y, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, c.stream));
  const size_t smem = sizeof(double) * 2 * (size_t)n;
  if (smem > 48 * 1024)
    RT_CUDA(cudaFuncSetAttribute(qr_global_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RT_LAUNCH(c, qr_global_kernel, 1, kQRG, smem, W.p, m, n, Q);
}

void sym_eig(Ctx &c, const double *A, int n, double *w, double *V, int *sweeps) {
  const int np = n + (n & 1);
  const size_t need = sizeof(double) * (2 * (size_t)np * np + np);
  const double tol = 1e-15;
  const int max_sweeps = 30;
  DevBuf<double> ws;
  if (need <= 200 * 1024) {
    RT_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
    RT_LAUNCH(c, jacobi_kernel, 1, kEigT, need, A, n, w, V, (double *)nullptr, tol, max_sweeps, sweeps);
  } else {
    ws.alloc(c, need / sizeof(double) + 1);
    RT_LAUNCH(c, jacobi_kernel, 1, kEigT, 0, A, n, w, V, ws.p, tol, max_sweeps, sweeps);
  }
}

}  // namespace rt
