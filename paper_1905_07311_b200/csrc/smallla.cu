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
//                   barrier.
//  canonical_signs  the sign convention of DESIGN reading R4b.
#include <cstdio>
#include <cooperative_groups.h>

#include "kernels.h"
#include "kernels_extra.h"

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

constexpr int kMaxCTA = 16;

// Cluster-wide sums of slots [s0, s1) of every CTA's message buffer `buf`: all threads
// gather the remote slots into `gat` in one parallel sweep (one DSMEM round trip), then
// slot s is summed over CTAs 0..ncta-1 in that fixed order, so every CTA derives
// bit-identical values.  Ends with a CTA barrier; `tot` holds the sums.
__device__ __forceinline__ void cluster_allsum(cg::cluster_group &cl, double *buf, double *gat, double *tot,
                                               int s0, int s1, int ncta) {
  const int w = s1 - s0;
  for (int e = threadIdx.x; e < ncta * w; e += kQRT) {
    const int k = e / w, s = s0 + e % w;
    gat[k * 2 * kMaxN + s] = cl.map_shared_rank(buf, k)[s];
  }
  __syncthreads();
  for (int s = s0 + (int)threadIdx.x; s < s1; s += kQRT) {
    double v = 0.0;
    for (int k = 0; k < ncta; ++k) v += gat[k * 2 * kMaxN + s];
    tot[s] = v;
  }
  __syncthreads();
}

// Householder QR of the m x n sketch with its rows split over the CTAs of a cluster (row
// slab of W and Q in each CTA's shared memory).  Per column j: partial dots x_j^T w_c and
// the row-j entries -> one cluster barrier -> gathered, summed in fixed order -> every CTA
// forms the same reflector v = x_j + sign(alpha) ||x_j|| e_j, beta = 1/(||x|| (||x|| + |alpha|))
// and updates its rows; v^T w_c = x_j^T w_c + (v_0 - alpha) w_c[j].  Q = H_0 .. H_{n-1} [I; 0]
// is then accumulated backwards the same way.
__global__ void __launch_bounds__(kQRT) qr_cluster_kernel(const double *__restrict__ Y, int64_t m, int n,
                                                          int rows, double *__restrict__ Q,
                                                          const int *__restrict__ gate) {
  if (gate && *gate == 0) return;  // uniform across the cluster
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
  double *msg = Qs + (size_t)rows * n;   // [2 parity][2 kMaxN]: (partial dot, row-j entry)
  double *gat = msg + 4 * kMaxN;         // [kMaxCTA][2 kMaxN]
  double *tot = gat + 2 * kMaxN * kMaxCTA;  // [2 kMaxN]
  double *beta = tot + 2 * kMaxN;        // [kMaxN]
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
    cluster_allsum(cl, buf, gat, tot, 2 * j, 2 * n, ncta);
    const double nrm = sqrt(tot[2 * j]);
    const double alpha = tot[2 * j + 1];
    double b = 0.0, v0 = 0.0;
    if (nrm > 0.0) {
      v0 = alpha + (alpha >= 0.0 ? nrm : -nrm);
      b = 1.0 / (nrm * (nrm + fabs(alpha)));
    }
    if (tid == 0) beta[j] = b;
    if (b != 0.0) {
      for (int c = j + 1 + warp; c < n; c += kNW) {      // warp per column, lanes over rows
        const double f = b * (tot[2 * c] + (v0 - alpha) * tot[2 * c + 1]);  // beta v^T w_c
        for (int i = i0 + lane; i < nloc; i += 32) {
          const double vi = (i == jl) ? v0 : W[i + rows * j];
          W[i + rows * c] -= f * vi;
        }
      }
    }
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
      if (lane == 0) buf[c] = d;
    }
    cl.sync();
    cluster_allsum(cl, buf, gat, tot, j, n, ncta);
    for (int c = j + warp; c < n; c += kNW) {
      const double f = b * tot[c];
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
                                                         double *__restrict__ Q, const int *__restrict__ gate) {
  if (gate && *gate == 0) return;
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
#ifndef RT_EIG_PROBE
#define RT_EIG_PROBE(k)
#define RT_EIG_PROBE_INIT()
#endif
constexpr int kEigT = 1024;

// Pair k of round t of the round-robin tournament on np (even) indices.
__device__ __forceinline__ void rr_pair(int k, int t, int np, int &p, int &q) {
  auto pos = [&](int i) { return i == 0 ? 0 : ((i - 1 + t) % (np - 1)) + 1; };
  p = pos(k);
  q = pos(np - 1 - k);
  if (p > q) { const int s = p; p = q; q = s; }
}

// One-sided (Hestenes) Jacobi on the Gram itself: M <- M J, V <- V J on column pairs
// until the columns of M = G V are mutually orthogonal; then G V = V diag(lambda) with
// lambda_k = v_k^T m_k.  Round-robin ordering (pair table precomputed in shared memory);
// each pair of a round is owned by a group of kL lanes (8 for np <= 64, so a warp handles
// 4 pairs and the dot product needs 3 shuffle levels); one CTA barrier per round.  The
// squared column norms a_k are carried from round to round with the exact update
// a_p' = a_p - t g, a_q' = a_q + t g and recomputed at every sweep start (dgesvj
// practice), so a round reduces only g = m_p.m_q.  A pair is skipped when
// g^2 <= tol^2 a_p a_q (relative test; tol ~ sqrt(n) eps, just above the rounding of g, so
// the angle left between converged columns is <= tol lambda_q / lambda_p).
template <int kL, bool kSmem>
__global__ void __launch_bounds__(kL == 8 ? 256 : (kL == 16 ? 512 : kEigT)) jacobi_kernel(const double *__restrict__ Ain, int n, double *__restrict__ w,
                                                       double *__restrict__ Vout, double *__restrict__ gws,
                                                       double tol, int max_sweeps, int *__restrict__ info,
                                                       const int *__restrict__ gate, unsigned *__restrict__ status) {
  if (gate && *gate == 0) return;  // the preconditioned solver's result was accurate enough
  extern __shared__ double esm[];
  const int np = n + (n & 1);
  double *__restrict__ M = kSmem ? esm : gws;   // np x np, column-major
  double *__restrict__ V = M + (size_t)np * np;
  double *__restrict__ lam = V + (size_t)np * np;  // np (column norms^2 during the sweeps)
  short2 *ptab = reinterpret_cast<short2 *>(lam + np);  // [(np-1) * np/2], shared-memory variant only
  __shared__ int sconv;
  __shared__ double sfro[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x, nw = nthr >> 5;
  constexpr int kGroups = 32 / kL;                 // pairs per warp
  const int sub = lane / kL, gl = lane % kL;       // group within warp, lane within group
  const unsigned gmask = (kL == 32) ? 0xffffffffu : (((1u << kL) - 1u) << (sub * kL));
  const int npairs = np / 2;
  RT_EIG_PROBE_INIT();

  double fro = 0.0;
  for (int e = tid; e < np * np; e += nthr) {
    const int i = e % np, j = e / np;
    const double v = (i < n && j < n) ? 0.5 * (Ain[i + (size_t)n * j] + Ain[j + (size_t)n * i]) : 0.0;
    M[e] = v;
    V[e] = (i == j) ? 1.0 : 0.0;
    fro = fma(v, v, fro);
  }
  if (kSmem)
    for (int e = tid; e < (np - 1) * npairs; e += nthr) {
      int p, q;
      rr_pair(e % npairs, e / npairs, np, p, q);
      ptab[e] = make_short2((short)p, (short)q);
    }
  fro = warp_sum(fro);
  if (lane == 0) sfro[warp] = fro;
  __syncthreads();
  double f2 = 0.0;
  for (int k = 0; k < nw; ++k) f2 += sfro[k];
  const double tol2 = tol * tol;
  const int kstride = kGroups * nw;
  int sweeps = 0;
  bool converged = false;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    // column norms^2 (fresh every sweep)
    for (int k = warp; k < np; k += nw) {
      double d = 0.0;
      for (int r = lane; r < np; r += 32) { const double x = M[r + (size_t)np * k]; d = fma(x, x, d); }
      d = warp_sum(d);
      if (lane == 0) lam[k] = d;
    }
    if (tid == 0) sconv = 1;
    __syncthreads();
    for (int t = 0; t < np - 1; ++t) {
      const short2 *row = ptab + t * npairs;
      for (int k0 = warp * kGroups; k0 < npairs; k0 += kstride) {
        const int k = k0 + sub;
        const bool act = k < npairs;
        int p, q;
        if (kSmem) {
          const short2 pq = row[act ? k : 0];
          p = pq.x;
          q = pq.y;
        } else {
          rr_pair(act ? k : 0, t, np, p, q);
        }
        double *__restrict__ mp = M + (size_t)np * p;
        double *__restrict__ mq = M + (size_t)np * q;
        RT_EIG_PROBE(0);
        constexpr int kR = (kL < 32) ? 64 / kL : 1;   // rows per lane held in registers (np <= 64)
        double xp[kR], xq[kR];
        double g = 0.0;
        if (kL < 32) {
#pragma unroll
          for (int u = 0; u < kR; ++u) {
            const int r = gl + kL * u;
            xp[u] = r < np ? mp[r] : 0.0;
            xq[u] = r < np ? mq[r] : 0.0;
          }
          double pr[kR];
#pragma unroll
          for (int u = 0; u < kR; ++u) pr[u] = xp[u] * xq[u];   // independent products, then a tree
#pragma unroll
          for (int h = kR / 2; h; h >>= 1)
#pragma unroll
            for (int u = 0; u < h; ++u) pr[u] += pr[u + h];
          g = pr[0];
        } else {
          for (int r = gl; r < np; r += kL) g = fma(mp[r], mq[r], g);
        }
#pragma unroll
        for (int o = kL / 2; o; o >>= 1) g += __shfl_xor_sync(gmask, g, o, kL);
        const double a = lam[p], b = lam[q];
        const bool rot = act && g != 0.0 && g * g > tol2 * a * b;
        RT_EIG_PROBE(1);
        if (rot) {  // group-uniform
          if (gl == 0) sconv = 0;
          const double zeta = (b - a) / (2.0 * g);
          const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          const double c = rsqrt(fma(tt, tt, 1.0)), s = tt * c;
          RT_EIG_PROBE(2);
          double *__restrict__ vp = V + (size_t)np * p;
          double *__restrict__ vq = V + (size_t)np * q;
          if (kL < 32) {
            double yp[kR], yq[kR];
#pragma unroll
            for (int u = 0; u < kR; ++u) {
              const int r = gl + kL * u;
              yp[u] = r < np ? vp[r] : 0.0;
              yq[u] = r < np ? vq[r] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kR; ++u) {
              const int r = gl + kL * u;
              if (r < np) {
                mp[r] = c * xp[u] - s * xq[u];
                mq[r] = s * xp[u] + c * xq[u];
                vp[r] = c * yp[u] - s * yq[u];
                vq[r] = s * yp[u] + c * yq[u];
              }
            }
          } else {
            for (int r = gl; r < np; r += kL) {
              const double x = mp[r], y = mq[r];
              const double u = vp[r], z = vq[r];
              mp[r] = c * x - s * y;
              mq[r] = s * x + c * y;
              vp[r] = c * u - s * z;
              vq[r] = s * u + c * z;
            }
          }
          if (gl == 0) {  // exact for the exact angle; refreshed every sweep
            lam[p] = a - tt * g;
            lam[q] = b + tt * g;
          }
          RT_EIG_PROBE(3);
        }
      }
      __syncthreads();
      RT_EIG_PROBE(4);
    }
    sweeps = sweep + 1;
    const int done = sconv;
    __syncthreads();
    if (done) {
      converged = true;
      break;
    }
  }
  if (tid == 0 && info) *info = sweeps;
  if (tid == 0 && !converged && status) atomicOr(status, (unsigned)ST_EIG_NOT_CONVERGED);
  // lambda_k = v_k^T m_k
  for (int k = warp; k < np; k += nw) {
    double d = 0.0;
    for (int r = lane; r < np; r += 32) d = fma(V[r + (size_t)np * k], M[r + (size_t)np * k], d);
    d = warp_sum(d);
    if (lane == 0) lam[k] = d;
  }
  __syncthreads();
  // sort descending (ties by index), drop the padding index
  for (int i = tid; i < n; i += nthr) {
    const double di = lam[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = lam[j];
      if (dj > di || (dj == di && j < i)) ++rank;
    }
    w[rank] = di;
    for (int r = 0; r < n; ++r) Vout[r + (int64_t)n * rank] = V[r + (size_t)np * i];
  }
}

// Large-n variant of jacobi_kernel (matrices in global memory / L2) on the whole GPU: a
// cooperative grid, one warp per column pair of a round (pairs strided over all warps of the
// grid), grid.sync() between rounds.  A one-CTA sweep over n ~ 700 took ~0.3 s (3 s per
// eigensolve in the adaptive C4 run, ranks ~700); the arithmetic and the round-robin order are
// jacobi_kernel's, so the result is the same up to the order of the column-norm refreshes.
// The convergence flag rotates over three slots (reset for sweep s while sweep s - 1's slot is
// still being read).
constexpr int kEigGT = 256;
__global__ void __launch_bounds__(kEigGT) jacobi_grid_kernel(const double *__restrict__ Ain, int n,
                                                          double *__restrict__ w, double *__restrict__ Vout,
                                                          double *__restrict__ gws, int *__restrict__ conv,
                                                          double tol, int max_sweeps, int *__restrict__ info,
                                                          const int *__restrict__ gate, unsigned *__restrict__ status) {
  if (gate && *gate == 0) return;
  cg::grid_group grid = cg::this_grid();
  const int np = n + (n & 1);
  double *__restrict__ M = gws;                    // np x np, column-major
  double *__restrict__ V = M + (size_t)np * np;
  double *__restrict__ lam = V + (size_t)np * np;  // np
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gthr = (int64_t)gridDim.x * blockDim.x;
  const int gw = (int)(gtid >> 5), nw = (int)(gthr >> 5);
  const int npairs = np / 2;
  for (int64_t e = gtid; e < (int64_t)np * np; e += gthr) {
    const int i = (int)(e % np), j = (int)(e / np);
    M[e] = (i < n && j < n) ? 0.5 * (Ain[i + (size_t)n * j] + Ain[j + (size_t)n * i]) : 0.0;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  const double tol2 = tol * tol;
  int sweeps = 0;
  bool converged = false;
  grid.sync();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int k = gw; k < np; k += nw) {  // column norms^2 (fresh every sweep)
      double d = 0.0;
      for (int r = lane; r < np; r += 32) { const double x = M[r + (size_t)np * k]; d = fma(x, x, d); }
      d = warp_sum(d);
      if (lane == 0) lam[k] = d;
    }
    if (gtid == 0) conv[sweep % 3] = 1;
    grid.sync();
    for (int t = 0; t < np - 1; ++t) {
      for (int k = gw; k < npairs; k += nw) {
        int p, q;
        rr_pair(k, t, np, p, q);
        double *__restrict__ mp = M + (size_t)np * p;
        double *__restrict__ mq = M + (size_t)np * q;
        double g = 0.0;
        for (int r = lane; r < np; r += 32) g = fma(mp[r], mq[r], g);
        g = warp_sum(g);
        const double a = lam[p], b = lam[q];
        if (g != 0.0 && g * g > tol2 * a * b) {  // warp-uniform
          if (lane == 0) conv[sweep % 3] = 0;
          const double zeta = (b - a) / (2.0 * g);
          const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          const double c = rsqrt(fma(tt, tt, 1.0)), s = tt * c;
          double *__restrict__ vp = V + (size_t)np * p;
          double *__restrict__ vq = V + (size_t)np * q;
          for (int r = lane; r < np; r += 32) {
            const double x = mp[r], y = mq[r];
            const double u = vp[r], z = vq[r];
            mp[r] = c * x - s * y;
            mq[r] = s * x + c * y;
            vp[r] = c * u - s * z;
            vq[r] = s * u + c * z;
          }
          if (lane == 0) {
            lam[p] = a - tt * g;
            lam[q] = b + tt * g;
          }
        }
      }
      grid.sync();
    }
    sweeps = sweep + 1;
    if (*(volatile int *)&conv[sweep % 3]) {  // identical in every thread after the sync
      converged = true;
      break;
    }
  }
  if (gtid == 0 && info) *info = sweeps;
  if (gtid == 0 && !converged && status) atomicOr(status, (unsigned)ST_EIG_NOT_CONVERGED);
  for (int k = gw; k < np; k += nw) {  // lambda_k = v_k^T m_k
    double d = 0.0;
    for (int r = lane; r < np; r += 32) d = fma(V[r + (size_t)np * k], M[r + (size_t)np * k], d);
    d = warp_sum(d);
    if (lane == 0) lam[k] = d;
  }
  grid.sync();
  for (int64_t i = gtid; i < n; i += gthr) {  // sort descending (ties by index)
    const double di = lam[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = lam[j];
      if (dj > di || (dj == di && j < i)) ++rank;
    }
    w[rank] = di;
    for (int r = 0; r < n; ++r) Vout[r + (int64_t)n * rank] = V[r + (size_t)np * i];
  }
}

// Eigenpairs of a PSD Gram G (n <= 64), preconditioned one-sided Jacobi (Drmac-Veselic
// style): pivoted Cholesky G = M M^T with M = P L (diagonal pivoting, ties to the smallest
// index, stops at rank when the largest remaining diagonal is <= n eps max diag(G); rows are
// not exchanged, so M keeps G's index order), then one-sided Jacobi orthogonalises the
// columns of M (M J = U Sigma), so G = U Sigma^2 U^T: lambda_k = |m_k|^2, v_k = m_k / |m_k|.
// The pivoted factor is already close to column-orthogonal, so the Jacobi needs a handful of
// sweeps instead of the 13-25 sweeps of Jacobi on G itself; no rotation matrix is
// accumulated.  Eigenvectors are accurate to ~eps sigma_1 / sigma_k, i.e. for the leading part
// of the spectrum that the truncation keeps.
//
// Jacobi schedule (register resident, block ordered): the columns of M form nb (even) blocks
// of 8.  A sweep visits every column pair once: first the pairs inside each block (warp w
// holds blocks 2w, 2w+1, one column of each per 4-lane slot; round m = 1..7 pairs slot k with
// slot k ^ m, both slots evaluate the pair on shuffled copies and each updates its own column),
// then the pairs between blocks (nb - 1 outer rounds; in round t warp w takes the block pair
// rr(w, t) and its 64 column pairs in 8 rounds, the B columns shifting one slot per round).
// Lane (slot k = lane / 4, quarter q = lane % 4) keeps rows q + 4v of its columns in
// registers; g = m_p^T m_q and the two squared norms are reduced over the slot's 4 lanes
// (exact every round, nothing carried); one CTA barrier per outer round.
constexpr int kGramT = 256;

__device__ __forceinline__ double rcp_approx_f64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

// Rotation (c, s) annihilating g for squared norms a (column p), b (column q).  t is evaluated
// with fp32 approximations (a rotation that leaves ~1e-7 g behind still converges
// quadratically); c = (1 + t^2)^{-1/2} to working precision, so the rotation is orthogonal.
__device__ __forceinline__ void jac_angle(double a, double b, double g, double &c, double &s) {
  const double zeta = (b - a) * rcp_approx_f64(2.0 * g);
  double t;
  if (fabs(zeta) > 1e7) {
    t = 0.5 * rcp_approx_f64(zeta);
  } else {  // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), fp32 approximations
    const float zf = (float)zeta;
    const float s1 = fmaf(zf, zf, 1.0f);
    float r1, r2;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(s1));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(fabsf(zf) + s1 * r1));
    t = (double)copysignf(r2, zf);
  }
  // c = (1 + t^2)^{-1/2} to working precision: approximate rsqrt + two Newton steps
  const double u = fma(t, t, 1.0), hu = 0.5 * u;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(c) : "d"(u));
  c = c * fma(-hu * c, c, 1.5);
  c = c * fma(-hu * c, c, 1.5);
  s = t * c;
}

template <int kV, int LPS>
__device__ __forceinline__ void jac_pair(double (&x)[kV], double (&y)[kV], double tol2, int &rot) {
  double g0 = 0.0, g1 = 0.0, a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
  for (int v = 0; v < kV; v += 2) {  // six independent chains
    g0 = fma(x[v], y[v], g0);
    g1 = fma(x[v + 1], y[v + 1], g1);
    a0 = fma(x[v], x[v], a0);
    a1 = fma(x[v + 1], x[v + 1], a1);
    b0 = fma(y[v], y[v], b0);
    b1 = fma(y[v + 1], y[v + 1], b1);
  }
  double g = g0 + g1, a = a0 + a1, b = b0 + b1;
#pragma unroll
  for (int o = 1; o < LPS; o <<= 1) {  // the slot's LPS lanes; identical sums in all of them
    g += __shfl_xor_sync(0xffffffffu, g, o);
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (g != 0.0 && g * g > tol2 * a * b) {
    rot = 1;
    double c, s;
    jac_angle(a, b, g, c, s);
#pragma unroll
    for (int v = 0; v < kV; ++v) {
      const double xv = x[v], yv = y[v];
      x[v] = fma(c, xv, -s * yv);
      y[v] = fma(s, xv, c * yv);
    }
  }
}

// Pair (p, q) evaluated on BOTH slots that hold copies of the two columns (XOR schedule): the
// slot owning column p passes (own = m_p, oth = m_q, own_is_p = true), the slot owning q the
// mirror; the sums are formed in the same order on both (x*y == y*x exactly), so both take
// the identical rotation and each updates its own column only.
template <int kV, int LPS>
__device__ __forceinline__ void jac_half(double (&own)[kV], const double (&oth)[kV], bool own_is_p, double tol2,
                                         int &rot) {
  double g0 = 0.0, g1 = 0.0, o0 = 0.0, o1 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
  for (int v = 0; v < kV; v += 2) {
    g0 = fma(own[v], oth[v], g0);
    g1 = fma(own[v + 1], oth[v + 1], g1);
    o0 = fma(own[v], own[v], o0);
    o1 = fma(own[v + 1], own[v + 1], o1);
    t0 = fma(oth[v], oth[v], t0);
    t1 = fma(oth[v + 1], oth[v + 1], t1);
  }
  double g = g0 + g1, so = o0 + o1, st = t0 + t1;
#pragma unroll
  for (int o = 1; o < LPS; o <<= 1) {
    g += __shfl_xor_sync(0xffffffffu, g, o);
    so += __shfl_xor_sync(0xffffffffu, so, o);
    st += __shfl_xor_sync(0xffffffffu, st, o);
  }
  const double a = own_is_p ? so : st, b = own_is_p ? st : so;
  if (g != 0.0 && g * g > tol2 * a * b) {
    rot = 1;
    double c, s;
    jac_angle(a, b, g, c, s);
    if (own_is_p) {
#pragma unroll
      for (int v = 0; v < kV; ++v) own[v] = fma(c, own[v], -s * oth[v]);
    } else {
#pragma unroll
      for (int v = 0; v < kV; ++v) own[v] = fma(s, oth[v], c * own[v]);
    }
  }
}

// Pivoted Cholesky of the np x np Gram G (column-major, shared memory) without row exchanges,
// left-looking, one CTA barrier per step (256 threads: 4 per row):
//   p = argmax of the remaining diagonal d (first index on ties; every warp evaluates it
//   redundantly from d in shared memory, so no barrier publishes it), stop once d_p <= n eps
//   max diag(G);  M[i, k] = (G[i, p] - sum_{k' < k} M[i, k'] M[p, k']) / sqrt(d_p) on the rows
//   not yet pivoted (4 threads per row split the dot product), d_i -= M[i, k]^2.
//   M = P L (P the pivot permutation): its columns have the preconditioning of L, and
//   M M^T = G in the original index order.  (Right-looking with a rank-1 update of G and a
//   separate pivot pass cost 3 barriers and ~2100 cycles per step: 125k cycles at n = 60.)
// M (ldm x >= np) must be zero on entry; lc, lam: np-double scratch each.  Returns the number
// of pivots taken (the numerical rank); the columns of M beyond it stay zero.
__device__ int chol_pivoted_left(const double *__restrict__ G, int np, int n, double *__restrict__ M, int ldm,
                                 double *__restrict__ lc, double *__restrict__ lam, int ldg) {
  const int tid = threadIdx.x, lane = tid & 31;
  // remaining diagonal, double-buffered (step k reads lc / lam by parity, writes the other); -inf
  // marks a pivoted (or padding) row; a remaining diagonal that rounds below zero stays live
  for (int i = tid; i < np; i += blockDim.x) lc[i] = i < n ? G[i + ldg * i] : -INFINITY;
  double dmax = 0.0;
  for (int i = lane; i < n; i += 32) dmax = fmax(dmax, G[i + ldg * i]);
  for (int o = 16; o; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const double thresh = n * 2.2e-16 * dmax;
  __syncthreads();
  const int ci = tid >> 2, cs = tid & 3;  // row ci, dot-product quarter cs
#ifdef RTUCKER_EIG_PROF_BUILD
  long long cpa[5] = {0, 0, 0, 0, 0}, cpt = clock64();
#define CHP(i) { const long long t_ = clock64(); cpa[i] += t_ - cpt; cpt = t_; }
#else
#define CHP(i)
#endif
  int k = 0;
  for (; k < n; ++k) {
    CHP(0);
    const double *dc = (k & 1) ? lam : lc;
    double *dnx = (k & 1) ? lc : lam;
    // pivot = argmax of the remaining diagonal to fp32 resolution by ONE warp reduction: key =
    // fp32 bits of d_i (non-negative floats order like their bit patterns) with the low 6 bits
    // replaced by 63 - i (ties, and values equal to 2^-17 relative, go to the smallest index);
    // the pivot only has to be near-maximal (for the grading), and the choice is deterministic.
    // Negative entries (pivoted rows, diagonals rounded below 0) count as 0.  (Three dependent
    // redux.sync for the exact fp64 maximum cost ~700 cycles per step.)
    uint32_t key = 0;
    for (int i = lane; i < n; i += 32) {
      const double v = dc[i];
      const uint32_t kb = v > 0.0 ? ((__float_as_uint((float)v) & ~63u) | (uint32_t)(63 - i)) : 0u;
      key = max(key, kb);
    }
    key = __reduce_max_sync(0xffffffffu, key);
    const int bi = 63 - (int)(key & 63u);
    const double bv = key ? dc[bi] : 0.0;
    if (!(bv > thresh)) break;  // rank reached (same decision in every warp): the rest of M is zero
    const int p = bi;
    double inv;  // bv^{-1/2}: approximate rsqrt + two Newton steps (no slow-path subroutine)
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(bv));
    inv = inv * fma(-0.5 * bv * inv, inv, 1.5);
    inv = inv * fma(-0.5 * bv * inv, inv, 1.5);
    CHP(1);
    double dot = 0.0;
    if (ci < np) {  // four independent chains (loads of 4 steps in flight)
      double d1 = 0.0, d2 = 0.0, d3 = 0.0;
      int kk = cs;
      for (; kk + 12 < k; kk += 16) {
        dot = fma(M[ci + ldm * kk], M[p + ldm * kk], dot);
        d1 = fma(M[ci + ldm * (kk + 4)], M[p + ldm * (kk + 4)], d1);
        d2 = fma(M[ci + ldm * (kk + 8)], M[p + ldm * (kk + 8)], d2);
        d3 = fma(M[ci + ldm * (kk + 12)], M[p + ldm * (kk + 12)], d3);
      }
      for (; kk < k; kk += 4) dot = fma(M[ci + ldm * kk], M[p + ldm * kk], dot);
      dot = (dot + d1) + (d2 + d3);
    }
    dot += __shfl_xor_sync(0xffffffffu, dot, 1);
    dot += __shfl_xor_sync(0xffffffffu, dot, 2);
    CHP(2);
    if (cs == 0 && ci < np) {
      const double dci = dc[ci];
      const bool done = dci == -INFINITY;
      const double l = done ? 0.0 : (G[ci + ldg * p] - dot) * inv;
      M[ci + ldm * k] = l;
      dnx[ci] = (done || ci == p) ? -INFINITY : dci - l * l;
    }
    CHP(3);
    __syncthreads();
    CHP(4);
  }
#ifdef RTUCKER_EIG_PROF_BUILD
  if (tid == 0 || tid == 255)
    printf("[chol prof] tid %d steps %d: top %lld argmax %lld dot %lld write %lld barrier %lld\n", tid, k, cpa[0], cpa[1],
           cpa[2], cpa[3], cpa[4]);
#endif
#undef CHP
  return k;
}

template <int kV, int LPS>
__device__ void gram_eig_body(double *__restrict__ gsm2, const double *__restrict__ Ain, int n,
                              double *__restrict__ w, double *__restrict__ Vout, double tol, int max_sweeps,
                              int *__restrict__ info, int r_need, int *__restrict__ refine,
                              unsigned *__restrict__ status) {
#ifdef RTUCKER_EIG_PROF_BUILD
  long long et_[6];
  int en_ = 0;
#define EGP() if (threadIdx.x == 0 && en_ < 6) et_[en_++] = clock64()
#else
#define EGP()
#endif
  EGP();
  constexpr int SPW = 32 / LPS;        // column slots per warp = block size
  const int np = n + (n & 1);
  const int nb = ((n + 2 * SPW - 1) / (2 * SPW)) * 2;  // column blocks of SPW (even count)
  const int ncol = SPW * nb;
  constexpr int ldm = LPS * kV + LPS;  // = LPS mod 16: conflict-free slot loads
  double *G = gsm2;                    // np x np working copy (column-major)
  double *M = G + np * np;             // ldm x ncol: P L, then M J
  double *lam = M + ldm * ncol;        // ncol
  double *lc = lam + ncol;             // np: current column of L
  int *dn = reinterpret_cast<int *>(lc + np);  // np: row already pivoted
  __shared__ int spiv, sflag;
  __shared__ double sdmax;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < np * np; e += kGramT) {
    const int i = e % np, j = e / np;
    G[e] = (i < n && j < n) ? 0.5 * (Ain[i + (size_t)n * j] + Ain[j + (size_t)n * i]) : 0.0;
  }
  for (int e = tid; e < ldm * ncol; e += kGramT) M[e] = 0.0;
  for (int i = tid; i < np; i += kGramT) dn[i] = i < n ? 0 : 1;
  __syncthreads();
  chol_pivoted_left(G, np, n, M, ldm, lc, lam, np);
  EGP();
  // ---- block-ordered one-sided Jacobi on the columns of M
  const double tol2 = tol * tol;
  const int slot = lane / LPS, q = lane % LPS;
  const int nwk = nb / 2;  // working warps
  int sweeps = 0;
  bool converged = false;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) sflag = 0;
    __syncthreads();
    int rot = 0;
    if (warp < nwk) {  // pairs inside blocks 2w (x) and 2w + 1 (y): round m pairs slot k with k ^ m
      double *c1 = M + ldm * (2 * SPW * warp + slot), *c2 = c1 + SPW * ldm;
      double x[kV], y[kV];
#pragma unroll
      for (int v = 0; v < kV; ++v) { x[v] = c1[q + LPS * v]; y[v] = c2[q + LPS * v]; }
#pragma unroll 1
      for (int m = 1; m < SPW; ++m) {
        const int src = (slot ^ m) * LPS + q;
        const bool own_p = slot < (slot ^ m);
        double px[kV], py[kV];
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          px[v] = __shfl_sync(0xffffffffu, x[v], src);
          py[v] = __shfl_sync(0xffffffffu, y[v], src);
        }
        jac_half<kV, LPS>(x, px, own_p, tol2, rot);
        jac_half<kV, LPS>(y, py, own_p, tol2, rot);
      }
#pragma unroll
      for (int v = 0; v < kV; ++v) { c1[q + LPS * v] = x[v]; c2[q + LPS * v] = y[v]; }
    }
    __syncthreads();
    for (int t = 0; t < nb - 1; ++t) {  // pairs between blocks
      if (warp < nwk) {
        int bA, bB;
        rr_pair(warp, t, nb, bA, bB);
        double *c1 = M + ldm * (SPW * bA + slot), *c2 = M + ldm * (SPW * bB + slot);
        double x[kV], y[kV];
#pragma unroll
        for (int v = 0; v < kV; ++v) { x[v] = c1[q + LPS * v]; y[v] = c2[q + LPS * v]; }
        const int nxt = ((slot + 1) % SPW) * LPS + q;
#pragma unroll 1
        for (int r = 0; r < SPW; ++r) {
          jac_pair<kV, LPS>(x, y, tol2, rot);
#pragma unroll
          for (int v = 0; v < kV; ++v) y[v] = __shfl_sync(0xffffffffu, y[v], nxt);
        }
#pragma unroll
        for (int v = 0; v < kV; ++v) { c1[q + LPS * v] = x[v]; c2[q + LPS * v] = y[v]; }
      }
      __syncthreads();
    }
    if (rot) sflag = 1;
    __syncthreads();
    sweeps = sweep + 1;
    const int more = sflag;
    __syncthreads();
    if (!more) {
      converged = true;
      break;
    }
  }
  EGP();
  if (tid == 0 && info) *info = sweeps;
  if (tid == 0 && !converged && status) atomicOr(status, (unsigned)ST_EIG_NOT_CONVERGED);
  for (int k = warp; k < np; k += kGramT / 32) {  // exact column norms
    double d = 0.0;
    for (int r = lane; r < np; r += 32) { const double x = M[r + ldm * k]; d = fma(x, x, d); }
    d = warp_sum(d);
    if (lane == 0) lam[k] = d;
  }
  __syncthreads();
  // sort descending (ties by index), drop the padding column, v_k = P m_k / |m_k|
  for (int i = tid; i < n; i += kGramT) {
    const double di = lam[i];
    int rank = 0;
    for (int j = 0; j < np; ++j) {
      const double dj = lam[j];
      if (j != i && (dj > di || (dj == di && j < i))) ++rank;
    }
    if (rank >= n) continue;
    w[rank] = di;
    const double inv = di > 0.0 ? 1.0 / sqrt(di) : 0.0;
    for (int r = 0; r < n; ++r) Vout[r + (int64_t)n * rank] = M[r + ldm * i] * inv;
  }
  EGP();
#ifdef RTUCKER_EIG_PROF_BUILD
  if (threadIdx.x == 0) printf("[eig prof] n %d sweeps %d: init %lld chol %lld jacobi %lld final %lld\n", n, sweeps,
                               et_[1] - et_[0], et_[2] - et_[1], et_[3] - et_[2], et_[4] - et_[3]);
#endif
  // v_k from a normalised column is accurate to ~eps sqrt(lambda_0 / lambda_k): request the
  // unpreconditioned solver when the wanted rank reaches lambda_k < 1e-8 lambda_0
  if (refine) {
    __syncthreads();  // w (global) written above by the sorting threads
    if (tid == 0) *refine = (w[r_need - 1] >= 1e-8 * w[0]) ? 0 : 1;
  }
}

template <int kV, int LPS>
__global__ void __launch_bounds__(kGramT) gram_eig_kernel(const double *__restrict__ Ain, int n, double *__restrict__ w,
                                                          double *__restrict__ Vout, double tol, int max_sweeps,
                                                          int *__restrict__ info, int r_need, int *__restrict__ refine,
                                                          unsigned *__restrict__ status) {
  extern __shared__ double gsm_dyn[];
  gram_eig_body<kV, LPS>(gsm_dyn, Ain, n, w, Vout, tol, max_sweeps, info, r_need, refine, status);
}

// ----------------------------------------------------- mixed-precision Gram eigensolver ----
// fp32 data, n <= 64 (the fixed-rank truncation of Alg 1 line 4, eigenpairs of the l x l
// Gram B B^T): the fp32 criteria need the eigenvectors to the absolute accuracy ~eps lambda_1 /
// gap (the class of the tridiagonal solver used above 64), which an fp64 Newton refinement of
// an fp32 starting basis reaches in two or three GEMM-shaped steps:
//   1. pivoted Cholesky G = M M^T in fp64 (chol_pivoted_left: M keeps the column grading);
//   2. block-ordered one-sided Jacobi on an fp32 copy of M (same schedule as gram_eig_kernel)
//      to column orthogonality ~4e-6; X = normalised columns of M J (eigenvector estimates of
//      G, angles ~4e-6 / relative gap thanks to the grading);
//   3. Ogita-Aishima refinement in fp64 (Newton steps on X^T X = I, X^T G X diagonal):
//        R = I - X^T X, S = X^T G X, lambda_i = S_ii / (1 - R_ii),
//        E_ij = (S_ij + lambda_j R_ij) / (lambda_j - lambda_i)   (i != j, |E_ij| <= 1/8),
//        E_ij = R_ij / 2                                        (otherwise: a cluster),
//        X <- X + X E,
//      the four 64^3 products on the fp64 tensor cores (mma.sync m8n8k4), until max |E| <= 1e-8
//      (the next correction would be below 1e-16) or four steps.
// A rank-deficient Gram (the Cholesky stops early) or a pair of the final step that is still
// unresolved across the wanted rank r_need with a gap above 1e-12 lambda_1 raises *fallback,
// which runs the fp64 Jacobi kernel (device-side gate, no host sync).
constexpr int kMxT = 256;
constexpr int kMxLd = 66;  // 64 x 64 fp64 tiles: 2-wavefront m8n8k4 fragment loads both ways

__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// C = op(A) B (+ Cin) for 64 x 64 column-major shared-memory operands (ld kMxLd); 8 warps, warp w
// computes rows 16 (w & 3) .. + 15 and columns 32 (w >> 2) .. + 31 as 2 x 4 tiles of 8 x 8.
template <bool TA>
__device__ __forceinline__ void mx_gemm64(const double *__restrict__ A, const double *__restrict__ B,
                                          double *__restrict__ C, const double *__restrict__ Cin) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int i0 = 16 * (warp & 3), j0 = 32 * (warp >> 2);
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = i0 + 8 * i + g, cc = j0 + 8 * j + 2 * t;
      acc[i][j][0] = Cin ? Cin[r + kMxLd * cc] : 0.0;
      acc[i][j][1] = Cin ? Cin[r + kMxLd * (cc + 1)] : 0.0;
    }
#pragma unroll 4
  for (int k0 = 0; k0 < 64; k0 += 4) {
    double a[2], b[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = i0 + 8 * i + g;
      a[i] = TA ? A[(k0 + t) + kMxLd * r] : A[r + kMxLd * (k0 + t)];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = B[(k0 + t) + kMxLd * (j0 + 8 * j + g)];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = i0 + 8 * i + g, cc = j0 + 8 * j + 2 * t;
      C[r + kMxLd * cc] = acc[i][j][0];
      C[r + kMxLd * (cc + 1)] = acc[i][j][1];
    }
}

// fp32 rotation (c, s) annihilating g for squared column norms a (p), b (q)
// fp32 rotation (c, s) annihilating g for squared column norms a (p), b (q) in two dependent
// MUFU steps: with d = b - a and r = sqrt(d^2 + 4 g^2), cos 2theta = |d| / r, c = sqrt((1 +
// cos 2theta) / 2), s = sgn(d) g / (r c) (|theta| <= pi/4; the usual t = sgn(zeta) / (|zeta| +
// sqrt(1 + zeta^2)) chain cost five dependent MUFU operations).  g = 0 gives the identity.
__device__ __forceinline__ float rsqrt_ftz_f32(float x) {  // bare MUFU.RSQ (no denormal fix-up code)
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void jac_angle_f32(float a, float b, float g, float &c, float &s) {
  const float d = b - a;
  const float q = rsqrt_ftz_f32(fmaf(d, d, 4.0f * g * g));
  const float h = fmaf(fabsf(d), 0.5f * q, 0.5f);
  const float rh = rsqrt_ftz_f32(h);
  const bool id = g == 0.0f;
  c = id ? 1.0f : h * rh;
  s = id ? 0.0f : copysignf(1.0f, d) * (g * q * rh);
}

// convergence test g^2 > tol^2 a b, off the rotation's critical path: every pair is rotated, a
// converged one by an angle below tol.  (Columns are scaled to max norm 1 and the Cholesky stops
// at n eps max diag, so tol^2 a b >= 1e-6 (64 eps)^2 stays a normal fp32 number.)
__device__ __forceinline__ bool jac_needs_f32(float a, float b, float g, float tol) {
  return g * g > (tol * tol) * (a * b);
}

template <int kV, int LPS>
__device__ __forceinline__ void jac_pair_f32(float (&x)[kV], float (&y)[kV], float tol, int &rot) {
  float g0 = 0.f, g1 = 0.f, a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll
  for (int v = 0; v < kV; v += 2) {
    g0 = fmaf(x[v], y[v], g0);
    g1 = fmaf(x[v + 1], y[v + 1], g1);
    a0 = fmaf(x[v], x[v], a0);
    a1 = fmaf(x[v + 1], x[v + 1], a1);
    b0 = fmaf(y[v], y[v], b0);
    b1 = fmaf(y[v + 1], y[v + 1], b1);
  }
  float g = g0 + g1, a = a0 + a1, b = b0 + b1;
#pragma unroll
  for (int o = 1; o < LPS; o <<= 1) {
    g += __shfl_xor_sync(0xffffffffu, g, o);
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  rot |= jac_needs_f32(a, b, g, tol) ? 1 : 0;
  float c, s;
  jac_angle_f32(a, b, g, c, s);
#pragma unroll
  for (int v = 0; v < kV; ++v) {
    const float xv = x[v], yv = y[v];
    x[v] = fmaf(c, xv, -s * yv);
    y[v] = fmaf(s, xv, c * yv);
  }
}

template <int kV, int LPS>
__device__ __forceinline__ void jac_half_f32(float (&own)[kV], const float (&oth)[kV], bool own_is_p, float tol,
                                             int &rot) {
  float g0 = 0.f, g1 = 0.f, o0 = 0.f, o1 = 0.f, t0 = 0.f, t1 = 0.f;
#pragma unroll
  for (int v = 0; v < kV; v += 2) {
    g0 = fmaf(own[v], oth[v], g0);
    g1 = fmaf(own[v + 1], oth[v + 1], g1);
    o0 = fmaf(own[v], own[v], o0);
    o1 = fmaf(own[v + 1], own[v + 1], o1);
    t0 = fmaf(oth[v], oth[v], t0);
    t1 = fmaf(oth[v + 1], oth[v + 1], t1);
  }
  float g = g0 + g1, so = o0 + o1, st = t0 + t1;
#pragma unroll
  for (int o = 1; o < LPS; o <<= 1) {
    g += __shfl_xor_sync(0xffffffffu, g, o);
    so += __shfl_xor_sync(0xffffffffu, so, o);
    st += __shfl_xor_sync(0xffffffffu, st, o);
  }
  const float a = own_is_p ? so : st, b = own_is_p ? st : so;
  rot |= jac_needs_f32(a, b, g, tol) ? 1 : 0;
  float c, s;
  jac_angle_f32(a, b, g, c, s);
  // p: c own - s oth;  q: s oth + c own  (the mirror slot applies the other half)
  const float so_ = own_is_p ? -s : s;
#pragma unroll
  for (int v = 0; v < kV; ++v) own[v] = fmaf(so_, oth[v], c * own[v]);
}

constexpr int kMxLdm = 68;  // fp32 Jacobi columns: 4 lanes x 16 rows + 4 (conflict-free slot loads)
constexpr size_t kMxSmem = sizeof(double) * (5 * 64 * kMxLd + 6 * 64) + 64;

// A (64 x 64, ld kMxLd) -= P P^T for a 64 x 8 panel P (column-major, ld ldp) on the fp64 tensor
// cores (the trailing update of the blocked Cholesky below; same warp tiling as mx_gemm64)
__device__ __forceinline__ void mx_syrk8(double *__restrict__ A, const double *__restrict__ P, int ldp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int i0 = 16 * (warp & 3), j0 = 32 * (warp >> 2);
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = i0 + 8 * i + g, cc = j0 + 8 * j + 2 * t;
      acc[i][j][0] = A[r + kMxLd * cc];
      acc[i][j][1] = A[r + kMxLd * (cc + 1)];
    }
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += 4) {
    double a[2], b[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = -P[(i0 + 8 * i + g) + ldp * (k0 + t)];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = P[(j0 + 8 * j + g) + ldp * (k0 + t)];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = i0 + 8 * i + g, cc = j0 + 8 * j + 2 * t;
      A[r + kMxLd * cc] = acc[i][j][0];
      A[r + kMxLd * (cc + 1)] = acc[i][j][1];
    }
}

// Blocked pivoted Cholesky G = M M^T (M = P L, rows in the original order, no row exchanges) for
// the mixed solver, 256 threads, n <= 64.  Panels of 8 columns: ONE warp factors the panel
// (rows lane and lane + 32 in registers, the remaining diagonal d in registers, pivot = argmax d
// by one redux.sync as in chol_pivoted_left, earlier panel columns of the pivot row by shuffles:
// no CTA barrier inside a panel), then all warps apply the trailing update A -= P P^T on the
// fp64 tensor cores.  ~250 cycles per column instead of ~1900 for the one-barrier-per-column
// left-looking form.  A (ld kMxLd) is a working copy of G and is destroyed; M (ld ldm) must be
// zero on entry.  Returns the number of pivots (numerical rank, threshold n eps max diag).
__device__ int chol_pivoted_panel(double *__restrict__ A, int n, double *__restrict__ M, int ldm, int *sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double d0 = -1.0, d1 = -1.0;  // remaining diagonal of rows lane, lane + 32 (-1: pivoted / padding)
  double thresh = 0.0;
  if (warp == 0) {
    if (lane < n) d0 = A[lane * (kMxLd + 1)];
    if (lane + 32 < n) d1 = A[(lane + 32) * (kMxLd + 1)];
    double dm = fmax(d0, d1);
    for (int o = 16; o; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    thresh = n * 2.2e-16 * dm;
  }
  int k = 0;
  for (int j0 = 0; j0 < n; j0 += 8) {
    if (warp == 0) {
      double P0[8], P1[8];
      int stop = 0;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        P0[jj] = 0.0;
        P1[jj] = 0.0;
        if (stop || j0 + jj >= n) continue;
        uint32_t key0 = d0 > 0.0 ? ((__float_as_uint((float)d0) & ~63u) | (uint32_t)(63 - lane)) : 0u;
        uint32_t key1 = d1 > 0.0 ? ((__float_as_uint((float)d1) & ~63u) | (uint32_t)(31 - lane)) : 0u;
        const uint32_t key = __reduce_max_sync(0xffffffffu, max(key0, key1));
        const int p = 63 - (int)(key & 63u), pl = p & 31;
        const bool hi = p >= 32;
        const double bv = __shfl_sync(0xffffffffu, hi ? d1 : d0, pl);
        if (!key || !(bv > thresh)) {
          stop = 1;
          continue;
        }
        double inv;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(bv));
        inv = inv * fma(-0.5 * bv * inv, inv, 1.5);
        inv = inv * fma(-0.5 * bv * inv, inv, 1.5);
        double a0 = A[lane + kMxLd * p], a1 = A[lane + 32 + kMxLd * p];
#pragma unroll
        for (int q = 0; q < jj; ++q) {
          const double pp = __shfl_sync(0xffffffffu, hi ? P1[q] : P0[q], pl);
          a0 = fma(-P0[q], pp, a0);
          a1 = fma(-P1[q], pp, a1);
        }
        const double l0 = d0 < 0.0 && lane != p ? 0.0 : a0 * inv;
        const double l1 = d1 < 0.0 && lane + 32 != p ? 0.0 : a1 * inv;
        P0[jj] = l0;
        P1[jj] = l1;
        M[lane + ldm * (j0 + jj)] = l0;
        M[lane + 32 + ldm * (j0 + jj)] = l1;
        d0 = (d0 < 0.0 || lane == p) ? -1.0 : d0 - l0 * l0;
        d1 = (d1 < 0.0 || lane + 32 == p) ? -1.0 : d1 - l1 * l1;
      }
      if (lane == 0) {
        sh[0] = stop;
        sh[1] = stop ? -1 : 0;
      }
      // pivots taken in this panel: columns j0.. until the stop
      int taken = 0;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) taken += (j0 + jj < n) ? 1 : 0;
      (void)taken;
    }
    __syncthreads();
    const int stopped = sh[0];
    if (stopped || j0 + 8 >= n) {
      // count the columns actually taken (nonzero pivot entries) in this last panel
      k = j0;
      for (int jj = 0; jj < 8 && j0 + jj < n; ++jj) {
        bool nz = false;
        for (int r = 0; r < n; ++r) nz |= M[r + ldm * (j0 + jj)] != 0.0;
        if (!nz) break;
        ++k;
      }
      break;
    }
    mx_syrk8(A, M + ldm * j0, ldm);
    __syncthreads();
  }
  return k;
}



__global__ void __launch_bounds__(kMxT) gram_eig_mixed_kernel(const double *__restrict__ Ain, int n,
                                                              double *__restrict__ w, double *__restrict__ Vout,
                                                              int *__restrict__ info, int r_need, int max_sweeps,
                                                              double tol64, int *__restrict__ refine,
                                                              unsigned *__restrict__ status) {
  constexpr int kV = 16, LPS = 4, SPW = 8, NB = 8;  // 64 columns of 64 rows, 8 blocks of 8
  extern __shared__ double mxs[];
#ifdef RTUCKER_EIG_PROF_BUILD
  long long mt_[12];
  int mn_ = 0;
#define MXP() if (threadIdx.x == 0 && mn_ < 12) mt_[mn_++] = clock64()
#else
#define MXP()
#endif
  MXP();
  double *Gs = mxs;                   // 64 x 64 (ld kMxLd), zero padded
  double *buf1 = Gs + 64 * kMxLd;     // M32 (fp32 Jacobi columns), later a product buffer
  double *buf2 = buf1 + 64 * kMxLd;   // M (fp64, ld kMxLdm, spans buf2..buf3), later X
  double *buf3 = buf2 + 64 * kMxLd;
  double *Eb = buf3 + 64 * kMxLd;     // the refinement's correction E
  double *lc = Eb + 64 * kMxLd, *lam = lc + 64, *lamv = lam + 64, *rowoff = lamv + 64, *rowr = rowoff + 64;
  int *rkv = reinterpret_cast<int *>(rowr + 64);
  float *M32 = reinterpret_cast<float *>(buf1);
  double *M = buf2;
  __shared__ int sflag, sbad;
  __shared__ float smaxe;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int np = n + (n & 1);
  for (int e = tid; e < 64 * kMxLd; e += kMxT) {
    const int i = e % kMxLd, j = e / kMxLd;
    const double gv = (i < n && j < n) ? 0.5 * (Ain[i + (size_t)n * j] + Ain[j + (size_t)n * i]) : 0.0;
    Gs[e] = gv;
    Eb[e] = gv;  // the Cholesky's working copy
    buf2[e] = 0.0;
    buf3[e] = 0.0;
  }
  if (tid == 0) {
    sbad = 0;
    if (refine) *refine = 0;  // set again by the fp64 fallback when it needs the unpreconditioned solver
  }
  __syncthreads();
  // ---- 1. pivoted Cholesky (fp64, blocked)
  __shared__ int csh[2];
  const int rank = chol_pivoted_panel(Eb, n, M, kMxLdm, csh);
  (void)np;
  MXP();
  if (rank < n) {  // rank-deficient Gram: the fp64 Jacobi (null space as zero columns)
    __syncthreads();
    gram_eig_body<16, 4>(mxs, Ain, n, w, Vout, tol64, 40, info, r_need, refine, status);
    return;
  }
  // ---- 2. fp32 one-sided Jacobi on M / sqrt(max column norm^2) (no fp32 overflow / underflow)
  double dmx = 0.0;
  for (int i = 0; i < n; ++i) dmx = fmax(dmx, Gs[i + kMxLd * i]);
  const double sc = dmx > 0.0 ? 1.0 / sqrt(dmx) : 1.0;
  for (int e = tid; e < kMxLdm * 64; e += kMxT) M32[e] = (float)(M[e] * sc);
  __syncthreads();
  // a start to ~1e-3: the refinement's Newton steps converge quadratically from there
  const float tol = 1e-3f;
  const int slot = lane / LPS, q = lane % LPS;
  int sweeps = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) sflag = 0;
    __syncthreads();
    int rot = 0;
    if (warp < NB / 2) {
      float *c1 = M32 + kMxLdm * (2 * SPW * warp + slot), *c2 = c1 + SPW * kMxLdm;
      float x[kV], y[kV];
#pragma unroll
      for (int v = 0; v < kV; ++v) { x[v] = c1[q + LPS * v]; y[v] = c2[q + LPS * v]; }
#pragma unroll 1
      for (int m = 1; m < SPW; ++m) {
        const int src = (slot ^ m) * LPS + q;
        const bool own_p = slot < (slot ^ m);
        float px[kV], py[kV];
#pragma unroll
        for (int v = 0; v < kV; ++v) {
          px[v] = __shfl_sync(0xffffffffu, x[v], src);
          py[v] = __shfl_sync(0xffffffffu, y[v], src);
        }
        jac_half_f32<kV, LPS>(x, px, own_p, tol, rot);
        jac_half_f32<kV, LPS>(y, py, own_p, tol, rot);
      }
#pragma unroll
      for (int v = 0; v < kV; ++v) { c1[q + LPS * v] = x[v]; c2[q + LPS * v] = y[v]; }
    }
    __syncthreads();
    for (int t = 0; t < NB - 1; ++t) {
      if (warp < NB / 2) {
        int bA, bB;
        rr_pair(warp, t, NB, bA, bB);
        float *c1 = M32 + kMxLdm * (SPW * bA + slot), *c2 = M32 + kMxLdm * (SPW * bB + slot);
        float x[kV], y[kV];
#pragma unroll
        for (int v = 0; v < kV; ++v) { x[v] = c1[q + LPS * v]; y[v] = c2[q + LPS * v]; }
        const int nxt = ((slot + 1) % SPW) * LPS + q;
#pragma unroll 1
        for (int r = 0; r < SPW; ++r) {
          jac_pair_f32<kV, LPS>(x, y, tol, rot);
#pragma unroll
          for (int v = 0; v < kV; ++v) y[v] = __shfl_sync(0xffffffffu, y[v], nxt);
        }
#pragma unroll
        for (int v = 0; v < kV; ++v) { c1[q + LPS * v] = x[v]; c2[q + LPS * v] = y[v]; }
      }
      __syncthreads();
    }
    if (rot) sflag = 1;
    __syncthreads();
    sweeps = sweep + 1;
    const int more = sflag;
    __syncthreads();
    if (!more) break;
  }
  MXP();
  // X = normalised columns of M32 J (fp64), columns >= n and rows >= n zero
  double *X = buf2, *T1 = buf1, *T2 = buf3;
  for (int k = warp; k < 64; k += kMxT / 32) {
    double d = 0.0;
    for (int r = lane; r < 64; r += 32) { const double v = (double)M32[r + kMxLdm * k]; d = fma(v, v, d); }
    d = warp_sum(d);
    if (lane == 0) lc[k] = d;
  }
  __syncthreads();
  // column k of M32 -> column k of X (M32 lives in buf1, X in buf2: no overlap)
  for (int e = tid; e < 64 * 64; e += kMxT) {
    const int r = e & 63, k = e >> 6;
    const double d = lc[k];
    X[r + kMxLd * k] = (r < n && k < n && d > 0.0) ? (double)M32[r + kMxLdm * k] / sqrt(d) : 0.0;
  }
  __syncthreads();
  MXP();
  // ---- 3. Ogita-Aishima refinement (fp64 tensor cores).  S and I - R are read symmetrised (the
  // GEMMs leave ~eps ||G|| asymmetry, which the 1 / (lambda_j - lambda_i) of small eigenvalues
  // would amplify into a loss of orthogonality: with symmetric S, E + E^T = R exactly).  A pair
  // takes the Newton correction when it is separated at this step's resolution,
  //   |lambda_j - lambda_i| > 4 |S_ij| + 2 lambda_max |R_ij|  and  |E_ij| <= 1/100
  // (a per-pair form of Ogita and Aishima's separation bound; the second condition keeps the
  // first-order step inside its domain), else it is orthogonalised only (a cluster: any basis of
  // a numerically degenerate pair is as good, a split across r_need raises the fallback).
  const double floor_num = n * 2.2e-16 * dmx;
  int it = 0, more = 1, unresolved = 0;
  while (it < 4 && more) {
    mx_gemm64<false>(Gs, X, T1, nullptr);  // A X
    __syncthreads();
    mx_gemm64<true>(X, T1, T2, nullptr);  // S = X^T (A X)
    __syncthreads();
    mx_gemm64<true>(X, X, T1, nullptr);  // X^T X = I - R
    __syncthreads();
    if (tid < 64) lamv[tid] = tid < n ? T2[tid * (kMxLd + 1)] / T1[tid * (kMxLd + 1)] : 0.0;
    __syncthreads();
    double ml = fmax(lamv[lane], lamv[lane + 32]);
    for (int o = 16; o; o >>= 1) ml = fmax(ml, __shfl_xor_sync(0xffffffffu, ml, o));
    int lmore = 0, bad = 0;
    for (int e = tid; e < 64 * 64; e += kMxT) {
      const int i = e & 63, j = e >> 6;
      double E = 0.0;
      if (i < n && j < n) {
        if (i == j) {
          E = 0.5 * (1.0 - T1[i * (kMxLd + 1)]);
        } else {
          const double sij = 0.5 * (T2[i + kMxLd * j] + T2[j + kMxLd * i]);
          const double rij = -0.5 * (T1[i + kMxLd * j] + T1[j + kMxLd * i]);
          const double num = fma(lamv[j], rij, sij), den = lamv[j] - lamv[i];
          const double aden = fabs(den);
          if (aden > 4.0 * fabs(sij) + 2.0 * ml * fabs(rij) && fabs(num) <= 0.01 * aden) {
            double rd = rcp_approx_f64(den);  // + two Newton steps: ~1e-16 relative, no division subroutine
            rd = rd * fma(-den, rd, 2.0);
            rd = rd * fma(-den, rd, 2.0);
            E = num * rd;
            // another step unless this correction already leaves ~|E|^2 <= 1e-14 (or sits at the noise floor)
            if (fabs(E) > 1e-7 && fabs(num) > floor_num) lmore = 1;
          } else {
            E = 0.5 * rij;  // a cluster at this step's resolution: orthogonalise only
            // harmful only when the pair straddles the wanted rank with a real gap
            if (aden > 1e-12 * dmx) {
              int ri = 0, rj = 0;
              for (int k = 0; k < n; ++k) {
                ri += (lamv[k] > lamv[i] || (lamv[k] == lamv[i] && k < i));
                rj += (lamv[k] > lamv[j] || (lamv[k] == lamv[j] && k < j));
              }
              if ((ri < r_need) != (rj < r_need)) bad = 1;
            }
          }
        }
      }
      Eb[i + kMxLd * j] = E;
    }
    more = __syncthreads_or(lmore);
    unresolved = __syncthreads_or(bad);
    mx_gemm64<false>(X, Eb, T1, X);  // X + X E
    __syncthreads();
    double *tmp = X;
    X = T1;
    T1 = tmp;
    ++it;
    MXP();
  }
  if (tid == 0 && info) *info = sweeps + 1000 * it;
  if (unresolved || more) {  // a straddling cluster, or no convergence in four steps: fp64 Jacobi
    __syncthreads();
    gram_eig_body<16, 4>(mxs, Ain, n, w, Vout, tol64, 40, info, r_need, refine, status);
    return;
  }
  // eigenvalues: the last step's Rayleigh quotients (second order in the remaining error);
  // eigenvectors: the refined columns, normalised
  for (int k = warp; k < n; k += kMxT / 32) {
    double d = 0.0;
    for (int r = lane; r < n; r += 32) { const double v = X[r + kMxLd * k]; d = fma(v, v, d); }
    d = warp_sum(d);
    if (lane == 0) lc[k] = 1.0 / sqrt(d);
  }
  for (int i = tid; i < n; i += kMxT) {  // rank of each eigenvalue: descending, ties by index
    const double di = lamv[i];
    int rk = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = lamv[j];
      if (j != i && (dj > di || (dj == di && j < i))) ++rk;
    }
    rkv[i] = rk;
    w[rk] = di;
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += kMxT) {  // coalesced: consecutive threads, consecutive rows
    const int i = e / n, r = e - i * n;
    Vout[r + (int64_t)n * rkv[i]] = X[r + kMxLd * i] * lc[i];
  }
  MXP();
#ifdef RTUCKER_EIG_PROF_BUILD
  if (threadIdx.x == 0) {
    printf("[mixed prof] n %d sweeps %d iters %d:", n, sweeps, it);
    for (int i = 1; i < mn_; ++i) printf(" %lld", mt_[i] - mt_[i - 1]);
    printf("\n");
  }
#endif
#undef MXP
}

// ------------------------------------------------------------- CholeskyQR2 ----------
// Thin QR of a well-conditioned tall sketch in 2 x (Gram, Cholesky, Y R^{-1}) passes
// (Yamamoto et al.'s CholeskyQR2; orthogonality ~eps while kappa(Y) < ~1e7).  The Cholesky
// flags ill-conditioning (a pivot d_k < 1e-13 of its original diagonal, i.e. a column that is
// numerically in the span of the previous ones); the Householder kernel then recomputes Q
// (device-side gate, no host sync).  Only the range of Q enters the method (B = Q^T X and
// A = Q U_B, or the oblique factor Q Q_S^{-1}), and both routes span range(Y).
__global__ void __launch_bounds__(256) chol_inv_kernel(const double *__restrict__ G, int n, double *__restrict__ Rinv,
                                                       int *__restrict__ bad) {
  extern __shared__ double cs[];
  double *R = cs;              // n x n, row-major upper (R[k*n + j])
  double *diag0 = R + n * n;   // original diagonal
  __shared__ int sbad;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    R[e] = 0.5 * (G[i + n * j] + G[j + n * i]);
  }
  for (int i = tid; i < n; i += blockDim.x) diag0[i] = G[i + n * i];
  if (tid == 0) sbad = 0;
  __syncthreads();
  // right-looking Cholesky G = R^T R (upper R), 16 x 16 thread tiling of the trailing update
  for (int k = 0; k < n; ++k) {
    const double d = R[k * n + k];
    if (!(d > 1e-13 * diag0[k] && d > 0.0)) {  // uniform
      if (tid == 0) sbad = 1;
      break;
    }
    const double inv = rsqrt(d);
    for (int i = k + 1 + ty; i < n; i += 16)
      for (int j = i + tx; j < n; j += 16) R[i * n + j] -= (R[k * n + i] * inv) * (R[k * n + j] * inv);
    __syncthreads();
    for (int j = k + 1 + tid; j < n; j += blockDim.x) R[k * n + j] *= inv;
    if (tid == 0) R[k * n + k] = d * inv;
    __syncthreads();
  }
  if (sbad) {
    if (tid == 0) *bad = 1;
    return;
  }
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    Rinv[i + n * j] = (j >= i) ? R[e] : 0.0;  // R itself (column-major upper)
  }
}

// Inverse of an upper-triangular n x n matrix (column-major, n <= 256): thread j solves column j
// of R X = I by back substitution (R in shared memory).
__global__ void tri_inv_upper_kernel(const double *__restrict__ Rg, int n, double *__restrict__ X,
                                     const int *__restrict__ bad) {
  if (*bad) return;
  extern __shared__ double rs2[];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) rs2[e] = Rg[e];
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    for (int i = n - 1; i >= 0; --i) {
      double s = (i == j) ? 1.0 : 0.0;
      if (i > j) {
        X[i + (int64_t)n * j] = 0.0;
        continue;
      }
      for (int t = i + 1; t <= j; ++t) s = fma(-rs2[i + n * t], X[t + (int64_t)n * j], s);
      X[i + (int64_t)n * j] = s / rs2[i + n * i];
    }
  }
}

// Q = Y R^{-1} by forward substitution, one row of Y per thread (x R = y), R in shared memory.
__global__ void __launch_bounds__(128) trsm_rows_kernel(const double *__restrict__ Y, int64_t m, int n,
                                                        const double *__restrict__ Rg, double *__restrict__ Q,
                                                        const int *__restrict__ bad) {
  if (*bad) return;
  extern __shared__ double rs[];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) rs[e] = Rg[e];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double x[64];
    for (int j = 0; j < n; ++j) {
      double s = Y[i + m * j];
      for (int t = 0; t < j; ++t) s = fma(-x[t], rs[t + n * j], s);
      x[j] = s / rs[j + n * j];
      Q[i + m * j] = x[j];
    }
  }
}

// ------------------------------------------------- cluster CholeskyQR2 (dense) --------
// Thin QR of a sketch with m <= 8 * 256 rows and n <= 64 columns in ONE cluster kernel.
// Each CTA keeps its row slab in shared memory (column-major, ld = ldY).  Per pass:
//  1. partial Gram Y_slab^T Y_slab on the fp64 tensor cores (mma.m8n8k4, upper 8x8 tiles);
//  2. cluster-wide sum through DSMEM in a fixed CTA order, straight into registers: thread t
//     owns row i = t / 8 of G and the columns j = t % 8 + 8u, u < 8 (every CTA derives the
//     bitwise identical Gram);
//  3. elimination of [G | I] (right-looking Cholesky as Gaussian elimination: step k scales
//     row k by d_k^{-1/2}, publishes it, every row i > k subtracts G_ik d_k^{-1/2} times it)
//     -> the published rows are R (upper, G = R^T R) and E = R^{-T}; one barrier per step;
//  4. slab <- slab R^{-1} = slab E^T on the tensor cores (warp per 8-row block, in place).
// Two passes (CholeskyQR2).  A pivot d_k <= 1e-13 of its original diagonal (or NaN) marks
// the sketch as too ill-conditioned: the kernel flags it and Householder recomputes Q.
constexpr int kCQT = 512;
constexpr int kCQN = 64;                // max columns
constexpr size_t kCQSmem = 225 * 1024;  // dynamic shared memory budget of one CTA

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
// Gram G = Y^T Y of a tall m x n fp64 matrix (column-major, ld m), n <= 8 NA, on the fp64
// tensor cores: warp = a run of rows, fragments F_a = Y[k0 + (lane & 3), 8a + (lane >> 2)]
// serve as both operands of the NA(NA+1)/2 upper 8 x 8 tiles (m8n8k4: A = F_a, B = F_b);
// the 8 warps of a CTA add into shared memory in warp order, CTA partials are summed in block
// order by tall_gram_reduce_kernel (deterministic).
template <int NA>
__global__ void __launch_bounds__(256) tall_gram_kernel(const double *__restrict__ Y, int64_t m, int n,
                                                       int64_t rpw, double *__restrict__ part) {
  constexpr int N8 = 8 * NA, NT = NA * (NA + 1) / 2;
  __shared__ double buf[N8 * N8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < N8 * N8; t += 256) buf[t] = 0.0;
  const int64_t r0 = ((int64_t)blockIdx.x * 8 + warp) * rpw, r1 = min(m, r0 + rpw);
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int kr = lane & 3, cr = lane >> 2;
#pragma unroll 4
  for (int64_t k0 = r0; k0 < r1; k0 += 4) {
    const int64_t row = k0 + kr;
    double f[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const int col = 8 * a + cr;
      f[a] = (row < r1 && col < n) ? Y[(int64_t)col * m + row] : 0.0;
    }
    int t = 0;
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int b = a; b < NA; ++b, ++t) dmma884(acc[t][0], acc[t][1], f[a], f[b]);
  }
  for (int w = 0; w < 8; ++w) {
    __syncthreads();
    if (warp == w) {
      int t = 0;
#pragma unroll
      for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int b = a; b < NA; ++b, ++t) {
          const int i = 8 * a + cr, j = 8 * b + 2 * kr;  // C fragment: row lane >> 2, cols 2 (lane & 3) + {0, 1}
          buf[i * N8 + j] += acc[t][0];
          buf[i * N8 + j + 1] += acc[t][1];
        }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < N8 * N8; t += 256) part[(int64_t)blockIdx.x * N8 * N8 + t] = buf[t];
}
// G (n x n, column-major, both triangles) = sum over the CTA partials: one CTA per entry, a fixed
// partition of the partials over its threads and a fixed-shape tree (deterministic)
__global__ void tall_gram_reduce_kernel(const double *__restrict__ part, int nblk, int n, int n8,
                                        double *__restrict__ G) {
  __shared__ double sr[4];
  const int e = blockIdx.x;
  int i = e % n, j = e / n;
  if (i > j) { const int t = i; i = j; j = t; }  // upper tile entry (i <= j)
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += 128) s += part[(int64_t)b * n8 * n8 + i * n8 + j];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sr[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) G[e] = (sr[0] + sr[1]) + (sr[2] + sr[3]);
}

void tall_gram(Ctx &c, const double *Y, int64_t m, int n, double *G) {
  RT_REQUIRE(n >= 1 && n <= 64, "tall_gram: 1 <= n <= 64");
  const int64_t rpw = std::max<int64_t>(64, ((m + (int64_t)c.num_sms * 64 - 1) / ((int64_t)c.num_sms * 64) + 3) / 4 * 4);
  const int nblk = (int)((m + 8 * rpw - 1) / (8 * rpw));
  const int na = (n + 7) / 8, n8 = 8 * (na <= 2 ? 2 : (na <= 4 ? 4 : 8));
  DevBuf<double> part(c, (size_t)nblk * n8 * n8);
  if (na <= 2) RT_LAUNCH(c, tall_gram_kernel<2>, nblk, 256, 0, Y, m, n, rpw, part.p);
  else if (na <= 4) RT_LAUNCH(c, tall_gram_kernel<4>, nblk, 256, 0, Y, m, n, rpw, part.p);
  else RT_LAUNCH(c, tall_gram_kernel<8>, nblk, 256, 0, Y, m, n, rpw, part.p);
  RT_LAUNCH(c, tall_gram_reduce_kernel, n * n, 128, 0, part.p, nblk, n, n8, G);
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kCQT, 1) cholqr2_cluster_kernel(const double *__restrict__ Y, int64_t m, int n,
                                                                  int rows, int ldY, int ldG, int ldE,
                                                                  double *__restrict__ Q, int *__restrict__ bad) {
  extern __shared__ __align__(16) double cq[];
#ifdef RTUCKER_CQ_PROF_BUILD
  long long pt[12];
  int np_ = 0;
#define CQP() if (threadIdx.x == 0 && np_ < 12) pt[np_++] = clock64()
#else
#define CQP()
#endif
  CQP();
  cg::cluster_group cl = cg::this_cluster();
  const int ncta = (int)cl.num_blocks();
  const int me = (int)cl.block_rank();
  const int64_t r0 = (int64_t)me * rows;
  const int64_t left_ = m - r0;
  const int nloc = left_ <= 0 ? 0 : (left_ < rows ? (int)left_ : rows);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n8 = (n + 7) & ~7, nbk = n8 >> 3;
  double *Yl = cq;                 // ldY x n8 slab (column-major), zero padded
  double *Gp = Yl + ldY * n8;      // n8 x ldG partial Gram (row-major)
  double *E = Gp + n8 * ldG;       // n8 x ldE, row k = row k of R^{-T} (column k of R^{-1})
  double *pv = E + n8 * ldE;       // [2 buffers][R row | E row][kCQN]
  double *d0 = pv + 4 * kCQN;      // original diagonal of the pass's Gram
  __shared__ int sbad;
  for (int e = tid; e < ldY * n8; e += kCQT) {
    const int i = e % ldY, c = e / ldY;
    Yl[e] = (i < nloc && c < n) ? Y[r0 + i + m * c] : 0.0;
  }
  if (tid == 0) sbad = 0;
  CQP();
  const int ri = tid >> 3, g = tid & 7;  // elimination ownership: row ri, columns g + 8u
  const unsigned gmask = 0xFFu << (8 * (ri & 3));
  const int kend = (nloc + 3) & ~3;      // slab rows past nloc are zero
  const int ntiles = nbk * (nbk + 1) / 2;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) cluster_wait();  // every CTA has read the pass-0 partial Grams
    // ---- 1. partial Gram, upper tiles (a <= b), mirrored
    for (int tile = warp; tile < ntiles; tile += kCQT / 32) {
      int a = 0, rem = tile;
      while (rem >= nbk - a) { rem -= nbk - a; ++a; }
      const int b = a + rem;
      const double *pa = Yl + (size_t)ldY * (8 * a + (lane >> 2)) + (lane & 3);
      const double *pb = Yl + (size_t)ldY * (8 * b + (lane >> 2)) + (lane & 3);
      double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
      int k0 = 0;
      for (; k0 + 8 <= kend; k0 += 8) {  // two independent accumulator chains
        dmma884(c0, c1, pa[k0], pb[k0]);
        dmma884(e0, e1, pa[k0 + 4], pb[k0 + 4]);
      }
      if (k0 < kend) dmma884(c0, c1, pa[k0], pb[k0]);
      c0 += e0; c1 += e1;
      const int gi = 8 * a + (lane >> 2), gj = 8 * b + 2 * (lane & 3);
      Gp[gi * ldG + gj] = c0; Gp[gi * ldG + gj + 1] = c1;
      if (a != b) { Gp[gj * ldG + gi] = c0; Gp[(gj + 1) * ldG + gi] = c1; }
    }
    CQP();
    cluster_arrive();
    cluster_wait();
    CQP();
    // ---- 2. cluster sum into registers (fixed CTA order)
    double gr[8], er[8], diag = 0.0;  // diag: running G[ri][ri], kept by its owner (g == ri % 8)
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = g + 8 * u;
      double s = 0.0;
      if (ri < n && j < n)
        for (int q = 0; q < ncta; ++q) s += cl.map_shared_rank(Gp, q)[ri * ldG + j];
      gr[u] = s;
      er[u] = (j == ri) ? 1.0 : 0.0;
      if (j == ri && ri < n) { d0[ri] = s; diag = s; }
    }
    cluster_arrive();  // matched by the wait before the next Gram (or before exit)
    __syncthreads();
    CQP();
    // ---- 3. elimination of [G | I]
    for (int k = 0; k < n; ++k) {
      double *pR = pv + (k & 1) * 2 * kCQN, *pE = pR + kCQN;
      if (ri == k) {  // the 8 owners of row k (one lane group of warp k / 4)
        const double dk = __shfl_sync(gmask, diag, k & 7, 8);
        if (g == 0 && !(dk > 1e-13 * d0[k])) sbad = 1;
        const double inv = rsqrt(dk);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = g + 8 * u;
          pR[j] = (j >= k) ? gr[u] * inv : 0.0;
          const double ev = er[u] * inv;
          pE[j] = ev;
          if (j < n8) E[k * ldE + j] = ev;
        }
      }
      __syncthreads();
      if (ri > k && ri < n) {
        const double f = pR[ri];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = g + 8 * u;
          gr[u] = fma(-f, pR[j], gr[u]);
          er[u] = fma(-f, pE[j], er[u]);
        }
        diag = fma(-f, f, diag);  // == gr[ri >> 3] in the owner of G[ri][ri] (same operands)
      }
    }
    // rows n..n8-1 of E (padding) stay as written by a previous pass or zero them once
    for (int e = n * ldE + tid; e < n8 * ldE; e += kCQT) E[e] = 0.0;
    __syncthreads();
    CQP();
    // ---- 4. slab <- slab E^T (W = R^{-1} upper: W[t][j] = E[j][t], only t <= j contributes)
    for (int rb = warp; 8 * rb < nloc; rb += kCQT / 32) {
      double acc[8][2];
#pragma unroll
      for (int cb = 0; cb < 8; ++cb) acc[cb][0] = acc[cb][1] = 0.0;
      const double *pa = Yl + 8 * rb + (lane >> 2) + (size_t)ldY * (lane & 3);
#pragma unroll
      for (int tb = 0; tb < 8; ++tb) {
        if (tb < nbk) {
#pragma unroll
          for (int kh = 0; kh < 2; ++kh) {
            const int t0 = 8 * tb + 4 * kh;
            const double av = pa[(size_t)ldY * t0];
#pragma unroll
            for (int cb = tb; cb < 8; ++cb)
              if (cb < nbk) dmma884(acc[cb][0], acc[cb][1], av, E[(8 * cb + (lane >> 2)) * ldE + t0 + (lane & 3)]);
          }
        }
      }
      __syncwarp();
      const int row = 8 * rb + (lane >> 2);
#pragma unroll
      for (int cb = 0; cb < 8; ++cb)
        if (cb < nbk) {
          const int col = 8 * cb + 2 * (lane & 3);
          Yl[row + (size_t)ldY * col] = acc[cb][0];
          Yl[row + (size_t)ldY * (col + 1)] = acc[cb][1];
        }
    }
    __syncthreads();
  }
  cluster_wait();  // no CTA leaves while others may still read its partial Gram
  CQP();
#ifdef RTUCKER_CQ_PROF_BUILD
  if (threadIdx.x == 0 && me == 0) {
    printf("[cq prof] m %lld n %d:", (long long)m, n);
    for (int i = 1; i < np_; ++i) printf(" %lld", pt[i] - pt[i - 1]);
    printf("\n");
  }
#endif
  if (sbad) {
    if (me == 0 && tid == 0) *bad = 1;
    return;
  }
  for (int e = tid; e < nloc * n; e += kCQT) {
    const int i = e % nloc, c = e / nloc;
    Q[r0 + i + m * c] = Yl[i + (size_t)ldY * c];
  }
}

// ------------------------------------- cluster CholeskyQR2, blocked Cholesky (dense) --------
// Same data flow as cholqr2_cluster_kernel (row slabs in the CTAs of one cluster, partial Grams
// on the fp64 tensor cores, fixed-order DSMEM sum so every CTA holds the bit-identical Gram),
// but the factorisation is blocked in 8 x 8 tiles instead of 60 single-pivot elimination steps
// with a CTA barrier each:
//   for each diagonal block kb:  warp 0 factors the 8 x 8 block (8 shuffle-broadcast pivots)
//                                and inverts its triangle (D_kb = R_kb,kb^{-1}, one column per lane);
//                                the panel R_kb,jb = D_kb^T G_kb,jb and the trailing update
//                                G_ib,jb -= R_kb,ib^T R_kb,jb run on the fp64 tensor cores, one
//                                block per warp (3 CTA barriers per block row, 24 in all);
//   slab <- slab R^{-1} by a blocked triangular solve on the tensor cores, one 8-row block per
//   warp: X_kb = (Y_kb - sum_{jb < kb} X_jb R_jb,kb) D_kb.
// A pivot <= 1e-13 of its original diagonal (or NaN) flags the sketch as too ill-conditioned
// and the Householder kernel recomputes Q (device-side gate), as before.
constexpr int kBQT = 512;
__device__ __forceinline__ void mma_blk8(double &c0, double &c1, const double *A, int lda_r, int lda_c,
                                         const double *B, int ldb_r, int ldb_c, int lane) {
  // C(8x8) += A(8x8) B(8x8): A(i, k) = A[i * lda_r + k * lda_c], B(k, j) = B[k * ldb_r + j * ldb_c]
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += 4) {
    const int kk = k0 + (lane & 3), r = lane >> 2;
    dmma884(c0, c1, A[r * lda_r + kk * lda_c], B[kk * ldb_r + r * ldb_c]);
  }
}

__global__ void __launch_bounds__(kBQT, 1) cholqr2_blk_kernel(const double *__restrict__ Y, int64_t m, int n,
                                                              int rows, int ldY, int ldG, double *__restrict__ Q,
                                                              int *__restrict__ bad, double orth_tol) {
  extern __shared__ __align__(16) double bq[];
  cg::cluster_group cl = cg::this_cluster();
  const int ncta = (int)cl.num_blocks();
  const int me = (int)cl.block_rank();
  const int64_t r0 = (int64_t)me * rows;
  const int64_t left_ = m - r0;
  const int nloc = left_ <= 0 ? 0 : (left_ < rows ? (int)left_ : rows);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kW = kBQT / 32;
  const int n8 = (n + 7) & ~7, nbk = n8 >> 3;
  double *Yl = bq;                 // ldY x n8 slab (column-major), zero padded
  double *Gp = Yl + ldY * n8;      // n8 x ldG partial Gram (row-major)
  double *G = Gp + n8 * ldG;       // n8 x ldG summed Gram, then R (upper) in place
  double *D = G + n8 * ldG;        // nbk x 64: D_kb (8 x 8 row-major)
  double *tmp = D + 8 * 64;        // kW x 64 scratch (one 8 x 8 tile per warp)
  double *d0 = tmp + kW * 64;      // 64: original diagonal
  __shared__ int sbad;
  for (int e = tid; e < ldY * n8; e += kBQT) {
    const int i = e % ldY, c = e / ldY;
    Yl[e] = (i < nloc && c < n) ? Y[r0 + i + m * c] : 0.0;
  }
  if (tid == 0) sbad = 0;
  const int kend = (nloc + 3) & ~3;
  const int ntiles = nbk * (nbk + 1) / 2;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) cluster_wait();  // every CTA has read the pass-0 partial Grams
    // ---- 1. partial Gram, upper tiles (a <= b), mirrored
    for (int tile = warp; tile < ntiles; tile += kW) {
      int a = 0, rem = tile;
      while (rem >= nbk - a) { rem -= nbk - a; ++a; }
      const int b = a + rem;
      const double *pa = Yl + (size_t)ldY * (8 * a + (lane >> 2)) + (lane & 3);
      const double *pb = Yl + (size_t)ldY * (8 * b + (lane >> 2)) + (lane & 3);
      double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
      int k0 = 0;
      for (; k0 + 8 <= kend; k0 += 8) {
        dmma884(c0, c1, pa[k0], pb[k0]);
        dmma884(e0, e1, pa[k0 + 4], pb[k0 + 4]);
      }
      if (k0 < kend) dmma884(c0, c1, pa[k0], pb[k0]);
      c0 += e0; c1 += e1;
      const int gi = 8 * a + (lane >> 2), gj = 8 * b + 2 * (lane & 3);
      Gp[gi * ldG + gj] = c0; Gp[gi * ldG + gj + 1] = c1;
      if (a != b) { Gp[gj * ldG + gi] = c0; Gp[(gj + 1) * ldG + gi] = c1; }
    }
    cluster_arrive();
    cluster_wait();
    // ---- 2. cluster sum (fixed CTA order) into G
    int far = 0;  // pass 1: an entry of Q^T Q - I above orth_tol
    for (int e = tid; e < n8 * n8; e += kBQT) {
      const int i = e / n8, j = e % n8;
      double sum = 0.0;
      for (int q = 0; q < ncta; ++q) sum += cl.map_shared_rank(Gp, q)[i * ldG + j];
      G[i * ldG + j] = sum;
      if (i == j) d0[i] = sum;
      if (i < n && j < n) far |= !(fabs(sum - (i == j ? 1.0 : 0.0)) <= orth_tol);
    }
    cluster_arrive();  // matched by the wait before the next Gram (or before exit)
    // the Gram is bit-identical in every CTA of the cluster, so every CTA takes the same decision
    if (__syncthreads_or(far) == 0 && pass == 1) break;  // the first pass is orthonormal enough
    // ---- 3. blocked Cholesky G = R^T R (upper R in place) with D_kb = R_kb,kb^{-1}
    for (int kb = 0; kb < nbk; ++kb) {
      if (warp == 0) {
        // (a) 8 x 8 diagonal block: lane holds entries e = lane, lane + 32 (i = e >> 3, j = e & 7)
        double bv[2];
        int bi[2], bj[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = lane + 32 * h;
          bi[h] = e >> 3;
          bj[h] = e & 7;
          bv[h] = G[(8 * kb + bi[h]) * ldG + 8 * kb + bj[h]];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int gk = 8 * kb + k;
          const int ek = 9 * k;  // entry (k, k)
          double piv = __shfl_sync(0xffffffffu, bv[ek >> 5], ek & 31);
          if (gk >= n) piv = 1.0;  // padding pivot: identity
          else if (!(piv > 1e-13 * d0[gk])) {
            if (lane == 0) sbad = 1;
            piv = 1.0;
          }
          double rinv;  // piv^{-1/2}: approximate rsqrt + two Newton steps (no slow-path subroutine)
          asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rinv) : "d"(piv));
          rinv = rinv * fma(-0.5 * piv * rinv, rinv, 1.5);
          rinv = rinv * fma(-0.5 * piv * rinv, rinv, 1.5);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (bi[h] == k && bj[h] > k) bv[h] *= rinv;
            if (bi[h] == k && bj[h] == k) bv[h] = piv * rinv;
          }
          // rank-1 update of the trailing entries (i, j), k < i <= j: R_ki R_kj from row k
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int ea = 8 * k + bi[h], eb = 8 * k + bj[h];
            const double rki = __shfl_sync(0xffffffffu, bv[ea >> 5], ea & 31);
            const double rkj = __shfl_sync(0xffffffffu, bv[eb >> 5], eb & 31);
            if (bi[h] > k && bj[h] >= bi[h]) bv[h] = fma(-rki, rkj, bv[h]);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double &g = G[(8 * kb + bi[h]) * ldG + 8 * kb + bj[h]];
          g = bj[h] >= bi[h] ? bv[h] : 0.0;
        }
        __syncwarp();
        // (b) D = R_kb,kb^{-1} (upper): lane j < 8 solves column j by back substitution
        double *Dk = D + 64 * kb;
        if (lane < 8) {
          const int j = lane;
          const double *Rb = G + (8 * kb) * ldG + 8 * kb;
          double x[8];
#pragma unroll
          for (int i = 7; i >= 0; --i) {
            double s2 = (i == j) ? 1.0 : 0.0;
#pragma unroll
            for (int t = i + 1; t < 8; ++t) s2 = fma(-Rb[i * ldG + t], x[t], s2);
            const double di = Rb[i * ldG + i];
            double rd = rcp_approx_f64(di);  // 1 / R_ii: approximate reciprocal + two Newton steps
            rd = rd * fma(-di, rd, 2.0);
            rd = rd * fma(-di, rd, 2.0);
            x[i] = (i <= j) ? s2 * rd : 0.0;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) Dk[i * 8 + j] = x[i];
        }
      }
      __syncthreads();
      // (c) panel: R_kb,jb = D^T G_kb,jb for jb > kb (one block per warp)
      const double *Dk = D + 64 * kb;
      for (int jb = kb + 1 + warp; jb < nbk; jb += kW) {
        double c0 = 0.0, c1 = 0.0;
        // A(i, k) = D^T(i, k) = D[k][i];  B(k, j) = G[8kb + k][8jb + j]
        mma_blk8(c0, c1, Dk, 1, 8, G + (8 * kb) * ldG + 8 * jb, ldG, 1, lane);
        __syncwarp();
        const int r = lane >> 2, cc = 2 * (lane & 3);
        G[(8 * kb + r) * ldG + 8 * jb + cc] = c0;
        G[(8 * kb + r) * ldG + 8 * jb + cc + 1] = c1;
      }
      __syncthreads();
      // (d) trailing update G_ib,jb -= R_kb,ib^T R_kb,jb for kb < ib <= jb
      const int rem = nbk - kb - 1;
      for (int t = warp; t < rem * (rem + 1) / 2; t += kW) {
        int ib = 0, r2 = t;
        while (r2 >= rem - ib) { r2 -= rem - ib; ++ib; }
        const int jb = ib + r2;
        ib += kb + 1;
        const int jj = jb + kb + 1;
        const int r = lane >> 2, cc = 2 * (lane & 3);
        double c0 = G[(8 * ib + r) * ldG + 8 * jj + cc], c1 = G[(8 * ib + r) * ldG + 8 * jj + cc + 1];
        // A(i, k) = -R_kb,ib^T(i, k) = -G[8kb + k][8ib + i] (negated via the B operand sign below)
        double n0 = 0.0, n1 = 0.0;
        mma_blk8(n0, n1, G + (8 * kb) * ldG + 8 * ib, 1, ldG, G + (8 * kb) * ldG + 8 * jj, ldG, 1, lane);
        G[(8 * ib + r) * ldG + 8 * jj + cc] = c0 - n0;
        G[(8 * ib + r) * ldG + 8 * jj + cc + 1] = c1 - n1;
      }
      __syncthreads();
    }
    // ---- 4. slab <- slab R^{-1}: X_kb = (Y_kb - sum_{jb<kb} X_jb R_jb,kb) D_kb per 8-row block
    double *tw = tmp + 64 * warp;
    for (int rb = warp; 8 * rb < nloc; rb += kW) {
      double *yr = Yl + 8 * rb;  // rows 8rb.., column c at yr[ldY * c]
      for (int kb = 0; kb < nbk; ++kb) {
        const int r = lane >> 2, cc = 2 * (lane & 3);
        double c0 = yr[r + (size_t)ldY * (8 * kb + cc)], c1 = yr[r + (size_t)ldY * (8 * kb + cc + 1)];
        for (int jb = 0; jb < kb; ++jb) {
          double n0 = 0.0, n1 = 0.0;
          // A(i, k) = X[8rb + i][8jb + k];  B(k, j) = R[8jb + k][8kb + j]
          mma_blk8(n0, n1, yr + (size_t)ldY * 8 * jb, 1, ldY, G + (8 * jb) * ldG + 8 * kb, ldG, 1, lane);
          c0 -= n0;
          c1 -= n1;
        }
        tw[r * 8 + cc] = c0;
        tw[r * 8 + cc + 1] = c1;
        __syncwarp();
        double x0 = 0.0, x1 = 0.0;
        mma_blk8(x0, x1, tw, 8, 1, D + 64 * kb, 8, 1, lane);  // (Y - ...) D_kb
        __syncwarp();
        yr[r + (size_t)ldY * (8 * kb + cc)] = x0;
        yr[r + (size_t)ldY * (8 * kb + cc + 1)] = x1;
        __syncwarp();
      }
    }
    __syncthreads();
  }
  cluster_wait();  // no CTA leaves while others may still read its partial Gram
  if (sbad) {
    if (me == 0 && tid == 0) *bad = 1;
    return;
  }
  for (int e = tid; e < nloc * n; e += kBQT) {
    const int i = e % nloc, c = e / nloc;
    Q[r0 + i + m * c] = Yl[i + (size_t)ldY * c];
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

// Alg 1 line 5 + reading R4b + the residual of the truncation (ell, r <= 64), two launches:
//   factor_gemm_kernel: CTA b forms rows 16b .. 16b + 15 of A = Q U(:, 1:r) from shared-memory
//     copies of its Q slab and of U (fixed summation order over the ell columns of Q) and
//     records, per column, the largest |A_ij| of its rows and its first row index;
//   factor_sign_kernel: CTA j reduces those partials in block order (largest value, smallest
//     row on ties), flips A(:, j) and U(:, j) when that entry is negative, and CTA 0 writes
//     ||G||^2 - sum_{i<r} w_i (the truncated mode's residual, P:133 / Alg 3).
// (One CTA per column reading all of Q measured 61 us: dependent L2 loads per thread.)
constexpr int kFeRows = 16;
__global__ void __launch_bounds__(256) factor_gemm_kernel(const double *__restrict__ Q, int64_t m, int ell,
                                                          const double *__restrict__ U, int r, double *__restrict__ A,
                                                          double *__restrict__ pmax, int *__restrict__ pidx) {
  __shared__ double us[64][64], qs[kFeRows][64];  // (row reads broadcast, column reads consecutive)
  __shared__ double bm[4][64];
  __shared__ int bi[4][64];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kFeRows;
  for (int e = tid; e < ell * r; e += 256) us[e % ell][e / ell] = U[(e % ell) + (int64_t)ell * (e / ell)];
  for (int e = tid; e < kFeRows * ell; e += 256) {
    const int i = e % kFeRows, t = e / kFeRows;
    qs[i][t] = r0 + i < m ? Q[r0 + i + m * t] : 0.0;
  }
  __syncthreads();
  const int j = tid & 63, g = tid >> 6;
  double best = -1.0;
  int besti = 0;
  if (j < r) {
    for (int k = 0; k < kFeRows / 4; ++k) {
      const int i = g + 4 * k;
      double acc = 0.0;
      for (int t = 0; t < ell; ++t) acc = fma(qs[i][t], us[t][j], acc);
      if (r0 + i < m) {
        A[r0 + i + m * j] = acc;
        const double v = fabs(acc);
        if (v > best) { best = v; besti = (int)(r0 + i); }  // rows ascending: first index kept on ties
      }
    }
  }
  bm[g][j] = best;
  bi[g][j] = besti;
  __syncthreads();
  if (g == 0 && j < r) {
    double b = bm[0][j];
    int ii = bi[0][j];
    for (int q = 1; q < 4; ++q)
      if (bm[q][j] > b || (bm[q][j] == b && bi[q][j] < ii)) { b = bm[q][j]; ii = bi[q][j]; }
    pmax[(int64_t)blockIdx.x * r + j] = b;
    pidx[(int64_t)blockIdx.x * r + j] = ii;
  }
}

__global__ void __launch_bounds__(32) factor_sign_kernel(double *__restrict__ A, int64_t m, int ell,
                                                         double *__restrict__ U, int r, int nblk,
                                                         const double *__restrict__ pmax, const int *__restrict__ pidx,
                                                         const double *__restrict__ w, const double *__restrict__ nsq,
                                                         double *__restrict__ res) {
  const int j = blockIdx.x, lane = threadIdx.x;
  if (res && j == 0 && lane == 0) {
    double s = 0.0;
    for (int i = 0; i < r; ++i) s += w[i];
    *res = *nsq - s;
  }
  double best = -1.0;
  int bi = 0;
  for (int b = lane; b < nblk; b += 32) {  // blocks ascending per lane
    const double v = pmax[(int64_t)b * r + j];
    const int ii = pidx[(int64_t)b * r + j];
    if (v > best) { best = v; bi = ii; }
  }
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  double *a = A + m * j;
  if (a[bi] >= 0.0) return;
  for (int64_t i = lane; i < m; i += 32) a[i] = -a[i];
  for (int t = lane; t < ell; t += 32) U[t + (int64_t)ell * j] = -U[t + (int64_t)ell * j];
}

}  // namespace

void canonical_signs(Ctx &c, double *A, int64_t m, int r, double *U, int64_t ldu, int ell) {
  RT_LAUNCH(c, canonical_signs_kernel, r, 256, 0, A, m, U, ldu, ell);
}

void factor_epilogue(Ctx &c, const double *Q, int64_t m, int ell, double *U, int r, double *A, const double *w,
                     const double *normsq, double *residual) {
  if (ell > 64) {  // the adaptive truncation's large bases: tensor-core GEMM + separate passes
    gemm_small(c, false, Q, m, U, ell, A, m, m, r, ell);
    canonical_signs(c, A, m, r, U, ell, ell);
    if (w) residual_from_eigs(c, w, r, normsq, residual);
    return;
  }
  const int nblk = (int)((m + kFeRows - 1) / kFeRows);
  DevBuf<double> pmax(c, (size_t)nblk * r);
  DevBuf<int> pidx(c, (size_t)nblk * r);
  RT_LAUNCH(c, factor_gemm_kernel, nblk, 256, 0, Q, m, ell, (const double *)U, r, A, pmax.p, pidx.p);
  RT_LAUNCH(c, factor_sign_kernel, r, 32, 0, A, m, ell, U, r, nblk, (const double *)pmax.p, (const int *)pidx.p, w,
            normsq, w ? residual : nullptr);
}

void householder_qr(Ctx &c, const double *Y, int64_t m, int n, double *Q, const int *gate) {
  RT_REQUIRE(m >= n && n >= 1, "qr: need m >= n >= 1");
  RT_REQUIRE(n <= 4096, "qr: more than 4096 columns is not supported");
  // smallest cluster whose row slabs fit in shared memory (RTUCKER_QR_NCTA forces a size,
  // for testing the multi-CTA path on small inputs)
  static const int forced = [] {
    const char *e = RT_EXP_GETENV("RTUCKER_QR_NCTA");
    return e ? atoi(e) : 0;
  }();
  for (int ncta : {1, 2, 4, 8, 16}) {
    if (n > kMaxN) break;
    if (forced > 0 && ncta != forced) continue;
    const int rows = (int)((m + ncta - 1) / ncta);
    if (forced == 0 && rows > 256 && ncta < 16) continue;  // keep per-CTA slabs short (latency)
    const size_t smem = sizeof(double) * ((size_t)2 * rows * n + (7 + 2 * kMaxCTA) * kMaxN);
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
    smem_attr(qr_cluster_kernel, smem);
    if (ncta > 8)
      RT_CUDA(cudaFuncSetAttribute(qr_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RT_CUDA(cudaLaunchKernelEx(&cfg, qr_cluster_kernel, Y, m, n, rows, Q, gate));
    c.launches++;
    return;
  }
  DevBuf<double> W(c, (size_t)m * n);
  RT_CUDA(cudaMemcpyAsync(W.p, Y, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, c.stream));
  const size_t smem = sizeof(double) * 2 * (size_t)n;
  if (smem > 48 * 1024)
    smem_attr(qr_global_kernel, smem);
  RT_LAUNCH(c, qr_global_kernel, 1, kQRG, smem, W.p, m, n, Q, gate);
}

void gram_eig(Ctx &c, const double *A, int n, double *w, double *V, int *sweeps, int r_need, bool rel_acc) {
  const int np = n + (n & 1);
  // fp32 data (rel_acc = false): Householder tridiagonalisation + multisection + twisted
  // eigenvectors (trideig.cu; one CTA for n <= 64, the whole GPU above), eigenvectors to
  // ~eps lambda_1 / gap, ample for the fp32 criteria.  fp64 data: the preconditioned Jacobi below
  // (pivoted Cholesky + one-sided Jacobi on the factor: ~eps sigma_1 / (sigma gap)), which the
  // 1e-10 fp64 projector criterion of graded spectra needs (SURVEY c.4)
  // n <= 64 stays on the register Jacobi: the one-CTA tridiagonal kernel measured slower at
  // n = 60 (362 vs 300 us: fp64-issue-bound Sturm rounds and 58 barrier-bound Householder steps,
  // DESIGN §12); it remains available in experiments builds (RTUCKER_EIG_TRID_CTA)
  if (!rel_acc && (np > 64 || RT_EXP_GETENV("RTUCKER_EIG_TRID_CTA")) && trid_eig(c, A, n, w, V, sweeps)) return;
  if (np > 64) return sym_eig(c, A, n, w, V, sweeps);
  // 4 lanes per column slot (blocks of 8 columns, nb / 2 busy warps).  RTUCKER_EIG_LPS8 (n > 32):
  // 8 lanes (blocks of 4, all 8 warps busy, 8 rows per lane) measured no faster at n = 60
  // (405 vs 412 us): a round is bound by its dependent latency chain (reductions, angle),
  // not by the per-lane work.
  static const bool lps8 = RT_EXP_GETENV("RTUCKER_EIG_LPS8") != nullptr;
  const int lps = (np > 32 && lps8) ? 8 : 4, spw = 32 / lps;
  const int nb = ((n + 2 * spw - 1) / (2 * spw)) * 2, ncol = spw * nb;
  const int kv = (np + lps - 1) / lps <= 4 ? 4 : ((np + lps - 1) / lps <= 8 ? 8 : 16);
  const int ldm = lps * kv + lps;
  const size_t need = sizeof(double) * ((size_t)np * np + (size_t)ldm * ncol + ncol + np) + sizeof(int) * np + 64;
  DevBuf<int> refine(c, 1);
  const double tol = 3e-15 * std::sqrt((double)n);
  const int rn = std::max(1, std::min(r_need, n));
  // fp32 data, 32 < n <= 64: the mixed-precision solver; the fp64 Jacobi below runs only when it
  // raises its fallback flag (rank-deficient Gram, unresolved pair across r_need)
  static const bool no_mixed = RT_EXP_GETENV("RTUCKER_EIG_NO_MIXED") != nullptr;
  if (!rel_acc && n > 32 && !no_mixed && lps == 4 && kv == 16) {
    // the fp64 Jacobi runs inside the same launch when the solver falls back
    smem_attr(gram_eig_mixed_kernel, kMxSmem);
    RT_LAUNCH(c, gram_eig_mixed_kernel, 1, kMxT, kMxSmem, A, n, w, V, sweeps, rn, 15, tol, refine.p, c.status);
    sym_eig(c, A, n, w, V, nullptr, refine.p);  // no-op unless the fallback's gate asks for it
    return;
  }
#define RT_GE(KV, L)                                                                                      \
  smem_attr(gram_eig_kernel<KV, L>, need);                                                                 \
  RT_LAUNCH(c, (gram_eig_kernel<KV, L>), 1, kGramT, need, A, n, w, V, tol, 40, sweeps, rn, refine.p, c.status)
  if (lps == 8) {
    RT_GE(8, 8);
  } else if (kv == 4) {
    RT_GE(4, 4);
  } else if (kv == 8) {
    RT_GE(8, 4);
  } else {
    RT_GE(16, 4);
  }
#undef RT_GE
  sym_eig(c, A, n, w, V, nullptr, refine.p);  // no-op unless the gate asks for it
}

void chol_rinv(Ctx &c, const double *G, int n, double *Rinv, int *bad) {
  RT_REQUIRE(n >= 1 && n <= 256, "chol_rinv: 1 <= n <= 256");
  DevBuf<double> R(c, (size_t)n * n);
  const size_t csm = sizeof(double) * ((size_t)n * n + n);
  smem_attr(chol_inv_kernel, csm);
  RT_LAUNCH(c, chol_inv_kernel, 1, 256, csm, G, n, R.p, bad);
  smem_attr(tri_inv_upper_kernel, sizeof(double) * n * n);
  RT_LAUNCH(c, tri_inv_upper_kernel, 1, 256, sizeof(double) * n * n, R.p, n, Rinv, bad);
}

void thin_qr(Ctx &c, const double *Y, int64_t m, int n, double *Q, double orth_tol) {
  RT_REQUIRE(m >= n && n >= 1, "qr: need m >= n >= 1");
  if (n > 64) return householder_qr(c, Y, m, n, Q, nullptr);
  static const bool no_chol = RT_EXP_GETENV("RTUCKER_QR_HOUSEHOLDER") != nullptr;
  if (no_chol) return householder_qr(c, Y, m, n, Q, nullptr);
  DevBuf<int> bad(c, 1);
  bad.zero();
  if (m <= 8 * 256) {
    // one portable cluster: CholeskyQR2 in shared memory (row slabs of <= 256 rows per CTA)
    int ncta = 1;
    while (ncta < 8 && (m + ncta - 1) / ncta > 256) ncta *= 2;
    const int rows = (int)((m + ncta - 1) / ncta);
    const int n8 = (n + 7) & ~7;
    const int ldY = ((rows + 7) / 8 * 8 + 11) / 16 * 16 + 4;  // >= rows rounded to 8, = 4 mod 16
    const int ldG = (n8 + 15) / 16 * 16 + 8, ldE = (n8 + 15) / 16 * 16 + 4;
    const bool blk = !RT_EXP_GETENV("RTUCKER_QR_ELIM");  // blocked Cholesky (default) or the elimination kernel
    const size_t smem = blk ? sizeof(double) * ((size_t)ldY * n8 + 2 * (size_t)n8 * ldG + 8 * 64 + (kBQT / 32) * 64 + 64)
                            : sizeof(double) * ((size_t)ldY * n8 + (size_t)n8 * ldG + (size_t)n8 * ldE + 4 * kCQN + kCQN);
    RT_REQUIRE(smem <= kCQSmem, "qr: CholeskyQR2 slab does not fit shared memory");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(blk ? kBQT : kCQT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ncta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (blk) {
      smem_attr(cholqr2_blk_kernel, smem);
      RT_CUDA(cudaLaunchKernelEx(&cfg, cholqr2_blk_kernel, Y, m, n, rows, ldY, ldG, Q, bad.p, orth_tol));
    } else {
      smem_attr(cholqr2_cluster_kernel, smem);
      RT_CUDA(cudaLaunchKernelEx(&cfg, cholqr2_cluster_kernel, Y, m, n, rows, ldY, ldG, ldE, Q, bad.p));
    }
    c.launches++;
  } else {
    // tall sketches (sparse modes, I_n ~ 1e5): CholeskyQR2 over the whole grid
    DevBuf<double> G(c, (size_t)n * n), Ri(c, (size_t)n * n), Q1(c, (size_t)m * n);
    const size_t csm = sizeof(double) * ((size_t)n * n + n);
    smem_attr(chol_inv_kernel, csm);
    const double *src = Y;
    for (int pass = 0; pass < 2; ++pass) {
      double *dst = pass == 0 ? Q1.p : Q;
      tall_gram(c, src, m, n, G.p);
      RT_LAUNCH(c, chol_inv_kernel, 1, 256, csm, G.p, n, Ri.p, bad.p);
      RT_LAUNCH(c, trsm_rows_kernel, std::max(1, std::min(c.num_sms * 8, ceil_div(m, 128))), 128,
                sizeof(double) * n * n, src, m, n, Ri.p, dst, bad.p);
      src = dst;
    }
  }
  householder_qr(c, Y, m, n, Q, bad.p);  // runs only when a Cholesky pass flagged
}

void sym_eig(Ctx &c, const double *A, int n, double *w, double *V, int *sweeps, const int *gate) {
  const int np = n + (n & 1);
  const size_t tab = sizeof(short2) * (size_t)(np - 1) * (np / 2) + 16;
  const size_t need = sizeof(double) * (2 * (size_t)np * np + np) + tab;
  const double tol = 3e-15 * std::sqrt((double)n);
  const int max_sweeps = 40;
  const int thr = np <= 64 ? std::max(64, ((np / 2) * 8 + 31) / 32 * 32) : kEigT;
  if (need <= 200 * 1024) {
#define RT_EIG(KL)                                                                                   \
  smem_attr(jacobi_kernel<KL, true>, need);                                                                 \
  RT_LAUNCH(c, (jacobi_kernel<KL, true>), 1, thr, need, A, n, w, V, (double *)nullptr, tol, max_sweeps, sweeps, gate, \
            c.status)
    if (np <= 64) { RT_EIG(8); } else { RT_EIG(32); }
#undef RT_EIG
  } else {  // matrices in global memory (L2): the whole GPU, one warp per pair, grid-synchronised
    static const bool one_cta = RT_EXP_GETENV("RTUCKER_EIG_ONE_CTA") != nullptr;
    DevBuf<double> ws(c, 2 * (size_t)np * np + np);
    if (one_cta) {
      RT_LAUNCH(c, (jacobi_kernel<32, false>), 1, kEigT, 0, A, n, w, V, ws.p, tol, max_sweeps, sweeps, gate, c.status);
    } else {
      DevBuf<int> conv(c, 3);
      int nb = 0;
      RT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, jacobi_grid_kernel, kEigGT, 0));
      const int grid = std::max(1, std::min(c.num_sms * std::max(nb, 1), (np / 2 + 7) / 8));
      double *wsp = ws.p;
      int *convp = conv.p;
      double tl = tol;
      int ms = max_sweeps;
      unsigned *stp = c.status;
      void *args[] = {(void *)&A, (void *)&n, (void *)&w, (void *)&V, (void *)&wsp, (void *)&convp,
                      (void *)&tl, (void *)&ms, (void *)&sweeps, (void *)&gate, (void *)&stp};
      RT_CUDA(cudaLaunchCooperativeKernel((const void *)jacobi_grid_kernel, dim3(grid), dim3(kEigGT), args, 0, c.stream));
      c.launches++;
    }
  }
}

}  // namespace rt
