// Symmetric eigensolver for the small Grams of the hot path (Alg 1 line 4: the thin SVD
// of B through the eigenpairs of B B^T), n <= 64, in ONE CTA of 1024 threads:
//
//  A. Householder tridiagonalisation  Q^T A Q = T  (A in shared memory; per step one fused
//     round of matvecs y = A_sub x, u = Q x, then the rank-2 update A -= v w^T + w v^T and
//     Q -= (Q v)(tau v)^T, two CTA barriers per step: the reflector v = x - alpha e_1 is never
//     needed before its dot products, since A v = A x - alpha A e_1 and v^T A v follows from
//     x^T A x, (A x)_1 and a_11)
//  B. eigenvalues of T by multisection on Sturm counts (16 threads per eigenvalue, 17 points
//     per round, 14 rounds from the Gershgorin interval: ~eps ||T|| absolute)
//  C. eigenvectors of T by twisted factorisations T - lambda I = N_k D_k N_k^T (one warp per
//     eigenvalue pair; z_k = 1 at the twist index minimising |gamma_k|), Gram-Schmidt inside
//     clusters of eigenvalues closer than 1e-12 ||T||, then Newton-Schulz steps
//     Z <- Z (3 I - Z^T Z) / 2 on the fp64 tensor cores (orthogonality to O(eps^2))
//  D. V = Q Z on the fp64 tensor cores; eigenvalues descending.
//
// Accuracy: backward stable; eigenvalues to ~eps ||A|| absolute and eigenvectors to
// ~eps ||A|| / gap, the accuracy the fp64 Gram itself carries (its entries are rounded at
// eps ||B||^2 = eps lambda_1).  The dependent chain is ~58 tridiagonalisation steps of ~500
// cycles plus 14 Sturm rounds of n steps, instead of the 8-11 Jacobi sweeps x 63 rounds of
// the register Jacobi (gram_eig_kernel).
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace rt {

namespace {

constexpr int kTeT = 1024;
constexpr int kNP = 64;        // padded size
constexpr int kLd = kNP + 2;   // shared-memory row stride (doubles)

__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// C (64 x 64, row stride kLd) = op(A) B with A, B row-major 64 x 64 (stride kLd) in shared
// memory; transA: C = A^T B.  32 warps x 2 tiles of 8 x 8 (m8n8k4 fp64 tensor-core MMAs).
__device__ void gemm64(const double *A, const double *B, double *C, bool transA) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int tile = warp; tile < 64; tile += 32) {
    const int ti = tile >> 3, tj = tile & 7;
    double c0 = 0.0, c1 = 0.0;
    const int ar = 8 * ti + (lane >> 2), bc = 8 * tj + (lane >> 2);
#pragma unroll 4
    for (int k0 = 0; k0 < kNP; k0 += 4) {
      const int kk = k0 + (lane & 3);
      const double a = transA ? A[kk * kLd + ar] : A[ar * kLd + kk];
      const double b = B[kk * kLd + bc];
      dmma884(c0, c1, a, b);
    }
    const int r = 8 * ti + (lane >> 2), cc = 8 * tj + 2 * (lane & 3);
    C[r * kLd + cc] = c0;
    C[r * kLd + cc + 1] = c1;
  }
}

__device__ __forceinline__ double half_sum(double v) {  // sum over the 16-lane half warp
#pragma unroll
  for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sturm count: number of eigenvalues of T (d, e2 = e^2) below x (LDL^T pivots < 0).
__device__ __forceinline__ int sturm_count(const double *d, const double *e2, int n, double x, double pivmin) {
  double q = d[0] - x;
  int cnt = q < 0.0;
#pragma unroll 4
  for (int i = 1; i < n; ++i) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = (d[i] - x) - e2[i - 1] * rcp_nr(q);
    cnt += q < 0.0;
  }
  return cnt;
}

#ifdef RT_TRID_PROGRESS
__device__ volatile int *g_trid_progress;
__device__ long long g_trid_clk[8];
#define TPROG(v) do { if (threadIdx.x == 0) { g_trid_progress[0] = (v); if ((v) < 8) g_trid_clk[(v)] = clock64(); \
                       __threadfence_system(); } } while (0)
#else
#define TPROG(v)
#endif
__global__ void __launch_bounds__(kTeT, 1) trid_eig_kernel(const double *__restrict__ Ain, int n,
                                                         double *__restrict__ w, double *__restrict__ Vout,
                                                         int *__restrict__ info) {
  extern __shared__ __align__(16) double tsm[];
  double *A = tsm;                  // 64 x kLd, row-major (symmetric); later D / 1/D of phase C
  double *Q = A + kNP * kLd;        // 64 x kLd: accumulated reflectors (row i, column j)
  double *Z = Q + kNP * kLd;        // 64 x kLd: eigenvectors of T (row = component, column = eigenvalue)
  double *Z2 = Z + kNP * kLd;       // 64 x kLd: scratch (R / 1/R of phase C, Newton-Schulz)
  double *ys = Z2 + kNP * kLd;      // 64: y = A_sub x of the step
  double *ac = ys + kNP;            // 64: column k+1 of A_sub (before the update)
  double *part = ac + kNP;          // 2 x 32: warp partials of x.x and x.y
  double *d = part + 64;            // 64: diagonal of T
  double *e = d + kNP;              // 64: off-diagonal of T (e[i] = T[i+1][i])
  double *e2 = e + kNP;             // 64: e^2
  double *lam = e2 + kNP;           // 64: eigenvalues ascending
  __shared__ double sscale;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ri = tid >> 4, pt = tid & 15;  // phase A: row ri, column part pt
  TPROG(0);

  // ---- load (symmetrised, padded with zeros), scale to max |a_ij| = 1
  double amax = 0.0;
  for (int e0 = tid; e0 < kNP * kNP; e0 += kTeT) {
    const int i = e0 >> 6, j = e0 & 63;
    const double v = (i < n && j < n) ? 0.5 * (Ain[i + (size_t)n * j] + Ain[j + (size_t)n * i]) : 0.0;
    A[i * kLd + j] = v;
    Q[i * kLd + j] = (i == j) ? 1.0 : 0.0;
    amax = fmax(amax, fabs(v));
  }
  for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) part[warp] = amax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int q = 0; q < 32; ++q) m = fmax(m, part[q]);
    sscale = m > 0.0 ? m : 1.0;
  }
  __syncthreads();
  const double scale = sscale, iscale = 1.0 / scale;
  for (int e0 = tid; e0 < kNP * kNP; e0 += kTeT) A[(e0 >> 6) * kLd + (e0 & 63)] *= iscale;
  __syncthreads();

  // ---- A. tridiagonalisation
  TPROG(1);
  for (int k = 0; k + 2 < n; ++k) {
    TPROG(100 + k);
    const int c0 = k + 1;                        // x = A[c0.., k]
    // fused matvecs over the columns j >= c0: y_i = sum_j A[i][j] x_j (rows i >= c0),
    // u_i = sum_j Q[i][j] x_j (all rows)
    double ya = 0.0, yq = 0.0;
    for (int j = c0 + pt; j < n; j += 16) {
      const double xj = A[j * kLd + k];
      if (ri >= c0) ya = fma(A[ri * kLd + j], xj, ya);
      yq = fma(Q[ri * kLd + j], xj, yq);
    }
    ya = half_sum(ya);
    yq = half_sum(yq);
    const double xi = (ri >= c0 && ri < n) ? A[ri * kLd + k] : 0.0;
    const double aik1 = (ri >= c0 && ri < n) ? A[ri * kLd + c0] : 0.0;
    const double qik1 = Q[ri * kLd + c0];
    double pxx = pt == 0 ? xi * xi : 0.0, pxy = pt == 0 ? xi * ya : 0.0;
    pxx += __shfl_xor_sync(0xffffffffu, pxx, 16);
    pxy += __shfl_xor_sync(0xffffffffu, pxy, 16);
    if (lane == 0) {
      part[warp] = pxx;
      part[32 + warp] = pxy;
    }
    if (pt == 0 && ri < n) {
      ys[ri] = ya;
      ac[ri] = aik1;
    }
    __syncthreads();
    // every warp reduces the partials (identical sums): x.x, x.y
    double sxx = part[lane], sxy = part[32 + lane];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
      sxy += __shfl_xor_sync(0xffffffffu, sxy, o);
    }
    const double x1 = A[c0 * kLd + k];
    if (sxx > 0.0) {
      const double nx = sqrt(sxx);
      const double alpha = x1 >= 0.0 ? -nx : nx;   // H x = alpha e_1
      const double h = sxx - alpha * x1;           // |v|^2 / 2
      const double tau = 1.0 / h;                  // H = I - tau v v^T
      const double y1 = ys[c0], a11 = ac[c0];
      // p = tau A v = tau (y - alpha a),  p.v = tau (x.y - 2 alpha y_1 + alpha^2 a_11)
      const double pv = tau * (sxy - 2.0 * alpha * y1 + alpha * alpha * a11);
      const double kc = 0.5 * tau * pv;
      // rank-2 update of rows ri >= c0 (w_j = tau (y_j - alpha a_j) - kc v_j)
      if (ri >= c0 && ri < n) {
        const double vi = (ri == c0) ? xi - alpha : xi;
        const double wi = tau * (ya - alpha * aik1) - kc * vi;
        for (int j = c0 + pt; j < n; j += 16) {
          const double xj = A[j * kLd + k];
          const double vj = (j == c0) ? xj - alpha : xj;
          const double wj = tau * (ys[j] - alpha * ac[j]) - kc * vj;
          A[ri * kLd + j] -= fma(vi, wj, wi * vj);
        }
      }
      // Q <- Q H: Q -= (Q v)(tau v)^T, (Q v)_i = u_i - alpha Q[i][c0]
      if (ri < n) {
        const double qv = tau * (yq - alpha * qik1);
        for (int j = c0 + pt; j < n; j += 16) {
          const double xj = A[j * kLd + k];
          const double vj = (j == c0) ? xj - alpha : xj;
          Q[ri * kLd + j] -= qv * vj;
        }
      }
      if (tid == 0) {
        d[k] = A[k * kLd + k];
        e[k] = alpha;
      }
    } else if (tid == 0) {  // column already reduced
      d[k] = A[k * kLd + k];
      e[k] = 0.0;
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (n >= 2) {
      d[n - 2] = A[(n - 2) * kLd + n - 2];
      e[n - 2] = A[(n - 1) * kLd + n - 2];
    }
    d[n - 1] = A[(n - 1) * kLd + n - 1];
  }
  __syncthreads();
  for (int i = tid; i < kNP; i += kTeT) e2[i] = (i + 1 < n) ? e[i] * e[i] : 0.0;
  // ---- B. eigenvalues: Gershgorin interval, multisection (16 threads per eigenvalue)
  TPROG(2);
  double glo = 1e300, ghi = -1e300;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
    glo = fmin(glo, d[i] - r);
    ghi = fmax(ghi, d[i] + r);
  }
  const double tnorm = fmax(fabs(glo), fabs(ghi));
  const double pm = 1e-280;  // LDL pivot floor (T is scaled to max |a_ij| = 1)
  {
    const int q = tid >> 4;  // eigenvalue index (ascending), 0..63
    double lo = glo - 2.2e-16 * tnorm - 1e-300, hi = ghi + 2.2e-16 * tnorm + 1e-300;
    for (int round = 0; round < 16; ++round) {
      const double x = lo + (hi - lo) * (double)(pt + 1) * (1.0 / 17.0);
      const int cnt = (q < n) ? sturm_count(d, e2, n, x, pm) : 0;
      // smallest sample point whose count exceeds q (eigenvalue q lies below it)
      const unsigned m = __ballot_sync(0xffffffffu, cnt > q) >> ((lane >> 4) << 4) & 0xFFFFu;
      const int t = m ? __ffs(m) - 1 : 16;  // first point above eigenvalue q
      const double nlo = lo + (hi - lo) * (double)t * (1.0 / 17.0);
      const double nhi = t < 16 ? lo + (hi - lo) * (double)(t + 1) * (1.0 / 17.0) : hi;
      lo = nlo;
      hi = nhi;
      // both eigenvalues of the warp converged (the ballot above needs all 32 lanes)
      if (__all_sync(0xffffffffu, hi - lo <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300)) break;
    }
    if (pt == 0 && q < n) lam[q] = 0.5 * (lo + hi);
  }
  __syncthreads();
  // ---- C. eigenvectors of T: twisted factorisations T - lambda I = L D L^T = U R U^T, two
  // threads per eigenvalue (top-down D, bottom-up R), all eigenvalues at once.  The
  // reciprocals 1/D_i, 1/R_i of the recurrences are kept for the eigenvector recurrences.
  // Storage (A and Z2 are free now): column q of A holds D (rows 0..63) ... as [q][i] planes.
  double *Dq = A, *Rq = Z2;  // Dq[q * kLd + i] = 1/D_i, Rq[q * kLd + i] = 1/R_i
  TPROG(3);
  if (tid < 2 * n) {
    const int q = tid >> 1;
    const double l = lam[q];
    if ((tid & 1) == 0) {
      double v = d[0] - l;
      for (int i = 0;; ++i) {
        if (fabs(v) < pm) v = -pm;
        const double r = rcp_nr(v);
        Dq[q * kLd + i] = r;
        if (i + 1 >= n) break;
        v = (d[i + 1] - l) - e2[i] * r;
      }
    } else {
      double v = d[n - 1] - l;
      for (int i = n - 1;; --i) {
        if (fabs(v) < pm) v = -pm;
        const double r = rcp_nr(v);
        Rq[q * kLd + i] = r;
        if (i == 0) break;
        v = (d[i - 1] - l) - e2[i - 1] * r;
      }
    }
  }
  __syncthreads();
  __shared__ int twist[kNP];
  if (tid < n) {  // twist index: argmin_k |gamma_k|, gamma_k = D_k + R_k - (d_k - lambda), first on ties
    const int q = tid;
    const double l = lam[q];
    double best = 1e308;
    int bk = 0;
    for (int i = 0; i < n; ++i) {
      const double g = fabs(1.0 / Dq[q * kLd + i] + 1.0 / Rq[q * kLd + i] - (d[i] - l));
      if (g < best) { best = g; bk = i; }
    }
    twist[q] = bk;
  }
  __syncthreads();
  if (tid < 2 * n) {  // z_k = 1; z_i = -(e_i / D_i) z_{i+1} (i < k); z_{i+1} = -(e_i / R_{i+1}) z_i (i >= k)
    const int q = tid >> 1, bk = twist[q];
    if ((tid & 1) == 0) {
      Z[bk * kLd + q] = 1.0;
      double z = 1.0;
      for (int i = bk - 1; i >= 0; --i) {
        z = -(e[i] * Dq[q * kLd + i]) * z;
        Z[i * kLd + q] = z;
      }
    } else {
      double z = 1.0;
      for (int i = bk; i + 1 < n; ++i) {
        z = -(e[i] * Rq[q * kLd + i + 1]) * z;
        Z[(i + 1) * kLd + q] = z;
      }
    }
  }
  __syncthreads();
  for (int q = warp; q < kNP; q += 32) {  // normalise; padding columns = unit vectors
    if (q < n) {
      double s2 = 0.0;
      for (int i = lane; i < n; i += 32) s2 = fma(Z[i * kLd + q], Z[i * kLd + q], s2);
      for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      const double inv = 1.0 / sqrt(s2);
      for (int i = lane; i < kNP; i += 32) Z[i * kLd + q] = i < n ? Z[i * kLd + q] * inv : 0.0;
    } else {
      for (int i = lane; i < kNP; i += 32) Z[i * kLd + q] = (i == q) ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  // Gram-Schmidt (twice) inside clusters of eigenvalues closer than 1e-12 ||T|| (warp 0); a
  // vector that collapses onto the earlier members (a numerically degenerate cluster, e.g. the
  // zero eigenvalues of a rank-deficient Gram) is replaced by a unit vector orthogonalised
  // against every other column except the cluster's later members (orthonormal completion)
  if (warp == 0) {
    const double ctol = 1e-12 * tnorm;
    for (int q = 1; q < n; ++q) {
      if (lam[q] - lam[q - 1] > ctol) continue;
      int s0 = q - 1;
      while (s0 > 0 && lam[s0] - lam[s0 - 1] <= ctol) --s0;
      int s1 = q;
      while (s1 + 1 < n && lam[s1 + 1] - lam[s1] <= ctol) ++s1;
      for (int attempt = 0; attempt <= n; ++attempt) {
        const int pe = attempt == 0 ? q : n;   // columns to orthogonalise against: [s0, q) or all others
        for (int pass = 0; pass < 2; ++pass) {
          for (int p = attempt == 0 ? s0 : 0; p < pe; ++p) {
            if (attempt > 0 && (p == q || (p > q && p <= s1))) continue;
            double dt = 0.0;
            for (int i = lane; i < n; i += 32) dt = fma(Z[i * kLd + p], Z[i * kLd + q], dt);
            for (int o = 16; o; o >>= 1) dt += __shfl_xor_sync(0xffffffffu, dt, o);
            for (int i = lane; i < n; i += 32) Z[i * kLd + q] -= dt * Z[i * kLd + p];
            __syncwarp();
          }
        }
        double s2 = 0.0;
        for (int i = lane; i < n; i += 32) s2 = fma(Z[i * kLd + q], Z[i * kLd + q], s2);
        for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (s2 > 1e-2) {
          const double inv = 1.0 / sqrt(s2);
          for (int i = lane; i < n; i += 32) Z[i * kLd + q] *= inv;
          __syncwarp();
          break;
        }
        const int t = (q + attempt) % n;  // collapsed: restart from a unit vector
        for (int i = lane; i < n; i += 32) Z[i * kLd + q] = (i == t) ? 1.0 : 0.0;
        __syncwarp();
      }
    }
  }
  __syncthreads();
  TPROG(4);
  // Newton-Schulz: Z <- Z (3 I - Z^T Z) / 2 (S = Z^T Z in A's storage)
  double *S = A;
  gemm64(Z, Z, S, true);
  __syncthreads();
  for (int e0 = tid; e0 < kNP * kNP; e0 += kTeT) {
    const int i = e0 >> 6, j = e0 & 63;
    S[i * kLd + j] = ((i == j) ? 1.5 : 0.0) - 0.5 * S[i * kLd + j];
  }
  __syncthreads();
  gemm64(Z, S, Z2, false);  // Z2 = Z (1.5 I - 0.5 Z^T Z)
  __syncthreads();
  // ---- D. V = Q Z2 (into Z's storage), eigenvalues descending
  gemm64(Q, Z2, Z, false);
  __syncthreads();
  for (int e0 = tid; e0 < n * n; e0 += kTeT) {
    const int row = e0 % n, col = e0 / n;  // output column col = eigenvalue n-1-col (descending)
    Vout[row + (size_t)n * col] = Z[row * kLd + (n - 1 - col)];
  }
  for (int i = tid; i < n; i += kTeT) w[i] = lam[n - 1 - i] * scale;
  if (tid == 0 && info) *info = 1;
  TPROG(5);
}


// ------------------------------------------------------------------------------------------
// Large n (adaptive truncation, n ~ 100..4096): the same three phases on the whole GPU in one
// cooperative kernel (matrices in global memory, L2 resident): one warp per matrix row for the
// fused matvecs and the rank-2 / Q updates, two grid barriers per Householder step; one warp
// per eigenvalue for the multisection (33 points per round); two threads per eigenvalue for
// the twisted factorisations; Gram-Schmidt inside clusters by the warp that owns the cluster's
// first eigenvalue.  Newton-Schulz and V = Q Z run on the fp64 tensor cores afterwards
// (gemm_f64).  Layouts: A, Q row-major n x n (ld n); Z column-major (eigenvector q at Z + q n).
struct TridGridWs {
  double *A, *Q, *Z, *Dinv, *Rinv;   // n x n each
  double *ys, *ac, *qc, *d, *e, *e2, *lam;  // n each
  double *pxx, *pxy;                 // grid partials
  int *twist;                        // n
};

__global__ void __launch_bounds__(256) trid_eig_grid_kernel(const double *__restrict__ Ain, int n, TridGridWs ws,
                                                          double *__restrict__ scale_out) {
  cg::grid_group grid = cg::this_grid();
#ifdef RTUCKER_TRID_PROF_BUILD
  long long tg_[4] = {0, 0, 0, 0};
  const long long tg0_ = clock64();
#define TGP(i) if (blockIdx.x == 0 && threadIdx.x == 0) tg_[i] = clock64() - tg0_
#else
#define TGP(i)
#endif
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gthr = (int64_t)gridDim.x * blockDim.x;
  const int gw = (int)(gtid >> 5), nw = (int)(gthr >> 5);
  double *__restrict__ A = ws.A;
  double *__restrict__ Q = ws.Q;
  __shared__ double red[8];
  __shared__ double bc[2];
  // ---- load, symmetrise, scale by max |a_ij| (order-independent maximum)
  double amax = 0.0;
  for (int64_t e0 = gtid; e0 < (int64_t)n * n; e0 += gthr) {
    const int i = (int)(e0 / n), j = (int)(e0 % n);
    const double v = 0.5 * (Ain[i + (int64_t)n * j] + Ain[j + (int64_t)n * i]);
    A[e0] = v;
    Q[e0] = (i == j) ? 1.0 : 0.0;
    amax = fmax(amax, fabs(v));
  }
  for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    ws.pxx[blockIdx.x] = m;
  }
  grid.sync();
  double scale = 0.0;
  for (int q = 0; q < (int)gridDim.x; ++q) scale = fmax(scale, ws.pxx[q]);
  if (!(scale > 0.0)) scale = 1.0;
  const double iscale = 1.0 / scale;
  if (gtid == 0) *scale_out = scale;
  for (int64_t e0 = gtid; e0 < (int64_t)n * n; e0 += gthr) A[e0] *= iscale;
  grid.sync();
  TGP(0);
  // ---- A. tridiagonalisation (x = row k of A, j >= k+1; A stays symmetric)
  for (int k = 0; k + 2 < n; ++k) {
    const int c0 = k + 1;
    const double *xr = A + (int64_t)k * n;
    double pxx = 0.0, pxy = 0.0;
    for (int i = gw; i < n; i += nw) {
      double ya = 0.0, yq = 0.0;
      const double *ar = A + (int64_t)i * n, *qr = Q + (int64_t)i * n;
      for (int j = c0 + lane; j < n; j += 32) {
        const double xj = xr[j];
        if (i >= c0) ya = fma(ar[j], xj, ya);
        yq = fma(qr[j], xj, yq);
      }
      for (int o = 16; o; o >>= 1) {
        ya += __shfl_xor_sync(0xffffffffu, ya, o);
        yq += __shfl_xor_sync(0xffffffffu, yq, o);
      }
      if (lane == 0) {
        ws.qc[i] = yq;            // u_i = (Q x)_i ...
        ws.e2[i] = qr[c0];        // ... and Q[i][c0] (e2 is free until phase B)
        if (i >= c0) {
          const double xi = xr[i];
          ws.ys[i] = ya;
          ws.ac[i] = ar[c0];
          pxx = fma(xi, xi, pxx);
          pxy = fma(xi, ya, pxy);
        }
      }
    }
    // per-CTA partials in a fixed order (warp lane 0 values, then warps)
    pxx = __shfl_sync(0xffffffffu, pxx, 0);
    pxy = __shfl_sync(0xffffffffu, pxy, 0);
    __syncthreads();
    if (lane == 0) {
      red[threadIdx.x >> 5] = pxx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      ws.pxx[blockIdx.x] = t;
    }
    __syncthreads();
    if (lane == 0) red[threadIdx.x >> 5] = pxy;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      ws.pxy[blockIdx.x] = t;
    }
    grid.sync();
    if (threadIdx.x < 32) {  // the CTA partials by one warp: lane-strided sums, fixed-order tree
      double sxx = 0.0, sxy = 0.0;
      for (int q = lane; q < (int)gridDim.x; q += 32) {
        sxx += ws.pxx[q];
        sxy += ws.pxy[q];
      }
      for (int o = 16; o; o >>= 1) {
        sxx += __shfl_xor_sync(0xffffffffu, sxx, o);
        sxy += __shfl_xor_sync(0xffffffffu, sxy, o);
      }
      if (lane == 0) {
        bc[0] = sxx;
        bc[1] = sxy;
      }
    }
    __syncthreads();
    const double sxx = bc[0], sxy = bc[1];
    const double x1 = xr[c0];
    if (sxx > 0.0) {
      const double nx = sqrt(sxx);
      const double alpha = x1 >= 0.0 ? -nx : nx;
      const double tau = 1.0 / (sxx - alpha * x1);
      const double pv = tau * (sxy - 2.0 * alpha * ws.ys[c0] + alpha * alpha * ws.ac[c0]);
      const double kc = 0.5 * tau * pv;
      for (int i = gw; i < n; i += nw) {
        double *ar = A + (int64_t)i * n, *qr = Q + (int64_t)i * n;
        if (i >= c0) {
          const double xi = xr[i];
          const double vi = (i == c0) ? xi - alpha : xi;
          const double wi = tau * (ws.ys[i] - alpha * ws.ac[i]) - kc * vi;
          for (int j = c0 + lane; j < n; j += 32) {
            const double xj = xr[j];
            const double vj = (j == c0) ? xj - alpha : xj;
            const double wj = tau * (ws.ys[j] - alpha * ws.ac[j]) - kc * vj;
            ar[j] -= fma(vi, wj, wi * vj);
          }
        }
        const double qv = tau * (ws.qc[i] - alpha * ws.e2[i]);
        for (int j = c0 + lane; j < n; j += 32) {
          const double xj = xr[j];
          const double vj = (j == c0) ? xj - alpha : xj;
          qr[j] -= qv * vj;
        }
      }
      if (gtid == 0) {
        ws.d[k] = xr[k];
        ws.e[k] = alpha;
      }
    } else if (gtid == 0) {
      ws.d[k] = xr[k];
      ws.e[k] = 0.0;
    }
    grid.sync();
  }
  if (gtid == 0) {
    if (n >= 2) {
      ws.d[n - 2] = A[(int64_t)(n - 2) * n + n - 2];
      ws.e[n - 2] = A[(int64_t)(n - 1) * n + n - 2];
    }
    ws.d[n - 1] = A[(int64_t)n * n - 1];
  }
  grid.sync();
  for (int64_t i = gtid; i < n; i += gthr) ws.e2[i] = (i + 1 < n) ? ws.e[i] * ws.e[i] : 0.0;
  grid.sync();
  const double *d = ws.d, *e = ws.e, *e2 = ws.e2;
  double glo = 1e300, ghi = -1e300;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
    glo = fmin(glo, d[i] - r);
    ghi = fmax(ghi, d[i] + r);
  }
  const double tnorm = fmax(fabs(glo), fabs(ghi));
  const double pm = 1e-280;
  TGP(1);
  // ---- B. eigenvalues: one warp per eigenvalue, 33-section
  for (int q = gw; q < n; q += nw) {
    double lo = glo - 2.2e-16 * tnorm - 1e-300, hi = ghi + 2.2e-16 * tnorm + 1e-300;
    for (int round = 0; round < 16; ++round) {
      const double x = lo + (hi - lo) * (double)(lane + 1) * (1.0 / 33.0);
      const int cnt = sturm_count(d, e2, n, x, pm);
      const unsigned m = __ballot_sync(0xffffffffu, cnt > q);
      const int t = m ? __ffs(m) - 1 : 32;
      const double nlo = lo + (hi - lo) * (double)t * (1.0 / 33.0);
      const double nhi = t < 32 ? lo + (hi - lo) * (double)(t + 1) * (1.0 / 33.0) : hi;
      lo = nlo;
      hi = nhi;
      if (hi - lo <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300) break;  // warp-uniform
    }
    if (lane == 0) ws.lam[q] = 0.5 * (lo + hi);
  }
  grid.sync();
  TGP(2);
  // ---- C. eigenvectors of T (twisted factorisations), eigenvector q in Z + q n
  for (int64_t t = gtid; t < 2 * (int64_t)n; t += gthr) {
    const int q = (int)(t >> 1);
    const double l = ws.lam[q];
    if ((t & 1) == 0) {
      double *Di = ws.Dinv + (int64_t)q * n;
      double v = d[0] - l;
      for (int i = 0;; ++i) {
        if (fabs(v) < pm) v = -pm;
        const double r = rcp_nr(v);
        Di[i] = r;
        if (i + 1 >= n) break;
        v = (d[i + 1] - l) - e2[i] * r;
      }
    } else {
      double *Ri = ws.Rinv + (int64_t)q * n;
      double v = d[n - 1] - l;
      for (int i = n - 1;; --i) {
        if (fabs(v) < pm) v = -pm;
        const double r = rcp_nr(v);
        Ri[i] = r;
        if (i == 0) break;
        v = (d[i - 1] - l) - e2[i - 1] * r;
      }
    }
  }
  grid.sync();
  for (int q = gw; q < n; q += nw) {  // twist: argmin |gamma_k| (warp reduction, first on ties)
    const double l = ws.lam[q];
    const double *Di = ws.Dinv + (int64_t)q * n, *Ri = ws.Rinv + (int64_t)q * n;
    double best = 1e308;
    int bk = 0;
    for (int i = lane; i < n; i += 32) {
      const double g = fabs(1.0 / Di[i] + 1.0 / Ri[i] - (d[i] - l));
      if (g < best) { best = g; bk = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bk, o);
      if (ob < best || (ob == best && oi < bk)) { best = ob; bk = oi; }
    }
    if (lane == 0) ws.twist[q] = bk;
  }
  grid.sync();
  for (int64_t t = gtid; t < 2 * (int64_t)n; t += gthr) {
    const int q = (int)(t >> 1), bk = ws.twist[q];
    double *z = ws.Z + (int64_t)q * n;
    if ((t & 1) == 0) {
      const double *Di = ws.Dinv + (int64_t)q * n;
      z[bk] = 1.0;
      double zv = 1.0;
      for (int i = bk - 1; i >= 0; --i) {
        zv = -(e[i] * Di[i]) * zv;
        z[i] = zv;
      }
    } else {
      const double *Ri = ws.Rinv + (int64_t)q * n;
      double zv = 1.0;
      for (int i = bk; i + 1 < n; ++i) {
        zv = -(e[i] * Ri[i + 1]) * zv;
        z[i + 1] = zv;
      }
    }
  }
  grid.sync();
  for (int q = gw; q < n; q += nw) {  // normalise
    double *z = ws.Z + (int64_t)q * n;
    double s2 = 0.0;
    for (int i = lane; i < n; i += 32) s2 = fma(z[i], z[i], s2);
    for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    const double inv = 1.0 / sqrt(s2);
    for (int i = lane; i < n; i += 32) z[i] *= inv;
  }
  grid.sync();
  // Gram-Schmidt (twice) inside clusters closer than 1e-12 ||T||: the warp of a cluster's first
  // eigenvalue orthogonalises the cluster's later vectors in order (warp 0 takes the clusters in
  // turn, so a replacement reads settled columns only); a collapsed vector is
  // replaced by a unit vector orthogonalised against every column outside the cluster's
  // unprocessed part (as in the one-CTA kernel)
  const double ctol = 1e-12 * tnorm;
  for (int s0 = 0; gw == 0 && s0 + 1 < n; ++s0) {  // one warp, clusters in order (deterministic)
    if (ws.lam[s0 + 1] - ws.lam[s0] > ctol || (s0 > 0 && ws.lam[s0] - ws.lam[s0 - 1] <= ctol)) continue;
    int s1 = s0 + 1;
    while (s1 + 1 < n && ws.lam[s1 + 1] - ws.lam[s1] <= ctol) ++s1;
    for (int q = s0 + 1; q <= s1; ++q) {
      double *zq = ws.Z + (int64_t)q * n;
      for (int attempt = 0; attempt <= n; ++attempt) {
        const int pe = attempt == 0 ? q : n;
        for (int pass = 0; pass < 2; ++pass) {
          for (int p = attempt == 0 ? s0 : 0; p < pe; ++p) {
            if (attempt > 0 && (p == q || (p > q && p <= s1))) continue;
            const double *zp = ws.Z + (int64_t)p * n;
            double dt = 0.0;
            for (int i = lane; i < n; i += 32) dt = fma(zp[i], zq[i], dt);
            for (int o = 16; o; o >>= 1) dt += __shfl_xor_sync(0xffffffffu, dt, o);
            for (int i = lane; i < n; i += 32) zq[i] -= dt * zp[i];
            __syncwarp();
          }
        }
        double s2 = 0.0;
        for (int i = lane; i < n; i += 32) s2 = fma(zq[i], zq[i], s2);
        for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (s2 > 1e-2) {
          const double inv = 1.0 / sqrt(s2);
          for (int i = lane; i < n; i += 32) zq[i] *= inv;
          __syncwarp();
          break;
        }
        const int t = (q + attempt) % n;
        for (int i = lane; i < n; i += 32) zq[i] = (i == t) ? 1.0 : 0.0;
        __syncwarp();
      }
    }
  }
#ifdef RTUCKER_TRID_PROF_BUILD
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("[trid prof] n %d grid %d: load %lld tridiag %lld eigvals %lld eigvecs %lld cycles\n", n, (int)gridDim.x, tg_[0], tg_[1] - tg_[0], tg_[2] - tg_[1], clock64() - tg0_ - tg_[2]);
#endif
#undef TGP
}

// S <- 1.5 I - 0.5 S (n x n)
__global__ void ns_shift_kernel(double *__restrict__ S, int n) {
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 < (int64_t)n * n;
       e0 += (int64_t)gridDim.x * blockDim.x)
    S[e0] = ((e0 % n) == (e0 / n) ? 1.5 : 0.0) - 0.5 * S[e0];
}

// w descending (unscaled), V columns in the same order (V = P Vasc, column q <- n-1-q).
__global__ void trid_out_kernel(const double *__restrict__ lam, const double *__restrict__ scale,
                                const double *__restrict__ Vasc, int n, double *__restrict__ w,
                                double *__restrict__ V) {
  const double s = *scale;
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 < (int64_t)n * n;
       e0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e0 % n, col = e0 / n;
    V[e0] = Vasc[row + (int64_t)n * (n - 1 - col)];
    if (row == 0) w[col] = lam[n - 1 - col] * s;
  }
}

}  // namespace

size_t trid_eig_smem() {
  // A, Q, Z, Z2 (64 x kLd each) + ys, ac, part (2 x 32), d, e, e2, lam
  return sizeof(double) * (4 * (size_t)kNP * kLd + 7 * kNP) + 64;
}

void trid_eig_large(Ctx &c, const double *A, int n, double *w, double *V) {
  const size_t nn = (size_t)n * n;
  DevBuf<double> big(c, 5 * nn + 7 * (size_t)n + 2 * 4096 + 1);
  DevBuf<int> tw(c, n);
  TridGridWs ws;
  ws.A = big.p;
  ws.Q = ws.A + nn;
  ws.Z = ws.Q + nn;
  ws.Dinv = ws.Z + nn;
  ws.Rinv = ws.Dinv + nn;
  ws.ys = ws.Rinv + nn;
  ws.ac = ws.ys + n;
  ws.qc = ws.ac + n;
  ws.d = ws.qc + n;
  ws.e = ws.d + n;
  ws.e2 = ws.e + n;
  ws.lam = ws.e2 + n;
  ws.pxx = ws.lam + n;
  ws.pxy = ws.pxx + 4096;
  double *scale = ws.pxy + 4096;
  ws.twist = tw.p;
  int per_sm = 0;
  RT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trid_eig_grid_kernel, 256, 0));
  // one warp per matrix row (ceil(n / 8) CTAs of 8 warps): the two grid barriers per Householder
  // step dominate phase A and cost more with more CTAs; at n = 760 phase A measured 26 ms with
  // 96 CTAs, 30 ms with 148, 38 ms with 48 and 53 ms with all 592 resident CTAs
  static const int gover = RT_EXP_GETENV("RTUCKER_TRID_GRID") ? atoi(RT_EXP_GETENV("RTUCKER_TRID_GRID")) : 0;
  const int gmax = std::max(1, std::min(c.num_sms * std::max(per_sm, 1), 4096));
  const int grid = gover > 0 ? std::min(gover, gmax) : std::min(gmax, (n + 7) / 8);
  void *args[] = {(void *)&A, (void *)&n, (void *)&ws, (void *)&scale};
  RT_CUDA(cudaLaunchCooperativeKernel((const void *)trid_eig_grid_kernel, dim3(grid), dim3(256), args, 0, c.stream));
  c.launches++;
  // Newton-Schulz: Z <- Z (1.5 I - 0.5 Z^T Z); then V = Q Z (Q row-major = Q^T column-major)
  // (two iterations: outside clusters (gaps > 1e-12 ||T||) the twisted vectors are orthogonal to
  // ~eps ||T|| / gap <= 1e-4, and each iteration squares the defect)
  double *S = ws.Dinv, *Z2 = ws.Rinv;
  for (int it = 0; it < 2; ++it) {
    double *src = it == 0 ? ws.Z : Z2, *dst = it == 0 ? Z2 : ws.Z;
    gemm_f64(c, true, src, n, src, n, S, n, n, n, n);
    RT_LAUNCH(c, ns_shift_kernel, std::max(1, std::min(4096, ceil_div((int64_t)nn, 256))), 256, 0, S, n);
    gemm_f64(c, false, src, n, S, n, dst, n, n, n, n);
  }
  gemm_f64(c, true, ws.Q, n, ws.Z, n, Z2, n, n, n, n);
  std::swap(ws.Z, Z2);
  RT_LAUNCH(c, trid_out_kernel, std::max(1, std::min(4096, ceil_div((int64_t)nn, 256))), 256, 0, ws.lam, scale,
            ws.Z, n, w, V);
}

bool trid_eig(Ctx &c, const double *A, int n, double *w, double *V, int *info) {
  if (n < 1) return false;
  if (n > kNP || RT_EXP_GETENV("RTUCKER_EIG_TRID_GRID")) {
    trid_eig_large(c, A, n, w, V);
    if (info) RT_CUDA(cudaMemsetAsync(info, 0, sizeof(int), c.stream));
    return true;
  }
  const size_t smem = trid_eig_smem();
  smem_attr(trid_eig_kernel, smem);
  RT_LAUNCH(c, trid_eig_kernel, 1, kTeT, smem, A, n, w, V, info);
  return true;
}

}  // namespace rt
