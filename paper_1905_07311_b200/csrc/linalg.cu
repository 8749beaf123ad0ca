// Small dense linear algebra on the device, fp64 (latency-bound steps of the path):
//   (householder_qr and sym_eig live in smallla.cu)
//   gemm_small      A_n = Q U_B(:, 1:r) (Alg 1 line 5) and friends
//   reductions      deterministic two-stage sums (norms, residuals)
#include "kernels.h"

namespace rt {

namespace {


__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// C = op(A) B, one thread per output element (small sizes only).
__global__ void gemm_small_kernel(bool transA, const double *__restrict__ A, int64_t lda,
                                  const double *__restrict__ B, int64_t ldb, double *__restrict__ C,
                                  int64_t ldc, int64_t m, int64_t n, int64_t k) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    double s = 0.0;
    if (transA)
      for (int64_t t = 0; t < k; ++t) s += A[t + lda * i] * B[t + ldb * j];
    else
      for (int64_t t = 0; t < k; ++t) s += A[i + lda * t] * B[t + ldb * j];
    C[i + ldc * j] = s;
  }
}

// C (m x n) = beta C + alpha op(A) (m x k) op(B) (k x n), column-major fp64 on the fp64 tensor
// cores (mma.sync m8n8k4): CTA tile 64 x 64, K steps of 16 staged in shared memory, 8 warps of
// 32 x 16; fixed summation order (deterministic); blockIdx.z = batch (strides sA, sB, sC).
constexpr int kGm = 64, kGk = 16;
__global__ void __launch_bounds__(256) gemm_f64_kernel(bool transA, bool transB, const double *__restrict__ A,
                                                       int64_t lda, int64_t sA, const double *__restrict__ B,
                                                       int64_t ldb, int64_t sB, double *__restrict__ C, int64_t ldc,
                                                       int64_t sC, int64_t m, int64_t n, int64_t k, double beta,
                                                       double alpha) {
  __shared__ double As[kGk][kGm + 1], Bs[kGk][kGm + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  A += sA * blockIdx.z;
  B += sB * blockIdx.z;
  C += sC * blockIdx.z;
  const int64_t i0 = (int64_t)blockIdx.x * kGm, j0 = (int64_t)blockIdx.y * kGm;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int64_t k0 = 0; k0 < k; k0 += kGk) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (!transA) {
        const int ii = tid & 63, kk = (tid >> 6) + 4 * s;
        const int64_t gi = i0 + ii, gk = k0 + kk;
        As[kk][ii] = (gi < m && gk < k) ? A[gi + lda * gk] : 0.0;
      } else {
        const int kk = tid & 15, ii = (tid >> 4) + 16 * s;
        const int64_t gi = i0 + ii, gk = k0 + kk;
        As[kk][ii] = (gi < m && gk < k) ? A[gk + lda * gi] : 0.0;
      }
      if (!transB) {
        const int kk = tid & 15, jj = (tid >> 4) + 16 * s;
        const int64_t gj = j0 + jj, gk = k0 + kk;
        Bs[kk][jj] = (gj < n && gk < k) ? B[gk + ldb * gj] : 0.0;
      } else {
        const int jj = tid & 63, kk = (tid >> 6) + 4 * s;
        const int64_t gj = j0 + jj, gk = k0 + kk;
        Bs[kk][jj] = (gj < n && gk < k) ? B[gj + ldb * gk] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kGk; ks += 4) {
      const int kk = ks + (lane & 3);
      double bv[2];
#pragma unroll
      for (int b = 0; b < 2; ++b) bv[b] = Bs[kk][wn + 8 * b + (lane >> 2)];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double av = As[kk][wm + 8 * a + (lane >> 2)];
#pragma unroll
        for (int b = 0; b < 2; ++b)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                       : "d"(av), "d"(bv[b]));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gi = i0 + wm + 8 * a + (lane >> 2), gj = j0 + wn + 8 * b + 2 * (lane & 3) + h;
        if (gi < m && gj < n) {
          double *cp = C + gi + ldc * gj;
          const double v = alpha * acc[a][b][h];
          *cp = beta == 0.0 ? v : fma(beta, *cp, v);
        }
      }
}

// Large GEMMs (adaptive truncation: Gram and shrink with k, r ~ 700): CTA tile 64 x 128, 8 warps
// of 32 x 32 (16 m8n8k4 tiles each: 8 fragment loads feed 16 MMAs), K tiles of 16 in a 3-stage
// cp.async ring (8-byte copies: leading dimensions need not be even), zero fill at the edges.
// Shared layouts follow the global ones (no transposition): A as [k][m] (TA = false) or [m][k],
// B as [n][k] (TB = false) or [k][n].
constexpr int kBm = 64, kBn = 128, kBk = 16, kBs = 3;
constexpr int kPadM = kBm + 2, kPadN = kBn + 2, kPadK = kBk + 2;
// GA (Gram of a mode unfolding, L > 1): op(A)(i, t) = A[(t % L) + L i + L Km (t / L)] and
// op(B)(t, j) the same with j; blockIdx.z = K chunk [z kc, (z+1) kc) with C + z sC its partial.
template <bool TA, bool TB, bool GA = false>
__global__ void __launch_bounds__(256) gemm_f64_big_kernel(const double *__restrict__ A, int64_t lda, int64_t sA,
                                                           const double *__restrict__ B, int64_t ldb, int64_t sB,
                                                           double *__restrict__ C, int64_t ldc, int64_t sC, int64_t m,
                                                           int64_t n, int64_t k, double beta, double alpha,
                                                           int64_t gL = 1, int64_t gKm = 1, int64_t kc = 0,
                                                           int upper = 0) {
  // upper (Grams): tiles entirely below the diagonal (every row > every column) are not computed
  if (upper && (int64_t)blockIdx.x * kBm > (int64_t)blockIdx.y * kBn + kBn - 1) return;
  extern __shared__ __align__(16) double gsm[];
  constexpr int kAst = TA ? kBm * kPadK : kBk * kPadM;  // doubles per A stage
  constexpr int kBst = TB ? kBk * kPadN : kBn * kPadK;  // doubles per B stage
  double *As = gsm, *Bs = gsm + kBs * kAst;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t kbeg = 0;
  if (GA) {
    kbeg = (int64_t)blockIdx.z * kc;
    k = min(k, kbeg + kc);
  } else {
    A += sA * blockIdx.z;
    B += sB * blockIdx.z;
  }
  C += sC * blockIdx.z;
  const int64_t i0 = (int64_t)blockIdx.x * kBm, j0 = (int64_t)blockIdx.y * kBn;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int nkt = (int)((k - kbeg + kBk - 1) / kBk);
  auto load_stage = [&](int kt, int st) {
    const int64_t k0 = kbeg + (int64_t)kt * kBk;
    double *as = As + st * kAst, *bs = Bs + st * kBst;
    // GA: the K index t = l + gL r of this tile, split once per stage (per-element 64-bit
    // divisions were subroutine calls: 12 per thread and stage, the gather Gram ran at 12 TF/s)
    int64_t r0 = 0, l0 = 0;
    if (GA) {
      r0 = k0 / gL;
      l0 = k0 - r0 * gL;
    }
    auto gsplit = [&](int kk, int64_t &l, int64_t &r) {
      l = l0 + kk;
      r = r0;
      while (l >= gL) { l -= gL; ++r; }
    };
    // A: 64 x 16 = 1024 elements, 4 per thread
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + 256 * q;
      int mm, kk;
      if (!TA) { mm = e & 63; kk = e >> 6; } else { kk = e & 15; mm = e >> 4; }
      const int64_t gi = i0 + mm, gk = k0 + kk;
      const bool ok = gi < m && gk < k;
      const double *src = A;
      if (ok) {
        if (GA) {
          int64_t l, r;
          gsplit(kk, l, r);
          src = A + l + gL * gi + gL * gKm * r;
        }
        else src = TA ? A + gk + lda * gi : A + gi + lda * gk;
      }
      double *dst = TA ? as + mm * kPadK + kk : as + kk * kPadM + mm;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(src), "r"(ok ? 8 : 0));
    }
    // B: 16 x 128 = 2048 elements, 8 per thread
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + 256 * q;
      int nn, kk;
      if (!TB) { kk = e & 15; nn = e >> 4; } else { nn = e & 127; kk = e >> 7; }
      const int64_t gj = j0 + nn, gk = k0 + kk;
      const bool ok = gj < n && gk < k;
      const double *src = B;
      if (ok) {
        if (GA) {
          int64_t l, r;
          gsplit(kk, l, r);
          src = B + l + gL * gj + gL * gKm * r;
        }
        else src = TB ? B + gj + ldb * gk : B + gk + ldb * gj;
      }
      double *dst = TB ? bs + kk * kPadN + nn : bs + nn * kPadK + kk;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(src), "r"(ok ? 8 : 0));
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int st = 0; st < kBs - 1; ++st) {
    if (st < nkt) load_stage(st, st);
    asm volatile("cp.async.commit_group;");
  }
  for (int kt = 0; kt < nkt; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kBs - 2));
    __syncthreads();
    if (kt + kBs - 1 < nkt) load_stage(kt + kBs - 1, (kt + kBs - 1) % kBs);
    asm volatile("cp.async.commit_group;");
    const double *as = As + (kt % kBs) * kAst, *bs = Bs + (kt % kBs) * kBst;
#pragma unroll
    for (int ks = 0; ks < kBk; ks += 4) {
      const int kk = ks + (lane & 3), r = lane >> 2;
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = TA ? as[(wm + 8 * a + r) * kPadK + kk] : as[kk * kPadM + wm + 8 * a + r];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = TB ? bs[kk * kPadN + wn + 8 * b + r] : bs[(wn + 8 * b + r) * kPadK + kk];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                       : "d"(av[a]), "d"(bv[b]));
    }
  }
  asm volatile("cp.async.wait_group 0;");
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gi = i0 + wm + 8 * a + (lane >> 2), gj = j0 + wn + 8 * b + 2 * (lane & 3) + h;
        if (gi < m && gj < n) {
          double *cp = C + gi + ldc * gj;
          const double v = alpha * acc[a][b][h];
          *cp = beta == 0.0 ? v : fma(beta, *cp, v);
        }
      }
}
constexpr size_t kBigSmem(bool ta, bool tb) {
  return sizeof(double) * kBs * ((ta ? kBm * kPadK : kBk * kPadM) + (tb ? kBk * kPadN : kBn * kPadK));
}

// Gram C = X X^T (K x K) of the mode unfolding of a (L, K, R) fp64 tensor B: X(i, t) =
// B[(t % L) + L (i + K (t / L))], t < L R, on the fp64 tensor cores.  Upper 64 x 64 tiles,
// K dimension split over gridDim.z chunks (partials summed in a fixed order by
// gram_split_reduce_kernel: deterministic).
__global__ void __launch_bounds__(256) gram_gather_kernel(const double *__restrict__ B, int64_t L, int64_t K, int64_t R,
                                                          int64_t chunk, double *__restrict__ part) {
  const int ti = blockIdx.x, tj = blockIdx.y;
  if (ti > tj) return;
  __shared__ double As[kGk][kGm + 1], Bs[kGk][kGm + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t T = L * R;
  const int64_t t0 = (int64_t)blockIdx.z * chunk, t1 = min(T, t0 + chunk);
  const int64_t i0 = (int64_t)ti * kGm, j0 = (int64_t)tj * kGm;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int64_t k0 = t0; k0 < t1; k0 += kGk) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      int ii, kk;
      if (L == 1) { ii = tid & 63; kk = (tid >> 6) + 4 * s; }   // B[i + K t]: i contiguous
      else { kk = tid & 15; ii = (tid >> 4) + 16 * s; }         // t contiguous within a row l
      const int64_t gt = k0 + kk;
      double va = 0.0, vb = 0.0;
      if (gt < t1) {
        const int64_t l = gt % L, r = gt / L;
        const int64_t base = l + L * K * r;
        if (i0 + ii < K) va = B[base + L * (i0 + ii)];
        if (j0 + ii < K) vb = B[base + L * (j0 + ii)];
      }
      As[kk][ii] = va;
      Bs[kk][ii] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kGk; ks += 4) {
      const int kk = ks + (lane & 3);
      double bv[2];
#pragma unroll
      for (int b = 0; b < 2; ++b) bv[b] = Bs[kk][wn + 8 * b + (lane >> 2)];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double av = As[kk][wm + 8 * a + (lane >> 2)];
#pragma unroll
        for (int b = 0; b < 2; ++b)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                       : "d"(av), "d"(bv[b]));
      }
    }
    __syncthreads();
  }
  double *P = part + (int64_t)blockIdx.z * K * K;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gi = i0 + wm + 8 * a + (lane >> 2), gj = j0 + wn + 8 * b + 2 * (lane & 3) + h;
        if (gi < K && gj < K) P[gi + K * gj] = acc[a][b][h];
      }
}

__global__ void gram_reduce_full_kernel(const double *__restrict__ part, int nsplit, int64_t K,
                                        double *__restrict__ C) {
  // fixed-order sum of the split partials of the upper triangle (the GEMM computed only the tiles
  // touching it), mirrored: C is exactly symmetric
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K * K; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % K, j = e / K;
    if (i > j) continue;
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += part[(int64_t)q * K * K + e];
    C[i + K * j] = s;
    C[j + K * i] = s;
  }
}

__global__ void gram_split_reduce_kernel(const double *__restrict__ part, int nsplit, int64_t K,
                                         double *__restrict__ C) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K * K; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % K, j = e / K;
    if ((i / kGm) > (j / kGm)) continue;  // lower tiles were not computed: mirrored below
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += part[(int64_t)q * K * K + e];
    C[i + K * j] = s;
    C[j + K * i] = s;
  }
}

template <typename S, typename D>
__global__ void convert_kernel(const S *__restrict__ s, D *__restrict__ d, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    d[e] = (D)s[e];
}

constexpr int kRedBlocks = 1024;

template <typename T>
__global__ void sumsq_stage1(const T *__restrict__ x, const double *__restrict__ y, int64_t n,
                             double *__restrict__ part) {
  __shared__ double sred[8];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)x[e] - (y ? y[e] : 0.0);
    s += v * v;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sred[k];
    part[blockIdx.x] = t;
  }
}

__global__ void sum_vec_kernel(const double *__restrict__ x, int64_t n, double *__restrict__ out) {
  __shared__ double sred[32];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) s += x[e];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sred[k];
    *out = t;
  }
}

__global__ void sub_scalar_kernel(const double *a, const double *b, double *out) { *out = *a - *b; }

}  // namespace

void gemm_small(Ctx &c, bool transA, const double *A, int64_t lda, const double *B, int64_t ldb,
                double *C, int64_t ldc, int64_t m, int64_t n, int64_t k) {
  if (m * n * k >= (1 << 20)) return gemm_f64(c, transA, A, lda, B, ldb, C, ldc, m, n, k, 0.0, 1.0);
  const int g = std::max(1, std::min(2048, ceil_div(m * n, 256)));
  RT_LAUNCH(c, gemm_small_kernel, g, 256, 0, transA, A, lda, B, ldb, C, ldc, m, n, k);
}

void gemm_f64(Ctx &c, bool transA, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
              int64_t ldc, int64_t m, int64_t n, int64_t k, double beta, double alpha) {
  gemm_f64_batched(c, transA, false, A, lda, 0, B, ldb, 0, C, ldc, 0, m, n, k, 1, beta, alpha);
}

void gemm_f64_batched(Ctx &c, bool transA, bool transB, const double *A, int64_t lda, int64_t sA, const double *B,
                      int64_t ldb, int64_t sB, double *C, int64_t ldc, int64_t sC, int64_t m, int64_t n, int64_t k,
                      int64_t batch, double beta, double alpha) {
  if (m <= 0 || n <= 0 || batch <= 0) return;
  RT_REQUIRE(batch <= 65535, "gemm: more than 65535 batches");
  if (m * n * k * batch >= (int64_t)1 << 28) {  // large: the pipelined 64 x 128 kernel
    const dim3 g((unsigned)((m + kBm - 1) / kBm), (unsigned)((n + kBn - 1) / kBn), (unsigned)batch);
#define RT_BIG(TA_, TB_)                                                                                      \
  do {                                                                                                       \
    smem_attr(gemm_f64_big_kernel<TA_, TB_>, kBigSmem(TA_, TB_));                                            \
    RT_LAUNCH(c, (gemm_f64_big_kernel<TA_, TB_>), g, 256, kBigSmem(TA_, TB_), A, lda, sA, B, ldb, sB, C, ldc, sC, m, \
              n, k, beta, alpha);                                                                            \
  } while (0)
    if (!transA && !transB) RT_BIG(false, false);
    else if (transA && !transB) RT_BIG(true, false);
    else if (!transA && transB) RT_BIG(false, true);
    else RT_BIG(true, true);
#undef RT_BIG
    return;
  }
  const dim3 grid((unsigned)((m + kGm - 1) / kGm), (unsigned)((n + kGm - 1) / kGm), (unsigned)batch);
  RT_LAUNCH(c, gemm_f64_kernel, grid, 256, 0, transA, transB, A, lda, sA, B, ldb, sB, C, ldc, sC, m, n, k, beta,
            alpha);
}

void gram_f64(Ctx &c, const double *B, int64_t L, int64_t K, int64_t R, double *C) {
  const int64_t T = L * R;
  if (K * K * T < ((int64_t)1 << 28)) {  // small: the simple tiled kernel (upper tiles, split K)
    const int tiles = (int)((K + kGm - 1) / kGm);
    const int ntile = tiles * (tiles + 1) / 2;
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>((2 * c.num_sms + ntile - 1) / ntile, (T + 4095) / 4096));
    const int64_t chunk = ((T + nsplit - 1) / nsplit + kGk - 1) / kGk * kGk;
    nsplit = (int)((T + chunk - 1) / chunk);
    DevBuf<double> part(c, (size_t)nsplit * K * K);
    RT_LAUNCH(c, gram_gather_kernel, dim3(tiles, tiles, nsplit), 256, 0, B, L, K, R, chunk, part.p);
    RT_LAUNCH(c, gram_split_reduce_kernel, std::max(1, std::min(4096, ceil_div(K * K, 256))), 256, 0, part.p,
              nsplit, K, C);
    return;
  }
  // large: the pipelined kernel on the tiles touching the upper triangle (58 % of them at K = 760),
  // K chunks over ~2 waves, partials summed in a fixed order and mirrored
  int64_t tiles = 0;  // tiles touching the upper triangle
  for (int64_t by = 0; by < (K + kBn - 1) / kBn; ++by)
    for (int64_t bx = 0; bx < (K + kBm - 1) / kBm; ++bx) tiles += bx * kBm <= by * kBn + kBn - 1;
  int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>((2 * c.num_sms + tiles - 1) / tiles, T / 2048));
  const int64_t chunk = ((T + nsplit - 1) / nsplit + kBk - 1) / kBk * kBk;
  nsplit = (int)((T + chunk - 1) / chunk);
  DevBuf<double> part(c, (size_t)nsplit * K * K);
  const dim3 g((unsigned)((K + kBm - 1) / kBm), (unsigned)((K + kBn - 1) / kBn), (unsigned)nsplit);
  if (L == 1) {  // X = B (K x R, column-major): C = X X^T, full K chunks as batches, then the tail
    const int64_t nfull = T / chunk, tl = T - nfull * chunk;
    smem_attr(gemm_f64_big_kernel<false, true, false>, kBigSmem(false, true));
    if (nfull > 0) {
      const dim3 gf(g.x, g.y, (unsigned)nfull);
      RT_LAUNCH(c, (gemm_f64_big_kernel<false, true, false>), gf, 256, kBigSmem(false, true), B, K, chunk * K, B, K,
                chunk * K, part.p, K, K * K, K, K, chunk, 0.0, 1.0, (int64_t)1, (int64_t)1, (int64_t)0, 1);
    }
    if (tl > 0) {
      const dim3 g1(g.x, g.y, 1);
      RT_LAUNCH(c, (gemm_f64_big_kernel<false, true, false>), g1, 256, kBigSmem(false, true), B + nfull * chunk * K, K,
                0, B + nfull * chunk * K, K, 0, part.p + nfull * K * K, K, 0, K, K, tl, 0.0, 1.0, (int64_t)1,
                (int64_t)1, (int64_t)0, 1);
    }
  } else {
    smem_attr(gemm_f64_big_kernel<true, false, true>, kBigSmem(true, false));
    RT_LAUNCH(c, (gemm_f64_big_kernel<true, false, true>), g, 256, kBigSmem(true, false), B, 0, 0, B, 0, 0, part.p, K,
              K * K, K, K, T, 0.0, 1.0, L, K, chunk, 1);
  }
  RT_LAUNCH(c, gram_reduce_full_kernel, std::max(1, std::min(4096, ceil_div(K * K, 256))), 256, 0, part.p, nsplit,
            K, C);
}

void convert(Ctx &c, const void *src, DT s, void *dst, DT d, int64_t n) {
  const int g = std::max(1, std::min(4096, ceil_div(n, 256)));
  if (s == DT::F32 && d == DT::F64)
    RT_LAUNCH(c, (convert_kernel<float, double>), g, 256, 0, (const float *)src, (double *)dst, n);
  else if (s == DT::F64 && d == DT::F32)
    RT_LAUNCH(c, (convert_kernel<double, float>), g, 256, 0, (const double *)src, (float *)dst, n);
  else
    RT_CUDA(cudaMemcpyAsync(dst, src, n * dt_size(s), cudaMemcpyDeviceToDevice, c.stream));
}

static void sumsq_impl(Ctx &c, const void *X, DT t, const double *Y, int64_t n, double *out) {
  DevBuf<double> part(c, kRedBlocks);
  if (t == DT::F32)
    RT_LAUNCH(c, sumsq_stage1<float>, kRedBlocks, 256, 0, (const float *)X, Y, n, part.p);
  else
    RT_LAUNCH(c, sumsq_stage1<double>, kRedBlocks, 256, 0, (const double *)X, Y, n, part.p);
  sum_vec(c, part.p, kRedBlocks, out);
}

void sumsq(Ctx &c, const void *X, DT t, int64_t n, double *out) { sumsq_impl(c, X, t, nullptr, n, out); }

void diff_sumsq(Ctx &c, const void *X, DT t, const double *Y, int64_t n, double *out) {
  sumsq_impl(c, X, t, Y, n, out);
}

void sum_vec(Ctx &c, const double *x, int64_t n, double *out) {
  RT_LAUNCH(c, sum_vec_kernel, 1, 1024, 0, x, n, out);
}

void sub_scalar(Ctx &c, const double *a, const double *b, double *out) {
  RT_LAUNCH(c, sub_scalar_kernel, 1, 1, 0, a, b, out);
}

}  // namespace rt
