// Mode-n products out = X x_n A^T used for
//   the B-pass   B = Q^T X_(n)            (Alg 1 line 3)  + fused Gram B B^T (fp64)
//   the shrink   G_(n) <- U_B(:,1:r)^T B  (= Sigma_hat V_hat^T, Alg 3 line 6)
//   the core chain G = X x_1 A_1^T ... x_d A_d^T (Alg 2 line 5).
// SIMT kernel: each CTA walks tiles of TP output columns p = l + L*r (grid-stride), streams
// the mode-n index i in chunks of CI through smem (X tile coalesced along the contiguous
// index, A chunk), 4x4 register blocks, fp64 accumulation (fp32 products are flushed into
// fp64 every CI terms).  The optional Gram of the produced tile is accumulated per CTA in
// fp64 and reduced in a fixed order (deterministic).
#include "kernels.h"

namespace rt {

namespace {

constexpr int kThreads = 256;
constexpr int kCI = 32;

template <typename Tin, typename Tout, typename Tmul, int JP, bool STORE, bool GRAM>
__global__ void __launch_bounds__(kThreads) ttm_simt_kernel(
    const Tin *__restrict__ X, int64_t L, int64_t I, int64_t R, const double *__restrict__ A, int64_t lda,
    int J, int64_t Jst, Tout *__restrict__ out, double *__restrict__ gram_partial) {
  // J: active output columns of this launch (<= JP); Jst: size of the output mode
  // (stride of r in the output layout; > J when the caller blocks over j).
  constexpr int TP = 4096 / JP;
  constexpr int NJ = JP / 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tmul *sX = reinterpret_cast<Tmul *>(smem_raw);   // [kCI][TP]
  Tmul *sA = sX + kCI * TP;                         // [kCI][JP]
  double *sB = reinterpret_cast<double *>(smem_raw); // [TP][JP+1] (after the main loop)

  const int tid = threadIdx.x;
  const int tj = tid % NJ, tp = tid / NJ;
  const int64_t P = L * R;
  const int64_t ntiles = (P + TP - 1) / TP;

  double g[GRAM ? (JP * JP + kThreads - 1) / kThreads : 1];
  if (GRAM) {
#pragma unroll
    for (int e = 0; e < (JP * JP + kThreads - 1) / kThreads; ++e) g[e] = 0.0;
  }

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p0 = tile * TP;
    double accd[4][4];
    Tmul acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) { accd[a][b] = 0.0; acc[a][b] = Tmul(0); }

    const int64_t pl0 = p0 % L, pr0 = p0 / L;  // one 64-bit divide per tile
    for (int64_t i0 = 0; i0 < I; i0 += kCI) {
      __syncthreads();
      for (int e = tid; e < kCI * TP; e += kThreads) {
        int ii, pp;
        if (L == 1) { ii = e % kCI; pp = e / kCI; } else { pp = e % TP; ii = e / TP; }
        const int64_t i = i0 + ii, p = p0 + pp;
        Tmul x = Tmul(0);
        if (i < I && p < P) {
          int64_t off;
          if (L == 1) {
            off = i + I * p;
          } else {
            int64_t l = pl0 + pp, r = pr0;
            while (l >= L) { l -= L; ++r; }
            off = l + L * (i + I * r);
          }
          x = (Tmul)__ldg(X + off);
        }
        sX[ii * TP + pp] = x;
      }
      for (int e = tid; e < kCI * JP; e += kThreads) {
        const int ii = e / JP, j = e % JP;
        const int64_t i = i0 + ii;
        sA[ii * JP + j] = (i < I && j < J) ? (Tmul)__ldg(A + i + lda * j) : Tmul(0);
      }
      __syncthreads();
#pragma unroll 8
      for (int ii = 0; ii < kCI; ++ii) {
        Tmul a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { a[q] = sX[ii * TP + tp * 4 + q]; b[q] = sA[ii * JP + tj * 4 + q]; }
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) { accd[p][q] += (double)acc[p][q]; acc[p][q] = Tmul(0); }
    }
    // ---- epilogue: stage the tile (rounded to the stored precision) in smem
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int pp = tp * 4 + p, j = tj * 4 + q;
        const bool valid = (p0 + pp < P) && (j < J);
        sB[pp * (JP + 1) + j] = valid ? (double)(Tout)accd[p][q] : 0.0;
      }
    __syncthreads();
    if (STORE) {
      // out(l, j, r) at l + L*(j + J*r); coalesce along l (L > 1) or j (L == 1)
      for (int e = tid; e < TP * JP; e += kThreads) {
        int pp, j;
        if (L == 1) { j = e % JP; pp = e / JP; } else { pp = e % TP; j = e / TP; }
        const int64_t p = p0 + pp;
        if (p < P && j < J) {
          int64_t off;
          if (L == 1) {
            off = j + Jst * p;
          } else {
            int64_t l = pl0 + pp, r = pr0;
            while (l >= L) { l -= L; ++r; }
            off = l + L * (j + Jst * r);
          }
          out[off] = (Tout)sB[pp * (JP + 1) + j];
        }
      }
    }
    if (GRAM) {
#pragma unroll
      for (int e = 0; e < (JP * JP + kThreads - 1) / kThreads; ++e) {
        const int idx = tid + e * kThreads;
        if (idx < JP * JP) {
          const int j1 = idx / JP, j2 = idx % JP;
          double s = 0.0;
          for (int pp = 0; pp < TP; ++pp) s = fma(sB[pp * (JP + 1) + j1], sB[pp * (JP + 1) + j2], s);
          g[e] += s;
        }
      }
    }
  }
  if (GRAM) {
#pragma unroll
    for (int e = 0; e < (JP * JP + kThreads - 1) / kThreads; ++e) {
      const int idx = tid + e * kThreads;
      if (idx < JP * JP) gram_partial[(int64_t)blockIdx.x * JP * JP + idx] = g[e];
    }
  }
}

// gram[j1 + J*j2] = sum_b partial[b][j1*JP + j2]: one CTA per entry, fixed-shape tree
// (deterministic).
__global__ void gram_reduce_kernel(const double *__restrict__ partial, int nblk, int JP, int J,
                                   double *__restrict__ gram) {
  __shared__ double sred[4];
  const int e = blockIdx.x;
  const int j1 = e % J, j2 = e / J;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partial[(int64_t)b * JP * JP + j1 * JP + j2];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) gram[e] = (sred[0] + sred[1]) + (sred[2] + sred[3]);
}

template <typename Tin, typename Tout, typename Tmul, int JP>
void launch_ttm(Ctx &c, const Tin *X, ModeView v, const double *A, int64_t lda, int J, int64_t Jst,
                Tout *out, double *gram) {
  constexpr int TP = 4096 / JP;
  const int64_t P = v.L * v.R;
  const int64_t ntiles = (P + TP - 1) / TP;
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)c.num_sms * 4));
  const size_t sm_main = (size_t)kCI * (TP + JP) * sizeof(Tmul);
  const size_t sm_epi = (size_t)TP * (JP + 1) * sizeof(double);
  const size_t smem = std::max(sm_main, sm_epi);
  DevBuf<double> part;
  if (gram) part.alloc(c, (size_t)nblk * JP * JP);
#define RT_TTM_CASE(ST, GR)                                                                   \
  do {                                                                                        \
    auto k = ttm_simt_kernel<Tin, Tout, Tmul, JP, ST, GR>;                                    \
    smem_attr(k, smem); \
    RT_LAUNCH(c, k, nblk, kThreads, smem, X, v.L, v.I, v.R, A, lda, J, Jst, out, part.p);     \
  } while (0)
  if (out && gram) RT_TTM_CASE(true, true);
  else if (out) RT_TTM_CASE(true, false);
  else RT_TTM_CASE(false, true);
#undef RT_TTM_CASE
  if (gram) RT_LAUNCH(c, gram_reduce_kernel, J * J, 128, 0, part.p, nblk, JP, J, gram);
}

// Gram of the mode-n unfolding of a (stored) tensor B with mode size J:
// gram[j1 + J*j2] = sum_{l,r} B(l, j1, r) B(l, j2, r), computed per 64 x 64 block pair.
constexpr int kGB = 64;
template <typename T>
__global__ void __launch_bounds__(kThreads) mode_gram_kernel(const T *__restrict__ B, int64_t L, int64_t J,
                                                             int64_t R, int jb1, int jb2,
                                                             double *__restrict__ partial) {
  constexpr int TPc = 32;
  __shared__ double s1[TPc][kGB + 1], s2[TPc][kGB + 1];
  const int tid = threadIdx.x;
  const int64_t P = L * R;
  double acc[kGB * kGB / kThreads];
#pragma unroll
  for (int e = 0; e < kGB * kGB / kThreads; ++e) acc[e] = 0.0;
  for (int64_t p0 = (int64_t)blockIdx.x * TPc; p0 < P; p0 += (int64_t)gridDim.x * TPc) {
    __syncthreads();
    for (int e = tid; e < TPc * kGB; e += kThreads) {
      int pp, j;
      if (L == 1) { j = e % kGB; pp = e / kGB; } else { pp = e % TPc; j = e / TPc; }
      const int64_t p = p0 + pp;
      const int64_t j1 = (int64_t)jb1 * kGB + j, j2 = (int64_t)jb2 * kGB + j;
      double a = 0.0, b = 0.0;
      if (p < P) {
        const int64_t l = p % L, r = p / L;
        if (j1 < J) a = (double)B[l + L * (j1 + J * r)];
        if (j2 < J) b = (double)B[l + L * (j2 + J * r)];
      }
      s1[pp][j] = a;
      s2[pp][j] = b;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < kGB * kGB / kThreads; ++e) {
      const int idx = tid + e * kThreads;
      const int a = idx / kGB, b = idx % kGB;
      double s = 0.0;
#pragma unroll 8
      for (int pp = 0; pp < TPc; ++pp) s = fma(s1[pp][a], s2[pp][b], s);
      acc[e] += s;
    }
  }
#pragma unroll
  for (int e = 0; e < kGB * kGB / kThreads; ++e)
    partial[(int64_t)blockIdx.x * kGB * kGB + tid + e * kThreads] = acc[e];
}

__global__ void mode_gram_reduce_kernel(const double *__restrict__ partial, int nblk, int jb1, int jb2, int64_t J,
                                        double *__restrict__ gram) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kGB * kGB; e += gridDim.x * blockDim.x) {
    const int a = e / kGB, b = e % kGB;
    const int64_t j1 = (int64_t)jb1 * kGB + a, j2 = (int64_t)jb2 * kGB + b;
    if (j1 >= J || j2 >= J) continue;
    double s = 0.0;
    for (int k = 0; k < nblk; ++k) s += partial[(int64_t)k * kGB * kGB + e];
    gram[j1 + J * j2] = s;
    gram[j2 + J * j1] = s;
  }
}

// Gram of the mode-n unfolding for J <= 64 (fp64 DFMA, register-tiled): 256 threads in 4
// groups of 64; a group owns every 4th column of the CTA's chunk and each of its threads an
// 8 x 8 tile of the 64 x 64 Gram; columns p = l + L r are staged 32 at a time in shared
// memory (coalesced along l, or along j when L == 1).  Per-CTA partials are summed in a
// fixed order by gram_reduce2_kernel (deterministic).
constexpr int kGP = 32;  // columns per staged chunk
template <typename T>
__global__ void __launch_bounds__(256) gram64_kernel(const T *__restrict__ B, int64_t L, int J, int64_t R,
                                                     int64_t pchunk, double *__restrict__ partial) {
  __shared__ double sB[kGP][65];
  const int tid = threadIdx.x, grp = tid >> 6, t = tid & 63;
  const int ta = t >> 3, tb = t & 7;  // tile rows 8ta.., cols 8tb..
  const int64_t P = L * R;
  const int64_t pbeg = (int64_t)blockIdx.x * pchunk, pend = min(P, pbeg + pchunk);
  double acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  for (int64_t p0 = pbeg; p0 < pend; p0 += kGP) {
    __syncthreads();
    const int np_ = (int)((pend - p0) < kGP ? (pend - p0) : kGP);
    if (L == 1) {  // columns contiguous: B[j + J p]
      const T *src = B + p0 * J;
      for (int e = tid; e < kGP * 64; e += 256) {
        const int pp = e >> 6, j = e & 63;
        sB[pp][j] = (pp < np_ && j < J) ? (double)src[(int64_t)pp * J + j] : 0.0;
      }
    } else {
      const int64_t l0 = p0 % L, r0 = p0 / L;
      for (int e = tid; e < kGP * 64; e += 256) {
        const int pp = e % kGP, j = e / kGP;
        double v = 0.0;
        if (pp < np_ && j < J) {
          int64_t l = l0 + pp, r = r0;
          while (l >= L) { l -= L; ++r; }
          v = (double)B[l + L * (j + (int64_t)J * r)];
        }
        sB[pp][j] = v;
      }
    }
    __syncthreads();
#pragma unroll 2
    for (int pp = grp; pp < kGP; pp += 4) {
      double x[8], y[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { x[u] = sB[pp][8 * ta + u]; y[u] = sB[pp][8 * tb + u]; }
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
    }
  }
  // combine the 4 groups in a fixed order into the CTA partial [64 x 64] (global, L2)
  for (int g = 0; g < 4; ++g) {
    __syncthreads();
    if (grp == g) {
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const int64_t o = (int64_t)blockIdx.x * 4096 + (8 * ta + a) * 64 + 8 * tb + b;
          partial[o] = (g == 0 ? 0.0 : partial[o]) + acc[a][b];
        }
    }
  }
}

__global__ void gram_reduce2_kernel(const double *__restrict__ partial, int nblk, int J, double *__restrict__ gram) {
  __shared__ double sred[4];
  const int e = blockIdx.x;
  const int j1 = e % J, j2 = e / J;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partial[(int64_t)b * 4096 + j1 * 64 + j2];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) gram[e] = (sred[0] + sred[1]) + (sred[2] + sred[3]);
}

// Gram of the middle index for L, J <= 64 (B(l, j, r), slabs B(:, :, r) of L J contiguous
// doubles): each CTA sums M_r^T M_r over its contiguous range of r, thread = 4 x 4 tile of the
// 64 x 64 partial, one partial per CTA, reduced in a fixed order by gram_reduce2_kernel.
constexpr int kSGs = 68;  // slab row stride (doubles)
__global__ void __launch_bounds__(256) slab_gram_kernel(const double *__restrict__ B, int L, int J, int64_t R,
                                                        double *__restrict__ partial) {
  __shared__ __align__(16) double sM[64 * kSGs];
  const int tid = threadIdx.x, ta = tid >> 4, tb = tid & 15;
  const int64_t r0 = (int64_t)blockIdx.x * R / gridDim.x, r1 = (int64_t)(blockIdx.x + 1) * R / gridDim.x;
  for (int e = tid; e < 64 * kSGs; e += 256) sM[e] = 0.0;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  const int LJ = L * J;
  double pre[16];  // the next slab, prefetched into registers (L J <= 4096: 16 per thread)
  auto load = [&](int64_t r) {
    const double *src = B + r * (int64_t)LJ;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int e = tid + 256 * t;
      pre[t] = e < LJ ? src[e] : 0.0;
    }
  };
  if (r0 < r1) load(r0);
  for (int64_t r = r0; r < r1; ++r) {
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int e = tid + 256 * t;
      if (e < LJ) {
        const int j = e / L, l = e - j * L;
        sM[l * kSGs + j] = pre[t];
      }
    }
    __syncthreads();
    if (r + 1 < r1) load(r + 1);
    for (int l = 0; l < L; ++l) {
      const double2 x0 = *(const double2 *)&sM[l * kSGs + 4 * ta], x1 = *(const double2 *)&sM[l * kSGs + 4 * ta + 2];
      const double2 y0 = *(const double2 *)&sM[l * kSGs + 4 * tb], y1 = *(const double2 *)&sM[l * kSGs + 4 * tb + 2];
      const double x[4] = {x0.x, x0.y, x1.x, x1.y}, y[4] = {y0.x, y0.y, y1.x, y1.y};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(x[u], y[v], acc[u][v]);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) partial[(int64_t)blockIdx.x * 4096 + (4 * ta + u) * 64 + 4 * tb + v] = acc[u][v];
}

template <typename T>
void mode_gram_t(Ctx &c, const T *B, ModeView v, double *gram) {
  const int64_t P = v.L * v.R;
  if (v.I <= 64) {
    const int64_t nchunk = (P + kGP - 1) / kGP;
    const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(nchunk, (int64_t)c.num_sms * 3));
    const int64_t pchunk = ((nchunk + nblk - 1) / nblk) * kGP;
    const int g = (int)((P + pchunk - 1) / pchunk);
    DevBuf<double> part(c, (size_t)std::max(g, 1) * 4096);
    RT_LAUNCH(c, gram64_kernel<T>, g, 256, 0, B, v.L, (int)v.I, v.R, pchunk, part.p);
    RT_LAUNCH(c, gram_reduce2_kernel, (int)(v.I * v.I), 128, 0, part.p, g, (int)v.I, gram);
    return;
  }
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((P + 31) / 32, (int64_t)c.num_sms * 2));
  const int nb = ceil_div(v.I, kGB);
  DevBuf<double> part(c, (size_t)nblk * kGB * kGB);
  for (int b1 = 0; b1 < nb; ++b1)
    for (int b2 = b1; b2 < nb; ++b2) {
      RT_LAUNCH(c, mode_gram_kernel<T>, nblk, kThreads, 0, B, v.L, v.I, v.R, b1, b2, part.p);
      RT_LAUNCH(c, mode_gram_reduce_kernel, 16, 256, 0, part.p, nblk, b1, b2, v.I, gram);
    }
}

// ---------------------------------------------------------------- fp64 (DFMA) TTM ----
// out(l, j, r) = sum_i A[i, j] X(l, i, r) with fp64 products and sums (X fp32 or fp64), J <= 64,
// optional fp64 Gram of the output.  DFMA-bound (2 J flop per element of X), so the kernel is
// built for DFMA issue: a CTA owns a 64 (j) x 256 (p = l + L r) output tile, warp w the j-block
// 8w..8w+7 (A reads are warp broadcasts), lane the 8 consecutive columns 8 lane..; 8 x 8 fp64
// register tile per thread; X and A staged 16 values of i at a time in shared memory (X
// converted to fp64 once, at staging), next chunk prefetched into registers.  Persistent CTAs
// stride over column tiles; the Gram of each finished tile is accumulated per thread (4 x 4 of
// the 64 x 64) and written once per CTA (fixed-order reduction afterwards: deterministic).
constexpr int kDT = 256;   // threads
constexpr int kDP = 256;   // columns per tile
constexpr int kDK = 16;    // values of i per chunk
constexpr int kDS = kDP + 2;  // padded X row stride (doubles): 16-B aligned rows, fewer staging conflicts
template <typename Tin, bool STORE, bool GRAM>
__global__ void __launch_bounds__(kDT, 1) ttm_dfma_kernel(const Tin *__restrict__ X, int64_t L, int64_t I, int64_t R,
                                                          const double *__restrict__ A, int64_t lda, int J,
                                                          double *__restrict__ out, double *__restrict__ gram_partial) {
  extern __shared__ __align__(16) double dsm[];
  double *Xs = dsm;                        // [kDK][kDS]
  double *As = Xs + kDK * kDS;             // [kDK][64]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t P = L * R;
  const int64_t ntiles = (P + kDP - 1) / kDP;
  const int nchunk = (int)((I + kDK - 1) / kDK);
  double g[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) g[e] = 0.0;
  const int gj1 = (tid >> 4) * 4, gj2 = (tid & 15) * 4;  // Gram block of this thread
  // staging map (16 values per thread and chunk)
  //   L == 1: unit k = tid + 256 q (q < 4): column pp = k / 4, rows 4 (k % 4) .. +3
  //   L > 1 : element k = tid + 256 q (q < 16): column pp = tid (coalesced), row q
  Tin pre[16];
  double apre[4];

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p0 = tile * kDP;
    const int64_t pl0 = p0 % L, pr0 = p0 / L;
    int64_t mycol = -1;  // base offset of this thread's staging column (L > 1)
    if (L > 1) {
      const int64_t p = p0 + tid;
      if (p < P) {
        int64_t l = pl0 + tid, r = pr0;
        while (l >= L) { l -= L; ++r; }
        mycol = l + L * I * r;
      }
    }
    auto load_chunk = [&](int ch) {
      const int64_t i0 = (int64_t)ch * kDK;
      if (L == 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = tid + kDT * q, pp = k >> 2, iq = k & 3;
          const int64_t p = p0 + pp, i = i0 + 4 * iq;
#pragma unroll
          for (int u = 0; u < 4; ++u) pre[4 * q + u] = (p < P && i + u < I) ? X[(i + u) + I * p] : Tin(0);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t i = i0 + q;
          pre[q] = (mycol >= 0 && i < I) ? X[mycol + L * i] : Tin(0);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = tid + kDT * q, ii = e >> 6, j = e & 63;
        const int64_t i = i0 + ii;
        apre[q] = (i < I && j < J) ? A[i + lda * j] : 0.0;
      }
    };
    auto store_chunk = [&]() {
      if (L == 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = tid + kDT * q, pp = k >> 2, iq = k & 3;
#pragma unroll
          for (int u = 0; u < 4; ++u) Xs[(4 * iq + u) * kDS + pp] = (double)pre[4 * q + u];
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) Xs[q * kDS + tid] = (double)pre[q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) As[tid + kDT * q] = apre[q];
    };
    double acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
    load_chunk(0);
    for (int ch = 0; ch < nchunk; ++ch) {
      __syncthreads();
      store_chunk();
      __syncthreads();
      if (ch + 1 < nchunk) load_chunk(ch + 1);  // in flight during the DFMA block
#pragma unroll 4
      for (int ii = 0; ii < kDK; ++ii) {
        const double2 *ar = reinterpret_cast<const double2 *>(As + ii * 64 + 8 * warp);
        double a[8], x[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 av = ar[q];
          a[2 * q] = av.x;
          a[2 * q + 1] = av.y;
        }
#pragma unroll
        for (int w2 = 0; w2 < 4; ++w2) {  // columns 2 lane + 64 w2 + {0, 1}: conflict-free LDS.128
          const double2 xv = *reinterpret_cast<const double2 *>(Xs + ii * kDS + 2 * lane + 64 * w2);
          x[2 * w2] = xv.x;
          x[2 * w2 + 1] = xv.y;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int v = 0; v < 8; ++v) acc[u][v] = fma(a[u], x[v], acc[u][v]);
      }
    }
    // ---- epilogue: thread holds out(j = 8 warp + u, p = p0 + 2 lane + 64 (v / 2) + v % 2)
    if (STORE && L == 1) {
      // out[j + J p]: the tile is ONE contiguous range of J * 256 doubles; stage it [p][J] in
      // shared memory (two halves of 128 columns) and write it with coalesced 16-B stores
      for (int h = 0; h < 2; ++h) {
        __syncthreads();
        double *T = dsm;  // [128][J]
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int pp = 2 * lane + 64 * (v >> 1) + (v & 1);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int j = 8 * warp + u;
            if (j < J) T[pp * J + j] = acc[u][4 * h + v];
          }
        }
        __syncthreads();
        const int64_t pb = p0 + 128 * h;
        const int64_t ncol = P - pb < 128 ? (P - pb) : 128;
        if (ncol > 0) {
          const int64_t n = ncol * J;
          double *dst = out + pb * J;
          if (((J & 1) == 0)) {
            for (int64_t e = 2 * tid; e < n; e += 2 * kDT)
              *reinterpret_cast<double2 *>(dst + e) = *reinterpret_cast<const double2 *>(T + e);
          } else {
            for (int64_t e = tid; e < n; e += kDT) dst[e] = T[e];
          }
        }
      }
    } else if (STORE) {
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int pp = 2 * lane + 64 * (v >> 1) + (v & 1);
        const int64_t p = p0 + pp;
        if (p >= P) continue;
        int64_t l = pl0 + pp, r = pr0;
        while (l >= L) { l -= L; ++r; }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = 8 * warp + u;
          if (j < J) out[l + L * (j + (int64_t)J * r)] = acc[u][v];
        }
      }
    }
    if (GRAM) {  // stage the tile [p][64] in two halves of 128 columns, 4 x 4 Gram blocks
      for (int h = 0; h < 2; ++h) {
        __syncthreads();
        double *T = dsm;  // [128][65]
#pragma unroll
        for (int v = 0; v < 4; ++v) {  // register columns 4h .. 4h+3 = tile columns 128 h + 2 lane + 64 (v/2) + v%2 - 128 h
          const int pp = 2 * lane + 64 * (v >> 1) + (v & 1);  // column within the half
          const bool ok = p0 + 128 * h + pp < P;
#pragma unroll
          for (int u = 0; u < 8; ++u) T[pp * 65 + 8 * warp + u] = ok ? acc[u][4 * h + v] : 0.0;
        }
        __syncthreads();
        for (int pp = 0; pp < 128; ++pp) {
          double a4[4], b4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) { a4[q] = T[pp * 65 + gj1 + q]; b4[q] = T[pp * 65 + gj2 + q]; }
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int s = 0; s < 4; ++s) g[q * 4 + s] = fma(a4[q], b4[s], g[q * 4 + s]);
        }
      }
    }
  }
  if (GRAM) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int s = 0; s < 4; ++s) gram_partial[(int64_t)blockIdx.x * 4096 + (gj1 + q) * 64 + gj2 + s] = g[q * 4 + s];
  }
}

// ------------------------------------------------------ fp64 tensor-core (DMMA) TTM ----
// Same contraction and tiling contract as ttm_dfma_kernel, on the fp64 tensor cores
// (mma.sync.m8n8k4.f64: 256 FMA per warp instruction; the measured B200 peak equals DFMA's
// 37 TF/s, scripts/dbg/dmma_probe.cu, but the 8x lower instruction count leaves issue slots
// for the operand loads).  CTA tile 64 (j) x 256 (p); warp (wj = w & 1, wp = w >> 1) owns
// 32 j x 64 p = 4 x 8 MMA tiles (64 fp64 accumulators per thread).  Per chunk of 16 values of
// i: A staged [i][68] (A_mma[m][k] = A[i0 + k][j0 + m]), X staged [p][20] (B_mma[k][n] =
// X(i0 + k, p0 + n)); the paddings make both fragment loads bank-conflict-free per half warp.
// Fragment layouts (PTX m8n8k4 .f64): A row-major, lane -> (m = lane >> 2, k = lane & 3);
// B col-major, lane -> (k = lane & 3, n = lane >> 2); C lane -> (m = lane >> 2, n = 2 (lane & 3) + {0, 1}).
constexpr int kMA = 68;  // As row stride (doubles)
constexpr int kMX = 20;  // Xs row stride (doubles), rows = p
// Epilogue tile T[p][kTS] (kTS = 4 mod 16 doubles): conflict-free for the accumulator stores
// and for the Gram's DMMA fragment loads.  The Gram partial G += T^T T runs on the fp64 tensor
// cores too: the 36 upper 8x8 tiles of the 64 x 64 Gram are spread over the 8 warps.
constexpr int kTS = 68;
__device__ __forceinline__ void gram_tile_ab(int t, int &a, int &b) {
  a = 0;
  while (t >= 8 - a) { t -= 8 - a; ++a; }
  b = a + t;
}

// Stream-K work split (Osama et al. style): the ntiles x nchunk MAC iterations are divided
// evenly over the persistent grid, so a short tile list (P = L R of a few hundred columns)
// still fills every SM.  CTA b owns iterations [b T / G, (b+1) T / G).  A segment that starts
// mid-tile can only be the CTA's FIRST segment: it runs first, its accumulators go to fix[b]
// and flags[b] is set to this launch's epoch.  The CTA that runs a tile's chunk 0 (late in
// its own range) adds the partials of the CTAs b+1, b+2, .. that cover the rest of the tile
// (fixed order, deterministic), then runs the epilogue.  Partials are produced before any
// CTA waits, all CTAs are co-resident (grid = #SMs, one CTA per SM), so the hand-off
// neither serialises nor deadlocks.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename Tin, bool STORE, bool GRAM>
__global__ void __launch_bounds__(kDT, 1) ttm_dmma_kernel(const Tin *__restrict__ X, int64_t L, int64_t I, int64_t R,
                                                          const double *__restrict__ A, int64_t lda, int J,
                                                          double *__restrict__ out, double *__restrict__ gram_partial,
                                                          double *__restrict__ fix, unsigned *__restrict__ flags,
                                                          unsigned epoch) {
  extern __shared__ __align__(16) double dsm[];
  double *Xs = dsm;                        // [kDP][kMX]
  double *As = Xs + kDP * kMX;             // [kDK][kMA]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wj = warp & 1, wp = warp >> 1;
  const int fr = lane >> 2, fc = lane & 3;  // fragment row / column
  const int64_t P = L * R;
  const int64_t ntiles = (P + kDP - 1) / kDP;
  const int nchunk = (int)((I + kDK - 1) / kDK);
  const int64_t total = ntiles * nchunk, G = gridDim.x, b = blockIdx.x;
  auto seg_start = [&](int64_t cta) { return cta * total / G; };
  double gacc[5][2];
#pragma unroll
  for (int s5 = 0; s5 < 5; ++s5) gacc[s5][0] = gacc[s5][1] = 0.0;
  Tin pre[16];
  double apre[4];

  int64_t it = seg_start(b);
  const int64_t it_end = seg_start(b + 1);
  while (it < it_end) {
    const int64_t tile = it / nchunk;
    const int c0 = (int)(it - tile * nchunk);
    const int64_t rem = it_end - it;
    const int c1 = (c0 + rem < nchunk) ? (int)(c0 + rem) : nchunk;
    it += c1 - c0;
    const int64_t p0 = tile * kDP;
    const int64_t pl0 = p0 % L, pr0 = p0 / L;
    int64_t mycol = -1;
    if (L > 1) {
      const int64_t p = p0 + tid;
      if (p < P) {
        int64_t l = pl0 + tid, r = pr0;
        while (l >= L) { l -= L; ++r; }
        mycol = l + L * I * r;
      }
    }
    auto load_chunk = [&](int ch) {
      const int64_t i0 = (int64_t)ch * kDK;
      if (L == 1) {  // unit k = tid + 256 q: column pp = k / 4, rows 4 (k % 4) .. +3
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = tid + kDT * q, pp = k >> 2, iq = k & 3;
          const int64_t p = p0 + pp, i = i0 + 4 * iq;
#pragma unroll
          for (int u = 0; u < 4; ++u) pre[4 * q + u] = (p < P && i + u < I) ? X[(i + u) + I * p] : Tin(0);
        }
      } else {  // column pp = tid, rows q
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t i = i0 + q;
          pre[q] = (mycol >= 0 && i < I) ? X[mycol + L * i] : Tin(0);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = tid + kDT * q, ii = e >> 6, j = e & 63;
        const int64_t i = i0 + ii;
        apre[q] = (i < I && j < J) ? A[i + lda * j] : 0.0;
      }
    };
    auto store_chunk = [&]() {
      if (L == 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = tid + kDT * q, pp = k >> 2, iq = k & 3;
          double2 *d = reinterpret_cast<double2 *>(Xs + pp * kMX + 4 * iq);
          d[0] = make_double2((double)pre[4 * q], (double)pre[4 * q + 1]);
          d[1] = make_double2((double)pre[4 * q + 2], (double)pre[4 * q + 3]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) Xs[tid * kMX + q] = (double)pre[q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = tid + kDT * q, ii = e >> 6, j = e & 63;
        As[ii * kMA + j] = apre[q];
      }
    };
    double acc[4][8][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int bb = 0; bb < 8; ++bb) { acc[a][bb][0] = 0.0; acc[a][bb][1] = 0.0; }
    load_chunk(c0);
    for (int ch = c0; ch < c1; ++ch) {
      __syncthreads();
      store_chunk();
      __syncthreads();
      if (ch + 1 < c1) load_chunk(ch + 1);
#pragma unroll
      for (int ks = 0; ks < kDK / 4; ++ks) {
        double af[4], bf[8];
#pragma unroll
        for (int jt = 0; jt < 4; ++jt) af[jt] = As[(4 * ks + fc) * kMA + 32 * wj + 8 * jt + fr];
#pragma unroll
        for (int pt = 0; pt < 8; ++pt) bf[pt] = Xs[(64 * wp + 8 * pt + fr) * kMX + 4 * ks + fc];
#pragma unroll
        for (int jt = 0; jt < 4; ++jt)
#pragma unroll
          for (int pt = 0; pt < 8; ++pt)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(acc[jt][pt][0]), "+d"(acc[jt][pt][1])
                         : "d"(af[jt]), "d"(bf[pt]));
      }
    }
    if (c0 > 0) {  // tile begun by a lower CTA (this CTA's first segment): hand the partial over
      double *f = fix + b * (int64_t)(64 * kDT);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int bb = 0; bb < 8; ++bb)
#pragma unroll
          for (int h = 0; h < 2; ++h) f[((a * 8 + bb) * 2 + h) * kDT + tid] = acc[a][bb][h];
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release_u32(flags + b, epoch);
      continue;
    }
    if (c1 < nchunk) {  // add the partials of the CTAs that run the rest of this tile
      const int64_t tend = (tile + 1) * nchunk;
      for (int64_t bn = b + 1; bn < G; ++bn) {
        const int64_t se = seg_start(bn + 1);
        if (seg_start(bn) == se) continue;  // empty range (more CTAs than iterations)
        if (tid == 0) {
          const long long t0 = clock64();
          while (ld_acquire_u32(flags + bn) != epoch) {  // a lost hand-off traps instead of hanging
            __nanosleep(32);
            if (clock64() - t0 > 8000000000LL) __trap();
          }
        }
        __syncthreads();
        const double *f = fix + bn * (int64_t)(64 * kDT);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int bb = 0; bb < 8; ++bb)
#pragma unroll
            for (int h = 0; h < 2; ++h) acc[a][bb][h] += __ldcg(f + ((a * 8 + bb) * 2 + h) * kDT + tid);
        if (se >= tend) break;
      }
    }
    // ---- epilogue: acc[jt][pt][h] = out(j = 32 wj + 8 jt + fr, p = 64 wp + 8 pt + 2 fc + h)
    if (STORE || GRAM) {
      for (int half = 0; half < 2; ++half) {  // stage 128 columns at a time: T[p][kTS]
        __syncthreads();
        double *T = dsm;
        if ((wp >> 1) == half) {
#pragma unroll
          for (int jt = 0; jt < 4; ++jt)
#pragma unroll
            for (int pt = 0; pt < 8; ++pt)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int pp = 64 * (wp & 1) + 8 * pt + 2 * fc + h;
                T[pp * kTS + 32 * wj + 8 * jt + fr] = acc[jt][pt][h];
              }
        }
        __syncthreads();
        const int64_t pb = p0 + 128 * half;
        const int64_t ncol = P - pb < 128 ? (P - pb) : 128;
        if (STORE && ncol > 0) {
          if (L == 1) {  // contiguous J x ncol range out[pb J ..]
            double *dst = out + pb * J;
            for (int64_t e = tid; e < ncol * J; e += kDT) {
              const int pp = (int)(e / J), j = (int)(e - (int64_t)pp * J);
              dst[e] = T[pp * kTS + j];
            }
          } else {
            for (int e = tid; e < 128 * 64; e += kDT) {
              const int pp = e & 127, j = e >> 7;
              if (pp < ncol && j < J) {
                int64_t l = pl0 + 128 * half + pp, r = pr0;
                while (l >= L) { l -= L; ++r; }
                out[l + L * (j + (int64_t)J * r)] = T[pp * kTS + j];
              }
            }
          }
        }
        if (GRAM) {  // G += T^T T on the tensor cores (columns p >= P of T are zero)
#pragma unroll
          for (int s5 = 0; s5 < 5; ++s5) {
            const int t = warp + 8 * s5;
            if (t < 36) {
              int ga, gb;
              gram_tile_ab(t, ga, gb);
              const double *ta = T + fc * kTS + 8 * ga + fr;
              const double *tb = T + fc * kTS + 8 * gb + fr;
#pragma unroll 8
              for (int k0 = 0; k0 < 128; k0 += 4)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(gacc[s5][0]), "+d"(gacc[s5][1])
                             : "d"(ta[k0 * kTS]), "d"(tb[k0 * kTS]));
            }
          }
        }
      }
    }
  }
  if (GRAM) {
    double *gp = gram_partial + b * 4096;
#pragma unroll
    for (int s5 = 0; s5 < 5; ++s5) {
      const int t = warp + 8 * s5;
      if (t < 36) {
        int ga, gb;
        gram_tile_ab(t, ga, gb);
        const int gi = 8 * ga + fr, gj = 8 * gb + 2 * fc;
        gp[gi * 64 + gj] = gacc[s5][0];
        gp[gi * 64 + gj + 1] = gacc[s5][1];
        if (ga != gb) {
          gp[gj * 64 + gi] = gacc[s5][0];
          gp[(gj + 1) * 64 + gi] = gacc[s5][1];
        }
      }
    }
  }
}

// L == 1 variant of ttm_dmma_kernel with a 3-stage cp.async pipeline: X(i, p) = X[i + I p]
// (i contiguous) and A[i + lda j] are copied raw (16-byte units, zero-filled out of range)
// into [p][20] / [j][20] stage buffers, so no register staging pass and two chunks in
// flight while the tensor cores work on the third; X is converted to fp64 at fragment load.
constexpr int kNST = 3;
template <typename Tin>
__host__ __device__ constexpr int l1_chunk() { return sizeof(Tin) == 4 ? 32 : 16; }
__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Epilogue staging of the L == 1 kernel: kTP columns of the tile at a time in its own buffer
// (after the stage ring), so the copies of the next tile's first chunks run during the
// epilogue of this one (the chunk sequence is flat across the CTA's tiles).
template <typename Tin>
__host__ __device__ constexpr int l1_tp() { return sizeof(Tin) == 4 ? 64 : 128; }
template <typename Tin>
__host__ __device__ constexpr size_t l1_stage_bytes() {
  return (size_t)kDP * (l1_chunk<Tin>() + 4) * sizeof(Tin) + 64 * (l1_chunk<Tin>() + 4) * 8;
}

template <typename Tin, bool STORE, bool GRAM>
__global__ void __launch_bounds__(kDT, 1) ttm_dmma_l1_kernel(const Tin *__restrict__ X, int64_t I, int64_t P,
                                                             const double *__restrict__ A, int64_t lda, int J,
                                                             double *__restrict__ out, double *__restrict__ gram_partial) {
  extern __shared__ __align__(16) double dsm[];
  constexpr int kDKt = l1_chunk<Tin>(), kSt = kDKt + 4;  // i per chunk; stage row stride (= 4 mod 16)
  constexpr int kVX = 16 / sizeof(Tin);                 // elements of X per 16-byte unit
  constexpr int kXStage = kDP * kSt * (int)sizeof(Tin);  // bytes
  constexpr int kAStage = 64 * kSt * 8;
  constexpr int kQX = kDKt / kVX;                        // 16-byte units per X row of a chunk
  constexpr int kUXT = kDP * kQX / kDT;                 // X units per thread per chunk
  constexpr int kUAT = 64 * (kDKt / 2) / kDT;            // A units per thread per chunk
  constexpr int kTP = l1_tp<Tin>();                     // epilogue columns per pass
  static_assert(kDP * kQX % kDT == 0 && 64 * (kDKt / 2) % kDT == 0, "unit split");
  unsigned char *sbase = reinterpret_cast<unsigned char *>(dsm);
  double *T = reinterpret_cast<double *>(sbase + kNST * (kXStage + kAStage));  // [kTP][kTS]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wj = warp & 1, wp = warp >> 1;
  const int fr = lane >> 2, fc = lane & 3;
  const int64_t ntiles = (P + kDP - 1) / kDP;
  const int nchunk = (int)((I + kDKt - 1) / kDKt);
  const int64_t mytiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = mytiles * nchunk;
  // Gram tiles of this warp: t = warp + 8 s (s < 5, t < 36)
  double gacc[5][2];
#pragma unroll
  for (int s5 = 0; s5 < 5; ++s5) gacc[s5][0] = gacc[s5][1] = 0.0;
  // per-thread copy assignment (fixed for every chunk): X unit k -> row pp = xr + (kDT / kQX) k,
  // column iq = xq; A unit k -> row j = ar + (kDT / (kDKt / 2)) k, column aq
  const int xr = tid / kQX, xq = tid % kQX;
  const int ar = tid / (kDKt / 2), aq = tid % (kDKt / 2);
  const double *abase = A + 2 * aq + lda * ar;

  auto issue = [&](int64_t g) {  // flat chunk g of this CTA: tile g / nchunk, chunk g % nchunk
    const int64_t tk = g / nchunk;
    const int ch = (int)(g - tk * nchunk);
    const int64_t p0 = (blockIdx.x + tk * gridDim.x) * kDP;
    const Tin *xbase = X + kVX * xq + I * (p0 + xr);
    const int st = (int)(g % kNST);
    Tin *xs = reinterpret_cast<Tin *>(sbase + st * (kXStage + kAStage));
    double *as = reinterpret_cast<double *>(sbase + st * (kXStage + kAStage) + kXStage);
    const int64_t i0 = (int64_t)ch * kDKt;
    const bool iok = i0 + kVX * xq < I;
#pragma unroll
    for (int k = 0; k < kUXT; ++k) {
      const int pp = xr + (kDT / kQX) * k;
      const bool ok = iok && p0 + pp < P;
      cp_async16(xs + pp * kSt + kVX * xq, ok ? (const void *)(xbase + i0 + I * (int64_t)((kDT / kQX) * k)) : (const void *)X,
                 ok);
    }
    const bool aiok = i0 + 2 * aq < I;
#pragma unroll
    for (int k = 0; k < kUAT; ++k) {
      const int j = ar + (kDT / (kDKt / 2)) * k;
      const bool ok = aiok && j < J;
      cp_async16(as + j * kSt + 2 * aq, ok ? (const void *)(abase + i0 + lda * (int64_t)((kDT / (kDKt / 2)) * k)) : (const void *)A,
                 ok);
    }
  };

#pragma unroll
  for (int s = 0; s < kNST - 1; ++s) {
    if (s < total) issue(s);
    cp_async_commit();
  }
  double acc[4][8][2];
  int ch = 0;
  int64_t tk = 0;
  for (int64_t g = 0; g < total; ++g) {
    if (ch == 0) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) { acc[a][b][0] = 0.0; acc[a][b][1] = 0.0; }
    }
    cp_async_wait<kNST - 2>();
    __syncthreads();
    if (g + kNST - 1 < total) issue(g + kNST - 1);
    cp_async_commit();
    const int st = (int)(g % kNST);
    const Tin *xs = reinterpret_cast<const Tin *>(sbase + st * (kXStage + kAStage));
    const double *as = reinterpret_cast<const double *>(sbase + st * (kXStage + kAStage) + kXStage);
#pragma unroll
    for (int ks = 0; ks < kDKt / 4; ++ks) {
      double af[4], bf[8];
#pragma unroll
      for (int jt = 0; jt < 4; ++jt) af[jt] = as[(32 * wj + 8 * jt + fr) * kSt + 4 * ks + fc];
#pragma unroll
      for (int pt = 0; pt < 8; ++pt) bf[pt] = (double)xs[(64 * wp + 8 * pt + fr) * kSt + 4 * ks + fc];
#pragma unroll
      for (int jt = 0; jt < 4; ++jt)
#pragma unroll
        for (int pt = 0; pt < 8; ++pt)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[jt][pt][0]), "+d"(acc[jt][pt][1])
                       : "d"(af[jt]), "d"(bf[pt]));
    }
    if (++ch < nchunk) continue;
    // ---- tile done: epilogue (L == 1: the tile is one contiguous range out[p0 J ..]); columns
    // p >= P and rows j >= J of the tile are exact zeros (zero-filled copies)
    ch = 0;
    const int64_t p0 = (blockIdx.x + tk * gridDim.x) * kDP;
    ++tk;
    if (STORE || GRAM) {
#pragma unroll 1
      for (int part = 0; part < kDP / kTP; ++part) {
        __syncthreads();  // T free (previous pass / tile done reading it)
        if ((64 * wp) / kTP == part) {
#pragma unroll
          for (int jt = 0; jt < 4; ++jt)
#pragma unroll
            for (int pt = 0; pt < 8; ++pt)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int pp = (64 * wp) % kTP + 8 * pt + 2 * fc + h;
                T[pp * kTS + 32 * wj + 8 * jt + fr] = acc[jt][pt][h];
              }
        }
        __syncthreads();
        const int64_t pb = p0 + kTP * part;
        const int64_t ncol = P - pb < kTP ? (P - pb) : kTP;
        if (STORE && ncol > 0) {
          double *dst = out + pb * J;
          for (int e = tid; e < (int)ncol * J; e += kDT) {
            const int pp = e / J, j = e - pp * J;
            dst[e] = T[pp * kTS + j];
          }
        }
        if (GRAM) {
#pragma unroll
          for (int s5 = 0; s5 < 5; ++s5) {
            const int t = warp + 8 * s5;
            if (t < 36) {
              int a, b;
              gram_tile_ab(t, a, b);
              const double *ta = T + fc * kTS + 8 * a + fr;
              const double *tb = T + fc * kTS + 8 * b + fr;
#pragma unroll 8
              for (int k0 = 0; k0 < kTP; k0 += 4)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(gacc[s5][0]), "+d"(gacc[s5][1])
                             : "d"(ta[k0 * kTS]), "d"(tb[k0 * kTS]));
            }
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  if (GRAM) {
    double *gp = gram_partial + (int64_t)blockIdx.x * 4096;
#pragma unroll
    for (int s5 = 0; s5 < 5; ++s5) {
      const int t = warp + 8 * s5;
      if (t < 36) {
        int a, b;
        gram_tile_ab(t, a, b);
        const int gi = 8 * a + fr, gj = 8 * b + 2 * fc;
        gp[gi * 64 + gj] = gacc[s5][0];
        gp[gi * 64 + gj + 1] = gacc[s5][1];
        if (a != b) {
          gp[gj * 64 + gi] = gacc[s5][0];
          gp[(gj + 1) * 64 + gi] = gacc[s5][1];
        }
      }
    }
  }
}

template <typename Tin>
void launch_ttm_dfma(Ctx &c, const Tin *X, ModeView v, const double *A, int64_t lda, int J, double *out, double *gram) {
  const int64_t P = v.L * v.R;
  const int64_t ntiles = (P + kDP - 1) / kDP;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, c.num_sms));
  static const bool use_dfma = RT_EXP_GETENV("RTUCKER_NO_DMMA") != nullptr;
  DevBuf<double> part;
  if (gram) part.alloc(c, (size_t)grid * 4096);
  // cp.async pipeline for L == 1 with 16-byte aligned rows of X and A
  const bool l1 = !use_dfma && v.L == 1 && (v.I % (16 / sizeof(Tin))) == 0 && (lda % 2) == 0 &&
                  (((uintptr_t)X) & 15) == 0 && (((uintptr_t)A) & 15) == 0;
  if (l1) {
    const size_t smem = kNST * l1_stage_bytes<Tin>() + sizeof(double) * l1_tp<Tin>() * kTS;
#define RT_DL(ST, GR)                                                                                 \
  do {                                                                                                \
    auto k = ttm_dmma_l1_kernel<Tin, ST, GR>;                                                         \
    smem_attr(k, smem);         \
    RT_LAUNCH(c, k, grid, kDT, smem, X, v.I, P, A, lda, J, out, part.p);                              \
  } while (0)
    if (out && gram) RT_DL(true, true);
    else if (out) RT_DL(true, false);
    else RT_DL(false, true);
#undef RT_DL
  } else if (use_dfma) {
    const size_t smem = std::max(sizeof(double) * (kDK * kDS + kDK * 64), sizeof(double) * 128 * 65);
#define RT_DF(ST, GR)                                                                                 \
  do {                                                                                                \
    auto k = ttm_dfma_kernel<Tin, ST, GR>;                                                            \
    smem_attr(k, smem);         \
    RT_LAUNCH(c, k, grid, kDT, smem, X, v.L, v.I, v.R, A, lda, J, out, part.p);                       \
  } while (0)
    if (out && gram) RT_DF(true, true);
    else if (out) RT_DF(true, false);
    else RT_DF(false, true);
#undef RT_DF
  } else {
    // stream-K over all SMs (the tile list alone is often shorter than the SM count)
    const int sk_grid = c.num_sms;
    if (c.sk_n < sk_grid) {
      if (c.sk_flags) RT_CUDA(cudaFree(c.sk_flags));
      RT_CUDA(cudaMalloc((void **)&c.sk_flags, sizeof(unsigned) * sk_grid));
      RT_CUDA(cudaMemsetAsync(c.sk_flags, 0, sizeof(unsigned) * sk_grid, c.stream));
      c.sk_n = sk_grid;
    }
    if (++c.sk_epoch == 0) ++c.sk_epoch;  // 0 is the initial flag value
    // a captured launch replays with the same epoch: reset the flags inside the graph
    if (c.capturing) RT_CUDA(cudaMemsetAsync(c.sk_flags, 0, sizeof(unsigned) * sk_grid, c.stream));
    DevBuf<double> fix(c, (size_t)sk_grid * 64 * kDT);
    if (gram) part.alloc(c, (size_t)sk_grid * 4096);
    const size_t smem = std::max(sizeof(double) * (kDP * kMX + kDK * kMA), sizeof(double) * 128 * kTS);
#define RT_DM(ST, GR)                                                                                 \
  do {                                                                                                \
    auto k = ttm_dmma_kernel<Tin, ST, GR>;                                                            \
    smem_attr(k, smem);         \
    RT_LAUNCH(c, k, sk_grid, kDT, smem, X, v.L, v.I, v.R, A, lda, J, out, part.p, fix.p, c.sk_flags, c.sk_epoch); \
  } while (0)
    if (out && gram) RT_DM(true, true);
    else if (out) RT_DM(true, false);
    else RT_DM(false, true);
#undef RT_DM
    if (gram) RT_LAUNCH(c, gram_reduce2_kernel, J * J, 128, 0, part.p, sk_grid, J, gram);
    return;
  }
  if (gram) RT_LAUNCH(c, gram_reduce2_kernel, J * J, 128, 0, part.p, grid, J, gram);
}

template <typename Tin, typename Tout, typename Tmul>
void ttm_dispatch(Ctx &c, const Tin *X, ModeView v, const double *A, int64_t lda, int J, Tout *out,
                  double *gram) {
  if (J <= 16) return launch_ttm<Tin, Tout, Tmul, 16>(c, X, v, A, lda, J, J, out, gram);
  if (J <= 32) return launch_ttm<Tin, Tout, Tmul, 32>(c, X, v, A, lda, J, J, out, gram);
  if (J <= 64) return launch_ttm<Tin, Tout, Tmul, 64>(c, X, v, A, lda, J, J, out, gram);
  // J > 64: blocks of 64 output columns, then the Gram of the stored output
  DevBuf<Tout> tmp;
  Tout *o = out;
  if (!o) {
    tmp.alloc(c, (size_t)v.L * J * v.R);
    o = tmp.p;
  }
  for (int j0 = 0; j0 < J; j0 += 64)
    launch_ttm<Tin, Tout, Tmul, 64>(c, X, v, A + lda * j0, lda, std::min(64, J - j0), J, o + v.L * j0, nullptr);
  if (gram) mode_gram_t<Tout>(c, o, ModeView{v.L, J, v.R}, gram);
}

}  // namespace

void slab_gram(Ctx &c, const double *B, ModeView v, double *gram) {
  RT_REQUIRE(v.L <= 64 && v.I <= 64, "slab_gram: L, J <= 64");
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(v.R, (int64_t)c.num_sms * 2));
  DevBuf<double> part(c, (size_t)g * 4096);
  RT_LAUNCH(c, slab_gram_kernel, g, 256, 0, B, (int)v.L, (int)v.I, v.R, part.p);
  RT_LAUNCH(c, gram_reduce2_kernel, (int)(v.I * v.I), 128, 0, part.p, g, (int)v.I, gram);
}

void mode_gram(Ctx &c, const void *B, DT t, ModeView v, double *gram) {
  if (t == DT::F64) mode_gram_t<double>(c, (const double *)B, v, gram);
  else mode_gram_t<float>(c, (const float *)B, v, gram);
}

bool ttm_dense_tc(Ctx &c, const void *X, DT in, ModeView v, const double *A, int64_t lda, int J, void *out, DT outT,
                  bool mul_f64, double *gram);

void ttm_dense(Ctx &c, const void *X, DT in, ModeView v, const double *A, int64_t lda, int J,
               void *out, DT outT, bool mul_f64, double *gram, const uint32_t *colmax) {
  RT_REQUIRE(out || gram, "ttm: nothing to compute");
  if (ttm_dense_tc(c, X, in, v, A, lda, J, out, outT, mul_f64, gram)) return;
  // HYBRID mode-1 B-pass on fp32 data: fp64-level products from exact int8 tensor-core slices
  if (in == DT::F32 && !mul_f64 && (!out || outT == DT::F64) &&
      ttm_ozaki(c, (const float *)X, v, A, lda, J, (double *)out, gram, colmax))
    return;
  // fp64 output (HYBRID / FP64 policies, fp64 data): DFMA kernel
  if (J <= 64 && (!out || outT == DT::F64) && (in == DT::F64 || mul_f64 || outT == DT::F64)) {
    if (in == DT::F64) launch_ttm_dfma<double>(c, (const double *)X, v, A, lda, J, (double *)out, gram);
    else launch_ttm_dfma<float>(c, (const float *)X, v, A, lda, J, (double *)out, gram);
    return;
  }
  if (in == DT::F64) {
    RT_REQUIRE(outT == DT::F64, "ttm: fp64 input needs fp64 output");
    ttm_dispatch<double, double, double>(c, (const double *)X, v, A, lda, J, (double *)out, gram);
  } else if (outT == DT::F64 || mul_f64) {
    RT_REQUIRE(outT == DT::F64, "ttm: fp64 products imply fp64 output");
    ttm_dispatch<float, double, double>(c, (const float *)X, v, A, lda, J, (double *)out, gram);
  } else {
    ttm_dispatch<float, float, float>(c, (const float *)X, v, A, lda, J, (float *)out, gram);
  }
}

bool ttm_dense_tc(Ctx &c, const void *X, DT in, ModeView v, const double *A, int64_t lda, int J, void *out, DT outT,
                  bool mul_f64, double *gram) {
  // tensor-core B-pass: FAST policy only (fp32 data, fp32 B, mode with L == 1).  Under HYBRID
  // the B-pass on the fp32 input keeps fp64 products: at C4 (rank-50 gap ~5e-7 lambda_1) an
  // fp32-accurate B moves the relative error by 5e-4 (3xTF32) / 9e-5 (FFMA), beyond the 1e-5
  // parity bound (scripts/dbg_c4_policy.py)
  if (in != DT::F32 || mul_f64 || !out || v.L != 1 || outT != DT::F32) return false;
  if (!bpass_tc_mn(c, (const float *)X, v, A, lda, J, out, outT == DT::F64)) return false;
  if (gram) mode_gram(c, out, outT, ModeView{1, J, v.R}, gram);
  return true;
}

}  // namespace rt
