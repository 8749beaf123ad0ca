// Dense mode-n sketch Y = X_(n) Omega_n (Alg 1 line 1; Alg 2 line 2, Alg 3 line 2)
// without materialising the unfolding, Omega generated on the fly.
//
// SIMT kernel (the tensor-core 3xTF32 variant lives in sketch_tc.cu).  Each CTA owns a
// tile of TI rows i and a contiguous range of unfolding columns c = l + L*r; it streams
// CK columns at a time: X tile -> smem (coalesced along the contiguous index of the
// (L, I, R) view), Omega chunk generated into smem, register-blocked 4x4 FMAs.  Per-CTA
// partial Y tiles are summed in a fixed order by reduce_splits (deterministic).
// The squared Frobenius norm of X is fused in (each element is read exactly once).
#include "kernels.h"
#include "philox.cuh"
#include <type_traits>

namespace rt {

namespace {

constexpr int kThreads = 256;
template <int LP> constexpr int chunk_cols() { return LP >= 32 ? 32 : 16; }  // columns per chunk

template <typename Tin, typename Tmul, int LP>
__global__ void __launch_bounds__(kThreads) sketch_simt_kernel(
    const Tin *__restrict__ X, int64_t L, int64_t I, int64_t R, int64_t cols_per_split,
    uint64_t seed, int mode, int ell, int64_t k0, int64_t col_offset,
    double *__restrict__ partial, double *__restrict__ norm_partial) {
  constexpr int TI = 4096 / LP;   // rows per tile
  constexpr int NK = LP / 4;      // k-groups
  constexpr int kCK = chunk_cols<LP>();
  __shared__ __align__(16) Tmul sX[kCK][TI];
  __shared__ __align__(16) Tmul sO[kCK][LP];
  __shared__ double sred[kThreads / 32];

  const int tid = threadIdx.x;
  const int tk = tid % NK, ti = tid / NK;
  const int64_t i0 = (int64_t)blockIdx.x * TI;
  const int64_t C = L * R;
  const int64_t cbeg = (int64_t)blockIdx.y * cols_per_split;
  const int64_t cend = min(C, cbeg + cols_per_split);

  // Philox blocks that cover global sketch columns [k0, k0 + ell).
  const int64_t jb0 = k0 >> 2;
  const int nb = (int)(((k0 + ell - 1) >> 2) - jb0 + 1);

  // zero the padding columns of the Omega tile once
  for (int e = tid; e < kCK * LP; e += kThreads) sO[e / LP][e % LP] = Tmul(0);

  double accd[4][4];
  Tmul acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) { accd[a][b] = 0.0; acc[a][b] = Tmul(0); }
  double nsq = 0.0;

  for (int64_t c0 = cbeg; c0 < cend; c0 += kCK) {
    __syncthreads();
    const int64_t l0 = c0 % L, rb = c0 / L;  // one 64-bit divide per chunk
    // ---- X tile: (ii, cc) -> X[l + L*(i + I*r)] with c = l + L*r
    for (int e = tid; e < kCK * TI; e += kThreads) {
      int ii, cc;
      if (L == 1) { ii = e % TI; cc = e / TI; } else { cc = e % kCK; ii = e / kCK; }
      const int64_t i = i0 + ii, c = c0 + cc;
      Tmul x = Tmul(0);
      if (i < I && c < cend) {
        int64_t off;
        if (L == 1) {
          off = i + I * c;
        } else {
          int64_t l = l0 + cc, r = rb;
          while (l >= L) { l -= L; ++r; }
          off = l + L * (i + I * r);
        }
        const Tin xv = __ldg(X + off);
        x = (Tmul)xv;
        nsq += (double)xv * (double)xv;
      }
      sX[cc][ii] = x;
    }
    // ---- Omega chunk: rows c0..c0+CK, columns k0..k0+ell (Philox block granularity)
    for (int e = tid; e < kCK * nb; e += kThreads) {
      const int cc = e / nb, jb = e % nb;
      const int64_t c = c0 + cc;
      if (c >= cend) continue;
      const uint4 w = omega_words(seed, mode, 0, (uint64_t)(c + col_offset), (uint32_t)(jb0 + jb));
      Normal4<Tmul> z(w);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t kk = 4 * (jb0 + jb) + q - k0;
        if (kk >= 0 && kk < ell) sO[cc][kk] = z.v[q];
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int cc = 0; cc < kCK; ++cc) {
      Tmul a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = sX[cc][ti * 4 + q]; b[q] = sO[cc][tk * 4 + q]; }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
    }
    // flush the chunk sum (<= 32 products) into the fp64 accumulators
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) { accd[p][q] += (double)acc[p][q]; acc[p][q] = Tmul(0); }
  }
  // ---- per-CTA partial: partial[split][k*I + i]
  double *dst = partial + (int64_t)blockIdx.y * I * ell;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int64_t i = i0 + ti * 4 + p;
    if (i >= I) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = tk * 4 + q;
      if (k < ell) dst[(int64_t)k * I + i] = accd[p][q];
    }
  }
  if (norm_partial) {
    for (int o = 16; o; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
    if ((tid & 31) == 0) sred[tid >> 5] = nsq;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) s += sred[w];
      norm_partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
  }
}

// Y[e] = sum_s partial[s*n + e], fixed order.
__global__ void reduce_splits_kernel(const double *__restrict__ partial, int nsplit, int64_t n,
                                     double *__restrict__ Y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nsplit; ++k) s += partial[(int64_t)k * n + e];
    Y[e] = s;
  }
}

template <typename Tout>
__global__ void omega_rows_kernel(uint64_t seed, int mode, const int64_t *__restrict__ cols,
                                  int64_t n, int ell, int64_t k0, Tout *__restrict__ out) {
  const int64_t jb0 = k0 >> 2;
  const int nb = (int)(((k0 + ell - 1) >> 2) - jb0 + 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * nb;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / nb;
    const int jb = (int)(e % nb);
    const uint4 w = omega_words(seed, mode, 0, (uint64_t)cols[i], (uint32_t)(jb0 + jb));
    Normal4<Tout> z(w);
    for (int q = 0; q < 4; ++q) {
      const int64_t kk = 4 * (jb0 + jb) + q - k0;
      if (kk >= 0 && kk < ell) out[i + n * kk] = z.v[q];
    }
  }
}

__global__ void philox_raw_kernel(const uint32_t *__restrict__ ctr, int64_t n, uint32_t k0,
                                  uint32_t k1, uint32_t *__restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint4 c = make_uint4(ctr[4 * e], ctr[4 * e + 1], ctr[4 * e + 2], ctr[4 * e + 3]);
    uint4 w = philox4x32_10(c, k0, k1);
    out[4 * e] = w.x; out[4 * e + 1] = w.y; out[4 * e + 2] = w.z; out[4 * e + 3] = w.w;
  }
}

template <typename Tin, typename Tmul, int LP>
void launch_sketch(Ctx &c, const Tin *X, ModeView v, int mode, int ell, int64_t k0, uint64_t seed,
                   int64_t col_offset, double *Y, double *normsq) {
  constexpr int TI = 4096 / LP;
  constexpr int kCK = chunk_cols<LP>();
  const int gx = ceil_div(v.I, TI);
  const int64_t C = v.L * v.R;
  // enough CTAs for ~4 per SM, each with at least 4 chunks of columns
  int64_t target = std::max<int64_t>(1, (int64_t)c.num_sms * 4 / gx);
  int64_t maxsplit = std::max<int64_t>(1, C / (4 * kCK));
  int64_t nsplit = std::min<int64_t>(target, maxsplit);
  int64_t cps = ((C + nsplit - 1) / nsplit + kCK - 1) / kCK * kCK;
  nsplit = (C + cps - 1) / cps;
  DevBuf<double> part(c, (size_t)nsplit * v.I * ell);
  DevBuf<double> npart;
  if (normsq) npart.alloc(c, (size_t)nsplit * gx);
  dim3 grid(gx, (unsigned)nsplit);
  RT_LAUNCH(c, (sketch_simt_kernel<Tin, Tmul, LP>), grid, kThreads, 0, X, v.L, v.I, v.R, cps,
            seed, mode, ell, k0, col_offset, part.p, normsq ? npart.p : nullptr);
  const int64_t n = v.I * ell;
  RT_LAUNCH(c, reduce_splits_kernel, ceil_div(n, 256) > 1024 ? 1024 : ceil_div(n, 256), 256, 0,
            part.p, (int)nsplit, n, Y);
  if (normsq) sum_vec(c, npart.p, (int64_t)nsplit * gx, normsq);
}

// ------------------------------------------------------------ fp64-product sketch ----
// Y[i, k] = sum_p X(l, i, r) Omega(p, k), p = l + L r, with fp64 products and sums (X fp32
// or fp64; normals fp32 or fp64 per reading R3), on the fp64 tensor cores (mma.m8n8k4).
// A CTA owns 128 rows x 64 sketch columns and a contiguous range of p (split-K); warp
// (wm = w & 3, wn = w >> 2) the 32 x 32 block rows 32 wm.., columns 32 wn.. (4 x 4 MMA
// tiles).  X and Omega are staged 16 values of p at a time (Omega generated into shared
// memory: ceil(I/128) row tiles regenerate it); partials per split are summed in a fixed
// order (deterministic).
constexpr int kSP = 16;   // p per chunk
constexpr int kSX = 136;  // Xs row stride (doubles, = 8 mod 16): conflict-free A fragments
constexpr int kSO = 72;   // Os row stride
// Shared memory is double buffered (dynamic, kSketchDfmaSmem bytes): per chunk a warp stores the
// NEXT chunk (register-prefetched X, generated or explicit Omega) into the other buffer, issues
// the global loads of the chunk after it and then runs the MMAs of the current buffer: one CTA
// barrier per chunk, and the loads are in flight during the MMA block.  L1 (mode-1 layout) is a
// template parameter and CTAs whose 128 rows are all inside I take unpredicated loads (ncu on
// the C4 mode-2 sketch of B: the single-buffered form issued ~20 instructions per DMMA).  The
// (l, r) split of a thread's column p is advanced incrementally (one division per CTA).
constexpr size_t kSketchDfmaSmem = (size_t)2 * kSP * (kSX + kSO) * sizeof(double);
template <typename Tin, typename TN, bool L1>
__global__ void __launch_bounds__(256, 2) sketch_dfma_kernel(const Tin *__restrict__ X, int64_t L, int64_t I, int64_t R,
                                                             int64_t cols_per_split, uint64_t seed, int mode, int ell,
                                                             int64_t k0, int64_t col_offset, double *__restrict__ partial,
                                                             double *__restrict__ norm_partial,
                                                             const double *__restrict__ Om = nullptr) {
  extern __shared__ __align__(16) double sk_smem[];
  double *const XsB = sk_smem;                  // [2][kSP * kSX]
  double *const OsB = sk_smem + 2 * kSP * kSX;  // [2][kSP * kSO]
  __shared__ double sred[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2, fr = lane >> 2, fc = lane & 3;
  const int64_t i0 = (int64_t)blockIdx.x * 128;
  const int64_t P = L * R;
  const int64_t pbeg = (int64_t)blockIdx.y * cols_per_split, pend = min(P, pbeg + cols_per_split);
  const int64_t jb0 = k0 >> 2;
  const int nb = (int)(((k0 + ell - 1) >> 2) - jb0 + 1);
  const bool rows_full = i0 + 128 <= I;
  const bool want_norm = norm_partial != nullptr;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[a][q][0] = acc[a][q][1] = 0.0;
  double nsq = 0.0;
  for (int e = tid; e < 2 * kSP * kSO; e += 256) OsB[e] = 0.0;
  __syncthreads();  // the zero fill precedes every Omega store
  // X staging with a register prefetch (8 values per thread and chunk)
  //   L1 : element e = tid + 256 q: row ii = tid & 127, column pp = (tid >> 7) + 2 q (coalesced along i)
  //   !L1: column pp = tid % 16, row ii = tid / 16 + 16 q (coalesced along p = l)
  constexpr int NQ = kSP * 128 / 256;
  Tin pre[NQ];
  double opre[4];
  const int xoff = L1 ? (tid >> 7) * kSX + (tid & 127) : (tid % kSP) * kSX + tid / kSP;
  constexpr int xstep = L1 ? 2 * kSX : 16;
  // column (tid % 16) of the chunk: p = l + L r, advanced by kSP per chunk
  const int ppc = tid % kSP;
  int64_t cl = 0, cr = 0;
  if (!L1 || Om) {
    const int64_t p = pbeg + ppc;
    cr = p / L;
    cl = p - cr * L;
  }
  auto advance = [&]() {
    if (L1) {
      cr += kSP;  // l = 0, r = p
    } else {
      cl += kSP;
      while (cl >= L) { cl -= L; ++cr; }
    }
  };
  // loads of the chunk at p0; (cl, cr) must describe column p0 + ppc
  auto load_chunk = [&](int64_t p0) {
    if (Om) {
      const bool pok = p0 + ppc < pend;
      const double *om = Om + cl + L * (int64_t)ell * cr;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int kk = tid / kSP + 16 * t;
        opre[t] = (pok && kk < ell) ? om[L * kk] : 0.0;
      }
    }
    if (L1) {
      const int64_t i = i0 + (tid & 127);
      const int64_t pf = p0 + (tid >> 7);
      const Tin *src = X + i + I * pf;
      if (rows_full && p0 + kSP <= pend) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) pre[q] = src[(int64_t)(2 * q) * I];
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q) pre[q] = (i < I && pf + 2 * q < pend) ? src[(int64_t)(2 * q) * I] : Tin(0);
      }
    } else {
      const bool pok = p0 + ppc < pend;
      const int64_t ib = i0 + tid / kSP;
      const Tin *src = X + cl + L * I * cr + L * ib;
      if (rows_full && p0 + kSP <= pend) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) pre[q] = src[(int64_t)(16 * q) * L];
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q) pre[q] = (pok && ib + 16 * q < I) ? src[(int64_t)(16 * q) * L] : Tin(0);
      }
    }
  };
  // stores of the prefetched chunk at p0 into buffer b (Omega generated here when not explicit)
  auto store_chunk = [&](int64_t p0, int b) {
    double *Xs = XsB + b * (kSP * kSX);
    double *Os = OsB + b * (kSP * kSO);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double v = (double)pre[q];
      if (want_norm) nsq = fma(v, v, nsq);
      Xs[xoff + q * xstep] = v;
    }
    // Omega chunk: rows p0.., columns k0.. (Philox block granularity); rows past pend are 0.
    // Explicit Omega (subspace iteration, deferred shrink): Om stored (L, ell, R), Omega(p, k) = Om(l, k, r).
    if (Om) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int kk = tid / kSP + 16 * t;
        if (kk < ell) Os[ppc * kSO + kk] = opre[t];
      }
    } else {
      for (int e = tid; e < kSP * nb; e += 256) {
        const int pp = e / nb, jb = e - pp * nb;
        const int64_t p = p0 + pp;
        const uint4 w = omega_words(seed, mode, 0, (uint64_t)(p + col_offset), (uint32_t)(jb0 + jb));
        Normal4<TN> z(w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t kk = 4 * (jb0 + jb) + q - k0;
          if (kk >= 0 && kk < ell) Os[pp * kSO + kk] = p < pend ? (double)z.v[q] : 0.0;
        }
      }
    }
  };
  if (pbeg < pend) {
    load_chunk(pbeg);
    store_chunk(pbeg, 0);
    if (pbeg + kSP < pend) {
      advance();
      load_chunk(pbeg + kSP);
    }
  }
  __syncthreads();
  int buf = 0;
  for (int64_t p0 = pbeg; p0 < pend; p0 += kSP, buf ^= 1) {
    if (p0 + kSP < pend) {
      store_chunk(p0 + kSP, buf ^ 1);
      if (p0 + 2 * kSP < pend) {  // in flight during the MMA block
        advance();
        load_chunk(p0 + 2 * kSP);
      }
    }
    const double *Xs = XsB + buf * (kSP * kSX);
    const double *Os = OsB + buf * (kSP * kSO);
#pragma unroll
    for (int ks = 0; ks < kSP / 4; ++ks) {
      double af[4], bf[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) af[mt] = Xs[(4 * ks + fc) * kSX + 32 * wm + 8 * mt + fr];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = Os[(4 * ks + fc) * kSO + 32 * wn + 8 * nt + fr];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1])
                       : "d"(af[mt]), "d"(bf[nt]));
    }
    __syncthreads();
  }
  // C fragment: acc[mt][nt][h] = Y(i = 32 wm + 8 mt + fr, k = 32 wn + 8 nt + 2 fc + h)
  double *dst = partial + (int64_t)blockIdx.y * I * ell;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int64_t i = i0 + 32 * wm + 8 * mt + fr;
    if (i >= I) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 32 * wn + 8 * nt + 2 * fc + h;
        if (k < ell) dst[(int64_t)k * I + i] = acc[mt][nt][h];
      }
  }
  if (norm_partial) {
    for (int o = 16; o; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
    if ((tid & 31) == 0) sred[tid >> 5] = nsq;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += sred[w];
      norm_partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
  }
}

template <typename Tin, typename TN>
void launch_sketch_dfma(Ctx &c, const Tin *X, ModeView v, int mode, int ell, int64_t k0, uint64_t seed,
                        int64_t col_offset, double *Y, double *normsq, const double *Om = nullptr) {
  const int gx = ceil_div(v.I, 128);
  const int64_t P = v.L * v.R;
  // one full wave: 2 CTAs of 256 threads per SM (126 registers per thread)
  int64_t target = std::max<int64_t>(1, (int64_t)c.num_sms * 2 / gx);
  int64_t maxsplit = std::max<int64_t>(1, P / (4 * kSP));
  int64_t nsplit = std::min<int64_t>(target, maxsplit);
  int64_t cps = ((P + nsplit - 1) / nsplit + kSP - 1) / kSP * kSP;
  nsplit = (P + cps - 1) / cps;
  DevBuf<double> part(c, (size_t)nsplit * v.I * ell);
  DevBuf<double> npart;
  if (normsq) npart.alloc(c, (size_t)nsplit * gx);
  dim3 grid(gx, (unsigned)nsplit);
  if (v.L == 1) {
    smem_attr(sketch_dfma_kernel<Tin, TN, true>, kSketchDfmaSmem);
    RT_LAUNCH(c, (sketch_dfma_kernel<Tin, TN, true>), grid, 256, kSketchDfmaSmem, X, v.L, v.I, v.R, cps, seed, mode, ell,
              k0, col_offset, part.p, normsq ? npart.p : nullptr, Om);
  } else {
    smem_attr(sketch_dfma_kernel<Tin, TN, false>, kSketchDfmaSmem);
    RT_LAUNCH(c, (sketch_dfma_kernel<Tin, TN, false>), grid, 256, kSketchDfmaSmem, X, v.L, v.I, v.R, cps, seed, mode, ell,
              k0, col_offset, part.p, normsq ? npart.p : nullptr, Om);
  }
  const int64_t n = v.I * ell;
  RT_LAUNCH(c, reduce_splits_kernel, ceil_div(n, 256) > 1024 ? 1024 : ceil_div(n, 256), 256, 0, part.p, (int)nsplit, n,
            Y);
  if (normsq) sum_vec(c, npart.p, (int64_t)nsplit * gx, normsq);
}

template <typename Tin, typename Tmul>
void sketch_dispatch(Ctx &c, const Tin *X, ModeView v, int mode, int ell, int64_t k0,
                     uint64_t seed, int64_t col_offset, double *Y, double *normsq, uint32_t *colmax = nullptr) {
  // Column blocks of <= 64 sketch columns; the norm is fused into the first block only.
  for (int kb = 0; kb < ell; kb += 64) {
    const int e = std::min(64, ell - kb);
    double *Yb = Y + (int64_t)kb * v.I;
    double *ns = kb == 0 ? normsq : nullptr;
    if constexpr (std::is_same<Tin, float>::value && std::is_same<Tmul, float>::value) {
      if (sketch_tc_mn(c, X, v, mode, e, k0 + kb, seed, col_offset, Yb, ns, kb == 0 ? colmax : nullptr)) continue;
      if (kb == 0 && colmax) column_maxima(c, (const float *)X, v, colmax);  // TC path declined
    }
    if (e <= 16)
      launch_sketch<Tin, Tmul, 16>(c, X, v, mode, e, k0 + kb, seed, col_offset, Yb, ns);
    else if (e <= 32)
      launch_sketch<Tin, Tmul, 32>(c, X, v, mode, e, k0 + kb, seed, col_offset, Yb, ns);
    else
      launch_sketch<Tin, Tmul, 64>(c, X, v, mode, e, k0 + kb, seed, col_offset, Yb, ns);
  }
}

}  // namespace

void sketch_dense(Ctx &c, const void *X, DT in, ModeView v, int mode, int ell, int64_t k0,
                  uint64_t seed, int64_t col_offset, bool mul_f64, double *Y, double *normsq, bool normals_f32,
                  uint32_t *colmax) {
  // the column maxima must be valid whenever requested: the tcgen05 mode-1 sketch records them
  // on the fly; any other path computes them here
  if (colmax && (in != DT::F32 || mul_f64)) {
    RT_REQUIRE(in == DT::F32, "sketch: column maxima need fp32 data");
    column_maxima(c, (const float *)X, v, colmax);
    colmax = nullptr;
  }
  if (in == DT::F64 || mul_f64) {
    // fp64 products: DFMA kernel in column blocks of <= 64 (norm fused into the first block)
    for (int kb = 0; kb < ell; kb += 64) {
      const int e = std::min(64, ell - kb);
      double *Yb = Y + (int64_t)kb * v.I;
      double *ns = kb == 0 ? normsq : nullptr;
      if (in == DT::F64) {
        if (normals_f32) launch_sketch_dfma<double, float>(c, (const double *)X, v, mode, e, k0 + kb, seed, col_offset, Yb, ns);
        else launch_sketch_dfma<double, double>(c, (const double *)X, v, mode, e, k0 + kb, seed, col_offset, Yb, ns);
      } else {  // fp32 data with the FP64 policy
        if (normals_f32) launch_sketch_dfma<float, float>(c, (const float *)X, v, mode, e, k0 + kb, seed, col_offset, Yb, ns);
        else launch_sketch_dfma<float, double>(c, (const float *)X, v, mode, e, k0 + kb, seed, col_offset, Yb, ns);
      }
    }
    return;
  }
  sketch_dispatch<float, float>(c, (const float *)X, v, mode, ell, k0, seed, col_offset, Y, normsq, colmax);
}


// Om(l', k, r') = sum_a V[k_n + ell_n a] Omega_m(p(a), k) for the mode-m unfolding columns
// p' = l' + L' r' of B (mode n of size ell_n); p(a) is the column of G = B x_n V(:, :r)^T with
// i_n = a (deferred shrink).  One CTA per (p_lo, p_hi): the r x ell block of
// Omega_m it needs is generated once (the sketch kernels' stream: key (seed, m), counter
// (k >> 2, m, p)), the ell_n x ell outputs are sums over a in index order (deterministic).
template <typename TN>
__global__ void __launch_bounds__(256) omega_fold_kernel(int64_t sn, int r, int ell_n, int ell, int64_t Lb,
                                                         uint64_t seed, int mode, const double *__restrict__ V,
                                                         double *__restrict__ Om) {
  extern __shared__ __align__(16) double fsm[];
  const int ep = (ell + 3) & ~3, kp = (ell_n + 3) & ~3;  // rows padded to 4 (zero-filled)
  double *Os = fsm;                                      // [a][kk], stride ep
  double *Vs = Os + (size_t)r * ep;                      // [a][k], stride kp
  const int64_t plo = (int64_t)blockIdx.x % sn, phi = (int64_t)blockIdx.x / sn;
  const int nb = ep >> 2, tid = threadIdx.x;
  for (int e = tid; e < r * nb; e += blockDim.x) {
    const int a = e / nb, jb = e - a * nb;
    const uint4 w = omega_words(seed, mode, 0, (uint64_t)(plo + sn * (a + (int64_t)r * phi)), (uint32_t)jb);
    Normal4<TN> z(w);
#pragma unroll
    for (int q = 0; q < 4; ++q) Os[a * ep + 4 * jb + q] = 4 * jb + q < ell ? (double)z.v[q] : 0.0;
  }
  for (int e = tid; e < kp * r; e += blockDim.x) {
    const int a = e / kp, k = e - a * kp;
    Vs[a * kp + k] = k < ell_n ? V[k + (int64_t)ell_n * a] : 0.0;
  }
  __syncthreads();
  // thread = 4 k x 4 kk outputs: per a two 32-byte loads of each operand and 16 independent FMAs
  const int nkb = kp >> 2;
  for (int e = tid; e < nkb * nb; e += blockDim.x) {
    const int q = e / nkb, kb = e - q * nkb;
    double s[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int u = 0; u < 4; ++u) s[i][u] = 0.0;
#pragma unroll 2
    for (int a = 0; a < r; ++a) {
      const double2 v0 = *(const double2 *)&Vs[a * kp + 4 * kb], v1 = *(const double2 *)&Vs[a * kp + 4 * kb + 2];
      const double2 o0 = *(const double2 *)&Os[a * ep + 4 * q], o1 = *(const double2 *)&Os[a * ep + 4 * q + 2];
      const double vv[4] = {v0.x, v0.y, v1.x, v1.y}, oo[4] = {o0.x, o0.y, o1.x, o1.y};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int u = 0; u < 4; ++u) s[i][u] = fma(vv[i], oo[u], s[i][u]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = 4 * kb + i;
      if (k >= ell_n) break;
      const int64_t pq = plo + sn * (k + (int64_t)ell_n * phi);
      const int64_t rq = pq / Lb, lq = pq - rq * Lb;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (4 * q + u < ell) Om[lq + Lb * (4 * q + u + (int64_t)ell * rq)] = s[i][u];
    }
  }
}

void omega_fold(Ctx &c, const int64_t *gdims, int d, int n, int m, int ell_n, const double *V, int ell, uint64_t seed,
                bool normals_f32, double *Om) {
  RT_REQUIRE(n != m && ell >= 1 && ell <= 64 && ell_n >= 1 && ell_n <= 64, "omega_fold: bad shape");
  const int r = (int)gdims[n];
  int64_t sn = 1, P = 1, Lb = 1;
  for (int k = 0; k < d; ++k) {
    if (k == m) continue;
    P *= gdims[k];
    if (k < n) sn *= gdims[k];
  }
  for (int k = 0; k < m; ++k) Lb *= (k == n ? ell_n : gdims[k]);
  const int64_t nhi = P / (sn * r);
  if (sn == 0 || nhi == 0) return;
  RT_REQUIRE(sn * nhi < (1ll << 31) && r <= 64, "omega_fold: grid too large");
  const size_t smem = sizeof(double) * (size_t)r * (((ell + 3) & ~3) + ((ell_n + 3) & ~3));
  const unsigned grid = (unsigned)(sn * nhi);
  if (normals_f32) {
    smem_attr(omega_fold_kernel<float>, smem);
    RT_LAUNCH(c, omega_fold_kernel<float>, grid, 256, smem, sn, r, ell_n, ell, Lb, seed, m, V, Om);
  } else {
    smem_attr(omega_fold_kernel<double>, smem);
    RT_LAUNCH(c, omega_fold_kernel<double>, grid, 256, smem, sn, r, ell_n, ell, Lb, seed, m, V, Om);
  }
}

void sketch_explicit(Ctx &c, const void *X, DT in, ModeView v, const double *Om, int ell, double *Y) {
  RT_REQUIRE(ell >= 1 && ell <= 64, "explicit sketch: 1 <= l <= 64");
  if (in == DT::F64) launch_sketch_dfma<double, double>(c, (const double *)X, v, 0, ell, 0, 0, 0, Y, nullptr, Om);
  else launch_sketch_dfma<float, double>(c, (const float *)X, v, 0, ell, 0, 0, 0, Y, nullptr, Om);
}

void omega_rows(Ctx &c, DT out, uint64_t seed, int mode, const int64_t *cols, int64_t n, int ell,
                int64_t k0, void *dst) {
  const int g = std::max(1, std::min(4096, ceil_div(n * ((ell + 7) / 4), 256)));
  if (out == DT::F64)
    RT_LAUNCH(c, omega_rows_kernel<double>, g, 256, 0, seed, mode, cols, n, ell, k0, (double *)dst);
  else
    RT_LAUNCH(c, omega_rows_kernel<float>, g, 256, 0, seed, mode, cols, n, ell, k0, (float *)dst);
}

void philox_raw(Ctx &c, const uint32_t *ctr, int64_t n, uint32_t k0, uint32_t k1, uint32_t *out) {
  const int g = std::max(1, std::min(4096, ceil_div(n, 256)));
  RT_LAUNCH(c, philox_raw_kernel, g, 256, 0, ctr, n, k0, k1, out);
}

}  // namespace rt
