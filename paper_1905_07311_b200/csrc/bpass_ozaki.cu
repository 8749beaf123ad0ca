// Mode-1 B-pass B = Q^T X_(1) (+ its Gram) for fp32 X under the HYBRID policy, with fp64-level
// products from EXACT int8 tensor-core products (Ozaki-style splitting, tcgen05 kind::i8).
//
// Why: R16 needs B to ~1e-9 relative, which fp32/TF32 accumulation cannot give; the
// fp64 tensor cores give it at 37 TF/s (the previous kernel, 71 % of that peak).  Here every
// column p of X_(1) is scaled by 2^-e_p (e_p: exponent of max_i |X_ip|, computed beforehand) and
// every column j of Q by 2^-f_j; the scaled values (|.| < 1) are cut into S = 5 signed slices
// by rounding to nearest:  x = sum_{s=1..5} x_s 2^{1-7s} + O(2^-35),  x_s in [-64, 64]
// (first slice of x 2^6, then 7 more bits per slice; the rounding is done with the fp32 magic
// constant 1.5 2^23, whose sum's low byte IS the int8 slice: FMA-pipe work only, no F2I).
// Then  B_jp = 2^{e_p + f_j} sum_{L=2..6} 2^{2-7L} acc_L,  acc_L = sum_{s+t=L} sum_i q_t[i,j] x_s[i,p],
// each acc_L an exact int32 sum of int8 products (|acc_L| <= 5 * I * 64^2 < 2^31 for I <= 100000)
// accumulated in TMEM; levels L >= 7 (and the slice residuals) are dropped: |error| ~
// 2^-35 relative to the scaled magnitudes, i.e. ~1e-10 relative to |B_jp| for
// random-sign sums (measured against fp64 products in tests/test_gpu_kernels.py).
//
// Layout of one CTA (persistent, one per SM; tile = 128 columns p, all I rows i):
//   warp 0       TMA producer: per chunk (32 values of i) an X box {32 i, 128 p} (fp32) into a
//                staging ring, and the chunk's pre-sliced Q (5 slices, K-major int8, 10 KB) by
//                a bulk copy from the qslice buffer
//   warp 1       TMEM owner + MMA issuer: the 15 slice pairs of a chunk in 10 kind::i8 MMAs
//                (M = 128 p, N = 128 j x 2 levels or 64, K = 32, A from TMEM, B from shared
//                memory), pair (s, t) into the level-(s+t) accumulator (5 x 64 TMEM columns)
//   warps 2-9    slicers: thread = one column p of the tile (its TMEM lane) and 16 values of i;
//                X staging (128B-swizzled TMA box, conflict-free row reads) -> 5 int8 slices
//                stored straight into the A-operand buffers in TMEM (tcgen05.st): no shared-
//                memory round trip for the slices, the MMAs read only the small B operand
//   warps 10-13  epilogue (one per TMEM lane quadrant): levels -> fp64 B tile (scales
//                applied) -> shared T -> coalesced store of B and the tile's Gram on the fp64
//                tensor cores (36 upper 8 x 8 tiles, mma.m8n8k4)
// Everything else (scales, Q slices) is computed by two small kernels below.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "kernels.h"
#include "tc.cuh"

namespace rt {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();  // sketch_tc.cu

namespace {

constexpr int kOP = 128;       // columns p per tile (MMA M)
constexpr int kOK = 32;        // values of i per chunk (MMA K for int8)
constexpr int kOS = 5;         // slices per operand
constexpr int kOLv = 5;        // levels L = 2 .. 6
constexpr int kON = 64;        // MMA N (j, ell <= 64)
constexpr int kONSS = 6;       // X staging ring depth
constexpr int kONQ = 3;        // Q slice ring depth
constexpr int kOSlicers = 8;   // slicer warps
constexpr int kOEpi = 4;       // epilogue warps
constexpr int kOThreads = 32 * (2 + kOSlicers + kOEpi + 1);  // + the Q producer warp
constexpr int kOTP = 132;      // epilogue tile T[j][p] stride (doubles, = 4 mod 16): lane-per-p
                               // rows and the DMMA Gram fragments both conflict-free
constexpr int kXStB = kOP * kOK * 4;         // staging bytes per chunk (16 KB)
constexpr int kQChB = kOS * kON * kOK;       // pre-sliced Q bytes per chunk (10 KB)

__device__ __forceinline__ int kmaj8(int r, int k) {  // byte offset, K-major int8 core matrices
  return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}
__host__ __device__ constexpr uint32_t idesc_s8(int M, int N) {  // s32 <- s8 x s8, K-major
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Cut a scaled value r (|r| < 1) into 5 slices rounded to nearest (exact fp32 arithmetic):
// u = r 2^k + 1.5 2^23 holds round(r 2^k) in its low bits (two's complement byte), t = u -
// 1.5 2^23 is that integer as a float, r <- r 2^k - t stays exact.  Returns the raw bits of u.
__device__ __forceinline__ void slice5(float r, uint32_t (&q)[kOS]) {
  constexpr float M = 12582912.0f;  // 1.5 * 2^23
#pragma unroll
  for (int s = 0; s < kOS; ++s) {
    const float k = s == 0 ? 64.0f : 128.0f;
    const float u = fmaf(r, k, M);
    const float t = u - M;
    r = fmaf(r, k, -t);
    q[s] = __float_as_uint(u);
  }
}

// Two values at a time on the paired fp32 pipe (FFMA2 / FADD2, sm_100): the same exact steps as
// slice5, carried on the NEGATED residual r' = -r so that no operand needs a sign flip:
//   u = fma(r', -k, M) = fl(r k + M),  t = u + (-M) = u - M,  r' <- fma(r', k, t) = -(r k - t).
// Bit-identical slices; half the FP instructions of two slice5 calls (the slicers bound the
// B-pass: DESIGN §7).
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
// slices of x0 * sc and x1 * sc into q0, q1 (raw bits of u, as slice5)
__device__ __forceinline__ void slice5x2(float x0, float x1, float sc, uint32_t (&q0)[kOS], uint32_t (&q1)[kOS]) {
  const uint64_t M2 = f2_pack(12582912.0f, 12582912.0f), nM2 = f2_pack(-12582912.0f, -12582912.0f);
  uint64_t r = f2_mul(f2_pack(x0, x1), f2_pack(-sc, -sc));  // r' = -x sc (exact: sc is a power of 2)
#pragma unroll
  for (int s = 0; s < kOS; ++s) {
    const float k = s == 0 ? 64.0f : 128.0f;
    const uint64_t u = f2_fma(r, f2_pack(-k, -k), M2);
    const uint64_t t = f2_add(u, nM2);
    r = f2_fma(r, f2_pack(k, k), t);
    q0[s] = (uint32_t)u;
    q1[s] = (uint32_t)(u >> 32);
  }
}

// m_p = max_i |X(i, p)| as fp32 bits (the scale exponent is taken from it), one warp per column.
// The R-STHOSVD path gets these from the mode-1 sketch instead (sketch_tc.cu, colmax).
__global__ void colmax_kernel(const float *__restrict__ X, int64_t I, int64_t P, uint32_t *__restrict__ cm) {
  const int lane = threadIdx.x & 31;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float *col = X + I * p;
    float m = 0.f;
    if (((I & 3) == 0)) {
      for (int64_t i = 4 * lane; i < I; i += 128) {
        const float4 v = *(const float4 *)(col + i);
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
    } else {
      for (int64_t i = lane; i < I; i += 32) m = fmaxf(m, fabsf(col[i]));
    }
    const uint32_t r = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
    if (lane == 0) cm[p] = r;
  }
}
// exponent e with m < 2^e (frexp convention), 0 for m == 0
__device__ __forceinline__ int exp_of(uint32_t mbits) {
  if (mbits == 0) return 0;
  int e;
  frexpf(__uint_as_float(mbits), &e);
  return e;
}

// m_p = max_i |X(l, i, r)| for p = l + L r (strided contraction index): thread per column,
// consecutive threads consecutive l (coalesced rows).
__global__ void colmax_l_kernel(const float *__restrict__ X, int64_t L, int64_t I, int64_t P, uint32_t *__restrict__ cm) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = p / L, l = p - r * L;
    const float *col = X + l + L * I * r;
    float m = 0.f;
    for (int64_t i = 0; i < I; ++i) m = fmaxf(m, fabsf(col[L * i]));
    cm[p] = __float_as_uint(m);
  }
}

// Q (I x J fp64, column-major) -> per chunk c: 5 slices, each [64 j][32 i] K-major int8 (rows
// j >= J and i >= I zero); f_j = exponent of max_i |Q(i, j)|.  One CTA per column j.
__global__ void qslice_kernel(const double *__restrict__ Q, int64_t I, int64_t lda, int J, int nchunk,
                              int8_t *__restrict__ qs, int *__restrict__ f) {
  const int j = blockIdx.x;  // 0 .. 63
  __shared__ double red[32];
  double m = 0.0;
  if (j < J)
    for (int64_t i = threadIdx.x; i < I; i += blockDim.x) m = fmax(m, fabs(Q[i + lda * j]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  int ex = 0;
  if (red[0] > 0.0) frexp(red[0], &ex);
  if (threadIdx.x == 0) f[j] = ex;
  for (int64_t i = threadIdx.x; i < (int64_t)nchunk * kOK; i += blockDim.x) {
    double r = (j < J && i < I) ? ldexp(Q[i + lda * j], -ex) : 0.0;
    const int c = (int)(i / kOK), k = (int)(i % kOK);
    int8_t *dst = qs + (size_t)c * kQChB;
#pragma unroll
    for (int s = 0; s < kOS; ++s) {  // same convention as slice5: x 2^6, then x 2^7, nearest
      r *= (s == 0) ? 64.0 : 128.0;
      const double t = rint(r);
      r -= t;
      dst[s * (kON * kOK) + kmaj8(j, k)] = (int8_t)(int)t;
    }
  }
}

struct OzParams {
  int64_t I, P;
  int64_t L, tpr;       // LG layout: extent of the contiguous index l and 128-column tiles per r
  int J, nchunk;
  const int8_t *qs;     // [nchunk][5][64 x 32]
  const uint32_t *cm;   // [P] fp32 bits of the column maxima of X
  const int *f;         // [64]
  double *out;          // B: (J x P) column-major, or null
  double *gram_partial; // [grid][64 x 64] or null
  long long *prof;      // CTA 0 wait-cycle counters (builds with -DRTUCKER_OZ_PROF_BUILD only)
};

#ifdef RTUCKER_OZ_PROF_BUILD
#define OZP(...) __VA_ARGS__
#else
#define OZP(...)
#endif

// Tile -> column p of tile row `row` (-1 past the end).  Mode 1 (L == 1): tiles of 128
// consecutive p.  LG (L > 1, Gram only): tile (r, l0) = 128 consecutive l of one r, p = l + L r.
__device__ __forceinline__ void tma_load_3d(void *dst, const void *tmap, uint64_t *bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(tc::smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(tc::smem_u32(bar))
      : "memory");
}

template <bool LG>
__device__ __forceinline__ int64_t oz_col(const OzParams &p, int64_t tile, int row) {
  if (!LG) {
    const int64_t pp = tile * kOP + row;
    return pp < p.P ? pp : -1;
  }
  const int64_t r = tile / p.tpr, l = (tile - r * p.tpr) * kOP + row;
  return l < p.L ? l + p.L * r : -1;
}

// 2^k as a double for k in the normal range (clamped)
__device__ __forceinline__ double pow2d(int k) {
  k = k < -1022 ? -1022 : (k > 1023 ? 1023 : k);
  return __longlong_as_double((long long)(k + 1023) << 52);
}
__device__ __forceinline__ void mma_i8_ta(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// TMEM map: columns [0, 320): the 5 level accumulators (64 columns each); columns
// [320 + 40 b, +40): A-operand buffer b (5 X slices x 8 columns: lane = column p of the tile,
// column c of a slice = int8 values k = 4c .. 4c + 3 of the chunk).
constexpr int kOXB = 4;          // A-operand buffers in TMEM
constexpr uint32_t kOAcol = 320;

// LG: the contraction index i is strided (mode n > 1 with L > 1: X(l, i, r)); 3-D TMA boxes of
// 128 l x 32 i (plain layout [i][l]) and a Gram-only epilogue.
template <bool LG>
__global__ void __launch_bounds__(kOThreads, 1)
    bpass_ozaki_kernel(const __grid_constant__ CUtensorMap tmap, const OzParams p) {
  extern __shared__ __align__(1024) unsigned char ozs[];
  const uint32_t pad = (1024u - (tc::smem_u32(ozs) & 1023u)) & 1023u;
  unsigned char *base = ozs + pad;
  unsigned char *stg = base;                             // [kONSS][16 KB] fp32 X boxes (128B swizzle)
  unsigned char *qb = stg + kONSS * kXStB;               // [kONQ][10 KB] Q slices
  double *T = reinterpret_cast<double *>(qb + kONQ * kQChB);  // [64 j][kOTP] (p = 0 .. 127)
  uint64_t *full = reinterpret_cast<uint64_t *>(T + kON * kOTP);  // X stage landed
  uint64_t *sfree = full + kONSS;                        // X stage consumed by the slicers
  uint64_t *qfull = sfree + kONSS, *qfree = qfull + kONQ;
  uint64_t *xready = qfree + kONQ, *xempty = xready + kOXB;
  uint64_t *accfull = xempty + kOXB, *accempty = accfull + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(accempty + 1);
  double *fpw = reinterpret_cast<double *>(tslot + 2);  // [64] 2^{f_j}

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = LG ? p.tpr * (p.P / p.L) : (p.P + kOP - 1) / kOP;
  const int64_t mytiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nchunk = p.nchunk;
  const int64_t total = mytiles * nchunk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kONSS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&sfree[s], 32 * kOSlicers);
    }
    for (int s = 0; s < kONQ; ++s) {
      tc::mbar_init(&qfull[s], 1);
      tc::mbar_init(&qfree[s], 1);
    }
    for (int s = 0; s < kOXB; ++s) {
      tc::mbar_init(&xready[s], 32 * kOSlicers);
      tc::mbar_init(&xempty[s], 1);
    }
    tc::mbar_init(accfull, 1);
    tc::mbar_init(accempty, 32 * kOEpi);
    tc::fence_barrier_init();
  }
  for (int j = threadIdx.x; j < kON; j += kOThreads) fpw[j] = pow2d(p.f[j]);
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------------- TMA producer
    if (lane == 0) {
      tc::tma_prefetch_desc(&tmap);
      int s = 0;
      uint32_t ph = 0;
      for (int64_t g = 0; g < total; ++g) {
        const int64_t tk = g / nchunk;
        const int ch = (int)(g - tk * nchunk);
        const int64_t tile = blockIdx.x + tk * gridDim.x;
        if (g >= kONSS) tc::mbar_wait(&sfree[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&full[s], kXStB);
        if (LG) {
          const int64_t r = tile / p.tpr;
          tma_load_3d(stg + s * kXStB, &tmap, &full[s], (int)((tile - r * p.tpr) * kOP), ch * kOK, (int)r);
        } else {
          tc::tma_load_2d(stg + s * kXStB, &tmap, &full[s], ch * kOK, (int)(tile * kOP));
        }
        if (++s == kONSS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------- MMA issuer (warp-wide,
    // elect.sync inside the MMA asm: uniform operands, see tc::mma_tf32_w)
    {
      constexpr uint32_t idesc = idesc_s8(kOP, kON), idesc2 = idesc_s8(kOP, 2 * kON);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t qb0 = __shfl_sync(0xffffffffu, tc::smem_u32(qb), 0);
      int s = 0, x = 0;  // s: Q ring slot
      uint32_t ph = 0, phx = 0;
      int ch = 0;
      int64_t tt = 0;
      OZP(long long w0 = 0, w1 = 0, w2 = 0, t0 = clock64();)
      for (int64_t g = 0; g < total; ++g) {
        OZP(const long long c0 = clock64();)
        if (ch == 0 && tt > 0) tc::mbar_wait(accempty, (uint32_t)((tt - 1) & 1));  // TMEM drained
        OZP(const long long c1 = clock64();)
        tc::mbar_wait(&qfull[s], ph);
        OZP(const long long c2 = clock64();)
        tc::mbar_wait(&xready[x], phx);
        OZP(w0 += c1 - c0; w1 += c2 - c1; w2 += clock64() - c2;)
        tc::tc_fence_after();
        const uint32_t xa = tm + kOAcol + 40 * x;
        const uint64_t bd0 = tc::smem_desc(qb0 + s * kQChB, 128, 256, tc::kSwNone);
        // pairs (sx, t) and (sx, t + 1) in ONE N = 128 MMA: the B slices q_t, q_{t+1} are
        // adjacent 64-row tiles in shared memory, and the levels sx + t, sx + t + 1 adjacent
        // 64-column accumulators in TMEM (10 MMAs per chunk instead of 15)
#pragma unroll
        for (int sx = 0; sx < kOS; ++sx)
#pragma unroll
          for (int sq = 0; sx + sq < kOLv; sq += 2) {
            const int L = sx + sq;  // level - 2 (slices are 1-based in the derivation)
            const bool two = L + 1 < kOLv;
            // the first products of a level in a tile (sx = 0) overwrite the accumulators
            tc::mma_i8_ta_w(tm + L * kON, xa + 8 * sx, bd0 + (uint64_t)(sq * ((kON * kOK) >> 4)), two ? idesc2 : idesc,
                      (ch == 0 && sx == 0) ? 0u : 1u);
          }
        tc::mma_commit_w(&xempty[x]);
        tc::mma_commit_w(&qfree[s]);
        if (++ch == nchunk) {
          ch = 0;
          tc::mma_commit_w(accfull);
          ++tt;
        }
        if (++s == kONQ) { s = 0; ph ^= 1; }
        if (++x == kOXB) { x = 0; phx ^= 1; }
      }
      OZP(if (p.prof && blockIdx.x == 0 && lane == 0) {
        p.prof[0] = w0; p.prof[1] = w1; p.prof[2] = w2; p.prof[3] = clock64() - t0; p.prof[15] = total;
      })
    }
  } else if (warp == 2 + kOSlicers + kOEpi) {
    // ------------------------------------------------------------------- Q producer
    if (lane == 0) {  // pre-sliced Q chunks (L2-resident, the same for every tile)
      int s = 0;
      uint32_t ph = 0;
      for (int64_t g = 0; g < total; ++g) {
        const int64_t tk = g / nchunk;
        const int ch = (int)(g - tk * nchunk);
        if (g >= kONQ) tc::mbar_wait(&qfree[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&qfull[s], kQChB);
        bulk_g2s(qb + s * kQChB, p.qs + (size_t)ch * kQChB, kQChB, &qfull[s]);
        if (++s == kONQ) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp < 2 + kOSlicers) {
    // ------------------------------------------------------------------- slicers
    // warp -> TMEM lane quadrant q = warp % 4 (tile rows 32 q ..) and half of the chunk's i
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int row = 32 * q + lane;
    int s = 0, x = 0;
    uint32_t ph = 0, phx = 0;
    int ch = 0;
    int64_t tk = 0;
    float sc = 0.f;  // 2^-e_p of this thread's column
    OZP(long long w4 = 0, w5 = 0, t0 = clock64();)
    for (int64_t g = 0; g < total; ++g) {
      if (ch == 0) {
        const int64_t pp = oz_col<LG>(p, blockIdx.x + tk * gridDim.x, row);
        sc = pp >= 0 ? ldexpf(1.0f, -exp_of(p.cm[pp])) : 0.f;
      }
      OZP(const long long c0 = clock64();)
      tc::mbar_wait(&full[s], ph);
      OZP(const long long c1 = clock64();)
      if (g >= kOXB) tc::mbar_wait(&xempty[x], phx ^ 1);
      OZP(w4 += c1 - c0; w5 += clock64() - c1;)
      tc::tc_fence_after();
      // mode 1: staging row `row` = 32 floats (128 B, 16-byte chunks XOR-swizzled by row % 8);
      // LG: staging [32 i][128 l], this thread's values at stride 128 floats (conflict-free)
      const unsigned char *srow = stg + s * kXStB + row * 128;
      const float *scol = reinterpret_cast<const float *>(stg + s * kXStB) + row;
      uint32_t w[kOS][4];
#pragma unroll
      for (int cq = 0; cq < 4; ++cq) {  // 16-byte chunk j = 4 half + cq: values k = 4 j .. 4 j + 3
        const int j = 4 * half + cq;
        float4 v;
        if (LG) {
          v = make_float4(scol[(4 * j) * kOP], scol[(4 * j + 1) * kOP], scol[(4 * j + 2) * kOP], scol[(4 * j + 3) * kOP]);
        } else {
          v = *reinterpret_cast<const float4 *>(srow + ((j ^ (row & 7)) << 4));
        }
        uint32_t a[kOS], b[kOS], c[kOS], d[kOS];
        slice5x2(v.x, v.y, sc, a, b);
        slice5x2(v.z, v.w, sc, c, d);
#pragma unroll
        for (int t = 0; t < kOS; ++t)
          w[t][cq] = __byte_perm(__byte_perm(a[t], b[t], 0x0040), __byte_perm(c[t], d[t], 0x0040), 0x5410);
      }
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + kOAcol + 40 * x + 4 * half;
#pragma unroll
      for (int t = 0; t < kOS; ++t) tmem_st4(ta + 8 * t, w[t][0], w[t][1], w[t][2], w[t][3]);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      // the staging slot is released only after every slice has been formed and stored: with
      // the paired-pipe slicing, ptxas issued this arrive between the staging loads and their
      // first use, and the refill raced with them (nondeterministic B, caught by rerunning C4)
      tc::mbar_arrive(&sfree[s]);  // staging slot may be refilled
      tc::tc_fence_before();
      tc::mbar_arrive(&xready[x]);
      if (++ch == nchunk) { ch = 0; ++tk; }
      if (++s == kONSS) { s = 0; ph ^= 1; }
      if (++x == kOXB) { x = 0; phx ^= 1; }
    }
    OZP(if (p.prof && blockIdx.x == 0 && threadIdx.x == 64) { p.prof[4] = w4; p.prof[5] = w5; p.prof[6] = clock64() - t0; })
  } else {
    // ------------------------------------------------------------------- epilogue
    const int q4 = warp & 3;            // TMEM lane quadrant
    const int et = threadIdx.x - 32 * (2 + kOSlicers);  // 0 .. 127
    const int row = 32 * q4 + lane;     // tile row (column p)
    double gacc[9][2];
#pragma unroll
    for (int u = 0; u < 9; ++u) gacc[u][0] = gacc[u][1] = 0.0;
    const int ew = warp - (2 + kOSlicers);  // 0 .. 3
    long long *Ti = reinterpret_cast<long long *>(T);
    OZP(long long e0 = 0, e1 = 0, e2 = 0, e3 = 0, e4 = 0, et0 = clock64();)
    for (int64_t tt = 0; tt < mytiles; ++tt) {
      const int64_t pp = oz_col<LG>(p, blockIdx.x + tt * gridDim.x, row);
      OZP(const long long c0 = clock64();)
      tc::mbar_wait(accfull, (uint32_t)(tt & 1));
      OZP(const long long c1 = clock64(); e0 += c1 - c0;)
      tc::tc_fence_after();
      // phase 1 (holds TMEM): S = sum_L acc_L 2^{7 (4 - L)} exactly in int64 (|S| < 2^60 for
      // I <= 100000), parked in T; then release the accumulators
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        long long S[32];
#pragma unroll
        for (int L = 0; L < kOLv; ++L) {
          uint32_t r[32];
          tc::tmem_ld32(tmem + ((uint32_t)(32 * q4) << 16) + L * kON + 32 * h, r);
#pragma unroll
          for (int j = 0; j < 32; ++j) S[j] = (L == 0 ? 0ll : (S[j] << 7)) + (long long)(int)r[j];
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) Ti[(32 * h + j) * kOTP + row] = S[j];
      }
      tc::tc_fence_before();
      tc::mbar_arrive(accempty);  // the MMA warp may overwrite the accumulators
      OZP(const long long c2 = clock64(); e1 += c2 - c1;)
      // phase 2: B_jp = S 2^{e_p - 40} 2^{f_j} (level weights 2^{2 - 7 (L + 2)}, L = 0 .. 4),
      // kept in T (fp64, in place) for the Gram and stored straight to B = out[p J + j]: a row
      // of B is one thread's 60 contiguous doubles (16-byte stores; L2 merges the sectors)
      const bool pok = pp >= 0;
      const int ep = pok ? exp_of(p.cm[pp]) : 0;
      const double rs = pow2d(ep - 40);
      double *orow = (!LG && p.out) ? p.out + pp * p.J : nullptr;
      const bool vec = (p.J & 1) == 0;
#pragma unroll 4
      for (int jj = 0; jj < kON; jj += 2) {
        const double v0 = (pok && jj < p.J) ? (double)Ti[jj * kOTP + row] * rs * fpw[jj] : 0.0;
        const double v1 = (pok && jj + 1 < p.J) ? (double)Ti[(jj + 1) * kOTP + row] * rs * fpw[jj + 1] : 0.0;
        T[jj * kOTP + row] = v0;
        T[(jj + 1) * kOTP + row] = v1;
        if (orow && pok) {
          if (vec) {
            if (jj < p.J) *reinterpret_cast<double2 *>(orow + jj) = make_double2(v0, v1);
          } else {
            if (jj < p.J) orow[jj] = v0;
            if (jj + 1 < p.J) orow[jj + 1] = v1;
          }
        }
      }
      named_bar(1, 32 * kOEpi);
      OZP(const long long c3 = clock64(); e2 += c3 - c2;)
      OZP(const long long c4 = clock64(); e3 += c4 - c3;)
      if (p.gram_partial) {  // G += T^T T, 36 upper 8x8 tiles over the 4 epilogue warps
        const int fr = lane >> 2, fc = lane & 3;
        // three tiles at a time, k inner: three independent DMMA accumulation chains in flight
        // (one tile at a time left a dependent chain of 32 DMMAs: 22k cycles per tile; all
        // nine at once spills)
#pragma unroll
        for (int u0 = 0; u0 < 9; u0 += 3) {
          int oa[3], ob[3];
#pragma unroll
          for (int v = 0; v < 3; ++v) {
            const int t = ew + 4 * (u0 + v);
            int a = 0, rem = t;
            while (rem >= 8 - a) { rem -= 8 - a; ++a; }
            oa[v] = (8 * a + fr) * kOTP + fc;
            ob[v] = (8 * (a + rem) + fr) * kOTP + fc;
          }
#pragma unroll 4
          for (int k0 = 0; k0 < kOP; k0 += 4) {
#pragma unroll
            for (int v = 0; v < 3; ++v)  // non-volatile: pure register op, freely scheduled
              asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                           : "+d"(gacc[u0 + v][0]), "+d"(gacc[u0 + v][1])
                           : "d"(T[oa[v] + k0]), "d"(T[ob[v] + k0]));
          }
        }
      }
      OZP(e4 += clock64() - c4;)
      named_bar(1, 32 * kOEpi);  // T free for the next tile
    }
    OZP(if (p.prof && blockIdx.x == 0 && et == 0) {
      p.prof[7] = e0; p.prof[8] = e1; p.prof[9] = e2; p.prof[10] = e3; p.prof[11] = e4; p.prof[12] = clock64() - et0;
    })
    if (p.gram_partial) {
      const int fr = lane >> 2, fc = lane & 3;
      double *gp = p.gram_partial + (int64_t)blockIdx.x * 4096;
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        const int t = ew + 4 * u;
        int a = 0, rem = t;
        while (rem >= 8 - a) { rem -= 8 - a; ++a; }
        const int b = a + rem;
        const int gi = 8 * a + fr, gj = 8 * b + 2 * fc;
        gp[gi * 64 + gj] = gacc[u][0];
        gp[gi * 64 + gj + 1] = gacc[u][1];
        if (a != b) {
          gp[gj * 64 + gi] = gacc[u][0];
          gp[(gj + 1) * 64 + gi] = gacc[u][1];
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

__global__ void oz_gram_reduce_kernel(const double *__restrict__ part, int nblk, int J, double *__restrict__ gram) {
  // four lanes per entry: lane q sums the CTA partials b = q, q + 4, ... in order, then
  // (q0 + q1) + (q2 + q3) (a serial chain over ~148 partials per thread was latency-bound)
  const int e4 = blockIdx.x * blockDim.x + threadIdx.x, q = threadIdx.x & 3, e = e4 >> 2;
  if (e >= J * J) return;  // (J * J * 4 and the block size are multiples of 4: groups exit together)
  const int i = e % J, j = e / J;
  double s = 0.0;
  for (int b = q; b < nblk; b += 4) s += part[(int64_t)b * 4096 + i * 64 + j];
  const unsigned gm = 0xFu << (threadIdx.x & 28);
  s += __shfl_xor_sync(gm, s, 1);
  s += __shfl_xor_sync(gm, s, 2);
  if (q == 0) gram[i + (int64_t)J * j] = s;
}

}  // namespace

void column_maxima(Ctx &c, const float *X, ModeView v, uint32_t *cm) {
  const int64_t P = v.L * v.R;
  if (v.L > 1) {
    RT_LAUNCH(c, colmax_l_kernel, (int)std::min<int64_t>((P + 255) / 256, (int64_t)c.num_sms * 32), 256, 0, X, v.L,
              v.I, P, cm);
  } else {
    RT_LAUNCH(c, colmax_kernel, std::max(1, std::min(c.num_sms * 16, (int)((P + 7) / 8))), 256, 0, X, v.I, P, cm);
  }
}

bool ozaki_bpass_enabled() {
  static const bool off = RT_EXP_GETENV("RTUCKER_NO_OZAKI") != nullptr;
  return !off;
}

// B = A^T X_(1) (J x P fp64, column-major) and/or its Gram for fp32 X with L == 1.
// Returns false outside the kernel's envelope (caller falls back to the fp64 tensor cores).
bool ttm_ozaki(Ctx &c, const float *X, ModeView v, const double *A, int64_t lda, int J, double *out, double *gram,
               const uint32_t *colmax) {
  const bool lg = v.L > 1;  // strided contraction index: Gram-only variant (R-HOSVD modes n > 1)
  if (!ozaki_bpass_enabled() || J < 1 || J > kON || (v.I % 4) != 0 || v.I > 26000 ||
      (((uintptr_t)X) & 15) != 0 || v.R > (int64_t)INT32_MAX - kOP)
    return false;
  if (lg && (out || !gram || (v.L % 4) != 0 || v.L > (int64_t)INT32_MAX - kOP || RT_EXP_GETENV("RTUCKER_NO_OZAKI_LG")))
    return false;
  const int64_t I = v.I, P = v.L * v.R;
  const int nchunk = (int)((I + kOK - 1) / kOK);
  DevBuf<int8_t> qs(c, (size_t)nchunk * kQChB);
  DevBuf<int> fexp(c, kON);
  DevBuf<uint32_t> cmown;
  RT_LAUNCH(c, qslice_kernel, kON, 256, 0, A, I, lda, J, nchunk, qs.p, fexp.p);
  if (!colmax) {
    cmown.alloc(c, (size_t)P);
    column_maxima(c, X, v, cmown.p);
    colmax = cmown.p;
  }
  const int64_t tpr = (v.L + kOP - 1) / kOP;
  const int64_t ntiles = lg ? tpr * v.R : (P + kOP - 1) / kOP;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, c.num_sms));
  DevBuf<double> part;
  OzParams prm{};
  prm.I = I;
  prm.P = P;
  prm.L = v.L;
  prm.tpr = tpr;
  prm.J = J;
  prm.nchunk = nchunk;
  prm.qs = qs.p;
  prm.cm = colmax;
  prm.f = fexp.p;
  prm.out = out;
  // Gram of B in the epilogue (DMMA, 36 upper 8x8 tiles per 128-column tile).  The alternative,
  // a separate pass over B (gram64_kernel, RTUCKER_OZ_GRAM_SEPARATE), measured slower at C4
  // (B-pass + Gram 1.37 vs 0.82 ms).
  static const bool gsep_env = RT_EXP_GETENV("RTUCKER_OZ_GRAM_SEPARATE") != nullptr;
  const bool gsep = gram && out && gsep_env;
  if (gram && !gsep) part.alloc(c, (size_t)grid * 4096);
  prm.gram_partial = (gram && !gsep) ? part.p : nullptr;
  CUtensorMap tm;
  CUresult r;
  if (lg) {  // (l, i, r), box 128 l x 32 i x 1 r, plain [i][l] staging
    cuuint64_t dims[3] = {(cuuint64_t)v.L, (cuuint64_t)I, (cuuint64_t)v.R};
    cuuint64_t strides[2] = {(cuuint64_t)v.L * 4, (cuuint64_t)v.L * I * 4};
    cuuint32_t box[3] = {kOP, kOK, 1};
    cuuint32_t es[3] = {1, 1, 1};
    r = tensor_map_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)X, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)I, (cuuint64_t)P};
    cuuint64_t strides[1] = {(cuuint64_t)I * 4};
    cuuint32_t box[2] = {kOK, kOP};
    cuuint32_t es[2] = {1, 1};
    r = tensor_map_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)X, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) throw Error(RTUCKER_ECUDA, "cuTensorMapEncodeTiled failed for the Ozaki B-pass");
  const size_t smem = 1024 + (size_t)kONSS * kXStB + (size_t)kONQ * kQChB + sizeof(double) * kON * kOTP +
                      8 * (2 * kONSS + 2 * kONQ + 2 * kOXB + 2) + 16 + 8 * kON;
  auto kern = lg ? bpass_ozaki_kernel<true> : bpass_ozaki_kernel<false>;
  smem_attr(kern, smem);
  static const bool prof = RT_EXP_GETENV("RTUCKER_OZ_PROF") != nullptr;
  DevBuf<long long> pbuf;
  if (prof) {
    pbuf.alloc(c, 16);
    RT_CUDA(cudaMemsetAsync(pbuf.p, 0, 128, c.stream));
    prm.prof = pbuf.p;
  }
  RT_LAUNCH(c, kern, grid, kOThreads, smem, tm, prm);
  if (prof) {
    long long h[16];
    RT_CUDA(cudaMemcpyAsync(h, pbuf.p, 128, cudaMemcpyDeviceToHost, c.stream));
    RT_CUDA(cudaStreamSynchronize(c.stream));
    fprintf(stderr,
            "[oz prof] chunks %lld | mma: wait accempty %lld qfull %lld xready %lld total %lld | slicer: wait full %lld "
            "xempty %lld total %lld | epi: wait accfull %lld ph1 %lld ph2 %lld store %lld gram %lld total %lld\n",
            h[15], h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], h[10], h[11], h[12]);
  }
  if (gsep) mode_gram(c, out, DT::F64, ModeView{1, J, P}, gram);
  else if (gram) RT_LAUNCH(c, oz_gram_reduce_kernel, (4 * J * J + 127) / 128, 128, 0, part.p, grid, J, gram);
  return true;
}

}  // namespace rt
