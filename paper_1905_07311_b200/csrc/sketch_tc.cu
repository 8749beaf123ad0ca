// Tensor-core (tcgen05, 3xTF32) mode-n sketch Y = X_(n) Omega_n (Alg 1 line 1) for
// fp32 data whose mode-n rows are the contiguous index (L == 1: mode 1, or any mode whose
// lower modes are all 1), i.e. X_(n) is stored column-major I x C and the MMA A operand
// is MN-major.  Omega is generated on the fly into shared memory; it is never read
// from HBM.
//
// Layout of one CTA (persistent, one per SM, split-K over the unfolding columns c):
//   warp 0       TMA producer: per stage, nbox boxes of BR rows x 8 columns of X into a
//                staging buffer (plain [c][i] tiles), NSS stages deep
//   warp 1       TMEM allocation + MMA issuer (one elected thread)
//   warps 2-5    Omega generators: Omega(c0:c0+8, k0:k0+N) with Philox4x32-10 + Box-Muller
//                (fp32, DESIGN reading R3), one Philox block per thread and stage, split into
//                hi/lo tf32 K-major tiles (NSG stages deep, so the long RNG dependency chain
//                runs ahead of the X pipeline)
//   warps 6-13   X workers: split X = hi + lo (both rounded to the tf32 grid, R15) and
//                write both TRANSPOSED into K-major no-swizzle operand tiles (MN-major tf32
//                operands need the SWIZZLE_128B_BASE32B layout; this kernel keeps
//                the K-major split); accumulate ||X||^2; after the last stage: TMEM -> fp64
//                partial Y.
//   The accumulator of M-tile mt (rows 128 mt ..) lives in TMEM columns [mt N, mt N + N):
//   3 MMAs per M-tile and stage, D += Xhi*Ohi + Xhi*Olo + Xlo*Ohi (M=128, N, K=8), fp32
//   accumulation in TMEM (BASELINE "3xTF32"; the dropped Xlo*Olo term is 2^-22 relative).
//   K-major no-swizzle operand tile (rows r, 8 K): byte (r/8)*256 + (k/4)*128 + (r%8)*16 + (k%4)*4.
// Per-CTA partial sketches are reduced in a fixed order by the caller (deterministic).
//
// KM variant (L > 1: every mode but the first, e.g. R-HOSVD's modes 2..d on the input): the
// contraction index p = l + L r has l contiguous, so X_(n) is already K-major for the MMA.
// One 5-D TMA box per stage, dims (l%4, i%8, l/4, i/8, r), lands the tile of 8 consecutive l
// (fixed r) x all rows i directly in the K-major core-matrix layout; the X workers only split
// it into hi / lo planes (elementwise, no transposition).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>

#include "kernels.h"
#include "philox.cuh"
#include "tc.cuh"

namespace rt {

namespace {

constexpr int kBK = 8;               // unfolding columns per stage (= MMA K for tf32)
constexpr int kGen = 4;              // Omega generator warps
constexpr int kWorkers = 8;          // X worker warps
constexpr int kThreads = 32 * (2 + kGen + kWorkers);
constexpr int kNSG = 4;              // Omega stages

struct SketchTcParams {
  int64_t I, C;          // rows, unfolding columns
  int64_t L;             // KM variant: extent of the contiguous lower index (C = L R)
  int64_t cps;           // columns per CTA (multiple of kBK)
  int NT;                // M-tiles of 128 rows
  int nbox, BR;          // TMA boxes per stage and rows per box (nbox * BR >= I, BR <= 256)
  int NSS, NSO;          // staging stages (TMA depth), X operand stages
  int ell;               // valid sketch columns (<= N)
  int64_t k0;            // first global sketch column
  uint64_t seed;
  int mode;
  int64_t col_offset;    // global unfolding-column offset of this shard
  float *partial;        // [grid][ell][I]: the CTA's fp32 TMEM sums (exact copies; summed in fp64)
  double *norm_partial;  // [grid] or null
  uint32_t *colmax;      // [C] fp32 bits of max_i |X(i, c)| (atomic max), or null
};

__device__ __forceinline__ int kmaj_off(int r, int k) {  // byte offset in a K-major tile
  return (r >> 3) * 256 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

template <int N, bool KM>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_tc_mn_kernel(const __grid_constant__ CUtensorMap tmap, const SketchTcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // offsets from smem_raw (kept as shared-window pointers so that the compiler emits LDS/STS)
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char *base = smem_raw + pad;
  const int NT = p.NT, NSS = p.NSS, NSO = p.NSO;
  const int sbytes = p.nbox * p.BR * kBK * 4;      // staging (raw X) per stage
  const int abytes = NT * 128 * kBK * 4;           // one operand plane (all M-tiles)
  constexpr int obytes = N * kBK * 4;              // one Omega tile
  unsigned char *hb = base;                        // [NSO][abytes]  X hi (K-major)
  unsigned char *lb = hb + (size_t)NSO * abytes;   // [NSO][abytes]  X lo
  unsigned char *ohb = lb + (size_t)NSO * abytes;  // [kNSG][obytes]
  unsigned char *olb = ohb + (size_t)kNSG * obytes;// [kNSG][obytes]
  unsigned char *sb = olb + (size_t)kNSG * obytes; // [NSS][sbytes]
  uint64_t *full = (uint64_t *)(sb + (size_t)NSS * sbytes);
  uint64_t *sfree = full + NSS;
  uint64_t *xready = sfree + NSS;
  uint64_t *xempty = xready + NSO;
  uint64_t *oready = xempty + NSO;
  uint64_t *oempty = oready + kNSG;
  uint64_t *done = oempty + kNSG;
  uint32_t *tslot = (uint32_t *)(done + 1);
  double *wsum = (double *)(tslot + 2);            // [kWorkers]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cbeg = (int64_t)blockIdx.x * p.cps;
  const int64_t cend = min(p.C, cbeg + p.cps);
  const int nst = (int)((cend - cbeg + kBK - 1) / kBK);
  const uint32_t tcols = NT * N <= 32 ? 32 : NT * N <= 64 ? 64 : NT * N <= 128 ? 128 : NT * N <= 256 ? 256 : 512;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&sfree[s], 32 * kWorkers);
    }
    for (int s = 0; s < NSO; ++s) {
      tc::mbar_init(&xready[s], 32 * kWorkers);
      tc::mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < kNSG; ++s) {
      tc::mbar_init(&oready[s], 32 * kGen);
      tc::mbar_init(&oempty[s], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, tcols);
  // Omega tiles: columns n >= ell stay zero for the whole kernel
  for (int e = threadIdx.x; e < 2 * kNSG * obytes / 4; e += kThreads) ((float *)ohb)[e] = 0.f;
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (lane == 0 && nst > 0) {
      tc::tma_prefetch_desc(&tmap);
      const uint32_t bytes = (uint32_t)sbytes;
      const int boxb = p.BR * kBK * 4;
      for (int it = 0; it < nst; ++it) {
        const int s = it % NSS;
        if (it >= NSS) tc::mbar_wait(&sfree[s], ((it / NSS) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&full[s], bytes);
        const int c0 = (int)(cbeg + (int64_t)it * kBK);
        unsigned char *dst = sb + (size_t)s * sbytes;
        if (KM) {  // 8 consecutive l of one r (L % 8 == 0): tile already K-major
          const int r = c0 / (int)p.L, l0 = c0 - r * (int)p.L;
          tc::tma_load_5d(dst, &tmap, &full[s], 0, 0, l0 >> 2, 0, r);
        } else {
          for (int b = 0; b < p.nbox; ++b) tc::tma_load_2d(dst + b * boxb, &tmap, &full[s], p.BR * b, c0);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer (warp-wide)
    if (nst > 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(128, N, false, false);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t hb0 = __shfl_sync(0xffffffffu, tc::smem_u32(hb), 0);
      const uint32_t lb0 = __shfl_sync(0xffffffffu, tc::smem_u32(lb), 0);
      const uint32_t obh = __shfl_sync(0xffffffffu, tc::smem_u32(ohb), 0);
      const uint32_t obl = __shfl_sync(0xffffffffu, tc::smem_u32(olb), 0);
      for (int it = 0; it < nst; ++it) {
        const int s = it % NSO, g = it % kNSG;
        tc::mbar_wait(&oready[g], (it / kNSG) & 1);
        tc::mbar_wait(&xready[s], (it / NSO) & 1);
        tc::tc_fence_after();
        const uint32_t ha = hb0 + s * abytes, la = lb0 + s * abytes;
        const uint64_t bh = tc::smem_desc(obh + g * obytes, 128, 256, tc::kSwNone);
        const uint64_t bl = tc::smem_desc(obl + g * obytes, 128, 256, tc::kSwNone);
        for (int mt = 0; mt < NT; ++mt) {
          const uint64_t ah = tc::smem_desc(ha + mt * 128 * kBK * 4, 128, 256, tc::kSwNone);
          const uint64_t al = tc::smem_desc(la + mt * 128 * kBK * 4, 128, 256, tc::kSwNone);
          const uint32_t d = tm + mt * N;
          tc::mma_tf32_w(d, ah, bh, idesc, it > 0 ? 1u : 0u);
          tc::mma_tf32_w(d, ah, bl, idesc, 1u);
          tc::mma_tf32_w(d, al, bh, idesc, 1u);
        }
        tc::mma_commit_w(&xempty[s]);
        tc::mma_commit_w(&oempty[g]);
      }
      tc::mma_commit_w(done);
    }
  } else if (warp < 2 + kGen) {
    // ------------------------------------------------------------- Omega generators
    const int gt = threadIdx.x - 64;  // 0 .. 32*kGen-1
    const int64_t jb0 = p.k0 >> 2;
    const int nb = (int)(((p.k0 + p.ell - 1) >> 2) - jb0 + 1);
    for (int it = 0; it < nst; ++it) {
      const int g = it % kNSG;
      const int64_t c0 = cbeg + (int64_t)it * kBK;
      if (it >= kNSG) tc::mbar_wait(&oempty[g], ((it / kNSG) & 1) ^ 1);
      float *oh = (float *)(ohb + (size_t)g * obytes), *ol = (float *)(olb + (size_t)g * obytes);
      for (int t = gt; t < kBK * nb; t += 32 * kGen) {
        const int kk = t & (kBK - 1), jb = t >> 3;
        const int64_t c = c0 + kk;
        const bool valid = c < cend;
        const uint4 w = omega_words(p.seed, p.mode, 0, (uint64_t)(c + p.col_offset), (uint32_t)(jb0 + jb));
        Normal4<float> z(w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t n = 4 * (jb0 + jb) + q - p.k0;
          if (n >= 0 && n < p.ell) {
            const float v = valid ? z.v[q] : 0.f;
            const float hi = tc::tf32_hi(v);
            const int off = kmaj_off((int)n, kk) >> 2;
            oh[off] = hi;
            ol[off] = tc::tf32_lo(v, hi);
          }
        }
      }
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&oready[g]);
    }
  } else {
    // ------------------------------------------------------------- X workers
    const int wt = threadIdx.x - 32 * (2 + kGen);  // 0 .. 32*kWorkers-1
    const int rows_st = min(NT * 128, p.nbox * p.BR);  // operand rows filled from staging
    // rows i = wt + 32 kWorkers j of every stage: staging offsets (floats) and operand offsets
    // (bytes) are fixed, computed once
    constexpr int kRJ = (8 * 128 + 32 * kWorkers - 1) / (32 * kWorkers);  // NT <= 8
    int soff[kRJ], ooff[kRJ];
#pragma unroll
    for (int j = 0; j < kRJ; ++j) {
      const int i = wt + 32 * kWorkers * j;
      soff[j] = (i / p.BR) * (p.BR * kBK) + i % p.BR;
      ooff[j] = (i >> 3) * 256 + (i & 7) * 16;
    }
    double nsq = 0.0;
    int so = 0, ss = 0;
    uint32_t po = 0, ps = 0;  // phase parities of the current operand / staging slot
    for (int it = 0; it < nst; ++it) {
      // the MMAs of this operand slot's previous use must have finished reading it
      if (it >= NSO) tc::mbar_wait(&xempty[so], po ^ 1);
      // X staging [box][c][BR rows] -> hi / lo K-major tiles (rows i, K = c); rows >= I are
      // zero-filled by the TMA, rows beyond the staging extent are never read by a valid D row
      tc::mbar_wait(&full[ss], ps);
      const float *st = (const float *)(sb + (size_t)ss * sbytes);
      unsigned char *hs = hb + (size_t)so * abytes, *ls = lb + (size_t)so * abytes;
      float acc = 0.f;
      float cm[8];  // this thread's column maxima of the stage's 8 columns c0 .. c0+7
#pragma unroll
      for (int u = 0; u < 8; ++u) cm[u] = 0.f;
      if (KM) {  // staging and operand planes share the K-major layout: elementwise split
        const int nun = p.nbox * p.BR * kBK / 4;  // float4 units
        for (int u = wt; u < nun; u += 32 * kWorkers) {
          const float4 x = *(const float4 *)(st + 4 * u);
          if (p.colmax) {  // unit u = (i % 8) + 8 (l / 4) + 16 (i / 8): columns 4 (l / 4) + 0..3
            const float m0 = fabsf(x.x), m1 = fabsf(x.y), m2 = fabsf(x.z), m3 = fabsf(x.w);
            if ((u >> 3) & 1) {
              cm[4] = fmaxf(cm[4], m0); cm[5] = fmaxf(cm[5], m1); cm[6] = fmaxf(cm[6], m2); cm[7] = fmaxf(cm[7], m3);
            } else {
              cm[0] = fmaxf(cm[0], m0); cm[1] = fmaxf(cm[1], m1); cm[2] = fmaxf(cm[2], m2); cm[3] = fmaxf(cm[3], m3);
            }
          }
          float4 h, l;
          h.x = tc::tf32_hi(x.x); h.y = tc::tf32_hi(x.y); h.z = tc::tf32_hi(x.z); h.w = tc::tf32_hi(x.w);
          l.x = tc::tf32_lo(x.x, h.x); l.y = tc::tf32_lo(x.y, h.y); l.z = tc::tf32_lo(x.z, h.z); l.w = tc::tf32_lo(x.w, h.w);
          *(float4 *)(hs + 16 * u) = h;
          *(float4 *)(ls + 16 * u) = l;
          acc = fmaf(x.x, x.x, acc); acc = fmaf(x.y, x.y, acc); acc = fmaf(x.z, x.z, acc); acc = fmaf(x.w, x.w, acc);
        }
      }
#pragma unroll
      for (int j = 0; j < kRJ; ++j) {
        if (!KM && wt + 32 * kWorkers * j < rows_st) {
          const float *src = st + soff[j];
          float x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = src[u * p.BR];
#pragma unroll
          for (int cq = 0; cq < 2; ++cq) {
            float4 h, l;
            h.x = tc::tf32_hi(x[4 * cq]); h.y = tc::tf32_hi(x[4 * cq + 1]);
            h.z = tc::tf32_hi(x[4 * cq + 2]); h.w = tc::tf32_hi(x[4 * cq + 3]);
            l.x = tc::tf32_lo(x[4 * cq], h.x); l.y = tc::tf32_lo(x[4 * cq + 1], h.y);
            l.z = tc::tf32_lo(x[4 * cq + 2], h.z); l.w = tc::tf32_lo(x[4 * cq + 3], h.w);
            *(float4 *)(hs + ooff[j] + cq * 128) = h;
            *(float4 *)(ls + ooff[j] + cq * 128) = l;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            acc = fmaf(x[u], x[u], acc);
            cm[u] = fmaxf(cm[u], fabsf(x[u]));
          }
        }
      }
      if (p.colmax) {
        // warp max per column by a transposing butterfly: at distance 16, 8, 4 each lane keeps
        // half of its columns and takes the partner's maxima of them (4 + 2 + 1 shuffles), so
        // lane l ends with column l / 4 over 8 lanes; distances 2, 1 finish the warp.  Then
        // lanes 4u issue the 8 atomics in one instruction.  Values are |x| >= 0, so the fp32
        // maximum equals the maximum of the bit patterns the B-pass reads.
        const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float keep = u16 ? cm[k + 4] : cm[k], send = u16 ? cm[k] : cm[k + 4];
          cm[k] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 16));
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float keep = u8 ? cm[k + 2] : cm[k], send = u8 ? cm[k] : cm[k + 2];
          cm[k] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 8));
        }
        {
          const float keep = u4 ? cm[1] : cm[0], send = u4 ? cm[0] : cm[1];
          cm[0] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 4));
        }
        cm[0] = fmaxf(cm[0], __shfl_xor_sync(0xffffffffu, cm[0], 2));
        cm[0] = fmaxf(cm[0], __shfl_xor_sync(0xffffffffu, cm[0], 1));
        const int64_t c = cbeg + (int64_t)it * kBK + (lane >> 2);
        if ((lane & 3) == 0 && c < cend) atomicMax(p.colmax + c, __float_as_uint(cm[0]));
      }
      nsq += (double)acc;
      tc::mbar_arrive(&sfree[ss]);       // staging slot may be refilled
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&xready[so]);
      if (++so == NSO) { so = 0; po ^= 1; }
      if (++ss == NSS) { ss = 0; ps ^= 1; }
    }
    // ---- epilogue: TMEM -> fp64 partial[blockIdx.x][k * I + i]
    const int q4 = warp & 3;                       // TMEM lane quadrant of this warp
    const int half = (warp - 2 - kGen) >> 2;       // 0 / 1: which 32 of the N columns
    if (nst > 0) {
      tc::mbar_wait(done, 0);
      tc::tc_fence_after();
    }
    float *dst = p.partial + (int64_t)blockIdx.x * p.ell * p.I;
    if (half * 32 < N) {
      for (int mt = 0; mt < NT; ++mt) {
        uint32_t rr[32];
        if (nst > 0) tc::tmem_ld32(tmem + ((uint32_t)(32 * q4) << 16) + mt * N + half * 32, rr);
        const int64_t i = (int64_t)mt * 128 + 32 * q4 + lane;
        if (i < p.I) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = half * 32 + j;
            if (k < p.ell) dst[(int64_t)k * p.I + i] = nst > 0 ? __uint_as_float(rr[j]) : 0.f;
          }
        }
      }
    }
    if (p.norm_partial) {
      for (int o = 16; o; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
      if (lane == 0) wsum[warp - 2 - kGen] = nsq;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (p.norm_partial && threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kWorkers; ++w) s += wsum[w];
    p.norm_partial[blockIdx.x] = s;
  }
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, tcols);
  }
}

// ---------------------------------------------------------------------------------------------
// L == 1, MN-major A (sketch_tc_mna_kernel, round 2): X_(1) tiles go from TMA straight into the
// MMA's A-operand layout.  tcgen05 kind::tf32 reads an MN-major operand in the SWIZZLE_128B_BASE32B
// layout (atoms of 4 K-rows x 128 B along M, 32-byte chunk j of K-row k stored at j ^ (k % 4)),
// and TMA's CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B writes exactly that for a box of 32 rows i x 8
// columns c (measured, scripts/dbg/tma_swz_probe.cu).  So one stage = ceil(I / 32) boxes of 1 KB,
// M-tile mt = 4 boxes (LBO = 1 KB between 32-row atoms, SBO = 512 B between the two 4-column
// groups), and the raw fp32 X IS the hi operand: the tensor core truncates it to tf32, x_t =
// trunc(x).  The X workers no longer transpose: they write X_lo = rn_tf32(x - x_t) elementwise
// in the same layout (exact difference, rounded to the tf32 grid: residual <= 2^-11 |x - x_t|
// <= 2^-21 |x|, unbiased), and keep ||X||^2 and the Ozaki column maxima (a thread's chunks all
// lie in one column c of the stage).  D += x_t Ohi + x_t Olo + X_lo Ohi as in R15 (hi split by
// truncation instead of rounding; same tf32 grid).  Shared-memory traffic per X byte: TMA write,
// one worker read, the lo write and three operand reads (the K-major kernel also wrote the hi
// plane and transposed through shared memory).
//   warp 0 TMA producer, warp 1 TMEM + MMA issuer, warps 2-5 Omega generators (as in
//   sketch_tc_mn_kernel), warps 6-13 X workers; stage s = (x plane, lo plane), NS deep.
constexpr int kMW = 12;   // X worker warps of the MN-major kernel (its longest pipeline stage)
constexpr int kMThreads = 32 * (2 + kGen + kMW);
constexpr int kMnaJ = (7 * 256 + 32 * kMW - 1) / (32 * kMW);  // 16-byte chunks per worker and stage (NT <= 7)

template <int N>
__global__ void __launch_bounds__(kMThreads, 1)
    sketch_tc_mna_kernel(const __grid_constant__ CUtensorMap tmap, const SketchTcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char *base = smem_raw + pad;
  const int NT = p.NT, NS = p.NSS, nbox = p.nbox;
  const int abytes = NT * 4096;                    // one plane: NT M-tiles x (128 rows x 8 K fp32)
  constexpr int obytes = N * kBK * 4;
  unsigned char *xb = base;                        // [NS][abytes] X as loaded (the hi operand)
  unsigned char *lb = xb + (size_t)NS * abytes;    // [NS][abytes] X_lo
  unsigned char *ohb = lb + (size_t)NS * abytes;   // [kNSG][obytes]
  unsigned char *olb = ohb + (size_t)kNSG * obytes;// [kNSG][obytes]
  uint64_t *full = (uint64_t *)(olb + (size_t)kNSG * obytes);
  uint64_t *sfree = full + NS;    // the MMAs of stage s finished reading both planes
  uint64_t *xready = sfree + NS;  // workers wrote X_lo of stage s
  uint64_t *oready = xready + NS;
  uint64_t *oempty = oready + kNSG;
  uint64_t *done = oempty + kNSG;
  uint32_t *tslot = (uint32_t *)(done + 1);
  double *wsum = (double *)(tslot + 2);            // [kMW]

#ifdef RTUCKER_SK_PROF_BUILD
  long long skp[5] = {0, 0, 0, 0, 0}, skp_t = 0;
  const long long skp_start = clock64();
#define SKP_T0() skp_t = clock64()
#define SKP_ACC(i) skp[i] += clock64() - skp_t
#else
#define SKP_T0()
#define SKP_ACC(i)
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cbeg = (int64_t)blockIdx.x * p.cps;
  const int64_t cend = min(p.C, cbeg + p.cps);
  const int nst = (int)((cend - cbeg + kBK - 1) / kBK);
  const uint32_t tcols = NT * N <= 32 ? 32 : NT * N <= 64 ? 64 : NT * N <= 128 ? 128 : NT * N <= 256 ? 256 : 512;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&sfree[s], 1);
      tc::mbar_init(&xready[s], 32 * kMW);
    }
    for (int s = 0; s < kNSG; ++s) {
      tc::mbar_init(&oready[s], 32 * kGen);
      tc::mbar_init(&oempty[s], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, tcols);
  // Omega tiles: columns n >= ell stay zero; atoms past the last TMA box (rows >= 32 nbox, only
  // ever read into D rows >= I, which are discarded) are zeroed once in both planes
  for (int e = threadIdx.x; e < 2 * kNSG * obytes / 4; e += kMThreads) ((float *)ohb)[e] = 0.f;
  {
    const int pad_f = (4 * NT - nbox) * 256;  // floats per plane past the boxes
    for (int e = threadIdx.x; e < 2 * NS * pad_f; e += kMThreads) {
      const int pl = e / pad_f, f = e % pad_f;
      ((float *)(xb + (size_t)pl * abytes + (size_t)nbox * 1024))[f] = 0.f;
    }
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (lane == 0 && nst > 0) {
      tc::tma_prefetch_desc(&tmap);
      const uint32_t bytes = (uint32_t)nbox * 1024u;
      for (int it = 0; it < nst; ++it) {
        const int s = it % NS;
        SKP_T0();
        if (it >= NS) tc::mbar_wait(&sfree[s], ((it / NS) & 1) ^ 1);
        SKP_ACC(0);
        tc::mbar_arrive_expect_tx(&full[s], bytes);
        const int c0 = (int)(cbeg + (int64_t)it * kBK);
        unsigned char *dst = xb + (size_t)s * abytes;
        if (p.L == 3)  // 3-D map (32 rows, columns, row blocks): all nbox boxes in one instruction
          tc::tma_load_3d(dst, &tmap, &full[s], 0, c0, 0);
        else  // (one TMA instruction per 1 KB box: the producer's issue rate bounds the kernel)
          for (int b = 0; b < nbox; ++b) tc::tma_load_2d(dst + b * 1024, &tmap, &full[s], 32 * b, c0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer (warp-wide)
    if (nst > 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(128, N, true, false);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t xb0 = __shfl_sync(0xffffffffu, tc::smem_u32(xb), 0);
      const uint32_t lb0 = __shfl_sync(0xffffffffu, tc::smem_u32(lb), 0);
      const uint32_t obh = __shfl_sync(0xffffffffu, tc::smem_u32(ohb), 0);
      const uint32_t obl = __shfl_sync(0xffffffffu, tc::smem_u32(olb), 0);
      for (int it = 0; it < nst; ++it) {
        const int s = it % NS, g = it % kNSG;
        SKP_T0();
        tc::mbar_wait(&oready[g], (it / kNSG) & 1);
        SKP_ACC(1);
        tc::mbar_wait(&xready[s], (it / NS) & 1);
        SKP_ACC(2);
        tc::tc_fence_after();
        const uint32_t xa = xb0 + s * abytes, la = lb0 + s * abytes;
        const uint64_t bh = tc::smem_desc(obh + g * obytes, 128, 256, tc::kSwNone);
        const uint64_t bl = tc::smem_desc(obl + g * obytes, 128, 256, tc::kSwNone);
        for (int mt = 0; mt < NT; ++mt) {
          const uint64_t ah = tc::smem_desc(xa + mt * 4096, 1024, 512, tc::kSw128Base32);
          const uint64_t al = tc::smem_desc(la + mt * 4096, 1024, 512, tc::kSw128Base32);
          const uint32_t d = tm + mt * N;
          tc::mma_tf32_w(d, ah, bh, idesc, it > 0 ? 1u : 0u);
          tc::mma_tf32_w(d, ah, bl, idesc, 1u);
          tc::mma_tf32_w(d, al, bh, idesc, 1u);
        }
        tc::mma_commit_w(&sfree[s]);
        tc::mma_commit_w(&oempty[g]);
      }
      tc::mma_commit_w(done);
    }
  } else if (warp < 2 + kGen) {
    // ------------------------------------------------------------- Omega generators
    const int gt = threadIdx.x - 64;  // 0 .. 32*kGen-1
    const int64_t jb0 = p.k0 >> 2;
    const int nb = (int)(((p.k0 + p.ell - 1) >> 2) - jb0 + 1);
    for (int it = 0; it < nst; ++it) {
      const int g = it % kNSG;
      const int64_t c0 = cbeg + (int64_t)it * kBK;
      SKP_T0();
      if (it >= kNSG) tc::mbar_wait(&oempty[g], ((it / kNSG) & 1) ^ 1);
      SKP_ACC(3);
      float *oh = (float *)(ohb + (size_t)g * obytes), *ol = (float *)(olb + (size_t)g * obytes);
      for (int t = gt; t < kBK * nb; t += 32 * kGen) {
        const int kk = t & (kBK - 1), jb = t >> 3;
        const int64_t c = c0 + kk;
        const bool valid = c < cend;
        const uint4 w = omega_words(p.seed, p.mode, 0, (uint64_t)(c + p.col_offset), (uint32_t)(jb0 + jb));
        Normal4<float> z(w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t n = 4 * (jb0 + jb) + q - p.k0;
          if (n >= 0 && n < p.ell) {
            const float v = valid ? z.v[q] : 0.f;
            const float hi = tc::tf32_hi(v);
            const int off = kmaj_off((int)n, kk) >> 2;
            oh[off] = hi;
            ol[off] = tc::tf32_lo(v, hi);
          }
        }
      }
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&oready[g]);
    }
  } else {
    // ------------------------------------------------------------- X workers
    const int wt = threadIdx.x - 32 * (2 + kGen);  // 0 .. 32*kMW-1
    const int nch = nbox * 64;                     // 16-byte chunks per stage
    const int ccol = (wt & 63) >> 3;               // the stage column all of this thread's chunks hold
    double nsq = 0.0;
    for (int it = 0; it < nst; ++it) {
      const int s = it % NS;
      SKP_T0();
      tc::mbar_wait(&full[s], (it / NS) & 1);  // (TMA refilled stage s only after its MMAs finished)
      SKP_ACC(4);
      const unsigned char *xs = xb + (size_t)s * abytes;
      unsigned char *ls = lb + (size_t)s * abytes;
      float acc = 0.f, cm = 0.f;
      // all of the thread's chunks (<= kMnaJ) loaded first, then split and stored: the loads
      // are independent, so their latency overlaps instead of chaining per chunk
      float4 xv[kMnaJ];
#pragma unroll
      for (int j = 0; j < kMnaJ; ++j) {
        const int q = wt + 32 * kMW * j;
        xv[j] = q < nch ? *(const float4 *)(xs + 16 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < kMnaJ; ++j) {
        const int q = wt + 32 * kMW * j;
        const float4 x = xv[j];
        float4 l;
        l.x = tc::tf32_rn(x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u));
        l.y = tc::tf32_rn(x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u));
        l.z = tc::tf32_rn(x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u));
        l.w = tc::tf32_rn(x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u));
        if (q < nch) *(float4 *)(ls + 16 * q) = l;
        acc = fmaf(x.x, x.x, acc); acc = fmaf(x.y, x.y, acc); acc = fmaf(x.z, x.z, acc); acc = fmaf(x.w, x.w, acc);
        cm = fmaxf(cm, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
      }
      if (p.colmax) {  // lanes 8g .. 8g + 7 of a warp share one column: 3 shuffles, one atomic
        cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
        cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
        cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 4));
        const int64_t c = cbeg + (int64_t)it * kBK + ccol;
        if ((lane & 7) == 0 && c < cend) atomicMax(p.colmax + c, __float_as_uint(cm));
      }
      nsq += (double)acc;
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&xready[s]);
    }
    // ---- epilogue: TMEM -> fp64 partial[blockIdx.x][k * I + i]
    const int q4 = warp & 3;                       // TMEM lane quadrant of this warp
    const int half = (warp - 2 - kGen) >> 2;       // 0 / 1: which 32 of the N columns
    if (nst > 0) {
      tc::mbar_wait(done, 0);
      tc::tc_fence_after();
    }
    float *dst = p.partial + (int64_t)blockIdx.x * p.ell * p.I;
    if (half * 32 < N) {
      for (int mt = 0; mt < NT; ++mt) {
        uint32_t rr[32];
        if (nst > 0) tc::tmem_ld32(tmem + ((uint32_t)(32 * q4) << 16) + mt * N + half * 32, rr);
        const int64_t i = (int64_t)mt * 128 + 32 * q4 + lane;
        if (i < p.I) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = half * 32 + j;
            if (k < p.ell) dst[(int64_t)k * p.I + i] = nst > 0 ? __uint_as_float(rr[j]) : 0.f;
          }
        }
      }
    }
    if (p.norm_partial) {
      for (int o = 16; o; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
      if (lane == 0) wsum[warp - 2 - kGen] = nsq;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (p.norm_partial && threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kMW; ++w) s += wsum[w];
    p.norm_partial[blockIdx.x] = s;
  }
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, tcols);
  }
#ifdef RTUCKER_SK_PROF_BUILD
  if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 64 || threadIdx.x == 192))
    printf("[mna prof] tid %d nst %d: wait sfree %lld oready %lld xready %lld oempty %lld full %lld total %lld\n",
           threadIdx.x, nst, skp[0], skp[1], skp[2], skp[3], skp[4], clock64() - skp_start);
#endif
}

#ifdef RTUCKER_EXPERIMENTS  // TMEM-A variant: measured slower, kept for experiments builds only
// ---------------------------------------------------------------------------------------------
// L == 1 variant with the A operand in TMEM (sketch_tc_ta_kernel).  The smem-operand kernel
// above spends ~70 % of the shared-memory bandwidth on the X operand (hi / lo planes written
// by the workers, read 3x by the MMAs: ~1900 wavefronts per 8-column stage, measured).  Here
// the workers split the staged X rows and store hi / lo straight into TMEM (tcgen05.st, lane =
// row i, one tf32 value per 32-bit column, K = 8 columns per MMA), so shared memory carries
// only the TMA staging, its one read and the small Omega tiles.  TMEM then holds the
// accumulators (<= 4 M-tiles x N columns, [0, 256)) and a ring of A stages ([256, 512):
// tile t of stage s at 256 + 16 (s NTg + t), hi in its first 8 columns, lo in the next 8), so
// a CTA covers at most 512 rows: the rows are split into ng = ceil(NT / 4) groups and CTA b
// takes row group b % ng of column range b / ng (X is still read once; Omega is generated
// by both CTAs of a column range).
//   warp 0 TMA (boxes of BR rows x 8 columns of the CTA's row group), warp 1 MMA issuer,
//   warps 2-5 Omega generators (as above), warps 6-13 workers: warp w owns TMEM lane quadrant
//   q = w % 4 and the tiles t = (w - 6) / 4 + 2 u, i.e. rows r = 128 t + 32 q + lane.
// D rows of rows outside the group (r >= rvalid) are never read, so their A lanes may hold
// anything.
constexpr int kTaCol = 256;  // first TMEM column of the A ring
constexpr int kTaGen = 8;    // Omega generator warps (groups of 4 warps share the stages)
constexpr int kTaWork = 8;   // X worker warps (kTaWq per TMEM lane quadrant)
constexpr int kTaWq = kTaWork / 4;
constexpr int kTaTpw = 4 / kTaWq;  // M-tiles per worker warp
constexpr int kTaNSG = 8;    // Omega stages
constexpr int kTaThreads = 32 * (2 + kTaGen + kTaWork);
static_assert(kTaGen % 4 == 0 && kTaWork % 4 == 0, "TA warp roles");

struct SketchTaParams {
  int64_t I, C, cps;
  int ng, RG, NTg, nbox, BR, NSS, NSA;
  int gsplit;            // Omega generator groups (stages round-robin over the groups)
  int acol;              // first TMEM column of the A ring (= NTg N)
  int ell;
  int64_t k0;
  uint64_t seed;
  int mode;
  int64_t col_offset;
  double *partial;       // [C ranges][ell][I]
  double *norm_partial;  // [grid] or null
  uint32_t *colmax;      // [C] or null
  long long *prof;       // optional: CTA 0 wait-cycle counters (RTUCKER_TA_PROF)
};

__device__ __forceinline__ void mma_tf32_ta(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b),
               "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

template <int N>
__global__ void __launch_bounds__(kTaThreads, 1)
    sketch_tc_ta_kernel(const __grid_constant__ CUtensorMap tmap, const SketchTaParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char *base = smem_raw + pad;
  const int NSS = p.NSS, NSA = p.NSA, NTg = p.NTg, BR = p.BR;
  const int sbytes = p.nbox * BR * kBK * 4;
  constexpr int obytes = N * kBK * 4;
  unsigned char *ohb = base;                          // [kTaNSG][obytes]
  unsigned char *olb = ohb + (size_t)kTaNSG * obytes; // [kTaNSG][obytes]
  unsigned char *sb = olb + (size_t)kTaNSG * obytes;  // [NSS][sbytes]
  uint64_t *full = (uint64_t *)(sb + (size_t)NSS * sbytes);
  uint64_t *sfree = full + NSS;
  uint64_t *aready = sfree + NSS;
  uint64_t *aempty = aready + NSA;
  uint64_t *oready = aempty + NSA;
  uint64_t *oempty = oready + kTaNSG;
  uint64_t *done = oempty + kTaNSG;
  uint32_t *tslot = (uint32_t *)(done + 1);
  double *wsum = (double *)(tslot + 2);  // [kTaWork]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = blockIdx.x % p.ng, cr = blockIdx.x / p.ng;
  const int64_t row0 = (int64_t)grp * p.RG;
  const int rvalid = (int)min((int64_t)p.RG, p.I - row0);
  const int64_t cbeg = (int64_t)cr * p.cps;
  const int64_t cend = min(p.C, cbeg + p.cps);
  const int nst = cend > cbeg ? (int)((cend - cbeg + kBK - 1) / kBK) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&sfree[s], 32 * kTaWork);
    }
    for (int s = 0; s < NSA; ++s) {
      tc::mbar_init(&aready[s], 32 * kTaWork);
      tc::mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < kTaNSG; ++s) {
      tc::mbar_init(&oready[s], 32 * kTaGen / p.gsplit);
      tc::mbar_init(&oempty[s], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 512);
  for (int e = threadIdx.x; e < 2 * kTaNSG * obytes / 4; e += kTaThreads) ((float *)ohb)[e] = 0.f;
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (lane == 0 && nst > 0) {
      tc::tma_prefetch_desc(&tmap);
      const int boxb = BR * kBK * 4;
      for (int it = 0; it < nst; ++it) {
        const int s = it % NSS;
        if (it >= NSS) tc::mbar_wait(&sfree[s], ((it / NSS) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&full[s], (uint32_t)sbytes);
        const int c0 = (int)(cbeg + (int64_t)it * kBK);
        unsigned char *dst = sb + (size_t)s * sbytes;
        for (int b = 0; b < p.nbox; ++b) tc::tma_load_2d(dst + b * boxb, &tmap, &full[s], (int)row0 + BR * b, c0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer (warp-wide)
    if (nst > 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(128, N, false, false);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t obh = __shfl_sync(0xffffffffu, tc::smem_u32(ohb), 0);
      const uint32_t obl = __shfl_sync(0xffffffffu, tc::smem_u32(olb), 0);
      long long w0 = 0, w1 = 0, w2 = 0;
      for (int it = 0; it < nst; ++it) {
        const int s = it % NSA, g = it % kTaNSG;
        const long long c0 = clock64();
        tc::mbar_wait(&oready[g], (it / kTaNSG) & 1);
        const long long c1 = clock64();
        tc::mbar_wait(&aready[s], (it / NSA) & 1);
        const long long c2 = clock64();
        w0 += c1 - c0; w1 += c2 - c1;
        tc::tc_fence_after();
        const uint64_t bh = tc::smem_desc(obh + g * obytes, 128, 256, tc::kSwNone);
        const uint64_t bl = tc::smem_desc(obl + g * obytes, 128, 256, tc::kSwNone);
        const uint32_t a0 = tm + p.acol + 16 * s * NTg;
        for (int t = 0; t < NTg; ++t) {
          const uint32_t d = tm + t * N, ah = a0 + 16 * t;
          tc::mma_tf32_ta_w(d, ah, bh, idesc, it > 0 ? 1u : 0u);
          tc::mma_tf32_ta_w(d, ah, bl, idesc, 1u);
          tc::mma_tf32_ta_w(d, ah + 8, bh, idesc, 1u);
        }
        tc::mma_commit_w(&aempty[s]);
        tc::mma_commit_w(&oempty[g]);
        w2 += clock64() - c2;
      }
      tc::mma_commit_w(done);
      if (p.prof && blockIdx.x == 0 && lane == 0) { p.prof[0] = w0; p.prof[1] = w1; p.prof[2] = w2; p.prof[3] = nst; }
    }
  } else if (warp < 2 + kTaGen) {
    // ------------------------------------------------------------- Omega generators
    // group gg = 0 / 1 of 4 warps fills the even / odd stages
    const int gsz = 32 * kTaGen / p.gsplit;
    const int gg = (threadIdx.x - 64) / gsz, gt = threadIdx.x - 64 - gsz * gg;
    const int64_t jb0 = p.k0 >> 2;
    const int nb = (int)(((p.k0 + p.ell - 1) >> 2) - jb0 + 1);
    for (int it = gg; it < nst; it += p.gsplit) {
      const int g = it % kTaNSG;
      const int64_t c0 = cbeg + (int64_t)it * kBK;
      if (it >= kTaNSG) tc::mbar_wait(&oempty[g], ((it / kTaNSG) & 1) ^ 1);
      float *oh = (float *)(ohb + (size_t)g * obytes), *ol = (float *)(olb + (size_t)g * obytes);
      for (int t = gt; t < kBK * nb; t += gsz) {
        const int kk = t & (kBK - 1), jb = t >> 3;
        const int64_t c = c0 + kk;
        const bool valid = c < cend;
        const uint4 w = omega_words(p.seed, p.mode, 0, (uint64_t)(c + p.col_offset), (uint32_t)(jb0 + jb));
        Normal4<float> z(w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t n = 4 * (jb0 + jb) + q - p.k0;
          if (n >= 0 && n < p.ell) {
            const float v = valid ? z.v[q] : 0.f;
            const float hi = tc::tf32_hi(v);
            const int off = kmaj_off((int)n, kk) >> 2;
            oh[off] = hi;
            ol[off] = tc::tf32_lo(v, hi);
          }
        }
      }
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&oready[g]);
    }
  } else {
    // ------------------------------------------------------------- X workers
    const int q = warp & 3, hw = (warp - 2 - kTaGen) >> 2;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    int soff[kTaTpw];
    bool rok[kTaTpw];
#pragma unroll
    for (int u = 0; u < kTaTpw; ++u) {
      const int t = hw + kTaWq * u;
      const int r = 128 * t + 32 * q + lane;
      rok[u] = t < NTg && r < rvalid;
      soff[u] = (r / BR) * (BR * kBK) + r % BR;
    }
    float acc = 0.f;
    double nsq = 0.0;
    int ss = 0, sa = 0;
    uint32_t ps = 0, pa = 0;
    long long w3 = 0, w4 = 0, tw0 = clock64();
    for (int it = 0; it < nst; ++it) {
      const long long c0 = clock64();
      if (it >= NSA) tc::mbar_wait(&aempty[sa], pa ^ 1);
      const long long c1 = clock64();
      tc::mbar_wait(&full[ss], ps);
      w3 += c1 - c0; w4 += clock64() - c1;
      tc::tc_fence_after();
      const float *st = (const float *)(sb + (size_t)ss * sbytes);
      float cm[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cm[u] = 0.f;
#pragma unroll
      for (int u = 0; u < kTaTpw; ++u) {
        const int t = hw + kTaWq * u;
        if (t < NTg) {  // warp-uniform
          float x[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) x[k] = rok[u] ? st[soff[u] + k * BR] : 0.f;
          uint32_t v[16];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float h = tc::tf32_hi(x[k]);
            v[k] = __float_as_uint(h);
            v[8 + k] = __float_as_uint(tc::tf32_lo(x[k], h));
            acc = fmaf(x[k], x[k], acc);
            cm[k] = fmaxf(cm[k], fabsf(x[k]));
          }
          tmem_st16(tmem + lane_base + p.acol + 16 * (sa * NTg + t), v);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc::mbar_arrive(&sfree[ss]);
      tc::tc_fence_before();
      tc::mbar_arrive(&aready[sa]);
      if (p.colmax) {  // transposing butterfly (see sketch_tc_mn_kernel)
        const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float keep = u16 ? cm[k + 4] : cm[k], send = u16 ? cm[k] : cm[k + 4];
          cm[k] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 16));
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float keep = u8 ? cm[k + 2] : cm[k], send = u8 ? cm[k] : cm[k + 2];
          cm[k] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 8));
        }
        {
          const float keep = u4 ? cm[1] : cm[0], send = u4 ? cm[0] : cm[1];
          cm[0] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 4));
        }
        cm[0] = fmaxf(cm[0], __shfl_xor_sync(0xffffffffu, cm[0], 2));
        cm[0] = fmaxf(cm[0], __shfl_xor_sync(0xffffffffu, cm[0], 1));
        const int64_t c = cbeg + (int64_t)it * kBK + (lane >> 2);
        if ((lane & 3) == 0 && c < cend) atomicMax(p.colmax + c, __float_as_uint(cm[0]));
      }
      nsq += (double)acc;
      acc = 0.f;
      if (++sa == NSA) { sa = 0; pa ^= 1; }
      if (++ss == NSS) { ss = 0; ps ^= 1; }
    }
    if (p.prof && blockIdx.x == 0 && threadIdx.x == 32 * (2 + kTaGen)) {
      p.prof[4] = w3; p.prof[5] = w4; p.prof[6] = clock64() - tw0;
    }
    // ---- epilogue: TMEM -> fp64 partial[cr][k * I + i]
    if (nst > 0) {
      tc::mbar_wait(done, 0);
      tc::tc_fence_after();
    }
    double *dst = p.partial + (int64_t)cr * p.ell * p.I;
    for (int t = hw; t < NTg; t += kTaWq) {
      for (int h = 0; h * 32 < N; ++h) {
        uint32_t rr[32];
        if (nst > 0) tc::tmem_ld32(tmem + lane_base + t * N + h * 32, rr);
        const int r = 128 * t + 32 * q + lane;
        if (r < rvalid) {
          const int64_t i = row0 + r;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = h * 32 + j;
            if (k < p.ell) dst[(int64_t)k * p.I + i] = nst > 0 ? __uint_as_float(rr[j]) : 0.f;
          }
        }
      }
    }
    if (p.norm_partial) {
      for (int o = 16; o; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
      if (lane == 0) wsum[warp - 2 - kTaGen] = nsq;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (p.norm_partial && threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kTaWork; ++w) s += wsum[w];
    p.norm_partial[blockIdx.x] = s;
  }
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

#endif  // RTUCKER_EXPERIMENTS

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    RT_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (!ptr || q != cudaDriverEntryPointSuccess) throw Error(RTUCKER_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
  }
  return fn;
}

// Y = sum over the CTAs of their fp32 partials, in fp64 and in CTA order (deterministic; the fp32
// partials are the TMEM values themselves, so this is the same sum as over fp64 copies at half
// the bytes)
__global__ void reduce_partials_f32_kernel(const float *__restrict__ partial, int nsplit, int64_t n,
                                           double *__restrict__ Y) {
  // four lanes per output (a serial chain over ~148 CTAs per thread was latency-bound): lane q of
  // the group sums the partials k = q, q + 4, ... in order, then (q0 + q1) + (q2 + q3)
  const int q = threadIdx.x & 3;
  for (int64_t e4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e4 < 4 * n; e4 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = e4 >> 2;  // (4 n is a multiple of 4 and the stride is too: groups stay aligned)
    double s = 0.0;
    for (int k = q; k < nsplit; k += 4) s += (double)partial[(int64_t)k * n + e];
    const unsigned gm = 0xFu << (threadIdx.x & 28);  // this group's four lanes (always all active)
    s += __shfl_xor_sync(gm, s, 1);
    s += __shfl_xor_sync(gm, s, 2);
    if (q == 0) Y[e] = s;
  }
}

__global__ void reduce_partials_kernel(const double *__restrict__ partial, int nsplit, int64_t n,
                                       double *__restrict__ Y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nsplit; ++k) s += partial[(int64_t)k * n + e];
    Y[e] = s;
  }
}

#ifdef RTUCKER_EXPERIMENTS
template <int N>
void launch_ta(Ctx &c, const CUtensorMap &tm, SketchTaParams &p, int grid, size_t smem) {
  auto k = sketch_tc_ta_kernel<N>;
  smem_attr(k, smem);
  RT_LAUNCH(c, k, grid, kTaThreads, smem, tm, p);
}

// L == 1 sketch with the A operand in TMEM (sketch_tc_ta_kernel).
bool sketch_ta(Ctx &c, const float *X, ModeView v, int mode, int ell, int64_t k0, uint64_t seed, int64_t col_offset,
               double *Y, double *normsq, uint32_t *colmax) {
  const int N = ell <= 32 ? 32 : 64;
  const int NT = (int)((v.I + 127) / 128);
  SketchTaParams p{};
  p.I = v.I;
  p.C = v.R;
  p.ng = (NT + 3) / 4;
  if (const char *e = RT_EXP_GETENV("RTUCKER_TA_NG")) p.ng = std::max(p.ng, atoi(e));  // experiments
  p.RG = (int)(((v.I + p.ng - 1) / p.ng + 7) / 8 * 8);
  p.NTg = (p.RG + 127) / 128;
  p.nbox = (p.RG + 255) / 256;
  p.BR = ((p.RG + p.nbox - 1) / p.nbox + 7) / 8 * 8;
  p.acol = p.NTg * N;
  p.NSA = std::min(8, (512 - p.acol) / (16 * p.NTg));
  p.gsplit = kTaGen / 4;
  static const bool prof = RT_EXP_GETENV("RTUCKER_TA_PROF") != nullptr;
  DevBuf<long long> pbuf;
  if (prof) {
    pbuf.alloc(c, 8);
    RT_CUDA(cudaMemsetAsync(pbuf.p, 0, 64, c.stream));
    p.prof = pbuf.p;
  }
  const size_t sbytes = (size_t)p.nbox * p.BR * kBK * 4, obytes = (size_t)N * kBK * 4;
  const size_t budget = 200 * 1024, fixed = 1024 + 2 * kTaNSG * obytes + 512;
  p.NSS = (int)std::min<size_t>(8, (budget - fixed) / sbytes);
  if (p.NSS < 2) return false;
  const size_t smem = fixed + p.NSS * sbytes;
  const int64_t nchunks = (p.C + kBK - 1) / kBK;
  const int ncr = (int)std::max<int64_t>(1, std::min<int64_t>(c.num_sms / p.ng, nchunks / 4));
  p.cps = ((nchunks + ncr - 1) / ncr) * kBK;
  const int ncr_used = (int)((p.C + p.cps - 1) / p.cps);
  const int grid = ncr_used * p.ng;
  p.ell = ell;
  p.k0 = k0;
  p.seed = seed;
  p.mode = mode;
  p.col_offset = col_offset;
  DevBuf<double> part(c, (size_t)ncr_used * ell * v.I);
  DevBuf<double> npart;
  if (normsq) npart.alloc(c, grid);
  p.partial = part.p;
  p.norm_partial = normsq ? npart.p : nullptr;
  p.colmax = colmax;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)v.I, (cuuint64_t)p.C};
  cuuint64_t strides[1] = {(cuuint64_t)v.I * 4};
  cuuint32_t box[2] = {(cuuint32_t)p.BR, kBK};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)X, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(RTUCKER_ECUDA, "cuTensorMapEncodeTiled failed for the sketch operand");
  if (N == 32) launch_ta<32>(c, tm, p, grid, smem);
  else launch_ta<64>(c, tm, p, grid, smem);
  if (prof) {
    long long h[8];
    RT_CUDA(cudaMemcpyAsync(h, pbuf.p, 64, cudaMemcpyDeviceToHost, c.stream));
    RT_CUDA(cudaStreamSynchronize(c.stream));
    fprintf(stderr, "[ta prof] nst %lld  mma: wait oready %lld aready %lld issue %lld | worker: wait aempty %lld full %lld total %lld\n",
            h[3], h[0], h[1], h[2], h[4], h[5], h[6]);
  }
  const int64_t n = v.I * ell;
  RT_LAUNCH(c, reduce_partials_kernel, (int)std::min<int64_t>(1024, (n + 255) / 256), 256, 0, part.p, ncr_used, n, Y);
  if (normsq) sum_vec(c, npart.p, grid, normsq);
  return true;
}

#endif  // RTUCKER_EXPERIMENTS

template <int N>
void launch_mna(Ctx &c, const CUtensorMap &tm, SketchTcParams &p, int grid, size_t smem) {
  auto k = sketch_tc_mna_kernel<N>;
  smem_attr(k, smem);
  RT_LAUNCH(c, k, grid, kMThreads, smem, tm, p);
}

// The MN-major-A route for L == 1 (sketch_tc_mna_kernel).  Returns false outside its envelope.
bool sketch_tc_mna(Ctx &c, const float *X, ModeView v, int mode, int ell, int64_t k0, uint64_t seed,
                   int64_t col_offset, double *Y, double *normsq, uint32_t *colmax) {
  const int N = ell <= 32 ? 32 : 64;
  const int NT = (int)((v.I + 127) / 128);
  if (NT * N > 512 || NT > 7 || (v.I % 4) != 0 || (((uintptr_t)X) & 15) != 0) return false;
  const int64_t C = v.L * v.R;
  if (C > (int64_t)INT32_MAX - 64) return false;
  SketchTcParams p{};
  p.I = v.I;
  p.C = C;
  p.NT = NT;
  p.nbox = (int)((v.I + 31) / 32);
  const size_t abytes = (size_t)NT * 4096, obytes = (size_t)N * kBK * 4;
  const size_t budget = 220 * 1024;
  const size_t fixed = 1024 + 2 * kNSG * obytes + 512;
  if (fixed + 2 * 2 * abytes > budget) return false;
  p.NSS = (int)std::min<size_t>(4, (budget - fixed) / (2 * abytes));
  const size_t smem = fixed + (size_t)p.NSS * 2 * abytes;
  const int64_t nchunks = (C + kBK - 1) / kBK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(c.num_sms, nchunks / 4));
  p.cps = ((nchunks + grid - 1) / grid) * kBK;
  const int g = (int)((C + p.cps - 1) / p.cps);
  p.ell = ell;
  p.k0 = k0;
  p.seed = seed;
  p.mode = mode;
  p.col_offset = col_offset;
  DevBuf<float> part(c, (size_t)g * ell * v.I);
  DevBuf<double> npart;
  if (normsq) npart.alloc(c, g);
  p.partial = part.p;
  p.norm_partial = normsq ? npart.p : nullptr;
  p.colmax = colmax;
  CUtensorMap tm;
  CUresult r;
  // p.L is reused as the map's rank: 3 when I % 32 == 0 and nbox <= 256 (dims: 32 rows i % 32,
  // columns c, row blocks i / 32 at a 128-byte stride, one box = a whole stage), else 2
  if (v.I % 32 == 0 && p.nbox <= 256) {
    p.L = 3;
    cuuint64_t dims[3] = {32, (cuuint64_t)C, (cuuint64_t)p.nbox};
    cuuint64_t strides[2] = {(cuuint64_t)v.I * 4, 128};
    cuuint32_t box[3] = {32, kBK, (cuuint32_t)p.nbox};
    cuuint32_t es[3] = {1, 1, 1};
    r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)X, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    p.L = 2;
    cuuint64_t dims[2] = {(cuuint64_t)v.I, (cuuint64_t)C};
    cuuint64_t strides[1] = {(cuuint64_t)v.I * 4};
    cuuint32_t box[2] = {32, kBK};
    cuuint32_t es[2] = {1, 1};
    r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)X, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) throw Error(RTUCKER_ECUDA, "cuTensorMapEncodeTiled failed for the MN-major sketch operand");
  if (N == 32) launch_mna<32>(c, tm, p, g, smem);
  else launch_mna<64>(c, tm, p, g, smem);
  const int64_t n = v.I * ell;
  RT_LAUNCH(c, reduce_partials_f32_kernel, (int)std::min<int64_t>(4096, (4 * n + 255) / 256), 256, 0, part.p, g, n, Y);
  if (normsq) sum_vec(c, npart.p, g, normsq);
  return true;
}

template <int N, bool KM>
void launch(Ctx &c, const CUtensorMap &tm, SketchTcParams &p, int grid, size_t smem) {
  auto k = sketch_tc_mn_kernel<N, KM>;
  smem_attr(k, smem);
  RT_LAUNCH(c, k, grid, kThreads, smem, tm, p);
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return encode_fn(); }

bool sketch_tc_enabled() {
  static const bool off = RT_EXP_GETENV("RTUCKER_NO_TC") != nullptr;
  return !off;
}

// Y (I x ell fp64, column-major) = X_(n) Omega(:, k0:k0+ell) for fp32 X (L == 1, or L > 1 with
// L and I multiples of 8: the K-major variant).
// Returns false when the shape is outside this kernel's envelope (caller falls back).
bool sketch_tc_mn(Ctx &c, const float *X, ModeView v, int mode, int ell, int64_t k0, uint64_t seed,
                  int64_t col_offset, double *Y, double *normsq, uint32_t *colmax) {
  static const bool off = RT_EXP_GETENV("RTUCKER_NO_TC_SKETCH") != nullptr;
  if (off || !sketch_tc_enabled() || ell > 64 || ell < 1) return false;
  const bool km = v.L > 1;  // K-major variant: l contiguous (5-D TMA box, no transposition)
  if (!km && (v.I % 4) != 0) return false;
  if (km && ((v.L % 8) != 0 || (v.I % 8) != 0 || v.I / 8 > 256)) return false;
  // L == 1: X tiles straight into the MN-major A operand (RTUCKER_SKETCH_KMAJOR in experiments
  // builds selects the transposing K-major kernel below)
  static const bool kmajor = RT_EXP_GETENV("RTUCKER_SKETCH_KMAJOR") != nullptr;
  if (!km && !kmajor && sketch_tc_mna(c, X, v, mode, ell, k0, seed, col_offset, Y, normsq, colmax)) return true;
#ifdef RTUCKER_EXPERIMENTS
  static const bool ta = RT_EXP_GETENV("RTUCKER_SKETCH_TA") != nullptr;  // TMEM-A variant (experimental)
  if (!km && ta && (((uintptr_t)X) & 15) == 0 && v.I <= 2048 && v.L * v.R <= (int64_t)INT32_MAX - 64)
    return sketch_ta(c, X, v, mode, ell, k0, seed, col_offset, Y, normsq, colmax);
#endif
  const int N = ell <= 32 ? 32 : 64;
  const int NT = (int)((v.I + 127) / 128);
  if (NT * N > 512 || (((uintptr_t)X) & 15) != 0) return false;
  const int64_t C = v.L * v.R;
  if (C > (int64_t)INT32_MAX - 64) return false;
  SketchTcParams p{};
  p.I = v.I;
  p.C = C;
  p.L = v.L;
  p.NT = NT;
  p.nbox = km ? 1 : (int)((v.I + 255) / 256);
  p.BR = km ? (int)v.I : (int)(((v.I + p.nbox - 1) / p.nbox + 7) / 8 * 8);
  const size_t sbytes = (size_t)p.nbox * p.BR * kBK * 4, abytes = (size_t)NT * 128 * kBK * 4,
               obytes = (size_t)N * kBK * 4;
  const size_t budget = 220 * 1024;
  p.NSO = 2;
  const size_t fixed = 1024 + 2 * p.NSO * abytes + 2 * kNSG * obytes + 512;
  if (fixed + 2 * sbytes > budget) return false;
  p.NSS = (int)std::min<size_t>(4, (budget - fixed) / sbytes);
  const size_t smem = fixed + p.NSS * sbytes;
  const int64_t nchunks = (C + kBK - 1) / kBK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(c.num_sms, nchunks / 4));
  p.cps = ((nchunks + grid - 1) / grid) * kBK;
  const int g = (int)((C + p.cps - 1) / p.cps);
  p.ell = ell;
  p.k0 = k0;
  p.seed = seed;
  p.mode = mode;
  p.col_offset = col_offset;
  DevBuf<float> part(c, (size_t)g * ell * v.I);
  DevBuf<double> npart;
  if (normsq) npart.alloc(c, g);
  p.partial = part.p;
  p.norm_partial = normsq ? npart.p : nullptr;
  p.colmax = colmax;

  CUtensorMap tm;
  CUresult r;
  if (!km) {
    cuuint64_t dims[2] = {(cuuint64_t)v.I, (cuuint64_t)C};
    cuuint64_t strides[1] = {(cuuint64_t)v.I * 4};
    cuuint32_t box[2] = {(cuuint32_t)p.BR, kBK};
    cuuint32_t es[2] = {1, 1};
    r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)X, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    // (l % 4, i % 8, l / 4, i / 8, r): the box lands as K-major core matrices of 8 rows x 16 B
    cuuint64_t dims[5] = {4, 8, (cuuint64_t)v.L / 4, (cuuint64_t)v.I / 8, (cuuint64_t)v.R};
    cuuint64_t strides[4] = {(cuuint64_t)v.L * 4, 16, (cuuint64_t)v.L * 32, (cuuint64_t)v.L * v.I * 4};
    cuuint32_t box[5] = {4, 8, 2, (cuuint32_t)(v.I / 8), 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, (void *)X, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) throw Error(RTUCKER_ECUDA, "cuTensorMapEncodeTiled failed for the sketch operand");
  if (km) {
    if (N == 32) launch<32, true>(c, tm, p, g, smem);
    else launch<64, true>(c, tm, p, g, smem);
  } else {
    if (N == 32) launch<32, false>(c, tm, p, g, smem);
    else launch<64, false>(c, tm, p, g, smem);
  }
  const int64_t n = v.I * ell;
  RT_LAUNCH(c, reduce_partials_f32_kernel, (int)std::min<int64_t>(4096, (4 * n + 255) / 256), 256, 0, part.p, g, n, Y);
  if (normsq) sum_vec(c, npart.p, g, normsq);
  return true;
}

}  // namespace rt
