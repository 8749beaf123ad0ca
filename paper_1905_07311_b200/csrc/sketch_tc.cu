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
//                write both TRANSPOSED into K-major operand tiles (the tensor core reads tf32
//                operands K-major only: MN-major tf32 A or B measured as all-zero output on
//                this B200, scripts/dbg/tc_probe.cu); accumulate ||X||^2; after the last
//                stage: TMEM -> fp64 partial Y.
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
  double *partial;       // [grid][ell][I]
  double *norm_partial;  // [grid] or null
  uint32_t *colmax;      // [C] fp32 bits of max_i |X(i, c)| (atomic max), or null (L == 1 only)
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
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0 && nst > 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(128, N, false, false);
      for (int it = 0; it < nst; ++it) {
        const int s = it % NSO, g = it % kNSG;
        tc::mbar_wait(&oready[g], (it / kNSG) & 1);
        tc::mbar_wait(&xready[s], (it / NSO) & 1);
        tc::tc_fence_after();
        const uint32_t ha = tc::smem_u32(hb + (size_t)s * abytes);
        const uint32_t la = tc::smem_u32(lb + (size_t)s * abytes);
        const uint64_t bh = tc::smem_desc(tc::smem_u32(ohb + (size_t)g * obytes), 128, 256, tc::kSwNone);
        const uint64_t bl = tc::smem_desc(tc::smem_u32(olb + (size_t)g * obytes), 128, 256, tc::kSwNone);
        for (int mt = 0; mt < NT; ++mt) {
          const uint64_t ah = tc::smem_desc(ha + mt * 128 * kBK * 4, 128, 256, tc::kSwNone);
          const uint64_t al = tc::smem_desc(la + mt * 128 * kBK * 4, 128, 256, tc::kSwNone);
          const uint32_t d = tmem + mt * N;
          tc::mma_tf32(d, ah, bh, idesc, it > 0 ? 1u : 0u);
          tc::mma_tf32(d, ah, bl, idesc, 1u);
          tc::mma_tf32(d, al, bh, idesc, 1u);
        }
        tc::mma_commit(&xempty[s]);
        tc::mma_commit(&oempty[g]);
      }
      tc::mma_commit(done);
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
      if (KM) {  // staging and operand planes share the K-major layout: elementwise split
        const int nun = p.nbox * p.BR * kBK / 4;  // float4 units
        for (int u = wt; u < nun; u += 32 * kWorkers) {
          const float4 x = *(const float4 *)(st + 4 * u);
          float4 h, l;
          h.x = tc::tf32_hi(x.x); h.y = tc::tf32_hi(x.y); h.z = tc::tf32_hi(x.z); h.w = tc::tf32_hi(x.w);
          l.x = tc::tf32_lo(x.x, h.x); l.y = tc::tf32_lo(x.y, h.y); l.z = tc::tf32_lo(x.z, h.z); l.w = tc::tf32_lo(x.w, h.w);
          *(float4 *)(hs + 16 * u) = h;
          *(float4 *)(ls + 16 * u) = l;
          acc = fmaf(x.x, x.x, acc); acc = fmaf(x.y, x.y, acc); acc = fmaf(x.z, x.z, acc); acc = fmaf(x.w, x.w, acc);
        }
      }
      float cm[8];  // this thread's column maxima of the stage (L == 1: 8 columns c0 .. c0+7)
#pragma unroll
      for (int u = 0; u < 8; ++u) cm[u] = 0.f;
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
      if (!KM && p.colmax) {  // warp max per column, one atomic per warp and column
        const int64_t c0 = cbeg + (int64_t)it * kBK;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t m = __reduce_max_sync(0xffffffffu, __float_as_uint(cm[u]));
          if (lane == 0 && c0 + u < cend) atomicMax(p.colmax + c0 + u, m);
        }
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
    double *dst = p.partial + (int64_t)blockIdx.x * p.ell * p.I;
    if (half * 32 < N) {
      for (int mt = 0; mt < NT; ++mt) {
        uint32_t rr[32];
        if (nst > 0) tc::tmem_ld32(tmem + ((uint32_t)(32 * q4) << 16) + mt * N + half * 32, rr);
        const int64_t i = (int64_t)mt * 128 + 32 * q4 + lane;
        if (i < p.I) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = half * 32 + j;
            if (k < p.ell) dst[(int64_t)k * p.I + i] = nst > 0 ? (double)__uint_as_float(rr[j]) : 0.0;
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

__global__ void reduce_partials_kernel(const double *__restrict__ partial, int nsplit, int64_t n,
                                       double *__restrict__ Y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nsplit; ++k) s += partial[(int64_t)k * n + e];
    Y[e] = s;
  }
}

template <int N, bool KM>
void launch(Ctx &c, const CUtensorMap &tm, SketchTcParams &p, int grid, size_t smem) {
  auto k = sketch_tc_mn_kernel<N, KM>;
  RT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RT_LAUNCH(c, k, grid, kThreads, smem, tm, p);
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return encode_fn(); }

bool sketch_tc_enabled() {
  static const bool off = getenv("RTUCKER_NO_TC") != nullptr;
  return !off;
}

// Y (I x ell fp64, column-major) = X_(n) Omega(:, k0:k0+ell) for fp32 X (L == 1, or L > 1 with
// L and I multiples of 8: the K-major variant).
// Returns false when the shape is outside this kernel's envelope (caller falls back).
bool sketch_tc_mn(Ctx &c, const float *X, ModeView v, int mode, int ell, int64_t k0, uint64_t seed,
                  int64_t col_offset, double *Y, double *normsq, uint32_t *colmax) {
  static const bool off = getenv("RTUCKER_NO_TC_SKETCH") != nullptr;
  if (off || !sketch_tc_enabled() || ell > 64 || ell < 1) return false;
  const bool km = v.L > 1;  // K-major variant: l contiguous (5-D TMA box, no transposition)
  if (!km && (v.I % 4) != 0) return false;
  if (km && ((v.L % 8) != 0 || (v.I % 8) != 0 || v.I / 8 > 256)) return false;
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
  DevBuf<double> part(c, (size_t)g * ell * v.I);
  DevBuf<double> npart;
  if (normsq) npart.alloc(c, g);
  p.partial = part.p;
  p.norm_partial = normsq ? npart.p : nullptr;
  p.colmax = km ? nullptr : colmax;

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
  RT_LAUNCH(c, reduce_partials_kernel, (int)std::min<int64_t>(1024, (n + 255) / 256), 256, 0, part.p, g, n, Y);
  if (normsq) sum_vec(c, npart.p, g, normsq);
  return true;
}

}  // namespace rt
