// Tensor-core (tcgen05, 3xTF32) B-pass of mode n for fp32 data with L == 1 (mode 1):
//   B = Q^T X_(n)   (Alg 1 line 3),  B stored (L=1, l, R): B[k + l c]
// X_(n) is I x C column-major, so the contraction index i is the contiguous one and the
// X tile is a K-major operand without any transpose: a 4-D TMA map (i_in 4, c_in 8,
// i_out I/4, c_out C/8) writes the canonical no-swizzle K-major layout (8 rows x 16 B core
// matrices, LBO = 128 B along K, SBO = 1024 B along M) straight from HBM.
//
//   warp 0       TMA producer: per stage (32 values of i) the X box (128 c x 32 i, 16 KB) and
//                the pre-split Q chunk (hi/lo, 64 k x 32 i, 16 KB, bulk copy from L2)
//   warp 1       TMEM allocation + MMA issuer: per stage 4 k-steps x 3 MMAs
//                D = Xhi Qhi + Xhi Qlo + Xlo Qhi (M=128, N=64, K=8) into a FRESH accumulator
//                (two TMEM buffers of 64 columns, alternating per stage)
//   warps 2-5    epilogue: per stage, TMEM -> registers, added into fp64 running sums (one
//                row c per thread, 64 doubles); after a unit's last stage B(c, :) is stored.
//                fp32 accumulation therefore spans only the 32 terms of one stage: summing the
//                whole I = 800 terms in TMEM gave a B error of 6e-6 relative at C4, which moved
//                the rank-50 eigen-subspace of the Gram (gap ~5e-7 of lambda_1) and the C4
//                relative error by 1e-2
//   warps 6-9    split workers: X = hi + lo in place (both rounded to the tf32 grid, DESIGN
//                R15; lo to a buffer of the same layout; elementwise, layout-agnostic)
// A work unit is 128 consecutive columns c; CTAs are persistent and stride over units.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels.h"
#include "tc.cuh"

namespace rt {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();  // sketch_tc.cu

namespace {

constexpr int kUnit = 128;            // columns per work unit (1 M-tile)
constexpr int kKC = 32;               // values of i per stage
constexpr int kXBytes = kUnit * kKC * 4;   // 16 KB
constexpr int kQBytes = 64 * kKC * 4;      // one Q plane chunk, 8 KB
constexpr int kNS = 4;
constexpr int kEpi = 4, kSplit = 4;
constexpr int kThreads = 32 * (2 + kEpi + kSplit);

struct BpassParams {
  int64_t I, C;
  int ell;
  int nkc;                 // K chunks (ceil(I / 32))
  int64_t nunits;
  const float *qp;         // [nkc][2][64][32] in the smem operand layout
  void *B;                 // output, B[k + ell * c]
  int out_f64;
};

template <bool kF64>
__global__ void __launch_bounds__(kThreads, 1)
    bpass_tc_kernel(const __grid_constant__ CUtensorMap tmap, const BpassParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char *base = smem_raw + pad;
  unsigned char *xb = base;                             // [kNS][kXBytes]  X (hi after split)
  unsigned char *lb = xb + kNS * kXBytes;               // [kNS][kXBytes]  X lo
  unsigned char *qb = lb + kNS * kXBytes;               // [kNS][2 * kQBytes] Q hi, Q lo
  uint64_t *full = (uint64_t *)(qb + kNS * 2 * kQBytes);
  uint64_t *ready = full + kNS;
  uint64_t *empty = ready + kNS;
  uint64_t *accfull = empty + kNS;     // [2]
  uint64_t *accempty = accfull + 2;    // [2]
  uint32_t *tslot = (uint32_t *)(accempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nmine = p.nunits > blockIdx.x ? (p.nunits - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t nst = nmine * p.nkc;   // stages of this CTA

  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&ready[s], 32 * kSplit);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&accfull[b], 1);
      tc::mbar_init(&accempty[b], 32 * kEpi);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tslot, 128);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (lane == 0) {
      tc::tma_prefetch_desc(&tmap);
      for (int64_t it = 0; it < nst; ++it) {
        const int s = (int)(it % kNS);
        if (it >= kNS) tc::mbar_wait(&empty[s], (uint32_t)((it / kNS) & 1) ^ 1);
        const int64_t u = blockIdx.x + (it / p.nkc) * gridDim.x;
        const int kc = (int)(it % p.nkc);
        tc::mbar_arrive_expect_tx(&full[s], kXBytes + 2 * kQBytes);
        // X box: i_in 0..3, c_in 0..7, i_out 8 kc .. +8, c_out 16 u .. +16
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5}], [%6];" ::"r"(tc::smem_u32(xb + s * kXBytes)),
            "l"(&tmap), "r"(0), "r"(0), "r"(8 * kc), "r"((int)(16 * u)), "r"(tc::smem_u32(&full[s]))
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                tc::smem_u32(qb + s * 2 * kQBytes)),
            "l"(p.qp + (size_t)kc * 2 * 64 * kKC), "r"(2 * kQBytes), "r"(tc::smem_u32(&full[s]))
            : "memory");
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer (warp-wide)
    {
      constexpr uint32_t idesc = tc::idesc_tf32(128, 64, false, false);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t xb0 = __shfl_sync(0xffffffffu, tc::smem_u32(xb), 0);
      const uint32_t lb0 = __shfl_sync(0xffffffffu, tc::smem_u32(lb), 0);
      const uint32_t qb0 = __shfl_sync(0xffffffffu, tc::smem_u32(qb), 0);
      for (int64_t it = 0; it < nst; ++it) {
        const int s = (int)(it % kNS);
        const int ab = (int)(it & 1);          // accumulator buffer
        if (it >= 2) tc::mbar_wait(&accempty[ab], (uint32_t)(((it / 2) & 1) ^ 1));
        tc::mbar_wait(&ready[s], (uint32_t)((it / kNS) & 1));
        tc::tc_fence_after();
        const uint32_t xa = xb0 + s * kXBytes, la = lb0 + s * kXBytes;
        const uint32_t qh = qb0 + s * 2 * kQBytes, ql = qh + kQBytes;
        const uint32_t d = tm + ab * 64;
        for (int ks = 0; ks < kKC / 8; ++ks) {
          const uint64_t ah = tc::smem_desc(xa + ks * 256, 128, 1024, tc::kSwNone);
          const uint64_t al = tc::smem_desc(la + ks * 256, 128, 1024, tc::kSwNone);
          const uint64_t bh = tc::smem_desc(qh + ks * 256, 128, 1024, tc::kSwNone);
          const uint64_t bl = tc::smem_desc(ql + ks * 256, 128, 1024, tc::kSwNone);
          tc::mma_tf32_w(d, ah, bh, idesc, ks ? 1u : 0u);
          tc::mma_tf32_w(d, ah, bl, idesc, 1u);
          tc::mma_tf32_w(d, al, bh, idesc, 1u);
        }
        tc::mma_commit_w(&empty[s]);
        tc::mma_commit_w(&accfull[ab]);
      }
    }
  } else if (warp < 2 + kEpi) {
    // ------------------------------------------------------------- epilogue
    const int q4 = warp & 3;  // TMEM lane quadrant = rows 32 q4 .. of the M-tile
    double acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0;
    for (int64_t it = 0; it < nst; ++it) {
      const int ab = (int)(it & 1);
      tc::mbar_wait(&accfull[ab], (uint32_t)((it / 2) & 1));
      tc::tc_fence_after();
      {
        uint32_t r[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q4) << 16) + ab * 64, r);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] += (double)__uint_as_float(r[j]);
        tc::tmem_ld32(tmem + ((uint32_t)(32 * q4) << 16) + ab * 64 + 32, r);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[32 + j] += (double)__uint_as_float(r[j]);
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&accempty[ab]);
      if ((int)(it % p.nkc) == p.nkc - 1) {  // unit complete: store B(c, :) and reset
        const int64_t u = blockIdx.x + (it / p.nkc) * gridDim.x;
        const int64_t c = u * kUnit + 32 * q4 + lane;
        if (c < p.C) {
          if (kF64) {
            double *dst = (double *)p.B + c * p.ell;
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (j < p.ell) dst[j] = acc[j];
          } else {
            float *dst = (float *)p.B + c * p.ell;
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (j < p.ell) dst[j] = (float)acc[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 64; ++j) acc[j] = 0.0;
      }
    }
  } else {
    // ------------------------------------------------------------- split workers
    const int wt = threadIdx.x - 32 * (2 + kEpi);
    for (int64_t it = 0; it < nst; ++it) {
      const int s = (int)(it % kNS);
      tc::mbar_wait(&full[s], (uint32_t)((it / kNS) & 1));
      float4 *xv = (float4 *)(xb + s * kXBytes);
      float4 *lv = (float4 *)(lb + s * kXBytes);
#pragma unroll 4
      for (int e = wt; e < kXBytes / 16; e += 32 * kSplit) {
        const float4 x = xv[e];
        float4 h, l;
        h.x = tc::tf32_hi(x.x); h.y = tc::tf32_hi(x.y); h.z = tc::tf32_hi(x.z); h.w = tc::tf32_hi(x.w);
        l.x = tc::tf32_lo(x.x, h.x); l.y = tc::tf32_lo(x.y, h.y); l.z = tc::tf32_lo(x.z, h.z); l.w = tc::tf32_lo(x.w, h.w);
        xv[e] = h;
        lv[e] = l;
      }
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&ready[s]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 128);
  }
}

// Q (I x ell fp64, leading dim ldq) -> [nkc][hi/lo][64 k][32 i] fp32 in the K-major
// no-swizzle operand layout: element (k, i) at (k/8)*1024 + (i/4)*128 + (k%8)*16 + (i%4)*4 B.
__global__ void prep_q_kernel(const double *__restrict__ Q, int64_t ldq, int64_t I, int ell, int nkc,
                              float *__restrict__ out) {
  const int64_t n = (int64_t)nkc * 64 * kKC;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int kc = (int)(e / (64 * kKC));
    const int rem = (int)(e % (64 * kKC));
    const int k = rem / kKC, ii = rem % kKC;
    const int64_t i = (int64_t)kc * kKC + ii;
    const float v = (k < ell && i < I) ? (float)Q[i + ldq * k] : 0.f;
    const float hi = tc::tf32_hi(v);
    const int off = ((k >> 3) * 1024 + (ii >> 2) * 128 + (k & 7) * 16 + (ii & 3) * 4) >> 2;
    float *dst = out + (size_t)kc * 2 * 64 * kKC;
    dst[off] = hi;
    dst[64 * kKC + off] = tc::tf32_lo(v, hi);
  }
}

}  // namespace

// B = Q^T X_(n) for fp32 X with L == 1 (B[k + ell c]); Q fp64 I x ell (ld = ldq).  Returns
// false outside the kernel's envelope (caller falls back to the SIMT TTM).
bool bpass_tc_mn(Ctx &c, const float *X, ModeView v, const double *Q, int64_t ldq, int ell, void *B, bool out_f64) {
  static const bool off = RT_EXP_GETENV("RTUCKER_NO_TC_BPASS") != nullptr;
  if (off || !sketch_tc_enabled() || v.L != 1 || (v.I % 4) != 0 || (v.R % 8) != 0 || ell > 64 || ell < 1) return false;
  if ((((uintptr_t)X) & 15) != 0 || v.R / 8 > (int64_t)INT32_MAX / 2) return false;
  BpassParams p{};
  p.I = v.I;
  p.C = v.R;
  p.ell = ell;
  p.nkc = (int)((v.I + kKC - 1) / kKC);
  p.nunits = (v.R + kUnit - 1) / kUnit;
  p.B = B;
  p.out_f64 = out_f64;
  DevBuf<float> qp(c, (size_t)p.nkc * 2 * 64 * kKC);
  p.qp = qp.p;
  {
    const int64_t n = (int64_t)p.nkc * 64 * kKC;
    RT_LAUNCH(c, prep_q_kernel, (int)std::min<int64_t>(1024, (n + 255) / 256), 256, 0, Q, ldq, v.I, ell, p.nkc, qp.p);
  }
  CUtensorMap tm;
  const uint64_t C = (uint64_t)v.R, I = (uint64_t)v.I;
  cuuint64_t dims[4] = {4, 8, I / 4, C / 8};
  cuuint64_t strides[3] = {I * 4, 16, I * 32};  // bytes of dims 1..3
  cuuint32_t box[4] = {4, 8, kKC / 4, kUnit / 8};  // 4 x 8 x 8 x 16 = 128 c x 32 i
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = tensor_map_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void *)X, dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(RTUCKER_ECUDA, "cuTensorMapEncodeTiled failed for the B-pass operand");
  const size_t smem = 1024 + kNS * (2 * kXBytes + 2 * kQBytes) + 256;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(c.num_sms, p.nunits));
  if (out_f64) {
    smem_attr(bpass_tc_kernel<true>, smem);
    RT_LAUNCH(c, bpass_tc_kernel<true>, grid, kThreads, smem, tm, p);
  } else {
    smem_attr(bpass_tc_kernel<false>, smem);
    RT_LAUNCH(c, bpass_tc_kernel<false>, grid, kThreads, smem, tm, p);
  }
  return true;
}

}  // namespace rt
