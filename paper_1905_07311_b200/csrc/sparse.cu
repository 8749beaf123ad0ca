// Structure-preserving SP-STHOSVD (Alg 6) for COO tensors:
//   for j in rho:  Y = G_(j) Omega_j                 (sketch over the nonzeros)
//                  Q = qr(Y)
//                  S = strong RRQR on Q^T, eta       (DESIGN reading R9: CPQR + maxvol)
//                  A_j = Q (P^T Q)^{-1}
//                  G_(j) <- P^T G_(j)                (keep the selected slices, renumber)
// The core keeps the input values bit-exactly.
//
// Determinism (RTUCKER_DETERMINISTIC): the sketch sums in FIXED POINT.  Every
// product v * omega (exact or fp64-rounded, as in the oracle) is scaled by 2^S and split into
// an integer part H (units of 2^32) and a 32-bit fraction L; all reductions (lanes, warps,
// CTAs, and the ranks of a multi-GPU run through an integer allreduce) add int64 words, which
// is associative, so Y is bit-identical for any launch shape, schedule or GPU count.  S is
// chosen from max|v| and the global nnz so that no partial sum overflows (|omega| < 8 since
// u >= 2^-33): the resolution is 2^-65 of the largest term, below fp64 rounding.
//
// Nothing here synchronises the host until the end of the call: the current nnz stays on
// the device (kernels are sized for the input nnz and read the live count), the sRRQR
// selection runs in one cooperative kernel, and the final sizes are read back once.
//
// Multi-GPU: nnz-partitioned.  Each rank sketches its own nonzeros, the
// integer partial sketches are allreduced (exact), QR and sRRQR run redundantly (identical
// inputs, deterministic kernels -> identical selections), each rank filters its own nonzeros,
// and the core nonzeros are gathered in rank order at the end (= the single-GPU order when
// the partition is contiguous in the input order).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "comm.h"
#include "kernels_extra.h"
#include "orchestrate.h"
#include "philox.cuh"

namespace cg = cooperative_groups;

namespace rt {

namespace {

constexpr int kCooT = 256;
constexpr int kMaxEll = 64;

// ------------------------------------------------------------ fixed-point scale --
struct FixScale {
  double mul;    // 2^S: product -> fixed point (units of 2^-S... split at 2^32 below)
  double outH;   // 2^(32 - S): weight of the H word
  double outL;   // 2^-S: weight of the L word
  int S;
};

template <typename TV>
__global__ void abs_max_kernel(const TV *__restrict__ v, int64_t n, unsigned long long *__restrict__ out) {
  double m = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs((double)v[e]));
  // a non-negative double orders like its bit pattern: the maximum is order-independent
  unsigned long long b = (unsigned long long)__double_as_longlong(m);
  for (int o = 16; o; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, b, o);
    b = t > b ? t : b;
  }
  if ((threadIdx.x & 31) == 0 && b) atomicMax(out, b);
}

// S = 91 - ceil(log2 N) - e with max|v| < 2^e: |v omega 2^S| < 2^(94 - ceil(log2 N)), so the
// H words (|H| < 2^(62 - ceil(log2 N))) and the L words (< 2^32 each) of N terms never overflow.
__global__ void fix_scale_kernel(const unsigned long long *__restrict__ maxbits, const int64_t *__restrict__ nglob,
                                 FixScale *__restrict__ fs) {
  const double m = __longlong_as_double((long long)*maxbits);
  int e = 0;
  if (m > 0.0) frexp(m, &e);
  const int64_t N = *nglob > 1 ? *nglob : 1;
  const int lg = N > 1 ? 64 - __clzll((unsigned long long)(N - 1)) : 0;
  int S = 91 - lg - e;
  S = S > 1000 ? 1000 : (S < -1000 ? -1000 : S);
  fs->S = S;
  fs->mul = ldexp(1.0, S);
  fs->outH = ldexp(1.0, 32 - S);
  fs->outL = ldexp(1.0, -S);
}

__device__ __forceinline__ void to_fixed(double prod, double mul, long long &H, long long &L) {
  const double T = prod * mul;                 // exact power-of-two scaling
  const double hf = floor(T * 0x1p-32);
  H = (long long)hf;
  L = __double2ll_rn(T - hf * 0x1p32);         // exact difference in [0, 2^32), fraction rounded
}

// ---------------------------------------------------------------- COO sketch (a8) --
// Y[i_j, k] += v * Omega_j[c, k], c = sum_{m != j} i_m prod_{m' < m, m' != j} I_m', in fixed
// point (see the file header).  Count tensors are heavy-tailed (BASELINE configs[4]: Zipf(1.1)
// indices; the heaviest mode-3 row holds ~9 % of the nonzeros), so lanes holding the same row
// are first combined (__match_any_sync + a shuffle tree over the group), rows < hot (the heavy
// rows of these tensors) go to warp-private shared-memory accumulators (one writer lane per
// row and instruction) flushed once per CTA, other rows to global int64 atomics (one per
// distinct row and warp).  Integer adds make every one of these orders give the same sum.
template <typename TV, typename TN>
__global__ void __launch_bounds__(kCooT) sketch_coo_kernel(CooDev g, const int64_t *__restrict__ nnz_dev, int mode,
                                                           int ell, int hot, uint64_t seed,
                                                           const FixScale *__restrict__ fs,
                                                           unsigned long long *__restrict__ YH,
                                                           unsigned long long *__restrict__ YL) {
  extern __shared__ long long hsm[];  // [warps][hot][ell] H, then the same for L
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kW = kCooT / 32;
  const int64_t I = g.dims[mode];
  const int hrows = (int)(I < hot ? I : hot);
  long long *hH = hsm + (size_t)warp * hot * ell;
  long long *hL = hsm + (size_t)(kW + warp) * hot * ell;
  for (int e = threadIdx.x; e < 2 * kW * hot * ell; e += kCooT) hsm[e] = 0;
  __syncthreads();
  int64_t stride[kMaxModes];
  int64_t s = 1;
  for (int k = 0; k < g.d; ++k) {
    stride[k] = (k == mode) ? 0 : s;
    if (k != mode) s *= g.dims[k];
  }
  const double mul = fs->mul;
  const TV *vals = (const TV *)g.vals;
  const int nb = (ell + 3) >> 2;
  const int64_t nnz = nnz_dev ? *nnz_dev : g.nnz;
  const int64_t nper = (nnz + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = (int64_t)blockIdx.x * nper, e1 = min(nnz, e0 + nper);
  for (int64_t base = e0 + (int64_t)warp * 32; base < e1; base += kCooT) {  // uniform trip count per warp
    const int64_t e = base + lane;
    const bool act = e < e1;
    int64_t c = 0;
    int row = -1;
    double v = 0.0;
    if (act) {
      for (int k = 0; k < g.d; ++k) c += (int64_t)g.idx[k][e] * stride[k];
      row = g.idx[mode][e];
      v = (double)vals[e];
    }
    const unsigned grp = __match_any_sync(0xffffffffu, row);
    const int leader = __ffs(grp) - 1;
    const bool big = __any_sync(0xffffffffu, __popc(grp) > 2);
    unsigned src[5];
    const int rank = __popc(grp & ((1u << lane) - 1u));
    if (big) {
#pragma unroll
      for (int k = 0; k < 5; ++k) src[k] = __fns(grp, lane, 1 + (1 << k));
    }
    for (int jb = 0; jb < nb; ++jb) {
      long long h[4] = {0, 0, 0, 0}, l[4] = {0, 0, 0, 0};
      if (act) {
        const uint4 w = omega_words(seed, mode, 0, (uint64_t)c, (uint32_t)jb);
        Normal4<TN> z(w);
#pragma unroll
        for (int q = 0; q < 4; ++q) to_fixed(v * (double)z.v[q], mul, h[q], l[q]);
      }
      if (!big) {  // groups of <= 2 lanes: every member adds the others' words
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          long long th = 0, tl = 0;
          unsigned m = grp;
          while (m) {
            const int sl = __ffs(m) - 1;
            th += __shfl_sync(grp, h[q], sl);
            tl += __shfl_sync(grp, l[q], sl);
            m &= m - 1;
          }
          h[q] = th;
          l[q] = tl;
        }
      } else {  // tree over the group: partner = the member 2^k ranks further (__fns)
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const bool take = src[k] != 0xffffffffu && (rank & ((2 << k) - 1)) == 0;
          const int sl = (src[k] != 0xffffffffu) ? (int)src[k] : lane;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const long long oh = __shfl_sync(0xffffffffu, h[q], sl);
            const long long ol = __shfl_sync(0xffffffffu, l[q], sl);
            if (take) {
              h[q] += oh;
              l[q] += ol;
            }
          }
        }
      }
      if (act && lane == leader) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = 4 * jb + q;
          if (k < ell) {
            if (row < hrows) {
              hH[row * ell + k] += h[q];
              hL[row * ell + k] += l[q];
            } else {
              atomicAdd(&YH[row + I * k], (unsigned long long)h[q]);
              atomicAdd(&YL[row + I * k], (unsigned long long)l[q]);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < hrows * ell; e += kCooT) {
    long long th = 0, tl = 0;
    for (int w = 0; w < kW; ++w) {
      th += hsm[(size_t)w * hot * ell + e];
      tl += hsm[(size_t)(kW + w) * hot * ell + e];
    }
    const int r = e / ell, k = e % ell;
    if (th) atomicAdd(&YH[r + I * k], (unsigned long long)th);
    if (tl) atomicAdd(&YL[r + I * k], (unsigned long long)tl);
  }
}

// ------------------------------------------- bucketed COO sketch (default, a8) --
// Count tensors are heavy-tailed (BASELINE configs[4]: Zipf(1.1) indices; in mode 3 the
// heaviest row holds ~9 % of the nonzeros and every one of the 200000 rows a few), so a
// per-nonzero global atomic (2 words x ell columns) is what bounds a direct scatter into Y.
// Instead:
//   pass 0  bucket_hist     nonzeros per bucket of kBR consecutive rows (per-CTA shared-
//                           memory counters, one global atomic per CTA and bucket)
//   scan    bucket_scan     bucket offsets and the work units (<= unit nonzeros of one bucket)
//   pass 1  bucket_scatter  every nonzero to its bucket: key = Omega column index c | local row
//                           << 56, value; per chunk one cursor atomic per bucket reserves a
//                           contiguous range (the write frontiers, one per bucket, stay in L2)
//   pass 2  bucket_sketch   one work item per CTA iteration: Y rows of the bucket accumulate in
//                           shared memory (int64 fixed point) with ONE writer per address: warp
//                           w owns columns 4(w & 3) .. +3 of copy (w >> 2), lanes of a warp
//                           holding the same row are combined by a shuffle tree first; then one
//                           global atomic pair per touched (row, column) of the item.
// Integer additions make the result independent of every order involved (R20).
constexpr int kBR = 128;          // rows per bucket (local row: 7 bits of the key)
constexpr int kMaxBk = 8192;      // buckets (I <= 2^20)
constexpr int kBT = 256;          // threads of the bucket kernels
constexpr int kBChunk = 8192;     // nonzeros per scatter chunk
constexpr int kItemMax = 65536;   // nonzeros per sketch work unit (at most; see bucket_scan)
constexpr int kSub = 2048, kRun = kSub / kBT;  // bucket_sketch sub-chunk, nonzeros per lane
constexpr uint64_t kKeyMask = (1ull << 56) - 1;

__global__ void __launch_bounds__(kBT) bucket_hist(CooDev g, const int64_t *__restrict__ nnz_dev, int mode, int nbk,
                                                  unsigned *__restrict__ gcnt) {
  extern __shared__ unsigned cnt[];  // nbk
  for (int t = threadIdx.x; t < nbk; t += kBT) cnt[t] = 0;
  __syncthreads();
  const int64_t nnz = nnz_dev ? *nnz_dev : g.nnz;
  const int lane = threadIdx.x & 31;
  for (int64_t base = ((int64_t)blockIdx.x * kBT + threadIdx.x) & ~(int64_t)31; base < nnz;
       base += (int64_t)gridDim.x * kBT) {
    const int64_t e = base + lane;
    const int bk = e < nnz ? g.idx[mode][e] / kBR : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, bk);
    if (bk >= 0 && lane == __ffs(grp) - 1) atomicAdd(&cnt[bk], (unsigned)__popc(grp));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nbk; t += kBT)
    if (cnt[t]) atomicAdd(&gcnt[t], cnt[t]);
}

// One CTA: bstart[b] (exclusive scan of the counts, bstart[nbk] = nnz), cursor = bstart, and
// istart[b] = first work unit of bucket b (ceil(cnt / unit) of them), istart[nbk] = units.
__device__ __forceinline__ int64_t block_excl_scan(int64_t x, int64_t *sh, int64_t &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int64_t s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
    int64_t si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += y;
    }
    sh[lane] = si - s;
    if (lane == 31) sh[32] = si;
  }
  __syncthreads();
  const int64_t r = sh[w] + inc - x;
  total = sh[32];
  __syncthreads();
  return r;
}
constexpr int kScanT = 1024, kScanPer = kMaxBk / kScanT;
__global__ void __launch_bounds__(kScanT) bucket_scan(const unsigned *__restrict__ cnt, int nbk,
                                                     unsigned *__restrict__ bstart, unsigned *__restrict__ cur,
                                                     int *__restrict__ istart, int *__restrict__ work, int grid) {
  __shared__ int64_t sh[33];
  unsigned v[kScanPer];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int i = threadIdx.x * kScanPer + k;
    v[k] = i < nbk ? cnt[i] : 0u;
    s += v[k];
  }
  int64_t tot, itot;
  int64_t run = block_excl_scan(s, sh, tot);
  // work-unit size from the live nonzero count: ~4 units per CTA of bucket_sketch, a multiple
  // of its sub-chunk, at most kItemMax
  const int64_t u = (tot / (4 * (int64_t)grid) + kSub - 1) / kSub * kSub;
  const int unit = (int)(u < kSub ? kSub : (u > kItemMax ? kItemMax : u));
  int64_t si = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) si += (v[k] + unit - 1) / unit;
  int64_t irun = block_excl_scan(si, sh, itot);
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int i = threadIdx.x * kScanPer + k;
    if (i < nbk) {
      bstart[i] = (unsigned)run;
      cur[i] = (unsigned)run;
      istart[i] = (int)irun;
    }
    run += v[k];
    irun += (v[k] + unit - 1) / unit;
  }
  if (threadIdx.x == 0) {
    bstart[nbk] = (unsigned)tot;
    istart[nbk] = (int)itot;
    work[0] = 0;
    work[1] = unit;
  }
}

template <typename TV>
__global__ void __launch_bounds__(kBT) bucket_scatter(CooDev g, const int64_t *__restrict__ nnz_dev, int mode, int nbk,
                                                     unsigned *__restrict__ cur, uint64_t *__restrict__ skey,
                                                     TV *__restrict__ sval) {
  extern __shared__ unsigned bsc[];
  unsigned *lcnt = bsc, *lbase = bsc + nbk;
  const int64_t nnz = nnz_dev ? *nnz_dev : g.nnz;
  const int lane = threadIdx.x & 31;
  int64_t stride[kMaxModes];
  int64_t s = 1;
  for (int k = 0; k < g.d; ++k) {
    stride[k] = (k == mode) ? 0 : s;
    if (k != mode) s *= g.dims[k];
  }
  const TV *vals = (const TV *)g.vals;
  for (int64_t c0 = (int64_t)blockIdx.x * kBChunk; c0 < nnz; c0 += (int64_t)gridDim.x * kBChunk) {
    const int64_t c1 = min(nnz, c0 + kBChunk);
    for (int t = threadIdx.x; t < nbk; t += kBT) lcnt[t] = 0;
    __syncthreads();
    for (int64_t b0 = c0 + (threadIdx.x & ~31); b0 < c1; b0 += kBT) {
      const int64_t e = b0 + lane;
      const int bk = e < c1 ? g.idx[mode][e] / kBR : -1;
      const unsigned grp = __match_any_sync(0xffffffffu, bk);
      if (bk >= 0 && lane == __ffs(grp) - 1) atomicAdd(&lcnt[bk], (unsigned)__popc(grp));
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nbk; t += kBT) {
      if (lcnt[t]) lbase[t] = atomicAdd(&cur[t], lcnt[t]);
      lcnt[t] = 0;
    }
    __syncthreads();
    for (int64_t b0 = c0 + (threadIdx.x & ~31); b0 < c1; b0 += kBT) {
      const int64_t e = b0 + lane;
      const bool act = e < c1;
      int row = -1, bk = -1;
      uint64_t c = 0;
      TV v = TV(0);
      if (act) {
        for (int k = 0; k < g.d; ++k) c += (uint64_t)((int64_t)g.idx[k][e] * stride[k]);
        row = g.idx[mode][e];
        bk = row / kBR;
        v = vals[e];
      }
      const unsigned grp = __match_any_sync(0xffffffffu, bk);
      const int leader = __ffs(grp) - 1;
      unsigned pos = 0;
      if (act && lane == leader) pos = lbase[bk] + atomicAdd(&lcnt[bk], (unsigned)__popc(grp));
      pos = __shfl_sync(0xffffffffu, pos, leader) + (unsigned)__popc(grp & ((1u << lane) - 1u));
      if (act) {
        skey[pos] = c | ((uint64_t)(row - bk * kBR) << 56);
        sval[pos] = v;
      }
    }
    __syncthreads();
  }
}

// Pass 2 work unit: <= unit consecutive nonzeros of one bucket, taken by a CTA from a global
// counter.  The unit's Y rows (kBR x 16 columns x (H, L) int64) accumulate in shared memory
// and are flushed once (one global atomic pair per touched word).  The unit is processed in
// sub-chunks of kSub nonzeros, each first counting-sorted by local row in shared memory; then
// every lane sums a run of kRun consecutive sorted nonzeros in registers and emits per row
// segment: segments strictly inside its run belong to this lane alone (plain add), its first
// segment may continue the previous lane's (shared-memory atomic), and the runs' last segments
// are combined across the warp by a segmented shuffle reduction (rows are sorted, so equal rows
// sit in consecutive lanes) whose head lane adds atomically.
constexpr size_t kBSmem = sizeof(long long) * 2 * kBR * 16   // accumulators
                          + sizeof(uint64_t) * kSub + sizeof(double) * kSub  // sorted keys, values
                          + sizeof(int) * 2 * kBR + 16;                     // row counts, offsets

__device__ __forceinline__ void seg_add(long long *aH, long long *aL, int lr, int nq, const long long (&H)[16],
                                        const long long (&L)[16]) {
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    if (q < nq) {
      aH[lr * 16 + q] += H[q];
      aL[lr * 16 + q] += L[q];
    }
  }
}

template <typename TV, typename TN>
__global__ void __launch_bounds__(kBT, 3) bucket_sketch(const uint64_t *__restrict__ skey, const TV *__restrict__ sval,
                                                       const unsigned *__restrict__ bstart,
                                                       const int *__restrict__ istart, int nbk, int64_t I, int mode,
                                                       int ell, uint64_t seed, const FixScale *__restrict__ fs,
                                                       int *__restrict__ work, unsigned long long *__restrict__ YH,
                                                       unsigned long long *__restrict__ YL) {
  extern __shared__ __align__(16) long long bsm[];
  long long *aH = bsm, *aL = aH + kBR * 16;
  uint64_t *sk = (uint64_t *)(aL + kBR * 16);
  double *sv = (double *)(sk + kSub);
  int *lcnt = (int *)(sv + kSub), *loff = lcnt + kBR;
  __shared__ int sunit;
  __shared__ int brow[kBT / 32];
  __shared__ long long bH[kBT / 32 * 16], bL[kBT / 32 * 16];
  const int lane = threadIdx.x & 31, tid = threadIdx.x;
  const double mul = fs->mul;
  const int nunits = istart[nbk];
  const int unit = work[1];
  while (true) {
    if (tid == 0) sunit = atomicAdd(work, 1);
    __syncthreads();
    const int it = sunit;
    __syncthreads();
    if (it >= nunits) break;
    int lo = 0, hi = nbk - 1;  // bucket of unit it: largest b with istart[b] <= it
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (istart[mid] <= it) lo = mid;
      else hi = mid - 1;
    }
    const int b = lo;
    const int64_t u0 = (int64_t)bstart[b] + (int64_t)(it - istart[b]) * unit;
    const int64_t u1 = min((int64_t)bstart[b + 1], u0 + unit);
    for (int cb = 0; cb < ell; cb += 16) {
      const int nq = min(16, ell - cb);
      for (int t = tid; t < 2 * kBR * 16; t += kBT) aH[t] = 0;  // aH and aL are contiguous
      for (int64_t s0 = u0; s0 < u1; s0 += kSub) {
        const int n = (int)min((int64_t)kSub, u1 - s0);
        for (int t = tid; t < kBR; t += kBT) lcnt[t] = 0;
        __syncthreads();
        // local counting sort by row (rank inside a row from warp-aggregated smem atomics)
        uint64_t kk[kRun];
        double vv[kRun];
        int rk[kRun];
#pragma unroll
        for (int k = 0; k < kRun; ++k) {
          const int i = tid + kBT * k;
          const bool act = i < n;
          kk[k] = act ? skey[s0 + i] : 0;
          vv[k] = act ? (double)sval[s0 + i] : 0.0;
          const int lr = act ? (int)(kk[k] >> 56) : -1;
          const unsigned grp = __match_any_sync(0xffffffffu, lr);
          const int leader = __ffs(grp) - 1;
          int base = 0;
          if (act && lane == leader) base = atomicAdd(&lcnt[lr], __popc(grp));
          rk[k] = __shfl_sync(0xffffffffu, base, leader) + __popc(grp & ((1u << lane) - 1u));
        }
        __syncthreads();
        if (tid < 32) {  // exclusive scan of the kBR = 128 counts, 4 per lane
          int c4[4], t4 = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) { c4[j] = lcnt[4 * lane + j]; t4 += c4[j]; }
          int inc = t4;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
          }
          int run = inc - t4;
#pragma unroll
          for (int j = 0; j < 4; ++j) { loff[4 * lane + j] = run; run += c4[j]; }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kRun; ++k) {
          if (tid + kBT * k < n) {
            const int o = loff[(int)(kk[k] >> 56)] + rk[k];
            sk[o] = kk[k];
            sv[o] = vv[k];
          }
        }
        __syncthreads();
        // lane-serial segments over the sorted sub-chunk.  Rows a lane completes inside its run
        // (its first segment included) are distinct across all lanes of the CTA, so they are
        // added without atomics; the runs' last segments are added after a barrier.
        const int i0 = tid * kRun, i1 = min(n, i0 + kRun);
        long long H[16], L[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) H[q] = L[q] = 0;
        int cur = i0 < i1 ? (int)(sk[i0] >> 56) : -1;
        for (int i = i0; i < i1; ++i) {
          const uint64_t key = sk[i];
          const int r = (int)(key >> 56);
          if (r != cur) {
            seg_add(aH, aL, cur, nq, H, L);
#pragma unroll
            for (int q = 0; q < 16; ++q) H[q] = L[q] = 0;
            cur = r;
          }
          const double v = sv[i];
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) {
            if (4 * jb < nq) {
              const uint4 w = omega_words(seed, mode, 0, key & kKeyMask, (uint32_t)(cb / 4 + jb));
              Normal4<TN> z(w);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                long long h, l;
                to_fixed(v * (double)z.v[q], mul, h, l);
                H[4 * jb + q] += h;
                L[4 * jb + q] += l;
              }
            }
          }
        }
        // last segments: suffix sums over consecutive lanes holding the same row (sorted)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int ro = __shfl_down_sync(0xffffffffu, cur, o);
          const bool take = lane + o < 32 && ro == cur;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const long long oh = __shfl_down_sync(0xffffffffu, H[q], o);
            const long long ol = __shfl_down_sync(0xffffffffu, L[q], o);
            if (take) {
              H[q] += oh;
              L[q] += ol;
            }
          }
        }
        const int rp = __shfl_up_sync(0xffffffffu, cur, 1);
        __syncthreads();  // every in-run segment added
        // group heads: the group of lane 0 may continue the previous warp's last group -> its
        // warp's boundary slot; every other group's row is this warp's alone
        const int warp = tid >> 5;
        if (lane == 0) {
          brow[warp] = cur;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            bH[warp * 16 + q] = H[q];
            bL[warp * 16 + q] = L[q];
          }
        } else if (cur >= 0 && rp != cur) {
          seg_add(aH, aL, cur, nq, H, L);
        }
        __syncthreads();
        if (tid < 32) {  // boundary slots in warp order, one thread per word
          const int q = tid & 15;
          long long *dst = tid < 16 ? aH : aL;
          const long long *src = tid < 16 ? bH : bL;
          for (int w = 0; w < kBT / 32; ++w)
            if (brow[w] >= 0 && q < nq) dst[brow[w] * 16 + q] += src[w * 16 + q];
        }
        __syncthreads();
      }
      for (int t = tid; t < kBR * 16; t += kBT) {
        const int r = t >> 4, q = t & 15;
        const int64_t row = (int64_t)b * kBR + r;
        if (q >= nq || row >= I) continue;
        const int64_t o = row + I * (cb + q);
        if (aH[t]) atomicAdd(&YH[o], (unsigned long long)aH[t]);
        if (aL[t]) atomicAdd(&YL[o], (unsigned long long)aL[t]);
      }
      __syncthreads();
    }
  }
}

__global__ void y_from_fixed_kernel(const long long *__restrict__ YH, const long long *__restrict__ YL, int64_t n,
                                    const FixScale *__restrict__ fs, double *__restrict__ Y) {
  const double oh = fs->outH, ol = fs->outL;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    Y[e] = fma((double)YH[e], oh, (double)YL[e] * ol);
}

// ------------------------------------------------------------- argmax helpers --
struct ArgMax {
  double v;
  int64_t i;
};
__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
  return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}
// CTA-wide argmax (ties to the smallest index); the result is returned to every thread.
__device__ ArgMax block_argmax_all(ArgMax m) {
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  __shared__ ArgMax res;
  for (int o = 16; o; o >>= 1) {
    ArgMax t{__shfl_xor_sync(0xffffffffu, m.v, o), __shfl_xor_sync(0xffffffffu, m.i, o)};
    m = better(m, t);
  }
  __syncthreads();  // sv/si/res may still be read by a previous call
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = m.v;
    si[threadIdx.x >> 5] = m.i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = better(m, ArgMax{sv[w], si[w]});
    res = m;
  }
  __syncthreads();
  return res;
}

// ------------------------------------------ sRRQR selection (a9), one cooperative kernel --
// Reading R9 (oracle/srrqr.py): Businger-Golub CPQR on Q^T (pivot = largest residual column
// norm sum_{t >= j} r_i[t]^2, ties to the smallest index; Householder reflector in the oracle's
// form) gives the initial S; then, while max_{i not in S, k} |A_ik| > eta with A = Q Q_S^{-1}
// (ties: smallest i, then smallest k), swap S_k <- i; finally S is sorted and A is formed for
// the sorted selection.  Each step's reduction is over all rows of the grid (per-CTA argmax,
// grid.sync, every CTA reduces the partials in the same order -> identical decisions).
// Q_S^{-1} by Gauss-Jordan with partial pivoting, redundantly in every CTA; a pivot below
// l eps max|Q_S| marks P^T Q singular (status ST_SINGULAR_PQ -> ENUMERIC).
constexpr int kSrT = 256;

// Gauss-Jordan inverse of Q[sel, :] (l x l) into inv (column-major), M scratch (l x 2l row-major).
// Returns false when singular.  All threads of the CTA call it.
__device__ bool gj_inverse(const double *__restrict__ Q, int64_t m, int l, const int64_t *sel, double *M, double *inv) {
  __shared__ int piv;
  __shared__ double amax;
  __shared__ int bad;
  const int w = 2 * l;
  for (int e = threadIdx.x; e < l * w; e += blockDim.x) {
    const int r = e / w, cc = e % w;
    M[e] = cc < l ? Q[sel[r] + m * cc] : (cc - l == r ? 1.0 : 0.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int r = 0; r < l; ++r)
      for (int cc = 0; cc < l; ++cc) a = fmax(a, fabs(M[r * w + cc]));
    amax = a;
    bad = 0;
  }
  __syncthreads();
  for (int col = 0; col < l; ++col) {
    if (threadIdx.x == 0) {
      int best = col;
      for (int r = col + 1; r < l; ++r)
        if (fabs(M[r * w + col]) > fabs(M[best * w + col])) best = r;
      piv = best;
      if (!(fabs(M[best * w + col]) > l * 2.2e-16 * amax)) bad = 1;
    }
    __syncthreads();
    const int pr = piv;
    if (pr != col)
      for (int cc = threadIdx.x; cc < w; cc += blockDim.x) {
        const double t = M[col * w + cc];
        M[col * w + cc] = M[pr * w + cc];
        M[pr * w + cc] = t;
      }
    __syncthreads();
    const double dinv = 1.0 / M[col * w + col];
    __syncthreads();
    for (int cc = threadIdx.x; cc < w; cc += blockDim.x) M[col * w + cc] *= dinv;
    __syncthreads();
    for (int e = threadIdx.x; e < l * w; e += blockDim.x) {
      const int r = e / w, cc = e % w;
      if (r != col && cc != col) M[e] -= M[r * w + col] * M[col * w + cc];
    }
    __syncthreads();
    for (int r = threadIdx.x; r < l; r += blockDim.x)
      if (r != col) M[r * w + col] = 0.0;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) {
    const int a = e % l, b = e / l;
    inv[e] = M[a * w + l + b];
  }
  __syncthreads();
  return bad == 0;
}

__global__ void __launch_bounds__(kSrT) srrqr_coop_kernel(const double *__restrict__ Q, int64_t m, int l, double eta,
                                                          int max_swaps, double *__restrict__ r, int *__restrict__ mark,
                                                          double *__restrict__ pv, int64_t *__restrict__ pi,
                                                          int64_t *__restrict__ sel_out, double *__restrict__ A,
                                                          int *__restrict__ swaps_out, unsigned *__restrict__ status) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sh[];
  double *M = sh;                        // l x 2l
  double *inv = M + 2 * l * l;           // l x l
  double *hv = inv + l * l;              // Householder vector (l)
  __shared__ int64_t ssel[kMaxEll];
  __shared__ int hv_ok;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = gt; e < m * l; e += gs) {
    const int64_t i = e / l;
    const int t = (int)(e % l);
    r[e] = Q[i + m * t];
  }
  for (int64_t i = gt; i < m; i += gs) mark[i] = 0;
  grid.sync();
  // Per-CTA candidates go to alternating halves of pv / pi (2 gridDim.x entries each): a CTA that
  // runs ahead writes the other half, and it cannot reach the call after that (the same half
  // again) before every CTA has passed this call's barrier, i.e. finished reading: one grid
  // barrier per reduction instead of two.
  int am_par = 0;
  auto global_argmax = [&](ArgMax b) -> ArgMax {
    b = block_argmax_all(b);
    double *pvh = pv + (size_t)am_par * gridDim.x;
    int64_t *pih = pi + (size_t)am_par * gridDim.x;
    am_par ^= 1;
    if (threadIdx.x == 0) {
      pvh[blockIdx.x] = b.v;
      pih[blockIdx.x] = b.i;
    }
    grid.sync();
    ArgMax gb{-1.0, INT64_MAX};
    for (int q = threadIdx.x; q < (int)gridDim.x; q += blockDim.x) gb = better(gb, ArgMax{pvh[q], pih[q]});
    gb = block_argmax_all(gb);
    return gb;
  };
  // ---- Businger-Golub CPQR on Q^T
  for (int j = 0; j < l; ++j) {
    ArgMax b{-1.0, INT64_MAX};
    for (int64_t i = gt; i < m; i += gs) {
      if (mark[i]) continue;
      double s2 = 0.0;
      for (int t = j; t < l; ++t) s2 += r[i * l + t] * r[i * l + t];
      b = better(b, ArgMax{s2, i});
    }
    const int64_t p = global_argmax(b).i;
    if (threadIdx.x == 0) {
      ssel[j] = p;
      // reflector from row p, rows j..l-1 (alpha = -sign(v0) ||v||, v0 -= alpha, v /= ||v||)
      double nv = 0.0;
      for (int t = j; t < l; ++t) {
        hv[t] = r[p * l + t];
        nv += hv[t] * hv[t];
      }
      nv = sqrt(nv);
      hv_ok = 0;
      if (nv != 0.0) {
        const double alpha = hv[j] >= 0.0 ? -nv : nv;
        hv[j] -= alpha;
        double vn = 0.0;
        for (int t = j; t < l; ++t) vn += hv[t] * hv[t];
        vn = sqrt(vn);
        if (vn != 0.0) {
          for (int t = j; t < l; ++t) hv[t] /= vn;
          hv_ok = 1;
        }
      }
    }
    __syncthreads();
    if (hv_ok)
      for (int64_t i = gt; i < m; i += gs) {
        if (i == p) continue;  // read by every CTA above; never used again
        double s2 = 0.0;
        for (int t = j; t < l; ++t) s2 += hv[t] * r[i * l + t];
        for (int t = j; t < l; ++t) r[i * l + t] -= 2.0 * s2 * hv[t];
      }
    if (gt == 0) mark[p] = 1;
    grid.sync();
  }
  // ---- maxvol swaps while max_{i not in S} |A_ik| > eta
  int swaps = 0;
  bool singular = false;
  while (true) {
    if (!gj_inverse(Q, m, l, ssel, M, inv)) {
      singular = true;
      break;
    }
    ArgMax b{-1.0, INT64_MAX};
    for (int64_t i = gt; i < m; i += gs) {
      if (mark[i]) continue;
      for (int k = 0; k < l; ++k) {
        double s2 = 0.0;
        for (int t = 0; t < l; ++t) s2 = fma(Q[i + m * t], inv[t + l * k], s2);
        b = better(b, ArgMax{fabs(s2), i * l + k});
      }
    }
    const ArgMax gb = global_argmax(b);
    if (!(gb.v > eta) || swaps >= max_swaps) break;
    const int64_t i = gb.i / l;
    const int k = (int)(gb.i % l);
    const int64_t old = ssel[k];
    __syncthreads();
    if (threadIdx.x == 0) ssel[k] = i;
    if (gt == 0) {
      mark[old] = 0;
      mark[i] = 1;
    }
    ++swaps;
    grid.sync();
  }
  if (singular) {
    if (gt == 0) atomicOr(status, (unsigned)ST_SINGULAR_PQ);
    return;  // uniform over the grid (every CTA computed the same inverse)
  }
  // ---- sort S ascending; A = Q Q_S^{-1} for the sorted selection
  if (threadIdx.x == 0)
    for (int a = 1; a < l; ++a)
      for (int b2 = a; b2 > 0 && ssel[b2 - 1] > ssel[b2]; --b2) {
        const int64_t t = ssel[b2];
        ssel[b2] = ssel[b2 - 1];
        ssel[b2 - 1] = t;
      }
  __syncthreads();
  gj_inverse(Q, m, l, ssel, M, inv);
  for (int64_t i = gt; i < m; i += gs)
    for (int k = 0; k < l; ++k) {
      double s2 = 0.0;
      for (int t = 0; t < l; ++t) s2 = fma(Q[i + m * t], inv[t + l * k], s2);
      A[i + m * k] = s2;
    }
  if (gt == 0) *swaps_out = swaps;
  if (blockIdx.x == 0)
    for (int t = threadIdx.x; t < l; t += blockDim.x) sel_out[t] = ssel[t];
}

// ------------------------------------------------------- selection / compaction (a10) --
// Keep the nonzeros whose mode-n index is selected and renumber it to its position in the
// sorted selection; order-preserving (per-block counts, one exclusive scan, scatter).  The
// live nnz is read from the device; grids are sized for the input nnz (an upper bound) and
// blocks past the live count exit.
__global__ void build_lookup(const int64_t *__restrict__ sel, int ell, int32_t *__restrict__ lut) {
  for (int t = threadIdx.x; t < ell; t += blockDim.x) lut[sel[t]] = t;
}

constexpr int kCompactB = 1024;

// Per-mode lookup tables of a selection: lut[m][i] = position of i in S_m, or -1; a null table
// keeps every index of that mode (single-mode filter of SP-STHOSVD, all-mode filter of SP-HOSVD).
struct LutSet {
  const int32_t *lut[kMaxModes];
};

__device__ __forceinline__ bool keep_entry(const CooDev &in, const LutSet &ls, int64_t e) {
  for (int k = 0; k < in.d; ++k)
    if (ls.lut[k] && ls.lut[k][in.idx[k][e]] < 0) return false;
  return true;
}

// Order-preserving compaction with a fixed grid: CTA b owns the contiguous range
// [b chunk, (b+1) chunk) of the live nonzeros (chunk from the live nnz on the device), counts its
// survivors, a one-CTA scan turns the per-CTA counts into offsets, and the scatter pass re-walks
// the range in 1024-entry steps with a running offset.  The grid does not depend on the live nnz,
// so nothing waits for the host.
constexpr int kCompactG = 1024;  // max CTAs
__device__ __forceinline__ void compact_range(int64_t nnz, int64_t &b0, int64_t &b1) {
  const int64_t chunk = ((nnz + gridDim.x - 1) / gridDim.x + kCompactB - 1) / kCompactB * kCompactB;
  b0 = min(nnz, (int64_t)blockIdx.x * chunk);
  b1 = min(nnz, b0 + chunk);
}

__global__ void __launch_bounds__(kCompactB) compact_count(CooDev in, const int64_t *__restrict__ nnz_dev, LutSet ls,
                                                           int64_t *__restrict__ counts) {
  __shared__ int sc[32];
  int64_t b0, b1;
  compact_range(*nnz_dev, b0, b1);
  int mine = 0;
  for (int64_t e = b0 + threadIdx.x; e < b1; e += kCompactB) mine += keep_entry(in, ls, e) ? 1 : 0;
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0) sc[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kCompactB / 32; ++w) t += sc[w];
    counts[blockIdx.x] = t;
  }
}

// One CTA: exclusive scan of n <= kCompactG values (thread t owns entry t), total to *total.
__global__ void exclusive_scan_single(int64_t *__restrict__ v, int64_t n, int64_t *__restrict__ total) {
  __shared__ int64_t sh[kCompactG];
  const int t = threadIdx.x;
  const int64_t x = t < n ? v[t] : 0;
  sh[t] = x;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // Hillis-Steele inclusive scan
    const int64_t y = t >= o ? sh[t - o] : 0;
    __syncthreads();
    sh[t] += y;
    __syncthreads();
  }
  if (t < n) v[t] = sh[t] - x;
  if (t == (int)blockDim.x - 1) *total = sh[t];
}

template <typename TV>
__global__ void __launch_bounds__(kCompactB) compact_scatter(CooDev in, const int64_t *__restrict__ nnz_dev, LutSet ls,
                                                             const int64_t *__restrict__ offs,
                                                             int32_t *const *__restrict__ oidx, TV *__restrict__ ovals) {
  // steps of 4 kCompactB entries, thread t owning the 4 consecutive entries 4t .. 4t + 3 of
  // the step: survivors' offsets from a warp scan of the per-thread counts and a scan of the
  // 32 warp totals (2 barriers per step)
  __shared__ int wsum[33];
  __shared__ int64_t base;
  int64_t b0, b1;
  compact_range(*nnz_dev, b0, b1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = offs[blockIdx.x];
  for (int64_t s0 = b0; s0 < b1; s0 += 4 * kCompactB) {
    const int64_t e0 = s0 + 4 * (int64_t)threadIdx.x;
    bool keep[4];
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      keep[k] = e0 + k < b1 && keep_entry(in, ls, e0 + k);
      cnt += keep[k] ? 1 : 0;
    }
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();  // wsum written; base of this step visible
    if (w == 0) {
      const int x = wsum[lane];
      int xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += y;
      }
      wsum[lane] = xi - x;
      if (lane == 31) wsum[32] = xi;
    }
    __syncthreads();
    int64_t o = base + wsum[w] + inc - cnt;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (keep[k]) {
        const int64_t e = e0 + k;
        for (int m = 0; m < in.d; ++m) {
          const int32_t i = in.idx[m][e];
          oidx[m][o] = ls.lut[m] ? ls.lut[m][i] : i;
        }
        ovals[o] = ((const TV *)in.vals)[e];
        ++o;
      }
    }
    __syncthreads();  // base and wsum consumed
    if (threadIdx.x == 0) base += wsum[32];
  }
}

__global__ void fill_i32(int32_t *p, int64_t n, int32_t v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) p[e] = v;
}

// Debug-checks flag: every index of the COO input in range (status bit on failure).
__global__ void check_indices(const int32_t *__restrict__ idx, int64_t n, int64_t dim, unsigned *__restrict__ status) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    if (idx[e] < 0 || idx[e] >= dim) atomicOr(status, (unsigned)ST_BAD_INDEX);
}

// Rank-order gather of the core nonzeros: rank q's block [q * cap, q * cap + cnt[q]) of the
// allgathered arrays goes to offset sum_{q' < q} cnt[q'].
template <typename TV>
__global__ void gather_core(const int32_t *__restrict__ gidx, const TV *__restrict__ gvals, int d, int nranks,
                            int64_t cap, const int64_t *__restrict__ cnt, int32_t *const *__restrict__ oidx,
                            TV *__restrict__ ovals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)nranks * cap;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(e / cap);
    const int64_t t = e % cap;
    if (t >= cnt[q]) continue;
    int64_t o = t;
    for (int q2 = 0; q2 < q; ++q2) o += cnt[q2];
    for (int k = 0; k < d; ++k) oidx[k][o] = gidx[((int64_t)q * d + k) * cap + t];
    ovals[o] = gvals[(int64_t)q * cap + t];
  }
}

int grid_for(Ctx &c, int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * 8, (n + threads - 1) / threads));
}

// Fixed-point scale of a sketch: max|v| over this rank's values, maximum and nnz over the
// ranks, then S (device-side; no host synchronisation).
void fix_scale(Ctx &c, const void *vals, DT vt, int64_t nnz, FixScale *fs) {
  DevBuf<unsigned long long> mb(c, 1);
  DevBuf<int64_t> nb(c, 1);
  mb.zero();
  if (nnz > 0) {
    const int g = grid_for(c, nnz);
    if (vt == DT::F64) RT_LAUNCH(c, abs_max_kernel<double>, g, 256, 0, (const double *)vals, nnz, mb.p);
    else RT_LAUNCH(c, abs_max_kernel<float>, g, 256, 0, (const float *)vals, nnz, mb.p);
  }
  RT_CUDA(cudaMemcpyAsync(nb.p, &nnz, sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
  allreduce_u64_max(c, mb.p, 1);
  allreduce_i64_sum(c, nb.p, 1);
  RT_LAUNCH(c, fix_scale_kernel, 1, 1, 0, mb.p, nb.p, fs);
}

}  // namespace

// Y (I x ell, fp64) = G_(n) Omega_n over the (live) nonzeros of g, summed over the ranks.
void sketch_coo(Ctx &c, const CooDev &g, int mode, int ell, uint64_t seed, bool normals_f64, double *Y,
                const int64_t *nnz_dev, const void *fs_dev) {
  const int64_t I = g.dims[mode];
  RT_REQUIRE(ell <= kMaxEll, "sparse sketch: l > 64 is not supported");
  const FixScale *fs = (const FixScale *)fs_dev;
  DevBuf<FixScale> own;
  if (!fs) {  // standalone use: scale from this tensor
    own.alloc(c, 1);
    fix_scale(c, g.vals, g.vt, g.nnz, own.p);
    fs = own.p;
  }
  DevBuf<long long> Yf(c, 2 * (size_t)I * ell);  // [H | L]
  Yf.zero();
  static const bool unsorted = RT_EXP_GETENV("RTUCKER_COO_UNSORTED") != nullptr;
  bool key_fits = true;  // Omega column index c < prod_{k != mode} I_k must fit 56 bits of the key
  int64_t others = 1;
  for (int k = 0; k < g.d; ++k) {
    if (k == mode) continue;
    if (others > (int64_t)(kKeyMask / (uint64_t)g.dims[k])) key_fits = false;
    else others *= g.dims[k];
  }
  const int64_t nbk64 = (I + kBR - 1) / kBR;
  if (g.nnz > 0 && !unsorted && nbk64 <= kMaxBk && key_fits && g.nnz < INT32_MAX) {
    const int nbk = (int)nbk64;
    DevBuf<unsigned> cnt(c, (size_t)nbk), bstart(c, (size_t)nbk + 1), cur(c, (size_t)nbk);
    DevBuf<int> istart(c, (size_t)nbk + 3);  // + bucket_sketch's work-unit counter and unit size
    DevBuf<uint64_t> skey(c, (size_t)g.nnz);
    DevBuf<char> sval(c, (size_t)g.nnz * (g.vt == DT::F64 ? 8 : 4));
    cnt.zero();
    // latency-bound streaming passes: 8 CTAs (64 warps) per SM in flight
    const int gs = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * 8, (g.nnz + kBChunk - 1) / kBChunk));
    smem_attr(bucket_hist, sizeof(unsigned) * nbk);
    RT_LAUNCH(c, bucket_hist, gs, kBT, sizeof(unsigned) * nbk, g, nnz_dev, mode, nbk, cnt.p);
    const int gk = c.num_sms * 3;
    RT_LAUNCH(c, bucket_scan, 1, kScanT, 0, cnt.p, nbk, bstart.p, cur.p, istart.p, istart.p + nbk + 1, gk);
    unsigned long long *yh = (unsigned long long *)Yf.p, *yl = yh + (size_t)I * ell;
#define RT_BUCKETED(TV, TN)                                                                                  \
  do {                                                                                                       \
    smem_attr(bucket_scatter<TV>, 2 * sizeof(unsigned) * nbk);                                               \
    RT_LAUNCH(c, bucket_scatter<TV>, gs, kBT, 2 * sizeof(unsigned) * nbk, g, nnz_dev, mode, nbk, cur.p, skey.p,  \
              (TV *)sval.p);                                                                                 \
    smem_attr(bucket_sketch<TV, TN>, kBSmem);                                                                \
    RT_LAUNCH(c, (bucket_sketch<TV, TN>), gk, kBT, kBSmem, skey.p, (const TV *)sval.p, bstart.p, istart.p, nbk, \
              I, mode, ell, seed, fs, istart.p + nbk + 1, yh, yl);                                           \
  } while (0)
    if (g.vt == DT::F64) {
      RT_BUCKETED(double, double);
    } else if (normals_f64) {
      RT_BUCKETED(float, double);
    } else {
      RT_BUCKETED(float, float);
    }
#undef RT_BUCKETED
  } else if (g.nnz > 0) {
    constexpr int kW = kCooT / 32;
    const int hot = (int)std::max<int64_t>(1, std::min<int64_t>(32, (200 * 1024) / (2 * kW * ell * 8)));
    const size_t smem = (size_t)2 * kW * hot * ell * sizeof(long long);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * 4, (g.nnz + 1023) / 1024));
    unsigned long long *yh = (unsigned long long *)Yf.p, *yl = yh + (size_t)I * ell;
#define RT_COO(TV, TN)                                                                                     \
  do {                                                                                                     \
    smem_attr(sketch_coo_kernel<TV, TN>, smem);                                                            \
    RT_LAUNCH(c, (sketch_coo_kernel<TV, TN>), blocks, kCooT, smem, g, nnz_dev, mode, ell, hot, seed, fs, yh, yl); \
  } while (0)
    if (g.vt == DT::F64) {
      RT_COO(double, double);
    } else if (normals_f64) {
      RT_COO(float, double);
    } else {
      RT_COO(float, float);
    }
#undef RT_COO
  }
  allreduce_i64_sum(c, Yf.p, Yf.n);  // exact: integer words
  RT_LAUNCH(c, y_from_fixed_kernel, grid_for(c, I * ell), 256, 0, Yf.p, Yf.p + (size_t)I * ell, I * ell, fs, Y);
}

void srrqr(Ctx &c, const double *Q, int64_t m, int l, double eta, int64_t *sel_dev, double *A, int *swaps_dev) {
  RT_REQUIRE(l >= 1 && l <= kMaxEll && m >= l, "srrqr: need 1 <= l <= 64 and m >= l");
  const size_t smem = sizeof(double) * (3 * (size_t)l * l + l);
  smem_attr(srrqr_coop_kernel, smem);
  int per_sm = 0;
  RT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, srrqr_coop_kernel, kSrT, smem));
  // every resident CTA: a maxvol round recomputes A = Q Q_S^{-1} (m l^2 flops); one CTA per SM
  // (cheaper grid barriers) measured slower on C5's 200000-row mode (0.98 vs 0.59 ms)
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * std::max(per_sm, 1),
                                                               (m + kSrT - 1) / kSrT));
  DevBuf<double> r(c, (size_t)m * l), pv(c, 2 * (size_t)grid);
  DevBuf<int> mark(c, m);
  DevBuf<int64_t> pi(c, 2 * (size_t)grid);
  DevBuf<int> swl;
  if (!swaps_dev) {
    swl.alloc(c, 1);
    swaps_dev = swl.p;
  }
  double *rp = r.p, *pvp = pv.p;
  int *mp = mark.p;
  int64_t *pip = pi.p;
  int ms = 10000;
  unsigned *stp = c.status;
  void *args[] = {(void *)&Q, (void *)&m, (void *)&l, (void *)&eta, (void *)&ms, (void *)&rp, (void *)&mp,
                  (void *)&pvp, (void *)&pip, (void *)&sel_dev, (void *)&A, (void *)&swaps_dev, (void *)&stp};
  RT_CUDA(cudaLaunchCooperativeKernel((const void *)srrqr_coop_kernel, dim3(grid), dim3(kSrT), args, smem, c.stream));
  c.launches++;
}

// Keep the entries whose index is selected in every mode m with sel[m] != null (sorted, length
// l[m]) and renumber those modes; the live input nnz is read from nnz_dev, the new nnz written to
// nnz_out (device).  Order-preserving.
void coo_select_modes(Ctx &c, const CooDev &in, const int64_t *nnz_dev, const int64_t *const *sel, const int *l,
                      int32_t *const *out_idx, void *out_vals, int64_t *nnz_out) {
  LutSet ls{};
  DevBuf<int32_t> lut[kMaxModes];
  for (int m = 0; m < in.d; ++m) {
    if (!sel[m]) continue;
    const int64_t I = in.dims[m];
    lut[m].alloc(c, I);
    RT_LAUNCH(c, fill_i32, grid_for(c, I), 256, 0, lut[m].p, I, -1);
    RT_LAUNCH(c, build_lookup, 1, 256, 0, sel[m], l[m], lut[m].p);
    ls.lut[m] = lut[m].p;
  }
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)c.num_sms * 4, (int64_t)kCompactG,
                                                                 (in.nnz + kCompactB - 1) / kCompactB}));
  DevBuf<int64_t> offs(c, nblk);
  RT_LAUNCH(c, compact_count, nblk, kCompactB, 0, in, nnz_dev, ls, offs.p);
  RT_LAUNCH(c, exclusive_scan_single, 1, kCompactG, 0, offs.p, nblk, nnz_out);
  DevBuf<int32_t *> optr(c, kMaxModes);
  RT_CUDA(cudaMemcpyAsync(optr.p, out_idx, sizeof(int32_t *) * kMaxModes, cudaMemcpyHostToDevice, c.stream));
  if (in.vt == DT::F64)
    RT_LAUNCH(c, compact_scatter<double>, (int)nblk, kCompactB, 0, in, nnz_dev, ls, offs.p, optr.p, (double *)out_vals);
  else
    RT_LAUNCH(c, compact_scatter<float>, (int)nblk, kCompactB, 0, in, nnz_dev, ls, offs.p, optr.p, (float *)out_vals);
}

void coo_select(Ctx &c, const CooDev &in, const int64_t *nnz_dev, int mode, const int64_t *sel, int l,
                int32_t *const *out_idx, void *out_vals, int64_t *nnz_out) {
  const int64_t *sels[kMaxModes] = {nullptr};
  int ls[kMaxModes] = {0};
  sels[mode] = sel;
  ls[mode] = l;
  coo_select_modes(c, in, nnz_dev, sels, ls, out_idx, out_vals, nnz_out);
}

void debug_coo_sketch(Ctx &c, const rtucker_coo_desc *X, int mode, int ell, uint64_t seed, bool normals_f64,
                      double *Y) {
  const int d = X->d;
  const DT vt = X->dtype == RTUCKER_F64 ? DT::F64 : DT::F32;
  const int64_t nnz = X->nnz;
  CooDev g;
  g.d = d;
  g.nnz = nnz;
  g.vt = vt;
  for (int k = 0; k < d; ++k) {
    RT_REQUIRE(X->dims[k] >= 1 && X->dims[k] <= INT32_MAX, "every dim must lie in [1, 2^31)");
    RT_REQUIRE(nnz == 0 || X->idx[k] != nullptr, "null index array");
    g.dims[k] = X->dims[k];
  }
  RT_REQUIRE(nnz == 0 || X->vals != nullptr, "null value array");
  DevBuf<int32_t> ib;
  DevBuf<unsigned char> vb;
  if (X->memory == RTUCKER_HOST && nnz > 0) {
    ib.alloc(c, (size_t)nnz * d);
    vb.alloc(c, (size_t)nnz * dt_size(vt));
    for (int k = 0; k < d; ++k)
      RT_CUDA(cudaMemcpyAsync(ib.p + (size_t)k * nnz, X->idx[k], sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, c.stream));
    RT_CUDA(cudaMemcpyAsync(vb.p, X->vals, dt_size(vt) * nnz, cudaMemcpyHostToDevice, c.stream));
    for (int k = 0; k < d; ++k) g.idx[k] = ib.p + (size_t)k * nnz;
    g.vals = vb.p;
  } else {
    for (int k = 0; k < d; ++k) g.idx[k] = X->idx[k];
    g.vals = X->vals;
  }
  sketch_coo(c, g, mode, ell, seed, vt == DT::F64 || normals_f64, Y, nullptr, nullptr);
}

rtucker_result *run_sparse_sthosvd(Ctx &c, const rtucker_coo_desc *X, const int64_t *ranks, int p, uint64_t seed,
                                   const int32_t *order, double eta, uint32_t flags) {
  RT_REQUIRE(X != nullptr, "null tensor descriptor");
  if (X->d > kMaxModes) throw Error(RTUCKER_EUNSUPPORTED, "d > RTUCKER_MAX_MODES");
  RT_REQUIRE(X->d >= 1, "d must be >= 1");
  RT_REQUIRE(X->nnz >= 0 && X->nnz < INT32_MAX, "nnz must lie in [0, 2^31)");
  RT_REQUIRE(p >= 0, "p must be >= 0");
  RT_REQUIRE(eta >= 1.0, "eta must be >= 1 (P:379)");
  RT_REQUIRE(X->dtype == RTUCKER_F32 || X->dtype == RTUCKER_F64, "dtype must be RTUCKER_F32 or RTUCKER_F64");
  const int d = X->d;
  const DT vt = X->dtype == RTUCKER_F64 ? DT::F64 : DT::F32;
  const size_t vs = dt_size(vt);
  int64_t cur[kMaxModes] = {0};
  for (int k = 0; k < d; ++k) {
    RT_REQUIRE(X->dims[k] >= 1 && X->dims[k] <= INT32_MAX, "every dim must lie in [1, 2^31)");
    RT_REQUIRE(ranks[k] >= 1, "r_n must be >= 1");
    cur[k] = X->dims[k];
  }
  const bool hosvd = flags & RTUCKER_SP_HOSVD;  // SP-HOSVD: modes on X, one final filter
  int32_t ord[kMaxModes];
  check_order(hosvd ? nullptr : order, d, ord, cur, false);
  if (hosvd)
    for (int k = 0; k < d; ++k) ord[k] = k;
  const bool nf64 = vt == DT::F64 || (flags & RTUCKER_ACCUM_MASK) == RTUCKER_ACCUM_FP64;
  const bool dbg = flags & RTUCKER_DEBUG_CHECKS;
  ResultGuard rg{c, new_result(d)};
  rtucker_result *res = rg.r;
  res->dtype = X->dtype;
  for (int k = 0; k < d; ++k) {
    res->dims[k] = X->dims[k];
    res->order[k] = ord[k];
  }
  res->seed = seed;
  res->flags = flags;
  // working COO (ping-pong), device resident; nnz and its history live on the device
  const int64_t nnz0 = X->nnz;
  DevBuf<int32_t> ib[2];
  DevBuf<unsigned char> vb[2];
  for (int b = 0; b < 2; ++b) {
    ib[b].alloc(c, (size_t)std::max<int64_t>(nnz0, 1) * d);
    vb[b].alloc(c, (size_t)std::max<int64_t>(nnz0, 1) * vs);
  }
  const cudaMemcpyKind kind = X->memory == RTUCKER_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  for (int k = 0; k < d; ++k) {
    RT_REQUIRE(nnz0 == 0 || X->idx[k] != nullptr, "null index array");
    if (nnz0) RT_CUDA(cudaMemcpyAsync(ib[0].p + (size_t)k * nnz0, X->idx[k], sizeof(int32_t) * nnz0, kind, c.stream));
    if (dbg && nnz0)
      RT_LAUNCH(c, check_indices, grid_for(c, nnz0), 256, 0, ib[0].p + (size_t)k * nnz0, nnz0, cur[k], c.status);
  }
  RT_REQUIRE(nnz0 == 0 || X->vals != nullptr, "null value array");
  if (nnz0) RT_CUDA(cudaMemcpyAsync(vb[0].p, X->vals, vs * nnz0, kind, c.stream));
  if (dbg) check_status(c);
  DevBuf<int64_t> hist(c, kMaxModes + 1);  // nnz after each mode (device)
  DevBuf<int> swaps(c, kMaxModes);
  swaps.zero();
  RT_CUDA(cudaMemcpyAsync(hist.p, &nnz0, sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
  DevBuf<FixScale> fs(c, 1);
  fix_scale(c, vb[0].p, vt, nnz0, fs.p);  // max|v| bounds every later (filtered) mode too
  int cb = 0;
  for (int jj = 0; jj < d; ++jj) {
    const int n = ord[jj];
    int64_t others = 1;
    for (int k = 0; k < d; ++k)
      if (k != n) others *= cur[k];
    const int64_t ell64 = ranks[n] + p;
    RT_REQUIRE(ell64 < std::min<int64_t>(cur[n], others), "SP-STHOSVD needs r_n + p < min(I_n, prod_{k!=n} I_k) (P:372)");
    const int ell = (int)ell64;
    CooDev g;
    g.d = d;
    for (int k = 0; k < d; ++k) {
      g.dims[k] = cur[k];
      g.idx[k] = ib[cb].p + (size_t)k * nnz0;
    }
    g.nnz = nnz0;  // upper bound; the live count is hist[jj]
    g.vals = vb[cb].p;
    g.vt = vt;
    const int64_t I = cur[n];
    DevBuf<double> Y(c, (size_t)I * ell), Q(c, (size_t)I * ell);
    {
      PhaseScope ps(c, PH_SKETCH, jj);
      sketch_coo(c, g, n, ell, seed, nf64, Y.p, hist.p + (hosvd ? 0 : jj), fs.p);
      ps.next(PH_QR);
      thin_qr(c, Y.p, I, ell, Q.p);
    }
    double *A = (double *)dev_alloc(c, sizeof(double) * I * ell);
    res->factors[n] = A;
    int64_t *S = (int64_t *)dev_alloc(c, sizeof(int64_t) * ell);
    res->selection[n] = S;
    {
      PhaseScope ps(c, PH_EIG, jj);
      srrqr(c, Q.p, I, ell, eta, S, A, swaps.p + n);
    }
    res->ranks[n] = ell;
    res->ell[n] = ell;
    if (hosvd) continue;  // X itself is sketched for every mode; filtered once below
    // G_(n) <- P^T G_(n): keep the selected slices and renumber them 0..ell-1 (local nonzeros)
    int32_t *oidx[kMaxModes] = {nullptr};
    for (int k = 0; k < d; ++k) oidx[k] = ib[1 - cb].p + (size_t)k * nnz0;
    {
      PhaseScope ps(c, PH_SHRINK, jj);
      coo_select(c, g, hist.p + jj, n, S, ell, oidx, vb[1 - cb].p, hist.p + jj + 1);
    }
    cb = 1 - cb;
    cur[n] = ell;
  }
  if (hosvd) {  // core = X x_1 P_1^T ... x_d P_d^T: keep entries selected in every mode
    PhaseScope ps(c, PH_SHRINK, 0);
    CooDev g;
    g.d = d;
    for (int k = 0; k < d; ++k) {
      g.dims[k] = X->dims[k];
      g.idx[k] = ib[0].p + (size_t)k * nnz0;
    }
    g.nnz = nnz0;
    g.vals = vb[0].p;
    g.vt = vt;
    const int64_t *sels[kMaxModes] = {nullptr};
    int ls[kMaxModes] = {0};
    int32_t *oidx[kMaxModes] = {nullptr};
    for (int k = 0; k < d; ++k) {
      sels[k] = res->selection[k];
      ls[k] = (int)res->ranks[k];
      oidx[k] = ib[1].p + (size_t)k * nnz0;
      cur[k] = res->ranks[k];
    }
    coo_select_modes(c, g, hist.p, sels, ls, oidx, vb[1].p, hist.p + 1);
    for (int k = 2; k <= d; ++k)
      RT_CUDA(cudaMemcpyAsync(hist.p + k, hist.p + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, c.stream));
    cb = 1;
  }
  // ---- one host synchronisation: nnz history (summed over the ranks), swaps, status
  DevBuf<int64_t> hsum(c, kMaxModes + 1);
  RT_CUDA(cudaMemcpyAsync(hsum.p, hist.p, sizeof(int64_t) * (d + 1), cudaMemcpyDeviceToDevice, c.stream));
  allreduce_i64_sum(c, hsum.p, d + 1);
  std::vector<int64_t> hh(2 * (d + 1));
  int hsw[kMaxModes];
  RT_CUDA(cudaMemcpyAsync(hh.data(), hsum.p, sizeof(int64_t) * (d + 1), cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaMemcpyAsync(hh.data() + d + 1, hist.p, sizeof(int64_t) * (d + 1), cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaMemcpyAsync(hsw, swaps.p, sizeof(int) * d, cudaMemcpyDeviceToHost, c.stream));
  check_status(c);  // synchronises; ENUMERIC on a singular P^T Q
  for (int k = 0; k <= d; ++k) res->nnz_history[k] = hh[k];
  for (int k = 0; k < d; ++k) res->swaps[k] = hsw[k];
  const int64_t nnz_local = hh[d + 1 + d], nnz = hh[d];
  res->core_nnz = nnz;
  for (int k = 0; k < d; ++k) res->core_idx[k] = (int32_t *)dev_alloc(c, sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  res->core_vals = dev_alloc(c, vs * std::max<int64_t>(nnz, 1));
  if (c.nranks == 1) {
    for (int k = 0; k < d; ++k)
      if (nnz)
        RT_CUDA(cudaMemcpyAsync(res->core_idx[k], ib[cb].p + (size_t)k * nnz0, sizeof(int32_t) * nnz,
                                cudaMemcpyDeviceToDevice, c.stream));
    if (nnz) RT_CUDA(cudaMemcpyAsync(res->core_vals, vb[cb].p, vs * nnz, cudaMemcpyDeviceToDevice, c.stream));
  } else {
    // gather the core nonzeros of all ranks in rank order (padded blocks of cap entries)
    DevBuf<int64_t> cnt(c, 1), cnts(c, c.nranks), capd(c, 1);
    RT_CUDA(cudaMemcpyAsync(cnt.p, hist.p + d, sizeof(int64_t), cudaMemcpyDeviceToDevice, c.stream));
    allgather_i64(c, cnt.p, cnts.p, 1);
    std::vector<int64_t> hc(c.nranks);
    RT_CUDA(cudaMemcpyAsync(hc.data(), cnts.p, sizeof(int64_t) * c.nranks, cudaMemcpyDeviceToHost, c.stream));
    RT_CUDA(cudaStreamSynchronize(c.stream));
    int64_t cap = 1;
    for (int64_t v : hc) cap = std::max(cap, v);
    DevBuf<int32_t> sidx(c, (size_t)d * cap), gidx(c, (size_t)c.nranks * d * cap);
    DevBuf<unsigned char> sval(c, (size_t)cap * vs), gval(c, (size_t)c.nranks * cap * vs);
    for (int k = 0; k < d; ++k)
      if (nnz_local)
        RT_CUDA(cudaMemcpyAsync(sidx.p + (size_t)k * cap, ib[cb].p + (size_t)k * nnz0, sizeof(int32_t) * nnz_local,
                                cudaMemcpyDeviceToDevice, c.stream));
    if (nnz_local) RT_CUDA(cudaMemcpyAsync(sval.p, vb[cb].p, vs * nnz_local, cudaMemcpyDeviceToDevice, c.stream));
    allgather_bytes(c, sidx.p, gidx.p, sizeof(int32_t) * d * cap);
    allgather_bytes(c, sval.p, gval.p, vs * cap);
    DevBuf<int32_t *> optr(c, kMaxModes);
    RT_CUDA(cudaMemcpyAsync(optr.p, res->core_idx, sizeof(int32_t *) * kMaxModes, cudaMemcpyHostToDevice, c.stream));
    const int g = grid_for(c, (int64_t)c.nranks * cap);
    if (vt == DT::F64)
      RT_LAUNCH(c, gather_core<double>, g, 256, 0, gidx.p, (const double *)gval.p, d, c.nranks, cap, cnts.p, optr.p,
                (double *)res->core_vals);
    else
      RT_LAUNCH(c, gather_core<float>, g, 256, 0, gidx.p, (const float *)gval.p, d, c.nranks, cap, cnts.p, optr.p,
                (float *)res->core_vals);
  }
  finish_result(c, res, flags);
  RT_CUDA(cudaStreamSynchronize(c.stream));
  return rg.release();
}

}  // namespace rt
