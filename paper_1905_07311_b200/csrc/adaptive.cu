// Adaptive randomized Tucker: Alg 5 adaptive R-STHOSVD and, with
// RTUCKER_ADAPT_HOSVD, Alg 4 adaptive R-HOSVD.  The range finder
// AdaptRangeFinder is cited, not given, by the paper; this follows DESIGN
// reading R8, block by block:
//   E = ||G||^2;  k = 0
//   loop: stop if E <= tau^2 or k >= cap;  bb = min(b, cap - k)
//         W = G_(n) Omega(:, k:k+bb)            (sketch kernel, global column index k)
//         W <- (I - Q Q^T) W, twice              (fp64 tensor-core GEMMs)
//         stop ("floor") if ||W|| <= floor ||X|| (block discarded)
//         Q_i = qr(W);  B_i = Q_i^T G_(n) (+ Gram);  E -= ||B_i||^2;  k += bb
//   truncation (default): eigenpairs of B B^T, r = min{r : ||G||^2 - sum_{i<=r} s_i^2 <= tau^2},
//   A = Q U(:, 1:r) (signs per R4b), G <- U(:, 1:r)^T B.  ADAPT_NO_TRUNCATE keeps A = Q, G = B.
// tau_n = eps_n ||X||_F with eps_n = eps / sqrt(d) or the caller's mode_tol.
//
// Host synchronisation: ONE per block.  The floor test and the residual update are decided
// together after B_i: Q_i and B_i are formed speculatively and dropped when the projected
// block was below the floor (the only wasted pass is the final one of a floored mode).  The
// Ozaki B-pass's column maxima are computed once per mode (G does not change inside a mode).
//
// Multi-GPU: the dense input is sharded along its last mode, which is processed
// last.  Modes n < d: the block sketch W and ||B_i||^2 are allreduced (W is I_n x b), QR and the
// projections run redundantly, B stays sharded, the truncation Gram is allreduced and the
// shrink is local.  Mode d: W's rows are local and complete (placed and summed like the
// fixed-rank path), B_i = Q_i^T G_(d) sums over the sharded index and is allreduced
// (b x prod_{k<d} r_k per block: the known bandwidth limit of SURVEY §8(e)), and the core
// ends up replicated.
#include <cmath>
#include <cstring>
#include <vector>

#include "comm.h"
#include "kernels_extra.h"
#include "orchestrate.h"
#include "philox.cuh"

namespace rt {

namespace {

__global__ void trace_kernel(const double *__restrict__ A, int n, int64_t lda, double *__restrict__ out) {
  __shared__ double s[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += A[i + lda * i];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    *out = t;
  }
}

// W (m x b) -= Q (m x k) T (k x b), column-major, one thread per output element.
__global__ void sub_gemm_kernel(double *__restrict__ W, int64_t m, int b, const double *__restrict__ Q, int k,
                                const double *__restrict__ T) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * b; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    double s = 0.0;
    for (int t = 0; t < k; ++t) s += Q[i + m * t] * T[t + (int64_t)k * j];
    W[e] -= s;
  }
}

// Skinny projection W <- W - Q (Q^T W) of one block (m x b, b <= 16) against the basis so far
// (Q: m x k), fp64, fixed summation order (deterministic).  The tensor-core GEMM tiles of
// 64 x 64 left these k x b / m x b products at 12-25 CTAs and ~68 us each (4 per block, 59 ms
// of the C4 adaptive call); here:
//   proj_t_kernel:   T = Q^T W, one warp per row j of T (lanes stride the m rows, b running
//                    sums each, fixed-order warp tree); W staged once per CTA in shared memory;
//   proj_sub_kernel: W -= Q T, one CTA per 32 rows, its 8 warps split the k columns of Q, and
//                    the 8 partial sums are added in warp order through shared memory.
constexpr int kProjB = 16;
__global__ void __launch_bounds__(256) proj_t_kernel(const double *__restrict__ Q, int64_t m, int k,
                                                     const double *__restrict__ W, int b, double *__restrict__ T) {
  extern __shared__ double wsm[];  // m x b (column-major, ld m)
  for (int64_t e = threadIdx.x; e < m * b; e += blockDim.x) wsm[e] = W[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= k) return;
  double acc[kProjB];
#pragma unroll
  for (int c = 0; c < kProjB; ++c) acc[c] = 0.0;
  const double *qj = Q + m * j;
  for (int64_t i = lane; i < m; i += 32) {
    const double q = qj[i];
#pragma unroll
    for (int c = 0; c < kProjB; ++c)
      if (c < b) acc[c] = fma(q, wsm[i + m * c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < kProjB; ++c) {
    double v = acc[c];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && c < b) T[j + (int64_t)k * c] = v;
  }
}

__global__ void __launch_bounds__(256) proj_sub_kernel(double *__restrict__ W, int64_t m, int b,
                                                       const double *__restrict__ Q, int k,
                                                       const double *__restrict__ T) {
  __shared__ double part[8][32][kProjB + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  const int per = (k + 7) / 8, j0 = warp * per, j1 = min(k, j0 + per);
  double acc[kProjB];
#pragma unroll
  for (int c = 0; c < kProjB; ++c) acc[c] = 0.0;
  if (i < m)
    for (int j = j0; j < j1; ++j) {
      const double q = Q[i + m * j];
#pragma unroll
      for (int c = 0; c < kProjB; ++c)
        if (c < b) acc[c] = fma(q, T[j + (int64_t)k * c], acc[c]);
    }
#pragma unroll
  for (int c = 0; c < kProjB; ++c) part[warp][lane][c] = acc[c];
  __syncthreads();
  if (warp == 0 && i < m) {
    for (int c = 0; c < b; ++c) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += part[w][lane][c];
      W[i + m * c] -= s;
    }
  }
}

void project_out(Ctx &c, const double *Q, int64_t m, int k, double *W, int b, double *T) {
  const size_t sm = sizeof(double) * (size_t)m * b;
  if (b > kProjB || sm > 200 * 1024) {  // outside the skinny kernels' envelope: the GEMMs
    gemm_f64(c, true, Q, m, W, m, T, k, k, b, m);
    gemm_f64(c, false, Q, m, T, k, W, m, m, b, k, 1.0, -1.0);
    return;
  }
  if (sm > 48 * 1024) smem_attr(proj_t_kernel, sm);
  RT_LAUNCH(c, proj_t_kernel, (k + 7) / 8, 256, sm, Q, m, k, (const double *)W, b, T);
  RT_LAUNCH(c, proj_sub_kernel, (int)((m + 31) / 32), 256, 0, W, m, b, Q, k, (const double *)T);
}

// ---------------------------------------------------------------------------------------
// Fused block pass for fp64 cores (SURVEY §3.3 "B_i + next sketch"): ONE read of G_(n) gives
//   B_i     = Q_i^T G_(n)                      (b x P, stored (L, b, R)) and its Gram, and
//   W_{i+1} = G_(n) Omega(:, k1 : k1 + b1)     (I x b1, the next block's sketch)
// where the next sketch is formed before the stop test of block i decides whether it is needed
// (a wasted product on the last block of a mode).  G is (L, I, R), column p = l + L r; a tile is
// 32 consecutive l of one r, streamed in chunks of 32 rows i through a cp.async ring.  Per chunk
// (fp64 tensor cores, m8n8k4, one 8 x 8 output tile per warp and product):
//   B tile (16 j x 32 l) += Q_c^T (16 x 32 i) G_c (32 i x 32 l)    accumulated over the tile
//   W rows (32 i x 16 j') += G_c (32 i x 32 l) Omega_t (32 l x 16 j') into shared W (I x 16)
// Omega_t is generated per tile by the sketch's Philox stream (same counter layout as
// sketch_dfma_kernel).  Per-CTA W and Gram partials are summed in a fixed order afterwards.
constexpr int kFT = 256;              // threads
constexpr int kFS = 5;                // ring stages
constexpr int kFL = 64;               // columns l per tile
constexpr int kFG = kFL + 4;          // G chunk row stride (doubles, = 4 mod 16: conflict-free fragments)
constexpr int kFQ = 20;               // Q chunk / Omega row stride (= 4 mod 16)
constexpr int kFStage = 32 * kFG + 32 * kFQ;  // doubles per stage (G chunk + Q chunk)
__host__ __device__ constexpr int fused_ys(int bb1) { return bb1 <= 12 ? 12 : 16; }  // W row stride
__host__ __device__ constexpr size_t fused_smem(int64_t I, int ys) {
  return sizeof(double) * ((size_t)kFS * kFStage + kFL * kFQ + 16 * (kFL + 1) + (size_t)I * ys);
}

__device__ __forceinline__ void cp_async8(unsigned d, const double *src, bool ok) {
  const int n = ok ? 8 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(ok ? src : nullptr), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async16(unsigned d, const double *src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(bytes ? src : nullptr), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <typename TN, bool V16>
__global__ void __launch_bounds__(kFT, 1) adapt_fused_kernel(const double *__restrict__ G, int64_t L, int64_t I, int64_t R,
                                                           const double *__restrict__ Q, int bb, uint64_t seed, int mode,
                                                           int64_t k1, int bb1, int64_t col_offset, int ys,
                                                           double *__restrict__ Bi, double *__restrict__ ypart,
                                                           double *__restrict__ gpart) {
  extern __shared__ __align__(16) double fsm[];
  double *ring = fsm;                        // kFS x (G chunk [32][kFG], Q chunk [32][kFQ])
  double *Om = ring + kFS * kFStage;         // [kFL l][kFQ]
  double *Bs = Om + kFL * kFQ;               // [16 j][kFL + 1]
  double *Ys = Bs + 16 * (kFL + 1);          // [I][ys]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fa = lane & 3, fb = lane >> 2;
  const int64_t ntl = (L + kFL - 1) / kFL, ntiles = ntl * R, nch = (I + 31) / 32;
  for (int64_t e = tid; e < I * ys; e += kFT) Ys[e] = 0.0;
  // this CTA's tiles: blockIdx.x + t gridDim.x; steps = tiles x chunks.  Tile and chunk of the
  // consumed and of the issued step advance incrementally (no 64-bit divisions per step).
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t nsteps = my_tiles * nch;
  struct Cursor {
    int64_t t, r, l0, ch;
  };
  auto set_tile = [&](Cursor &cu, int64_t t) {
    cu.t = t;
    cu.r = t / ntl;
    cu.l0 = (t - cu.r * ntl) * kFL;
    cu.ch = 0;
  };
  auto advance = [&](Cursor &cu) {
    if (++cu.ch == nch) set_tile(cu, cu.t + gridDim.x);
  };
  // G chunk copies: V16 (L even, G 16-byte aligned): pairs of l per 16-byte cp.async, else 8-byte
  constexpr int kGW = V16 ? 2 : 1;                 // doubles per copy
  constexpr int kGQ = 32 * kFL / (kFT * kGW);      // copies per thread and chunk
  int64_t goff[kGQ];
  int gll[kGQ], gii[kGQ];
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
#pragma unroll
  for (int q = 0; q < kGQ; ++q) {
    const int e = (tid + kFT * q) * kGW;
    gii[q] = e / kFL;
    gll[q] = e % kFL;
    goff[q] = gll[q] + L * gii[q];
  }
  const int qii0 = tid >> 4, qj = tid & 15;  // Q chunk elements (qii0, qj) and (qii0 + 16, qj)
  Cursor ic;  // issue cursor
  set_tile(ic, blockIdx.x);
  int64_t is = 0;
  auto issue = [&]() {
    if (is < nsteps) {
      const int64_t i0 = ic.ch * 32;
      const unsigned st = ring_s + (unsigned)((is % kFS) * kFStage * sizeof(double));
      const double *gb = G + ic.l0 + L * (i0 + I * ic.r);
      const int64_t lrem = L - ic.l0, irem = I - i0;
#pragma unroll
      for (int q = 0; q < kGQ; ++q) {  // G chunk: 32 rows i x kFL l, coalesced along l
        const unsigned d = st + (unsigned)((gii[q] * kFG + gll[q]) * sizeof(double));
        if constexpr (V16) {
          const int nv = gii[q] < irem ? (int)min((int64_t)2, max((int64_t)0, lrem - gll[q])) : 0;
          cp_async16(d, gb + goff[q], 8 * nv);
        } else {
          cp_async8(d, gb + goff[q], gii[q] < irem && gll[q] < lrem);
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {  // Q chunk: 32 rows i x 16 j
        const int ii = qii0 + 16 * q;
        const bool ok = (ii < irem) && (qj < bb);
        cp_async8(st + (unsigned)((32 * kFG + ii * kFQ + qj) * sizeof(double)), Q + (i0 + ii) + I * qj, ok);
      }
      advance(ic);
    }
    ++is;
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < kFS - 1; ++s) issue();
  // Work split (every G element is read from shared memory once per product):
  //   B: warp w takes rows 4w .. 4w + 3 of the chunk (one k-step) for all 64 l and both j
  //      blocks; the 8 partial B tiles are summed in warp order at the tile's end
  //   W: warp w takes the 8-row block (w & 3) and the l half (w >> 2) for both j' blocks; the
  //      second half adds its partial after the next barrier (other rows: no conflict), Omega's
  //      fragments stay in registers for the whole tile
  double bacc[2][8][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int u = 0; u < 8; ++u) bacc[m][u][0] = bacc[m][u][1] = 0.0;
  double gacc = 0.0;                          // Gram entry (tid >> 4, tid & 15)
  const int ymt = warp & 3, yh = warp >> 2;   // W: row block, l half
  double omr[8][2];                           // Omega fragments of this warp's l half
  double ypend[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  int64_t ypend_i = -1;
  auto add_y = [&](int64_t i, const double (&y)[2][2]) {
    if (i < 0 || i >= I) return;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int jc = 8 * nt + 2 * fa;
      if (jc < bb1) Ys[i * ys + jc] += y[nt][0];
      if (jc + 1 < bb1) Ys[i * ys + jc + 1] += y[nt][1];
    }
  };
  Cursor cc;  // consume cursor
  set_tile(cc, blockIdx.x);
  for (int64_t s = 0; s < nsteps; ++s, advance(cc)) {
    const int64_t r = cc.r, l0 = cc.l0, ch = cc.ch, i0 = ch * 32;
    asm volatile("cp.async.wait_group %0;" ::"n"(kFS - 2) : "memory");
    __syncthreads();     // chunk s visible to all; every warp is past step s - 1
    issue();             // into the stage consumed at step s - 1
    if (yh == 1) {       // the second l half's partial of step s - 1 (rows differ from step s's: nch >= 2)
      add_y(ypend_i, ypend);
      ypend_i = -1;
    }
    if (ch == 0 && bb1 > 0) {  // Omega rows of this tile: p = l0 + ll + L r, columns k1 .. k1 + bb1
      const int64_t jb0 = k1 >> 2;
      const int nb = (int)(((k1 + bb1 - 1) >> 2) - jb0 + 1);
      for (int e = tid; e < kFL * nb; e += kFT) {
        const int ll = e / nb, jb = e % nb;
        const bool lok = l0 + ll < L;
        const uint64_t p = (uint64_t)(l0 + ll + L * r + col_offset);
        const uint4 w = omega_words(seed, mode, 0, p, (uint32_t)(jb0 + jb));
        Normal4<TN> z(w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t kk = 4 * (jb0 + jb) + q - k1;
          if (kk >= 0 && kk < bb1) Om[ll * kFQ + kk] = lok ? (double)z.v[q] : 0.0;
        }
      }
      for (int e = tid; e < kFL * 16; e += kFT)  // unused columns stay zero (disjoint entries)
        if ((e & 15) >= bb1) Om[(e >> 4) * kFQ + (e & 15)] = 0.0;
      __syncthreads();
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) omr[ks][nt] = Om[(4 * (8 * yh + ks) + fa) * kFQ + 8 * nt + fb];
    }
    const double *Gc = ring + (s % kFS) * kFStage, *Qc = Gc + 32 * kFG;
    {  // B partial += Q_c(rows 4w..)^T G_c(rows 4w.., all l)
      const double a0 = Qc[(4 * warp + fa) * kFQ + fb], a1 = Qc[(4 * warp + fa) * kFQ + 8 + fb];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double b = Gc[(4 * warp + fa) * kFG + 8 * u + fb];
        dmma(bacc[0][u][0], bacc[0][u][1], a0, b);
        dmma(bacc[1][u][0], bacc[1][u][1], a1, b);
      }
    }
    if (bb1 > 0) {  // W rows (8 ymt ..) += G_c(rows, l half) Omega(l half, :)
      double y[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const double a = Gc[(8 * ymt + fb) * kFG + 4 * (8 * yh + ks) + fa];
        dmma(y[0][0], y[0][1], a, omr[ks][0]);
        dmma(y[1][0], y[1][1], a, omr[ks][1]);
      }
      const int64_t i = i0 + 8 * ymt + fb;
      if (yh == 0) {
        add_y(i, y);
      } else {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) { ypend[nt][0] = y[nt][0]; ypend[nt][1] = y[nt][1]; }
        ypend_i = i;
      }
    }
    if (ch == nch - 1) {  // tile complete: sum the warps' B partials, store B_i, its Gram
      const int LB = kFL + 1;
      for (int w = 0; w < kFT / 32; ++w) {
        if (warp == w) {
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                double &d = Bs[(8 * m + fb) * LB + 8 * u + 2 * fa + h];
                d = (w == 0 ? 0.0 : d) + bacc[m][u][h];
                bacc[m][u][h] = 0.0;
              }
        }
        __syncthreads();
      }
      for (int e = tid; e < 16 * kFL; e += kFT) {
        const int j = e / kFL, ll = e % kFL;
        if (j < bb && l0 + ll < L) Bi[(l0 + ll) + L * (j + (int64_t)bb * r)] = Bs[j * LB + ll];
      }
      const int gj = tid >> 4, gk = tid & 15;
      double sacc = 0.0;
#pragma unroll 8
      for (int ll = 0; ll < kFL; ++ll) sacc = fma(Bs[gj * LB + ll], Bs[gk * LB + ll], sacc);
      gacc += sacc;
      // Bs is rewritten at the next tile's end, >= 1 barrier later
    }
  }
  __syncthreads();
  if (yh == 1) add_y(ypend_i, ypend);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  double *yp = ypart + (int64_t)blockIdx.x * I * ys;
  for (int64_t e = tid; e < I * ys; e += kFT) yp[e] = Ys[e];
  gpart[(int64_t)blockIdx.x * 256 + tid] = gacc;
}

// W (I x b1, column-major) and gram (bb x bb) from the per-CTA partials, summed in CTA order
__global__ void fused_reduce_kernel(const double *__restrict__ ypart, const double *__restrict__ gpart, int nblk,
                                    int64_t I, int bb1, int bb, int ys, double *__restrict__ W, double *__restrict__ gram) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < I * bb1) {
    const int64_t i = e % I;
    const int j = (int)(e / I);
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += ypart[((int64_t)b * I + i) * ys + j];
    W[e] = s;
  } else if (e < I * bb1 + bb * bb) {
    const int f = (int)(e - I * bb1), j = f % bb, k = f / bb;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += gpart[(int64_t)b * 256 + j * 16 + k];
    gram[f] = s;
  }
}

bool fused_ok(const ModeView &v, int bb) {
  static const bool off = RT_EXP_GETENV("RTUCKER_ADAPT_UNFUSED") != nullptr;
  return !off && v.L >= 32 && v.I > 32 && bb <= 16 && fused_smem(v.I, fused_ys(bb)) <= 225 * 1024;
}

// B_i (and its Gram) and, when bb1 > 0, the next block's sketch W1 in one pass over G (fp64)
void fused_block(Ctx &c, const double *G, const ModeView &v, int n, const double *Qi, int bb, uint64_t seed,
                 int64_t k1, int bb1, int64_t col_offset, bool normals_f32, double *Bi, double *gram, double *W1) {
  const int grid = c.num_sms;
  const int ys = fused_ys(bb1);
  const size_t smem = fused_smem(v.I, ys);
  DevBuf<double> yp(c, (size_t)grid * v.I * ys), gp(c, (size_t)grid * 256);
  const bool v16 = (v.L % 2 == 0) && ((uintptr_t)G % 16 == 0);
#define RT_FUSED(TN, V)                                                                                     \
  do {                                                                                                      \
    smem_attr(adapt_fused_kernel<TN, V>, smem);                                                             \
    RT_LAUNCH(c, (adapt_fused_kernel<TN, V>), grid, kFT, smem, G, v.L, v.I, v.R, Qi, bb, seed, n, k1, bb1,  \
              col_offset, ys, Bi, yp.p, gp.p);                                                              \
  } while (0)
  if (normals_f32) {
    if (v16) RT_FUSED(float, true); else RT_FUSED(float, false);
  } else {
    if (v16) RT_FUSED(double, true); else RT_FUSED(double, false);
  }
#undef RT_FUSED
  const int64_t tot = v.I * bb1 + (int64_t)bb * bb;
  RT_LAUNCH(c, fused_reduce_kernel, ceil_div(tot, 256), 256, 0, yp.p, gp.p, grid, v.I, bb1, bb, ys, W1, gram);
}

struct ModeOut {
  double *A = nullptr;  // I x r (owned by the result)
  int r = 0;            // realised rank
  int k = 0;            // columns drawn
  DevBuf<unsigned char> G;  // new core (L, r, R) in dtype `gt` (unless uncompressed)
  DT gt = DT::F64;
  bool replaced = false;
  bool rows_replicated = false;  // mode d of a sharded input: the new core is replicated
};

// scal[slot] = trace(gram) (||B_i||^2), slot+1 = ||W||^2 (from W), fetched together
__global__ void block_stats_kernel(const double *__restrict__ gram, int bb, const double *__restrict__ W,
                                   int64_t nw, double *__restrict__ out) {
  __shared__ double s[32];
  double v = 0.0, t = 0.0;
  for (int i = threadIdx.x; i < bb; i += blockDim.x) t += gram[i + (int64_t)bb * i];
  for (int64_t e = threadIdx.x; e < nw; e += blockDim.x) v = fma(W[e], W[e], v);
  for (int o = 16; o; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s[threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double w = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) w += s[k];
    out[0] = t;
    out[1] = w;
  }
}

template <typename T>
T fetch(Ctx &c, const T *dev) {
  T h;
  RT_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  return h;
}

struct Shard {
  bool on = false;        // input sharded along the last mode
  bool rows = false;      // this mode is the sharded last mode (local rows of G_(n))
  int64_t col_offset = 0; // global unfolding-column offset of the local slab (modes n < d)
  int64_t row_offset = 0; // shard offset along the last mode (rows of Q for mode d)
  int64_t I_glob = 0;     // global I_n
  bool rel_acc = false;   // fp64 data: relative-accuracy eigensolver (gram_eig)
};

// AdaptRangeFinder on the mode-n unfolding of G (local dims cur, global dims gcur), threshold
// tau2 = tau^2.
ModeOut adapt_mode(Ctx &c, const void *G, DT gt, const int64_t *cur, const int64_t *gcur, int d, int n, double tau2,
                   int block, uint64_t seed, double floor_abs, bool mul_f64, DT store, bool truncate, bool want_core,
                   double *gnorm2_dev, bool fp32_data, const Shard &sh) {
  const ModeView v = mode_view(cur, d, n);
  const int64_t I = gcur[n];  // global rows of W and Q
  ModeOut out;
  // ||G||^2 (fp64), summed over the ranks
  sumsq(c, G, gt, v.L * v.I * v.R, gnorm2_dev);
  if (sh.on) allreduce_sum_f64(c, gnorm2_dev, 1);
  const double gn2 = fetch(c, gnorm2_dev);
  if (!std::isfinite(gn2)) throw Error(RTUCKER_ENUMERIC, "adaptive: non-finite norm");
  int64_t others = 1;
  for (int k2 = 0; k2 < d; ++k2)
    if (k2 != n) others *= gcur[k2];
  const int cap = (int)std::min<int64_t>(I, others);  // column cap on the global dims (reading R8)
  // Ozaki column maxima of the fp32 input: once per mode (G is fixed inside the mode)
  DevBuf<uint32_t> colmax;
  if (gt == DT::F32 && !mul_f64 && store == DT::F64 && v.L == 1 && !sh.rows && ozaki_bpass_enabled()) {
    colmax.alloc(c, (size_t)v.R);
    column_maxima(c, (const float *)G, v, colmax.p);
  }
  DevBuf<double> Q(c, (size_t)I * cap);
  DevBuf<unsigned char> Bfull(c, (size_t)v.L * cap * v.R * dt_size(store));
  DevBuf<double> scal(c, 4), T(c, (size_t)cap * block);
  double E = gn2;
  int k = 0;
  // fp64 cores: B_i and the next block's sketch in one pass over G (fused_block)
  const bool fused = gt == DT::F64 && store == DT::F64 && !sh.rows && fused_ok(v, block);
  DevBuf<double> Wn;  // next block's sketch from the fused pass (local partial when sharded)
  int wn_cols = 0;
  while (true) {
    if (E <= tau2 || k >= cap) break;
    const int bb = std::min(block, cap - k);
    DevBuf<double> W(c, (size_t)I * bb + 1);
    {
      PhaseScope ps(c, PH_SKETCH, n);
      if (wn_cols == bb) {  // formed by the previous block's fused pass
        std::swap(W, Wn);
        wn_cols = 0;
        if (sh.on) allreduce_sum_f64(c, W.p, (size_t)I * bb);
      } else if (!sh.rows) {
        sketch_dense(c, G, gt, v, n, bb, k, seed, sh.col_offset, mul_f64, W.p, nullptr, fp32_data);
        if (sh.on) allreduce_sum_f64(c, W.p, (size_t)I * bb);
      } else {
        DevBuf<double> wl(c, (size_t)v.I * bb), cov(c, (size_t)I * (bb + 1));
        cov.zero();
        sketch_dense(c, G, gt, v, n, bb, k, seed, 0, mul_f64, wl.p, nullptr, fp32_data);
        place_rows(c, wl.p, v.I, bb, sh.row_offset, I, cov.p, cov.p + (size_t)I * bb);
        allreduce_sum_f64(c, cov.p, cov.n);
        check_cover(c, cov.p + (size_t)I * bb, I);
        RT_CUDA(cudaMemcpyAsync(W.p, cov.p, sizeof(double) * I * bb, cudaMemcpyDeviceToDevice, c.stream));
      }
    }
    PhaseScope ps(c, PH_QR, n);
    if (k > 0) {  // W <- (I - Q Q^T) W, twice (re-orthogonalisation)
      for (int rep = 0; rep < 2; ++rep) project_out(c, Q.p, I, k, W.p, bb, T.p);  // T = Q^T W, W -= Q T
    }
    double *Qi = Q.p + (size_t)I * k;
    householder_qr(c, W.p, I, bb, Qi);  // the basis of Q is the core basis with ADAPT_NO_TRUNCATE
    ps.next(PH_BPASS);
    // B_i = Q_i^T G_(n) written into rows k..k+bb of B (L, cap, R) via a strided copy
    DevBuf<double> gram(c, (size_t)bb * bb);
    DevBuf<unsigned char> Bi(c, (size_t)v.L * bb * v.R * dt_size(store));
    if (fused) {
      const int bb1 = std::max(0, std::min(block, cap - (k + bb)));
      Wn.alloc(c, (size_t)I * std::max(bb1, 1) + 1);
      fused_block(c, (const double *)G, v, n, Qi, bb, seed, k + bb, bb1, sh.col_offset, fp32_data, (double *)Bi.p,
                  gram.p, Wn.p);
      wn_cols = bb1;
      if (sh.on) allreduce_sum_f64(c, gram.p, (size_t)bb * bb);
    } else if (!sh.rows) {
      ttm_dense(c, G, gt, v, Qi, I, bb, Bi.p, store, mul_f64, gram.p, colmax.p);
      if (sh.on) allreduce_sum_f64(c, gram.p, (size_t)bb * bb);
    } else {
      ttm_dense(c, G, gt, v, Qi + sh.row_offset, I, bb, Bi.p, store, mul_f64, nullptr);
      allreduce_sum(c, Bi.p, (size_t)v.L * bb * v.R, store == DT::F64);  // sum over the sharded index
      mode_gram(c, Bi.p, store, ModeView{v.L, bb, v.R}, gram.p);
    }
    RT_CUDA(cudaMemcpy2DAsync((unsigned char *)Bfull.p + (size_t)v.L * k * dt_size(store),
                              (size_t)v.L * cap * dt_size(store), Bi.p, (size_t)v.L * bb * dt_size(store),
                              (size_t)v.L * bb * dt_size(store), v.R, cudaMemcpyDeviceToDevice, c.stream));
    RT_LAUNCH(c, block_stats_kernel, 1, 256, 0, gram.p, bb, W.p, (int64_t)I * bb, scal.p);
    double st[2];
    RT_CUDA(cudaMemcpyAsync(st, scal.p, sizeof st, cudaMemcpyDeviceToHost, c.stream));
    RT_CUDA(cudaStreamSynchronize(c.stream));
    // W was the PROJECTED block before its QR (householder_qr leaves W unchanged): the floor
    // test (range exhausted) discards this block and stops
    if (std::sqrt(st[1]) <= floor_abs) break;
    E -= st[0];  // E -= ||B_i||^2 (exact identity for orthonormal Q)
    k += bb;
  }
  out.k = k;
  // compact B to (L, k, R)
  DevBuf<unsigned char> B(c, (size_t)v.L * std::max(k, 1) * v.R * dt_size(store));
  if (k > 0)
    RT_CUDA(cudaMemcpy2DAsync(B.p, (size_t)v.L * k * dt_size(store), Bfull.p, (size_t)v.L * cap * dt_size(store),
                              (size_t)v.L * k * dt_size(store), v.R, cudaMemcpyDeviceToDevice, c.stream));
  Bfull.release();
  const ModeView vb{v.L, k, v.R};
  out.rows_replicated = sh.rows;
  if (!truncate || k == 0) {
    out.r = k;
    out.A = (double *)dev_alloc(c, sizeof(double) * I * std::max(k, 1));
    if (k > 0) RT_CUDA(cudaMemcpyAsync(out.A, Q.p, sizeof(double) * I * k, cudaMemcpyDeviceToDevice, c.stream));
    out.G = std::move(B);
    out.gt = store;
    out.replaced = true;
    return out;
  }
  // ---- truncation: eigenpairs of B B^T (thin SVD of B), r from the cumulative spectrum
  PhaseScope ps(c, PH_EIG, n);
  DevBuf<double> gram(c, (size_t)k * k), w(c, k), U(c, (size_t)k * k);
  if (store == DT::F64 && k > 64) gram_f64(c, (const double *)B.p, v.L, k, v.R, gram.p);  // tensor cores
  else mode_gram(c, B.p, store, vb, gram.p);
  if (sh.on && !sh.rows) allreduce_sum_f64(c, gram.p, (size_t)k * k);
  gram_eig(c, gram.p, k, w.p, U.p, nullptr, k, sh.rel_acc);  // r not known yet: the whole spectrum
  std::vector<double> hw(k);
  RT_CUDA(cudaMemcpyAsync(hw.data(), w.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  int r = k;
  double cum = 0.0;
  for (int i = 0; i < k; ++i) {
    cum += hw[i];
    if (gn2 - cum <= tau2) {
      r = i + 1;
      break;
    }
  }
  out.r = r;
  out.A = (double *)dev_alloc(c, sizeof(double) * I * r);
  gemm_small(c, false, Q.p, I, U.p, k, out.A, I, I, r, k);
  canonical_signs(c, out.A, I, r, U.p, k, k);
  if (want_core) {
    ps.next(PH_SHRINK);
    out.G.alloc(c, (size_t)v.L * r * v.R * dt_size(store));
    if (store == DT::F64 && r > 64) {  // G <- U_r^T B as GEMMs on the fp64 tensor cores
      if (v.L == 1)
        gemm_f64(c, true, U.p, k, (const double *)B.p, k, (double *)out.G.p, r, r, v.R, k);
      else  // per r-slab: G_r (L x r) = B_r (L x k) U_r (k x r)
        gemm_f64_batched(c, false, false, (const double *)B.p, v.L, v.L * k, U.p, k, 0, (double *)out.G.p, v.L,
                         v.L * r, v.L, r, k, v.R);
    } else {
      ttm_dense(c, B.p, store, vb, U.p, k, r, out.G.p, store, mul_f64 || store == DT::F64, nullptr);
    }
    out.gt = store;
    out.replaced = true;
  }
  return out;
}

}  // namespace

rtucker_result *run_adaptive(Ctx &c, const rtucker_dense_desc *X, double tol, int block, const double *mode_tol,
                             const int32_t *order, uint64_t seed, uint32_t flags) {
  DenseIn in;
  prepare_dense(c, X, in);
  RT_REQUIRE(tol > 0.0 && tol < 1.0, "tol must lie in (0, 1)");
  RT_REQUIRE(block >= 1, "block must be >= 1");
  const int d = in.d;
  std::vector<double> eps(d, tol / std::sqrt((double)d));
  if (mode_tol) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      RT_REQUIRE(mode_tol[k] >= 0.0, "mode_tol must be >= 0");
      eps[k] = mode_tol[k];
      s += mode_tol[k] * mode_tol[k];
    }
    RT_REQUIRE(std::fabs(s - tol * tol) <= 1e-12 * std::max(1.0, tol * tol), "sum mode_tol^2 must equal tol^2");
  }
  const bool hosvd = flags & RTUCKER_ADAPT_HOSVD;
  const bool truncate = !(flags & RTUCKER_ADAPT_NO_TRUNCATE);
  int32_t ord[kMaxModes];
  check_order(hosvd ? nullptr : order, d, ord, in.gdims, in.sharded);
  if (hosvd)
    for (int k = 0; k < d; ++k) ord[k] = k;
  RT_REQUIRE(!in.sharded || eps[d - 1] > 0.0, "a sharded last mode must be compressed (mode_tol[d-1] > 0)");
  // precision: fp64 data -> fp64; fp32 data -> FP64 / FAST per flag, AUTO = HYBRID (fp32
  // products on the fp32 input, fp64 B and intermediates)
  const uint32_t acc = flags & RTUCKER_ACCUM_MASK;
  const bool f64 = in.dt == DT::F64 || acc == RTUCKER_ACCUM_FP64;
  const DT store = (in.dt == DT::F64 || acc != RTUCKER_ACCUM_FAST) ? DT::F64 : DT::F32;
  ResultGuard rg{c, new_result(d)};
  rtucker_result *res = rg.r;
  for (int k = 0; k < d; ++k) {
    res->dims[k] = in.gdims[k];
    res->order[k] = ord[k];
  }
  res->seed = seed;
  res->flags = flags;
  DevBuf<double> scal(c, 4);
  sumsq(c, in.ptr, in.dt, prod(in.ldims, d), scal.p);
  if (in.sharded) allreduce_sum_f64(c, scal.p, 1);
  const double nx2 = fetch(c, scal.p);
  if (!std::isfinite(nx2)) throw Error(RTUCKER_ENUMERIC, "adaptive: non-finite ||X||");
  RT_REQUIRE(nx2 > 0.0, "adaptive: ||X|| = 0");
  res->norm_sq = nx2;
  const double nx = std::sqrt(nx2);
  // range-exhaustion floor (reading R8): 1e-13 ||X|| for fp64 data, 1e-6 ||X|| for fp32 data
  const double floor_abs = (in.dt == DT::F64 ? 1e-13 : 1e-6) * nx;

  int64_t cur[kMaxModes], gcur[kMaxModes];
  memcpy(cur, in.ldims, sizeof cur);
  memcpy(gcur, in.gdims, sizeof gcur);
  const void *G = in.ptr;
  DT gt = in.dt;
  bool g_sharded = in.sharded;  // the current core still holds only this rank's slab
  DevBuf<unsigned char> gown;
  for (int jj = 0; jj < d; ++jj) {
    const int n = ord[jj];
    res->order[jj] = n;
    if (eps[n] == 0.0) {  // mode not compressed: A = I (reading R8)
      double *A = (double *)dev_alloc(c, sizeof(double) * gcur[n] * gcur[n]);
      std::vector<double> eye((size_t)gcur[n] * gcur[n], 0.0);
      for (int64_t i = 0; i < gcur[n]; ++i) eye[i + gcur[n] * i] = 1.0;
      RT_CUDA(cudaMemcpyAsync(A, eye.data(), sizeof(double) * eye.size(), cudaMemcpyHostToDevice, c.stream));
      RT_CUDA(cudaStreamSynchronize(c.stream));
      res->factors[n] = A;
      res->ranks[n] = gcur[n];
      res->ell[n] = gcur[n];
      continue;
    }
    const double tau2 = (eps[n] * nx) * (eps[n] * nx);
    const void *src = hosvd ? in.ptr : G;
    const DT st = hosvd ? in.dt : gt;
    const int64_t *dims = hosvd ? in.ldims : cur;
    const int64_t *gdims = hosvd ? in.gdims : gcur;
    const bool mulf = f64 || st == DT::F64;
    Shard sh;
    sh.on = in.sharded;
    sh.rows = in.sharded && n == d - 1;
    sh.row_offset = in.offset;
    sh.col_offset = (in.sharded && n != d - 1) ? col_offset_for(in, dims, n) : 0;
    sh.rel_acc = in.dt == DT::F64;
    ModeOut mo = adapt_mode(c, src, st, dims, gdims, d, n, tau2, block, seed, floor_abs, mulf, store, truncate,
                            !hosvd, scal.p + 1, in.dt == DT::F32 && !f64, sh);
    res->factors[n] = mo.A;
    res->ranks[n] = mo.r;
    res->ell[n] = mo.k;
    if (!hosvd) {
      const double before = fetch(c, scal.p + 1);  // ||G_prev||^2 (global) computed in adapt_mode
      cur[n] = mo.r;
      gcur[n] = mo.r;
      gown = std::move(mo.G);
      G = gown.p;
      gt = mo.gt;
      if (mo.rows_replicated) g_sharded = false;
      sumsq(c, G, gt, prod(cur, d), scal.p + 2);
      if (g_sharded) allreduce_sum_f64(c, scal.p + 2, 1);
      res->mode_residual_sq[n] = before - fetch(c, scal.p + 2);
    }
  }
  if (hosvd) {  // G = X x_1 A_1^T ... x_d A_d^T (Alg 4 line 5); mode d of a sharded input: partial + allreduce
    PhaseScope ps(c, PH_SHRINK, 0);
    memcpy(cur, in.ldims, sizeof cur);
    DevBuf<unsigned char> g0, g1;
    const void *Gc = in.ptr;
    DT gc = in.dt;
    for (int n = 0; n < d; ++n) {
      const ModeView v = mode_view(cur, d, n);
      const int rr = (int)res->ranks[n];
      const bool last_sharded = in.sharded && n == d - 1;
      DevBuf<unsigned char> &dst = (Gc == g0.p) ? g1 : g0;
      const DT ot = last_sharded ? DT::F64 : store;
      dst.alloc(c, (size_t)v.L * rr * v.R * dt_size(ot));
      const double *An = (const double *)res->factors[n] + (last_sharded ? in.offset : 0);
      ttm_dense(c, Gc, gc, v, An, in.gdims[n], rr, dst.p, ot, f64 || gc == DT::F64 || ot == DT::F64, nullptr);
      if (last_sharded) allreduce_sum_f64(c, (double *)dst.p, (size_t)v.L * rr * v.R);
      Gc = dst.p;
      gc = ot;
      cur[n] = rr;
    }
    gown = std::move(Gc == g0.p ? g0 : g1);
    G = gown.p;
    gt = gc;
  }
  const int64_t ncore = prod(cur, d);
  res->core = dev_alloc(c, sizeof(double) * std::max<int64_t>(ncore, 1));
  convert(c, G, gt, res->core, DT::F64, ncore);
  finish_result(c, res, flags);
  check_status(c);  // synchronises
  return rg.release();
}

}  // namespace rt
