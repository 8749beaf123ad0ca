// Structure-preserving SP-STHOSVD (Alg 6) for COO tensors:
//   for j in rho:  Y = G_(j) Omega_j                 (sketch over the nonzeros)
//                  Q = qr(Y)                         (Householder)
//                  S = strong RRQR on Q^T, eta       (DESIGN reading R9: CPQR + maxvol)
//                  A_j = Q (P^T Q)^{-1}
//                  G_(j) <- P^T G_(j)                (keep the selected slices, renumber)
// The core keeps the input values bit-exactly.  The selection and the
// new nnz are data dependent, so the call synchronises the stream after every mode.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "comm.h"
#include "kernels_extra.h"
#include "orchestrate.h"
#include "philox.cuh"

namespace rt {

namespace {

constexpr int kHot = 32;      // hottest rows (smallest indices) kept warp-private per CTA
constexpr int kCooT = 256;
constexpr int kMaxEll = 64;

// ---------------------------------------------------------------- COO sketch (a8) --
// Y[i_j, k] += v * Omega_j[c, k0 + k], c = sum_{m != j} i_m prod_{m' < m, m' != j} I_m'.
// Products and sums in fp64.  Count tensors are heavy-tailed (BASELINE configs[4]: Zipf(1.1)
// indices, the heaviest mode-3 row holds ~9 % of the nonzeros), so naive atomics serialise
// on a few addresses.  Per warp instruction, lanes holding the same row are first combined
// with __match_any_sync + a leader reduction (one update per distinct row and warp); rows
// < kHot (the heavy rows of these tensors) then go to a warp-private shared-memory
// accumulator (no atomics: one writer lane per row per instruction), flushed once per CTA;
// other rows use one fp64 global atomic per distinct row and warp.  Global fp64 atomics make
// the sum order run-dependent (rounding-level differences only).
template <typename TV, typename TN>
__global__ void __launch_bounds__(kCooT) sketch_coo_kernel(CooDev g, int mode, int ell, uint64_t seed,
                                                           int64_t nper, double *__restrict__ Y) {
  extern __shared__ double hot[];  // [warps][kHot][ell]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t I = g.dims[mode];
  const int hrows = (int)(I < kHot ? I : kHot);
  double *myhot = hot + (size_t)warp * kHot * ell;
  for (int e = threadIdx.x; e < (kCooT / 32) * kHot * ell; e += kCooT) hot[e] = 0.0;
  __syncthreads();
  int64_t stride[kMaxModes];
  int64_t s = 1;
  for (int k = 0; k < g.d; ++k) {
    stride[k] = (k == mode) ? 0 : s;
    if (k != mode) s *= g.dims[k];
  }
  const TV *vals = (const TV *)g.vals;
  const int nb = (ell + 3) >> 2;
  const int64_t e0 = (int64_t)blockIdx.x * nper, e1 = min(g.nnz, e0 + nper);
  // warp-strided loop with uniform trip count (inactive lanes carry row = -1)
  for (int64_t base = e0 + (int64_t)warp * 32; base < e1; base += kCooT) {
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
    // rows shared by more than two lanes (the heavy rows of Zipf-like data): tree reduction over
    // the group in 5 shuffle steps (partner = the member 2^k ranks further, __fns) instead of
    // a serial loop over up to 32 members
    const bool big = __any_sync(0xffffffffu, __popc(grp) > 2);
    unsigned src[5];
    const int rank = __popc(grp & ((1u << lane) - 1u));
    if (big) {
#pragma unroll
      for (int k = 0; k < 5; ++k) src[k] = __fns(grp, lane, 1 + (1 << k));
    }
    for (int jb = 0; jb < nb; ++jb) {
      float4 dummy;
      (void)dummy;
      double pr[4] = {0.0, 0.0, 0.0, 0.0};
      if (act) {
        const uint4 w = omega_words(seed, mode, 0, (uint64_t)c, (uint32_t)jb);
        Normal4<TN> z(w);
#pragma unroll
        for (int q = 0; q < 4; ++q) pr[q] = v * (double)z.v[q];
      }
      // sum over the lanes of this row group (into the group's first lane)
      if (!big) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double t = 0.0;
          unsigned m = grp;
          while (m) {
            const int sl = __ffs(m) - 1;
            t += __shfl_sync(grp, pr[q], sl);
            m &= m - 1;
          }
          pr[q] = t;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const bool take = src[k] != 0xffffffffu && (rank & ((2 << k) - 1)) == 0;
          const int sl = (src[k] != 0xffffffffu) ? (int)src[k] : lane;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double o = __shfl_sync(0xffffffffu, pr[q], sl);
            if (take) pr[q] += o;
          }
        }
      }
      if (act && lane == leader) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = 4 * jb + q;
          if (k < ell) {
            if (row < hrows) myhot[row * ell + k] += pr[q];
            else atomicAdd(&Y[row + I * k], pr[q]);
          }
        }
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < hrows * ell; e += kCooT) {
    double t = 0.0;
    for (int w = 0; w < kCooT / 32; ++w) t += hot[(size_t)w * kHot * ell + e];
    if (t != 0.0) atomicAdd(&Y[(e / ell) + I * (e % ell)], t);
  }
}

// ------------------------------------------------------ CPQR on Q^T (a9, step 1) --
// r: I rows of length ell (row-major copy of Q); per step j the residual norms
// sum_{t >= j} r_i[t]^2 (fixed order), argmax with ties to the smallest index.
struct ArgMax {
  double v;
  int64_t i;
};
__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
  return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}
__device__ ArgMax block_argmax(ArgMax m) {
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  for (int o = 16; o; o >>= 1) {
    ArgMax t{__shfl_xor_sync(0xffffffffu, m.v, o), __shfl_xor_sync(0xffffffffu, m.i, o)};
    m = better(m, t);
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = m.v;
    si[threadIdx.x >> 5] = m.i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = better(m, ArgMax{sv[w], si[w]});
  }
  return m;
}

__global__ void cpqr_norm_argmax(const double *__restrict__ r, int64_t I, int ell, int j,
                                 const int *__restrict__ chosen, double *__restrict__ pv, int64_t *__restrict__ pi) {
  ArgMax m{-1.0, INT64_MAX};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x) {
    if (chosen[i]) continue;
    double s = 0.0;
    for (int t = j; t < ell; ++t) s += r[i * ell + t] * r[i * ell + t];
    m = better(m, ArgMax{s, i});
  }
  m = block_argmax(m);
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = m.v;
    pi[blockIdx.x] = m.i;
  }
}

__global__ void argmax_finish(const double *__restrict__ pv, const int64_t *__restrict__ pi, int n,
                              int64_t *__restrict__ out_i, double *__restrict__ out_v, int *__restrict__ chosen) {
  ArgMax m{-1.0, INT64_MAX};
  for (int b = threadIdx.x; b < n; b += blockDim.x) m = better(m, ArgMax{pv[b], pi[b]});
  m = block_argmax(m);
  if (threadIdx.x == 0) {
    *out_i = m.i;
    if (out_v) *out_v = m.v;
    if (chosen && m.i != INT64_MAX) chosen[m.i] = 1;
  }
}

// Householder reflector from column p's rows j..ell-1 (oracle form: alpha = -sign(v0)||v||,
// v0 -= alpha, v /= ||v||), applied to every column: r_i[j:] -= 2 (v . r_i[j:]) v.
__global__ void cpqr_reflect(double *__restrict__ r, int64_t I, int ell, int j, const int64_t *__restrict__ pivot) {
  __shared__ double v[256];
  __shared__ double scale;
  const int64_t p = *pivot;
  if (threadIdx.x == 0) {
    double nv = 0.0;
    for (int t = j; t < ell; ++t) { v[t] = r[p * ell + t]; nv += v[t] * v[t]; }
    nv = sqrt(nv);
    if (nv == 0.0) {
      scale = 0.0;
    } else {
      const double alpha = v[j] >= 0.0 ? -nv : nv;
      v[j] -= alpha;
      double vn = 0.0;
      for (int t = j; t < ell; ++t) vn += v[t] * v[t];
      vn = sqrt(vn);
      if (vn == 0.0) {
        scale = 0.0;
      } else {
        for (int t = j; t < ell; ++t) v[t] /= vn;
        scale = 1.0;
      }
    }
  }
  __syncthreads();
  if (scale == 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == p) continue;  // the pivot column is read by every CTA above and never used again
    double s = 0.0;
    for (int t = j; t < ell; ++t) s += v[t] * r[i * ell + t];
    for (int t = j; t < ell; ++t) r[i * ell + t] -= 2.0 * s * v[t];
  }
}

__global__ void transpose_q(const double *__restrict__ Q, int64_t I, int ell, double *__restrict__ r) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < I * ell; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ell;
    const int t = (int)(e % ell);
    r[e] = Q[i + I * t];
  }
}

// --------------------------------------- oblique factor A = Q Q_S^{-1} (a9, step 2) --
// Inverse of Q_S (ell x ell, rows sel of Q) by Gauss-Jordan with partial pivoting (one CTA).
// status = 1 when a pivot is below ell * eps * max|Q_S| (singular P^T Q, ENUMERIC).
__global__ void qs_inverse(const double *__restrict__ Q, int64_t I, int ell, const int64_t *__restrict__ sel,
                           double *__restrict__ inv, int *__restrict__ status) {
  extern __shared__ double sm[];
  double *M = sm;                 // ell x 2 ell, row-major
  const int w = 2 * ell;
  __shared__ int piv;
  __shared__ double amax;
  for (int e = threadIdx.x; e < ell * w; e += blockDim.x) {
    const int r = e / w, cc = e % w;
    M[e] = cc < ell ? Q[sel[r] + I * cc] : (cc - ell == r ? 1.0 : 0.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int r = 0; r < ell; ++r)
      for (int cc = 0; cc < ell; ++cc) a = fmax(a, fabs(M[r * w + cc]));
    amax = a;
    *status = 0;
  }
  __syncthreads();
  for (int col = 0; col < ell; ++col) {
    if (threadIdx.x == 0) {
      int best = col;
      for (int r = col + 1; r < ell; ++r)
        if (fabs(M[r * w + col]) > fabs(M[best * w + col])) best = r;
      piv = best;
      if (!(fabs(M[best * w + col]) > ell * 2.2e-16 * amax)) *status = 1;
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
    const double d = M[col * w + col];
    __syncthreads();
    for (int cc = threadIdx.x; cc < w; cc += blockDim.x) M[col * w + cc] /= d;
    __syncthreads();
    for (int e = threadIdx.x; e < ell * w; e += blockDim.x) {
      const int r = e / w, cc = e % w;
      if (r != col) {
        const double f = M[r * w + col];
        if (cc != col) M[e] -= f * M[col * w + cc];
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < ell; r += blockDim.x)
      if (r != col) M[r * w + col] = 0.0;
    __syncthreads();
  }
  // M[:, ell:] = Q_S^{-1}; store column-major inv[a + ell b]
  for (int e = threadIdx.x; e < ell * ell; e += blockDim.x) {
    const int a = e % ell, b = e / ell;
    inv[e] = M[a * w + ell + b];
  }
}

// A = Q inv (I x ell), and the argmax of |A_ik| over rows not in the selection (row-major
// flat order: smallest i, then smallest k on ties).
__global__ void oblique_apply(const double *__restrict__ Q, int64_t I, int ell, const double *__restrict__ inv,
                              const int *__restrict__ insel, double *__restrict__ A, double *__restrict__ pv,
                              int64_t *__restrict__ pi) {
  ArgMax m{-1.0, INT64_MAX};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < ell; ++k) {
      double s = 0.0;
      for (int t = 0; t < ell; ++t) s += Q[i + I * t] * inv[t + ell * k];
      A[i + I * k] = s;
      if (!insel[i]) m = better(m, ArgMax{fabs(s), i * ell + k});
    }
  }
  m = block_argmax(m);
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = m.v;
    pi[blockIdx.x] = m.i;
  }
}

// ------------------------------------------------------- selection / compaction (a10) --
__global__ void mark_sel(const int64_t *__restrict__ sel, int ell, int *__restrict__ mark) {
  for (int t = threadIdx.x; t < ell; t += blockDim.x) mark[sel[t]] = 1;
}

__global__ void build_lookup(const int64_t *__restrict__ sel, int ell, int32_t *__restrict__ lut) {
  for (int t = threadIdx.x; t < ell; t += blockDim.x) lut[sel[t]] = t;
}

constexpr int kCompactB = 1024;

__global__ void compact_count(const int32_t *__restrict__ idx, int64_t nnz, const int32_t *__restrict__ lut,
                              int64_t *__restrict__ counts) {
  __shared__ int64_t sc[32];
  const int64_t e = (int64_t)blockIdx.x * kCompactB + threadIdx.x;
  const int keep = (e < nnz && lut[idx[e]] >= 0) ? 1 : 0;
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if ((threadIdx.x & 31) == 0) sc[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int w = 0; w < kCompactB / 32; ++w) s += sc[w];
    counts[blockIdx.x] = s;
  }
}

__global__ void exclusive_scan_single(int64_t *__restrict__ v, int64_t n, int64_t *__restrict__ total) {
  // one CTA: chunked sequential scan with a per-thread chunk then a CTA scan of chunk sums
  __shared__ int64_t part[1024];
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per, e = min(n, b + per);
  int64_t s = 0;
  for (int64_t k = b; k < e; ++k) s += v[k];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const int64_t x = part[t];
      part[t] = acc;
      acc += x;
    }
    *total = acc;
  }
  __syncthreads();
  int64_t acc = part[threadIdx.x];
  for (int64_t k = b; k < e; ++k) {
    const int64_t x = v[k];
    v[k] = acc;
    acc += x;
  }
}

template <typename TV>
__global__ void compact_scatter(CooDev in, int mode, const int32_t *__restrict__ lut, const int64_t *__restrict__ offs,
                                int32_t *const *__restrict__ oidx, TV *__restrict__ ovals) {
  __shared__ int wsum[32];
  const int64_t e = (int64_t)blockIdx.x * kCompactB + threadIdx.x;
  int32_t pos = -1;
  if (e < in.nnz) pos = lut[in.idx[mode][e]];
  const int keep = pos >= 0;
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wsum[w] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < kCompactB / 32; ++k) {
      const int x = wsum[k];
      wsum[k] = acc;
      acc += x;
    }
  }
  __syncthreads();
  if (!keep) return;
  const int64_t o = offs[blockIdx.x] + wsum[w] + __popc(bal & ((1u << lane) - 1u));
  for (int k = 0; k < in.d; ++k) oidx[k][o] = (k == mode) ? pos : in.idx[k][e];
  ovals[o] = ((const TV *)in.vals)[e];
}

__global__ void fill_i32(int32_t *p, int64_t n, int32_t v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) p[e] = v;
}

template <typename T>
T fetch1(Ctx &c, const T *dev) {
  T h;
  RT_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  return h;
}

int grid_for(Ctx &c, int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * 8, (n + threads - 1) / threads));
}

}  // namespace

void sketch_coo(Ctx &c, const CooDev &g, int mode, int ell, uint64_t seed, bool normals_f64, double *Y) {
  const int64_t I = g.dims[mode];
  RT_REQUIRE(ell <= kMaxEll, "sparse sketch: l > 64 is not supported");
  RT_CUDA(cudaMemsetAsync(Y, 0, sizeof(double) * I * ell, c.stream));
  if (g.nnz == 0) return;
  const size_t smem = sizeof(double) * (kCooT / 32) * kHot * ell;
  const int64_t blocks = std::min<int64_t>((int64_t)c.num_sms * 4, (g.nnz + 1023) / 1024);
  const int64_t nper = (g.nnz + blocks - 1) / blocks;
#define RT_COO(TV, TN)                                                                                     \
  do {                                                                                                     \
    smem_attr(sketch_coo_kernel<TV, TN>, smem);                                                            \
    RT_LAUNCH(c, (sketch_coo_kernel<TV, TN>), (int)blocks, kCooT, smem, g, mode, ell, seed, nper, Y);      \
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

void srrqr(Ctx &c, const double *Q, int64_t m, int l, double eta, int64_t *sel_dev, double *A, int *swaps_host) {
  RT_REQUIRE(l >= 1 && l <= 256 && m >= l, "srrqr: need 1 <= l <= 256 and m >= l");
  DevBuf<double> r(c, (size_t)m * l);
  RT_LAUNCH(c, transpose_q, grid_for(c, m * l), 256, 0, Q, m, l, r.p);
  DevBuf<int> chosen(c, m);
  chosen.zero();
  const int g = grid_for(c, m);
  DevBuf<double> pv(c, g);
  DevBuf<int64_t> pi(c, g), piv(c, l);
  // Businger-Golub CPQR pivots (initial S)
  for (int j = 0; j < l; ++j) {
    RT_LAUNCH(c, cpqr_norm_argmax, g, 256, 0, r.p, m, l, j, chosen.p, pv.p, pi.p);
    RT_LAUNCH(c, argmax_finish, 1, 256, 0, pv.p, pi.p, g, piv.p + j, (double *)nullptr, chosen.p);
    RT_LAUNCH(c, cpqr_reflect, g, 256, 0, r.p, m, l, j, piv.p + j);
  }
  std::vector<int64_t> sel(l);
  RT_CUDA(cudaMemcpyAsync(sel.data(), piv.p, sizeof(int64_t) * l, cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  // maxvol swaps while max_{i not in S} |A_ik| > eta
  DevBuf<double> inv(c, (size_t)l * l), mv(c, 1);
  DevBuf<int> st(c, 1), insel(c, m);
  DevBuf<int64_t> dsel(c, l), mi(c, 1);
  const size_t qsm = sizeof(double) * l * 2 * l;
  if (qsm > 48 * 1024) smem_attr(qs_inverse, qsm);
  int swaps = 0;
  auto compute_A = [&](bool want_max) -> std::pair<double, int64_t> {
    RT_CUDA(cudaMemcpyAsync(dsel.p, sel.data(), sizeof(int64_t) * l, cudaMemcpyHostToDevice, c.stream));
    RT_LAUNCH(c, fill_i32, grid_for(c, m), 256, 0, insel.p, m, 0);
    RT_LAUNCH(c, mark_sel, 1, 256, 0, dsel.p, l, insel.p);
    RT_LAUNCH(c, qs_inverse, 1, 256, qsm, Q, m, l, dsel.p, inv.p, st.p);
    RT_LAUNCH(c, oblique_apply, g, 256, 0, Q, m, l, inv.p, insel.p, A, pv.p, pi.p);
    RT_LAUNCH(c, argmax_finish, 1, 256, 0, pv.p, pi.p, g, mi.p, mv.p, (int *)nullptr);
    const int status = fetch1(c, st.p);
    if (status) throw Error(RTUCKER_ENUMERIC, "SP-STHOSVD: singular P^T Q (fewer than l independent rows)");
    if (!want_max) return {0.0, 0};
    return {fetch1(c, mv.p), fetch1(c, mi.p)};
  };
  while (swaps < 10000) {
    auto best = compute_A(true);
    if (!(best.first > eta)) break;
    const int64_t i = best.second / l;
    const int k = (int)(best.second % l);
    sel[k] = i;
    ++swaps;
  }
  std::sort(sel.begin(), sel.end());
  compute_A(false);  // A for the sorted selection (its column order defines the renumbering)
  RT_CUDA(cudaMemcpyAsync(sel_dev, sel.data(), sizeof(int64_t) * l, cudaMemcpyHostToDevice, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  if (swaps_host) *swaps_host = swaps;
}

int64_t coo_select(Ctx &c, const CooDev &in, int mode, const int64_t *sel, int l, int32_t *const *out_idx,
                   void *out_vals) {
  const int64_t I = in.dims[mode];
  DevBuf<int32_t> lut(c, I);
  RT_LAUNCH(c, fill_i32, grid_for(c, I), 256, 0, lut.p, I, -1);
  RT_LAUNCH(c, build_lookup, 1, 256, 0, sel, l, lut.p);
  if (in.nnz == 0) return 0;
  const int64_t nblk = (in.nnz + kCompactB - 1) / kCompactB;
  DevBuf<int64_t> offs(c, nblk), total(c, 1);
  RT_LAUNCH(c, compact_count, (int)nblk, kCompactB, 0, in.idx[mode], in.nnz, lut.p, offs.p);
  RT_LAUNCH(c, exclusive_scan_single, 1, 1024, 0, offs.p, nblk, total.p);
  DevBuf<int32_t *> optr(c, kMaxModes);
  RT_CUDA(cudaMemcpyAsync(optr.p, out_idx, sizeof(int32_t *) * kMaxModes, cudaMemcpyHostToDevice, c.stream));
  if (in.vt == DT::F64)
    RT_LAUNCH(c, compact_scatter<double>, (int)nblk, kCompactB, 0, in, mode, lut.p, offs.p, optr.p, (double *)out_vals);
  else
    RT_LAUNCH(c, compact_scatter<float>, (int)nblk, kCompactB, 0, in, mode, lut.p, offs.p, optr.p, (float *)out_vals);
  return fetch1(c, total.p);
}

rtucker_result *run_sparse_sthosvd(Ctx &c, const rtucker_coo_desc *X, const int64_t *ranks, int p, uint64_t seed,
                                   const int32_t *order, double eta, uint32_t flags) {
  RT_REQUIRE(X != nullptr, "null tensor descriptor");
  if (X->d > kMaxModes) throw Error(RTUCKER_EUNSUPPORTED, "d > RTUCKER_MAX_MODES");
  RT_REQUIRE(X->d >= 1, "d must be >= 1");
  RT_REQUIRE(X->nnz >= 0, "nnz must be >= 0");
  RT_REQUIRE(p >= 0, "p must be >= 0");
  RT_REQUIRE(eta >= 1.0, "eta must be >= 1 (P:379)");
  RT_REQUIRE(X->dtype == RTUCKER_F32 || X->dtype == RTUCKER_F64, "dtype must be RTUCKER_F32 or RTUCKER_F64");
  RT_REQUIRE(c.nranks == 1, "rtucker_sparse_sthosvd: multi-rank contexts are not supported yet");
  const int d = X->d;
  const DT vt = X->dtype == RTUCKER_F64 ? DT::F64 : DT::F32;
  const size_t vs = dt_size(vt);
  int64_t cur[kMaxModes] = {0};
  for (int k = 0; k < d; ++k) {
    RT_REQUIRE(X->dims[k] >= 1 && X->dims[k] <= INT32_MAX, "every dim must lie in [1, 2^31)");
    RT_REQUIRE(ranks[k] >= 1, "r_n must be >= 1");
    cur[k] = X->dims[k];
  }
  int32_t ord[kMaxModes];
  check_order(order, d, ord, cur, false);
  const bool nf64 = vt == DT::F64 || (flags & RTUCKER_ACCUM_MASK) == RTUCKER_ACCUM_FP64;
  ResultGuard rg{c, new_result(d)};
  rtucker_result *res = rg.r;
  res->dtype = X->dtype;
  for (int k = 0; k < d; ++k) {
    res->dims[k] = X->dims[k];
    res->order[k] = ord[k];
  }
  res->seed = seed;
  res->flags = flags;
  // working COO (ping-pong), device resident
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
  }
  RT_REQUIRE(nnz0 == 0 || X->vals != nullptr, "null value array");
  if (nnz0) RT_CUDA(cudaMemcpyAsync(vb[0].p, X->vals, vs * nnz0, kind, c.stream));
  int cb = 0;
  int64_t nnz = nnz0;
  res->nnz_history[0] = nnz0;
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
    g.nnz = nnz;
    g.vals = vb[cb].p;
    g.vt = vt;
    const int64_t I = cur[n];
    DevBuf<double> Y(c, (size_t)I * ell), Q(c, (size_t)I * ell);
    {
      PhaseScope ps(c, PH_SKETCH, jj);
      sketch_coo(c, g, n, ell, seed, nf64, Y.p);
      ps.next(PH_QR);
      thin_qr(c, Y.p, I, ell, Q.p);
    }
    double *A = nullptr;
    A = (double *)dev_alloc(c, sizeof(double) * I * ell);
    res->factors[n] = A;
    int64_t *S = nullptr;
    S = (int64_t *)dev_alloc(c, sizeof(int64_t) * ell);
    res->selection[n] = S;
    {
      PhaseScope ps(c, PH_EIG, jj);
      int sw = 0;
      srrqr(c, Q.p, I, ell, eta, S, A, &sw);
      res->swaps[n] = sw;
    }
    // G_(n) <- P^T G_(n): keep the selected slices and renumber them 0..ell-1
    int32_t *oidx[kMaxModes] = {nullptr};
    for (int k = 0; k < d; ++k) oidx[k] = ib[1 - cb].p + (size_t)k * nnz0;
    {
      PhaseScope ps(c, PH_SHRINK, jj);
      nnz = coo_select(c, g, n, S, ell, oidx, vb[1 - cb].p);
    }
    cb = 1 - cb;
    cur[n] = ell;
    res->ranks[n] = ell;
    res->ell[n] = ell;
    res->nnz_history[jj + 1] = nnz;
  }
  res->core_nnz = nnz;
  for (int k = 0; k < d; ++k) {
    res->core_idx[k] = (int32_t *)dev_alloc(c, sizeof(int32_t) * std::max<int64_t>(nnz, 1));
    if (nnz)
      RT_CUDA(cudaMemcpyAsync(res->core_idx[k], ib[cb].p + (size_t)k * nnz0, sizeof(int32_t) * nnz,
                              cudaMemcpyDeviceToDevice, c.stream));
  }
  res->core_vals = dev_alloc(c, vs * std::max<int64_t>(nnz, 1));
  if (nnz) RT_CUDA(cudaMemcpyAsync(res->core_vals, vb[cb].p, vs * nnz, cudaMemcpyDeviceToDevice, c.stream));
  finish_result(c, res, flags);
  RT_CUDA(cudaStreamSynchronize(c.stream));
  return rg.release();
}

}  // namespace rt
