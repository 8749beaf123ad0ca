// Device generator of the Gaussian test matrices Omega_n.
//
// Binding definition: DESIGN.md reading R3 —
//   Philox4x32-10 (multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key increments
//   0x9E3779B9 / 0xBB67AE85, 10 rounds), key = (seed_lo, seed_hi),
//   counter = (k >> 2, mode | v << 8, c_lo, c_hi);  u_i = (w_i + 0.5) 2^-32;
//   Box-Muller: k&3 = 0,1 -> sqrt(-2 ln u0) (cos, sin)(2 pi u1); k&3 = 2,3 -> same on (u2, u3).
// fp64 Box-Muller uses log/sqrt/sincospi in double.  The fp32 variant evaluates the
// radius from log1p(-(1-u)) when u > 1/2 (1-u is exact from ~w), branch-free, and the angle
// through t = 2u-1 so that both stay within a few fp32 ulp of the fp64 values.
#pragma once
#include <stdint.h>

namespace rt {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// Words for Philox block j (= k >> 2) of unfolding column c of mode `mode`.
__device__ __forceinline__ uint4 omega_words(uint64_t seed, int mode, int v, uint64_t c,
                                             uint32_t j) {
  return philox4x32_10(make_uint4(j, (uint32_t)mode | ((uint32_t)v << 8), (uint32_t)c,
                                  (uint32_t)(c >> 32)),
                       (uint32_t)seed, (uint32_t)(seed >> 32));
}

__device__ __forceinline__ double2 box_muller_f64(uint32_t wa, uint32_t wb) {
  const double ua = ((double)wa + 0.5) * 0x1p-32;
  const double ub = ((double)wb + 0.5) * 0x1p-32;
  const double r = sqrt(-2.0 * log(ua));
  double s, c;
  sincospi(2.0 * ub, &s, &c);
  return make_double2(r * c, r * s);
}

__device__ __forceinline__ float2 box_muller_f32(uint32_t wa, uint32_t wb) {
  // ln u_a without branches (a warp evaluates one formula): u >= 1/2 -> log1p(-v) with
  // v = 1 - u taken from ~w (no cancellation near u = 1); u < 1/2 -> u = 2^e m with
  // m in [sqrt(1/2), sqrt(2)): e ln 2 + log1p(m - 1) (m - 1 exact).  log1p(z) = 2 atanh(s),
  // s = z / (2 + z), |s| <= 1/3, by its odd series to s^13 (truncation < 2^-26 relative);
  // the rounding of 2 + z is carried (tl) into s.  Max relative error of ln u vs fp64:
  // 2.2e-7, of which ~1e-7 is the fp32 rounding of u itself (scripts/dbg/bm_log.py model).
  const bool hi = (wa & 0x80000000u) != 0;
  const float v = ((float)(~wa) + 0.5f) * 0x1p-32f;
  const float u = ((float)wa + 0.5f) * 0x1p-32f;
  const int ib = (int)__float_as_uint(u) - 0x3f3504f3;
  const int e = ib >> 23;
  const float m = __uint_as_float(__float_as_uint(u) - ((uint32_t)e << 23));
  const float z = hi ? -v : m - 1.0f;
  const float ef = hi ? 0.0f : (float)e;
  const float t = 2.0f + z, tl = (2.0f - t) + z;
  float rc;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(t));
  float s = z * rc;
  s = fmaf(fmaf(-s, t, z), rc, s);
  s = fmaf(-s, tl * rc, s);
  const float x = s * s;
  float P = fmaf(x, 1.0f / 13.0f, 1.0f / 11.0f);
  P = fmaf(P, x, 1.0f / 9.0f);
  P = fmaf(P, x, 1.0f / 7.0f);
  P = fmaf(P, x, 1.0f / 5.0f);
  P = fmaf(P, x, 1.0f / 3.0f);
  P *= x;
  const float s2 = 2.0f * s;
  const float ln = fmaf(ef, 0.693145751953125f, fmaf(ef, 1.428606765330187e-6f, fmaf(s2, P, s2)));
  const float r = sqrtf(-2.0f * ln);
  const float tt = ((float)(int32_t)(wb ^ 0x80000000u) + 0.5f) * 0x1p-31f;  // 2 u_b - 1
  float sn, cs;
  sincospif(tt, &sn, &cs);  // (cos, sin)(2 pi u) = -(cos, sin)(pi t)
  return make_float2(-r * cs, -r * sn);
}

template <typename T>
struct Normal4;
template <>
struct Normal4<double> {
  double v[4];
  __device__ __forceinline__ Normal4(uint4 w) {
    double2 a = box_muller_f64(w.x, w.y), b = box_muller_f64(w.z, w.w);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};
template <>
struct Normal4<float> {
  float v[4];
  __device__ __forceinline__ Normal4(uint4 w) {
    float2 a = box_muller_f32(w.x, w.y), b = box_muller_f32(w.z, w.w);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};

}  // namespace rt
