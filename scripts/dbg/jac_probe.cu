// Latency of one register-resident Jacobi pair step (jac_pair) for a single warp: slot data
// kV = 16 rows per lane, as in gram_eig_kernel.  Prints cycles per step for variants.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_approx_f64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
template <int kV, int VAR>
__device__ __forceinline__ void jac_pair(double (&x)[kV], double (&y)[kV], double tol2, int &rot) {
  double g0 = 0.0, g1 = 0.0, a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
  for (int v = 0; v < kV; v += 2) {
    g0 = fma(x[v], y[v], g0); g1 = fma(x[v + 1], y[v + 1], g1);
    a0 = fma(x[v], x[v], a0); a1 = fma(x[v + 1], x[v + 1], a1);
    b0 = fma(y[v], y[v], b0); b1 = fma(y[v + 1], y[v + 1], b1);
  }
  double g = g0 + g1, a = a0 + a1, b = b0 + b1;
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    g += __shfl_xor_sync(0xffffffffu, g, o);
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (VAR == 2) { rot += (g != 0.0); return; }
  if (VAR == 6 && g != 0.0 && g * g > tol2 * a * b) {
    rot = 1;
    const double d = b - a, g2 = 2.0 * g;
    // common power-of-two scale so both fit fp32: exponent of max(|d|, |g2|)
    const int e = max((int)((__double2hiint(d) >> 20) & 0x7ff), (int)((__double2hiint(g2) >> 20) & 0x7ff));
    const double sc = __hiloint2double((2046 - e) << 20, 0);  // 2^(1023 - e)
    const float fd = (float)(d * sc), fg = (float)(g2 * sc);
    float r0, r1, r2, r3;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(fg));
    const float zf = fd * r0;
    const float s1 = fmaf(zf, zf, 1.0f);
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(s1));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(fabsf(zf) + s1 * r1));
    const float tf = copysignf(r2, zf);
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r3) : "f"(fmaf(tf, tf, 1.0f)));
    const double t = (double)tf, u = fma(t, t, 1.0);
    double c = (double)r3;
    c = fma(0.5 * c, fma(-u * c, c, 1.0), c);
    c = fma(0.5 * c, fma(-u * c, c, 1.0), c);
    const double s = t * c;
#pragma unroll
    for (int v = 0; v < kV; ++v) {
      const double xv = x[v], yv = y[v];
      x[v] = fma(c, xv, -s * yv);
      y[v] = fma(s, xv, c * yv);
    }
    return;
  }
  if (VAR != 6 && g != 0.0 && g * g > tol2 * a * b) {
    rot = 1;
    double t;
    if (VAR == 0 || VAR == 5) {
      const double zeta = (b - a) * rcp_approx_f64(2.0 * g);
      if (fabs(zeta) > 1e7) {
        t = 0.5 * rcp_approx_f64(zeta);
      } else {
        const float zf = (float)zeta;
        const float sq = sqrtf(fmaf(zf, zf, 1.0f));
        t = (double)copysignf(__frcp_rn(fabsf(zf) + sq), zf);
      }
    } else {
      const float zf = (float)((b - a) * rcp_approx_f64(2.0 * g));
      float r1, r2;
      const float s1 = fmaf(zf, zf, 1.0f);
      asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(s1));
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(fabsf(zf) + s1 * r1));
      t = (double)copysignf(r2, zf);
    }
    double c;
    if (VAR >= 3) {
      const double u = fma(t, t, 1.0);
      double r;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(u));
      const double hu = 0.5 * u;
      r = r * fma(-hu * r, r, 1.5);
      r = r * fma(-hu * r, r, 1.5);
      c = r;
    } else {
      c = rsqrt(fma(t, t, 1.0));
    }
    const double s = t * c;
    if (VAR == 4) { x[0] += c; y[0] += s; return; }
#pragma unroll
    for (int v = 0; v < kV; ++v) {
      const double xv = x[v], yv = y[v];
      x[v] = fma(c, xv, -s * yv);
      y[v] = fma(s, xv, c * yv);
    }
  }
}
template <int VAR>
__global__ void probe(double *out, long long *cyc, int iters) {
  constexpr int kV = 16;
  const int lane = threadIdx.x & 31, slot = lane >> 2, q = lane & 3;
  double x[kV], y[kV];
  for (int v = 0; v < kV; ++v) { x[v] = 1.0 / (1 + q + 4 * v + slot); y[v] = 1.0 / (2 + q + 4 * v + slot * 3); }
  int rot = 0;
  const int nxt = ((slot + 1) & 7) * 4 + q;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    jac_pair<kV, VAR>(x, y, 1e-30, rot);
#pragma unroll
    for (int v = 0; v < kV; ++v) y[v] = __shfl_sync(0xffffffffu, y[v], nxt);
  }
  long long t1 = clock64();
  double s = 0;
  for (int v = 0; v < kV; ++v) s += x[v] + y[v];
  out[threadIdx.x] = s + rot;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / iters;
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  long long h;
  probe<0><<<1, 32>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("fp32 IEEE angle: %lld cycles/step\n", h);
  probe<1><<<1, 32>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("approx angle:    %lld cycles/step\n", h);
  probe<3><<<1, 32>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("approx angle + NR rsqrt: %lld cycles/step\n", h);
  probe<4><<<1, 32>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("approx angle + NR, no rotation: %lld cycles/step\n", h);
  probe<6><<<1, 32>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("fp32 scaled angle + 2 NR: %lld cycles/step\n", h);
  probe<2><<<1, 32>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dots+move only:  %lld cycles/step\n", h);
  return 0;
}
