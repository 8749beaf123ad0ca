// fp64 / fp32 dependent-chain latency and warp-parallel throughput probe.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double *out, float *outf, long long *cyc, int iters) {
  double x = 1.0 + threadIdx.x * 1e-9, y = 0.999999, z = 1e-7;
  float xf = 1.0f + threadIdx.x * 1e-7f, yf = 0.999999f, zf = 1e-7f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, z);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = x * y + z * x;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) xf = fmaf(xf, yf, zf);
  long long t3 = clock64();
  double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
  for (int i = 0; i < iters; ++i) { a0 = fma(a0, y, z); a1 = fma(a1, y, z); a2 = fma(a2, y, z); a3 = fma(a3, y, z); a4 = fma(a4, y, z); a5 = fma(a5, y, z); a6 = fma(a6, y, z); a7 = fma(a7, y, z); }
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[threadIdx.x] = x + a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7; outf[threadIdx.x] = xf;
}
int main() {
  double *o; float *of; long long *c; cudaMalloc(&o, 8192 * 8); cudaMalloc(&of, 8192 * 4); cudaMallocManaged(&c, 64);
  int it = 4096;
  for (int bs : {32, 128, 512, 1024}) {
    probe<<<1, bs>>>(o, of, c, it); cudaDeviceSynchronize();
    printf("bs=%4d cyc/iter: dfma-chain %.1f  dmul+dfma-chain %.1f  ffma-chain %.1f  8x dfma indep %.1f (-> %.2f dfma/clk/SM)\n", bs,
           c[0] / (double)it, c[1] / (double)it, c[2] / (double)it, c[3] / (double)it, 8.0 * bs / (c[3] / (double)it));
  }
}
