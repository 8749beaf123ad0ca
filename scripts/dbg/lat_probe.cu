// Latency probe: cycles per __syncthreads round (1024 thr), fp64 sqrt/div chain, shfl chain.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double *out, long long *cyc, int iters, double seed) {
  __shared__ double s[64];
  double x = seed + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x * 1.0000001 + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 2.0);
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) { s[threadIdx.x & 63] = x; __syncthreads(); x += s[(threadIdx.x + 1) & 63]; __syncthreads(); }
  long long t5 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
  out[threadIdx.x] = x;
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 8192); cudaMallocManaged(&c, 64);
  int it = 1000;
  for (int bs : {32, 256, 1024}) {
    probe<<<1, bs>>>(o, c, it, 1.0); cudaDeviceSynchronize();
    printf("bs=%d cyc/iter: sync %.1f sqrt %.1f div %.1f shfl %.1f smem+2sync %.1f\n", bs, c[0] / (double)it,
           c[1] / (double)it, c[2] / (double)it, c[3] / (double)it, c[4] / (double)it);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock %d kHz\n", clk);
}
