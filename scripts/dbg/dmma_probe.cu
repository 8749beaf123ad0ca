// DMMA (mma.sync m8n8k4 f64) vs DFMA throughput per SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma(double *out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma(double *out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(a, b, c[i]);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// half the warps issue DMMA, the other half DFMA: do the two pipes overlap?
__global__ void mixed(double *out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double s = 0;
  if ((threadIdx.x >> 5) & 1) {
    double c[8][2];
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double c[16];
    for (int i = 0; i < 16; ++i) c[i] = i;
    for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) c[i] = fma(a, b, c[i]);
    }
    for (int i = 0; i < 16; ++i) s += c[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double *o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int it = 20000;
  for (int warps : {4, 8, 16, 32}) {
    dmma<<<148 * 2, 32 * warps>>>(o, 10); cudaDeviceSynchronize();
    cudaEventRecord(e0); dmma<<<148 * 2, 32 * warps>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)it * 148 * 2 * warps;  // 8x8x4 = 256 FMA per mma per warp
    printf("DMMA warps/CTA=%d: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
    dfma<<<148 * 2, 32 * warps>>>(o, 10); cudaDeviceSynchronize();
    cudaEventRecord(e0); dfma<<<148 * 2, 32 * warps>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * (double)it * 148 * 2 * warps * 32;
    printf("DFMA warps/CTA=%d: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
    mixed<<<148 * 2, 32 * warps>>>(o, 10); cudaDeviceSynchronize();
    cudaEventRecord(e0); mixed<<<148 * 2, 32 * warps>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    // per DMMA warp: 8 mma x 256 FMA per iter; per DFMA warp: 8 x 16 x 32 FMA per iter (equal work)
    flops = 2.0 * 2048 * (double)it * 148 * 2 * warps;
    printf("MIXED warps/CTA=%d: %.1f TFLOP/s (half DMMA, half DFMA, equal work)\n", warps, flops / ms / 1e9);
  }
}
