// Per-round latency breakdown of the Jacobi eig kernel (thread 0 clock64 stamps).
#include <cstdio>
__device__ long long g_probe[8];
__shared__ long long s_probe[8];
#define RT_EIG_PROBE(k) do { if (threadIdx.x == 0) { long long t_ = clock64(); if (k == 0) s_probe[7] = t_; else s_probe[k] += t_ - s_probe[7]; s_probe[7] = t_; if (k == 4) for (int i_ = 1; i_ < 5; ++i_) g_probe[i_] = s_probe[i_]; } } while (0)
#define RT_EIG_PROBE_INIT() do { if (threadIdx.x < 8) s_probe[threadIdx.x] = 0; } while (0)
#include "../../paper_1905_07311_b200/csrc/smallla.cu"
#include <vector>
#include <cmath>
int main() {
  int n = 60, np = 60;
  std::vector<double> a(n * n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) a[i + n * j] = 1.0 / (i + j + 1.0);  // Hilbert
  double *dA, *w, *V; int *info;
  cudaMalloc(&dA, 8 * n * n); cudaMalloc(&w, 8 * n); cudaMalloc(&V, 8 * n * n); cudaMallocManaged(&info, 4);
  cudaMemcpy(dA, a.data(), 8 * n * n, cudaMemcpyHostToDevice);
  size_t need = 8 * (2 * np * np + np) + 4 * (np - 1) * (np / 2) + 16;
  cudaFuncSetAttribute(rt::jacobi_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
  cudaFuncSetAttribute(rt::jacobi_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
  cudaFuncSetAttribute(rt::jacobi_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
  for (int rep = 0; rep < 3; ++rep) {
    long long z[8] = {0};
    cudaMemcpyToSymbol(g_probe, z, sizeof z);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    if (rep == 0) rt::jacobi_kernel<8, true><<<1, 256, need>>>(dA, n, w, V, nullptr, 2.3e-14, 40, info);
    if (rep == 1) rt::jacobi_kernel<16, true><<<1, 480, need>>>(dA, n, w, V, nullptr, 2.3e-14, 40, info);
    if (rep == 2) rt::jacobi_kernel<32, true><<<1, 960, need>>>(dA, n, w, V, nullptr, 2.3e-14, 40, info);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[8]; cudaMemcpyFromSymbol(h, g_probe, sizeof h);
    int rounds = *info * (np - 1);
    printf("err=%s sweeps=%d time=%.1f us; per round cycles: dot %.0f rot %.0f upd %.0f sync %.0f\n",
           cudaGetErrorString(cudaGetLastError()), *info, ms * 1e3, h[1] / (double)rounds, h[2] / (double)rounds,
           h[3] / (double)rounds, h[4] / (double)rounds);
  }
}
