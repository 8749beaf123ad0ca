// Phase profile of trid_eig_kernel (clock64 at phase boundaries) and event timing, n = argv[1].
#define RT_TRID_PROGRESS
#include "../../paper_1905_07311_b200/csrc/trideig.cu"
#include <cstdio>
#include <vector>
#include <random>
int main(int argc, char **argv) {
  int n = argc > 1 ? atoi(argv[1]) : 60;
  std::vector<double> a(n * n), b(n * n);
  std::mt19937 g(1);
  std::normal_distribution<double> nd;
  for (auto &v : b) v = nd(g);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < n; ++k) s += b[i + n * k] * b[j + n * k] * std::pow(k + 1.0, -3.0); a[i + n * j] = s; }
  double *dA, *dw, *dV; int *dinfo;
  cudaMalloc(&dA, 8 * n * n); cudaMalloc(&dw, 8 * n); cudaMalloc(&dV, 8 * n * n); cudaMalloc(&dinfo, 4);
  cudaMemcpy(dA, a.data(), 8 * n * n, cudaMemcpyHostToDevice);
  int *hp; cudaHostAlloc(&hp, 4, cudaHostAllocMapped);
  int *dp; cudaHostGetDevicePointer(&dp, hp, 0);
  cudaMemcpyToSymbol(rt::g_trid_progress, &dp, sizeof dp);
  size_t smem = rt::trid_eig_smem();
  cudaFuncSetAttribute(rt::trid_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) rt::trid_eig_kernel<<<1, 1024, smem>>>(dA, n, dw, dV, dinfo);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it) rt::trid_eig_kernel<<<1, 1024, smem>>>(dA, n, dw, dV, dinfo);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c[8]; cudaMemcpyFromSymbol(c, rt::g_trid_clk, sizeof c);
  printf("n=%d  %.1f us/launch  cycles: tridiag %lld  bisect %lld  vectors+GS %lld  NS+out %lld  (total %lld) err=%s\n", n,
         ms * 1000 / 20, c[2] - c[1], c[3] - c[2], c[4] - c[3], c[5] - c[4], c[5] - c[0], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
