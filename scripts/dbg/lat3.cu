// Dependent-chain latencies on one warp: DFMA, FFMA, LDS.64 (pointer chase), SHFL (64-bit),
// fp64 div / sqrt, MUFU.RCP64H.
#include <cstdio>
__global__ void k(double *out, long long *cyc, int n) {
  __shared__ double sm[1024];
  __shared__ int nx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; nx[i] = (i * 37 + 11) & 1023; }
  __syncthreads();
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999, c = 1e-7;
  float fa = a, fb = b, fc = c;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) fa = fmaf(fa, fb, fc);
  long long t2 = clock64();
  int p = threadIdx.x;
  double acc = 0;
  for (int i = 0; i < n; ++i) { p = nx[p]; }
  long long t3 = clock64();
  double x = a;
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * 1.0000001;
  long long t4 = clock64();
  double y = a + 2.0;
  for (int i = 0; i < n; ++i) y = 1.0 / y + 1.5;
  long long t5 = clock64();
  double z = a + 2.0;
  for (int i = 0; i < n; ++i) z = sqrt(z) + 1.5;
  long long t6 = clock64();
  double q = 0;
  for (int i = 0; i < n; ++i) { q += sm[p]; p = (int)q & 1023; }
  long long t7 = clock64();
  out[threadIdx.x] = a + fa + p + x + y + z + q + acc;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n; cyc[3] = (t4 - t3) / n;
    cyc[4] = (t5 - t4) / n; cyc[5] = (t6 - t5) / n; cyc[6] = (t7 - t6) / n;
  }
}
int main() {
  double *o; long long *c, h[7];
  cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 1000);
  k<<<1, 32>>>(o, c, 1000);
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  printf("DFMA %lld  FFMA %lld  LDS.32 chase %lld  SHFL64+DMUL %lld  div+add %lld  sqrt+add %lld  LDS.64+DADD chase %lld (cycles)\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
}
