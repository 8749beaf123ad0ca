// Dependent-chain latencies on one warp (B200): FFMA, DFMA, MUFU.RSQ (f32), rsqrt.approx.f64,
// SHFL.BFLY (32-bit), REDUX (u32 max), LDS (pointer chase), BAR.SYNC (8 warps), clock64 cost.
#include <cstdio>
__global__ void k(float *out, long long *cyc, int n) {
  __shared__ int nx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) nx[i] = (i * 37 + 11) & 1023;
  __syncthreads();
  float a = 1.0f + threadIdx.x * 1e-9f;
  double da = a;
  long long t[12];
  int c = 0;
  t[c++] = clock64();
  for (int i = 0; i < n; ++i) a = fmaf(a, 0.999f, 1e-7f);
  t[c++] = clock64();
  for (int i = 0; i < n; ++i) da = fma(da, 0.999, 1e-7);
  t[c++] = clock64();
  for (int i = 0; i < n; ++i) a = rsqrtf(a) + 0.5f;
  t[c++] = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(da)); da = r + 0.5; }
  t[c++] = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1) + 1e-7f;
  t[c++] = clock64();
  unsigned u = __float_as_uint(a);
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u) + (threadIdx.x & 1);
  t[c++] = clock64();
  int p = threadIdx.x;
  for (int i = 0; i < n; ++i) p = nx[p];
  t[c++] = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t[c++] = clock64();
  for (int i = 0; i < n; ++i) a = __fdividef(1.0f, a) + 0.5f;
  t[c++] = clock64();
  long long s = 0;
  for (int i = 0; i < n; ++i) s += clock64();
  t[c++] = clock64();
  out[threadIdx.x] = a + (float)da + (float)u + p + (float)s;
  if (threadIdx.x == 0)
    for (int i = 0; i + 1 < c; ++i) cyc[i] = t[i + 1] - t[i];
}
int main() {
  float *o; long long *cy;
  cudaMalloc(&o, 4096); cudaMallocManaged(&cy, 8 * 16);
  const char *nm[] = {"FFMA", "DFMA", "MUFU.RSQ f32", "rsqrt.approx.f64", "SHFL.BFLY", "REDUX.MAX", "LDS chase",
                      "BAR.SYNC 8w", "fdividef", "clock64"};
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 256>>>(o, cy, 256);
    cudaDeviceSynchronize();
  }
  for (int i = 0; i < 10; ++i) printf("%-18s %.1f cyc\n", nm[i], cy[i] / 256.0);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
