// __syncthreads cost per iteration for 256 / 512 threads: (0) barrier only, (1) one fp64 FMA
// chain of 8 + barrier, (2) thread t writes smem, barrier, reads a neighbour's value, (3) as (2)
// plus a rsqrt(double) on one warp (the Cholesky/QR step shape).
#include <cstdio>
template <int MODE>
__global__ void k(long long *out, double *sink, int iters) {
  __shared__ double sm[1024];
  double x = 1.0 + threadIdx.x * 1e-9;
  sm[threadIdx.x] = x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE >= 1) {
#pragma unroll
      for (int u = 0; u < 8; ++u) x = fma(x, 1.0000001, 1e-9);
    }
    if (MODE == 3 && threadIdx.x < 32) x = rsqrt(x * x + 1.0);
    if (MODE >= 2) sm[threadIdx.x] = x;
    __syncthreads();
    if (MODE >= 2) x += sm[(threadIdx.x + 37) % blockDim.x] * 1e-12;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[MODE] = (t1 - t0) / iters;
  sink[threadIdx.x] = x;
}
int main() {
  long long *o, h[4];
  double *s;
  cudaMalloc(&o, 64); cudaMalloc(&s, 8192);
  for (int nt : {64, 256, 512}) {
    k<0><<<1, nt>>>(o, s, 2000); k<1><<<1, nt>>>(o, s, 2000); k<2><<<1, nt>>>(o, s, 2000); k<3><<<1, nt>>>(o, s, 2000);
    cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
    printf("threads %3d: barrier %lld, fma8+barrier %lld, +smem exchange %lld, +rsqrt warp %lld cycles/iter\n", nt, h[0], h[1], h[2], h[3]);
  }
  return 0;
}
