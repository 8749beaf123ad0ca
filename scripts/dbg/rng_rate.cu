// Measured generation rate of the library's Omega entries (Philox4x32-10 + Box-Muller, fp32 and
// fp64, philox.cuh) on the whole GPU: the input of the fused all-mode R-HOSVD sketch model
// (DESIGN §13).  Each thread generates `per` Philox blocks (4 normals each) for consecutive
// columns and keeps a checksum so nothing is optimised away.
#include <cstdio>
#include "../../paper_1905_07311_b200/csrc/philox.cuh"
template <typename T>
__global__ void gen(int per, double *out) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (int j = 0; j < per; ++j) {
    const uint4 w = rt::omega_words(12345, 1, 0, t * per + j, 3);
    rt::Normal4<T> z(w);
    acc += (double)z.v[0] + (double)z.v[1] + (double)z.v[2] + (double)z.v[3];
  }
  if (acc == 1.2345) out[0] = acc;  // practically never true
}
int main() {
  double *d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, per = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int prec = 0; prec < 2; ++prec) {
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(a);
      if (prec == 0) gen<float><<<blocks, threads>>>(per, d);
      else gen<double><<<blocks, threads>>>(per, d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double normals = 4.0 * per * blocks * (double)threads;
    printf("%s normals: %.3e per s (%.3f ms for %.3e)\n", prec ? "fp64" : "fp32", normals / (ms * 1e-3), ms, normals);
  }
  return 0;
}
