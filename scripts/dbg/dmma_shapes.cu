// fp64 mma.sync shape throughput with ONE warp per SMSP (4 warps per CTA, 1 CTA per SM),
// NC independent accumulator chains: m8n8k4 (256 FMA), m16n8k4 (512), m16n8k8 (1024),
// m16n8k16 (2048 FMA per instruction).
#include <cstdio>
template <int SHAPE, int NC>
__global__ void k(double *out, int iters) {
  double a[8], b[4], c[NC][4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
  for (int i = 0; i < 4; ++i) b[i] = 0.999 + i * 1e-3;
  for (int j = 0; j < NC; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int j = 0; j < NC; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int SHAPE, int NC>
void run(double *o, int warps) {
  const int it = 4000;
  const double fma_per[4] = {256, 512, 1024, 2048};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<SHAPE, NC><<<148, 32 * warps>>>(o, 10); cudaDeviceSynchronize();
  cudaEventRecord(e0); k<SHAPE, NC><<<148, 32 * warps>>>(o, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * fma_per[SHAPE] * NC * (double)it * 148 * warps;
  printf("shape %d chains %d warps/SM %2d: %6.1f TFLOP/s  (%.1f cycles per instr per warp @1.965GHz)\n", SHAPE, NC, warps,
         fl / ms / 1e9, ms * 1e-3 * 1.965e9 / (it * NC));
}
int main() {
  double *o; cudaMalloc(&o, 148 * 1024 * 8);
  run<0, 3>(o, 4); run<0, 9>(o, 4); run<0, 8>(o, 8);
  run<1, 3>(o, 4); run<1, 8>(o, 4);
  run<2, 3>(o, 4); run<2, 8>(o, 4);
  run<3, 3>(o, 4); run<3, 8>(o, 4); run<3, 4>(o, 8);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
