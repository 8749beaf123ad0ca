// Where does TMA (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) put element (i, c) of a 32 (i, inner) x 8 (c)
// fp32 box?  Prints, for each c, the 32-byte chunk holding i = 0, 8, 16, 24, to compare with the
// UMMA SWIZZLE_128B_BASE32B layout (chunk j of K-row k at j ^ (k % 4), 128 B per K-row).
// Then runs one tcgen05 tf32 MMA with that TMA-loaded tile as an MN-major A (M = 128: 4 boxes).
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../../paper_1905_07311_b200/csrc/tc.cuh"
using namespace rt;
__global__ void k(const __grid_constant__ CUtensorMap tm, float *out, const float *B, float *D, int mode) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  unsigned char *sa = dyn + ((1024u - ((uint32_t)__cvta_generic_to_shared(dyn) & 1023u)) & 1023u);
  __shared__ __align__(1024) unsigned char sb[1024];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int e = t; e < 8192; e += blockDim.x) ((float *)sa)[e] = -1.f;
  // B (n, k) n < 32, k < 8: K-major no swizzle
  for (int idx = t; idx < 32 * 8; idx += blockDim.x) {
    int n = idx % 32, kk = idx / 32;
    *(float *)(sb + (n / 8) * 256 + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4) = B[n + 32 * kk];
  }
  if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&bar2, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&slot, 32);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (t == 0) {
    tc::mbar_arrive_expect_tx(&bar, 4 * 32 * 8 * 4);
    for (int b = 0; b < 4; ++b) tc::tma_load_2d(sa + 1024 * b, &tm, &bar, 32 * b, 0);
  }
  tc::mbar_wait(&bar, 0);
  for (int e = t; e < 1024; e += blockDim.x) out[e] = ((float *)sa)[e];
  tc::tc_fence_after();
  uint32_t tmv = slot;
  if (t == 0) {
    // A MN-major BASE32B: atoms of 4 K-rows x 128 B; K-group stride (SBO) 512, M-atom stride (LBO) 1024
    uint64_t ad = tc::smem_desc(tc::smem_u32(sa), 1024, 512, 1u);
    uint64_t bd = tc::smem_desc(tc::smem_u32(sb), 128, 256, tc::kSwNone);
    tc::mma_tf32(tmv, ad, bd, tc::idesc_tf32(128, 32, true, false), 0);
    tc::mma_commit(&bar2);
  }
  tc::mbar_wait(&bar2, 0);
  tc::tc_fence_after();
  uint32_t r[32];
  tc::tmem_ld32(tmv + ((uint32_t)(32 * warp) << 16), r);
  for (int j = 0; j < 32; ++j) D[(32 * warp + lane) + 128 * j] = __uint_as_float(r[j]);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmv, 32);
}
int main(int argc, char **argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 4;  // CUtensorMapSwizzle value
  const int I = 128, C = 8;
  float hX[I * C], hB[32 * 8], hD[128 * 32], hO[1024];
  for (int c = 0; c < C; ++c) for (int i = 0; i < I; ++i) hX[i + I * c] = (float)(i + 1000 * c);
  for (int e = 0; e < 256; ++e) hB[e] = (float)((e * 5) % 11) - 5.f;
  float *X, *B, *D, *O;
  cudaMalloc(&X, sizeof hX); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD); cudaMalloc(&O, sizeof hO);
  cudaMemcpy(X, hX, sizeof hX, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  void *ptr = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)I, (cuuint64_t)C};
  cuuint64_t strides[1] = {(cuuint64_t)I * 4};
  cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (CUtensorMapSwizzle)mode, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode(swizzle %d) = %d\n", mode, (int)r);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 64 * 1024>>>(tm, O, B, D, mode);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(hO, O, sizeof hO, cudaMemcpyDeviceToHost);
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  for (int c = 0; c < 8; ++c) {
    printf("c=%d:", c);
    for (int ch = 0; ch < 4; ++ch) { float v = hO[c * 32 + ch * 8]; printf(" chunk%d->i%d", ch, (int)v % 1000); }
    printf("\n");
  }
  double maxerr = 0; int bad = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < 32; ++n) {
    double s = 0; for (int kk = 0; kk < 8; ++kk) s += (double)hX[m + I * kk] * hB[n + 32 * kk];
    double d = fabs(hD[m + 128 * n] - s); if (d > maxerr) maxerr = d; if (d > 1e-2 * fabs(s) + 1e-3) ++bad;
  }
  printf("MMA from TMA tile (MN-major BASE32B): maxerr %g bad %d  D[0]=%g D[1]=%g\n", maxerr, bad, hD[0], hD[1]);
}
