// Single-MMA probe of the tcgen05 kind::tf32 path: A 128x8 (MN-major SW128, written by
// threads with the swizzle formula), B 32x8 (K-major, no swizzle), D read back via tcgen05.ld.
#include <cstdio>
#include <cstdint>
#include "../../paper_1905_07311_b200/csrc/tc.cuh"
using namespace rt;
__global__ void probe(const float *A, const float *B, float *D, int mode, int var) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  unsigned char *sa = dyn + ((1024u - ((uint32_t)__cvta_generic_to_shared(dyn) & 1023u)) & 1023u);
  __shared__ __align__(1024) unsigned char sb[1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // zero the operand area first (an earlier version zeroed it AFTER writing A: every mode read 0)
  for (int idx = t; idx < 190 * 1024 / 4; idx += blockDim.x) ((float *)sa)[idx] = 0.f;
  __syncthreads();
  // A(m, k) m<128, k<8: atom a = m/32, row r = k, 16B chunk j = (m%32)/4, within-chunk e = m%4
  for (int idx = t; idx < 128 * 8; idx += blockDim.x) {
    int m = idx % 128, k = idx / 128;
    int a = m / 32, j = (m % 32) / 4, e = m % 4;
    int off = a * 1024 + k * 128 + ((j ^ (k % 8)) * 16) + e * 4;
    *(float *)(sa + off) = A[m + 128 * k];
  }
  if (mode == 4) {  // A K-major, no swizzle: (m/8)*256 + (k/4)*128 + (m%8)*16 + (k%4)*4
    for (int idx = t; idx < 128 * 8; idx += blockDim.x) {
      int m = idx % 128, k = idx / 128;
      *(float *)(sa + (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4) = A[m + 128 * k];
    }
  }
  if (mode == 5 || mode == 6) {  // A MN-major, no swizzle: (m/4)*128 + k*16 + (m%4)*4
    for (int idx = t; idx < 128 * 8; idx += blockDim.x) {
      int m = idx % 128, k = idx / 128;
      *(float *)(sa + (m / 4) * 128 + k * 16 + (m % 4) * 4) = A[m + 128 * k];
    }
  }
  // B(n, k) n<32, k<8: (n/8)*256 + (k/4)*128 + (n%8)*16 + (k%4)*4
  for (int idx = t; idx < 32 * 8; idx += blockDim.x) {
    int n = idx % 32, k = idx / 32;
    *(float *)(sb + (n / 8) * 256 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4) = B[n + 32 * k];
  }
  if (mode == 9) {  // B MN-major no swizzle: (n/4)*128 + k*16 + (n%4)*4
    for (int idx = t; idx < 32 * 8; idx += blockDim.x) {
      int n = idx % 32, k = idx / 32;
      *(float *)(sb + (n / 4) * 128 + k * 16 + (n % 4) * 4) = B[n + 32 * k];
    }
  }
  if (mode == 10) {  // B MN-major SW128 atom: row k (128 B) holds n 0..31, chunk j = n/4 swizzled
    for (int idx = t; idx < 32 * 8; idx += blockDim.x) {
      int n = idx % 32, k = idx / 32;
      *(float *)(sb + k * 128 + (((n / 4) ^ (k % 8)) * 16) + (n % 4) * 4) = B[n + 32 * k];
    }
  }
  if (mode == 15) {  // A MN-major SWIZZLE_128B_BASE32B (CUTLASS Layout_MN_SW128_32B_Atom): atom = 4 k-rows x
    // 128 B (32 m), 32-byte chunk c = (m % 32) / 8 stored at c ^ (k % 4); atoms along m at LBO = 512,
    // k-groups of 4 at SBO = 2048
    for (int idx = t; idx < 128 * 8; idx += blockDim.x) {
      int m = idx % 128, k = idx / 128;
      int off = (m / 32) * 512 + (k / 4) * 2048 + (k % 4) * 128 + ((((m % 32) / 8) ^ (k % 4)) * 32) + (m % 8) * 4;
      *(float *)(sa + off) = A[m + 128 * k];
    }
  }
  if (mode == 16) {  // B MN-major SWIZZLE_128B_BASE32B: n < 32 = one atom along n, k-groups at SBO = 512
    for (int idx = t; idx < 32 * 8; idx += blockDim.x) {
      int n = idx % 32, k = idx / 32;
      *(float *)(sb + (k / 4) * 512 + (k % 4) * 128 + ((((n % 32) / 8) ^ (k % 4)) * 32) + (n % 8) * 4) = B[n + 32 * k];
    }
  }
  if (mode >= 9 && mode != 15) {  // A K-major no swizzle
    for (int idx = t; idx < 128 * 8; idx += blockDim.x) {
      int m = idx % 128, k = idx / 128;
      *(float *)(sa + (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4) = A[m + 128 * k];
    }
  }
  __syncthreads();
  if (mode == 14) {  // truncation test, K-major no swizzle: A(0,0) = 1+2^-11+2^-13, B(n,0) = 1
    for (int idx = t; idx < 128 * 8; idx += blockDim.x) {
      int m = idx % 128, k = idx / 128;
      float v = (m == 0 && k == 0) ? 1.0f + 0x1p-11f + 0x1p-13f : ((m == 1 && k == 0) ? -(1.0f + 0x1p-11f + 0x1p-13f) : 0.f);
      *(float *)(sa + (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4) = v;
    }
    for (int idx = t; idx < 32 * 8; idx += blockDim.x) { int n = idx % 32, k = idx / 32;
      *(float *)(sb + (n / 8) * 256 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4) = (k == 0) ? 1.f : 0.f; }
  }
  if (mode == 13 && var < 2) {  // A K-major SW128, K slice 0
    for (int idx = t; idx < 128 * 32; idx += blockDim.x) {
      int m = idx % 128, k = idx / 128;
      float v = (k < 8) ? A[m + 128 * k] : 1e30f;
      *(float *)(sa + m * 128 + (((k / 4) ^ (m % 8)) * 16) + (k % 4) * 4) = v;
    }
  }
  if (mode == 13 && var >= 2) {  // A K-major SW32: row m = 32 B, chunk j ^ ((m >> 2) & 1)
    for (int idx = t; idx < 128 * 8; idx += blockDim.x) {
      int m = idx % 128, k = idx / 128;
      *(float *)(sa + m * 32 + (((k / 4) ^ ((m >> 2) & 1)) * 16) + (k % 4) * 4) = A[m + 128 * k];
    }
  }
  if (mode == 11 || mode == 12) {  // A K-major SW128: row m = 128 B (32 k), chunk j ^ (m % 8); K slice 1 = k 8..15
    for (int idx = t; idx < 128 * 32; idx += blockDim.x) {
      int m = idx % 128, k = idx / 128;
      float v = (k >= 8 && k < 16) ? A[m + 128 * (k - 8)] : 1e30f;
      if (mode == 12) v = (k == 8) ? 1.0f + 0x1p-11f + 0x1p-13f : 0.f;
      *(float *)(sa + m * 128 + (((k / 4) ^ (m % 8)) * 16) + (k % 4) * 4) = v;
    }
    if (mode == 12) for (int idx = t; idx < 32 * 8; idx += blockDim.x) { int n = idx % 32, k = idx / 32;
      *(float *)(sb + (n / 8) * 256 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4) = (k == 0) ? 1.f : 0.f; }
  }
  if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&slot, 64);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  uint32_t tm = slot;
  if (t == 0) {
    uint64_t ad = tc::smem_desc(tc::smem_u32(sa), 1024, 4096, tc::kSw128);
    uint64_t bd = tc::smem_desc(tc::smem_u32(sb), 128, 256, tc::kSwNone);
    if (mode == 1) bd = tc::smem_desc(tc::smem_u32(sb), 256, 128, tc::kSwNone);
    if (mode == 2) ad = tc::smem_desc(tc::smem_u32(sa), 4096, 1024, tc::kSw128);
    if (mode == 4) ad = tc::smem_desc(tc::smem_u32(sa), 128, 256, tc::kSwNone);
    if (mode == 5) ad = tc::smem_desc(tc::smem_u32(sa), 1024, 128, tc::kSwNone);
    if (mode == 6) ad = tc::smem_desc(tc::smem_u32(sa), 128, 1024, tc::kSwNone);
    if (mode == 7) ad = tc::smem_desc(tc::smem_u32(sa), 1024, 1024, tc::kSw128);
    if (mode == 15) {
      ad = tc::smem_desc(tc::smem_u32(sa), 512, 2048, 1u);
      tc::mma_tf32(tm, ad, bd, tc::idesc_tf32(128, 32, true, false), 0);
    }
    if (mode == 16) {
      ad = tc::smem_desc(tc::smem_u32(sa), 128, 256, tc::kSwNone);
      bd = tc::smem_desc(tc::smem_u32(sb), 512, 512, 1u);
      tc::mma_tf32(tm, ad, bd, tc::idesc_tf32(128, 32, false, true), 0);
    }
    if (mode >= 9 && mode <= 10) {
      ad = tc::smem_desc(tc::smem_u32(sa), 128, 256, tc::kSwNone);
      bd = mode == 9 ? tc::smem_desc(tc::smem_u32(sb), 1024, 128, tc::kSwNone) : tc::smem_desc(tc::smem_u32(sb), 1024, 1024, tc::kSw128);
      tc::mma_tf32(tm, ad, bd, tc::idesc_tf32(128, 32, false, true), 0);
    }
    if (mode == 14) {
      ad = tc::smem_desc(tc::smem_u32(sa), 128, 256, tc::kSwNone);
      tc::mma_tf32(tm, ad, bd, tc::idesc_tf32(128, 32, false, false), 0);
    }
    if (mode == 13) {
      if (var == 0) ad = tc::smem_desc(tc::smem_u32(sa), 16, 1024, tc::kSw128);
      if (var == 1) ad = tc::smem_desc(tc::smem_u32(sa), 0, 1024, tc::kSw128);
      if (var == 2) ad = tc::smem_desc(tc::smem_u32(sa), 16, 256, tc::kSw32);
      if (var == 3) ad = tc::smem_desc(tc::smem_u32(sa), 0, 256, tc::kSw32);
      tc::mma_tf32(tm, ad, bd, tc::idesc_tf32(128, 32, false, false), 0);
    }
    if (mode == 11 || mode == 12) {
      ad = tc::smem_desc(tc::smem_u32(sa) + 32, 16, 1024, tc::kSw128);
      tc::mma_tf32(tm, ad, bd, tc::idesc_tf32(128, 32, false, false), 0);
    }
    if (mode != 3 && mode != 8 && mode < 9 && mode != 13 && mode != 14) tc::mma_tf32(tm, ad, bd, tc::idesc_tf32(128, 32, mode != 4, false), 0);
    tc::mma_commit(&bar);
  }
  if (mode == 8) {
    // A(m, k): thread = row m (warp w -> lanes 32w..), 8 columns at tm + 32
    uint32_t v[8];
    for (int k = 0; k < 8; ++k) v[k] = __float_as_uint(A[(32 * warp + lane) + 128 * k]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::
                 "r"(tm + 32 + ((uint32_t)(32 * warp) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (t == 0) {
      uint64_t bd = tc::smem_desc(tc::smem_u32(sb), 128, 256, tc::kSwNone);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(tm + 32), "l"(bd),
                   "r"(tc::idesc_tf32(128, 32, false, false)) : "memory");
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
  } else if (mode == 3) {
    uint32_t v = __float_as_uint((float)(lane + 1000 * warp));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(tm + ((uint32_t)(32 * warp) << 16)), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else {
    tc::mbar_wait(&bar, 0);
  }
  tc::tc_fence_after();
  uint32_t r[32];
  tc::tmem_ld32(tm + ((uint32_t)(32 * warp) << 16), r);
  for (int j = 0; j < 32; ++j) D[(32 * warp + lane) + 128 * j] = __uint_as_float(r[j]);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 64);
}
int main(int argc, char **argv) {
  float hA[128 * 8], hB[32 * 8], hD[128 * 32], ref[128 * 32];
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)((i * 7) % 13) - 6.f;
  for (int i = 0; i < 32 * 8; ++i) hB[i] = (float)((i * 5) % 11) - 5.f;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < 32; ++n) { double s = 0; for (int k = 0; k < 8; ++k) s += hA[m + 128 * k] * hB[n + 32 * k]; ref[m + 128 * n] = s; }
  float *A, *B, *D; cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  for (int mode = atoi(argv[1]); mode <= atoi(argv[1]); ++mode) {
    cudaMemset(D, 0, sizeof hD);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    probe<<<1, 128, 200 * 1024>>>(A, B, D, mode, argc > 2 ? atoi(argv[2]) : 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0; int bad = 0;
    for (int i = 0; i < 128 * 32; ++i) { double d = fabs(hD[i] - ref[i]); if (d > maxerr) maxerr = d; if (fabs(ref[i]) > maxref) maxref = fabs(ref[i]); if (d > 1e-3) ++bad; }
    if (mode == 14) { printf("trunc test: D[0]=%.9g D[1]=%.9g (1=truncation, %.9g=round-nearest)\n", hD[0], hD[1], 1.0 + 1.0 / 1024); continue; }
    if (mode == 12) { printf("trunc test: D[0]=%.9g (1=truncation, %.9g=round-nearest)\n", hD[0], 1.0 + 1.0 / 1024); continue; }
    printf("mode %d err=%s maxerr=%g maxref=%g bad=%d  D[0..3]=%g %g %g %g ref=%g %g %g %g D[128]=%g ref=%g\n", mode, cudaGetErrorString(e), maxerr, maxref, bad,
           hD[0], hD[1], hD[2], hD[3], ref[0], ref[1], ref[2], ref[3], hD[128], ref[128]);
  }
}
