// Probe of tcgen05.mma kind::i8 (signed int8 x int8 -> int32 in TMEM): A 128 x 32 and B 64 x 32,
// both K-major without swizzle (core matrices of 8 rows x 16 B, LBO = 128 B along K, SBO =
// 256 B along M/N), two MMAs accumulated (K = 64 in total).  Checks D against the exact
// integer product.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../../paper_1905_07311_b200/csrc/tc.cuh"
using namespace rt;

__host__ __device__ constexpr uint32_t idesc_s8(int M, int N) {
  // [4,6) D format 2 = s32; [7,10) A format 1 = signed 8-bit; [10,13) B format 1; K-major both
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
// K-major no-swizzle byte offset of (row r, k) in a [rows][32] int8 tile
__host__ __device__ inline int kmaj8(int r, int k) { return (r / 8) * 256 + (k / 16) * 128 + (r % 8) * 16 + (k % 16); }

__device__ __forceinline__ void mma_i8_ta(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__global__ void probe(const int8_t *A, const int8_t *B, int *D, int tmemA) {
  __shared__ __align__(1024) int8_t sa[2][128 * 32];
  __shared__ __align__(1024) int8_t sb[2][64 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int h = 0; h < 2; ++h) {
    for (int idx = t; idx < 128 * 32; idx += blockDim.x) { int m = idx / 32, k = idx % 32; sa[h][kmaj8(m, k)] = A[m * 64 + 32 * h + k]; }
    for (int idx = t; idx < 64 * 32; idx += blockDim.x) { int n = idx / 32, k = idx % 32; sb[h][kmaj8(n, k)] = B[n * 64 + 32 * h + k]; }
  }
  if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&slot, 128);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = slot;
  if (tmemA) {  // A rows -> TMEM columns 64 + 8 h .. : lane m, column c = bytes k 4c..4c+3
    const int m = 32 * warp + lane;
    for (int h = 0; h < 2; ++h) {
      uint32_t v[8];
      for (int c = 0; c < 8; ++c) {
        uint32_t w = 0;
        for (int b = 0; b < 4; ++b) w |= (uint32_t)(uint8_t)A[m * 64 + 32 * h + 4 * c + b] << (8 * b);
        v[c] = w;
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::
                   "r"(tm + 64 + 8 * h + ((uint32_t)(32 * warp) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),
                   "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
  }
  if (t == 0) {
    for (int h = 0; h < 2; ++h) {
      const uint64_t ad = tc::smem_desc(tc::smem_u32(sa[h]), 128, 256, tc::kSwNone);
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sb[h]), 128, 256, tc::kSwNone);
      if (tmemA) mma_i8_ta(tm, tm + 64 + 8 * h, bd, idesc_s8(128, 64), h);
      else mma_i8(tm, ad, bd, idesc_s8(128, 64), h);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  for (int half = 0; half < 2; ++half) {
    uint32_t r[32];
    tc::tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + 32 * half, r);
    for (int j = 0; j < 32; ++j) D[(32 * warp + lane) * 64 + 32 * half + j] = (int)r[j];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 128);
}

int main() {
  static int8_t hA[128 * 64], hB[64 * 64];
  static int hD[128 * 64];
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (int)((s >> 8) % 255) - 127; };
  for (auto &x : hA) x = (int8_t)rnd();
  for (auto &x : hB) x = (int8_t)rnd();
  int8_t *A, *B; int *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  int tmemA = 1;
  probe<<<1, 128>>>(A, B, D, tmemA);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      long ref = 0;
      for (int k = 0; k < 64; ++k) ref += (long)hA[m * 64 + k] * hB[n * 64 + k];
      if (ref != hD[m * 64 + n]) { if (bad < 5) printf("m=%d n=%d got %d ref %ld\n", m, n, hD[m * 64 + n], ref); ++bad; }
    }
  printf("i8 probe (A in TMEM=%d): %s, mismatches %ld of %d (D[0]=%d)\n", tmemA, cudaGetErrorString(e), bad, 128 * 64, hD[0]);
  return 0;
}
