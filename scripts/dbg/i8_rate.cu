// Issue-rate probe for tcgen05.mma kind::i8 from one thread: R MMAs back to back on the same
// smem operands (K-major, no swizzle), M = 128, N in {64, 128, 256}, one commit at the end.
#include <cstdio>
#include <cstdint>
#include "../../paper_1905_07311_b200/csrc/tc.cuh"
using namespace rt;
__host__ __device__ constexpr uint32_t idesc_s8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void mma_i8_ta(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
template <int N, bool TA>
__global__ void rate(long long *out, int R) {
  __shared__ __align__(1024) int8_t sa[128 * 32];
  __shared__ __align__(1024) int8_t sb[256 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 32; i += blockDim.x) sa[i] = (int8_t)(i % 7 - 3);
  for (int i = t; i < 256 * 32; i += blockDim.x) sb[i] = (int8_t)(i % 5 - 2);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (t == 0) {
    const uint64_t ad = tc::smem_desc(tc::smem_u32(sa), 128, 256, tc::kSwNone);
    const uint64_t bd = tc::smem_desc(tc::smem_u32(sb), 128, 256, tc::kSwNone);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      if (TA) mma_i8_ta(slot, slot + 256, bd, idesc_s8(128, N), r > 0);
      else mma_i8(slot, ad, bd, idesc_s8(128, N), r > 0);
    }
    tc::mma_commit(&bar);
    long long t1 = clock64();
    tc::mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(slot, 512);
}
int main() {
  long long *o, h[2];
  cudaMalloc(&o, 16);
  const int R = 4096;
  rate<64, false><<<148, 128>>>(o, R); cudaDeviceSynchronize();
  rate<64, false><<<148, 128>>>(o, R); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("N=64 : issue %.1f cyc/MMA, complete %.1f cyc/MMA -> %.0f MAC/clk/SM\n", (double)h[0] / R, (double)h[1] / R, 128.0 * 64 * 32 * R / h[1]);
  rate<128, false><<<148, 128>>>(o, R); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("N=128: issue %.1f cyc/MMA, complete %.1f cyc/MMA -> %.0f MAC/clk/SM\n", (double)h[0] / R, (double)h[1] / R, 128.0 * 128 * 32 * R / h[1]);
  rate<256, false><<<148, 128>>>(o, R); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("N=256: issue %.1f cyc/MMA, complete %.1f cyc/MMA -> %.0f MAC/clk/SM\n", (double)h[0] / R, (double)h[1] / R, 128.0 * 256 * 32 * R / h[1]);
  rate<64, true><<<148, 128>>>(o, R); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("TMEM-A N=64 : issue %.1f cyc/MMA, complete %.1f cyc/MMA -> %.0f MAC/clk/SM\n", (double)h[0] / R, (double)h[1] / R, 128.0 * 64 * 32 * R / h[1]);
  rate<128, true><<<148, 128>>>(o, R); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("TMEM-A N=128: issue %.1f cyc/MMA, complete %.1f cyc/MMA -> %.0f MAC/clk/SM\n", (double)h[0] / R, (double)h[1] / R, 128.0 * 128 * 32 * R / h[1]);
  return 0;
}
