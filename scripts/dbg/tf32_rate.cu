// Issue-rate probe for tcgen05.mma kind::tf32 from one thread: R MMAs back to back, M = 128,
// N in {64, 128, 256}, K = 8, A from smem or TMEM, one commit at the end (clock64 cycles).
#include <cstdio>
#include <cstdint>
#include "../../paper_1905_07311_b200/csrc/tc.cuh"
using namespace rt;
__device__ __forceinline__ void mma_ta(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
template <int N, bool TA, int KB>
__global__ void rate(long long *out, int R) {
  __shared__ __align__(1024) float sa[128 * 8 * KB];
  __shared__ __align__(1024) float sb[256 * 8 * KB];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 8 * KB; i += blockDim.x) sa[i] = (float)(i % 7 - 3);
  for (int i = t; i < 256 * 8 * KB; i += blockDim.x) sb[i] = (float)(i % 5 - 2);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (t == 0) {
    constexpr uint32_t id = tc::idesc_tf32(128, N, false, false);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      const int kb = r % KB;
      const uint64_t ad = tc::smem_desc(tc::smem_u32(sa + 128 * 8 * kb), 128, 256, tc::kSwNone);
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sb + 256 * 8 * kb), 128, 256, tc::kSwNone);
      if (TA) mma_ta(slot, slot + 256 + 8 * kb, bd, id, r > 0);
      else tc::mma_tf32(slot, ad, bd, id, r > 0);
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
// the sketch_tc_ta_kernel pattern: per stage 4 tiles x (Xhi*Bh, Xhi*Bl, Xlo*Bh), D tile t at
// column 64 t, A stage s of 4 at 256 + 16 (4 s + t)
__global__ void pattern(long long *out, int R, int ntile, int mode) {
  __shared__ __align__(1024) float sb[2 * 64 * 8 * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 2 * 64 * 8 * 4; i += blockDim.x) sb[i] = (float)(i % 5 - 2);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = slot;
  if (t == 0) {
    constexpr uint32_t id = tc::idesc_tf32(128, 64, false, false);
    long long t0 = clock64();
    for (int it = 0; it < R; ++it) {
      const int s = (mode & 1) ? (it & 3) : 0, g = (mode & 4) ? (it & 3) : 0;
      const uint64_t bh = tc::smem_desc(tc::smem_u32(sb + 64 * 8 * g), 128, 256, tc::kSwNone);
      const uint64_t bl = tc::smem_desc(tc::smem_u32(sb + 64 * 8 * (4 + g) - 64 * 8 * 4 + 64 * 8 * 4), 128, 256, tc::kSwNone);
      const uint32_t a0 = tb + 256 + 16 * s * ntile;
      #pragma unroll 1
      for (int tt = 0; tt < ntile; ++tt) {
        const uint32_t d = (mode & 64) ? tb : tb + 64 * tt, ah = a0 + 16 * tt;
        mma_ta(d, ah, bh, id, (mode & 32) ? 1u : (uint32_t)(it > 0));
        if (mode & 8) continue;
        mma_ta(d, ah, (mode & 4) ? bl : bh, id, 1u);
        if (mode & 16) continue;
        mma_ta(d, (mode & 2) ? ah + 8 : ah, bh, id, 1u);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t2 - t0; }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(slot, 512);
}
__device__ __forceinline__ void mma_ta_elect(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
// warp-wide issue loop (all lanes compute the same operands; elect.sync picks the issuer)
__global__ void pattern_w(long long *out, int R) {
  __shared__ __align__(1024) float sb[2 * 64 * 8 * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 2 * 64 * 8 * 4; i += blockDim.x) sb[i] = (float)(i % 5 - 2);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = __shfl_sync(0xffffffffu, slot, 0);
  if (warp == 0) {
    constexpr uint32_t id = tc::idesc_tf32(128, 64, false, false);
    const uint32_t sbase = __shfl_sync(0xffffffffu, tc::smem_u32(sb), 0);
    long long t0 = clock64();
    for (int it = 0; it < R; ++it) {
      const int s = it & 3, g = it & 3;
      const uint64_t bh = tc::smem_desc(sbase + 2048 * g, 128, 256, tc::kSwNone);
      const uint64_t bl = tc::smem_desc(sbase + 2048 * (4 + g), 128, 256, tc::kSwNone);
      const uint32_t a0 = tb + 256 + 64 * s;
#pragma unroll
      for (int tt = 0; tt < 4; ++tt) {
        const uint32_t d = tb + 64 * tt, ah = a0 + 16 * tt;
        mma_ta_elect(d, ah, bh, id, it > 0);
        mma_ta_elect(d, ah, bl, id, 1u);
        mma_ta_elect(d, ah + 8, bh, id, 1u);
      }
    }
    if (t == 0) tc::mma_commit(&bar);
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0 && t == 0) { out[0] = t2 - t0; }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(slot, 512);
}
template <int N, bool TA, int KB>
void run(long long *o, int R) {
  long long h[2];
  rate<N, TA, KB><<<148, 128>>>(o, R);
  cudaDeviceSynchronize();
  rate<N, TA, KB><<<148, 128>>>(o, R);
  cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("%s N=%3d KB=%d: issue %.1f cyc/MMA, complete %.1f cyc/MMA -> %.0f MAC/clk/SM\n", TA ? "TMEM-A" : "smem-A", N, KB,
         (double)h[0] / R, (double)h[1] / R, 128.0 * N * 8 * R / h[1]);
}
int main() {
  long long *o;
  cudaMalloc(&o, 16);
  const int R = 4096;
  run<64, false, 1>(o, R); run<128, false, 1>(o, R); run<256, false, 1>(o, R);
  run<64, true, 1>(o, R); run<128, true, 1>(o, R); run<256, true, 1>(o, R);
  run<64, false, 2>(o, R); run<64, true, 2>(o, R); run<256, true, 2>(o, R);
  for (int mode : {0, 8, 16, 64, 72})
  for (int nt = 1; nt <= 4; nt *= 4) {
    long long h[2];
    pattern<<<148, 128>>>(o, 1024, nt, mode); cudaDeviceSynchronize();
    pattern<<<148, 128>>>(o, 1024, nt, mode); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    const int per = (mode & 8) ? 1 : (mode & 16) ? 2 : 3;
    printf("pattern mode=%d (MMAs per tile-stage %d%s) ntile=%d: %.1f cyc/MMA\n", mode, per, (mode & 64) ? ", same D for all tiles" : "", nt, (double)h[0] / (1024.0 * per * nt));
  }
  {
    long long h[2];
    pattern_w<<<148, 128>>>(o, 1024); cudaDeviceSynchronize();
    pattern_w<<<148, 128>>>(o, 1024); cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("pattern_w (warp-wide, elect.sync) ntile=4: %.1f cyc/MMA\n", (double)h[0] / (1024.0 * 12));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
