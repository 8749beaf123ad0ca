#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void probe(double *out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  int me = cl.block_rank(), n = cl.num_blocks();
  if (threadIdx.x == 0) sm[5] = 100.0 + me;
  cl.sync();
  if (threadIdx.x < n) out[blockIdx.x * 16 + threadIdx.x] = cl.map_shared_rank(sm, threadIdx.x)[5];
  if (threadIdx.x == 0) printf("block %d rank %d of %d\n", blockIdx.x, me, n);
  cl.sync();
}
int main() {
  double *d; cudaMalloc(&d, 4 * 16 * 8); cudaMemset(d, 0, 4*16*8);
  for (int smem : {1024, 100000, 194560}) {
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(4); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d);
    cudaError_t e2 = cudaDeviceSynchronize();
    double h[64]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("smem %d launch %s sync %s: %g %g %g %g | %g %g\n", smem, cudaGetErrorString(e), cudaGetErrorString(e2), h[0], h[1], h[2], h[3], h[16], h[17]);
  }
}
