// How many CTAs of the count kernel's shape (256 threads, ~75 KB shared
// memory: 3 per SM) are co-resident at each cluster size: clusters cannot
// span GPCs, so slots are lost when a GPC's CTA slots are not a multiple.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/mb_clusters tools/mb_clusters.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 3) k(int* p) {
  extern __shared__ int s[];
  if (p) p[blockIdx.x] = s[threadIdx.x];
}
int main() {
  const int smem = 64 * 1024 + 8 * 1024 + 2600;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, smem);
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  printf("SMs %d, CTAs per SM %d, slots %d\n", pr.multiProcessorCount, per_sm, per_sm * pr.multiProcessorCount);
  for (int cs : {1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 1000);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int nc = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d CTAs (%s)\n", cs, nc, nc * cs, cudaGetErrorString(e));
  }
  return 0;
}
