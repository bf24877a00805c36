// How many 2-CTA clusters of a 1-CTA-per-SM, ~200 KB-smem kernel can be
// resident at once on this GPU (the persistent SM-pair GEMM assumes 74).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) k2(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}
__global__ void __launch_bounds__(256, 1) k1(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int smem : {100 << 10, 180 << 10, 200 << 10, 220 << 10}) {
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int clusters = -1, blocks = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, (void*)k2, &cfg);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k1, 256, smem);
    printf("sms %d smem %d KB: max active 2-CTA clusters %d (%s), 1-CTA blocks/SM %d\n", sms,
           smem >> 10, clusters, cudaGetErrorString(e), blocks);
  }
  return 0;
}
