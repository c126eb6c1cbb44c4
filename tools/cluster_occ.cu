// cluster_occ.cu — how many clusters of C CTAs (1 CTA/SM, ~200 KB smem,
// 768 threads) can be co-resident on this B200 (GPC packing).  Dev tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/cluster_occ.cu -o build/cluster_occ
#include <cstdio>

__global__ void __launch_bounds__(768, 1) k(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}

int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c = 1; c <= 16; ++c) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c * 64);
    cfg.blockDim = dim3(768);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d CTAs (%s)\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
