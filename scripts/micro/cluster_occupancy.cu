// How many clusters of 2 / 4 / 8 CTAs (one 200+ KB-smem CTA per SM) can be resident at once on this
// GPU: cudaOccupancyMaxActiveClusters. A 4-CTA cluster (two CTA pairs sharing operands through TMA
// multicast) only pays if it still covers every SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o cluster_occupancy cluster_occupancy.cu
#include <cstdio>
__global__ void k(int* p) { if (p) p[0] = 1; }
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d of %d SMs busy %s\n", cs, n, n * cs, sms,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
