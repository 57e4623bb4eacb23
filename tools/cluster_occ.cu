// Max co-resident clusters for a one-CTA-per-SM kernel (the int8 TRSM's footprint) at cluster
// sizes 1..16: how many SMs each cluster shape can use on this GPU (GPC packing).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int* p) {
  extern __shared__ int s[];
  if (p) p[threadIdx.x] = s[threadIdx.x];
}
int main() {
  const int smem = 190 * 1024;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 6, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, dummy, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d SMs (%s)\n", cs, nc, nc * cs,
           cudaGetErrorString(e));
  }
  return 0;
}
