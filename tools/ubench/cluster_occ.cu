#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* x) { extern __shared__ int s[]; if (x) x[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
  for (int cl : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * 64); cfg.blockDim = dim3(640); cfg.dynamicSmemBytes = 180 * 1024;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cl; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
    printf("cluster %d: max active clusters %d -> %d CTAs (%s)\n", cl, n, n * cl, cudaGetErrorString(e));
  }
}
