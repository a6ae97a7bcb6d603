// How many clusters of a 288-thread, ~206 KB / ~103 KB smem kernel fit at once (cudaOccupancyMaxActiveClusters)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* x) { extern __shared__ int s[]; if (threadIdx.x == 0 && x) x[0] = s[0]; }
int main() {
  int smems[2] = {206 * 1024, 103 * 1024};
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 206 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int si = 0; si < 2; ++si)
    for (int cs : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 16, 1);
      cfg.blockDim = dim3(288);
      cfg.dynamicSmemBytes = smems[si];
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %d KB cluster %d: max active clusters %d (%s) -> %d CTAs\n", smems[si] / 1024, cs, n, cudaGetErrorString(e), n * cs);
    }
  return 0;
}
