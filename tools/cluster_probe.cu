// cluster_probe.cu -- how many thread-block clusters of a 512-thread, ~212 KB-smem kernel fit
// on the device at once, per cluster size (cudaOccupancyMaxActiveClusters).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/cluster_probe tools/cluster_probe.cu
#include <cstdio>
__global__ void __launch_bounds__(512, 1) k(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  const size_t smem = 212 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * 32);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster size %2d: max active clusters %d (%d CTAs) %s\n", cl, n, n * cl, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
