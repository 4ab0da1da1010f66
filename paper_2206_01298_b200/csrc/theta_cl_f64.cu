// theta_cl_f64.cu -- cluster-resident-weights theta kernels (theta_cluster.cuh), fp64.
#define OB_THCL_KERNELS
#include "theta_cluster.cuh"

namespace ob {

void theta_cluster_geom(int N, int H, int R, int RC, bool second_x, int* region_doubles, int* cluster) {
  *region_doubles = thcl_geom(N, H, R, RC, second_x).total;
  *cluster = thcl::kCL;
}

// clusters of the kernel that can be resident at once with `smem` bytes of dynamic shared
// memory (GPC granularity: 15 clusters of 8 on a 148-SM B200)
int theta_cluster_max_active(size_t smem) {
  // (per thread and device: the answer depends on the device, and plans are made per thread)
  static thread_local int cached = -1, cached_dev = -1;
  static thread_local size_t cached_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cached >= 0 && cached_smem == smem && cached_dev == dev) return cached;
  if (cudaFuncSetAttribute(thcl_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(thcl::kCL * 32);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = thcl::kCL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, thcl_forward_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cached = n;
  cached_smem = smem;
  cached_dev = dev;
  return n;
}

cudaError_t launch_theta_cluster(const RkParams<double>& p, int tiles, size_t smem, cudaStream_t st, bool forward) {
  return forward ? thcl_launch(thcl_forward_kernel, tiles, smem, st, p)
                 : thcl_launch(thcl_reverse_kernel, tiles, smem, st, p);
}

}  // namespace ob
