// rk_cl_impl.cuh -- explicit-RK kernels (rk_impl.cuh) instantiated with the cluster MLP adapter
// (theta_cluster.cuh) for the cluster size OB_THCL_CL of the including translation unit: fp64
// two-layer MLP fields with the weights resident across a cluster.  Exports
// rk_cluster{2,8}_geom / _max_active / launch_rk_cluster{2,8}.
#pragma once
#include "theta_cluster.cuh"

#define OB_RKCL_CAT2(a, n, b) a##n##b
#define OB_RKCL_CAT(a, n, b) OB_RKCL_CAT2(a, n, b)
#define OB_RKCL(a, b) OB_RKCL_CAT(a, OB_THCL_CL, b)

namespace ob {

// shared-memory doubles of the cluster region for R rows per CTA (linearisation rows X and
// cotangent rows X2)
void OB_RKCL(rk_cluster, _geom)(int N, int H, int R, int* region_doubles) {
  *region_doubles = thcl_geom(N, H, R, thcl::kCL * R, true).total;
}

int OB_RKCL(rk_cluster, _max_active)(size_t smem) {
  // (per thread and device: the answer depends on the device, and plans are made per thread)
  static thread_local int cached = -1, cached_dev = -1;
  static thread_local size_t cached_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cached >= 0 && cached_smem == smem && cached_dev == dev) return cached;
  auto kf = rk_reverse_kernel<double, ClusterMlpAdapter>;
  if (cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(thcl::kCL * 32);
  cfg.blockDim = dim3(thcl::kRkThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = thcl::kCL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kf, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cached = n;
  cached_smem = smem;
  cached_dev = dev;
  return n;
}

cudaError_t OB_RKCL(launch_rk_cluster, )(const RkParams<double>& p, int tiles, size_t smem, cudaStream_t st,
                                         bool forward) {
  return forward ? thcl_launch(rk_forward_kernel<double, ClusterMlpAdapter>, tiles, smem, st, p, thcl::kRkThreads)
                 : thcl_launch(rk_reverse_kernel<double, ClusterMlpAdapter>, tiles, smem, st, p, thcl::kRkThreads);
}

}  // namespace ob
