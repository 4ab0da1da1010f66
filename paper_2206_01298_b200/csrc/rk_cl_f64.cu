// rk_cl_f64.cu -- explicit-RK kernels (rk_impl.cuh) instantiated with the cluster MLP adapter
// (theta_cluster.cuh): fp64 two-layer MLP fields with the weights resident across a cluster.
#include "theta_cluster.cuh"

namespace ob {

template <typename K>
static cudaError_t rkcl_launch(K kf, int grid, size_t smem, cudaStream_t st, const RkParams<double>& p) {
  return thcl_launch(kf, grid, smem, st, p);
}

int rk_cluster_max_active(size_t smem) {
  static int cached = -1;
  static size_t cached_smem = 0;
  if (cached >= 0 && cached_smem == smem) return cached;
  auto kf = rk_reverse_kernel<double, ClusterMlpAdapter>;
  if (cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
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
  if (cudaOccupancyMaxActiveClusters(&n, kf, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cached = n;
  cached_smem = smem;
  return n;
}

cudaError_t launch_rk_cluster(const RkParams<double>& p, int tiles, size_t smem, cudaStream_t st, bool forward) {
  return forward ? rkcl_launch(rk_forward_kernel<double, ClusterMlpAdapter>, tiles, smem, st, p)
                 : rkcl_launch(rk_reverse_kernel<double, ClusterMlpAdapter>, tiles, smem, st, p);
}

}  // namespace ob
