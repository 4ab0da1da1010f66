// cnf_tc.cu -- persistent explicit-RK kernels instantiated with the tcgen05 CNF tile
// (tc_cnf.cuh) for the C4 field shape, its weight packer and host geometry.
#include "tc_cnf.cuh"

namespace ob {

constexpr int kCnfD = 43, kCnfH = 860;   // BASELINE C4: (43 + t) -> 860 -> 860 -> 43, softplus

bool tc_cnf_shape(int D, int H) { return D == kCnfD && H == kCnfH; }

void tc_cnf_sizes(unsigned* packed_bytes, unsigned* smem_bytes, unsigned* log_record_bytes) {
  using G = CnfGeom<kCnfD, kCnfH>;
  *packed_bytes = G::Packed;
  *smem_bytes = G::Total;
  *log_record_bytes = G::Log;
}

cudaError_t launch_pack_tc_cnf(const Dims& d, const float* theta, void* img, cudaStream_t st) {
  pack_tc_cnf_kernel<kCnfD, kCnfH><<<148 * 4, 256, 0, st>>>(d, theta, static_cast<unsigned char*>(img));
  return cudaGetLastError();
}

// thread-block clusters of CL CTAs share every weight chunk (TMA multicast); the grid
// is a multiple of CL (the planner pads with empty tiles)
template <typename K, typename... A>
static cudaError_t launch_cluster(K kf, int grid, int cl, size_t smem, cudaStream_t st, A... args) {
  cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kf, args...);
}

template <int CL>
static cudaError_t launch_cl(const RkParams<float>& p, int tiles, size_t smem, cudaStream_t st, bool forward) {
  using F = TcCnfAdapter<float, kCnfD, kCnfH, CL>;
  return forward ? launch_cluster(rk_forward_kernel<float, F>, tiles, CL, smem, st, p)
                 : launch_cluster(rk_reverse_kernel<float, F>, tiles, CL, smem, st, p);
}

cudaError_t launch_cnf_tc(const RkParams<float>& p, int tiles, int cl, size_t smem, cudaStream_t st,
                          bool forward) {
  switch (cl) {
    case 1: return launch_cl<1>(p, tiles, smem, st, forward);
    case 2: return launch_cl<2>(p, tiles, smem, st, forward);
    case 4: return launch_cl<4>(p, tiles, smem, st, forward);
    default: return cudaErrorInvalidConfiguration;
  }
}

template <int CL>
static cudaError_t launch_field_cl(const RkParams<float>& p, int tiles, size_t smem, int mode, double t,
                                   const float* u, const float* w, float* out, cudaStream_t st) {
  using F = TcCnfAdapter<float, kCnfD, kCnfH, CL>;
  return launch_cluster(field_op_kernel<float, F>, tiles, CL, smem, st, p, mode, t, u, w, out);
}

cudaError_t launch_cnf_tc_field(const RkParams<float>& p, int tiles, int cl, size_t smem, int mode,
                                double t, const float* u, const float* w, float* out, cudaStream_t st) {
  switch (cl) {
    case 1: return launch_field_cl<1>(p, tiles, smem, mode, t, u, w, out, st);
    case 2: return launch_field_cl<2>(p, tiles, smem, mode, t, u, w, out, st);
    case 4: return launch_field_cl<4>(p, tiles, smem, mode, t, u, w, out, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace ob
