// rk_tc.cu -- persistent explicit-RK kernels instantiated with the tcgen05
// tensor-core MLP tile (tc_mlp.cuh) for each supported (state, hidden) shape,
// its weight packer and host geometry.
#include "tc_mlp.cuh"

namespace ob {

void tc_sizes(int D0, int H, int D2, unsigned* packed_bytes, unsigned* total_bytes) {
  const TcGeom g = tc_geom(D0, H, D2);
  *packed_bytes = g.packed;
  *total_bytes = g.total;
}

bool tc_shape_supported(int D0, int H, int D2) { return tc_shape_ok(D0, H, D2); }

cudaError_t launch_pack_tc(const Dims& d, const float* theta, float* packed, cudaStream_t st) {
  pack_tc_kernel<<<148, 256, 0, st>>>(d, theta, packed);
  return cudaGetLastError();
}

template <int D, int H>
static cudaError_t launch_shape(const RkParams<float>& p, int tiles, size_t smem, cudaStream_t st,
                               bool forward) {
  using F = TcMlpAdapter<float, D, H, D>;
  return forward ? launch_smem(rk_forward_kernel<float, F>, tiles, smem, st, p)
                 : launch_smem(rk_reverse_kernel<float, F>, tiles, smem, st, p);
}

cudaError_t launch_rk_tc(const RkParams<float>& p, int tiles, size_t smem, cudaStream_t st,
                         bool forward) {
  const int D = p.d.N, H = p.d.w[1];
#define OB_TC_CASE(d, h) \
  if (D == d && H == h) return launch_shape<d, h>(p, tiles, smem, st, forward);
  OB_TC_CASE(64, 256) OB_TC_CASE(64, 128) OB_TC_CASE(48, 256) OB_TC_CASE(48, 128)
  OB_TC_CASE(32, 256) OB_TC_CASE(32, 128) OB_TC_CASE(16, 256) OB_TC_CASE(16, 128)
#undef OB_TC_CASE
  return cudaErrorInvalidConfiguration;
}

}  // namespace ob
