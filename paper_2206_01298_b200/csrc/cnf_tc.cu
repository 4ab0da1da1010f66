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

cudaError_t launch_cnf_tc(const RkParams<float>& p, int tiles, size_t smem, cudaStream_t st, bool forward) {
  using F = TcCnfAdapter<float, kCnfD, kCnfH>;
  return forward ? launch_smem(rk_forward_kernel<float, F>, tiles, smem, st, p)
                 : launch_smem(rk_reverse_kernel<float, F>, tiles, smem, st, p);
}

cudaError_t launch_cnf_tc_field(const RkParams<float>& p, int tiles, size_t smem, int mode, double t,
                                const float* u, const float* w, float* out, cudaStream_t st) {
  using F = TcCnfAdapter<float, kCnfD, kCnfH>;
  return launch_smem(field_op_kernel<float, F>, tiles, smem, st, p, mode, t, u, w, out);
}

}  // namespace ob
