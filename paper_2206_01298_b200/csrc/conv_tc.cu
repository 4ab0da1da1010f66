// conv_tc.cu -- persistent explicit-RK kernels instantiated with the tcgen05 conv tile
// (tc_conv.cuh) for the C3 block, its weight packer and host geometry.
#include "tc_conv.cuh"

namespace ob {

void tc_conv_sizes(unsigned* packed_bytes, unsigned* smem_bytes) {
  *packed_bytes = conv_tc::kPacked;
  *smem_bytes = conv_tc::kTotal;
}

cudaError_t launch_pack_tc_conv(const Dims& d, const float* theta, void* img, cudaStream_t st) {
  pack_tc_conv_kernel<<<148, 256, 0, st>>>(d, theta, static_cast<unsigned char*>(img));
  return cudaGetLastError();
}

// dynamic shared memory starts after the 1 KB the system reserves per CTA and the kernel's
// static shared memory, at the array's 128-byte alignment (measured: 1280 for 256 static
// bytes; the tile checks the value on the device and fails loudly if it is off)
template <typename K>
static cudaError_t with_smem_base(K kf, const RkParams<float>& p, RkParams<float>& q) {
  cudaFuncAttributes at;
  cudaError_t e = cudaFuncGetAttributes(&at, kf);
  if (e != cudaSuccess) return e;
  q = p;
  q.tile_aux = 1024u + (unsigned)((at.sharedSizeBytes + 127) / 128 * 128);
  return cudaSuccess;
}

cudaError_t launch_conv_tc(const RkParams<float>& p, int tiles, size_t smem, cudaStream_t st, bool forward) {
  using F = TcConvAdapter<float>;
  RkParams<float> q;
  if (forward) {
    cudaError_t e = with_smem_base(rk_forward_kernel<float, F>, p, q);
    return e != cudaSuccess ? e : launch_smem(rk_forward_kernel<float, F>, tiles, smem, st, q);
  }
  cudaError_t e = with_smem_base(rk_reverse_kernel<float, F>, p, q);
  return e != cudaSuccess ? e : launch_smem(rk_reverse_kernel<float, F>, tiles, smem, st, q);
}

cudaError_t launch_conv_tc_field(const RkParams<float>& p, int tiles, size_t smem, int mode, double t,
                                 const float* u, const float* w, float* out, cudaStream_t st) {
  RkParams<float> q;
  cudaError_t e = with_smem_base(field_op_kernel<float, TcConvAdapter<float>>, p, q);
  return e != cudaSuccess ? e
                          : launch_smem(field_op_kernel<float, TcConvAdapter<float>>, tiles, smem, st, q, mode, t, u, w, out);
}

}  // namespace ob
