// conv_f32.cu -- explicit instantiation of the conv-block (C3) kernels, fp32.
#include "conv_impl.cuh"

namespace ob {
template cudaError_t launch_conv<float>(const RkParams<float>&, int, size_t, cudaStream_t, bool);
template cudaError_t launch_conv_field<float>(const RkParams<float>&, int, size_t, int, double,
                                              const float*, const float*, float*, cudaStream_t);
template cudaError_t launch_pack_conv<float>(const PackParams<float>&, cudaStream_t);
template cudaError_t launch_reduce_plain<float>(const float*, int, long long, long long, float*,
                                                cudaStream_t);
}  // namespace ob
