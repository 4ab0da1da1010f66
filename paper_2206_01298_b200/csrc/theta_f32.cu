// theta_f32.cu -- explicit instantiation of the theta-method kernels (fp32).
#include "theta_impl.cuh"

namespace ob {
template cudaError_t launch_theta<float>(const RkParams<float>&, int, int, size_t, cudaStream_t,
                                         bool);
}  // namespace ob
