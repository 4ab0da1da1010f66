// theta_f32_rev.cu -- explicit instantiation of the theta-method reverse kernels (f32).
#include "theta_impl.cuh"

namespace ob {
template cudaError_t launch_theta_dir<float, false>(const RkParams<float>&, int, int, size_t,
                                                     cudaStream_t);
}  // namespace ob
