// theta_f32_fwd.cu -- explicit instantiation of the theta-method forward kernels (f32).
#include "theta_impl.cuh"

namespace ob {
template cudaError_t launch_theta_dir<float, true>(const RkParams<float>&, int, int, size_t,
                                                     cudaStream_t);
}  // namespace ob
