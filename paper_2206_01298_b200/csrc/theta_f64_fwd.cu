// theta_f64_fwd.cu -- explicit instantiation of the theta-method forward kernels (f64).
#include "theta_impl.cuh"

namespace ob {
template cudaError_t launch_theta_dir<double, true>(const RkParams<double>&, int, int, size_t,
                                                     cudaStream_t);
}  // namespace ob
