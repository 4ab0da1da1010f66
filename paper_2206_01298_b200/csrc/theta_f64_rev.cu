// theta_f64_rev.cu -- explicit instantiation of the theta-method reverse kernels (f64).
#include "theta_impl.cuh"

namespace ob {
template cudaError_t launch_theta_dir<double, false>(const RkParams<double>&, int, int, size_t,
                                                     cudaStream_t);
}  // namespace ob
