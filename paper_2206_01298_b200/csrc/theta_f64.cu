// theta_f64.cu -- explicit instantiation of the theta-method kernels (fp64).
#include "theta_impl.cuh"

namespace ob {
template cudaError_t launch_theta<double>(const RkParams<double>&, int, int, size_t, cudaStream_t,
                                          bool);
}  // namespace ob
