// adaptive_f64.cu -- explicit instantiations of the adaptive-stepping kernels (fp64).
#include "adaptive_impl.cuh"

namespace ob {
template cudaError_t launch_adaptive_ws<double, false>(const RkParams<double>&, int, int, size_t,
                                                       cudaStream_t, bool);
}  // namespace ob
