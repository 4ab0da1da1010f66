// adaptive_f32.cu -- explicit instantiations of the adaptive-stepping kernels (fp32;
// weights in shared memory or L1/L2).
#include "adaptive_impl.cuh"

namespace ob {
template cudaError_t launch_adaptive_ws<float, true>(const RkParams<float>&, int, int, size_t,
                                                     cudaStream_t, bool);
template cudaError_t launch_adaptive_ws<float, false>(const RkParams<float>&, int, int, size_t,
                                                      cudaStream_t, bool);
}  // namespace ob
