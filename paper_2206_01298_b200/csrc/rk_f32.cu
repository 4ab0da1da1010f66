// rk_f32.cu -- explicit instantiations of the persistent RK kernels (fp32, weights in L1/L2); the
// kernel families are split across translation units so they compile in parallel.
#include "rk_impl.cuh"

namespace ob {
template cudaError_t launch_rk_ws<float, false>(const RkParams<float>&, int, int, size_t, cudaStream_t,
                                                bool);
template cudaError_t launch_field_ws<float, false>(const RkParams<float>&, int, int, size_t, int,
                                                   double, const float*, const float*, float*,
                                                   cudaStream_t);
template cudaError_t launch_pack<float>(const PackParams<float>&, cudaStream_t);
template cudaError_t launch_reduce<float>(const Dims&, const float*, int, long long, float*,
                                          const double*, double, double*, cudaStream_t,
                                          const float*);
template cudaError_t launch_cadj_ws<float, false>(const RkParams<float>&, int, int, size_t, double,
                                                   const float*, cudaStream_t);
}  // namespace ob
