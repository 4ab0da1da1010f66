// rk_f64.cu -- explicit instantiations of the persistent RK kernels (fp64); the
// kernel families are split across translation units so they compile in parallel.
#include "rk_impl.cuh"

namespace ob {
template cudaError_t launch_rk_ws<double, false>(const RkParams<double>&, int, int, size_t,
                                                 cudaStream_t, bool);
template cudaError_t launch_field_ws<double, false>(const RkParams<double>&, int, int, size_t, int,
                                                    double, const double*, const double*, double*,
                                                    cudaStream_t);
template cudaError_t launch_pack<double>(const PackParams<double>&, cudaStream_t);
template cudaError_t launch_reduce<double>(const Dims&, const double*, int, long long, double*,
                                           const double*, double, double*, cudaStream_t,
                                          const double*);
template cudaError_t launch_cadj_ws<double, false>(const RkParams<double>&, int, int, size_t, double,
                                                   const double*, cudaStream_t);
}  // namespace ob
