// cnf_f32.cu -- explicit instantiation of the CNF (C4) kernels, fp32.
#include "cnf_impl.cuh"

namespace ob {
template cudaError_t launch_cnf<float>(const RkParams<float>&, int, int, size_t, cudaStream_t, bool);
template cudaError_t launch_cnf_field<float>(const RkParams<float>&, int, int, size_t, int, double,
                                             const float*, const float*, float*, cudaStream_t);
}  // namespace ob
