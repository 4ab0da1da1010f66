// rk_cl_f64.cu -- cluster MLP adapter of the explicit-RK kernels, clusters of 8 CTAs
// (rk_cl_impl.cuh).
#define OB_THCL_CL 8
#include "rk_cl_impl.cuh"
