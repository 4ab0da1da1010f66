// rk_cl2_f64.cu -- cluster MLP adapter of the explicit-RK kernels, clusters of 2 CTAs: each CTA
// keeps half of both weight matrices and the parameter cotangents of its half in registers
// (rk_cl_impl.cuh, theta_cluster.cuh).
#define OB_THCL_CL 2
#include "rk_cl_impl.cuh"
