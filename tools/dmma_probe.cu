// dmma_probe.cu -- fp64 tensor-core MMA (mma.sync.m8n8k4.f64) rate on one SM: W warps, each a
// loop of 4 independent accumulator chains; cycles per DMMA per SM and the FMA rate, beside
// the same FMA count on the vector pipe.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k_dmma(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = c[0][0] + c[1][1] + c[2][0] + c[3][1];
}
__global__ void k_dfma(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = fma(a, b, c[j]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = c[0] + c[3] + c[7];
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  const int iters = 2000;
  for (int warps : {1, 4, 8, 16}) {
    long long h;
    k_dmma<<<1, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double nd = 4.0 * iters * warps;
    printf("DMMA  %2d warps: %8lld cycles, %.2f cycles per DMMA per SM, %.1f FMA/clk/SM\n", warps, h, h / nd, nd * 256 / h);
    k_dfma<<<1, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double nf = 8.0 * iters * warps * 32;
    printf("DFMA  %2d warps: %8lld cycles, %.1f FMA/clk/SM\n", warps, h, nf / h);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
