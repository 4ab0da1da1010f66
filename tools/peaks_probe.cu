// peaks_probe.cu -- measure the FP32 / FP64 FMA-pipe peaks of this B200
// (the roofline denominators MEASURED_PEAKS.json does not carry).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks_probe tools/peaks_probe.cu
//   tools/peaks_probe > profiles/fp_peaks.json
//
// Each thread runs 8 independent FMA chains (enough ILP to cover the 4-cycle
// latency), grid = 148 SMs x 4 CTAs x 512 threads.  Best of 5 CUDA-event timings.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_kernel(T* out, int iters, T b, T c) {
  T a0 = T(threadIdx.x) * T(1e-3), a1 = a0 + T(1), a2 = a0 + T(2), a3 = a0 + T(3);
  T a4 = a0 + T(4), a5 = a0 + T(5), a6 = a0 + T(6), a7 = a0 + T(7);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = a0 * b + c; a1 = a1 * b + c; a2 = a2 * b + c; a3 = a3 * b + c;
      a4 = a4 * b + c; a5 = a5 * b + c; a6 = a6 * b + c; a7 = a7 * b + c;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <typename T>
double measure(int iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512;
  T* out;
  cudaMalloc(&out, sizeof(T) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_kernel<T><<<blocks, threads>>>(out, iters / 10, T(0.999999), T(1e-7));
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_kernel<T><<<blocks, threads>>>(out, iters, T(0.999999), T(1e-7));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  const double f32 = measure<float>(20000);
  const double f64 = measure<double>(4000);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp32_tflops\": %.2f, \"fp64_tflops\": %.2f, \"how\": \"tools/peaks_probe.cu: "
         "8 independent FMA chains/thread, 148x4 CTAs x 512 threads, best of 5 CUDA-event "
         "timings\", \"sm_clock_attr_mhz\": %d}\n", f32, f64, clk / 1000);
  return 0;
}
