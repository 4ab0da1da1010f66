// mma_probe.cu -- throughput of warp-level mma.sync m16n8k8 TF32 on one SM
// (independent accumulators, operands in registers) vs SIMT FFMA.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

template <int CH>
__global__ void hmma_loop(float* out, int iters, uint32_t seed) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = (seed + threadIdx.x * 7 + i) & 0x3f800000u;
  for (int i = 0; i < 2; ++i) b[i] = (seed + threadIdx.x * 3 + i) & 0x3f800000u;
  float d[CH][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void bf16_loop(float* out, int iters, uint32_t seed) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = (seed + threadIdx.x * 7 + i) & 0x3f803f80u;
  for (int i = 0; i < 2; ++i) b[i] = (seed + threadIdx.x * 3 + i) & 0x3f803f80u;
  float d[CH][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
void run(const char* name, K kern, int threads, double macs_per_warp_iter, int iters) {
  float* out;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  int sms = 148;
  kern<<<sms, threads>>>(out, 10, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<sms, threads>>>(out, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double macs = macs_per_warp_iter * (threads / 32) * (double)iters * sms;
  const double tf = 2 * macs / (ms * 1e-3) / 1e12;
  const double per_sm_clk = macs / sms / (ms * 1e-3 * clk * 1e3);
  printf("%-28s threads %4d  %.3f ms  %.1f TFLOP/s  %.0f MAC/clk/SM (at %d MHz max)\n", name,
         threads, ms, tf, per_sm_clk, clk / 1000);
  cudaFree(out);
}

int main() {
  const int it = 20000;
  for (int th : {128, 256, 512, 1024}) {
    run("mma tf32 m16n8k8 x4", hmma_loop<4>, th, 4 * 16 * 8 * 8, it);
    run("mma tf32 m16n8k8 x8", hmma_loop<8>, th, 8 * 16 * 8 * 8, it);
    run("mma bf16 m16n8k16 x8", bf16_loop<8>, th, 8 * 16 * 8 * 16, it);
  }
  return 0;
}
