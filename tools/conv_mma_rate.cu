// conv_mma_rate.cu -- tensor-pipe rate of the conv tile's MMA pattern with ideal issue
// (compile-time descriptors, one issuing warp, no waits between units): 27 units of 12
// MMAs (M128 N64 K16, fp16, A = linear-position image K-major [LBO = plane 5008, SBO = 128],
// B = tap weights K-major [LBO 1024, SBO 128]) into three accumulators in turn.
//   MODE 0: the tile's order (4 x A_lo B_hi, then 4 x (A_hi B_lo keep-A, A_hi B_hi reuse-A))
//   MODE 1: no collector reuse     MODE 2: as 0 with N = 16     MODE 3: A planes dense (LBO 4096)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/conv_mma_rate tools/conv_mma_rate.cu
#include <cstdio>
#include <vector>
#include "../paper_2206_01298_b200/csrc/tc.cuh"
using namespace ob;

constexpr uint32_t kPlane = 5008, kPart = 8 * kPlane, kTile = 2 * kPart, kWPl = 1024, kTapHalf = 8192, kTap = 16384;
constexpr uint32_t kRing = 2 * kTile + 10112;

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(long long* out, int reps) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 220 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  if (threadIdx.x < 32) tc::tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) tc::bar_init(&bar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  uint32_t ph = 0;
  const uint32_t sb = tc::smem_u32(sm);
  constexpr int N = MODE == 2 ? 16 : 64;
  constexpr uint32_t id = tc::idesc_f16(128, N, false, false);
  constexpr uint32_t PL = MODE == 3 ? 4096u : kPlane;
  long long best = 1LL << 60, sum = 0, bissue = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    if (tc::uniform_warp() == 0) {
#pragma unroll
      for (int s = 0; s < 9; ++s) {
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const uint32_t a0 = sb + (18 + 128 * b + (s / 3 - 1) * 17 + (s % 3 - 1)) * 16;
          const uint32_t wb = sb + kRing + (s % 3) * kTap;
          const uint32_t d = 64 * b;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            tc::mma_bf16(d, tc::sdesc(a0 + kPart + 2 * ks * PL, PL, 128), tc::sdesc(wb + 2 * ks * kWPl, kWPl, 128), id,
                         ks > 0);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t Ah = tc::sdesc(a0 + 2 * ks * PL, PL, 128);
            if (MODE == 1) {
              tc::mma_bf16(d, Ah, tc::sdesc(wb + kTapHalf + 2 * ks * kWPl, kWPl, 128), id, 1u);
              tc::mma_bf16(d, Ah, tc::sdesc(wb + 2 * ks * kWPl, kWPl, 128), id, 1u);
            } else {
              tc::mma_bf16_keep_a(d, Ah, tc::sdesc(wb + kTapHalf + 2 * ks * kWPl, kWPl, 128), id, 1u);
              tc::mma_bf16_reuse_a(d, Ah, tc::sdesc(wb + 2 * ks * kWPl, kWPl, 128), id, 1u);
            }
          }
        }
      }
      tc::commit(&bar);
    }
    const long long t1 = clock64();
    tc::bar_wait(&bar, ph);
    ph ^= 1u;
    tc::fence_after();
    const long long t = clock64() - t0;
    if (r > 0 && threadIdx.x == 0) { best = min(best, t); sum += t; bissue = min(bissue, t1 - t0); }
  }
  if (threadIdx.x == 0) { out[0] = best; out[1] = sum / (reps - 1); out[2] = bissue; }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(slot, 512);
}

template <int MODE>
void run(const char* name, long long* d) {
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  kern<MODE><<<1, 512, 220 * 1024>>>(d, 10);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-44s 324 MMAs: total min %6lld avg %6lld (%.1f / MMA), issue min %6lld | floor %d | %s\n", name, h[0], h[1],
         h[0] / 324.0, h[2], 324 * 32, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<0>("conv pattern, tile order + collector", d);
  run<1>("conv pattern, no collector reuse", d);
  run<2>("conv pattern, N = 16", d);
  run<3>("conv pattern, dense A planes (LBO 4096)", d);
  return 0;
}
