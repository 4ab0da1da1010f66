// conv_probe.cu -- validates, on the device, the tcgen05 conventions the tensor-core conv
// tile (csrc/tc_conv.cuh) relies on:
//   1. kind::f16 with fp16 operands (instruction-descriptor formats 0);
//   2. a K-major A operand in the linear-position layout [channel/8][position][8 channels]
//      whose start address is displaced by any multiple of 16 bytes (a 3x3 tap is a
//      position offset), with a plane stride that is an odd multiple of 16 bytes;
//   3. the same weight bytes as a K-major B (N = cout, K = cin) and an MN-major B
//      (N = cin, K = cout: the transposed convolution);
//   4. MN-major A and B with K = positions (the weight-gradient products), M = 64;
//   5. whether an M = 64 accumulator may sit at TMEM lane offset 16 (two per column range).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/conv_probe tools/conv_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2206_01298_b200/csrc/tc.cuh"
using namespace ob;

constexpr int NP = 313;                 // positions per plane (odd: conflict-free 16-byte stores)
constexpr uint32_t PLANE = NP * 16;     // bytes per 8-channel plane
constexpr uint32_t WPL = 64 * 16;       // weight plane: 64 rows x 8 channels
constexpr uint32_t TILE = 8 * PLANE;

__device__ __forceinline__ uint32_t idesc_f16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// mode 0: D[m][n] = sum_k X[q0 + m][k] W[n][k]          (M = 128, N = 64, K = 64)
// mode 1: D[m][n] = sum_k X[q0 + m][k] W[k][n]          (B MN-major)
// mode 2: D[co][ci] = sum_{j < 32} V[q0 + j][co] X[q1 + j][ci]   (M = 64, N = 64, K = 32), lane offset dl
__global__ void probe(int mode, int q0, int q1, int dl, const float* X, const float* V, const float* W, float* D) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  unsigned char* Xs = sm;
  unsigned char* Vs = sm + TILE;
  unsigned char* Ws = sm + 2 * TILE;
  for (int i = threadIdx.x; i < NP * 64; i += blockDim.x) {
    const int q = i / 64, c = i % 64;
    const uint32_t off = (c >> 3) * PLANE + q * 16 + (c & 7) * 2;
    *reinterpret_cast<__half*>(Xs + off) = __float2half_rn(X[i]);
    *reinterpret_cast<__half*>(Vs + off) = __float2half_rn(V[i]);
  }
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64;   // W[r][c]: rows at 16 bytes, 8-column planes
    *reinterpret_cast<__half*>(Ws + (c >> 3) * WPL + r * 16 + (c & 7) * 2) = __float2half_rn(W[i]);
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 128);
  if (threadIdx.x == 0) tc::bar_init(&bar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tslot;
  // clear the accumulator columns so untouched lanes read as zero
  {
    float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int w = threadIdx.x / 32;
    for (int c = 0; c < 128; c += 8) tc::st8(tbase + ((uint32_t)(32 * w) << 16) + c, z);
    tc::wait_st();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x < 32) {
    const uint32_t xs = tc::smem_u32(Xs), vs = tc::smem_u32(Vs), ws = tc::smem_u32(Ws);
    if (mode == 0 || mode == 1) {
      const uint32_t id = idesc_f16(128, 64, false, mode == 1);
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t da = tc::sdesc(xs + ks * 2 * PLANE + q0 * 16, PLANE, 128);
        const uint64_t db = mode == 0 ? tc::sdesc(ws + ks * 2 * WPL, WPL, 128)      // K-major: LBO = K plane
                                      : tc::sdesc(ws + ks * 256, 128, WPL);         // MN-major: K rows, N planes
        tc::mma_bf16(tbase, da, db, id, ks > 0);
      }
    } else {
      const uint32_t id = idesc_f16(64, 64, true, true);
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t da = tc::sdesc(vs + q0 * 16 + ks * 256, 128, PLANE);
        const uint64_t db = tc::sdesc(xs + q1 * 16 + ks * 256, 128, PLANE);
        tc::mma_bf16(tbase + ((uint32_t)dl << 16), da, db, id, ks > 0);
      }
    }
    tc::commit(&bar);
  }
  tc::bar_wait(&bar, 0);
  tc::fence_after();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c = 0; c < 64; c += 8) {
    float v[8];
    tc::ld8(tbase + ((uint32_t)(32 * w) << 16) + c, v);
    for (int j = 0; j < 8; ++j) D[(32 * w + lane) * 64 + c + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(tbase, 128);
}

int main() {
  float *X, *V, *W, *D;
  cudaMallocManaged(&X, NP * 64 * 4);
  cudaMallocManaged(&V, NP * 64 * 4);
  cudaMallocManaged(&W, 64 * 64 * 4);
  cudaMallocManaged(&D, 128 * 64 * 4);
  srand(7);
  for (int i = 0; i < NP * 64; ++i) { X[i] = (rand() % 17 - 8) / 8.0f; V[i] = (rand() % 17 - 8) / 8.0f; }
  for (int i = 0; i < 64 * 64; ++i) W[i] = (rand() % 17 - 8) / 8.0f;
  const size_t smem = 2 * TILE + 8 * WPL + 256;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int fails = 0;
  auto run = [&](int mode, int q0, int q1, int dl) {
    cudaMemset(D, 0, 128 * 64 * 4);
    probe<<<1, 128, smem>>>(mode, q0, q1, dl, X, V, W, D);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d q0 %d q1 %d dl %d: CUDA error %s\n", mode, q0, q1, dl, cudaGetErrorString(e)); exit(1); }
  };
  for (int mode = 0; mode < 2; ++mode)
    for (int q0 : {0, 1, 3, 17, 18, 35, 146, 180}) {
      run(mode, q0, 0, 0);
      double err = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double ref = 0;
          for (int k = 0; k < 64; ++k)
            ref += (double)X[(q0 + m) * 64 + k] * (mode == 0 ? W[n * 64 + k] : W[k * 64 + n]);
          err = fmax(err, fabs(ref - D[m * 64 + n]));
        }
      printf("conv %s B, q0 %3d: max err %g\n", mode == 0 ? "K-major " : "MN-major", q0, err);
      if (err > 1e-3) ++fails;
    }
  for (int dl : {0, 16})
    for (int q0 : {18, 21})
      for (int q1 : {18, 0, 37}) {
        run(2, q0, q1, dl);
        double err = 0, stray = 0;
        for (int l = 0; l < 128; ++l) {
          const int in = (l % 32) - dl;                    // expected: rows 16 g + r at lane 32 g + dl + r
          const bool mine = in >= 0 && in < 16;
          for (int n = 0; n < 64; ++n) {
            if (!mine) { stray = fmax(stray, fabs(D[l * 64 + n])); continue; }
            const int co = 16 * (l / 32) + in;
            double ref = 0;
            for (int j = 0; j < 32; ++j) ref += (double)V[(q0 + j) * 64 + co] * X[(q1 + j) * 64 + n];
            err = fmax(err, fabs(ref - D[l * 64 + n]));
          }
        }
        printf("wgrad M64 lane offset %2d, q0 %2d q1 %2d: max err %g, stray %g\n", dl, q0, q1, err, stray);
        if (dl == 0 && (err > 1e-3 || stray != 0)) ++fails;
      }
  printf(fails ? "PROBE FAIL %d\n" : "PROBE OK\n", fails);
  return 0;
}
