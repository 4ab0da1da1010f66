// mma_timing.cu -- timing probe for the C2 tile's tcgen05 pattern on one SM per CTA:
// cycles from the first tcgen05.mma issue to the mbarrier completion of a group of
// MMAs (bf16, SS operands, no swizzle core blocks like csrc/tc.cuh), for M in {64,128},
// N in {16, 32, 64, 128}, the 3-pass split (collector reuse of A_hi) vs single pass;
// plus tcgen05.ld throughput of a 128-lane x 32-column fp32 accumulator read by 16 warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_timing tools/mma_timing.cu
#include <cstdio>
#include <vector>
#include "../paper_2206_01298_b200/csrc/tc.cuh"
using namespace ob;

struct Res { long long issue, total; };

template <int M, int N, int KS, int MODE>
__device__ void group(uint32_t sb, uint64_t* bar, uint32_t& ph, Res& r) {
  // A: [M][KS*16] K-major (core blocks: rows at SA = KS*2*128, k blocks at 128)
  constexpr uint32_t SA = KS * 2 * 128, BSA = KS * 2 * 128;
  constexpr uint32_t A_hi = 0, A_lo = M * KS * 16 * 2;
  constexpr uint32_t B_hi = 2 * M * KS * 16 * 2, B_lo = B_hi + N * KS * 16 * 2;
  constexpr uint32_t id = tc::idesc_bf16(M, N, false, false);
  long long t0 = clock64();
  if (tc::uniform_warp() == 0) {
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const uint64_t Ah = tc::sdesc(sb + A_hi + k * 256, 128, SA), Al = tc::sdesc(sb + A_lo + k * 256, 128, SA);
      const uint64_t Bh = tc::sdesc(sb + B_hi + k * 256, 128, BSA), Bl = tc::sdesc(sb + B_lo + k * 256, 128, BSA);
      if (MODE == 0) {
        tc::mma_bf16_keep_a(0, Ah, Bh, id, k > 0);
        tc::mma_bf16_reuse_a(0, Ah, Bl, id, 1u);
        tc::mma_bf16(0, Al, Bh, id, 1u);
      } else if (MODE == 1) {
        tc::mma_bf16(0, Ah, Bh, id, k > 0);
        tc::mma_bf16(0, Ah, Bl, id, 1u);
        tc::mma_bf16(0, Al, Bh, id, 1u);
      } else {
        tc::mma_bf16(0, Ah, Bh, id, k > 0);
      }
    }
    tc::commit(bar);
  }
  long long t1 = clock64();
  tc::bar_wait(bar, ph);
  ph ^= 1u;
  tc::fence_after();
  long long t2 = clock64();
  r.issue = t1 - t0;
  r.total = t2 - t0;
}

template <int M, int N, int KS, int MODE>
__global__ void __launch_bounds__(512, 1) kern(long long* out, int reps) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (threadIdx.x < 32) tc::tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) tc::bar_init(&bar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  uint32_t ph = 0;
  const uint32_t sb = tc::smem_u32(sm);
  long long bi = 1LL << 60, bt = 1LL << 60, si = 0, st = 0;
  for (int r = 0; r < reps; ++r) {
    Res x;
    group<M, N, KS, MODE>(sb, &bar, ph, x);
    __syncthreads();
    if (r > 0) {
      bi = min(bi, x.issue); bt = min(bt, x.total); si += x.issue; st += x.total;
    }
  }
  if (threadIdx.x == 0) {
    out[blockIdx.x * 4 + 0] = bi;
    out[blockIdx.x * 4 + 1] = bt;
    out[blockIdx.x * 4 + 2] = si / (reps - 1);
    out[blockIdx.x * 4 + 3] = st / (reps - 1);
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(slot, 512);
}

// tcgen05.ld of a 128 x 32 fp32 block (16 KB) by 16 warps (lane quarter w%4, 8 columns w/4)
__global__ void __launch_bounds__(512, 1) ldk(long long* out, int reps, int batch) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) tc::tmem_alloc(&slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const int w = threadIdx.x >> 5, q = w & 3, cg = w >> 2;
  long long best = 1LL << 60, sum = 0;
  float acc = 0.f;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    long long t0 = clock64();
    if (batch) {   // 4 independent lds (4 x 16 KB) then one wait
      uint32_t v[4][8];
#pragma unroll
      for (int b = 0; b < 4; ++b)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[b][0]), "=r"(v[b][1]), "=r"(v[b][2]), "=r"(v[b][3]), "=r"(v[b][4]),
                       "=r"(v[b][5]), "=r"(v[b][6]), "=r"(v[b][7])
                     : "r"(((uint32_t)(32 * q) << 16) + 32 * b + 8 * cg));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int b = 0; b < 4; ++b)
        for (int j = 0; j < 8; ++j) acc += __uint_as_float(v[b][j]);
    } else {       // 4 lds each waited (the tile's ld8 pattern)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        float v[8];
        tc::ld8(((uint32_t)(32 * q) << 16) + 32 * b + 8 * cg, v);
        for (int j = 0; j < 8; ++j) acc += v[j];
      }
    }
    __syncthreads();
    long long t = clock64() - t0;
    if (r > 0) { best = min(best, t); sum += t; }
  }
  if (threadIdx.x == 0) { out[blockIdx.x * 4] = best; out[blockIdx.x * 4 + 1] = sum / (reps - 1); }
  if (acc == 12345.f) out[0] = 0;
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(slot, 512);
}

template <int M, int N, int KS, int MODE>
void run(const char* name, long long* d, int grid) {
  cudaFuncSetAttribute(kern<M, N, KS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  kern<M, N, KS, MODE><<<grid, 512, 200 * 1024>>>(d, 20);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(grid * 4);
  cudaMemcpy(h.data(), d, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost);
  double ai = 0, at = 0;
  for (int b = 0; b < grid; ++b) { ai += h[b * 4 + 2]; at += h[b * 4 + 3]; }
  const int nmma = KS * (MODE == 2 ? 1 : 3);
  const double floor = (M > 128 ? M : 128) * N / 256.0 * nmma;
  printf("%-34s grid %3d  MMAs %3d  issue min %6lld avg %8.0f | total min %6lld avg %8.0f cyc | floor %6.0f | %s\n",
         name, grid, nmma, h[0], ai / grid, h[1], at / grid, floor, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 148 * 4);
  for (int grid : {1, 148}) {
    run<128, 32, 8, 0>("hidden M128 N32 K128 3pass+coll", d, grid);
    run<128, 32, 8, 1>("hidden M128 N32 K128 3pass", d, grid);
    run<128, 32, 8, 2>("hidden M128 N32 K128 1pass", d, grid);
    run<128, 16, 8, 0>("M128 N16 K128 3pass+coll", d, grid);
    run<128, 64, 8, 0>("M128 N64 K128 3pass+coll", d, grid);
    run<128, 128, 8, 0>("M128 N128 K128 3pass+coll", d, grid);
    run<64, 32, 16, 0>("out M64 N32 K256 3pass+coll", d, grid);
    run<64, 16, 16, 0>("out M64 N16 K256 3pass+coll", d, grid);
    run<64, 64, 16, 0>("out M64 N64 K256 3pass+coll", d, grid);
    run<64, 32, 16, 2>("out M64 N32 K256 1pass", d, grid);
    run<128, 32, 1, 2>("single M128 N32 K16", d, grid);
    run<64, 32, 1, 2>("single M64 N32 K16", d, grid);
  }
  for (int batch : {0, 1}) {
    ldk<<<148, 512>>>(d, 20, batch);
    cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("tcgen05.ld 4 x (128 lanes x 32 cols) = 64 KB by 16 warps, %s: min %lld avg %lld cyc\n",
           batch ? "batched, one wait" : "each waited", h[0], h[1]);
  }
  return 0;
}
