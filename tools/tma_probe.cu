// tma_probe.cu -- per-SM throughput of cp.async.bulk (global -> shared, mbarrier
// complete_tx) streaming an L2-resident buffer through a ring of shared-memory
// slots, the access pattern of the CNF tensor-core tile's weight stream
// (csrc/tc_cnf.cuh).  One CTA per SM, one elected thread issues; the ring keeps
// `depth` copies in flight; chunk bytes and depth are swept.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_probe tools/tma_probe.cu
#include <cstdio>
#include <vector>
#include "../paper_2206_01298_b200/csrc/tc.cuh"
using namespace ob;

__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(128, 1) stream(const unsigned char* src, size_t src_bytes, uint32_t chunk,
                                                 int depth, int n, long long* out, int split) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bars[32];
  if (threadIdx.x == 0)
    for (int i = 0; i < depth; ++i) tc::bar_init(&bars[i], 1);
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const size_t nch = src_bytes / chunk;
    auto load = [&](int i) {
      const int s = i % depth;
      expect_tx(&bars[s], chunk);
      const uint32_t piece = chunk / split;
      for (int q = 0; q < split; ++q)
        bulk_load(sm + (size_t)s * chunk + q * piece, src + ((size_t)(i + blockIdx.x * 7) % nch) * chunk + q * piece,
                  piece, &bars[s]);
    };
    for (int i = 0; i < depth && i < n; ++i) load(i);
    for (int i = 0; i < n; ++i) {
      tc::bar_wait(&bars[i % depth], (i / depth) & 1u);
      if (i + depth < n) load(i + depth);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  const size_t bytes = 7 << 20;   // ~ the packed CNF weights (L2-resident)
  unsigned char* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  for (int split : {1, 2, 8}) {
  for (uint32_t chunk : {16384u, 32768u, 65536u, 98304u}) {
    for (int depth : {1, 2, 3}) {
      const size_t smem = (size_t)chunk * depth;
      if (smem > 200 * 1024) continue;
      cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int n = (int)((64 << 20) / chunk);   // 64 MB per CTA
      for (int rep = 0; rep < 2; ++rep) {
        stream<<<148, 128, smem>>>(src, bytes, chunk, depth, n, d, split);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> h(148);
        cudaMemcpy(h.data(), d, sizeof(long long) * 148, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (long long x : h) avg += x;
        avg /= 148;
        if (rep == 1)
          printf("split %d  chunk %6u B  depth %2d  in flight %6u B:  %7.1f B/cycle/SM  (%5.2f TB/s at 1.965 GHz, all SMs) %s\n",
                 split, chunk, depth, chunk * depth, (double)n * chunk / avg, (double)n * chunk / avg * 148 * 1.965e9 / 1e12,
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  }
  return 0;
}
