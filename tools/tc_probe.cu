// tc_probe.cu -- validates the tcgen05 descriptor / core-block conventions of
// csrc/tc.cuh on the device: D = A . B^T for K-major and MN-major A and B,
// M in {64, 128}, several N, K = 64, exact small-integer bf16 data.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2206_01298_b200/csrc/tc.cuh"
using namespace ob;

constexpr int K = 64;
__global__ void probe(int M, int N, int amn, int bmn, const float* A, const float* B, float* D) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  unsigned char* As = sm;
  unsigned char* Bs = sm + 128 * K * 2;
  // strides (bytes): rows-of-blocks stride SA, block-column stride SB
  const uint32_t aSA = amn ? (M / 8) * 128 : (K / 8) * 128, aSB = 128;
  const uint32_t bSA = bmn ? (N / 8) * 128 : (K / 8) * 128, bSB = 128;
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    if (m < M) {
      const uint32_t off = amn ? tc::blk(k, m, aSA, aSB) : tc::blk(m, k, aSA, aSB);
      *reinterpret_cast<__nv_bfloat16*>(As + off) = __float2bfloat16_rn(A[m * K + k]);
    }
    if (m < N) {
      const uint32_t off = bmn ? tc::blk(k, m, bSA, bSB) : tc::blk(m, k, bSA, bSB);
      *reinterpret_cast<__nv_bfloat16*>(Bs + off) = __float2bfloat16_rn(B[m * K + k]);
    }
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 256);
  if (threadIdx.x == 0) tc::bar_init(&bar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    const uint32_t id = tc::idesc_bf16(M, N, amn, bmn);
    for (int ks = 0; ks < K / 16; ++ks) {
      // K-major: k blocks at SB (LBO); MN-major: k blocks at SA (LBO)
      const uint64_t da = amn ? tc::sdesc(tc::smem_u32(As) + ks * 2 * aSA, aSA, aSB)
                              : tc::sdesc(tc::smem_u32(As) + ks * 2 * aSB, aSB, aSA);
      const uint64_t db = bmn ? tc::sdesc(tc::smem_u32(Bs) + ks * 2 * bSA, bSA, bSB)
                              : tc::sdesc(tc::smem_u32(Bs) + ks * 2 * bSB, bSB, bSA);
      tc::mma_bf16(tbase, da, db, id, ks > 0);
    }
    tc::commit(&bar);
  }
  tc::bar_wait(&bar, 0);
  tc::fence_after();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tc::ld8(tbase + ((uint32_t)(32 * w) << 16) + c, v);
    for (int j = 0; j < 8; ++j) D[(32 * w + lane) * 256 + c + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_free(tbase, 256);
}

int main() {
  float *A, *B, *D;
  cudaMallocManaged(&A, 128 * K * 4);
  cudaMallocManaged(&B, 256 * K * 4);
  cudaMallocManaged(&D, 128 * 256 * 4);
  srand(1);
  for (int i = 0; i < 128 * K; ++i) A[i] = (rand() % 17 - 8) / 8.0f;
  for (int i = 0; i < 256 * K; ++i) B[i] = (rand() % 17 - 8) / 8.0f;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * K * 2 + 256 * K * 2);
  int fails = 0;
  for (int M : {128, 64})
    for (int N : {32, 64, 80, 128})
      for (int amn = 0; amn < 2; ++amn)
        for (int bmn = 0; bmn < 2; ++bmn) {
          cudaMemset(D, 0, 128 * 256 * 4);
          probe<<<1, 128, 128 * K * 2 + 256 * K * 2>>>(M, N, amn, bmn, A, B, D);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("M%d N%d amn%d bmn%d: CUDA error %s\n", M, N, amn, bmn, cudaGetErrorString(e)); return 1; }
          double err = 0;
          if (M == 128) {
            for (int m = 0; m < M; ++m)
              for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[n * K + k];
                err = fmax(err, fabs(ref - D[m * 256 + n]));
              }
            printf("M%d N%d amn%d bmn%d: max err %g\n", M, N, amn, bmn, err);
            if (err > 1e-3) ++fails;
          } else {
            // locate each D(m, n) in the TMEM dump: report the lane/column of a few rows
            int found = 0, tried = 0;
            printf("M64 N%d amn%d bmn%d rows->(lane,col):", N, amn, bmn);
            for (int m = 0; m < 64; m += 7) {
              double ref0 = 0, ref1 = 0;
              for (int k = 0; k < K; ++k) { ref0 += (double)A[m * K + k] * B[0 * K + k]; ref1 += (double)A[m * K + k] * B[1 * K + k]; }
              int hl = -1, hc = -1;
              for (int l = 0; l < 128 && hl < 0; ++l)
                for (int c = 0; c + 1 < 256; ++c)
                  if (D[l * 256 + c] == ref0 && D[l * 256 + c + 1] == ref1) { hl = l; hc = c; break; }
              ++tried; if (hl >= 0) ++found;
              printf(" %d->(%d,%d)", m, hl, hc);
            }
            printf("  [%d/%d located]\n", found, tried);
          }
        }
  printf(fails ? "PROBE FAIL %d\n" : "PROBE OK\n", fails);
  return 0;
}
