// tc.cuh -- thin sm_100a tcgen05 / TMEM / mbarrier layer used by the tensor-core
// MLP tile (tc_mlp.cuh) and the layout probe (tools/tc_probe.cu).
//
// Operand layout convention (SWIZZLE_NONE canonical UMMA layouts): every bf16
// operand lives in shared memory as 8x8 "core blocks" of 128 contiguous bytes,
// row q of a block = 16 bytes = 8 consecutive elements of the other index.
// For a matrix X[a][b] stored with rows indexed by `a`:
//     byte(a, b) = (a/8)*SA + (b/8)*SB + (a%8)*16 + (b%8)*2
// the same bytes are
//   * a K-major operand with M/N = a, K = b:   SBO = SA, LBO = SB
//   * an MN-major operand with M/N = b, K = a: SBO = SB, LBO = SA
// so one copy of a weight or activation tile serves both a product and its
// transpose (forward vs VJP, dX vs dW) -- only the descriptor changes.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace ob {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory matrix descriptor (sm_100: version 1, no swizzle)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (Blackwell)
  return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// instruction descriptor, kind::f16 with bf16 inputs and f32 accumulation
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                       // D format f32
       | (1u << 7) | (1u << 10)          // A, B format bf16
       | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16)
       | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// the same with fp16 inputs (format 0): 11-bit significands, used by the conv tile's
// scaled two-term split (tc_conv.cuh); the MMA instruction is kind::f16 either way
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Issue helpers are executed by a whole (warp-uniform) warp so the descriptors
// stay in uniform registers; elect.sync picks the one lane that issues.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// The same MMA keeping A in the tensor core's collector buffer for the next MMA
// (fill), and one reusing it instead of re-reading shared memory (lastuse)
__device__ __forceinline__ void mma_bf16_keep_a(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_bf16_reuse_a(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// ---- single-thread forms: the caller has already elected ONE thread (elect.sync region),
// which issues a whole group of MMAs and their commit (descriptors then stay in the uniform
// datapath without a per-instruction election)
__device__ __forceinline__ void mma1(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma1_keep_a(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma1_reuse_a(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit1(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// arrive on an mbarrier when every previously issued tcgen05.mma of the electing
// lane completes (whole warp calls; the same lane as mma_bf16 commits)
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

// warp index the compiler can treat as warp-uniform
__device__ __forceinline__ int uniform_warp() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }

__device__ __forceinline__ void bar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// The same wait executed by a whole converged warp with a warp-uniform exit (vote): the
// code after it stays provably convergent, so ptxas keeps descriptor arithmetic and the
// tcgen05 operands on the uniform datapath (after the per-thread exit of bar_wait it falls
// back to vector registers, R2UR moves and an election per MMA)
__device__ __forceinline__ void bar_wait_warp(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1, P2;\n"
      "WAITU_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "vote.sync.all.pred P2, P1, 0xffffffff;\n\t"
      "@P2 bra DONEU_%=;\n\t"
      "bra WAITU_%=;\n"
      "DONEU_%=:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// TMEM allocation: called by one whole warp; the base address lands in *slot
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t base, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols)
               : "memory");
}

// 32 lanes x 8 / 16 consecutive 32-bit columns: thread i of the warp gets lane
// (lane base + i).  The warp may only address its own sub-partition
// (lanes 32*(warp%4) .. +31).
__device__ __forceinline__ void ld8(uint32_t taddr, float v[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void ld16(uint32_t taddr, float v[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 columns without the wait: several loads in flight, then one wait_ld()
__device__ __forceinline__ void ld16_async(uint32_t taddr, uint32_t r[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// the wait names the loaded registers as in/out operands, so no use of them can be
// scheduled above it (call once per register group; later calls find nothing pending)
__device__ __forceinline__ void wait_ld(uint32_t r[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                 "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]),
                 "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}

__device__ __forceinline__ void st8(uint32_t taddr, const float v[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// fp32 -> (hi, lo) bf16 pair with hi + lo == x to ~2^-17 relative (round to nearest)
__device__ __forceinline__ void split_bf16(float x, uint16_t& hi, uint16_t& lo) {
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
  hi = __bfloat16_as_ushort(h);
  lo = __bfloat16_as_ushort(l);
}

// two fp32 -> two (hi, lo) bf16 pairs, packed (element a in the low half): one
// cvt.rn.bf16x2 per pair for hi and for lo
__device__ __forceinline__ void split2_bf16(float a, float b, uint32_t& hi2, uint32_t& lo2) {
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi2) : "f"(b), "f"(a));
  const float ha = __uint_as_float(hi2 << 16), hb = __uint_as_float(hi2 & 0xffff0000u);
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo2) : "f"(b - hb), "f"(a - ha));
}

// tanh with one MUFU op: e = 2^(-2|x| log2 e) (ex2.approx on the SFU), 1/(1 + e) by a
// linear guess and three Newton steps on the FMA pipe (1 + e lies in (1, 2]).  Absolute
// error ~1e-7 everywhere (relative error grows only where |tanh| is tiny, where the
// activation's contribution is equally tiny); far below the 3-pass split's 2^-16.
__device__ __forceinline__ float tanh_1sfu(float x) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-2.8853900817779268f * fabsf(x)));
  const float d = 1.0f + e;
  float r = fmaf(-0.5f, d, 1.4571068f);      // linear guess of 1/d on [1, 2] (~9 %)
  r = fmaf(r, fmaf(-d, r, 1.0f), r);
  r = fmaf(r, fmaf(-d, r, 1.0f), r);
  r = fmaf(r, fmaf(-d, r, 1.0f), r);
  return copysignf((1.0f - e) * r, x);
}

// ---- paired fp32 arithmetic (Blackwell FFMA2 / FADD2 / FMUL2: two lanes of work per
// instruction; each lane is the IEEE round-to-nearest operation of its scalar form)
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// tanh_1sfu of two values with the FMA-pipe work paired: bit-identical to two scalar
// calls (-(1 + e) and 1 - e are formed exactly as fma(e, -1, -/+1); -0.5 d = 0.5 (-d))
__device__ __forceinline__ void tanh2_1sfu(float x0, float x1, float& y0, float& y1) {
  float e0, e1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(-2.8853900817779268f * fabsf(x0)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(-2.8853900817779268f * fabsf(x1)));
  const uint64_t e = pk2(e0, e1), m1 = pk2(-1.f, -1.f), p1 = pk2(1.f, 1.f);
  const uint64_t nd = fma2(e, m1, m1);                                // -(1 + e)
  uint64_t r = fma2(pk2(0.5f, 0.5f), nd, pk2(1.4571068f, 1.4571068f));
  r = fma2(r, fma2(nd, r, p1), r);
  r = fma2(r, fma2(nd, r, p1), r);
  r = fma2(r, fma2(nd, r, p1), r);
  const uint64_t y = mul2(fma2(e, m1, p1), r);                        // (1 - e) r
  float a, b;
  upk2(y, a, b);
  y0 = copysignf(a, x0);
  y1 = copysignf(b, x1);
}

// byte offset of element (a, b) in a core-blocked operand (see the header comment)
__host__ __device__ __forceinline__ uint32_t blk(int a, int b, uint32_t SA, uint32_t SB) {
  return (uint32_t)(a >> 3) * SA + (uint32_t)(b >> 3) * SB + (uint32_t)(a & 7) * 16u +
         (uint32_t)(b & 7) * 2u;
}

}  // namespace tc
}  // namespace ob
