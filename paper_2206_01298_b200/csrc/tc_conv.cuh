// tc_conv.cuh -- tensor-core (tcgen05 / TMEM) tile for the image-classifier ODE block
// (config C3) in the persistent explicit-RK kernels:
//   f(u, t) = conv3x3(65 -> 64)(cat(u, t)) -> relu -> conv3x3(64 -> 64), padding 1,
// on a 16x16x64 NHWC state, one image per CTA.  Same maths as the SIMT ConvAdapter
// (conv_impl.cuh; restated oracle in oracle/fields_ext.py); every contraction is an
// implicit GEMM on the tensor cores.
//
// Layout.  An operand image lives in shared memory as eight 8-channel planes over a
// LINEAR position index with one shared zero column between image rows:
//     q(y, x) = 18 + 17 y + x,   byte(q, c) = (c / 8) * kPlane + q * 16 + (c % 8) * 2
// (positions 0..17 and 290..306 are the zero halo rows, q = 18 + 17 y + 16 the zero
// column).  A 3x3 tap (dy, dx) is the position offset 17 dy + dx, i.e. a displacement of
// the operand descriptor's START ADDRESS by 16 bytes per position (SWIZZLE_NONE
// descriptors take any 16-byte-aligned start; tools/conv_probe.cu validates it).  The
// same bytes serve as
//   * the K-major A operand of a convolution   (M = 128 positions, K = channels),
//   * the MN-major A / B operands of the weight gradient (M / N = channels, K = positions).
// The 272 output positions are three M = 128 blocks (rows past 289 and zero-column rows
// are discarded).  Tap weights [cin / 8][cout][8 cin] are the K-major B of the forward
// convolution (N = cout) and the MN-major B of the transposed one (N = cin).
//
// Precision.  The field has a ReLU: its discrete adjoint jumps where a pre-activation
// crosses zero, and a bf16 two-term split (2^-16 per product) moves most C3 images past
// the 1e-4 parity bar (profiles/r02/c3_kink_split.txt).  This tile splits into fp16
// pairs instead: x 2^e = hi + lo with hi = fp16(x 2^e), lo = fp16(x 2^e - hi), where the
// per-tile power of two 2^e puts the tile's largest magnitude in [2^14, 2^15).  fp16
// carries 11 significant bits, so hi + lo represents x to 2^-22 relative for every
// element within 2^17 of the tile maximum (smaller elements keep an absolute error below
// 2^-39 of the maximum), and A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in fp32 in
// TMEM is within a few 2^-22 of the fp32 product -- the rounding level of an fp32 FMA
// chain of this length (K = 576).  Scales are exact powers of two, undone in the epilogue.
//
// The time channel (constant t over the image, zero in the halo) never enters the MMAs:
// its contribution t * sum_{taps inside the image} W1[co][tap][64] is a per-border-class
// bias added in the epilogue, and its weight gradient t * sum_q dz[q][co] ind[q][tap]
// comes from one extra N = 16 product against a constant 0 / 1 indicator image (whose
// centre-tap column is the bias gradient).
//
// Accumulation.  The tensor core adds each MMA's products into the fp32 accumulator with
// truncation (round toward zero): a chain of L MMAs loses ~L/2 ulp, systematically.  One
// accumulator per output (108 MMAs: 9 taps x 4 K slices x 3 split products) measured
// 3.7e-6 on f -- 10x the fp32 FMA chain, enough to flip ReLU decisions the fp32 tile gets
// right -- while the split alone is exact to 1e-7 (emulated in fp64).  So a convolution
// accumulates only ONE TAP per TMEM accumulator (12 MMAs, the small cross products first
// so that only the last ones truncate at the full magnitude), and the nine tap partials
// are summed in registers with round-to-nearest adds: three 64-column accumulators
// (one per M block) form a ring that warp 0 refills one tap ahead of the drain.
//
// Weights stream from L2 one tap (16 KB: hi | lo) at a time through a ring of three
// shared-memory slots filled by the TMA (cp.async.bulk + mbarrier complete_tx) two taps
// ahead of the drain; the first taps of the next convolution are prefetched behind the
// current one.  Parameter cotangents are formed per VJP in TMEM (M = 64 x N = 64 per tap,
// K = 272 positions; two taps share 64 columns, see wgrad) and added to the CTA's private
// mu slot while the next taps' MMAs run (fixed order: bit-reproducible).
//
// The tile owns its RK steps (kOwnsStep): stage sums and cotangent combinations are formed
// in registers (same order and roundings as the generic loops) and split straight into
// the operand image; state-sized vectors live in L2-resident global scratch.
#pragma once

#include <cuda_fp16.h>
#include <cstdio>

#include "rk_impl.cuh"
#include "tc.cuh"

namespace ob {

#ifndef OB_CONV_GF
#define OB_CONV_GF 1   // taps per TMEM partial of the forward convolutions (experiments: 3, 9)
#endif
#ifndef OB_CONV_GT
#define OB_CONV_GT 3   // taps per TMEM partial of the transposed convolutions (experiments: 1, 9)
#endif

namespace conv_tc {
constexpr int kNP = 313;                       // positions per plane (odd: 16-byte stores of 8
                                               // consecutive planes hit distinct banks)
constexpr uint32_t kPlane = kNP * 16u;         // bytes per 8-channel plane
constexpr uint32_t kPart = 8u * kPlane;        // hi (or lo) part of an image tile
constexpr uint32_t kTile = 2u * kPart;         // hi | lo
constexpr int kQ0 = 18;                        // position of pixel (0, 0)
constexpr int kRow = 17;                       // positions per image row (16 pixels + zero column)
constexpr int kNOut = 16 * kRow;               // output positions 18 .. 289
constexpr uint32_t kWPl = 64u * 16u;           // weight plane: 64 rows x 8 channels
constexpr uint32_t kTapHalf = 8u * kWPl;       // one tap, hi (or lo): 8 KB
constexpr uint32_t kTap = 2u * kTapHalf;       // hi | lo
constexpr int kNS = 3;                         // weight ring slots
// packed image (global): header | border-class time bias | indicator image | tap weights
constexpr uint32_t kPkInvW = 0;                // float[2]: 2^-e of each conv's weights
constexpr uint32_t kPkTB = 64;                 // float[9][64]
constexpr uint32_t kPkInd = 4096;              // 2 planes (hi only)
constexpr uint32_t kPkW = 16384;               // [2 convs][9 taps][hi | lo]
constexpr uint32_t kPacked = kPkW + 2u * 9u * kTap;
// shared memory (bytes from the start of dynamic shared memory)
constexpr uint32_t kT0 = 0;                    // input image x / cotangent v
constexpr uint32_t kT1 = kTile;                // hidden image h / its cotangent dz
constexpr uint32_t kInd = 2u * kTile;          // indicator image (2 planes, padded)
constexpr uint32_t kRing = kInd + 10112u;
constexpr uint32_t kMask = kRing + kNS * kTap; // relu mask: 4 x uint16 per position
constexpr uint32_t kTBs = kMask + 2560u;       // float[9][64]
constexpr uint32_t kBias = kTBs + 2304u;       // float b1[64] | b2[64]
constexpr uint32_t kRed = kBias + 512u;        // float[2][16] block-max scratch
constexpr uint32_t kBars = kRed + 128u;        // full[3] acc_full[6] acc_empty[6] dw_full[5] wempty[3]
constexpr uint32_t kSlot = kBars + 192u;
constexpr uint32_t kTotal = (kSlot + 16u + 127u) / 128u * 128u;
static_assert(kRing % 128 == 0 && kInd % 128 == 0, "alignment");
static_assert(kTotal <= 227u * 1024u, "shared memory");
// TMEM columns: convolution accumulator ring (one 64-column tap partial per M block),
// weight-gradient tiles
constexpr uint32_t kAcc = 0;
constexpr uint32_t kDw = 192;                  // 5 x 64 columns: taps (2 j, 2 j + 1) | (8, indicator)

__host__ __device__ constexpr int tap_off(int s) { return (s / 3 - 1) * kRow + (s % 3 - 1); }
__device__ __forceinline__ bool q_valid(int q) {
  return q >= kQ0 && q < kQ0 + kNOut && (q - kQ0) % kRow != 16;
}
__device__ __forceinline__ int q_pixel(int q) { return ((q - kQ0) / kRow) * 16 + (q - kQ0) % kRow; }
__device__ __forceinline__ int pixel_q(int p) { return kQ0 + (p >> 4) * kRow + (p & 15); }
// border class of a pixel (3 x 3: first / interior / last row and column)
__device__ __forceinline__ int q_class(int q) {
  const int y = (q - kQ0) / kRow, x = (q - kQ0) % kRow;
  return (y == 0 ? 0 : y == 15 ? 2 : 1) * 3 + (x == 0 ? 0 : x == 15 ? 2 : 1);
}
__host__ __device__ constexpr bool tap_in_class(int s, int cls) {
  const int dy = s / 3 - 1, dx = s % 3 - 1, ry = cls / 3, rx = cls % 3;
  return !(ry == 0 && dy < 0) && !(ry == 2 && dy > 0) && !(rx == 0 && dx < 0) && !(rx == 2 && dx > 0);
}

// two fp32 -> packed fp16 (hi, lo) pairs (element a in the low half)
__device__ __forceinline__ void split2_f16(float a, float b, uint32_t& hi2, uint32_t& lo2) {
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi2) : "f"(b), "f"(a));
  const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&hi2));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo2) : "f"(b - h.y), "f"(a - h.x));
}
// eight consecutive channels (already scaled) -> one 16-byte row of the hi and lo planes
__device__ __forceinline__ void store8(unsigned char* tile, uint32_t off, const float v[8]) {
  uint4 h, l;
  split2_f16(v[0], v[1], h.x, l.x);
  split2_f16(v[2], v[3], h.y, l.y);
  split2_f16(v[4], v[5], h.z, l.z);
  split2_f16(v[6], v[7], h.w, l.w);
  *reinterpret_cast<uint4*>(tile + off) = h;
  *reinterpret_cast<uint4*>(tile + kPart + off) = l;
}
// power of two s with s * m in [2^14, 2^15) (1 for m = 0 or non-finite), and 1 / s
__device__ __forceinline__ void pow2_scale(float m, float& s, float& inv) {
  int ex = (int)((__float_as_uint(m) >> 23) & 0xffu) - 127;
  if (m == 0.0f || ex == 128) ex = 14;
  ex = max(-100, min(100, ex));
  s = __uint_as_float((uint32_t)(127 + 14 - ex) << 23);
  inv = __uint_as_float((uint32_t)(127 - 14 + ex) << 23);
}

__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}
#ifdef OB_DEBUG_WATCHDOG
// debugging aid: a wait that reports the barrier it starved on and gives up
__device__ __noinline__ void wd_report(int tag, int idx, uint32_t parity) {
  if ((threadIdx.x & 31) == 0)
    printf("WATCHDOG block %d warp %d tag %d barrier %d parity %u\n", (int)blockIdx.x, (int)(threadIdx.x >> 5), tag, idx,
           parity);
}
__device__ __forceinline__ void wd_wait(uint64_t* bar, uint32_t parity, int tag, uint64_t* base) {
  for (long long n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1, P2;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "vote.sync.all.pred P2, P1, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P2;\n\t}\n"
        : "=r"(ok)
        : "r"(tc::smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (n > (1LL << 21)) {
      wd_report(tag, (int)(bar - base), parity);
      return;
    }
  }
}
#define OB_WAIT(bar, parity, tag) conv_tc::wd_wait(bar, parity, tag, bars())
#else
#define OB_WAIT(bar, parity, tag) tc::bar_wait_warp(bar, parity)
#endif
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}\n"
               : "=r"(p));
  return p != 0;
}
}  // namespace conv_tc

// dynamic shared memory of the tile (shared with the other tensor-core tiles)
extern __shared__ __align__(128) unsigned char ob_tc_smem[];

template <typename T>
struct TcConvAdapter {
  static_assert(sizeof(T) == 4, "tensor-core conv tile is fp32");
  static constexpr bool kHasJvp = false;
  static constexpr bool kScaledVjp = false;   // vjp returns J^T w; mu += h P^T w
  static constexpr int kCombineBatch = 4;
  static constexpr bool kOwnsStep = true;     // step() / reverse_step() replace the generic stage loops
  static constexpr uint32_t kCols = 512;
  static constexpr int kN = 256 * 64;         // state elements of one image

  const RkParams<T>& p;
  float tcur;
  float* xin;                  // field input of the generic field ops, fp32 [256 pixels][64] (global)
  uint32_t wuse;               // weight-tap ordinal of the next convolution's first tap (9 per conv)
  int pref_layer;              // conv whose first three taps are already on their way (-1: none)
  uint32_t ta;                 // drain groups so far (accumulator barrier parity)
  uint32_t ndw;                // weight-gradient products so far (dw_full parity)
  uint32_t red_par;
  float invw[2];               // 2^-e of the packed conv weights
  float inv0, inv1;            // 2^-e of the images in T0 / T1
  PhaseTimer pt;               // OB_FLAG_PHASE_TIMING: 8 stage sums / splits, 10 conv MMA + drain,
                               // 11 epilogues, 12 weight gradients, 14 image loads

  OB_DEV unsigned char* sm() const { return ob_tc_smem; }
  OB_DEV uint64_t* bars() const { return reinterpret_cast<uint64_t*>(ob_tc_smem + conv_tc::kBars); }
  OB_DEV uint64_t* full(uint32_t s) const { return bars() + s; }
  OB_DEV uint64_t* acc_full(int slot) const { return bars() + 3 + slot; }
  OB_DEV uint64_t* acc_empty(int slot) const { return bars() + 9 + slot; }
  OB_DEV uint64_t* dw_full(int j) const { return bars() + 15 + j; }
  OB_DEV uint64_t* wempty(uint32_t s) const { return bars() + 20 + s; }
  OB_DEV const unsigned char* packed() const { return reinterpret_cast<const unsigned char*>(p.packed); }
  OB_DEV float* tb() const { return reinterpret_cast<float*>(ob_tc_smem + conv_tc::kTBs); }
  OB_DEV float* bias() const { return reinterpret_cast<float*>(ob_tc_smem + conv_tc::kBias); }

  OB_DEV TcConvAdapter(const RkParams<T>& p_, const Weights<T>&, MlpSmem<T>&, T*, int, int)
      : p(p_), tcur(0.f), wuse(0), pref_layer(-1), ta(0), ndw(0), red_par(0), inv0(1.f), inv1(1.f),
        pt(p_.prof ? p_.phase : nullptr) {
    xin = reinterpret_cast<float*>(p.cnf_pre) + (long long)blockIdx.x * p.cnf_pre_stride;
    // the kernel zeroed all dynamic shared memory: image halos / zero columns stay zero
    if (threadIdx.x < 32) tc::tmem_alloc(reinterpret_cast<uint32_t*>(ob_tc_smem + conv_tc::kSlot), kCols);
    if (threadIdx.x == 0) {
      for (int s = 0; s < 3; ++s) {
        tc::bar_init(full(s), 1);
        tc::bar_init(wempty(s), 6);                  // the six issuing warps release a weight slot
      }
      for (int s = 0; s < 6; ++s) {
        tc::bar_init(acc_full(s), 1);
        tc::bar_init(acc_empty(s), kThreads / 32);   // every warp drains its share of a partial
      }
      for (int j = 0; j < 5; ++j) tc::bar_init(dw_full(j), 1);
    }
    const float* hdr = reinterpret_cast<const float*>(packed());
    invw[0] = hdr[0];
    invw[1] = hdr[1];
    for (int i = threadIdx.x; i < 9 * 64; i += blockDim.x) tb()[i] = hdr[conv_tc::kPkTB / 4 + i];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) bias()[i] = float(p.W.bias[i >> 6][i & 63]);
    const uint4* ind = reinterpret_cast<const uint4*>(packed() + conv_tc::kPkInd);
    for (int i = threadIdx.x; i < (int)(2 * conv_tc::kPlane / 16); i += blockDim.x)
      reinterpret_cast<uint4*>(ob_tc_smem + conv_tc::kInd)[i] = ind[i];
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (threadIdx.x == 0 && p.status && *reinterpret_cast<volatile uint32_t*>(ob_tc_smem + conv_tc::kSlot) != 0u)
      set_status(p.status, OB_ERR_UNSUPPORTED, -2);   // TMEM not at column 0: shared SM
    if (threadIdx.x == 0 && p.status && tc::smem_u32(ob_tc_smem) != p.tile_aux)
      set_status(p.status, OB_ERR_UNSUPPORTED, -(int)tc::smem_u32(ob_tc_smem));   // the launcher's base is wrong: -(actual)
  }

  OB_DEV int nin() const { return p.d.N; }
  OB_DEV void set_scratch(T*, int) {}
  OB_DEV void jvp(const T*, T*) {}
  OB_DEV void put(int, int j, T v) { xin[j] = float(v); }
  OB_DEV void put_time(double t) { tcur = float(t); }

  // generic-proxy shared-memory writes -> visible to the MMA; TMEM reads retired
  OB_DEV void sync_issue() {
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }

  // ---- thread "units": unit u = threadIdx.x + 512 k (k < 4) is pixel u / 8, channels
  // 8 (u % 8) .. + 7, i.e. the eight consecutive floats at 8 u of a state-sized vector
  OB_DEV static int unit_off(int k) { return (int)(threadIdx.x + kThreads * k) * 8; }
  OB_DEV static void ld8(const T* g, float v[8]) {
    const float4 a = *reinterpret_cast<const float4*>(g), b = *reinterpret_cast<const float4*>(g + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  OB_DEV static void st8(T* g, const float v[8]) {
    *reinterpret_cast<float4*>(g) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(g + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }

  // block-wide maximum of |values| -> the tile's power-of-two scale (one barrier; the
  // scratch is double-buffered so consecutive reductions do not race)
  OB_DEV void tile_scale(float m, float& s, float& inv) {
    float* red = reinterpret_cast<float*>(ob_tc_smem + conv_tc::kRed) + 16 * red_par;
    red_par ^= 1u;
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    float mm = 0.f;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) mm = fmaxf(mm, red[w]);
    conv_tc::pow2_scale(mm, s, inv);
  }

  // the thread's units of an image (registers) -> split image tile; returns 2^-e of the tile
  OB_DEV float split_units(float v[4][8], uint32_t tile) {
    float m = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int e = 0; e < 8; ++e) m = fmaxf(m, fabsf(v[k][e]));
    float s, inv;
    tile_scale(m, s, inv);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int u = threadIdx.x + kThreads * k;
#pragma unroll
      for (int e = 0; e < 8; ++e) v[k][e] *= s;
      conv_tc::store8(sm() + tile, (uint32_t)(u & 7) * conv_tc::kPlane + (uint32_t)conv_tc::pixel_q(u >> 3) * 16u, v[k]);
    }
    return inv;
  }
  // fp32 image [256 pixels][64] (global) -> split image tile
  OB_DEV float load_image(uint32_t tile, const T* src) {
    float v[4][8];
#pragma unroll
    for (int k = 0; k < 4; ++k) ld8(src + unit_off(k), v[k]);
    return split_units(v, tile);
  }

  // ---- weight stream: tap ordinal o lands in ring slot o % 3 (caller: the slot is free)
  // (whole warp; one elected lane issues)
  OB_DEV void load_tap(uint32_t o, int layer, int s) {
    const uint32_t slot = o % 3u;
    if (conv_tc::elect_one()) {
      conv_tc::bar_expect_tx(full(slot), conv_tc::kTap);
      conv_tc::bulk_load(sm() + conv_tc::kRing + slot * conv_tc::kTap,
                         packed() + conv_tc::kPkW + (uint32_t)(layer * 9 + s) * conv_tc::kTap, conv_tc::kTap,
                         full(slot));
    }
    __syncwarp();
  }
  // one tap of one M block (all lanes of the issuing warp; elect.sync inside the MMA
  // helpers) into accumulator `slot`: the 128 positions 18 + 128 b ..  Cross products first:
  // within a fresh accumulator they stay 2^-11 of its final size, so only the A_hi B_hi
  // products truncate at full magnitude.
  template <bool TR, uint32_t TILE>
  OB_DEV void issue_unit(int s, int b, int slot, bool fresh) {
    const uint32_t sb = tc::smem_u32(ob_tc_smem);
    constexpr uint32_t id = tc::idesc_f16(128, 64, false, TR);
    const int off = TR ? -conv_tc::tap_off(s) : conv_tc::tap_off(s);
    const uint32_t wb = sb + conv_tc::kRing + (uint32_t)(s % 3) * conv_tc::kTap;
    const uint32_t a0 = sb + TILE + (uint32_t)(conv_tc::kQ0 + 128 * b + off) * 16u;
    const uint64_t Ah = tc::sdesc(a0, conv_tc::kPlane, 128);
    const uint64_t Al = Ah + (conv_tc::kPart >> 4);
    const uint64_t Bh = TR ? tc::sdesc(wb, 128, conv_tc::kWPl)      // MN-major: N = cin planes, K = cout rows
                           : tc::sdesc(wb, conv_tc::kWPl, 128);     // K-major: N = cout rows, K = cin planes
    const uint64_t Bl = Bh + (conv_tc::kTapHalf >> 4);
    constexpr uint64_t ak = (2u * conv_tc::kPlane) >> 4, bk = TR ? (256u >> 4) : ((2u * conv_tc::kWPl) >> 4);
    const uint32_t d = conv_tc::kAcc + 64u * (uint32_t)slot;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) tc::mma_bf16(d, Al + ks * ak, Bh + ks * bk, id, (ks > 0 || !fresh) ? 1u : 0u);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#ifdef OB_EXP_NO_COLLECTOR
      tc::mma_bf16(d, Ah + ks * ak, Bl + ks * bk, id, 1u);
      tc::mma_bf16(d, Ah + ks * ak, Bh + ks * bk, id, 1u);
#else
      tc::mma_bf16_keep_a(d, Ah + ks * ak, Bl + ks * bk, id, 1u);
      tc::mma_bf16_reuse_a(d, Ah + ks * ak, Bh + ks * bk, id, 1u);
#endif
    }
  }

  // v[b][.] = sum over taps and channels of image(TILE)[q +/- off(tap)] x W_layer[tap] for
  // the thread's rows (M block b, lane quarter, lane) and 16 output channels (TR: the input
  // cotangent of the convolution).  G taps accumulate in TMEM between drains: G = 1 where the
  // result decides ReLU masks downstream (the forward convolutions), G = 3 (a stencil row)
  // for the transposed ones, whose error only moves the cotangent smoothly.
  //
  // The product is bound by MMA ISSUE, not by the tensor pipe (shrinking every MMA to
  // N = 16 left its time unchanged; ~70-100 cycles of issue per tcgen05.mma from one warp
  // against 32 of execution), so SIX warps issue: each M block has two accumulators (one per
  // parity of the drain group) and warp parity * 3 + b owns accumulator (parity, b) -- a
  // group's MMAs all come from one thread, so its fresh MMA is ordered before the
  // accumulating ones.  At the top of tap s the issuing warps queue tap s + 1, then every
  // warp drains the group that tap s completes.  Warp 0
  // also streams the weights: tap s + 2 into the ring slot tap s - 1 released.  `next`: the
  // conv whose first taps are prefetched behind this product (-1: none).  Tap ordinals
  // advance by 9 per convolution: tap s sits in ring slot s % 3.
  template <bool TR, int G, uint32_t TILE>
  OB_DEV void conv(int layer, int next, float v[3][16]) {
    const int w = tc::uniform_warp();
    const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 3, cg = threadIdx.x >> 7;
    const uint32_t W0 = wuse;
    if (w == 0 && pref_layer != layer)
      for (int j = 0; j < 3; ++j) load_tap(W0 + j, layer, j);
    const uint32_t G0 = ta;     // drain groups so far: accumulator barrier phases
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int e = 0; e < 16; ++e) v[b][e] = 0.f;
    // (warp b < 3) tap s2 of block b: wait for the weights and, for a fresh accumulator, for
    // every warp's drain of its previous partial (two groups ago)
    // Every issuing warp observes EVERY phase of the weight barriers, and a slot is refilled
    // only when all six have released it: a warp that skipped a tap could otherwise test a
    // parity one phase ahead of the barrier, which reads as "complete" (measured: a hang).
    auto issue = [&](int s2) {
      const uint32_t gg = G0 + (uint32_t)(s2 / G);
      OB_WAIT(full(s2 % 3), ((W0 + s2) / 3u) & 1u, 2);
      if ((int)(gg & 1u) != w / 3) {   // the other warp of this block issues this group
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(wempty(s2 % 3))) : "memory");
        __syncwarp();
        return;
      }
      tc::fence_after();
      const int slot = w;              // = parity * 3 + block
      const bool fresh = s2 % G == 0;
      if (fresh && gg >= 2) {
        OB_WAIT(acc_empty(slot), ((gg >> 1) - 1) & 1u, 1);
        tc::fence_after();
      }
      issue_unit<TR, TILE>(s2, w % 3, slot, fresh);
      if (s2 % G == G - 1) tc::commit(acc_full(slot));
      tc::commit(wempty(s2 % 3));
    };
    if (w < 6) issue(0);
#pragma unroll 1
    for (int s = 0; s < 9; ++s) {
      if (w == 0 && s >= 1 && s + 2 < 9) {   // tap s - 1 completed: its ring slot takes tap s + 2
        OB_WAIT(wempty((s - 1) % 3), ((W0 + s - 1) / 3u) & 1u, 3);
        load_tap(W0 + s + 2, layer, s + 2);
      }
      if (w < 6 && s + 1 < 9) issue(s + 1);
      if (s % G != G - 1) continue;
      const uint32_t gg = G0 + (uint32_t)(s / G);
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int slot = (int)(gg & 1u) * 3 + b;
        OB_WAIT(acc_full(slot), (gg >> 1) & 1u, 4);
        tc::fence_after();
        if (b < 2 || q == 0) {   // block 2: only rows 0..15 (positions 274..289) are pixels
          float r[16];
          tc::ld16(((uint32_t)(32 * q) << 16) + conv_tc::kAcc + 64u * (uint32_t)slot + 16u * cg, r);
#pragma unroll
          for (int e = 0; e < 16; ++e) v[b][e] += r[e];
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(acc_empty(slot))) : "memory");
      }
    }
    ta = G0 + 9 / G;
    // every tap's MMAs completed (the last drain saw them); the last three release barriers
    // are consumed here so the phases stay aligned with the tap ordinals
    if (w == 0)
      for (int j = 6; j < 9; ++j) OB_WAIT(wempty(j % 3), ((W0 + j) / 3u) & 1u, 5);
    wuse = W0 + 9;
    pref_layer = next;
    if (w == 0 && next >= 0)
      for (int j = 0; j < 3; ++j) load_tap(wuse + j, next, j);
  }

  // ---- weight gradients.  D_s[cout][cin] = sum_q cot[q][cout] in[q + off(s)][cin] for all
  // nine taps.  An M = 64 accumulator occupies lanes 32 g + (0..15) of its columns and may
  // equally sit at lane offset 16 (tools/conv_probe.cu), so taps 2 j and 2 j + 1 share the 64
  // columns kDw + 64 j; the indicator product D[cout][16] = sum_q cot[q][cout] ind[q][.]
  // takes the free upper half beside tap 8.  Warp 0 issues the five column groups in turn,
  // committing each; every warp adds a finished group to mu while the next one runs:
  //   mu_layer[cout][tap][cin] += sc * D_tap, and from the indicator product (scale sci)
  //   the bias gradient (centre tap: every pixel) and, for conv 1, the time-channel weight
  //   gradient t * sum_q dz[q][co] ind[q][tap].
  // Warp (quarter, group): lane L holds row co = 16 quarter + L % 16 of tap 2 j + L / 16,
  // input channels 16 group .. + 15.
  OB_DEV static uint32_t dw_addr(int s) { return conv_tc::kDw + 64u * (uint32_t)(s >> 1) + ((uint32_t)(16 * (s & 1)) << 16); }
  template <uint32_t cot, uint32_t in>
  OB_DEV void wgrad(T* mu, int layer, float sc, float sci) {
    const uint32_t par = ndw & 1u;
    ++ndw;
#ifdef OB_EXP_NO_WGRAD
    return;
#endif
    const int w = tc::uniform_warp();
    const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 3, cg = threadIdx.x >> 7;
    const int co = 16 * q + (lane & 15);
    T* row = mu + p.d.mwoff[layer] + (long long)co * p.d.ldm[layer];
    auto issue = [&](int s) {   // tap s (s = 9: the indicator product)
      const uint32_t sb = tc::smem_u32(ob_tc_smem);
      constexpr uint32_t id = tc::idesc_f16(64, 64, true, true), id16 = tc::idesc_f16(64, 16, true, true);
      constexpr int KS = conv_tc::kNOut / 16;
      const uint32_t d = dw_addr(s);
      uint32_t a0 = sb + cot + (uint32_t)conv_tc::kQ0 * 16u;
      uint32_t b0 = sb + (s < 9 ? in + (uint32_t)(conv_tc::kQ0 + conv_tc::tap_off(s)) * 16u
                                : conv_tc::kInd + (uint32_t)conv_tc::kQ0 * 16u);
#ifndef OB_EXP_NO_UNIFORM
      a0 = __shfl_sync(0xffffffffu, a0, 0);
      b0 = __shfl_sync(0xffffffffu, b0, 0);
#endif
      const uint64_t Ah = tc::sdesc(a0, 128, conv_tc::kPlane);
      const uint64_t Al = Ah + (conv_tc::kPart >> 4);
      if (s < 9) {
        const uint64_t Bh = tc::sdesc(b0, 128, conv_tc::kPlane);
        const uint64_t Bl = Bh + (conv_tc::kPart >> 4);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)   // cross products first (see issue_unit)
          tc::mma_bf16(d, Al + 16u * ks, Bh + 16u * ks, id, ks > 0 ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          tc::mma_bf16_keep_a(d, Ah + 16u * ks, Bl + 16u * ks, id, 1u);
          tc::mma_bf16_reuse_a(d, Ah + 16u * ks, Bh + 16u * ks, id, 1u);
        }
      } else {
        const uint64_t Bi = tc::sdesc(b0, 128, conv_tc::kPlane);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) tc::mma_bf16(d, Al + 16u * ks, Bi + 16u * ks, id16, ks > 0 ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) tc::mma_bf16(d, Ah + 16u * ks, Bi + 16u * ks, id16, 1u);
      }
    };
    auto flush = [&](int j) {   // column group j: taps 2 j (lanes 0..15 of a quarter) and 2 j + 1
      const int s = 2 * j + (lane >> 4);
      // the mu values are loaded BEFORE the wait: their L2 round trip hides behind the MMAs
      float4* dst = reinterpret_cast<float4*>(row + (s < 9 ? s : 0) * 68 + 16 * cg);
      float4 m4[4];
#ifndef OB_EXP_NO_WFLUSH
      if (s < 9) {
#pragma unroll
        for (int e = 0; e < 4; ++e) m4[e] = dst[e];
      }
#endif
      OB_WAIT(dw_full(j), par, 6);
      tc::fence_after();
      float v[16];
      tc::ld16(((uint32_t)(32 * q) << 16) + conv_tc::kDw + 64u * (uint32_t)j + 16u * cg, v);
#ifdef OB_EXP_NO_WFLUSH
      return;
#endif
      if (s < 9) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          m4[e].x = fmaf(sc, v[4 * e], m4[e].x);
          m4[e].y = fmaf(sc, v[4 * e + 1], m4[e].y);
          m4[e].z = fmaf(sc, v[4 * e + 2], m4[e].z);
          m4[e].w = fmaf(sc, v[4 * e + 3], m4[e].w);
          dst[e] = m4[e];
        }
      } else if (cg == 0) {   // the indicator product
        mu[p.d.mboff[layer] + co] += T(sci * v[4]);
        if (layer == 0) {
#pragma unroll
          for (int t = 0; t < 9; ++t) row[t * 68 + 64] += T(sci * tcur * v[t]);
        }
      }
    };
    // Issue-bound like the convolutions: warps 0 and 1 issue alternate column groups (0, 2, 4
    // and 1, 3), each before it flushes the group two back, so the flushes of a pair overlap
    // the MMAs of the next pair (five warps issuing one group each measured slower: the
    // groups then finish together and no flush overlaps the MMAs).
#pragma unroll 1
    for (int j = 0; j < 5; ++j) {
      if (w < 2) {
        if ((j & 1) == w) {
          issue(2 * j);
          issue(2 * j + 1);
          tc::commit(dw_full(j));
        }
        if (j >= 2) flush(j - 2);
      } else {
        flush(j);
      }
    }
    if (w < 2) {
      flush(3);
      flush(4);
    }
    // the next convolution's accumulators (columns 0..383) overlap these tiles: every
    // warp's flush must have read them before any warp issues into them
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }

  // ---- convolution epilogues.  Thread rows: position 18 + 128 b + 32 quarter + lane of M
  // block b; channels 16 group .. + 15.
  // split the 16 channels of each valid row into image tile T1 (scaled by the tile maximum)
  OB_DEV float store_hidden(float v[3][16]) {
    const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 3, cg = threadIdx.x >> 7;
    float m = 0.f;
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int e = 0; e < 16; ++e) m = fmaxf(m, fabsf(v[b][e]));
    float s, inv;
    tile_scale(m, s, inv);
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int pos = conv_tc::kQ0 + 128 * b + 32 * q + lane;
      if (!conv_tc::q_valid(pos)) continue;
#pragma unroll
      for (int e = 0; e < 16; ++e) v[b][e] *= s;
      conv_tc::store8(sm() + conv_tc::kT1, (uint32_t)(2 * cg) * conv_tc::kPlane + (uint32_t)pos * 16u, v[b]);
      conv_tc::store8(sm() + conv_tc::kT1, (uint32_t)(2 * cg + 1) * conv_tc::kPlane + (uint32_t)pos * 16u, v[b] + 8);
    }
    return inv;
  }

  // T1 = relu(conv1(T0) + b1 + t * border-class time bias) from the image in T0 (scale inv0);
  // the relu mask is kept for the VJP
  OB_DEV void hidden_tile() {
    float v[3][16];
    conv<false, OB_CONV_GF, conv_tc::kT0>(0, 1, v);
    pt.mark(10);
    const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 3, cg = threadIdx.x >> 7;
    const float sc = inv0 * invw[0];
    uint16_t* mask = reinterpret_cast<uint16_t*>(sm() + conv_tc::kMask);
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int pos = conv_tc::kQ0 + 128 * b + 32 * q + lane;
      const bool ok = conv_tc::q_valid(pos);
      const float* tbc = tb() + (ok ? conv_tc::q_class(pos) : 0) * 64 + 16 * cg;
      uint32_t bits = 0;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float z = fmaf(v[b][e], sc, bias()[16 * cg + e]) + tcur * tbc[e];
        const bool on = ok && z > 0.0f;
        v[b][e] = on ? z : 0.0f;
        bits |= on ? (1u << e) : 0u;
      }
      if (ok) mask[pos * 4 + cg] = (uint16_t)bits;
    }
    inv1 = store_hidden(v);
    pt.mark(11);
  }

  // f(image in T0, tcur) -> out [256 pixels][64] (global)
  OB_DEV void eval_tile(T* out) {
    hidden_tile();
    sync_issue();
    float v[3][16];
    conv<false, OB_CONV_GF, conv_tc::kT1>(1, 0, v);
    pt.mark(10);
    const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 3, cg = threadIdx.x >> 7;
    const float sc = inv1 * invw[1];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int pos = conv_tc::kQ0 + 128 * b + 32 * q + lane;
      if (!conv_tc::q_valid(pos)) continue;
      float4* dst = reinterpret_cast<float4*>(out + conv_tc::q_pixel(pos) * 64 + 16 * cg);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        dst[e] = make_float4(fmaf(v[b][4 * e], sc, bias()[64 + 16 * cg + 4 * e]),
                             fmaf(v[b][4 * e + 1], sc, bias()[64 + 16 * cg + 4 * e + 1]),
                             fmaf(v[b][4 * e + 2], sc, bias()[64 + 16 * cg + 4 * e + 2]),
                             fmaf(v[b][4 * e + 3], sc, bias()[64 + 16 * cg + 4 * e + 3]));
    }
    tc::fence_before();
    __syncthreads();
    pt.mark(11);
  }

  // VJP at the stage state xsrc (global fp32 image): loadv fills the thread's units of the
  // cotangent w; out(pos, cg, j[16]) receives J^T w for one valid row (16 channels);
  // mu += hs P^T w (skipped when mu is null)
  template <class LoadV, class Out>
  OB_DEV void vjp_core(const T* xsrc, LoadV loadv, T* mu, float hs, bool want_jtv, Out out) {
    inv0 = load_image(conv_tc::kT0, xsrc);           // T0 = x
    sync_issue();
    pt.mark(14);
    hidden_tile();                                   // T1 = h1, mask
    sync_issue();
    float invv;
    {
      float vv[4][8];
      loadv(vv);
      invv = split_units(vv, conv_tc::kT0);          // T0 = v
    }
    sync_issue();
    pt.mark(8);
    if (mu) wgrad<conv_tc::kT0, conv_tc::kT1>(mu, 1, hs * invv * inv1, hs * invv);   // dW2 += h v (x) h1, db2
    pt.mark(12);
    const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 3, cg = threadIdx.x >> 7;
    {                                                // dz1 = relu'(z1) conv2^T v -> T1 (h1 is dead)
      float v[3][16];
      conv<true, OB_CONV_GT, conv_tc::kT0>(1, 0, v);
      pt.mark(10);
      const float sc = invv * invw[1];
      const uint16_t* mask = reinterpret_cast<const uint16_t*>(sm() + conv_tc::kMask);
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int pos = conv_tc::kQ0 + 128 * b + 32 * q + lane;
        const uint32_t bits = conv_tc::q_valid(pos) ? mask[pos * 4 + cg] : 0u;
#pragma unroll
        for (int e = 0; e < 16; ++e) v[b][e] = ((bits >> e) & 1u) ? v[b][e] * sc : 0.0f;
      }
      inv1 = store_hidden(v);
    }
    sync_issue();
    pt.mark(11);
    if (mu) {   // dW1 += h dz1 (x) x; time channel and db1 from the indicator product
      inv0 = load_image(conv_tc::kT0, xsrc);         // T0 = x again
      sync_issue();
      pt.mark(14);
      wgrad<conv_tc::kT1, conv_tc::kT0>(mu, 0, hs * inv1 * inv0, hs * inv1);
      pt.mark(12);
    }
    if (want_jtv) {
      float v[3][16];
      conv<true, OB_CONV_GT, conv_tc::kT1>(0, 0, v);            // J^T w = conv1^T dz1 (state channels)
      pt.mark(10);
      const float sc = inv1 * invw[0];
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int pos = conv_tc::kQ0 + 128 * b + 32 * q + lane;
        if (!conv_tc::q_valid(pos)) continue;
#pragma unroll
        for (int e = 0; e < 16; ++e) v[b][e] *= sc;
        out(pos, cg, v[b]);
      }
    }
    tc::fence_before();
    __syncthreads();
    pt.mark(11);
  }

  // ---- generic field ops (field_op_kernel): input through put() -> xin
  OB_DEV void eval(T* out) {
    inv0 = load_image(conv_tc::kT0, xin);
    sync_issue();
    eval_tile(out);
  }
  OB_DEV void vjp(const T* w, T* jtv, T* mu, double h, int) {
    vjp_core(
        xin,
        [&](float vv[4][8]) {
#pragma unroll
          for (int k = 0; k < 4; ++k) ld8(w + unit_off(k), vv[k]);
        },
        mu, float(h), jtv != nullptr,
        [&](int pos, int cg, const float* j) {
          float4* dst = reinterpret_cast<float4*>(jtv + conv_tc::q_pixel(pos) * 64 + 16 * cg);
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = make_float4(j[4 * e], j[4 * e + 1], j[4 * e + 2], j[4 * e + 3]);
        });
  }

  // ---- one explicit RK step of the image (explicit_rk_step, integrators.py:196-222): the
  // generic rk_step_tile with the stage sums formed in registers (same order, mul then add,
  // exact zeros skipped) and split straight into T0.  u, ks, rec: global memory.
  OB_DEV bool step(T* u, double t, double h, bool carry, T* rec, int row0, bool keep_last) {
    const int s = p.s;
    const long long vec = (long long)p.B * kN;
    T* ks = p.scratch + blockIdx.x * p.scratch_stride;
    T* recb = rec ? rec + (long long)row0 * kN : nullptr;
    for (int i = 0; i < s; ++i) {
      float v[4][8];
#pragma unroll
      for (int k = 0; k < 4; ++k) ld8(u + unit_off(k), v[k]);
      for (int qq = 0; qq < i; ++qq) {
        const double aiq = p.a[i * OB_MAX_STAGES + qq];
        if (aiq == 0.0) continue;
        const T c = T(h * aiq);
        float kv[4][8];
#pragma unroll
        for (int k = 0; k < 4; ++k) ld8(ks + (long long)qq * kN + unit_off(k), kv[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int e = 0; e < 8; ++e) v[k][e] = Num<T>::add(v[k][e], Num<T>::mul(c, kv[k][e]));
      }
      if (recb)
#pragma unroll
        for (int k = 0; k < 4; ++k) st8(recb + i * vec + unit_off(k), v[k]);
      tcur = float(t + p.c[i] * h);
      if (i == 0 && carry) {   // FSAL: k_0 of this step is k_{s-1} of the previous one
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float kv[8];
          ld8(ks + (long long)(s - 1) * kN + unit_off(k), kv);
          st8(ks + unit_off(k), kv);
        }
        __syncthreads();
      } else if (!((p.skip_vjp >> i) & 1u) || (keep_last && i == s - 1)) {
        inv0 = split_units(v, conv_tc::kT0);
        sync_issue();
        pt.mark(8);
        eval_tile(ks + (long long)i * kN);
      }
    }
    int bad = 0;
    {
      float v[4][8];
#pragma unroll
      for (int k = 0; k < 4; ++k) ld8(u + unit_off(k), v[k]);
      for (int i = 0; i < s; ++i) {
        if (p.b[i] == 0.0) continue;
        const T c = T(h * p.b[i]);
        float kv[4][8];
#pragma unroll
        for (int k = 0; k < 4; ++k) ld8(ks + (long long)i * kN + unit_off(k), kv[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int e = 0; e < 8; ++e) v[k][e] = Num<T>::add(v[k][e], Num<T>::mul(c, kv[k][e]));
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (!Num<T>::finite(v[k][e])) bad = 1;
        st8(u + unit_off(k), v[k]);
        if (recb) st8(recb + s * vec + unit_off(k), v[k]);
      }
    }
    return __syncthreads_or(bad) == 0;
  }

  // ---- the transposed step (rk_adjoint_step, adjoint.py:67-94): lam <- lam + sum_i Lam_i,
  // Lam_i = h J_i^T w_i, w_i = b_i lam + sum_{j > i} a_ji Lam_j, mu += h P_i^T w_i.
  // Returns false when lambda is no longer finite.
  OB_DEV bool reverse_step(T* lam, double t, double h, const T* rec, int row0, T* mu) {
    const int s = p.s;
    const long long vec = (long long)p.B * kN;
    T* Lam = p.scratch + blockIdx.x * p.scratch_stride + (long long)s * kN;
    T* lamn = p.state_glob + blockIdx.x * p.state_stride + 2LL * kN;
    const T* recb = rec + (long long)row0 * kN;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float v[8];
      ld8(lam + unit_off(k), v);
      st8(lamn + unit_off(k), v);
    }
    __syncthreads();
    const T hT = T(h);
    for (int i = s - 1; i >= 0; --i) {
      if (p.skip_vjp & (1u << i)) {   // w_i == 0 exactly: Lam_i = 0 (still counted, B8)
        const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 4; ++k) st8(Lam + (long long)i * kN + unit_off(k), z);
        __syncthreads();
        continue;
      }
      tcur = float(t + p.c[i] * h);
      T* Li = Lam + (long long)i * kN;
      vjp_core(
          recb + i * vec,
          [&](float vv[4][8]) {   // w_i in the generic order
            const T bi = T(p.b[i]);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              ld8(lam + unit_off(k), vv[k]);
#pragma unroll
              for (int e = 0; e < 8; ++e) vv[k][e] = Num<T>::mul(bi, vv[k][e]);
            }
            for (int j = i + 1; j < s; ++j) {
              const double aji = p.a[j * OB_MAX_STAGES + i];
              if (aji == 0.0) continue;
              const T c = T(aji);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                float lv[8];
                ld8(Lam + (long long)j * kN + unit_off(k), lv);
#pragma unroll
                for (int e = 0; e < 8; ++e) vv[k][e] = Num<T>::add(vv[k][e], Num<T>::mul(c, lv[e]));
              }
            }
          },
          mu, float(h), true,
          [&](int pos, int cg, const float* j) {   // Lam_i = h J^T w_i; lam_n += Lam_i
            const int o = conv_tc::q_pixel(pos) * 64 + 16 * cg;
            float4* dl = reinterpret_cast<float4*>(Li + o);
            float4* dn = reinterpret_cast<float4*>(lamn + o);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float4 li = make_float4(Num<T>::mul(hT, j[4 * e]), Num<T>::mul(hT, j[4 * e + 1]),
                                            Num<T>::mul(hT, j[4 * e + 2]), Num<T>::mul(hT, j[4 * e + 3]));
              float4 n = dn[e];
              n.x = Num<T>::add(n.x, li.x);
              n.y = Num<T>::add(n.y, li.y);
              n.z = Num<T>::add(n.z, li.z);
              n.w = Num<T>::add(n.w, li.w);
              dl[e] = li;
              dn[e] = n;
            }
          });
    }
    int bad = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float v[8];
      ld8(lamn + unit_off(k), v);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (!Num<T>::finite(v[e])) bad = 1;
      st8(lam + unit_off(k), v);
    }
    return __syncthreads_or(bad) == 0;
  }

  OB_DEV void finish(T*) {}
  OB_DEV void release() {
    // prefetched weight taps still in flight must land before the CTA's shared memory is freed
    if (tc::uniform_warp() == 0 && pref_layer >= 0)
      for (uint32_t o = wuse; o < wuse + 3; ++o) tc::bar_wait(full(o % 3u), (o / 3u) & 1u);
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_free(0u, kCols);
  }
};

// packed image of the conv block for the tensor-core tile (see conv_tc::kPk*): every block
// finds the power-of-two scale of each conv's weights, then the grid packs its share
__global__ void pack_tc_conv_kernel(const __grid_constant__ Dims d, const float* theta, unsigned char* img) {
  __shared__ float red[32];
  __shared__ float scale[2];
  for (int l = 0; l < 2; ++l) {
    const float* Wl = theta + d.woff[l];
    const int n = 64 * 9 * d.conv_cin[l];
    float m = 0.f;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if (i % d.conv_cin[l] < 64) m = fmaxf(m, fabsf(Wl[i]));   // the time channel stays fp32
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      float mm = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mm = fmaxf(mm, red[w]);
      float s, inv;
      conv_tc::pow2_scale(mm, s, inv);
      scale[l] = s;
      if (blockIdx.x == 0) reinterpret_cast<float*>(img + conv_tc::kPkInvW)[l] = inv;
    }
    __syncthreads();
  }
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gn = gridDim.x * blockDim.x;
  // border-class time bias: sum over the taps that stay inside the image (ascending)
  for (int i = gt; i < 9 * 64; i += gn) {
    const int cls = i / 64, co = i % 64;
    float acc = 0.f;
    for (int s = 0; s < 9; ++s)
      if (conv_tc::tap_in_class(s, cls)) acc += theta[d.woff[0] + (long long)(co * 9 + s) * 65 + 64];
    reinterpret_cast<float*>(img + conv_tc::kPkTB)[i] = acc;
  }
  // indicator image: ind[q][s] = 1 when q is a pixel and q + off(s) is one too
  for (int i = gt; i < conv_tc::kNP * 16; i += gn) {
    const int q = i / 16, s = i % 16;
    bool on = false;
    if (s < 9 && conv_tc::q_valid(q)) on = conv_tc::tap_in_class(s, conv_tc::q_class(q));
    *reinterpret_cast<__half*>(img + conv_tc::kPkInd + (uint32_t)(s >> 3) * conv_tc::kPlane + (uint32_t)q * 16u +
                               (uint32_t)(s & 7) * 2u) = __float2half_rn(on ? 1.0f : 0.0f);
  }
  // tap weights [layer][tap]: [cin / 8][cout][8 cin] fp16 hi then lo
  for (int i = gt; i < 2 * 9 * 64 * 64; i += gn) {
    const int l = i / (9 * 64 * 64), r = i % (9 * 64 * 64), s = r / 4096, co = (r / 64) % 64, ci = r % 64;
    const float x = theta[d.woff[l] + (long long)(co * 9 + s) * d.conv_cin[l] + ci] * scale[l];
    const __half hi = __float2half_rn(x);
    const __half lo = __float2half_rn(x - __half2float(hi));
    unsigned char* tap = img + conv_tc::kPkW + (uint32_t)(l * 9 + s) * conv_tc::kTap;
    const uint32_t off = (uint32_t)(ci >> 3) * conv_tc::kWPl + (uint32_t)co * 16u + (uint32_t)(ci & 7) * 2u;
    *reinterpret_cast<__half*>(tap + off) = hi;
    *reinterpret_cast<__half*>(tap + conv_tc::kTapHalf + off) = lo;
  }
}

}  // namespace ob
