// tc_mlp.cuh -- tensor-core (tcgen05 / TMEM) MLP field adapter for the
// persistent fp32 explicit-RK kernels.
//
// The field is the reference MlpField (integrators.py:76-102) with two affine
// layers, f(u, t) = W2 act(W1 [u | t] + b1) + b2 (kernels.py:122-183), evaluated
// for the CTA's tile of <= 32 samples.  Every contraction runs on the 5th-gen
// tensor cores as a 3-pass bf16 split: an fp32 operand x is held as the pair
// (hi, lo) = (bf16(x), bf16(x - hi)), and a product is accumulated in fp32 in
// TMEM as  A_hi B_hi + A_hi B_lo + A_lo B_hi  (relative error ~2^-16 per
// product; measured 3.6e-6 on the C2 gradient against the fp64 oracle, inside
// the 1e-4 fp32 parity bar -- single-pass TF32 is 2.9e-4).
//
// Orientation: features are the MMA M dimension (128-row blocks; M = 64 for
// the 64-wide state layers), the tile's samples are N = 32.  Weights are
// staged once per CTA in the core-block layout of tc.cuh, so W serves the
// forward (K-major) and W^T of the VJP (MN-major) from one copy; activations
// likewise serve the next layer and the weight-gradient product.
//
// Parameter cotangents never leave the SM during a reverse sweep: dW2^T and
// dW1 accumulate in TMEM across every stage VJP of the sweep (the VJP
// cotangent is pre-scaled by h, so Lambda_i = J^T (h w) and
// mu += P^T (h w) need no per-stage rescale), biases and the time column in
// fp32 shared-memory vectors; finish() adds them to the CTA's mu slot once.
//
// One thread issues the MMAs and commits them to an mbarrier; all threads
// wait on it, read accumulators with tcgen05.ld (each warp its TMEM lane
// quarter), apply the epilogue and write the next operand.
#pragma once

#include "rk_impl.cuh"
#include "tc.cuh"

namespace ob {

constexpr int kTcNS = 32;       // sample columns (MMA N) per tile
constexpr uint32_t kTcLB = 144; // activation block-column stride (128 + 16: conflict-free stores)

// shared-memory geometry of the tensor-core tile (bytes from the region base);
// used by the host planner and the device adapter alike
struct TcGeom {
  int D0, H, D2, nmb;
  uint32_t SA1, SA2, SAx, SAh, SAv;
  uint32_t W2h, W2l, W1h, W1l, fv, packed;
  uint32_t X0h, X0l, Hh, Hl, Vh, Vl, vec, bar, slot, total;
};

__host__ __device__ inline TcGeom tc_geom(int D0, int H, int D2) {
  TcGeom g{};
  g.D0 = D0; g.H = H; g.D2 = D2; g.nmb = H / 128;
  g.SA1 = (uint32_t)(D0 / 8) * 128u;
  g.SA2 = (uint32_t)(H / 8) * 128u;
  g.SAx = (uint32_t)(D0 / 8) * kTcLB;
  g.SAh = (uint32_t)(H / 8) * kTcLB;
  g.SAv = (uint32_t)(D2 / 8) * kTcLB;
  uint32_t o = 0;
  g.W2h = o; o += (uint32_t)D2 * H * 2;
  g.W2l = o; o += (uint32_t)D2 * H * 2;
  g.W1h = o; o += (uint32_t)H * D0 * 2;
  g.W1l = o; o += (uint32_t)H * D0 * 2;
  g.fv = o;  o += (uint32_t)(2 * H + D2) * 4;      // w1t[H] | b1[H] | b2[D2]
  o = (o + 127) & ~127u;
  g.packed = o;                                     // staged from global by setup_tile
  const uint32_t rb = kTcNS / 8;
  g.X0h = o; o += rb * g.SAx;
  g.X0l = o; o += rb * g.SAx;
  g.Hh = o;  o += rb * g.SAh;
  g.Hl = o;  o += rb * g.SAh;
  g.Vh = o;  o += rb * g.SAv;
  g.Vl = o;  o += rb * g.SAv;
  g.vec = o; o += (uint32_t)(2 * H + D2) * 4;       // db1[H] | dwt[H] | db2[D2]
  o = (o + 15) & ~15u;
  g.bar = o; o += 8;
  g.slot = o; o += 8;
  g.total = o;
  return g;
}

// eligibility (host): fp32 two-layer MLP field, explicit fixed-step scheme
__host__ inline bool tc_shape_ok(int D0, int H, int D2) {
  return D0 % 16 == 0 && D0 >= 16 && D0 <= 64 && D2 % 16 == 0 && D2 >= 16 && D2 <= 64 &&
         (H == 128 || H == 256);
}

template <typename T>
struct TcMlpAdapter {
  static_assert(sizeof(T) == 4, "tensor-core MLP tile is fp32");
  static constexpr bool kHasJvp = false;
  static constexpr bool kScaledVjp = true;   // vjp returns J^T (h w)
  static constexpr uint32_t kCols = 512;

  const RkParams<T>& p;
  TcGeom g;
  unsigned char* base;
  uint32_t sbase;       // shared address of base
  uint32_t tmem;        // TMEM base (lane 0, column 0)
  uint32_t phase;       // mbarrier parity
  float tcur;           // stage time (CTA-wide, set by put_time)
  int Rv, act;
  bool started;         // parameter-cotangent accumulators hold data
  uint64_t* bar;

  OB_DEV const float* w1t() const { return reinterpret_cast<const float*>(base + g.fv); }
  OB_DEV const float* b1() const { return w1t() + g.H; }
  OB_DEV const float* b2() const { return w1t() + 2 * g.H; }
  OB_DEV float* db1() const { return reinterpret_cast<float*>(base + g.vec); }
  OB_DEV float* dwt() const { return db1() + g.H; }
  OB_DEV float* db2() const { return db1() + 2 * g.H; }
  OB_DEV uint32_t t_acc1() const { return tmem; }
  OB_DEV uint32_t t_acc2() const { return tmem + 64; }
  OB_DEV uint32_t t_w2() const { return tmem + 128; }
  OB_DEV uint32_t t_w1() const { return tmem + 256; }

  OB_DEV TcMlpAdapter(const RkParams<T>& p_, const Weights<T>&, MlpSmem<T>&, T* sm, int, int Rv_)
      : p(p_), phase(0), tcur(0.f), Rv(Rv_), act(p_.d.act), started(false) {
    g = tc_geom(p.d.N, p.d.w[1], p.d.w[2]);
    base = reinterpret_cast<unsigned char*>(sm + p.sm.wts);
    sbase = tc::smem_u32(base);
    bar = reinterpret_cast<uint64_t*>(base + g.bar);
    // activation operands and accumulator vectors start at zero (padded samples stay 0)
    uint4* z = reinterpret_cast<uint4*>(base + g.X0h);
    const int n16 = (int)((g.bar - g.X0h) / 16);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) tc::tmem_alloc(reinterpret_cast<uint32_t*>(base + g.slot), kCols);
    if (threadIdx.x == 0) tc::bar_init(bar, 1);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    tmem = *reinterpret_cast<volatile uint32_t*>(base + g.slot);
  }

  OB_DEV T* x0() { return nullptr; }
  OB_DEV int nin() const { return p.d.N; }
  OB_DEV void set_scratch(T*, int) {}
  // stage state element j of row r (rows >= Rv are padding: kept at zero)
  OB_DEV void put(int r, int j, T v) {
    uint16_t hi, lo;
    tc::split_bf16(r < Rv ? v : 0.f, hi, lo);
    const uint32_t off = tc::blk(r, j, g.SAx, kTcLB);
    *reinterpret_cast<uint16_t*>(base + g.X0h + off) = hi;
    *reinterpret_cast<uint16_t*>(base + g.X0l + off) = lo;
  }
  OB_DEV void put_time(double t) { tcur = p.d.time_input ? float(t) : 0.f; }

  // ---- MMA issue (one thread) and completion wait (all threads)
  // 3-pass split product over ksteps K-slices of 16; a/b: (hi, lo) shared addresses
  OB_DEV void mma3(uint32_t d, uint32_t ah, uint32_t al, uint32_t alb, uint32_t asb, uint32_t ast,
                   uint32_t bh, uint32_t bl, uint32_t blb, uint32_t bsb, uint32_t bst, int ksteps,
                   uint32_t idesc, bool acc) {
    for (int k = 0; k < ksteps; ++k) {
      const uint64_t Ah = tc::sdesc(ah + k * ast, alb, asb), Al = tc::sdesc(al + k * ast, alb, asb);
      const uint64_t Bh = tc::sdesc(bh + k * bst, blb, bsb), Bl = tc::sdesc(bl + k * bst, blb, bsb);
      tc::mma_bf16(d, Ah, Bh, idesc, (acc || k > 0) ? 1u : 0u);
      tc::mma_bf16(d, Ah, Bl, idesc, 1u);
      tc::mma_bf16(d, Al, Bh, idesc, 1u);
    }
  }
  // operands written by the generic proxy -> visible to the MMA; accumulator reads retired
  OB_DEV void sync_issue() {
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  OB_DEV void wait() {
    tc::bar_wait(bar, phase);
    phase ^= 1u;
    tc::fence_after();
  }

  // hidden layer: z = W1 x + b1 + t w1t  (rows o of the hidden layer = MMA M)
  OB_DEV void issue_hidden() {
    const uint32_t id = tc::idesc_bf16(128, kTcNS, false, false);
    for (int mb = 0; mb < g.nmb; ++mb)
      mma3(t_acc1() + 32 * mb, sbase + g.W1h + mb * 16 * g.SA1, sbase + g.W1l + mb * 16 * g.SA1,
           128, g.SA1, 256, sbase + g.X0h, sbase + g.X0l, kTcLB, g.SAx, 2 * kTcLB, g.D0 / 16, id,
           false);
  }
  // epilogue of the hidden layer: act -> H (hi, lo); act' kept in registers for a VJP
  // warp w: lane quarter q = w % 4, column group cg = w / 4
  OB_DEV int hid_cols() const { return 8 * g.nmb; }
  template <bool kVjp>
  OB_DEV void epi_hidden(float ap[16]) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, cg = w >> 2;
    const int cw = hid_cols(), f0 = cg * cw, mb = f0 >> 5, c0 = f0 & 31;
    const int o = mb * 128 + q * 32 + lane;
    float v[16];
    const uint32_t ta = t_acc1() + ((uint32_t)(q * 32) << 16) + 32 * mb + c0;
    if (cw == 16) tc::ld16(ta, v); else tc::ld8(ta, v);
    const float bo = b1()[o], wt = w1t()[o];
    for (int j = 0; j < cw; ++j) {
      const float z = v[j] + bo + tcur * wt;
      float a;
      if (act == OB_ACT_TANH) a = fast_tanh(z);
      else if (act == OB_ACT_RELU) a = z > 0.f ? z : 0.f;
      else a = z;
      if (kVjp) ap[j] = act == OB_ACT_TANH ? 1.f - a * a : act == OB_ACT_RELU ? (a > 0.f ? 1.f : 0.f) : 1.f;
      uint16_t hi, lo;
      tc::split_bf16(a, hi, lo);
      const uint32_t off = tc::blk(c0 + j, o, g.SAh, kTcLB);
      *reinterpret_cast<uint16_t*>(base + g.Hh + off) = hi;
      *reinterpret_cast<uint16_t*>(base + g.Hl + off) = lo;
    }
  }

  // f(x0) -> out [Rt][ldn] (global or shared), columns >= N untouched
  OB_DEV void eval(T* out) {
    PhaseTimer pt(p.prof ? p.phase : nullptr);   // 10: MMA issue + wait, 11: epilogues
    sync_issue();
    if (threadIdx.x == 0) { issue_hidden(); tc::commit(bar); }
    wait();
    pt.mark(10);
    float ap[16];
    epi_hidden<false>(ap);
    sync_issue();
    pt.mark(11);
    if (threadIdx.x == 0) {
      mma3(t_acc2(), sbase + g.W2h, sbase + g.W2l, 128, g.SA2, 256, sbase + g.Hh, sbase + g.Hl,
           kTcLB, g.SAh, 2 * kTcLB, g.H / 16, tc::idesc_bf16(64, kTcNS, false, false), false);
      tc::commit(bar);
    }
    wait();
    pt.mark(10);
    epi_state(out, p.d.ldn, g.D2, true);
    tc::fence_before();
    __syncthreads();
    pt.mark(11);
  }

  // M = 64 accumulator (state-sized rows m = 16 q + lane, lanes < 16) -> dst[s][m]
  OB_DEV void epi_state(T* dst, int ldo, int rows, bool bias) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, cg = w >> 2;
    float v[8];
    tc::ld8(t_acc2() + ((uint32_t)(q * 32) << 16) + 8 * cg, v);
    const int m = 16 * q + lane;
    if (lane < 16 && m < rows) {
      const float bm = bias ? b2()[m] : 0.f;
      for (int j = 0; j < 8; ++j) {
        const int s = 8 * cg + j;
        if (s < p.Rt) dst[s * ldo + m] = v[j] + bm;
      }
    }
  }

  // jtv = J^T (h w); mu (nullable) += h P^T w, accumulated on chip until finish()
  OB_DEV void vjp(const T* wv, T* jtv, T* mu, double h, int) {
    const int N = p.d.N, ldn = p.d.ldn, D2 = g.D2, H = g.H;
    const float hf = float(h);
    PhaseTimer pt(p.prof ? p.phase : nullptr);   // 14: operand prep, 10: MMA waits, 11: epilogues
    // V = h w (rows >= Rv zero) as (hi, lo)
    for (int i = threadIdx.x; i < kTcNS * D2; i += blockDim.x) {
      const int s = i / D2, o2 = i % D2;
      const float v = s < Rv ? hf * wv[s * ldn + o2] : 0.f;
      uint16_t hi, lo;
      tc::split_bf16(v, hi, lo);
      const uint32_t off = tc::blk(s, o2, g.SAv, kTcLB);
      *reinterpret_cast<uint16_t*>(base + g.Vh + off) = hi;
      *reinterpret_cast<uint16_t*>(base + g.Vl + off) = lo;
    }
    sync_issue();
    pt.mark(14);
    if (threadIdx.x == 0) { issue_hidden(); tc::commit(bar); }
    if (mu && threadIdx.x < D2) {   // db2 += sum_s h w[s]
      float acc = 0.f;
      for (int s = 0; s < Rv; ++s) acc += hf * wv[s * ldn + threadIdx.x];
      db2()[threadIdx.x] += acc;
    }
    wait();
    pt.mark(10);
    float ap[16];
    epi_hidden<true>(ap);
    sync_issue();
    pt.mark(11);
    if (threadIdx.x == 0) {
      if (mu) {   // dW2^T[i2][o2] += sum_s H[s][i2] V[s][o2]
        const uint32_t id = tc::idesc_bf16(128, D2, true, true);
        for (int mb = 0; mb < g.nmb; ++mb)
          mma3(t_w2() + D2 * mb, sbase + g.Hh + mb * 16 * kTcLB, sbase + g.Hl + mb * 16 * kTcLB,
               g.SAh, kTcLB, 2 * g.SAh, sbase + g.Vh, sbase + g.Vl, g.SAv, kTcLB, 2 * g.SAv,
               kTcNS / 16, id, started);
      }
      // dH[i2][s] = sum_o2 W2[o2][i2] V[s][o2]
      const uint32_t id = tc::idesc_bf16(128, kTcNS, true, false);
      for (int mb = 0; mb < g.nmb; ++mb)
        mma3(t_acc1() + 32 * mb, sbase + g.W2h + mb * 16 * 128, sbase + g.W2l + mb * 16 * 128,
             g.SA2, 128, 2 * g.SA2, sbase + g.Vh, sbase + g.Vl, kTcLB, g.SAv, 2 * kTcLB, D2 / 16,
             id, false);
      tc::commit(bar);
    }
    wait();
    pt.mark(10);
    // dZ = dH * act'(z) overwrites H (its MMAs have completed); per-row partial sums
    {
      const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, cg = w >> 2;
      const int cw = hid_cols(), f0 = cg * cw, mb = f0 >> 5, c0 = f0 & 31;
      const int o = mb * 128 + q * 32 + lane;
      float v[16];
      const uint32_t ta = t_acc1() + ((uint32_t)(q * 32) << 16) + 32 * mb + c0;
      if (cw == 16) tc::ld16(ta, v); else tc::ld8(ta, v);
      float ps = 0.f;
      for (int j = 0; j < cw; ++j) {
        const float dz = v[j] * ap[j];
        ps += dz;
        uint16_t hi, lo;
        tc::split_bf16(dz, hi, lo);
        const uint32_t off = tc::blk(c0 + j, o, g.SAh, kTcLB);
        *reinterpret_cast<uint16_t*>(base + g.Hh + off) = hi;
        *reinterpret_cast<uint16_t*>(base + g.Hl + off) = lo;
      }
      // V is free now: partial sums part[k][o], k = column group within the row
      float* part = reinterpret_cast<float*>(base + g.Vh);
      part[(cg % (4 / g.nmb)) * H + o] = ps;
    }
    sync_issue();
    pt.mark(11);
    if (threadIdx.x == 0) {
      if (mu) {   // dW1[o][i] += sum_s dZ[s][o] X0[s][i]
        const uint32_t id = tc::idesc_bf16(128, g.D0, true, true);
        for (int mb = 0; mb < g.nmb; ++mb)
          mma3(t_w1() + g.D0 * mb, sbase + g.Hh + mb * 16 * kTcLB, sbase + g.Hl + mb * 16 * kTcLB,
               g.SAh, kTcLB, 2 * g.SAh, sbase + g.X0h, sbase + g.X0l, g.SAx, kTcLB, 2 * g.SAx,
               kTcNS / 16, id, started);
      }
      // dX[i][s] = sum_o W1[o][i] dZ[s][o]
      mma3(t_acc2(), sbase + g.W1h, sbase + g.W1l, g.SA1, 128, 2 * g.SA1, sbase + g.Hh,
           sbase + g.Hl, kTcLB, g.SAh, 2 * kTcLB, H / 16, tc::idesc_bf16(64, kTcNS, true, false),
           false);
      tc::commit(bar);
    }
    if (mu && threadIdx.x < H) {   // db1 += sum_s dZ, time column += t sum_s dZ
      const float* part = reinterpret_cast<const float*>(base + g.Vh);
      float s = 0.f;
      for (int k = 0; k < 4 / g.nmb; ++k) s += part[k * H + threadIdx.x];
      db1()[threadIdx.x] += s;
      dwt()[threadIdx.x] += tcur * s;
    }
    wait();
    pt.mark(10);
    epi_state(jtv, ldn, N, false);
    if (mu) started = true;
    tc::fence_before();
    __syncthreads();
    pt.mark(11);
  }

  // add the sweep's parameter cotangent to the CTA's padded mu slot
  OB_DEV void finish(T* mu) {
    if (!started || !mu) return;
    const Dims& d = p.d;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, cg = w >> 2;
    for (int mb = 0; mb < g.nmb; ++mb) {
      for (int c8 = cg; c8 < g.D2 / 8; c8 += 4) {   // dW2^T: lanes i2, columns o2
        float v[8];
        tc::ld8(t_w2() + ((uint32_t)(q * 32) << 16) + g.D2 * mb + 8 * c8, v);
        const int i2 = mb * 128 + q * 32 + lane;
        for (int j = 0; j < 8; ++j) mu[d.mwoff[1] + (long long)(8 * c8 + j) * d.ldm[1] + i2] += v[j];
      }
      for (int c8 = cg; c8 < g.D0 / 8; c8 += 4) {   // dW1: lanes o, columns i
        float v[8];
        tc::ld8(t_w1() + ((uint32_t)(q * 32) << 16) + g.D0 * mb + 8 * c8, v);
        const int o = mb * 128 + q * 32 + lane;
        for (int j = 0; j < 8; ++j) mu[d.mwoff[0] + (long long)o * d.ldm[0] + 8 * c8 + j] += v[j];
      }
    }
    for (int o = threadIdx.x; o < g.H; o += blockDim.x) {
      mu[d.mboff[0] + o] += db1()[o];
      if (d.time_input) mu[d.mwoff[0] + (long long)o * d.ldm[0] + g.D0] += dwt()[o];
    }
    for (int o = threadIdx.x; o < g.D2; o += blockDim.x) mu[d.mboff[1] + o] += db2()[o];
    __syncthreads();
  }

  OB_DEV void release() {
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_free(tmem, kCols);
  }
};

// packed image of the weights for the tensor-core tile (the staged part of TcGeom):
// W2 (hi, lo) | W1 state columns (hi, lo) | w1t | b1 | b2
__global__ void pack_tc_kernel(const __grid_constant__ Dims d, const float* theta, float* packed) {
  const TcGeom g = tc_geom(d.N, d.w[1], d.w[2]);
  unsigned char* img = reinterpret_cast<unsigned char*>(packed);
  const int D0 = g.D0, H = g.H, D2 = g.D2, w0 = d.w[0];
  const float* W1 = theta + d.woff[0];
  const float* W2 = theta + d.woff[1];
  const long long n = (long long)H * D0 + (long long)D2 * H + H;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    uint16_t hi, lo;
    if (i < (long long)H * D0) {
      const int o = (int)(i / D0), k = (int)(i % D0);
      const float x = W1[(long long)o * w0 + k];
      const __nv_bfloat16 bh = __float2bfloat16_rn(x);
      hi = __bfloat16_as_ushort(bh);
      lo = __bfloat16_as_ushort(__float2bfloat16_rn(x - __bfloat162float(bh)));
      const uint32_t off = tc::blk(o, k, g.SA1, 128);
      *reinterpret_cast<uint16_t*>(img + g.W1h + off) = hi;
      *reinterpret_cast<uint16_t*>(img + g.W1l + off) = lo;
    } else if (i < (long long)H * D0 + (long long)D2 * H) {
      const long long j = i - (long long)H * D0;
      const int o2 = (int)(j / H), k = (int)(j % H);
      const float x = W2[j];
      const __nv_bfloat16 bh = __float2bfloat16_rn(x);
      hi = __bfloat16_as_ushort(bh);
      lo = __bfloat16_as_ushort(__float2bfloat16_rn(x - __bfloat162float(bh)));
      const uint32_t off = tc::blk(o2, k, g.SA2, 128);
      *reinterpret_cast<uint16_t*>(img + g.W2h + off) = hi;
      *reinterpret_cast<uint16_t*>(img + g.W2l + off) = lo;
    } else {
      const int o = (int)(i - (long long)H * D0 - (long long)D2 * H);
      float* fv = reinterpret_cast<float*>(img + g.fv);
      fv[o] = d.time_input ? W1[(long long)o * w0 + D0] : 0.f;
      fv[H + o] = theta[d.boff[0] + o];
      if (o < D2) fv[2 * H + o] = theta[d.boff[1] + o];
    }
  }
}

}  // namespace ob
