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
// The tile runs whole RK steps (step(), reverse_step()): each stage's
// derivative / cotangent stays in its TMEM slot and the stage sums read it
// with tcgen05.ld.  One elected lane of warp 0 issues the MMAs and commits them
// to an mbarrier; all threads wait on it, read accumulators with tcgen05.ld
// (each warp its TMEM lane quarter), apply the epilogue and write the next
// operand.
#pragma once

#include "rk_impl.cuh"
#include "tc.cuh"

namespace ob {

constexpr int kTcNS = 32;       // sample columns (MMA N) per tile
constexpr uint32_t kTcRow = (kTcNS / 8) * 128u;   // activation tiles stored transposed [feature][sample]

// shared-memory geometry of the tensor-core tile (bytes from the start of dynamic
// shared memory, where the region sits); used by the host planner and, as
// compile-time constants, by the device adapter
struct TcGeom {
  int D0, H, D2, nmb;
  uint32_t SA1, SA2, SAx, SAh, SAv;
  uint32_t W2h, W2l, W1h, W1l, fv, packed;
  uint32_t X0h, X0l, Hh, Hl, Vh, Vl, vec, pw, bar, bar2, slot, total;
};

__host__ __device__ constexpr TcGeom tc_geom(int D0, int H, int D2) {
  TcGeom g{};
  g.D0 = D0; g.H = H; g.D2 = D2; g.nmb = H / 128;
  g.SA1 = (uint32_t)(D0 / 8) * 128u;
  g.SA2 = (uint32_t)(H / 8) * 128u;
  g.SAx = kTcRow;                                   // X0^T [i][s]: i-block stride
  g.SAh = (uint32_t)(kTcNS / 8) * 128u;             // H^T [o][s]: o-block stride
  g.SAv = kTcRow;                                   // V^T  [o2][s]
  uint32_t o = 0;
  g.W2h = o; o += (uint32_t)D2 * H * 2;
  g.W2l = o; o += (uint32_t)D2 * H * 2;
  g.W1h = o; o += (uint32_t)H * D0 * 2;
  g.W1l = o; o += (uint32_t)H * D0 * 2;
  g.fv = o;  o += (uint32_t)(2 * H + D2) * 4;      // w1t[H] | b1[H] | b2[D2]
  o = (o + 127) & ~127u;
  g.packed = o;                                     // staged from global by setup_tile
  g.X0h = o; o += (uint32_t)(D0 / 8) * g.SAx;
  g.X0l = o; o += (uint32_t)(D0 / 8) * g.SAx;
  g.Hh = o;  o += (uint32_t)(H / 8) * g.SAh;
  g.Hl = o;  o += (uint32_t)(H / 8) * g.SAh;
  g.Vh = o;  o += (uint32_t)(D2 / 8) * g.SAv;
  g.Vl = o;  o += (uint32_t)(D2 / 8) * g.SAv;
  g.vec = o; o += (uint32_t)(2 * H + D2) * 4;       // db1[H] | dwt[H] | db2[D2]
  g.pw = o;  o += (uint32_t)(4 * D2) * 4;           // db2 partials [4][D2] (reverse_step)
  o = (o + 15) & ~15u;
  g.bar = o; o += 8;
  g.bar2 = o; o += 8;                               // parameter-cotangent MMAs (off the critical path)
  g.slot = o; o += 8;
  o = (o + 31) & ~31u;
  g.total = o;
  return g;
}

// shapes with an instantiated tile (D0 = D2 = state dim, H hidden)
__host__ inline bool tc_shape_ok(int D0, int H, int D2) {
  return D0 == D2 && (D0 == 16 || D0 == 32 || D0 == 48 || D0 == 64) && (H == 128 || H == 256);
}

// dynamic shared memory (aliases every kernel's extern smem_raw); the tile's
// region starts at offset 0, so all operand addresses are link-time constants
extern __shared__ __align__(128) unsigned char ob_tc_smem[];

// 3-pass split product D (+)= A B over KS K-slices of 16, all geometry constant:
// (AH, AL) / (BH, BL): byte offsets of the hi / lo copies, *LB / *SB: the
// descriptor's leading / stride byte offsets, *ST: address step per K-slice
template <uint32_t AH, uint32_t AL, uint32_t ALB, uint32_t ASB, uint32_t AST,
          uint32_t BH, uint32_t BL, uint32_t BLB, uint32_t BSB, uint32_t BST, int KS, uint32_t ID>
OB_DEV void tc_mma3(uint32_t D, uint32_t first_acc) {
  const uint32_t sb = tc::smem_u32(ob_tc_smem);
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const uint64_t Ah = tc::sdesc(sb + AH + k * AST, ALB, ASB), Al = tc::sdesc(sb + AL + k * AST, ALB, ASB);
    const uint64_t Bh = tc::sdesc(sb + BH + k * BST, BLB, BSB), Bl = tc::sdesc(sb + BL + k * BST, BLB, BSB);
    // A_hi feeds two products: read once, reused from the collector buffer
    tc::mma_bf16_keep_a(D, Ah, Bh, ID, k > 0 ? 1u : first_acc);
    tc::mma_bf16_reuse_a(D, Ah, Bl, ID, 1u);
    tc::mma_bf16(D, Al, Bh, ID, 1u);
  }
}

template <typename T, int D0, int H, int D2>
struct TcMlpAdapter {
  static_assert(sizeof(T) == 4, "tensor-core MLP tile is fp32");
  static constexpr bool kHasJvp = false;
  static constexpr bool kScaledVjp = true;   // vjp returns J^T (h w)
  static constexpr bool kOwnsStep = true;    // step(): stage derivatives stay in TMEM
  static constexpr uint32_t kCols = 512;     // whole TMEM: one CTA per SM, base column 0
  static constexpr TcGeom G = tc_geom(D0, H, D2);
  static constexpr int NMB = H / 128;
  static constexpr int CW = 8 * NMB;         // hidden-epilogue columns per thread
  // TMEM columns (lane 0 base = 0: 512 columns allocated by the only CTA on the SM)
  // acc1: hidden accumulator; stage slots k (M = 64 out accumulators, the step's stage
  // derivatives kept on chip) at 64 + 32 k; acc2 (the VJP's dX) shares slot 0; dW2^T, dW1
  // of the reverse sweep.  The reverse kernel's replays use slots 0..5 only (see tc_eligible).
  static constexpr uint32_t T_ACC1 = 0, T_ACC2 = 64, T_W2 = 256, T_W1 = 384;
  static constexpr uint32_t slot_col(int k) { return 64u + 32u * (uint32_t)k; }

  const RkParams<T>& p;
  uint32_t phase;       // mbarrier parity
  uint32_t phase2;      // parity of bar2 (dW MMAs)
  bool pend2;           // a dW MMA group is still running (reads V / X0 / dZ)
  float tcur;           // stage time (CTA-wide, set by put_time)
  int Rv, act;
  bool started;         // parameter-cotangent accumulators hold data

  OB_DEV unsigned char* base() const { return ob_tc_smem; }
  OB_DEV uint64_t* bar() const { return reinterpret_cast<uint64_t*>(ob_tc_smem + G.bar); }
  OB_DEV uint64_t* bar2() const { return reinterpret_cast<uint64_t*>(ob_tc_smem + G.bar2); }
  OB_DEV const float* w1t() const { return reinterpret_cast<const float*>(ob_tc_smem + G.fv); }
  OB_DEV const float* b1() const { return w1t() + H; }
  OB_DEV const float* b2() const { return w1t() + 2 * H; }
  OB_DEV float* db1() const { return reinterpret_cast<float*>(ob_tc_smem + G.vec); }
  OB_DEV float* dwt() const { return db1() + H; }
  OB_DEV float* db2() const { return db1() + 2 * H; }

  OB_DEV TcMlpAdapter(const RkParams<T>& p_, const Weights<T>&, MlpSmem<T>&, T* sm, int, int Rv_)
      : p(p_), phase(0), phase2(0), pend2(false), tcur(0.f), Rv(Rv_), act(p_.d.act), started(false) {
    // operand tiles, accumulator vectors and the generic state buffers after the
    // region start at zero (padded samples stay 0)
    uint4* z = reinterpret_cast<uint4*>(ob_tc_smem + G.packed);
    const int n16 = (int)(((size_t)p.sm.total * sizeof(T) - G.packed) / 16);
    for (int i = threadIdx.x; i < n16; i += blockDim.x)
      if (i < (int)((G.bar - G.packed) / 16) || i >= (int)((G.total - G.packed) / 16))
        z[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) tc::tmem_alloc(reinterpret_cast<uint32_t*>(ob_tc_smem + G.slot), kCols);
    if (threadIdx.x == 0) {
      tc::bar_init(bar(), 1);
      tc::bar_init(bar2(), 1);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (threadIdx.x == 0 && *reinterpret_cast<volatile uint32_t*>(ob_tc_smem + G.slot) != 0u)
      set_status(p.status, OB_ERR_UNSUPPORTED, -2);   // TMEM not at column 0: shared SM
  }

  OB_DEV int nin() const { return D0; }
  OB_DEV void set_scratch(T*, int) {}
  // samples s0..s0+7 of state component m (rows >= Rv zero): two 16-byte stores
  OB_DEV void put8(int m, int s0, const float* v) {
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      tc::split2_bf16(s0 + 2 * q < Rv ? v[2 * q] : 0.f, s0 + 2 * q + 1 < Rv ? v[2 * q + 1] : 0.f, hw[q],
                      lw[q]);
    const uint32_t off = tc::blk(m, s0, G.SAx, 128);
    *reinterpret_cast<uint4*>(ob_tc_smem + G.X0h + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(ob_tc_smem + G.X0l + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
  OB_DEV void put_time(double t) { tcur = p.d.time_input ? float(t) : 0.f; }

  // operands written by the generic proxy -> visible to the MMA; accumulator reads retired
  OB_DEV void sync_issue() {
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  OB_DEV void wait() {
    tc::bar_wait(bar(), phase);
    phase ^= 1u;
    tc::fence_after();
  }
  // wait for the outstanding parameter-cotangent MMAs before their operands are rewritten
  OB_DEV void drain() {
    if (!pend2) return;
    tc::bar_wait(bar2(), phase2);
    phase2 ^= 1u;
    tc::fence_after();
    pend2 = false;
  }

  // ---- products (issued by warp 0; one elected lane)
  // z[o][s] = sum_i W1[o][i] X0[s][i]           (A = W1 K-major, B = X0^T MN-major)
  OB_DEV void issue_hidden() {
    constexpr uint32_t id = tc::idesc_bf16(128, kTcNS, false, true);
    tc_mma3<G.W1h, G.W1l, 128, G.SA1, 256, G.X0h, G.X0l, G.SAx, 128, 2 * G.SAx, D0 / 16, id>(T_ACC1, 0);
    if constexpr (NMB == 2)
      tc_mma3<G.W1h + 16 * G.SA1, G.W1l + 16 * G.SA1, 128, G.SA1, 256, G.X0h, G.X0l,
              G.SAx, 128, 2 * G.SAx, D0 / 16, id>(T_ACC1 + 32, 0);
  }
  // out[o2][s] = sum_i2 W2[o2][i2] H[s][i2]      (M = 64; B = H^T MN-major)
  OB_DEV void issue_out(uint32_t dst = T_ACC2) {
    constexpr uint32_t id = tc::idesc_bf16(64, kTcNS, false, true);
    tc_mma3<G.W2h, G.W2l, 128, G.SA2, 256, G.Hh, G.Hl, G.SAh, 128, 2 * G.SAh, H / 16, id>(dst, 0);
  }
  // dW2^T[i2][o2] += sum_s H[s][i2] V[s][o2]     (A = H^T K-major, B = V^T K-major)
  OB_DEV void issue_dw2(uint32_t acc) {
    constexpr uint32_t id = tc::idesc_bf16(128, D2, false, false);
    tc_mma3<G.Hh, G.Hl, 128, G.SAh, 256, G.Vh, G.Vl, 128, G.SAv, 256,
            kTcNS / 16, id>(T_W2, acc);
    if constexpr (NMB == 2)
      tc_mma3<G.Hh + 16 * G.SAh, G.Hl + 16 * G.SAh, 128, G.SAh, 256, G.Vh, G.Vl,
              128, G.SAv, 256, kTcNS / 16, id>(T_W2 + D2, acc);
  }
  // dH[i2][s] = sum_o2 W2[o2][i2] V[s][o2]       (A = W2 MN-major, B = V^T MN-major)
  OB_DEV void issue_dh() {
    constexpr uint32_t id = tc::idesc_bf16(128, kTcNS, true, true);
    tc_mma3<G.W2h, G.W2l, G.SA2, 128, 2 * G.SA2, G.Vh, G.Vl, G.SAv, 128, 2 * G.SAv,
            D2 / 16, id>(T_ACC1, 0);
    if constexpr (NMB == 2)
      tc_mma3<G.W2h + 16 * 128, G.W2l + 16 * 128, G.SA2, 128, 2 * G.SA2, G.Vh, G.Vl,
              G.SAv, 128, 2 * G.SAv, D2 / 16, id>(T_ACC1 + 32, 0);
  }
  // dW1[o][i] += sum_s dZ[s][o] X0[s][i]          (A = dZ^T K-major, B = X0^T K-major)
  OB_DEV void issue_dw1(uint32_t acc) {
    constexpr uint32_t id = tc::idesc_bf16(128, D0, false, false);
    tc_mma3<G.Hh, G.Hl, 128, G.SAh, 256, G.X0h, G.X0l, 128, G.SAx, 256,
            kTcNS / 16, id>(T_W1, acc);
    if constexpr (NMB == 2)
      tc_mma3<G.Hh + 16 * G.SAh, G.Hl + 16 * G.SAh, 128, G.SAh, 256, G.X0h,
              G.X0l, 128, G.SAx, 256, kTcNS / 16, id>(T_W1 + D0, acc);
  }
  // ---- epilogues (warp w: TMEM lane quarter q = w % 4, column group cg = w / 4)
  OB_DEV void ld_hidden(float v[16], int& o, int& c0, int& cg) const {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3;
    cg = w >> 2;
    const int f0 = cg * CW, mb = f0 >> 5;
    c0 = f0 & 31;
    o = mb * 128 + q * 32 + lane;
    const uint32_t ta = T_ACC1 + ((uint32_t)(q * 32) << 16) + 32 * mb + c0;
    if constexpr (CW == 16) tc::ld16(ta, v); else tc::ld8(ta, v);
  }
  // CW consecutive samples c0.. of hidden unit o -> H^T (hi, lo): 16-byte vector stores
  OB_DEV void put_hid(int c0, int o, const float* a) {
    const uint32_t off = tc::blk(o, c0, G.SAh, 128);
#pragma unroll
    for (int g8 = 0; g8 < CW / 8; ++g8) {
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) tc::split2_bf16(a[8 * g8 + 2 * q], a[8 * g8 + 2 * q + 1], hw[q], lw[q]);
      *reinterpret_cast<uint4*>(ob_tc_smem + G.Hh + off + 128 * g8) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(ob_tc_smem + G.Hl + off + 128 * g8) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
  }
  // act(z + b1 + t w1t) -> H (hi, lo); act' kept in registers for a VJP
  template <bool kVjp>
  OB_DEV void epi_hidden(float ap[16]) {
    float v[16];
    int o, c0, cg;
    ld_hidden(v, o, c0, cg);
    const float bo = b1()[o], wt = w1t()[o];
    float a[16];
    if (act == OB_ACT_TANH) {
#pragma unroll
      for (int j = 0; j < CW; j += 2) {
        const float z0 = v[j] + bo + tcur * wt, z1 = v[j + 1] + bo + tcur * wt;
        tc::tanh2_1sfu(z0, z1, a[j], a[j + 1]);
        if (kVjp) {
          ap[j] = 1.f - a[j] * a[j];
          ap[j + 1] = 1.f - a[j + 1] * a[j + 1];
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        a[j] = v[j] + bo + tcur * wt;
        if (kVjp) ap[j] = 1.f;
      }
    }
    put_hid(c0, o, a);
  }
  // f(x0) into stage slot k (TMEM, bias b2 not yet added); no epilogue
  OB_DEV void eval_slot(int k) {
    PhaseTimer pt(p.prof ? p.phase : nullptr);
    sync_issue();
    if (tc::uniform_warp() == 0) { issue_hidden(); tc::commit(bar()); }
    wait();
    pt.mark(10);
    float ap[16];
    epi_hidden<false>(ap);
    sync_issue();
    pt.mark(11);
    if (tc::uniform_warp() == 0) { issue_out(slot_col(k)); tc::commit(bar()); }
    wait();
    pt.mark(10);
  }

  // One explicit RK step of the tile (explicit_rk_step, integrators.py:196-222) with the
  // stage derivatives k_q = f(U_q) held in TMEM slots: the stage sums read them with
  // tcgen05.ld in the accumulator layout (warp w: state rows 16 (w%4) + lane for lanes < 16,
  // samples 8 (w/4) ..+7) -- same order and roundings as rk_step_tile (k = acc + b2, then
  // v + (h a_iq) k).  carry: FSAL (k_0 = previous k_{s-1}); keep_last: k_{s-1} is carried on.
  OB_DEV bool step(T* u, double t, double h, bool carry, T* rec, int row0, bool keep_last) {
    const int s = p.s, ldn = p.d.ldn, Rt = p.Rt;
    const long long vec = (long long)p.B * D0;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q4 = w & 3, cg = w >> 2;
    const int m = 16 * q4 + lane, s0 = 8 * cg;
    const bool mine = lane < 16 && m < D0;
    const uint32_t lrow = (uint32_t)(32 * q4) << 16;
    const float b2m = mine ? b2()[m] : 0.f;
    PhaseTimer pt(p.prof ? p.phase : nullptr);
    if (carry) {   // FSAL: this step's k_0 is the previous k_{s-1}
      float v[8];
      tc::ld8(slot_col(s - 1) + lrow + s0, v);
      tc::st8(slot_col(0) + lrow + s0, v);
      tc::wait_st();
    }
    for (int i = 0; i < s; ++i) {
      float ca[OB_MAX_STAGES];
      bool nz[OB_MAX_STAGES];
#pragma unroll
      for (int q = 0; q < OB_MAX_STAGES; ++q) {
        const double a = q < i ? p.a[i * OB_MAX_STAGES + q] : 0.0;
        nz[q] = a != 0.0;
        ca[q] = float(h * a);
      }
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (mine && s0 + j < Rt) ? u[(s0 + j) * ldn + m] : 0.f;
#pragma unroll
      for (int q = 0; q < OB_MAX_STAGES; ++q) {
        if (!nz[q]) continue;
        float k[8];
        tc::ld8(slot_col(q) + lrow + s0, k);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          v[j] = Num<float>::add(v[j], Num<float>::mul(ca[q], Num<float>::add(k[j], b2m)));
      }
      if (mine) {
        put8(m, s0, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = s0 + j;
          if (rec && r < Rv) rec[i * vec + (long long)(row0 + r) * D0 + m] = v[j];
        }
      }
      put_time(t + p.c[i] * h);
      pt.mark(8);
      if (i == 0 && carry) continue;
      if (!((p.skip_vjp >> i) & 1u) || (keep_last && i == s - 1)) eval_slot(i);
      pt.mark(9);
    }
    // u_next = u + sum_i (h b_i) k_i
    float cb[OB_MAX_STAGES];
    bool nzb[OB_MAX_STAGES];
#pragma unroll
    for (int q = 0; q < OB_MAX_STAGES; ++q) {
      const double b = q < s ? p.b[q] : 0.0;
      nzb[q] = b != 0.0;
      cb[q] = float(h * b);
    }
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (mine && s0 + j < Rt) ? u[(s0 + j) * ldn + m] : 0.f;
#pragma unroll
    for (int q = 0; q < OB_MAX_STAGES; ++q) {
      if (!nzb[q]) continue;
      float k[8];
      tc::ld8(slot_col(q) + lrow + s0, k);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v[j] = Num<float>::add(v[j], Num<float>::mul(cb[q], Num<float>::add(k[j], b2m)));
    }
    int bad = 0;
    if (mine) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = s0 + j;
        if (r < Rt) u[r * ldn + m] = v[j];
        if (r < Rv) {
          if (!Num<float>::finite(v[j])) bad = 1;
          if (rec) rec[s * vec + (long long)(row0 + r) * D0 + m] = v[j];
        }
      }
    }
    tc::fence_before();
    return __syncthreads_or(bad) == 0;
  }

  // The VJP pair on the operands already staged (V = h w split, X0 = stage state):
  // dX (= J^T (h w)) lands in TMEM column dx; parameter cotangents accumulate on chip.
  // db2_part: add the [4][D2] partial sums of h w in pw to db2 (reverse_step).
  OB_DEV void vjp_core(T* mu, uint32_t dx, bool db2_part) {
    PhaseTimer pt(p.prof ? p.phase : nullptr);
    sync_issue();
    pt.mark(14);
    if (tc::uniform_warp() == 0) { issue_hidden(); tc::commit(bar()); }
    if (mu && db2_part && threadIdx.x < D2) {
      const float* pw = reinterpret_cast<const float*>(ob_tc_smem + G.pw);
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc += pw[k * D2 + threadIdx.x];
      db2()[threadIdx.x] += acc;
    }
    wait();
    pt.mark(10);
    float ap[16];
    epi_hidden<true>(ap);
    sync_issue();
    pt.mark(11);
    const uint32_t acc = started ? 1u : 0u;
    // dH first (the critical path), dW2^T behind it on its own barrier
    if (tc::uniform_warp() == 0) {
      issue_dh();
      tc::commit(bar());
      if (mu) { issue_dw2(acc); tc::commit(bar2()); }
    }
    if (mu) pend2 = true;
    wait();
    pt.mark(10);
    {
      float v[16];
      int o, c0, cg;
      ld_hidden(v, o, c0, cg);
      float ps = 0.f;
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        v[j] *= ap[j];
        ps += v[j];
      }
      drain();   // dW2^T reads H: dZ may overwrite it only now
      put_hid(c0, o, v);
      float* part = reinterpret_cast<float*>(ob_tc_smem + G.Vh);
      part[(cg % (4 / NMB)) * H + o] = ps;
    }
    sync_issue();
    pt.mark(11);
    // dX first; dW1 keeps running into the next stage (drained before X0 / dZ change)
    if (tc::uniform_warp() == 0) {
      constexpr uint32_t id = tc::idesc_bf16(64, kTcNS, true, true);
      tc_mma3<G.W1h, G.W1l, G.SA1, 128, 2 * G.SA1, G.Hh, G.Hl, G.SAh, 128, 2 * G.SAh, H / 16, id>(dx, 0);
      tc::commit(bar());
      if (mu) { issue_dw1(acc); tc::commit(bar2()); }
    }
    if (mu) pend2 = true;
    if (mu && threadIdx.x < H) {
      const float* part = reinterpret_cast<const float*>(ob_tc_smem + G.Vh);
      float sm = 0.f;
#pragma unroll
      for (int k = 0; k < 4 / NMB; ++k) sm += part[k * H + threadIdx.x];
      db1()[threadIdx.x] += sm;
      dwt()[threadIdx.x] += tcur * sm;
    }
    wait();
    pt.mark(10);
    if (mu) started = true;
  }

  // One reverse step (rk_adjoint_step, adjoint.py:67-94) with the stage cotangents
  // Lambda_i = J^T (h w_i) held in TMEM slots: w_i = b_i lam + sum_{j>i} a_ji Lambda_j is
  // formed from tcgen05.ld in the accumulator layout, split straight into V; the
  // stage state U_i comes from the record (prefetched one stage ahead); at the end
  // lam += Lambda_{s-1} + ... + Lambda_0 (the reference's order).  Returns false on a
  // non-finite adjoint state (AdjointState.check_finite, adjoint.py:42-44).
  OB_DEV bool reverse_step(T* lam, double t, double h, const T* rec, int row0, T* mu) {
    const int s = p.s, ldn = p.d.ldn, Rt = p.Rt;
    const long long vec = (long long)p.B * D0;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q4 = w & 3, cg = w >> 2;
    const int m = 16 * q4 + lane, s0 = 8 * cg;
    const bool mine = lane < 16 && m < D0;
    const uint32_t lrow = (uint32_t)(32 * q4) << 16;
    const float hf = float(h);
    float lv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) lv[j] = (mine && s0 + j < Rt) ? lam[(s0 + j) * ldn + m] : 0.f;
    float un[8];   // stage state of the next stage to reverse (prefetched)
    auto load_u = [&](int i) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        un[j] = (mine && s0 + j < Rv) ? rec[i * vec + (long long)(row0 + s0 + j) * D0 + m] : 0.f;
    };
    load_u(s - 1);
    unsigned live = 0;   // slots holding a nonzero Lambda_i
    for (int i = s - 1; i >= 0; --i) {
      if ((p.skip_vjp >> i) & 1u) {   // w_i == 0 exactly: Lambda_i = 0 (still counted, B8)
        if (i > 0) load_u(i - 1);
        continue;
      }
      PhaseTimer ptr(p.prof ? p.phase : nullptr);
      float ca[OB_MAX_STAGES];
      bool nz[OB_MAX_STAGES];
#pragma unroll
      for (int j = 0; j < OB_MAX_STAGES; ++j) {
        const double a = (j > i && j < s && ((live >> j) & 1u)) ? p.a[j * OB_MAX_STAGES + i] : 0.0;
        nz[j] = a != 0.0;
        ca[j] = float(a);
      }
      const float bi = float(p.b[i]);
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = Num<float>::mul(bi, lv[j]);
#pragma unroll
      for (int j = 0; j < OB_MAX_STAGES; ++j) {
        if (!nz[j]) continue;
        float k[8];
        tc::ld8(slot_col(j) + lrow + s0, k);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = Num<float>::add(v[e], Num<float>::mul(ca[j], k[e]));
      }
      ptr.mark(12);   // cotangent combination from the TMEM slots
      // V = h w (padded samples zero), db2 partial, U_i into X0
      drain();   // the previous stage's dW1 reads X0 and dZ
      ptr.mark(13);   // wait for the previous stage's dW1 MMAs
      float ps = 0.f;
      if (mine) {
        float hv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          hv[e] = s0 + e < Rv ? hf * v[e] : 0.f;
          ps += hv[e];
        }
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) tc::split2_bf16(hv[2 * q], hv[2 * q + 1], hw[q], lw[q]);
        const uint32_t off = tc::blk(m, s0, G.SAv, 128);
        *reinterpret_cast<uint4*>(ob_tc_smem + G.Vh + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(ob_tc_smem + G.Vl + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        put8(m, s0, un);
        reinterpret_cast<float*>(ob_tc_smem + G.pw)[cg * D2 + m] = ps;
      }
      if (i > 0) load_u(i - 1);
      put_time(t + p.c[i] * h);
      ptr.mark(15);   // operand split + stores, next stage state load issued
      vjp_core(mu, slot_col(i), true);
      live |= 1u << i;
    }
    drain();
    // lam_n = lam_{n+1} + Lambda_{s-1} + ... + Lambda_0
    int bad = 0;
#pragma unroll
    for (int i = OB_MAX_STAGES - 1; i >= 0; --i) {
      if (i >= s || !((live >> i) & 1u)) continue;
      float k[8];
      tc::ld8(slot_col(i) + lrow + s0, k);
#pragma unroll
      for (int e = 0; e < 8; ++e) lv[e] = Num<float>::add(lv[e], k[e]);
    }
    if (mine) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int r = s0 + e;
        if (r < Rt) {
          lam[r * ldn + m] = lv[e];
          if (!Num<float>::finite(lv[e])) bad = 1;
        }
      }
    }
    tc::fence_before();
    return __syncthreads_or(bad) == 0;
  }

  // add the sweep's parameter cotangent to the CTA's padded mu slot
  OB_DEV void finish(T* mu) {
    if (!started || !mu) return;
    const Dims& d = p.d;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, cg = w >> 2;
#pragma unroll
    for (int mb = 0; mb < NMB; ++mb) {
      for (int c8 = cg; c8 < D2 / 8; c8 += 4) {   // dW2^T: lanes i2, columns o2
        float v[8];
        tc::ld8(T_W2 + ((uint32_t)(q * 32) << 16) + D2 * mb + 8 * c8, v);
        const int i2 = mb * 128 + q * 32 + lane;
        for (int j = 0; j < 8; ++j) mu[d.mwoff[1] + (long long)(8 * c8 + j) * d.ldm[1] + i2] += v[j];
      }
      for (int c8 = cg; c8 < D0 / 8; c8 += 4) {   // dW1: lanes o, columns i
        float v[8];
        tc::ld8(T_W1 + ((uint32_t)(q * 32) << 16) + D0 * mb + 8 * c8, v);
        const int o = mb * 128 + q * 32 + lane;
        for (int j = 0; j < 8; ++j) mu[d.mwoff[0] + (long long)o * d.ldm[0] + 8 * c8 + j] += v[j];
      }
    }
    for (int o = threadIdx.x; o < H; o += blockDim.x) {
      mu[d.mboff[0] + o] += db1()[o];
      if (d.time_input) mu[d.mwoff[0] + (long long)o * d.ldm[0] + D0] += dwt()[o];
    }
    for (int o = threadIdx.x; o < D2; o += blockDim.x) mu[d.mboff[1] + o] += db2()[o];
    __syncthreads();
  }

  OB_DEV void release() {
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_free(0u, kCols);
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
