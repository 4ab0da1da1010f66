// tc_cnf.cuh -- tensor-core (tcgen05 / TMEM) tile for the continuous-normalizing-flow
// right-hand side (config C4) in the persistent explicit-RK kernels:
//   f_aug([z, Delta], t) = [f(z, t), -eps^T (df/dz) eps],
//   f = W2 softplus(W1 softplus(W0 [z, t] + b0) + b1) + b2   (D + 1 -> H -> H -> D),
// one fixed Rademacher probe eps per sample (Hutchinson trace estimator).  The
// maths is the SIMT CnfAdapter's (cnf_impl.cuh; restated oracle in
// oracle/fields_ext.py): the tile stacks each sample's forward row and its
// eps-tangent row as the MMA N dimension (N = 16: forward rows 0..7, tangent rows
// 8..15, <= 8 samples per CTA), features are the MMA M dimension, and every
// contraction is a 3-pass bf16 split (A_hi B_hi + A_hi B_lo + A_lo B_hi, fp32
// accumulation in TMEM; see tc_mlp.cuh).
//
// Weights do not fit in shared memory (the H x H layer alone is 3 MB as hi/lo bf16),
// so they stream from L2 through a ring of shared-memory slots filled by the tensor
// memory accelerator (cp.async.bulk, mbarrier complete_tx): every product is a
// fixed sequence of 16 KB chunks (128 rows x 32 K, hi | lo), packed once per call in
// the order the tile consumes them (forward W_l and transposed W_l^T copies).
//
// Parameter cotangents are deferred: each VJP appends its stacked operand tiles
// (layer inputs [a; u] and output cotangents [zbar; sbar], bf16 hi/lo, exactly the
// shared-memory images the products used) to a per-tile log in global memory with
// bulk stores, and finish() forms dW_l = sum_vjp [zbar; sbar]^T [a; u] with tcgen05
// GEMMs over the log (K = 16 rows per VJP), then adds them to the CTA's mu slot once.
// Biases accumulate directly (fixed order).  The VJP seed is pre-scaled by h
// (kScaledVjp), so no per-VJP rescale is needed anywhere.
#pragma once

#include "rk_impl.cuh"
#include "tc.cuh"

namespace ob {

// ----------------------------------------------------------------- geometry
namespace cnf_tc {
constexpr int kRows = 16;         // MMA N: forward rows 0..7 | tangent rows 8..15
constexpr int kHalf = 8;          // samples per tile (max)
constexpr int kKc = 32;           // K per weight chunk (two 16-wide K slices)
constexpr int kNS = 6;            // weight ring slots
constexpr uint32_t kSlot = 16384; // bytes per slot (M = 128 chunk, hi | lo)
constexpr int kNW = 224;          // N per dW GEMM output tile (<= 256)

// stacked activation tile [kRows][K] (bf16) in core blocks: byte(row, k) =
// (row/8)*128 + (k/8)*256 + (row%8)*16 + (k%8)*2.  As a B operand (N = rows, K = k):
// K-major, LBO = 256, SBO = 128.  As an MN-major operand (M/N = k, K = rows) for the
// deferred dW GEMMs: LBO = 128, SBO = 256.
__host__ __device__ constexpr uint32_t tile_bytes(int K) { return (uint32_t)(K / 8) * 256u; }
__host__ __device__ constexpr uint32_t act_off(int row, int k) {
  return (uint32_t)(row >> 3) * 128u + (uint32_t)(k >> 3) * 256u + (uint32_t)(row & 7) * 16u +
         (uint32_t)(k & 7) * 2u;
}
// weight chunk [M][kKc] K-major: byte(m, k) = (m/8)*512 + (k/8)*128 + (m%8)*16 + (k%8)*2
__host__ __device__ constexpr uint32_t w_off(int m, int k) {
  return (uint32_t)(m >> 3) * 512u + (uint32_t)(k >> 3) * 128u + (uint32_t)(m & 7) * 16u +
         (uint32_t)(k & 7) * 2u;
}
}  // namespace cnf_tc

// One product of the tile: D[M-block][16] (+)= W_chunked x B-tile over K.
struct CnfProd {
  int nmb;            // M blocks
  int m;              // MMA M (128, or 64 for the D-row layers)
  int nkc;            // K chunks of kKc
  uint32_t src;       // byte offset of the first chunk in the packed weights
};

template <int D, int H>
struct CnfGeom {
  static constexpr int K0 = 64;                      // [z, t] padded (D + 1 <= 64)
  static constexpr int KH = (H + 31) / 32 * 32;      // hidden padded to whole chunks
  static constexpr int MB = (H + 127) / 128;         // M blocks of a hidden layer
  static constexpr uint32_t C128 = 2 * 128 * cnf_tc::kKc * 2;   // 16 KB chunk (hi | lo)
  static constexpr uint32_t C64 = 2 * 64 * cnf_tc::kKc * 2;     // 8 KB
  // products in streaming order: forward L0, L1, L2; backward L2^T, L1^T, L0^T
  static constexpr uint32_t P0f = 0;
  static constexpr uint32_t P1f = P0f + MB * (K0 / cnf_tc::kKc) * C128;
  static constexpr uint32_t P2f = P1f + MB * (KH / cnf_tc::kKc) * C128;
  static constexpr uint32_t P2b = P2f + (KH / cnf_tc::kKc) * C64;
  static constexpr uint32_t P1b = P2b + MB * (K0 / cnf_tc::kKc) * C128;
  static constexpr uint32_t P0b = P1b + MB * (KH / cnf_tc::kKc) * C128;
  static constexpr uint32_t Packed = P0b + (KH / cnf_tc::kKc) * C64;
  // shared memory (bytes from the start of dynamic shared memory)
  static constexpr uint32_t TX = cnf_tc::tile_bytes(K0);     // X0 / Z3 tiles (K = 64)
  static constexpr uint32_t TA = cnf_tc::tile_bytes(KH);     // hidden tiles
  static constexpr uint32_t X0h = 0, X0l = X0h + TX;
  static constexpr uint32_t Z3h = X0l + TX, Z3l = Z3h + TX;
  static constexpr uint32_t A1h = Z3l + TX, A1l = A1h + TA;
  static constexpr uint32_t A2h = A1l + TA, A2l = A2h + TA;
  static constexpr uint32_t Ring = A2l + TA;                  // kNS slots (contiguous after A2)
  static constexpr uint32_t Jeps = Ring + cnf_tc::kNS * cnf_tc::kSlot;   // fp32 [8][64]
  static constexpr uint32_t Bars = Jeps + 8 * 64 * 4;         // full[kNS] empty[kNS] done gemm[4]
  static constexpr uint32_t Slot = Bars + 8 * (2 * cnf_tc::kNS + 8);
  static constexpr uint32_t Total = (Slot + 8 + 127) / 128 * 128;
  // per-VJP log record (bytes): Z3 | A2 | Zb2 | A1 | Zb1 | X0, each hi | lo
  static constexpr uint32_t LZ3 = 0, LA2 = LZ3 + 2 * TX, LZ2 = LA2 + 2 * TA, LA1 = LZ2 + 2 * TA,
                            LZ1 = LA1 + 2 * TA, LX0 = LZ1 + 2 * TA, Log = LX0 + 2 * TX;
  // TMEM columns (fp32, N = 16 per M block)
  static constexpr uint32_t T_Z1 = 0, T_Z2 = T_Z1 + 16 * MB, T_OUT = T_Z2 + 16 * MB,
                            T_G2 = T_OUT + 16, T_G1 = T_G2 + 16 * MB, T_G0 = T_G1 + 16 * MB,
                            T_END = T_G0 + 16;
  static_assert(D + 1 <= K0, "state dim");
  static_assert(T_END <= 512, "TMEM");
};

// dynamic shared memory of the tile (shared with the other tensor-core tiles)
extern __shared__ __align__(128) unsigned char ob_tc_smem[];

namespace cnf_tc {
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// global -> shared bulk copy completing on an mbarrier (TMA engine)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}
// shared -> global bulk copy (bulk async-group)
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(tc::smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}\n"
               : "=r"(p));
  return p != 0;
}
// split x into (hi, lo) bf16 and store both at byte offset off of the hi / lo tiles
__device__ __forceinline__ void put_split(unsigned char* hi, unsigned char* lo, uint32_t off, float x) {
  uint16_t h, l;
  tc::split_bf16(x, h, l);
  *reinterpret_cast<uint16_t*>(hi + off) = h;
  *reinterpret_cast<uint16_t*>(lo + off) = l;
}
__device__ __forceinline__ float sigmoid_from_e(float z, float e) {   // e = exp(-|z|)
  const float r = recip_1p(e);
  return z >= 0.0f ? r : e * r;
}
}  // namespace cnf_tc

template <typename T, int D, int H>
struct TcCnfAdapter {
  static_assert(sizeof(T) == 4, "tensor-core CNF tile is fp32");
  using G = CnfGeom<D, H>;
  static constexpr bool kHasJvp = false;
  static constexpr bool kScaledVjp = true;    // vjp returns J^T (h w), mu += P^T (h w)
  static constexpr int kCombineBatch = 4;
  static constexpr bool kOwnsStep = false;
  static constexpr uint32_t kCols = 512;

  const RkParams<T>& p;
  int Rv, row0;
  float tcur;
  // weight-stream state (warp 0): chunk ordinals across all products of the sweep
  uint32_t head, tail, done_phase;
  int nlog;              // VJPs logged so far
  unsigned char* logp;   // this tile's log

  OB_DEV unsigned char* sm() const { return ob_tc_smem; }
  OB_DEV uint64_t* full(int s) const { return reinterpret_cast<uint64_t*>(ob_tc_smem + G::Bars) + s; }
  OB_DEV uint64_t* empty(int s) const {
    return reinterpret_cast<uint64_t*>(ob_tc_smem + G::Bars) + cnf_tc::kNS + s;
  }
  OB_DEV uint64_t* done() const { return reinterpret_cast<uint64_t*>(ob_tc_smem + G::Bars) + 2 * cnf_tc::kNS; }
  OB_DEV const unsigned char* packed() const { return reinterpret_cast<const unsigned char*>(p.packed); }

  OB_DEV TcCnfAdapter(const RkParams<T>& p_, const Weights<T>&, MlpSmem<T>&, T*, int row0_, int Rv_)
      : p(p_), Rv(Rv_), row0(row0_), tcur(0.f), head(0), tail(0), done_phase(0), nlog(0) {
    logp = reinterpret_cast<unsigned char*>(p.cnf_pre) + (long long)blockIdx.x * p.cnf_pre_stride * sizeof(T);
    // zero the operand tiles (padded rows / features stay exactly zero)
    uint4* z = reinterpret_cast<uint4*>(ob_tc_smem);
    for (int i = threadIdx.x; i < (int)(G::Ring / 16); i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) tc::tmem_alloc(reinterpret_cast<uint32_t*>(ob_tc_smem + G::Slot), kCols);
    if (threadIdx.x == 0) {
      for (int s = 0; s < cnf_tc::kNS; ++s) {
        tc::bar_init(full(s), 1);
        tc::bar_init(empty(s), 1);
      }
      tc::bar_init(done(), 1);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (threadIdx.x == 0 && p.status && *reinterpret_cast<volatile uint32_t*>(ob_tc_smem + G::Slot) != 0u)
      set_status(p.status, OB_ERR_UNSUPPORTED, -2);   // TMEM not at column 0: shared SM
    // Hutchinson probes: the tangent rows of X0 (time tangent 0)
    for (int i = threadIdx.x; i < Rv * D; i += blockDim.x) {
      const int r = i / D, j = i % D;
      cnf_tc::put_split(sm() + G::X0h, sm() + G::X0l, cnf_tc::act_off(cnf_tc::kHalf + r, j),
                        float(p.eps[(long long)(row0 + r) * D + j]));
    }
    __syncthreads();
  }

  OB_DEV int nin() const { return D; }
  OB_DEV void set_scratch(T*, int) {}
  OB_DEV void jvp(const T*, T*) {}
  // state component j of sample r -> forward row r of X0 (rows >= Rv stay zero)
  OB_DEV void put(int r, int j, T v) {
    if (r < Rv) cnf_tc::put_split(sm() + G::X0h, sm() + G::X0l, cnf_tc::act_off(r, j), float(v));
  }
  OB_DEV void put_time(double t) {
    tcur = float(t);
    if (threadIdx.x < Rv)
      cnf_tc::put_split(sm() + G::X0h, sm() + G::X0l, cnf_tc::act_off(threadIdx.x, D), tcur);
  }

  // generic-proxy shared-memory writes -> visible to the MMA / bulk copies; TMEM reads retired
  OB_DEV void sync_issue() {
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }

  // ---- weight stream (warp 0)
  OB_DEV void load_chunk(uint32_t idx, uint32_t src, uint32_t bytes) {
    const int s = (int)(idx % cnf_tc::kNS);
    if (cnf_tc::elect_one()) {
      cnf_tc::bar_expect_tx(full(s), bytes);
      cnf_tc::bulk_load(sm() + G::Ring + s * cnf_tc::kSlot, packed() + src, bytes, full(s));
    }
    __syncwarp();
  }
  // D[mb] (+)= W x B over the product's K: chunk c = (mb, kc); B = tile at smem offset bh / bl
  template <int M>
  OB_DEV void product(const CnfProd& pr, uint32_t dcol, uint32_t bh, uint32_t bl) {
    constexpr uint32_t id = tc::idesc_bf16(M, cnf_tc::kRows, false, false);
    const uint32_t cbytes = (uint32_t)M * cnf_tc::kKc * 2 * 2, half = cbytes / 2;
    const uint32_t n = (uint32_t)(pr.nmb * pr.nkc);
    const uint32_t sb = tc::smem_u32(ob_tc_smem);
    // prefetch kNS - 1 chunks (the ring is empty between products)
    for (; head < tail + cnf_tc::kNS - 1 && head < tail + n; ++head)
      load_chunk(head, pr.src + (head - tail) * cbytes, cbytes);
    for (uint32_t c = 0; c < n; ++c) {
      const uint32_t idx = tail + c;
      const int s = (int)(idx % cnf_tc::kNS);
      tc::bar_wait(full(s), (idx / cnf_tc::kNS) & 1u);
      tc::fence_after();
      const int mb = (int)(c / pr.nkc), kc = (int)(c % pr.nkc);
      const uint32_t a = sb + G::Ring + s * cnf_tc::kSlot;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t Ah = tc::sdesc(a + ks * 256, 128, 512), Al = tc::sdesc(a + half + ks * 256, 128, 512);
        const uint32_t bo = (uint32_t)(2 * kc + ks) * 512u;
        const uint64_t Bh = tc::sdesc(sb + bh + bo, 256, 128), Bl = tc::sdesc(sb + bl + bo, 256, 128);
        const uint32_t dt = dcol + 16u * mb;
        tc::mma_bf16_keep_a(dt, Ah, Bh, id, (kc > 0 || ks > 0) ? 1u : 0u);
        tc::mma_bf16_reuse_a(dt, Ah, Bl, id, 1u);
        tc::mma_bf16(dt, Al, Bh, id, 1u);
      }
      tc::commit(empty(s));
      // refill the previous chunk's slot (its MMAs were issued one chunk earlier)
      if (head < tail + n) {
        const uint32_t prev = head - cnf_tc::kNS;   // the chunk that last used head's slot
        if (head >= (uint32_t)cnf_tc::kNS) tc::bar_wait(empty((int)(prev % cnf_tc::kNS)), (prev / cnf_tc::kNS) & 1u);
        load_chunk(head, pr.src + (head - tail) * cbytes, cbytes);
        ++head;
      }
    }
    tail += n;
    tc::commit(done());
  }
  // every thread: wait for the product issued by warp 0
  OB_DEV void wait_done() {
    tc::bar_wait(done(), done_phase);
    done_phase ^= 1u;
    tc::fence_after();
  }
  // the ring slots are refilled only after their MMAs completed; drain the last
  // empties of a product so the next product's prefetch can reuse every slot
  OB_DEV void issue(int which, uint32_t dcol, uint32_t bh, uint32_t bl) {
    if (tc::uniform_warp() == 0) {
      const CnfProd pr = prod(which);
      if (pr.m == 128) product<128>(pr, dcol, bh, bl);
      else product<64>(pr, dcol, bh, bl);
      // wait for the product's remaining chunks' MMAs (slots free for the next prefetch)
      for (uint32_t j = (tail >= (uint32_t)cnf_tc::kNS ? tail - cnf_tc::kNS : 0); j < tail; ++j)
        tc::bar_wait(empty((int)(j % cnf_tc::kNS)), (j / cnf_tc::kNS) & 1u);
    }
    wait_done();
  }
  OB_DEV static CnfProd prod(int which) {
    constexpr int k0 = G::K0 / cnf_tc::kKc, kh = G::KH / cnf_tc::kKc;
    switch (which) {
      case 0: return CnfProd{G::MB, 128, k0, G::P0f};    // Z1 = W0 [x; e]
      case 1: return CnfProd{G::MB, 128, kh, G::P1f};    // Z2 = W1 [a1; u1]
      case 2: return CnfProd{1, 64, kh, G::P2f};         // OUT = W2 [a2; u2]
      case 3: return CnfProd{G::MB, 128, k0, G::P2b};    // G2 = W2^T Z3
      case 4: return CnfProd{G::MB, 128, kh, G::P1b};    // G1 = W1^T Zb2
      default: return CnfProd{1, 64, kh, G::P0b};        // G0 = W0^T Zb1
    }
  }

  // ---- epilogues (warp w: TMEM lane quarter q = w % 4, M blocks g, g + 4, ... with g = w / 4)
  // hidden layer l: pre-activations in TMEM (z forward cols 0..7, raw tangent s cols 8..15)
  // -> [softplus(z + b); sigmoid(z + b) s] into the stacked tile (hi | lo)
  OB_DEV void epi_hidden(uint32_t tcol, const T* bias, uint32_t oh, uint32_t ol) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3;
    for (int mb = w >> 2; mb < G::MB; mb += 4) {
      float v[16];
      tc::ld16(tcol + ((uint32_t)(32 * q) << 16) + 16u * mb, v);
      const int o = 128 * mb + 32 * q + lane;
      if (o >= H) continue;
      const float b = float(bias[o]);
#pragma unroll
      for (int c = 0; c < cnf_tc::kHalf; ++c) {
        if (c >= Rv) break;
        const float z = v[c] + b;
        const float e = ex2_fast(-1.4426950408889634f * fabsf(z));
        const float a = fmaxf(z, 0.0f) + 0.6931471805599453f * lg2_fast(1.0f + e);
        const float u = cnf_tc::sigmoid_from_e(z, e) * v[cnf_tc::kHalf + c];
        cnf_tc::put_split(sm() + oh, sm() + ol, cnf_tc::act_off(c, o), a);
        cnf_tc::put_split(sm() + oh, sm() + ol, cnf_tc::act_off(cnf_tc::kHalf + c, o), u);
      }
    }
  }

  // forward through the two hidden layers (pre-activations stay in TMEM Z1 / Z2)
  OB_DEV void hidden_forward() {
    sync_issue();
    issue(0, G::T_Z1, G::X0h, G::X0l);
    epi_hidden(G::T_Z1, p.W.bias[0], G::A1h, G::A1l);
    sync_issue();
    issue(1, G::T_Z2, G::A1h, G::A1l);
    epi_hidden(G::T_Z2, p.W.bias[1], G::A2h, G::A2l);
  }

  // f_aug(x0) -> out [Rt][ldn]: columns [0, D) = f, column D = -eps^T J eps
  OB_DEV void eval(T* out) {
    hidden_forward();
    sync_issue();
    issue(2, G::T_OUT, G::A2h, G::A2l);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* je = reinterpret_cast<float*>(sm() + G::Jeps);
    if (w < 4) {   // M = 64 accumulator: row n -> lane 32 (n / 16) + n % 16 (lanes < 16)
      float v[16];
      tc::ld16(G::T_OUT + ((uint32_t)(32 * w) << 16), v);   // collective: every lane
      const int n = 16 * w + lane;
      if (lane < 16 && n < D) {
        const float b = float(p.W.bias[2][n]);
        for (int c = 0; c < Rv; ++c) {
          out[c * p.d.ldn + n] = T(v[c] + b);
          je[c * 64 + n] = v[cnf_tc::kHalf + c];
        }
      }
    }
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < Rv) {   // -eps^T (J eps), fixed order
      const int c = threadIdx.x;
      float acc = 0.f;
      for (int n = 0; n < D; ++n) acc = fmaf(float(p.eps[(long long)(row0 + c) * D + n]), je[c * 64 + n], acc);
      out[c * p.d.ldn + D] = T(-acc);
    }
    __syncthreads();
  }

  // backward through hidden layer l: cotangents [abar; ubar] of the layer's outputs in
  // TMEM (tg), its pre-activations in TMEM (tz) -> [zbar; sbar] into the stacked tile:
  //   sbar = sigma(z) ubar,  zbar = sigma'(z) s ubar + sigma(z) abar   (softplus'' = sigma')
  // db_l (+)= sum over forward rows of zbar (fixed order)
  OB_DEV void epi_back(uint32_t tg, uint32_t tz, const T* bias, uint32_t oh, uint32_t ol, T* db) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3;
    for (int mb = w >> 2; mb < G::MB; mb += 4) {
      float g[16], zz[16];
      tc::ld16(tg + ((uint32_t)(32 * q) << 16) + 16u * mb, g);
      tc::ld16(tz + ((uint32_t)(32 * q) << 16) + 16u * mb, zz);
      const int o = 128 * mb + 32 * q + lane;
      if (o >= H) continue;
      const float b = float(bias[o]);
      float dbs = 0.f;
#pragma unroll
      for (int c = 0; c < cnf_tc::kHalf; ++c) {
        if (c >= Rv) break;
        const float z = zz[c] + b, s = zz[cnf_tc::kHalf + c];
        const float e = ex2_fast(-1.4426950408889634f * fabsf(z));
        const float sg = cnf_tc::sigmoid_from_e(z, e);
        const float sgp = sg * (1.0f - sg);
        const float ub = g[cnf_tc::kHalf + c], ab = g[c];
        const float sbar = sg * ub;
        const float zbar = sgp * s * ub + sg * ab;
        dbs += zbar;
        cnf_tc::put_split(sm() + oh, sm() + ol, cnf_tc::act_off(c, o), zbar);
        cnf_tc::put_split(sm() + oh, sm() + ol, cnf_tc::act_off(cnf_tc::kHalf + c, o), sbar);
      }
      if (db) db[o] += T(dbs);
    }
  }

  // log the stacked tile at smem offsets (hi, lo) -> this VJP's record at byte offset lo_
  OB_DEV void log_tile(uint32_t h, uint32_t l, uint32_t bytes, uint32_t rec_off) {
    if (threadIdx.x == 0) {
      unsigned char* dst = logp + (long long)nlog * G::Log + rec_off;
      cnf_tc::bulk_store(dst, sm() + h, bytes);
      cnf_tc::bulk_store(dst + bytes, sm() + l, bytes);
      cnf_tc::bulk_commit();
    }
  }
  // the logged shared-memory tiles have been read: they may be overwritten now
  OB_DEV void log_read_done() {
    if (threadIdx.x == 0) cnf_tc::bulk_wait_read();
    __syncthreads();
  }

  // (J_aug^T (h w), mu += P_aug^T (h w)) at x0; w: [Rt][ldn], columns [0, D) the cotangent
  // of f and column D that of Delta' (f_aug does not depend on Delta)
  OB_DEV void vjp(const T* w, T* jtv, T* mu, double h, int) {
    const Dims& d = p.d;
    const int ldn = d.ldn;
    const float hs = float(h);
    if (mu && (long long)(nlog + 1) * G::Log > p.cnf_pre_stride * (long long)sizeof(T)) {
      if (threadIdx.x == 0 && p.status) set_status(p.status, OB_ERR_UNSUPPORTED, -3);   // log capacity
      mu = nullptr;
    }
    hidden_forward();
    // output-layer cotangent Z3 = h [v_z ; -v_Delta eps]; db2 += h sum_rows v_z
    for (int i = threadIdx.x; i < cnf_tc::kHalf * D; i += blockDim.x) {
      const int c = i / D, n = i % D;
      float zf = 0.f, zt = 0.f;
      if (c < Rv) {
        zf = hs * float(w[c * ldn + n]);
        zt = hs * (-float(w[c * ldn + D]) * float(p.eps[(long long)(row0 + c) * D + n]));
      }
      cnf_tc::put_split(sm() + G::Z3h, sm() + G::Z3l, cnf_tc::act_off(c, n), zf);
      cnf_tc::put_split(sm() + G::Z3h, sm() + G::Z3l, cnf_tc::act_off(cnf_tc::kHalf + c, n), zt);
    }
    if (mu && threadIdx.x < D) {
      float s = 0.f;
      for (int c = 0; c < Rv; ++c) s += hs * float(w[c * ldn + threadIdx.x]);
      mu[d.mboff[2] + threadIdx.x] += T(s);
    }
    sync_issue();
    if (mu) {   // layer inputs of this VJP (final now): X0, A1, A2
      log_tile(G::X0h, G::X0l, G::TX, G::LX0);
      log_tile(G::A1h, G::A1l, G::TA, G::LA1);
      log_tile(G::A2h, G::A2l, G::TA, G::LA2);
      log_tile(G::Z3h, G::Z3l, G::TX, G::LZ3);
    }
    issue(3, G::T_G2, G::Z3h, G::Z3l);                   // [abar2; ubar2] = W2^T Z3
    if (mu) log_read_done();                             // A2 may be overwritten
    epi_back(G::T_G2, G::T_Z2, p.W.bias[1], G::A2h, G::A2l, mu ? mu + d.mboff[1] : nullptr);
    sync_issue();
    if (mu) log_tile(G::A2h, G::A2l, G::TA, G::LZ2);     // Zb2
    issue(4, G::T_G1, G::A2h, G::A2l);                   // [abar1; ubar1] = W1^T Zb2
    if (mu) log_read_done();
    epi_back(G::T_G1, G::T_Z1, p.W.bias[0], G::A1h, G::A1l, mu ? mu + d.mboff[0] : nullptr);
    sync_issue();
    if (mu) log_tile(G::A1h, G::A1l, G::TA, G::LZ1);     // Zb1
    issue(5, G::T_G0, G::A1h, G::A1l);                   // W0^T Zb1: rows 0..D-1 = J^T (h w)
    const int wp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (wp < 4) {
      float v[16];
      tc::ld16(G::T_G0 + ((uint32_t)(32 * wp) << 16), v);
      const int k = 16 * wp + lane;
      if (jtv && lane < 16 && k < D)
        for (int c = 0; c < Rv; ++c) jtv[c * ldn + k] = T(v[c]);
    }
    if (jtv)
      for (int c = threadIdx.x; c < p.Rt; c += blockDim.x) jtv[c * ldn + D] = T(0);
    if (mu) {
      log_read_done();
      ++nlog;
    }
    tc::fence_before();
    __syncthreads();
  }

  // ---- deferred parameter cotangents: dW_l = sum over logged VJPs of [zbar; sbar]^T [a; u]
  // D[M block of outputs][N chunk of inputs] accumulated in TMEM over K = 16 rows per VJP,
  // operand sub-blocks streamed from the log through the ring (A: outputs, B: inputs)
  OB_DEV void gemm_log(uint32_t zoff, uint32_t ztile, int mb_count, int mdim, uint32_t aoff,
                       uint32_t atile, int kin, T* dst, int ldm, int mrows) {
    const uint32_t sb = tc::smem_u32(ob_tc_smem);
    const int nch = (kin + cnf_tc::kNW - 1) / cnf_tc::kNW;
    // staging: two buffers of [A hi | A lo | B hi | B lo] in the A1 / A2 / ring region
    const uint32_t abytes = (uint32_t)mdim / 8 * 256;                 // M features x 16 rows
    for (int mb = 0; mb < mb_count; ++mb) {
      for (int c0 = 0; c0 < nch; c0 += 2) {
        reinit();   // fresh staging barriers per output tile (phases restart at v = 0)
        const int ncur = min(2, nch - c0);
        int nw[2] = {0, 0};
        for (int j = 0; j < ncur; ++j) nw[j] = min(cnf_tc::kNW, kin - (c0 + j) * cnf_tc::kNW);
        uint32_t bbytes[2] = {(uint32_t)nw[0] / 8 * 256, (uint32_t)nw[1] / 8 * 256};
        const uint32_t stage = 2 * abytes + 2 * (bbytes[0] + bbytes[1]);
        if (tc::uniform_warp() == 0) {
          for (int v = 0; v < nlog; ++v) {
            const int s = v & 1;
            const uint32_t base = G::A1h + s * 2 * 40960;   // two 80 KB stages
            const unsigned char* rec = logp + (long long)v * G::Log;
            if (v >= 2) tc::bar_wait(empty(s), ((v - 2) >> 1) & 1u);
            if (cnf_tc::elect_one()) {
              cnf_tc::bar_expect_tx(full(s), stage);
              const uint32_t ab = (uint32_t)(mb * mdim) / 8 * 256;
              cnf_tc::bulk_load(sm() + base, rec + zoff + ab, abytes, full(s));
              cnf_tc::bulk_load(sm() + base + abytes, rec + zoff + ztile + ab, abytes, full(s));
              uint32_t o = base + 2 * abytes;
              for (int j = 0; j < ncur; ++j) {
                const uint32_t bb = (uint32_t)((c0 + j) * cnf_tc::kNW) / 8 * 256;
                cnf_tc::bulk_load(sm() + o, rec + aoff + bb, bbytes[j], full(s));
                cnf_tc::bulk_load(sm() + o + bbytes[j], rec + aoff + atile + bb, bbytes[j], full(s));
                o += 2 * bbytes[j];
              }
            }
            __syncwarp();
            tc::bar_wait(full(s), (v >> 1) & 1u);
            tc::fence_after();
            const uint32_t a = sb + base;
            const uint64_t Ah = tc::sdesc(a, 128, 256), Al = tc::sdesc(a + abytes, 128, 256);
            uint32_t o = a + 2 * abytes;
            for (int j = 0; j < ncur; ++j) {
              const uint64_t Bh = tc::sdesc(o, 128, 256), Bl = tc::sdesc(o + bbytes[j], 128, 256);
              const uint32_t dt = (uint32_t)j * cnf_tc::kNW;
              const uint32_t id = mdim == 128 ? tc::idesc_bf16(128, nw[j], true, true)
                                              : tc::idesc_bf16(64, nw[j], true, true);
              tc::mma_bf16_keep_a(dt, Ah, Bh, id, v > 0 ? 1u : 0u);
              tc::mma_bf16_reuse_a(dt, Ah, Bl, id, 1u);
              tc::mma_bf16(dt, Al, Bh, id, 1u);
              o += 2 * bbytes[j];
            }
            tc::commit(empty(s));
          }
          for (int v = max(0, nlog - 2); v < nlog; ++v) tc::bar_wait(empty(v & 1), (v >> 1) & 1u);
          tc::commit(done());
        }
        tc::bar_wait(done(), done_phase);
        done_phase ^= 1u;
        tc::fence_after();
        // flush: rows (outputs) -> TMEM lanes (M = 128: lane = row; M = 64: 32 (r/16) + r%16)
        const int wq = threadIdx.x >> 5, lane = threadIdx.x & 31, q = wq & 3, cg = wq >> 2;
        int r;
        bool ok;
        if (mdim == 128) { r = 32 * q + lane; ok = true; }
        else { r = 16 * q + lane; ok = lane < 16; }
        const int orow = mb * mdim + r;
        for (int j = 0; j < ncur; ++j) {
          for (int cc = cg * 16; cc < nw[j]; cc += 64) {   // 16-column groups per warp group
            float v16[16];
            tc::ld16(((uint32_t)(32 * q) << 16) + (uint32_t)j * cnf_tc::kNW + cc, v16);
            if (ok && orow < mrows) {
              T* drow = dst + (long long)orow * ldm;
              const int k0 = (c0 + j) * cnf_tc::kNW + cc;
              for (int e = 0; e < 16; ++e)
                if (k0 + e < ldm) drow[k0 + e] += T(v16[e]);
            }
          }
        }
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
      }
    }
  }

  OB_DEV void finish(T* mu) {
    if (!mu || nlog == 0) return;
    const Dims& d = p.d;
    if (threadIdx.x == 0) {
      cnf_tc::bulk_wait_all();
      cnf_tc::fence_async_global();
    }
    __syncthreads();
    // dW1 [H][H] (mu row stride ldm[1]): zbar2 outputs x [a1; u1] inputs
    gemm_log(G::LZ2, G::TA, G::MB, 128, G::LA1, G::TA, G::KH, mu + d.mwoff[1], d.ldm[1], H);
    // dW0 [H][D + 1]: zbar1 x X0
    gemm_log(G::LZ1, G::TA, G::MB, 128, G::LX0, G::TX, G::K0, mu + d.mwoff[0], d.ldm[0], H);
    // dW2 [D][H]: Z3 x [a2; u2]
    gemm_log(G::LZ3, G::TX, 1, 64, G::LA2, G::TA, G::KH, mu + d.mwoff[2], d.ldm[2], D);
    __syncthreads();
  }
  OB_DEV void reinit() {
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int s = 0; s < 2; ++s) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(full(s))) : "memory");
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(empty(s))) : "memory");
        tc::bar_init(full(s), 1);
        tc::bar_init(empty(s), 1);
      }
    }
    __syncthreads();
  }

  OB_DEV void release() {
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_free(0u, kCols);
  }
};

// packed weight chunks in streaming order (forward W0, W1, W2; transposed W2^T, W1^T,
// W0^T), each [M][kKc] bf16 hi then lo in the K-major core-block layout of w_off
template <int D, int H>
__global__ void pack_tc_cnf_kernel(const __grid_constant__ Dims d, const float* theta, unsigned char* img) {
  using G = CnfGeom<D, H>;
  constexpr int kc = cnf_tc::kKc;
  const float* W0 = theta + d.woff[0];   // [H][D + 1]
  const float* W1 = theta + d.woff[1];   // [H][H]
  const float* W2 = theta + d.woff[2];   // [D][H]
  // element counts per product (chunks x M x kKc)
  const long long n0 = (long long)G::MB * (G::K0 / kc) * 128 * kc;
  const long long n1 = (long long)G::MB * (G::KH / kc) * 128 * kc;
  const long long n2 = (long long)(G::KH / kc) * 64 * kc;
  const long long tot = 2 * (n0 + n1 + n2);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    long long j = i;
    int prod = 0;
    const long long sizes[6] = {n0, n1, n2, n0, n1, n2};
    while (j >= sizes[prod]) { j -= sizes[prod]; ++prod; }
    const int M = (prod == 2 || prod == 5) ? 64 : 128;
    const int nkc = (prod == 0 || prod == 3) ? G::K0 / kc : G::KH / kc;
    const long long per = (long long)M * kc;
    const int chunk = (int)(j / per), e = (int)(j % per);
    const int m = e / kc, k = e % kc;
    const int mb = chunk / nkc, kcix = chunk % nkc;
    const int row = mb * M + m, col = kcix * kc + k;
    float x = 0.f;
    switch (prod) {
      case 0: if (row < H && col < D + 1) x = W0[(long long)row * (D + 1) + col]; break;
      case 1: if (row < H && col < H) x = W1[(long long)row * H + col]; break;
      case 2: if (row < D && col < H) x = W2[(long long)row * H + col]; break;
      case 3: if (row < H && col < D) x = W2[(long long)col * H + row]; break;   // W2^T
      case 4: if (row < H && col < H) x = W1[(long long)col * H + row]; break;   // W1^T
      default: if (row < D + 1 && col < H) x = W0[(long long)col * (D + 1) + row]; break;  // W0^T
    }
    const uint32_t base[6] = {G::P0f, G::P1f, G::P2f, G::P2b, G::P1b, G::P0b};
    const uint32_t cb = (uint32_t)M * kc * 2;
    unsigned char* c0 = img + base[prod] + (uint32_t)chunk * 2 * cb;
    uint16_t hi, lo;
    tc::split_bf16(x, hi, lo);
    *reinterpret_cast<uint16_t*>(c0 + cnf_tc::w_off(m, k)) = hi;
    *reinterpret_cast<uint16_t*>(c0 + cb + cnf_tc::w_off(m, k)) = lo;
  }
}

}  // namespace ob
