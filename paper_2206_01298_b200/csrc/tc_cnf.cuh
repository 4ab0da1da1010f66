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
// Weight chunks are large: a bulk copy costs ~600 cycles of TMA service per SM almost
// independently of its size up to ~64 KB (tools/tma_probe: 16 KB copies stream at
// 17-27 B/cycle/SM, 64 KB copies at 73 B/cycle/SM with one copy in flight behind the
// one being consumed), so the ring holds three 48 KB chunks (128 rows x 96 K, hi | lo):
// two copies stay in flight behind the chunk the MMAs consume.
constexpr int kKc = 96;           // K per weight chunk (six 16-wide K slices; 864 = 9 x 96)
constexpr int kNS = 3;            // weight ring slots
constexpr uint32_t kSlot = 49152; // bytes per slot (M = 128 chunk, hi | lo)
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
// weight chunk [M][kKc] K-major: byte(m, k) = (m/8)*kWSA + (k/8)*128 + (m%8)*16 + (k%8)*2
constexpr uint32_t kWSA = (uint32_t)(kKc / 8) * 128u;   // row-group stride (descriptor SBO)
__host__ __device__ constexpr uint32_t w_off(int m, int k) {
  return (uint32_t)(m >> 3) * kWSA + (uint32_t)(k >> 3) * 128u + (uint32_t)(m & 7) * 16u +
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
  static constexpr int K0 = cnf_tc::kKc;             // [z, t] padded to one chunk (D + 1 <= 64)
  static constexpr int KH = (H + cnf_tc::kKc - 1) / cnf_tc::kKc * cnf_tc::kKc;   // whole chunks
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
  static constexpr uint32_t TX = cnf_tc::tile_bytes(K0);     // X0 / Z3 tiles (K = K0)
  static constexpr uint32_t TA = cnf_tc::tile_bytes(KH);     // hidden tiles
  static constexpr uint32_t X0h = 0, X0l = X0h + TX;
  static constexpr uint32_t Z3h = X0l + TX, Z3l = Z3h + TX;
  // one stacked hidden tile serves every hidden-width operand in turn ([a1; u1], [a2; u2],
  // [zbar2; sbar2], [zbar1; sbar1]): each is logged and consumed by its product before the
  // next epilogue overwrites it, which leaves room for a deeper weight ring
  static constexpr uint32_t ABh = Z3l + TX, ABl = ABh + TA;
  static constexpr uint32_t Ring = ABl + TA;                  // kNS slots (contiguous after AB)
  static constexpr uint32_t Jeps = Ring + cnf_tc::kNS * cnf_tc::kSlot;   // fp32 [8][64]
  static constexpr uint32_t Bars = Jeps + 8 * 64 * 4;         // full[kNS] empty[kNS] done gemm[4]
  static constexpr uint32_t Slot = Bars + 8 * (2 * cnf_tc::kNS + 8);
  static constexpr uint32_t Total = (Slot + 8 + 127) / 128 * 128;
  // dW log, panel layout: for every operand tile a VJP logs, its blocks (the dW GEMMs'
  // M blocks / N chunks: 128 or 224 features x 16 rows) are stored [block][vjp][hi | lo],
  // so a dW output tile streams many VJPs of one block in a single bulk copy
  static constexpr int NC = (KH + cnf_tc::kNW - 1) / cnf_tc::kNW;       // N chunks of a hidden input
  static constexpr uint32_t BZ = 16 * 256;                             // 128-feature block (per copy)
  static constexpr uint32_t BA = (uint32_t)cnf_tc::kNW / 8 * 256;      // 224-feature chunk
  static constexpr uint32_t BZ3 = 8 * 256;                             // 64 features (M = 64)
  static constexpr uint32_t BX0 = TX;                                  // the whole X0 tile
  static constexpr uint32_t Log = 2 * (2 * MB * BZ + 2 * NC * BA + BZ3 + BX0);   // bytes per VJP
  // TMEM columns (fp32, N = 16 per M block)
  static constexpr uint32_t T_Z1 = 0, T_Z2 = T_Z1 + 16 * MB, T_OUT = T_Z2 + 16 * MB,
                            T_G2 = T_OUT + 16, T_G1 = T_G2 + 16 * MB, T_G0 = T_G1 + 16 * MB,
                            T_END = T_G0 + 16;
  static_assert(D + 1 <= 64, "state dim (M = 64 blocks for the D-row layers)");
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
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
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

template <typename T, int D, int H, int CL>
struct TcCnfAdapter {
  static_assert(sizeof(T) == 4, "tensor-core CNF tile is fp32");
  using G = CnfGeom<D, H>;
  static constexpr bool kHasJvp = false;
  static constexpr bool kScaledVjp = true;    // vjp returns J^T (h w), mu += P^T (h w)
  static constexpr int kCombineBatch = 4;
  static constexpr bool kOwnsStep = false;
  static constexpr bool kNoEarlyExit = CL > 1;   // the cluster streams weights together
  static constexpr uint32_t kCols = 512;
  static constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);

  const RkParams<T>& p;
  int Rv, row0;
  float tcur;
  // weight-stream state (warp 0): chunk ordinals across all products of the sweep
  uint32_t head, tail, done_phase;
  int nlog;              // VJPs logged so far
  unsigned char* logp;   // this tile's log
  uint32_t crank;        // rank in the thread-block cluster (chunk c is loaded by rank c % CL)

  OB_DEV unsigned char* sm() const { return ob_tc_smem; }
  OB_DEV uint64_t* full(int s) const { return reinterpret_cast<uint64_t*>(ob_tc_smem + G::Bars) + s; }
  OB_DEV uint64_t* empty(int s) const {
    return reinterpret_cast<uint64_t*>(ob_tc_smem + G::Bars) + cnf_tc::kNS + s;
  }
  OB_DEV uint64_t* done() const { return reinterpret_cast<uint64_t*>(ob_tc_smem + G::Bars) + 2 * cnf_tc::kNS; }
  OB_DEV const unsigned char* packed() const { return reinterpret_cast<const unsigned char*>(p.packed); }

  OB_DEV TcCnfAdapter(const RkParams<T>& p_, const Weights<T>&, MlpSmem<T>&, T*, int row0_, int Rv_)
      : p(p_), Rv(Rv_ > 0 ? Rv_ : 0), row0(row0_), tcur(0.f), head(0), tail(0), done_phase(0), nlog(0), crank(0) {
    if constexpr (CL > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    logp = reinterpret_cast<unsigned char*>(p.cnf_pre) + (long long)blockIdx.x * p.cnf_pre_stride * sizeof(T);
    // zero the operand tiles (padded rows / features stay exactly zero)
    uint4* z = reinterpret_cast<uint4*>(ob_tc_smem);
    for (int i = threadIdx.x; i < (int)(G::Ring / 16); i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) tc::tmem_alloc(reinterpret_cast<uint32_t*>(ob_tc_smem + G::Slot), kCols);
    if (threadIdx.x == 0) {
      for (int s = 0; s < cnf_tc::kNS; ++s) {
        tc::bar_init(full(s), 1);
        tc::bar_init(empty(s), CL);   // every CTA of the cluster releases the slot
      }
      tc::bar_init(done(), 1);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if constexpr (CL > 1) cluster_sync();   // barriers initialised cluster-wide before any multicast
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

  OB_DEV static void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  // MMA completion of this CTA -> the slot's empty barrier in every CTA of the cluster
  OB_DEV void commit_empty(int s) {
    if constexpr (CL == 1) {
      tc::commit(empty(s));
    } else {
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
              tc::smem_u32(empty(s))),
          "h"(kMask)
          : "memory");
    }
  }
  // ---- weight stream (warp 0): chunk idx lands in slot idx % kNS of every CTA of the
  // cluster; rank idx % CL issues it (multicast), every CTA expects its bytes
  OB_DEV void load_chunk(uint32_t idx, uint32_t src, uint32_t bytes) {
    const int s = (int)(idx % cnf_tc::kNS);
    if (cnf_tc::elect_one()) {
      cnf_tc::bar_expect_tx(full(s), bytes);
      if constexpr (CL == 1) {
        cnf_tc::bulk_load(sm() + G::Ring + s * cnf_tc::kSlot, packed() + src, bytes, full(s));
      } else if (idx % CL == crank) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
            " [%0], [%1], %2, [%3], %4;" ::"r"(tc::smem_u32(sm() + G::Ring + s * cnf_tc::kSlot)),
            "l"(packed() + src), "r"(bytes), "r"(tc::smem_u32(full(s))), "h"(kMask)
            : "memory");
      }
    }
    __syncwarp();
  }
  // ---- products, warp-specialised: warp 1 streams the weight chunks (TMA) as ring slots
  // free up, warp 0 issues the MMAs of each chunk as it lands; chunk ordinals run on
  // across products (slot = ordinal % kNS), so warp 1 may load the next product's first
  // chunks while the epilogue of this one runs.
  OB_DEV static uint32_t chunk_bytes(int m) { return (uint32_t)m * cnf_tc::kKc * 2 * 2; }
  OB_DEV void produce(uint32_t idx, uint32_t src, uint32_t bytes) {
    const int s = (int)(idx % cnf_tc::kNS);
    if (idx >= (uint32_t)cnf_tc::kNS) {   // every CTA of the cluster consumed the slot's last chunk
      const uint32_t prev = idx - cnf_tc::kNS;
      tc::bar_wait(empty(s), (prev / cnf_tc::kNS) & 1u);
    }
    load_chunk(idx, src, bytes);
  }
  // D[mb] (+)= W x B over the product's K: chunk c = (mb, kc); B = tile at smem offset bh / bl
  template <int M>
  OB_DEV void consume(const CnfProd& pr, uint32_t dcol, uint32_t bh, uint32_t bl) {
    constexpr uint32_t id = tc::idesc_bf16(M, cnf_tc::kRows, false, false);
    const uint32_t half = chunk_bytes(M) / 2;
    const uint32_t n = (uint32_t)(pr.nmb * pr.nkc);
    const uint32_t sb = tc::smem_u32(ob_tc_smem);
    constexpr int KS = cnf_tc::kKc / 16;   // K slices per chunk
    for (uint32_t c = 0; c < n; ++c) {
      const uint32_t idx = tail + c;
      const int s = (int)(idx % cnf_tc::kNS);
      tc::bar_wait(full(s), (idx / cnf_tc::kNS) & 1u);
      tc::fence_after();
      const int mb = (int)(c / pr.nkc), kc = (int)(c % pr.nkc);
      const uint32_t a = sb + G::Ring + s * cnf_tc::kSlot;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const uint64_t Ah = tc::sdesc(a + ks * 256, 128, cnf_tc::kWSA),
                       Al = tc::sdesc(a + half + ks * 256, 128, cnf_tc::kWSA);
        const uint32_t bo = (uint32_t)(KS * kc + ks) * 512u;
        const uint64_t Bh = tc::sdesc(sb + bh + bo, 256, 128), Bl = tc::sdesc(sb + bl + bo, 256, 128);
        const uint32_t dt = dcol + 16u * mb;
        tc::mma_bf16_keep_a(dt, Ah, Bh, id, (kc > 0 || ks > 0) ? 1u : 0u);
        tc::mma_bf16_reuse_a(dt, Ah, Bl, id, 1u);
        tc::mma_bf16(dt, Al, Bh, id, 1u);
      }
      commit_empty(s);
    }
    tc::commit(done());
  }
  // every thread: wait for the product issued by warp 0
  OB_DEV void wait_done() {
    tc::bar_wait(done(), done_phase);
    done_phase ^= 1u;
    tc::fence_after();
  }
  // product `which` into TMEM columns dcol from the B tile (bh, bl); `next`: the product
  // that follows within the same field call (its first chunks are prefetched), or -1
  OB_DEV void issue(int which, int next, uint32_t dcol, uint32_t bh, uint32_t bl) {
    const CnfProd pr = prod(which);
    const uint32_t n = (uint32_t)(pr.nmb * pr.nkc);
    const int w = tc::uniform_warp();
    if (w == 1) {
      const uint32_t cb = chunk_bytes(pr.m);
      for (uint32_t idx = head > tail ? head : tail; idx < tail + n; ++idx)
        produce(idx, pr.src + (idx - tail) * cb, cb);
      head = tail + n;
      if (next >= 0) {
        const CnfProd nx = prod(next);
        const uint32_t nn = (uint32_t)(nx.nmb * nx.nkc), ncb = chunk_bytes(nx.m);
        for (uint32_t k = 0; k + 1 < (uint32_t)cnf_tc::kNS && k < nn; ++k, ++head)
          produce(head, nx.src + k * ncb, ncb);
      }
    } else if (w == 0) {
      if (pr.m == 128) consume<128>(pr, dcol, bh, bl);
      else consume<64>(pr, dcol, bh, bl);
    }
    tail += n;
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
  // (log: the VJP's layer inputs are logged as they are produced)
  OB_DEV void hidden_forward(bool log, int next) {
    sync_issue();
    issue(0, 1, G::T_Z1, G::X0h, G::X0l);
    epi_hidden(G::T_Z1, p.W.bias[0], G::ABh, G::ABl);         // [a1; u1]
    sync_issue();
    if (log) log_panel(G::ABh, G::ABl, kSecA1, G::NC, G::BA);
    issue(1, next, G::T_Z2, G::ABh, G::ABl);
    epi_hidden(G::T_Z2, p.W.bias[1], G::ABh, G::ABl);         // [a2; u2] over [a1; u1]
  }

  // f_aug(x0) -> out [Rt][ldn]: columns [0, D) = f, column D = -eps^T J eps
  OB_DEV void eval(T* out) {
    hidden_forward(false, 2);
    sync_issue();
    issue(2, -1, G::T_OUT, G::ABh, G::ABl);
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

  // ---- dW log (panel layout, see CnfGeom): section offsets for this tile's capacity
  enum { kSecZ2 = 0, kSecZ1, kSecA1, kSecA2, kSecZ3, kSecX0 };
  OB_DEV long long cap() const { return p.cnf_pre_stride * (long long)sizeof(T) / G::Log; }
  OB_DEV long long sec_off(int sec) const {
    const long long c = cap();
    const long long z = (long long)G::MB * c * 2 * G::BZ, a = (long long)G::NC * c * 2 * G::BA;
    switch (sec) {
      case kSecZ2: return 0;
      case kSecZ1: return z;
      case kSecA1: return 2 * z;
      case kSecA2: return 2 * z + a;
      case kSecZ3: return 2 * z + 2 * a;
      default: return 2 * z + 2 * a + c * 2 * G::BZ3;
    }
  }
  // append the blocks of the stacked tile (hi, lo) to section sec for VJP nlog (all
  // threads, 16-byte copies; the tile may be overwritten after the next barrier)
  OB_DEV void log_panel(uint32_t h, uint32_t l, int sec, int nblk, uint32_t bb) {
#ifdef OB_EXP_NO_LOG
    return;
#endif
    uint4* dst0 = reinterpret_cast<uint4*>(logp + sec_off(sec));
    const int units = (int)(bb / 16);
    const long long c = cap();
    for (int i = threadIdx.x; i < nblk * 2 * units; i += blockDim.x) {
      const int blk = i / (2 * units), r = i % (2 * units), hl = r / units, u = r % units;
      const uint4 v = *reinterpret_cast<const uint4*>(sm() + (hl ? l : h) + blk * bb + u * 16);
      dst0[((blk * c + nlog) * 2 * bb + hl * bb) / 16 + u] = v;
    }
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
    hidden_forward(mu != nullptr, 3);
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
    if (mu) {   // the rest of this VJP's layer inputs and the output cotangent
      log_panel(G::X0h, G::X0l, kSecX0, 1, G::BX0);
      log_panel(G::ABh, G::ABl, kSecA2, G::NC, G::BA);
      log_panel(G::Z3h, G::Z3l, kSecZ3, 1, G::BZ3);
    }
    issue(3, 4, G::T_G2, G::Z3h, G::Z3l);                // [abar2; ubar2] = W2^T Z3
    epi_back(G::T_G2, G::T_Z2, p.W.bias[1], G::ABh, G::ABl, mu ? mu + d.mboff[1] : nullptr);
    sync_issue();
    if (mu) log_panel(G::ABh, G::ABl, kSecZ2, G::MB, G::BZ);   // Zb2
    issue(4, 5, G::T_G1, G::ABh, G::ABl);                // [abar1; ubar1] = W1^T Zb2
    epi_back(G::T_G1, G::T_Z1, p.W.bias[0], G::ABh, G::ABl, mu ? mu + d.mboff[0] : nullptr);
    sync_issue();
    if (mu) log_panel(G::ABh, G::ABl, kSecZ1, G::MB, G::BZ);   // Zb1
    issue(5, -1, G::T_G0, G::ABh, G::ABl);               // W0^T Zb1: rows 0..D-1 = J^T (h w)
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
    if (mu) ++nlog;
    tc::fence_before();
    __syncthreads();
  }

  // ---- deferred parameter cotangents: dW_l = sum over logged VJPs of [zbar; sbar]^T [a; u]
  // One output tile D[M block][N chunk] at a time, accumulated in TMEM over K = 16 rows per
  // VJP; the operands stream from the panel log kVB VJPs per stage (two bulk copies),
  // through three stages in the AB + ring region.
  static constexpr int kVB = 3;
  OB_DEV void gemm_panel(int secA, int nblkA, int mdim, uint32_t bbA, int secB, int nblkB,
                         uint32_t bbB, int kin, T* dst, int ldm, int mrows) {
    const uint32_t sb = tc::smem_u32(ob_tc_smem);
    const long long c = cap();
    const int nst = (nlog + kVB - 1) / kVB;
    const uint32_t stage = (uint32_t)kVB * 2 * (bbA + bbB);
    const unsigned char* pa = logp + sec_off(secA);
    const unsigned char* pb = logp + sec_off(secB);
    PhaseTimer pt(p.prof ? p.phase : nullptr);
    for (int mb = 0; mb < nblkA; ++mb) {
      for (int nc = 0; nc < nblkB; ++nc) {
        reinit();
        pt.mark(12);
        const int nw = min(cnf_tc::kNW, kin - nc * cnf_tc::kNW);
        const uint32_t id = mdim == 128 ? tc::idesc_bf16(128, nw, true, true) : tc::idesc_bf16(64, nw, true, true);
        // staging by every thread with 16-byte cp.async (the log lives in HBM: many
        // small requests in flight beat a few serialized bulk copies here)
        auto load = [&](int st) {
          const int v0 = st * kVB, nvb = min(kVB, nlog - v0), sl = st % 3;
          const uint32_t bytesA = (uint32_t)nvb * 2 * bbA, bytesB = (uint32_t)nvb * 2 * bbB;
          unsigned char* base = sm() + G::ABh + sl * stage;
          const unsigned char* ga = pa + ((long long)mb * c + v0) * 2 * bbA;
          const unsigned char* gb = pb + ((long long)nc * c + v0) * 2 * bbB;
          for (uint32_t o = threadIdx.x * 16u; o < bytesA; o += blockDim.x * 16u) cnf_tc::cp16(base + o, ga + o);
          for (uint32_t o = threadIdx.x * 16u; o < bytesB; o += blockDim.x * 16u)
            cnf_tc::cp16(base + kVB * 2 * bbA + o, gb + o);
          cnf_tc::cp_commit();
        };
        load(0);
        if (nst > 1) load(1); else cnf_tc::cp_commit();
        for (int st = 0; st < nst; ++st) {
          if (st + 2 < nst) {   // refill the slot of stage st - 1 once its MMAs completed
            if (st >= 1) {
              tc::bar_wait(empty((st - 1) % 3), ((st - 1) / 3) & 1u);
              tc::fence_after();
            }
            load(st + 2);
          } else {
            cnf_tc::cp_commit();   // keep one group per iteration
          }
          cnf_tc::cp_wait<2>();    // this thread's copies of stage st landed
          tc::fence_async_smem();
          __syncthreads();
          if (tc::uniform_warp() == 0) {
            tc::fence_after();
            const int sl = st % 3, v0 = st * kVB, nvb = min(kVB, nlog - v0);
            const uint32_t base = sb + G::ABh + sl * stage;
            for (int jv = 0; jv < nvb; ++jv) {
              const uint32_t a = base + jv * 2 * bbA, b = base + kVB * 2 * bbA + jv * 2 * bbB;
              const uint64_t Ah = tc::sdesc(a, 128, 256), Al = tc::sdesc(a + bbA, 128, 256);
              const uint64_t Bh = tc::sdesc(b, 128, 256), Bl = tc::sdesc(b + bbB, 128, 256);
              tc::mma_bf16_keep_a(0u, Ah, Bh, id, (v0 + jv) > 0 ? 1u : 0u);
              tc::mma_bf16_reuse_a(0u, Ah, Bl, id, 1u);
              tc::mma_bf16(0u, Al, Bh, id, 1u);
            }
            tc::commit(empty(sl));
            if (st == nst - 1) tc::commit(done());
          }
        }
        tc::bar_wait(done(), done_phase);
        done_phase ^= 1u;
        tc::fence_after();
        pt.mark(10);
        // flush: TMEM rows (M = 128: lane = row; M = 64: lane 32 (r/16) + r%16) -> a shared
        // fp32 tile -> coalesced 16-byte stores.  Every dW entry is produced by exactly one
        // output tile of one finish(), so it is stored, not accumulated (mu starts at zero).
        {
          constexpr int kLd = cnf_tc::kNW + 4;   // padded row stride (floats)
          float* tile = reinterpret_cast<float*>(sm() + G::ABh);
          const int wq = threadIdx.x >> 5, lane = threadIdx.x & 31, q = wq & 3, cg = wq >> 2;
          const int r = mdim == 128 ? 32 * q + lane : 16 * q + lane;
          const bool ok = mdim == 128 || lane < 16;
          for (int cc = cg * 16; cc < nw; cc += 64) {
            float v16[16];
            tc::ld16(((uint32_t)(32 * q) << 16) + (uint32_t)cc, v16);
            if (ok)
              for (int e = 0; e < 16; e += 4)
                *reinterpret_cast<float4*>(tile + r * kLd + cc + e) =
                    make_float4(v16[e], v16[e + 1], v16[e + 2], v16[e + 3]);
          }
          tc::fence_before();
          __syncthreads();
          const int rows = min(mdim, mrows - mb * mdim), k0 = nc * cnf_tc::kNW;
          const int ncol = min(nw, ldm - k0), n4 = (ncol + 3) / 4;
          for (int i = threadIdx.x; i < rows * n4; i += blockDim.x) {
            const int rr = i / n4, c4 = i % n4;
            const float4 v = *reinterpret_cast<const float4*>(tile + rr * kLd + 4 * c4);
            T* drow = dst + (long long)(mb * mdim + rr) * ldm + k0 + 4 * c4;
            if (4 * c4 + 3 < ncol) {
              *reinterpret_cast<float4*>(drow) = v;
            } else {
              const float e4[4] = {v.x, v.y, v.z, v.w};
              for (int e = 0; 4 * c4 + e < ncol; ++e) drow[e] = T(e4[e]);
            }
          }
        }
        tc::fence_before();
        __syncthreads();
        pt.mark(11);
      }
    }
  }

  OB_DEV void finish(T* mu) {
    // the cluster's weight multicasts into this CTA's ring are over before the ring
    // region is reused for the log GEMM staging
    if constexpr (CL > 1) {
      tc::fence_before();
      cluster_sync();
    }
    if (!mu || nlog == 0) return;
#ifdef OB_EXP_NO_FINISH
    return;
#endif
    const Dims& d = p.d;
    // the log was written by generic stores: visible to the bulk (async-proxy) loads
    cnf_tc::fence_async_global();
    __syncthreads();
    // dW1 [H][H] (mu row stride ldm[1]): [zbar2; sbar2] outputs x [a1; u1] inputs
    gemm_panel(kSecZ2, G::MB, 128, G::BZ, kSecA1, G::NC, G::BA, G::KH, mu + d.mwoff[1], d.ldm[1], H);
    // dW0 [H][D + 1]: [zbar1; sbar1] x [x; e]
    gemm_panel(kSecZ1, G::MB, 128, G::BZ, kSecX0, 1, G::BX0, G::K0, mu + d.mwoff[0], d.ldm[0], H);
    // dW2 [D][H]: Z3 x [a2; u2]
    gemm_panel(kSecZ3, 1, 64, G::BZ3, kSecA2, G::NC, G::BA, G::KH, mu + d.mwoff[2], d.ldm[2], D);
    __syncthreads();
  }
  OB_DEV void reinit() {
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int s = 0; s < 3; ++s) {
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
    if constexpr (CL > 1) cluster_sync();   // no CTA leaves while a partner may still multicast to it
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
