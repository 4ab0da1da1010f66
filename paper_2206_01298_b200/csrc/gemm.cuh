// gemm.cuh -- register-tiled CTA GEMMs for the persistent sample-tile kernels.
//
// A CTA holds R (<= 32) samples; its contractions are small GEMMs with the
// sample rows on one side and a weight matrix (shared memory when it fits,
// else L1/L2-resident global) on the other.  A thread owns a TR x TC output
// block; a warp's 32 lanes are arranged LR x LC (LR*LC = 32) so one warp covers
// a (TR*LR) x (TC*LC) tile.  Rows of a thread block are r0 + lr + LR*i and
// columns c0 + lc + LC*j (strided), which makes every 16-byte shared-memory
// access conflict-free when leading dimensions are "odd quads" (ld/4 odd).
// Activation operands are always shared memory and are read with explicit
// ld.shared vector loads; weights use ld.shared (WS) or ld.global.nc.
//
//   gemm_nt : Z[r][n] = sum_k X[r][k] W[n][k]        (forward / JVP, z = W x)
//   gemm_nn : O[r][k] = sum_n D[r][n] W[n][k]        (VJP input product d W)
//   gemm_tn : M[n][k] += s * sum_r D[r][n] X[r][k]   (parameter cotangent)
// Padding contract: operand rows up to the row tile and columns up to the next
// multiple of 4 (weights: up to the column tile the op reads) exist and are
// finite; weight padding is zero, so padded lanes contribute exact zeros.
#pragma once

#include "tile.cuh"

namespace ob {

OB_DEV uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <typename T> struct Ld;
template <> struct Ld<float> {
  static OB_DEV void s4(uint32_t a, float v[4]) {
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
  }
  static OB_DEV void g4(const float* p, float v[4]) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
};
template <> struct Ld<double> {
  static OB_DEV void s4(uint32_t a, double v[4]) {
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(a));
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v[2]), "=d"(v[3]) : "r"(a + 16));
  }
  static OB_DEV void g4(const double* p, double v[4]) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};

// weight operand: shared (byte address) or global pointer
template <typename T, bool WS> struct WOp;
template <typename T> struct WOp<T, true> {
  uint32_t base;
  OB_DEV WOp(const T* p) : base(smem_addr(p)) {}
  OB_DEV void ld4(long long off, T v[4]) const { Ld<T>::s4(base + (uint32_t)(off * sizeof(T)), v); }
};
template <typename T> struct WOp<T, false> {
  const T* base;
  OB_DEV WOp(const T* p) : base(p) {}
  OB_DEV void ld4(long long off, T v[4]) const { Ld<T>::g4(base + off, v); }
};

template <typename T> struct Vec4;
template <> struct Vec4<float> {
  static OB_DEV void ld(const float* p, float v[4]) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
  static OB_DEV void st(float* p, const float v[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct Vec4<double> {
  static OB_DEV void ld(const double* p, double v[4]) {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  static OB_DEV void st(double* p, const double v[4]) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
  }
};

OB_DEV int warp_id() { return threadIdx.x >> 5; }
OB_DEV int lane_id() { return threadIdx.x & 31; }
OB_DEV int n_warps() { return blockDim.x >> 5; }

template <typename T>
OB_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
OB_DEV T warp_dot(const T* a, const T* b, int n) {
  T s = T(0);
  for (int j = lane_id(); j < n; j += 32) s = Num<T>::fma(a[j], b[j], s);
  return warp_sum(s);
}

// ---- per-warp cp.async rings for weights streamed from L2 (WS = false): each warp
// copies the weight slice of k-step k + kRing - 1 into its private ring while it
// consumes step k, so kRing - 1 steps of 16-byte loads are in flight per lane
// without holding registers (one CTA per SM cannot hide L2 latency with 16 warps).
template <typename T> struct RingDepth { static constexpr int value = sizeof(T) == 4 ? 4 : 2; };
OB_DEV void ring_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
OB_DEV void ring_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> OB_DEV void ring_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Warp range executing an op: warps [w0, w0 + nw) of the CTA.
struct Warps {
  int w0, nw;
  OB_DEV static Warps all() { return {0, n_warps()}; }
  OB_DEV bool mine() const { return warp_id() >= w0 && warp_id() < w0 + nw; }
  OB_DEV int me() const { return warp_id() - w0; }
};

// Z[r][n] = sum_{k in [kb, ke)} X[r][k] * W[n][k];  epi(r, n, acc) for n < N.
// Rt: rows to compute (multiple of TR*LR).  split > 1 partitions k into
// `split` slices (multiples of 4) and calls epi(r, n, acc, slice).
template <typename T, int TR, int TC, int LR, bool WS, class Epi>
OB_DEV void gemm_nt(const T* X, int ldx, int Rt, const T* W, int ldw, int N, int Kp, Warps ws,
                    int split, Epi epi, T* ring = nullptr, int ring_elems = 0) {
  constexpr int LC = 32 / LR, RT = TR * LR, CT = TC * LC;
  if (!ws.mine()) return;
  const int lr = lane_id() % LR, lc = lane_id() / LR;
  const int rtiles = Rt / RT, ctiles = (N + CT - 1) / CT;
  const int kq = Kp / 4, per = (kq + split - 1) / split;
  const uint32_t xs = smem_addr(X);
  const WOp<T, WS> wo(W);
  if constexpr (!WS) {
    // ring slot: the task's CT weight rows x 4 k (row-major [CT][4])
    constexpr int kD = RingDepth<T>::value, kV = 16 / (int)sizeof(T), kPer = 4 / kV;
    constexpr int kSlot = CT * 4;
    if (ring && ring_elems / n_warps() >= kD * kSlot) {
      T* wr = ring + (long long)warp_id() * (ring_elems / n_warps());
      const int lane = lane_id();
      for (int task = ws.me(); task < rtiles * ctiles * split; task += ws.nw) {
        const int sl = task / (rtiles * ctiles), rc = task % (rtiles * ctiles);
        const int r0 = (rc % rtiles) * RT + lr, cb = (rc / rtiles) * CT, c0 = cb + lc;
        const int kb = sl * per * 4, ke = min(Kp, (sl + 1) * per * 4);
        auto issue = [&](int kk, int slot) {
          if (kk < ke)
            for (int c = lane; c < CT * kPer; c += 32) {
              const int r = c / kPer, hh = c % kPer;
              ring_cp16(wr + slot * kSlot + r * 4 + hh * kV, W + (long long)(cb + r) * ldw + kk + hh * kV);
            }
          ring_commit();
        };
        __syncwarp();   // the previous task's reads of the ring are complete
#pragma unroll
        for (int dd = 0; dd < kD - 1; ++dd) issue(kb + 4 * dd, dd);
        T acc[TR][TC];
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) acc[i][j] = T(0);
        int slot = 0;
        for (int k = kb; k < ke; k += 4) {
          __syncwarp();   // slot (slot - 1) mod kD was read last iteration; refill it
          issue(k + 4 * (kD - 1), (slot + kD - 1) % kD);
          ring_wait<kD - 1>();
          __syncwarp();
          T x[TR][4], w[TC][4];
#pragma unroll
          for (int j = 0; j < TC; ++j) {
            const T* src = wr + slot * kSlot + (lc + j * LC) * 4;
            if constexpr (sizeof(T) == 4) {
              Ld<T>::s4(smem_addr(src), w[j]);
            } else {
              Ld<T>::s4(smem_addr(src), w[j]);
            }
          }
#pragma unroll
          for (int i = 0; i < TR; ++i)
            Ld<T>::s4(xs + (uint32_t)(((r0 + i * LR) * ldx + k) * sizeof(T)), x[i]);
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int i = 0; i < TR; ++i)
#pragma unroll
              for (int j = 0; j < TC; ++j) acc[i][j] = Num<T>::fma(x[i][q], w[j][q], acc[i][j]);
          slot = slot + 1 == kD ? 0 : slot + 1;
        }
        ring_wait<0>();
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) {
            const int n = c0 + j * LC;
            if (n < N) epi(r0 + i * LR, n, acc[i][j], sl);
          }
      }
      return;
    }
  }
  for (int task = ws.me(); task < rtiles * ctiles * split; task += ws.nw) {
    const int sl = task / (rtiles * ctiles), rc = task % (rtiles * ctiles);
    const int r0 = (rc % rtiles) * RT + lr, c0 = (rc / rtiles) * CT + lc;
    const int kb = sl * per * 4, ke = min(Kp, (sl + 1) * per * 4);
    T acc[TR][TC];
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j) acc[i][j] = T(0);
    for (int k = kb; k < ke; k += 4) {
      T x[TR][4], w[TC][4];
#pragma unroll
      for (int i = 0; i < TR; ++i)
        Ld<T>::s4(xs + (uint32_t)(((r0 + i * LR) * ldx + k) * sizeof(T)), x[i]);
#pragma unroll
      for (int j = 0; j < TC; ++j) wo.ld4((long long)(c0 + j * LC) * ldw + k, w[j]);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) acc[i][j] = Num<T>::fma(x[i][q], w[j][q], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j) {
        const int n = c0 + j * LC;
        if (n < N) epi(r0 + i * LR, n, acc[i][j], sl);
      }
  }
}

// O[r][k] = sum_{n<Np} D[r][n] * W[n][k]; epi(r, k, acc) for k < K.  Thread
// columns here are contiguous (k = c0 + TC*lc + j) so W rows load as vectors.
template <typename T, int TR, int LR, bool WS, class Epi>
OB_DEV void gemm_nn(const T* D, int ldd, int Rt, const T* W, int ldw, int Np, int K, Warps ws,
                    Epi epi, int split = 1, T* ring = nullptr, int ring_elems = 0) {
  constexpr int TC = 4, LC = 32 / LR, RT = TR * LR, CT = TC * LC;
  if (!ws.mine()) return;
  const int lr = lane_id() % LR, lc = lane_id() / LR;
  const int rtiles = Rt / RT, ctiles = (K + CT - 1) / CT;
  const int nq = Np / 4, per = (nq + split - 1) / split;
  const uint32_t ds = smem_addr(D);
  const WOp<T, WS> wo(W);
  if constexpr (!WS) {
    // ring slot: 4 weight rows x the task's CT columns (row-major [4][CT])
    constexpr int kD = RingDepth<T>::value, kV = 16 / (int)sizeof(T), kCh = CT / kV;
    constexpr int kSlot = 4 * CT;
    if (ring && ring_elems / n_warps() >= kD * kSlot) {
      T* wr = ring + (long long)warp_id() * (ring_elems / n_warps());
      const int lane = lane_id();
      for (int task = ws.me(); task < rtiles * ctiles * split; task += ws.nw) {
        const int sl = task / (rtiles * ctiles), rc = task % (rtiles * ctiles);
        const int r0 = (rc % rtiles) * RT + lr, cb = (rc / rtiles) * CT, k0 = cb + TC * lc;
        const int nb = sl * per * 4, ne = min(Np, (sl + 1) * per * 4);
        auto issue = [&](int nn_, int slot) {
          if (nn_ < ne)
            for (int c = lane; c < 4 * kCh; c += 32) {
              const int q = c / kCh, hh = c % kCh;
              ring_cp16(wr + slot * kSlot + q * CT + hh * kV, W + (long long)(nn_ + q) * ldw + cb + hh * kV);
            }
          ring_commit();
        };
        __syncwarp();
#pragma unroll
        for (int dd = 0; dd < kD - 1; ++dd) issue(nb + 4 * dd, dd);
        T acc[TR][TC];
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) acc[i][j] = T(0);
        int slot = 0;
        for (int n = nb; n < ne; n += 4) {
          __syncwarp();
          issue(n + 4 * (kD - 1), (slot + kD - 1) % kD);
          ring_wait<kD - 1>();
          __syncwarp();
          T d[TR][4], w[4][4];
#pragma unroll
          for (int q = 0; q < 4; ++q) Ld<T>::s4(smem_addr(wr + slot * kSlot + q * CT + TC * lc), w[q]);
#pragma unroll
          for (int i = 0; i < TR; ++i)
            Ld<T>::s4(ds + (uint32_t)(((r0 + i * LR) * ldd + n) * sizeof(T)), d[i]);
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int i = 0; i < TR; ++i)
#pragma unroll
              for (int j = 0; j < TC; ++j) acc[i][j] = Num<T>::fma(d[i][q], w[q][j], acc[i][j]);
          slot = slot + 1 == kD ? 0 : slot + 1;
        }
        ring_wait<0>();
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j)
            if (k0 + j < K) epi(r0 + i * LR, k0 + j, acc[i][j], sl);
      }
      return;
    }
  }
  for (int task = ws.me(); task < rtiles * ctiles * split; task += ws.nw) {
    const int sl = task / (rtiles * ctiles), rc = task % (rtiles * ctiles);
    const int r0 = (rc % rtiles) * RT + lr, k0 = (rc / rtiles) * CT + TC * lc;
    const int nb = sl * per * 4, ne = min(Np, (sl + 1) * per * 4);
    T acc[TR][TC];
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j) acc[i][j] = T(0);
    for (int n = nb; n < ne; n += 4) {
      T d[TR][4], w[4][4];
#pragma unroll
      for (int i = 0; i < TR; ++i)
        Ld<T>::s4(ds + (uint32_t)(((r0 + i * LR) * ldd + n) * sizeof(T)), d[i]);
#pragma unroll
      for (int q = 0; q < 4; ++q) wo.ld4((long long)(n + q) * ldw + k0, w[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < TR; ++i)
#pragma unroll
          for (int j = 0; j < TC; ++j) acc[i][j] = Num<T>::fma(d[i][q], w[q][j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TC; ++j)
        if (k0 + j < K) epi(r0 + i * LR, k0 + j, acc[i][j], sl);
  }
}

// M[n][k] += scale * sum_{r<R} D[r][n] X[r][k]   (n < N, k < K; M row stride ldm,
// a multiple of 4) and mb[n] += scale * sum_r D[r][n].  Each thread owns a 4x4
// block of M held in registers for the R-loop, then one vector read-modify-write.
// The slot is private to the CTA, so plain RMW is race-free and deterministic.
template <typename T>
OB_DEV void gemm_tn_accum(const T* D, int ldd, const T* X, int ldx, int R, int N, int K, T scale,
                          T* __restrict__ M, int ldm, T* __restrict__ mb, Warps ws,
                          int bias_rows = -1) {
  if (bias_rows < 0) bias_rows = R;   // rows contributing to the bias (CNF: forward rows only)
  if (!ws.mine()) return;
  const int tid = ws.me() * 32 + lane_id(), nth = ws.nw * 32;
  const int nq = (N + 3) / 4, kq = (K + 3) / 4;
  const int items = nq * kq;
  const uint32_t ds = smem_addr(D), xs = smem_addr(X);
  for (int it = tid; it < items; it += nth) {
    const int n0 = (it / kq) * 4, k0 = (it % kq) * 4;
    // fp32: the slot's current values are fetched first so their L2 latency
    // overlaps the R-loop; fp64 reads them after (register budget)
    constexpr bool kPre = sizeof(T) == 4;
    T cur[4][4];
    if (kPre) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (n0 + i < N) Vec4<T>::ld(M + (long long)(n0 + i) * ldm + k0, cur[i]);
    }
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    for (int r = 0; r < R; ++r) {
      T d[4], x[4];
      Ld<T>::s4(ds + (uint32_t)((r * ldd + n0) * sizeof(T)), d);
      Ld<T>::s4(xs + (uint32_t)((r * ldx + k0) * sizeof(T)), x);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = Num<T>::fma(d[i], x[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (n0 + i < N) {
        if (!kPre) Vec4<T>::ld(M + (long long)(n0 + i) * ldm + k0, cur[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) cur[i][j] = Num<T>::add(cur[i][j], Num<T>::mul(scale, acc[i][j]));
        Vec4<T>::st(M + (long long)(n0 + i) * ldm + k0, cur[i]);
      }
    }
  }
  for (int n = tid; n < N; n += nth) {
    T s = T(0);
    for (int r = 0; r < bias_rows; ++r) s = Num<T>::add(s, D[r * ldd + n]);
    mb[n] = Num<T>::add(mb[n], Num<T>::mul(scale, s));
  }
}

}  // namespace ob
