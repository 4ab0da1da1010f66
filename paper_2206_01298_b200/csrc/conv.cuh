// conv.cuh -- 3x3 (padding 1) convolution GEMMs on one sample's 16x16 NHWC
// image held in shared memory with a one-pixel zero halo (18x18 pixels x CP
// channels, CP = 68 = an "odd quad" so 16-byte accesses of 8 consecutive pixels
// hit distinct banks).  Implicit GEMM: rows are the 256 pixels, the reduction
// runs over the 9 stencil taps x channels.  Thread tiles are 4 pixels x 4
// channels (pixels x + 8i, channels strided/contiguous as in gemm.cuh), so a
// warp covers 32 pixels x 16 channels.
//   conv_fwd  : out[p][co] = sum_{s,ci} X[p + off(s)][ci] Wf[co][s][ci]
//   conv_bwd  : out[p][ci] = sum_{s,co} D[p - off(s)][co] Wb[s][co][ci]   (transposed)
//   conv_wgrad: M[co][s][ci] += scale * sum_p D[p][co] X[p + off(s)][ci]; mb[co] += ...
// Weights stay in global memory (L1/L2 resident, 0.3 MB per conv pair).
#pragma once

#include "tile.cuh"   // (tile.cuh pulls gemm.cuh in at the right point)

namespace ob {

constexpr int kImg = 16;          // image side
constexpr int kHalo = 18;         // with the zero border
constexpr int kCP = 68;           // padded channel stride in shared memory
constexpr int kPix = kImg * kImg;

OB_DEV int halo_idx(int p, int dy, int dx) {   // pixel p shifted by (dy, dx) in [0, 2]
  return ((p / kImg) + dy) * kHalo + (p % kImg) + dx;
}

// ---- tap-staged variants: one tap's 64 weight rows (64 x kCP, 17 KB) are copied to
// shared memory with cp.async while the previous tap is consumed (double buffer), so
// the inner loops read weights with ld.shared instead of waiting on L2.  The warps of
// `ws` synchronise with a named barrier (ws may be half the CTA).
OB_DEV void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
OB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> OB_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
OB_DEV void warps_sync(const Warps& ws) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + (ws.w0 != 0 ? 1 : 0)), "r"(ws.nw * 32) : "memory");
}
template <typename T>
OB_DEV void stage_tap(T* dst, const T* src, long long rowstride, const Warps& ws) {
  constexpr int kV = 16 / sizeof(T), kChunks = kCP / kV;
  const int tid = ws.me() * 32 + lane_id(), nth = ws.nw * 32;
  for (int c = tid; c < 64 * kChunks; c += nth) {
    const int r = c / kChunks, q = c % kChunks;
    cp_async16(dst + r * kCP + q * kV, src + r * rowstride + q * kV);
  }
  cp_async_commit();
}

// out[p][co] = epi(sum_{s, k < K} X[p + off(s)][k] * Wt_s[co][k]) with Wt_s the staged tap
// rows (tap s at src + s * tapstride, row co at + co * rowstride).  bwd: D read at the
// flipped tap (transposed conv), thread columns contiguous (k0 + j) as in conv_bwd.
template <typename T, bool kBwd, class Epi>
OB_DEV void conv_staged(const T* Xh, const T* W, long long rowstride, long long tapstride, int Cout,
                        int K, Warps ws, T* stage, Epi epi) {
  constexpr int LR = 8, LC = 4, kMaxT = 2;
  if (!ws.mine()) return;
  const int lr = lane_id() % LR, lc = lane_id() / LR;
  const int ctiles = (Cout + 15) / 16, ntask = (kPix / 32) * ctiles;
  const int per = (ntask + ws.nw - 1) / ws.nw, groups = (per + kMaxT - 1) / kMaxT;
  const uint32_t xs = smem_addr(Xh);
  for (int g = 0; g < groups; ++g) {
    T acc[kMaxT][4][4];
#pragma unroll
    for (int t = 0; t < kMaxT; ++t)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[t][i][j] = T(0);
    stage_tap(stage, W, rowstride, ws);
    for (int s = 0; s < 9; ++s) {
      if (s + 1 < 9) {
        stage_tap(stage + ((s + 1) & 1) * 64 * kCP, W + (s + 1) * tapstride, rowstride, ws);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      warps_sync(ws);
      const uint32_t wsm = smem_addr(stage + (s & 1) * 64 * kCP);
      const int dy = kBwd ? 2 - s / 3 : s / 3, dx = kBwd ? 2 - s % 3 : s % 3;
#pragma unroll
      for (int t = 0; t < kMaxT; ++t) {
        const int task = ws.me() + (g * kMaxT + t) * ws.nw;
        if (task >= ntask) continue;
        const int p0 = (task % (kPix / 32)) * 32 + lr;
        const int c0 = kBwd ? (task / (kPix / 32)) * 16 + 4 * lc : (task / (kPix / 32)) * 16 + lc;
        int hx[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) hx[i] = halo_idx(p0 + i * LR, dy, dx) * kCP;
        for (int k = 0; k < K; k += 4) {
          T x[4][4], w[4][4];
#pragma unroll
          for (int i = 0; i < 4; ++i) Ld<T>::s4(xs + (uint32_t)((hx[i] + k) * sizeof(T)), x[i]);
          if constexpr (kBwd) {   // w[q][j] = Wt[k + q][c0 + j]
#pragma unroll
            for (int q = 0; q < 4; ++q) Ld<T>::s4(wsm + (uint32_t)(((k + q) * kCP + c0) * sizeof(T)), w[q]);
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[t][i][j] = Num<T>::fma(x[i][q], w[q][j], acc[t][i][j]);
          } else {                // w[j][q] = Wt[c0 + j LC][k + q]
#pragma unroll
            for (int j = 0; j < 4; ++j) Ld<T>::s4(wsm + (uint32_t)(((c0 + j * LC) * kCP + k) * sizeof(T)), w[j]);
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[t][i][j] = Num<T>::fma(x[i][q], w[j][q], acc[t][i][j]);
          }
        }
      }
      warps_sync(ws);   // every warp is done with this buffer before it is refilled
    }
#pragma unroll
    for (int t = 0; t < kMaxT; ++t) {
      const int task = ws.me() + (g * kMaxT + t) * ws.nw;
      if (task >= ntask) continue;
      const int p0 = (task % (kPix / 32)) * 32 + lr;
      const int c0 = kBwd ? (task / (kPix / 32)) * 16 + 4 * lc : (task / (kPix / 32)) * 16 + lc;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = kBwd ? c0 + j : c0 + j * LC;
          if (c < Cout) epi(p0 + i * LR, c, acc[t][i][j]);
        }
    }
  }
}

// out[p][co] (co < Cout) = sum over taps and ci < Kc of X[...] * Wf[co][s*kCP + ci]
template <typename T, class Epi>
OB_DEV void conv_fwd(const T* Xh, const T* Wf, int Cout, int Kc, Warps ws, Epi epi) {
  constexpr int LR = 8, LC = 4;
  if (!ws.mine()) return;
  const int lr = lane_id() % LR, lc = lane_id() / LR;
  const int ctiles = (Cout + 15) / 16;
  const uint32_t xs = smem_addr(Xh);
  const int ldw = 9 * kCP;
  for (int task = ws.me(); task < (kPix / 32) * ctiles; task += ws.nw) {
    const int p0 = (task % (kPix / 32)) * 32 + lr, c0 = (task / (kPix / 32)) * 16 + lc;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    for (int s = 0; s < 9; ++s) {
      const int dy = s / 3, dx = s % 3;
      int hx[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) hx[i] = halo_idx(p0 + i * LR, dy, dx) * kCP;
      const T* wrow = Wf + s * kCP;
      for (int ci = 0; ci < Kc; ci += 4) {
        T x[4][4], w[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) Ld<T>::s4(xs + (uint32_t)((hx[i] + ci) * sizeof(T)), x[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) Ld<T>::g4(wrow + (long long)(c0 + j * LC) * ldw + ci, w[j]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = Num<T>::fma(x[i][q], w[j][q], acc[i][j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (c0 + j * LC < Cout) epi(p0 + i * LR, c0 + j * LC, acc[i][j]);
  }
}

// transposed conv: out[p][ci] (ci < Cout) = sum_{s, co < 64} D[p - off(s)][co] * Wb[(s*64+co)][ci]
template <typename T, class Epi>
OB_DEV void conv_bwd(const T* Dh, const T* Wb, int ldw, int Cout, Warps ws, Epi epi) {
  constexpr int LR = 8, LC = 4;
  if (!ws.mine()) return;
  const int lr = lane_id() % LR, lc = lane_id() / LR;
  const int ctiles = (Cout + 15) / 16;
  const uint32_t ds = smem_addr(Dh);
  for (int task = ws.me(); task < (kPix / 32) * ctiles; task += ws.nw) {
    const int p0 = (task % (kPix / 32)) * 32 + lr, k0 = (task / (kPix / 32)) * 16 + 4 * lc;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    for (int s = 0; s < 9; ++s) {
      const int dy = 2 - s / 3, dx = 2 - s % 3;
      int hx[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) hx[i] = halo_idx(p0 + i * LR, dy, dx) * kCP;
      const T* wb = Wb + (long long)s * 64 * ldw + k0;
      for (int co = 0; co < 64; co += 4) {
        T d[4][4], w[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) Ld<T>::s4(ds + (uint32_t)((hx[i] + co) * sizeof(T)), d[i]);
#pragma unroll
        for (int q = 0; q < 4; ++q) Ld<T>::g4(wb + (long long)(co + q) * ldw, w[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = Num<T>::fma(d[i][q], w[q][j], acc[i][j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (k0 + j < Cout) epi(p0 + i * LR, k0 + j, acc[i][j]);
  }
}

// M[co][s*kCP + ci] += scale * sum_p D[p][co] X[p + off(s)][ci]  (ci < Kc, Kc % 4 == 0)
// mb[co] += scale * sum_p D[p][co].  D and X are halo buffers (D read at the centre).
template <typename T>
OB_DEV void conv_wgrad(const T* Dh, const T* Xh, int Kc, T scale, T* M, T* mb, Warps ws) {
  if (!ws.mine()) return;
  const int tid = ws.me() * 32 + lane_id(), nth = ws.nw * 32;
  const int kq = Kc / 4, items = 16 * 9 * kq;
  const uint32_t ds = smem_addr(Dh), xs = smem_addr(Xh);
  for (int it = tid; it < items; it += nth) {
    const int co0 = (it % 16) * 4, rest = it / 16, s = rest / kq, ci0 = (rest % kq) * 4;
    const int dy = s / 3, dx = s % 3;
    T cur[4][4];   // prefetch the slot (L2) so its latency overlaps the pixel loop
#pragma unroll
    for (int i = 0; i < 4; ++i) Vec4<T>::ld(M + (long long)(co0 + i) * (9 * kCP) + s * kCP + ci0, cur[i]);
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    for (int p = 0; p < kPix; ++p) {
      T d[4], x[4];
      Ld<T>::s4(ds + (uint32_t)((halo_idx(p, 1, 1) * kCP + co0) * sizeof(T)), d);
      Ld<T>::s4(xs + (uint32_t)((halo_idx(p, dy, dx) * kCP + ci0) * sizeof(T)), x);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = Num<T>::fma(d[i], x[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j) cur[i][j] = Num<T>::add(cur[i][j], Num<T>::mul(scale, acc[i][j]));
      Vec4<T>::st(M + (long long)(co0 + i) * (9 * kCP) + s * kCP + ci0, cur[i]);
    }
  }
  for (int co = tid; co < 64; co += nth) {
    T sacc = T(0);
    for (int p = 0; p < kPix; ++p) sacc = Num<T>::add(sacc, Dh[halo_idx(p, 1, 1) * kCP + co]);
    mb[co] = Num<T>::add(mb[co], Num<T>::mul(scale, sacc));
  }
}

}  // namespace ob
