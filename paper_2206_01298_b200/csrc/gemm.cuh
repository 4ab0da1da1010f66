// gemm.cuh -- register-tiled CTA GEMMs for the persistent sample-tile kernels.
//
// A CTA holds R (<= a few dozen) samples; its contractions are small GEMMs with
// the sample rows on one side and a weight matrix (shared memory when it fits,
// else L1/L2-resident global) on the other.  Every thread owns a 4 x 4 output
// block (16 FMAs per 8 vector loads); a warp's 32 lanes are arranged LR x LC
// (LR*LC = 32) so one warp covers a (4*LR) x (4*LC) tile.  Row r of a thread
// block is r0 + lr + LR*i and column n is c0 + lc + LC*j (strided), which makes
// every 16-byte shared-memory access conflict-free when leading dimensions are
// "odd quads" (ld/4 odd, see ld_quad_odd).
//
// Operands are row-major with the contraction dimension contiguous:
//   gemm_nt : Z[r][n] = sum_k X[r][k] W[n][k]        (forward / JVP, z = W x)
//   gemm_nn : O[r][k] = sum_n D[r][n] W[n][k]        (VJP input product d W)
//   gemm_tn : M[n][k] += s * sum_r D[r][n] X[r][k]   (parameter cotangent)
// Padding contract: X/D rows up to the row tile, columns up to the next 4 (and
// W rows / columns up to the tile the op reads) exist and are finite; weight
// padding is zero, so padded lanes contribute exact zeros.
#pragma once

#include "tile.cuh"

namespace ob {

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

// Z[r][n] = sum_{k<Kp} X[r][k] * W[n][k];  epi(r, n, acc) for r < Rv... (caller
// guards), n < N.  Rt = rows to compute (multiple of 4*LR).
template <typename T, int LR, class Epi>
OB_DEV void gemm_nt(const T* __restrict__ X, int ldx, int Rt, const T* __restrict__ W, int ldw,
                    int N, int Kp, Epi epi) {
  constexpr int LC = 32 / LR, RT = 4 * LR, CT = 4 * LC;
  const int lr = lane_id() % LR, lc = lane_id() / LR;
  const int rtiles = Rt / RT, ctiles = (N + CT - 1) / CT;
  for (int task = warp_id(); task < rtiles * ctiles; task += n_warps()) {
    const int r0 = (task % rtiles) * RT + lr, c0 = (task / rtiles) * CT + lc;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    const T* xp = X + r0 * ldx;
    const T* wp = W + c0 * ldw;
    for (int k = 0; k < Kp; k += 4) {
      T x[4][4], w[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) Vec4<T>::ld(xp + i * LR * ldx + k, x[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) Vec4<T>::ld(wp + j * LC * ldw + k, w[j]);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = Num<T>::fma(x[i][q], w[j][q], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = c0 + j * LC;
        if (n < N) epi(r0 + i * LR, n, acc[i][j]);
      }
  }
}

// O[r][k] = sum_{n<Np} D[r][n] * W[n][k]; epi(r, k, acc) for k < K.  Thread
// columns here are contiguous (k = c0 + 4*lc + j) so W rows load as one vector.
template <typename T, int LR, class Epi>
OB_DEV void gemm_nn(const T* __restrict__ D, int ldd, int Rt, const T* __restrict__ W, int ldw,
                    int Np, int K, Epi epi) {
  constexpr int LC = 32 / LR, RT = 4 * LR, CT = 4 * LC;
  const int lr = lane_id() % LR, lc = lane_id() / LR;
  const int rtiles = Rt / RT, ctiles = (K + CT - 1) / CT;
  for (int task = warp_id(); task < rtiles * ctiles; task += n_warps()) {
    const int r0 = (task % rtiles) * RT + lr, k0 = (task / rtiles) * CT + 4 * lc;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    const T* dp = D + r0 * ldd;
    const T* wp = W + k0;
    for (int n = 0; n < Np; n += 4) {
      T d[4][4], w[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) Vec4<T>::ld(dp + i * LR * ldd + n, d[i]);
#pragma unroll
      for (int q = 0; q < 4; ++q) Vec4<T>::ld(wp + (n + q) * ldw, w[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = Num<T>::fma(d[i][q], w[q][j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (k0 + j < K) epi(r0 + i * LR, k0 + j, acc[i][j]);
  }
}

// M[n][k] += scale * sum_{r<R} D[r][n] X[r][k]   (n < N, k < K; M row stride ldm,
// a multiple of 4) and mb[n] += scale * sum_r D[r][n].  Each thread owns a 4x4
// block of M held in registers for the R-loop, then one vector read-modify-write.
// The slot is private to the CTA, so plain RMW is race-free and deterministic.
template <typename T>
OB_DEV void gemm_tn_accum(const T* __restrict__ D, int ldd, const T* __restrict__ X, int ldx,
                          int R, int N, int K, T scale, T* __restrict__ M, int ldm,
                          T* __restrict__ mb) {
  const int nq = (N + 3) / 4, kq = (K + 3) / 4;
  const int items = nq * kq;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int n0 = (it / kq) * 4, k0 = (it % kq) * 4;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
    for (int r = 0; r < R; ++r) {
      T d[4], x[4];
      Vec4<T>::ld(D + r * ldd + n0, d);
      Vec4<T>::ld(X + r * ldx + k0, x);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = Num<T>::fma(d[i], x[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (n0 + i < N) {
        T* m = M + (long long)(n0 + i) * ldm + k0;
        T cur[4];
        Vec4<T>::ld(m, cur);
#pragma unroll
        for (int j = 0; j < 4; ++j) cur[j] = Num<T>::add(cur[j], Num<T>::mul(scale, acc[i][j]));
        Vec4<T>::st(m, cur);
      }
    }
  }
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    T s = T(0);
    for (int r = 0; r < R; ++r) s = Num<T>::add(s, D[r * ldd + n]);
    mb[n] = Num<T>::add(mb[n], Num<T>::mul(scale, s));
  }
}

}  // namespace ob
