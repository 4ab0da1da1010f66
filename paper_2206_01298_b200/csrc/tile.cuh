// tile.cuh -- CTA-level building blocks of the persistent ODE-block kernels.
//
// One CTA owns a fixed tile of R samples (rows) for a whole forward or reverse
// sweep: samples are independent given theta (nn.py:26-35 holds one sample per
// call), so the only cross-CTA data is the parameter cotangent,
// which every CTA accumulates into its own partial slot and a fixed-order
// reduction sums at the end (deterministic, no atomics).
//
// Activations live in shared memory as row-major [Rp][wp] tiles (wp = width
// padded to a multiple of 4 so 16-byte vector loads stay aligned; Rp = R padded
// to the row-block RB).  Padding is zero-filled once at kernel start and never
// written, so padded lanes contribute exact zeros.
//
// The MLP arithmetic follows kernels.py:122-225: z = W a + b (dot first, then
// bias), activation on hidden layers, linear output; VJP d *= act'(pre),
// dW += d x^T, db += d, d <- W^T d; JVP s <- act'(pre) * (W s).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/odeblock.h"

#define OB_DEV __device__ __forceinline__

namespace ob {

constexpr int kThreads = 512;

// ---------------------------------------------------------------- numerics
template <typename T> struct Num;
template <> struct Num<float> {
  static OB_DEV float mul(float a, float b) { return __fmul_rn(a, b); }
  static OB_DEV float add(float a, float b) { return __fadd_rn(a, b); }
  static OB_DEV float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
  static OB_DEV bool finite(float x) { return isfinite(x); }
};
template <> struct Num<double> {
  static OB_DEV double mul(double a, double b) { return __dmul_rn(a, b); }
  static OB_DEV double add(double a, double b) { return __dadd_rn(a, b); }
  static OB_DEV double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
  static OB_DEV bool finite(double x) { return isfinite(x); }
};

OB_DEV void load4(const float* p, float v[4]) {
  float4 q = *reinterpret_cast<const float4*>(p);
  v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
}
OB_DEV void load4(const double* p, double v[4]) {
  double2 a = *reinterpret_cast<const double2*>(p);
  double2 b = *reinterpret_cast<const double2*>(p + 2);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// activations: kernels.py:45-77 (+ softplus for the CNF config)
template <typename T> OB_DEV T act_fn(T x, int id) {
  switch (id) {
    case OB_ACT_IDENTITY: return x;
    case OB_ACT_RELU: return x > T(0) ? x : T(0);
    case OB_ACT_TANH: return tanh(x);
    case OB_ACT_GELU: return T(0.5) * x * (T(1) + erf(x * T(0.70710678118654752440)));
    default: {  // softplus, overflow-safe: max(x,0) + log1p(exp(-|x|))
      T ax = x < T(0) ? -x : x;
      return (x > T(0) ? x : T(0)) + log1p(exp(-ax));
    }
  }
}
template <typename T> OB_DEV T act_prime(T x, int id) {
  switch (id) {
    case OB_ACT_IDENTITY: return T(1);
    case OB_ACT_RELU: return x > T(0) ? T(1) : T(0);  // ReLU'(0) = 0 (kernels.py:68-70)
    case OB_ACT_TANH: { T t = tanh(x); return T(1) - t * t; }
    case OB_ACT_GELU:
      return T(0.5) * (T(1) + erf(x * T(0.70710678118654752440))) +
             x * T(0.39894228040143267794) * exp(T(-0.5) * x * x);
    default: return T(1) / (T(1) + exp(-x));  // softplus' = sigmoid
  }
}
template <typename T> OB_DEV T act_second(T x, int id) {
  switch (id) {
    case OB_ACT_TANH: { T t = tanh(x); return T(-2) * t * (T(1) - t * t); }
    case OB_ACT_SOFTPLUS: { T s = T(1) / (T(1) + exp(-x)); return s * (T(1) - s); }
    case OB_ACT_GELU: return T(0.39894228040143267794) * exp(T(-0.5) * x * x) * (T(2) - x * x);
    default: return T(0);
  }
}

OB_DEV int pad4(int n) { return (n + 3) & ~3; }

// ---------------------------------------------------------------- params
struct Dims {
  int L;                        // affine layers
  int w[OB_MAX_LAYERS + 1];     // widths
  int wp[OB_MAX_LAYERS + 1];    // widths padded to 4
  int N, Np;                    // state dim, padded
  int act, time_input;
  long long woff[OB_MAX_LAYERS], boff[OB_MAX_LAYERS];  // W / b offsets in theta
  int maxwp;
};

template <typename T>
struct Weights {
  const T* wt[OB_MAX_LAYERS];    // [wp_l][w_{l+1}]  W^T, zero rows for k >= w_l
  const T* wn[OB_MAX_LAYERS];    // [wp_{l+1}][w_l]  W,   zero rows for n >= w_{l+1}
  const T* bias[OB_MAX_LAYERS];  // [w_{l+1}] (into theta)
};

// shared-memory tile of one MLP evaluation
template <typename T>
struct MlpSmem {
  T* x0;                        // [Rp][wp0] layer-0 input (state | time)
  T* pre[OB_MAX_LAYERS];        // [Rp][wp_{l+1}] pre-activations (last = output)
  T* hid[OB_MAX_LAYERS];        // [Rp][wp_{l+1}] act(pre) for hidden layers
  T* dA;                        // [Rp][maxwp] cotangent / tangent ping-pong
  T* dB;
};

// ------------------------------------------------------------ affine ops
// Z[r][n] = sum_k X[r][k] * WT[k][n] (+ bias[n]);  rows r < Rp, n < N.
// Each thread owns RB rows x 1 column; k advances 4 at a time (X vector loads
// from smem, W^T coalesced across the warp from L1/L2).
template <typename T, int RB>
OB_DEV void affine_fwd(const T* __restrict__ X, int ldx, int Rp, int Kp,
                       const T* __restrict__ WT, const T* __restrict__ bias, int N,
                       T* __restrict__ Z, int ldz, T* __restrict__ A, int act) {
  const int nrb = Rp / RB;
  for (int item = threadIdx.x; item < nrb * N; item += blockDim.x) {
    const int n = item % N;
    const int r0 = (item / N) * RB;
    T acc[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) acc[j] = T(0);
    const T* xr = X + r0 * ldx;
    for (int k = 0; k < Kp; k += 4) {
      const T w0 = __ldg(WT + (k + 0) * N + n);
      const T w1 = __ldg(WT + (k + 1) * N + n);
      const T w2 = __ldg(WT + (k + 2) * N + n);
      const T w3 = __ldg(WT + (k + 3) * N + n);
#pragma unroll
      for (int j = 0; j < RB; ++j) {
        T x[4];
        load4(xr + j * ldx + k, x);
        acc[j] = Num<T>::fma(x[0], w0, acc[j]);
        acc[j] = Num<T>::fma(x[1], w1, acc[j]);
        acc[j] = Num<T>::fma(x[2], w2, acc[j]);
        acc[j] = Num<T>::fma(x[3], w3, acc[j]);
      }
    }
    const T b = bias ? __ldg(bias + n) : T(0);
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const T z = bias ? Num<T>::add(acc[j], b) : acc[j];
      Z[(r0 + j) * ldz + n] = z;
      if (A) A[(r0 + j) * ldz + n] = act_fn(z, act);
    }
  }
}

// Out[r][k] = sum_n D[r][n] * WN[n][k] for k < K  (input-side VJP product, d <- W^T d
// written as the row-vector product np.dot(d, w) of kernels.py:182).
template <typename T, int RB>
OB_DEV void affine_bwd(const T* __restrict__ D, int ldd, int Rp, int Np,
                       const T* __restrict__ WN, int Kfull, int K,
                       T* __restrict__ Out, int ldo) {
  const int nrb = Rp / RB;
  for (int item = threadIdx.x; item < nrb * K; item += blockDim.x) {
    const int k = item % K;
    const int r0 = (item / K) * RB;
    T acc[RB];
#pragma unroll
    for (int j = 0; j < RB; ++j) acc[j] = T(0);
    const T* dr = D + r0 * ldd;
    for (int n = 0; n < Np; n += 4) {
      const T w0 = __ldg(WN + (n + 0) * Kfull + k);
      const T w1 = __ldg(WN + (n + 1) * Kfull + k);
      const T w2 = __ldg(WN + (n + 2) * Kfull + k);
      const T w3 = __ldg(WN + (n + 3) * Kfull + k);
#pragma unroll
      for (int j = 0; j < RB; ++j) {
        T d[4];
        load4(dr + j * ldd + n, d);
        acc[j] = Num<T>::fma(d[0], w0, acc[j]);
        acc[j] = Num<T>::fma(d[1], w1, acc[j]);
        acc[j] = Num<T>::fma(d[2], w2, acc[j]);
        acc[j] = Num<T>::fma(d[3], w3, acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < RB; ++j) Out[(r0 + j) * ldo + k] = acc[j];
  }
}

// Parameter cotangent of one layer, summed over the tile's rows and scaled:
//   muW[n][k] += scale * sum_r D[r][n] X[r][k];   mub[n] += scale * sum_r D[r][n]
// (dW = outer(d, x), db = d per sample, kernels.py:177-179; mu += h*ptv,
// adjoint.py:91).  muW is this CTA's private slot -> plain read-modify-write.
template <typename T>
OB_DEV void accum_dparam(const T* __restrict__ D, int ldd, const T* __restrict__ X, int ldx,
                         int R, int N, int K, T scale, T* __restrict__ muW,
                         T* __restrict__ mub) {
  const int kq = (K + 3) / 4;
  const int items = N * kq;
  for (int item = threadIdx.x; item < items + N; item += blockDim.x) {
    if (item < items) {
      const int n = item / kq;
      const int k0 = (item % kq) * 4;
      T s[4] = {T(0), T(0), T(0), T(0)};
      for (int r = 0; r < R; ++r) {
        const T d = D[r * ldd + n];
        T x[4];
        load4(X + r * ldx + k0, x);
#pragma unroll
        for (int q = 0; q < 4; ++q) s[q] = Num<T>::fma(d, x[q], s[q]);
      }
      T* dst = muW + (long long)n * K + k0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (k0 + q < K) dst[q] = Num<T>::add(dst[q], Num<T>::mul(scale, s[q]));
    } else {
      const int n = item - items;
      T s = T(0);
      for (int r = 0; r < R; ++r) s = Num<T>::add(s, D[r * ldd + n]);
      mub[n] = Num<T>::add(mub[n], Num<T>::mul(scale, s));
    }
  }
}

// ------------------------------------------------------------- MLP tile
template <typename T, int RB>
struct MlpTile {
  const Dims& d;
  const Weights<T>& W;
  MlpSmem<T>& s;
  int Rp;

  OB_DEV MlpTile(const Dims& d_, const Weights<T>& W_, MlpSmem<T>& s_, int Rp_)
      : d(d_), W(W_), s(s_), Rp(Rp_) {}

  OB_DEV const T* in(int l) const { return l == 0 ? s.x0 : s.hid[l - 1]; }

  // x0 must be filled; output lands in s.pre[L-1] ([Rp][wp_L]).
  OB_DEV void forward() {
    for (int l = 0; l < d.L; ++l) {
      affine_fwd<T, RB>(in(l), d.wp[l], Rp, d.wp[l], W.wt[l], W.bias[l], d.w[l + 1],
                        s.pre[l], d.wp[l + 1], l < d.L - 1 ? s.hid[l] : nullptr, d.act);
      __syncthreads();
    }
  }

  // Reverse pass through the cached forward.  v: [Rp][ld_v] cotangent on the
  // output (not modified).  jtv (may be null): [Rp][ld_o] receives the state
  // part (k < N) of the input cotangent.  mu (may be null): this CTA's
  // parameter-cotangent slot; receives scale * sum_rows (df/dtheta)^T v.
  OB_DEV void vjp(const T* v, int ld_v, int R, T* jtv, int ld_o, T* mu, T scale) {
    T* cur = s.dA;
    T* nxt = s.dB;
    const int L = d.L;
    // copy the output cotangent into the ping-pong buffer
    for (int i = threadIdx.x; i < Rp * d.wp[L]; i += blockDim.x) {
      const int r = i / d.wp[L], n = i % d.wp[L];
      cur[r * d.maxwp + n] = v[r * ld_v + n];
    }
    __syncthreads();
    for (int l = L - 1; l >= 0; --l) {
      const int nout = d.w[l + 1];
      if (l < L - 1) {
        for (int i = threadIdx.x; i < Rp * nout; i += blockDim.x) {
          const int r = i / nout, n = i % nout;
          cur[r * d.maxwp + n] *= act_prime(s.pre[l][r * d.wp[l + 1] + n], d.act);
        }
        __syncthreads();
      }
      if (mu) accum_dparam<T>(cur, d.maxwp, in(l), d.wp[l], R, nout, d.w[l], scale,
                              mu + d.woff[l], mu + d.boff[l]);
      if (l > 0) {
        affine_bwd<T, RB>(cur, d.maxwp, Rp, d.wp[l + 1], W.wn[l], d.w[l], d.w[l], nxt, d.maxwp);
      } else if (jtv) {
        affine_bwd<T, RB>(cur, d.maxwp, Rp, d.wp[1], W.wn[0], d.w[0], d.N, jtv, ld_o);
      }
      __syncthreads();
      T* tmp = cur; cur = nxt; nxt = tmp;
    }
  }

  // Tangent pass through the cached linearisation (time tangent held at 0,
  // nn.py:177-180).  w: [Rp][ld_w] state tangent; out: [Rp][ld_o].
  OB_DEV void jvp(const T* w, int ld_w, T* out, int ld_o) {
    T* cur = s.dA;
    T* nxt = s.dB;
    for (int i = threadIdx.x; i < Rp * d.wp[0]; i += blockDim.x) {
      const int r = i / d.wp[0], k = i % d.wp[0];
      cur[r * d.maxwp + k] = k < d.N ? w[r * ld_w + k] : T(0);
    }
    __syncthreads();
    for (int l = 0; l < d.L; ++l) {
      const int nout = d.w[l + 1];
      T* dst = (l == d.L - 1) ? out : nxt;
      const int ldd = (l == d.L - 1) ? ld_o : d.maxwp;
      affine_fwd<T, RB>(cur, d.maxwp, Rp, d.wp[l], W.wt[l], nullptr, nout, dst, ldd, nullptr, 0);
      __syncthreads();
      if (l < d.L - 1) {
        for (int i = threadIdx.x; i < Rp * nout; i += blockDim.x) {
          const int r = i / nout, n = i % nout;
          nxt[r * d.maxwp + n] *= act_prime(s.pre[l][r * d.wp[l + 1] + n], d.act);
        }
        __syncthreads();
        T* tmp = cur; cur = nxt; nxt = tmp;
      }
    }
  }
};

}  // namespace ob
