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
// fp32 transcendentals go through the SFU's ex2/lg2 (one op each) with the reciprocal
// 1/(1 + e), e in (0, 1], refined by Newton steps on the FMA pipe: absolute error
// ~1e-7, far inside the fp32 parity bar and several times cheaper than the libm
// paths (exp2f / expf / log1pf / IEEE division); fp64 keeps libm (held to 1e-10).
OB_DEV float ex2_fast(float x) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x));
  return e;
}
OB_DEV float lg2_fast(float x) {
  float l;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(x));
  return l;
}
OB_DEV float recip_1p(float e) {   // 1 / (1 + e) for e in [0, 1]
  const float d = 1.0f + e;
  float r = fmaf(-0.5f, d, 1.4571068f);
  r = fmaf(r, fmaf(-d, r, 1.0f), r);
  r = fmaf(r, fmaf(-d, r, 1.0f), r);
  r = fmaf(r, fmaf(-d, r, 1.0f), r);
  return r;
}
OB_DEV float fast_tanh(float x) {
  const float e = ex2_fast(-2.8853900817779268f * fabsf(x));   // exp(-2|x|)
  return copysignf((1.0f - e) * recip_1p(e), x);
}
OB_DEV double fast_tanh(double x) { return tanh(x); }
OB_DEV float fast_sigmoid(float x) {       // 1 / (1 + exp(-x))
  const float e = ex2_fast(-1.4426950408889634f * fabsf(x));   // exp(-|x|)
  const float r = recip_1p(e);
  return x >= 0.0f ? r : e * r;
}
OB_DEV double fast_sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }
OB_DEV float fast_softplus(float x) {      // max(x, 0) + log1p(exp(-|x|))
  const float e = ex2_fast(-1.4426950408889634f * fabsf(x));
  return fmaxf(x, 0.0f) + 0.6931471805599453f * lg2_fast(1.0f + e);
}
OB_DEV double fast_softplus(double x) {
  const double ax = x < 0.0 ? -x : x;
  return (x > 0.0 ? x : 0.0) + log1p(exp(-ax));
}

template <typename T> OB_DEV T act_fn(T x, int id) {
  switch (id) {
    case OB_ACT_IDENTITY: return x;
    case OB_ACT_RELU: return x > T(0) ? x : T(0);
    case OB_ACT_TANH: return fast_tanh(x);
    case OB_ACT_GELU: return T(0.5) * x * (T(1) + erf(x * T(0.70710678118654752440)));
    default: return fast_softplus(x);   // overflow-safe form
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
    default: return fast_sigmoid(x);  // softplus' = sigmoid
  }
}
template <typename T> OB_DEV T act_second(T x, int id) {
  switch (id) {
    case OB_ACT_TANH: { T t = tanh(x); return T(-2) * t * (T(1) - t * t); }
    case OB_ACT_SOFTPLUS: { T s = fast_sigmoid(x); return s * (T(1) - s); }
    case OB_ACT_GELU: return T(0.39894228040143267794) * exp(T(-0.5) * x * x) * (T(2) - x * x);
    default: return T(0);
  }
}

OB_DEV int pad4(int n) { return (n + 3) & ~3; }

struct PhaseTimer {
  long long t0;
  unsigned long long* acc;
  __device__ __forceinline__ explicit PhaseTimer(unsigned long long* a) : t0(0), acc(a) {
#ifdef __CUDA_ARCH__
    if (acc) t0 = clock64();   // no clock read when profiling is off
#endif
  }
  __device__ __forceinline__ void mark(int ph) {   // call right after a __syncthreads
#ifdef __CUDA_ARCH__
    if (acc && threadIdx.x == 0) {
      const long long t = clock64();
      atomicAdd(&acc[ph], (unsigned long long)(t - t0));
      t0 = t;
    }
#endif
  }
};

// ---------------------------------------------------------------- params
// Host-computed geometry of one MLP (see capi.cu: make_dims / layout).
struct Dims {
  int L;                          // affine layers
  int w[OB_MAX_LAYERS + 1];       // widths
  int lda[OB_MAX_LAYERS + 1];     // leading dim of the activation buffer of width w[l]
  int ldw[OB_MAX_LAYERS];         // leading dim of packed W_l ([nrow_l][ldw_l])
  int nrow[OB_MAX_LAYERS];        // rows of packed W_l (w[l+1] rounded up to the col tile)
  long long woff[OB_MAX_LAYERS], boff[OB_MAX_LAYERS];    // W / b offsets in theta
  long long pwoff[OB_MAX_LAYERS];                        // packed W_l offsets (elements)
  long long mwoff[OB_MAX_LAYERS], mboff[OB_MAX_LAYERS];  // padded mu offsets
  int ldm[OB_MAX_LAYERS];         // padded mu row stride (w[l] rounded to 4)
  long long n_mu;                 // padded mu length
  long long n_packed;             // packed weights length
  int N, ldn;                     // state dim, its buffer leading dim
  int nin;                        // state components fed to the MLP (CNF: N - 1)
  int cnf;                        // 1: continuous normalizing flow field (C4)
  int conv;                       // 1: 3x3 conv block on a 16x16 NHWC image (C3)
  int conv_cin[OB_MAX_LAYERS];    // conv: input channels per stencil tap in theta
  int act, time_input;
  int need_pre;                   // act' needs the pre-activation (gelu / softplus)
  int maxw, ldt;                  // widest layer, tangent buffer leading dim
};

template <typename T>
struct Weights {
  const T* W[OB_MAX_LAYERS];      // packed W_l (shared memory or global)
  const T* bias[OB_MAX_LAYERS];   // [w_{l+1}] (into theta)
};

// shared-memory tile of one MLP evaluation
template <typename T>
struct MlpSmem {
  T* x0;                          // [Rt][lda0] layer-0 input (state | time)
  T* hid[OB_MAX_LAYERS];          // [Rt][lda_{l+1}] act(pre) of hidden layers, reused
                                  //   in place as the layer cotangent during a VJP
  T* pre[OB_MAX_LAYERS];          // pre-activations (only when need_pre)
  T* tA;                          // tangent ping-pong (JVP only) [Rt][ldt]
  T* tB;
  T* ring;                        // per-warp weight rings (streamed weights), or nullptr
  int ring_elems;                 // total elements (split evenly over the CTA's warps)
};

template <typename T> OB_DEV T act_prime_from(T a, T z, int id) {
  // derivative from the activation value when possible (tanh: 1 - a^2;
  // relu: a > 0 <=> z > 0), else from the pre-activation
  switch (id) {
    case OB_ACT_IDENTITY: return T(1);
    case OB_ACT_RELU: return a > T(0) ? T(1) : T(0);
    case OB_ACT_TANH: return T(1) - a * a;
    default: return act_prime(z, id);
  }
}

}  // namespace ob

#include "gemm.cuh"

namespace ob {

// ------------------------------------------------------------- MLP tile
// LR: lane rows of the wide 4x4 GEMM variant (row tile 4*LR); the narrow 2x4
// variant uses 2*LR lane rows (same row tile, half the column tile) so layers
// of width ~64 still occupy every warp.  WS: weights in shared memory.
template <typename T, int LR, bool WS>
struct MlpTile {
  const Dims& d;
  const Weights<T>& W;
  MlpSmem<T>& s;
  int Rt;
  T* scratch;          // split-K partials for narrow output layers (nullable)
  int scratch_elems;
  T* hscratch;         // split-K partials for hidden layers (dedicated region, nullable)
  int hscratch_elems;

  OB_DEV MlpTile(const Dims& d_, const Weights<T>& W_, MlpSmem<T>& s_, int Rt_)
      : d(d_), W(W_), s(s_), Rt(Rt_), scratch(nullptr), scratch_elems(0), hscratch(nullptr),
        hscratch_elems(0) {}

  OB_DEV const T* in(int l) const { return l == 0 ? s.x0 : s.hid[l - 1]; }

  static constexpr int kWideCT = 4 * (32 / LR);
  static constexpr int kNarrowCT = 4 * (32 / (2 * LR));
  OB_DEV int tasks_wide(int n) const { return (Rt / (4 * LR)) * ((n + kWideCT - 1) / kWideCT); }
  OB_DEV int tasks_narrow(int n) const { return (Rt / (4 * LR)) * ((n + kNarrowCT - 1) / kNarrowCT); }

  template <class Epi>
  OB_DEV void nt(const T* X, int ldx, int l, int split, Warps ws, Epi epi) {
    const int N = d.w[l + 1], Kp = (d.w[l] + 3) & ~3;
    if (tasks_wide(N) * split >= ws.nw || 2 * LR > 32)
      gemm_nt<T, 4, 4, LR, WS>(X, ldx, Rt, W.W[l], d.ldw[l], N, Kp, ws, split, epi, s.ring,
                               s.ring_elems);
    else
      gemm_nt<T, 2, 4, (2 * LR > 32 ? 32 : 2 * LR), WS>(X, ldx, Rt, W.W[l], d.ldw[l], N, Kp, ws,
                                                         split, epi, s.ring, s.ring_elems);
  }
  template <class Epi>
  OB_DEV void nn(const T* D, int ldD, int l, int K, Warps ws, Epi epi, int split = 1) {
    const int Np = (d.w[l + 1] + 3) & ~3;
    if (tasks_wide(K) * split >= ws.nw || 2 * LR > 32)
      gemm_nn<T, 4, LR, WS>(D, ldD, Rt, W.W[l], d.ldw[l], Np, K, ws, epi, split, s.ring,
                            s.ring_elems);
    else
      gemm_nn<T, 2, (2 * LR > 32 ? 32 : 2 * LR), WS>(D, ldD, Rt, W.W[l], d.ldw[l], Np, K, ws, epi,
                                                      split, s.ring, s.ring_elems);
  }

  // split-K factor for a narrow output product of n columns reducing over kred
  // (deterministic: partials in `scratch`, summed in slice order)
  OB_DEV int narrow_split(int n, int kred) const {
    if (!scratch) return 1;
    const int tn = tasks_narrow(n);
    if (tn >= n_warps()) return 1;
    int split = min(n_warps() / max(tn, 1), scratch_elems / (Rt * n));
    return max(1, min(split, kred / 4));
  }
  // reduce split partials [split][Rt][n] -> dst[r*ldo + c] (+ bias when given)
  OB_DEV void split_reduce(int split, int n, T* dst, int ldo, const T* bias) {
    const int pst = Rt * n;
    for (int i = threadIdx.x; i < Rt * n; i += blockDim.x) {
      T acc = scratch[i];
      for (int sl = 1; sl < split; ++sl) acc = Num<T>::add(acc, scratch[sl * pst + i]);
      dst[(i / n) * ldo + i % n] = bias ? Num<T>::add(acc, bias[i % n]) : acc;
    }
    __syncthreads();
  }

  // Layers [0, nl) from x0; when nl == L the last writes z = W a + b to
  // out[r*ldo+n] (hidden layers store act(z) into hid, and z into pre if needed).
  unsigned long long* prof_acc = nullptr;
  OB_DEV void forward(T* out, int ldo, int nl) {
    PhaseTimer pt(prof_acc);
    for (int l = 0; l < nl; ++l) {
      const T* b = W.bias[l];
      const bool last = (l == d.L - 1);
      const int ldh = d.lda[l + 1], N = d.w[l + 1];
      if (last) {
        // narrow output layer: deterministic split-K through the scratch partials
        int split = 1;
        const int tn = tasks_narrow(N);
        if (scratch && tn < n_warps()) {
          split = min(n_warps() / max(tn, 1), scratch_elems / (Rt * N));
          split = max(1, min(split, (d.w[l] + 3) / 4));
        }
        if (split == 1) {
          nt(in(l), d.lda[l], l, 1, Warps::all(),
             [&](int r, int n, T acc, int) { out[r * ldo + n] = Num<T>::add(acc, b[n]); });
          __syncthreads();
        } else {
          T* part = scratch;
          const int pst = Rt * N;
          nt(in(l), d.lda[l], l, split, Warps::all(),
             [&](int r, int n, T acc, int sl) { part[sl * pst + r * N + n] = acc; });
          __syncthreads();
          pt.mark(12);
          for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
            T acc = part[i];
            for (int sl = 1; sl < split; ++sl) acc = Num<T>::add(acc, part[sl * pst + i]);
            out[(i / N) * ldo + i % N] = Num<T>::add(acc, b[i % N]);
          }
          __syncthreads();
          pt.mark(13);
        }
      } else {
        T* hid = s.hid[l];
        T* pre = d.need_pre ? s.pre[l] : nullptr;
        const int act = d.act;
        // too few column tasks for the CTA (tiny tiles): deterministic split-K through
        // the dedicated partials region, summed in slice order
        int hsplit = 1;
        if (hscratch && tasks_narrow(N) * 2 <= n_warps()) {
          hsplit = min(n_warps() / max(tasks_narrow(N), 1), hscratch_elems / (Rt * N));
          hsplit = max(1, min(hsplit, (d.w[l] + 3) / 16));
        }
        if (hsplit > 1) {
          T* part = hscratch;
          const int pst = Rt * N;
          nt(in(l), d.lda[l], l, hsplit, Warps::all(),
             [&](int r, int n, T acc, int sl) { part[sl * pst + r * N + n] = acc; });
          __syncthreads();
          for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
            T acc = part[i];
            for (int sl = 1; sl < hsplit; ++sl) acc = Num<T>::add(acc, part[sl * pst + i]);
            const int r = i / N, n = i % N;
            const T z = Num<T>::add(acc, b[n]);
            hid[r * ldh + n] = act_fn(z, act);
            if (pre) pre[r * ldh + n] = z;
          }
        } else {
          nt(in(l), d.lda[l], l, 1, Warps::all(), [&](int r, int n, T acc, int) {
            const T z = Num<T>::add(acc, b[n]);
            hid[r * ldh + n] = act_fn(z, act);
            if (pre) pre[r * ldh + n] = z;
          });
        }
        __syncthreads();
        pt.mark(10);
      }
    }
  }

  // Reverse pass through the cached forward (forward(.., L-1) must have run).
  // v: [Rt][ldv] output cotangent (rows >= Rv zero).  jtv (nullable): state part
  // of the input cotangent.  mu (nullable): padded parameter-cotangent slot,
  // receives scale * sum_{r<Rv} (df/dtheta)^T v.  Hidden activations are
  // overwritten by the layer cotangents.
  OB_DEV void vjp(const T* v, int ldv, int Rv, T* jtv, int ldo, T* mu, T scale) {
    for (int l = d.L - 1; l >= 0; --l) {
      const T* D = (l == d.L - 1) ? v : s.hid[l];
      const int ldD = (l == d.L - 1) ? ldv : d.lda[l + 1];
      if (l > 0) {
        if (mu) {
          gemm_tn_accum<T>(D, ldD, in(l), d.lda[l], Rv, d.w[l + 1], d.w[l], scale,
                           mu + d.mwoff[l], d.ldm[l], mu + d.mboff[l], Warps::all());
          __syncthreads();
        }
        T* h = s.hid[l - 1];
        const T* z = d.need_pre ? s.pre[l - 1] : nullptr;
        const int ldh = d.lda[l], act = d.act, K = d.w[l];
        int hsplit = 1;   // tiny tiles: deterministic split-K as in forward()
        if (hscratch && tasks_narrow(K) * 2 <= n_warps()) {
          hsplit = min(n_warps() / max(tasks_narrow(K), 1), hscratch_elems / (Rt * K));
          hsplit = max(1, min(hsplit, (d.w[l + 1] + 3) / 16));
        }
        if (hsplit > 1) {
          T* part = hscratch;
          const int pst = Rt * K;
          nn(D, ldD, l, K, Warps::all(),
             [&](int r, int k, T acc, int sl) { part[sl * pst + r * K + k] = acc; }, hsplit);
          __syncthreads();
          for (int i = threadIdx.x; i < Rt * K; i += blockDim.x) {
            T acc = part[i];
            for (int sl = 1; sl < hsplit; ++sl) acc = Num<T>::add(acc, part[sl * pst + i]);
            const int r = i / K, k = i % K;
            const T a = h[r * ldh + k];
            h[r * ldh + k] = Num<T>::mul(acc, act_prime_from(a, z ? z[r * ldh + k] : a, act));
          }
        } else {
          nn(D, ldD, l, K, Warps::all(), [&](int r, int k, T acc, int) {
            const T a = h[r * ldh + k];
            h[r * ldh + k] = Num<T>::mul(acc, act_prime_from(a, z ? z[r * ldh + k] : a, act));
          });
        }
        __syncthreads();
      } else {
        // first layer: the input product (narrow, N columns) and the dW0
        // accumulation read the same operands -> one phase on split warps
        const int nw = n_warps();
        const bool both = mu && jtv;
        const Warps wn = both ? Warps{0, nw / 2} : Warps::all();
        const Warps wa = both ? Warps{nw / 2, nw - nw / 2} : Warps::all();
        if (jtv) nn(D, ldD, 0, d.N, wn, [&](int r, int k, T acc, int) { jtv[r * ldo + k] = acc; });
        if (mu)
          gemm_tn_accum<T>(D, ldD, s.x0, d.lda[0], Rv, d.w[1], d.w[0], scale, mu + d.mwoff[0],
                           d.ldm[0], mu + d.mboff[0], wa);
        __syncthreads();
      }
    }
  }

  // Reverse pass that keeps the cached forward intact (repeated transposed
  // products at one linearisation point, e.g. the adjoint GMRES): layer
  // cotangents ping-pong through tA/tB, and each layer's parameter
  // accumulation runs on half the warps beside its input product.
  OB_DEV void vjp_keep(const T* v, int ldv, int Rv, T* jtv, int ldo, T* mu, T scale) {
    const T* cur = v;
    int ldc = ldv;
    T* bufs[2] = {s.tA, s.tB};
    int nb = 0;
    const int nw = n_warps();
    for (int l = d.L - 1; l >= 0; --l) {
      const bool both = mu && (l > 0 || jtv);
      const Warps wn = both ? Warps{0, nw / 2} : Warps::all();
      const Warps wa = both ? Warps{nw / 2, nw - nw / 2} : Warps::all();
      T* dst = bufs[nb];
      if (l > 0) {
        const T* h = s.hid[l - 1];
        const T* z = d.need_pre ? s.pre[l - 1] : nullptr;
        const int ldh = d.lda[l], ldt = d.ldt, act = d.act;
        nn(cur, ldc, l, d.w[l], wn, [&](int r, int k, T acc, int) {
          const T a = h[r * ldh + k];
          dst[r * ldt + k] = Num<T>::mul(acc, act_prime_from(a, z ? z[r * ldh + k] : a, act));
        });
      } else if (jtv) {
        const int split = mu ? 1 : narrow_split(d.N, d.w[1]);
        if (split > 1) {
          T* part = scratch;
          const int pst = Rt * d.N, nn_ = d.N;
          nn(cur, ldc, 0, d.N, wn,
             [&](int r, int k, T acc, int sl) { part[sl * pst + r * nn_ + k] = acc; }, split);
          __syncthreads();
          split_reduce(split, d.N, jtv, ldo, nullptr);
        } else {
          nn(cur, ldc, 0, d.N, wn, [&](int r, int k, T acc, int) { jtv[r * ldo + k] = acc; });
        }
      }
      if (mu)
        gemm_tn_accum<T>(cur, ldc, in(l), d.lda[l], Rv, d.w[l + 1], d.w[l], scale,
                         mu + d.mwoff[l], d.ldm[l], mu + d.mboff[l], wa);
      __syncthreads();
      cur = dst;
      ldc = d.ldt;
      nb ^= 1;
    }
  }

  // Tangent pass through the cached linearisation (forward(.., L-1) must have
  // run; time tangent held at 0, nn.py:177-180).  w: [Rt][ldw_] (rows/cols
  // beyond the state zero); out: [Rt][ldo].
  OB_DEV void jvp(const T* w, int ldw_, T* out, int ldo) {
    T* cur = s.tA;
    T* nxt = s.tB;
    for (int i = threadIdx.x; i < Rt * d.ldt; i += blockDim.x) {
      const int r = i / d.ldt, k = i % d.ldt;
      cur[i] = k < d.N ? w[r * ldw_ + k] : T(0);
    }
    __syncthreads();
    for (int l = 0; l < d.L; ++l) {
      const bool last = (l == d.L - 1);
      const T* h = last ? nullptr : s.hid[l];
      const T* z = (last || !d.need_pre) ? nullptr : s.pre[l];
      const int ldh = d.lda[l + 1], ldt = d.ldt, act = d.act;
      T* dst = last ? out : nxt;
      const int split = last ? narrow_split(d.w[l + 1], d.w[l]) : 1;
      if (split > 1) {
        T* part = scratch;
        const int nn_ = d.w[l + 1], pst = Rt * nn_;
        nt(cur, ldt, l, split, Warps::all(),
           [&](int r, int n, T acc, int sl) { part[sl * pst + r * nn_ + n] = acc; });
        __syncthreads();
        split_reduce(split, nn_, out, ldo, nullptr);
      } else {
        nt(cur, ldt, l, 1, Warps::all(), [&](int r, int n, T acc, int) {
          if (last) {
            dst[r * ldo + n] = acc;
          } else {
            const T a = h[r * ldh + n];
            dst[r * ldt + n] = Num<T>::mul(acc, act_prime_from(a, z ? z[r * ldh + n] : a, act));
          }
        });
        __syncthreads();
      }
      T* tmp = cur; cur = nxt; nxt = tmp;
    }
  }
};

}  // namespace ob
