// cnf_impl.cuh -- continuous-normalizing-flow right-hand side (config C4) for
// the persistent RK kernels: f_aug([z, Delta], t) = [f(z, t), -eps^T (df/dz) eps]
// with one fixed Rademacher probe eps per sample (Hutchinson trace estimator).
//
// The tile stacks 2*Rt rows: rows [0, Rt) carry the forward activations of the
// Rt samples and rows [Rt, 2Rt) their tangents along eps, so every layer does
// ONE weight pass for both (forward z = W a + b and tangent s = W u) and the
// reverse pass does one input-product pass and one parameter accumulation for
// the first- and second-order terms together:
//   dW_l += zbar_l a_{l-1}^T + sbar_l u_{l-1}^T,  db_l += zbar_l,
//   sbar = act'(z) * ubar,  zbar = act''(z) * s * ubar + act'(z) * abar.
// Pre-activations (forward z | raw tangent s) live in a per-tile global
// scratch (L2-resident); activations and cotangents in shared memory.
// The reference has no CNF; the fp64 restatement in oracle/fields_ext.py is
// pinned by finite differences (tests/test_oracle_ext.py).
#pragma once

#include "rk_impl.cuh"

namespace ob {

template <typename T, int LR>
struct CnfAdapter {
  const RkParams<T>& p;
  MlpTile<T, LR, false> mt;   // stacked rows: 4*LR = 2*Rt
  T* P;                       // this tile's pre-activation scratch
  T* aux;                     // [2Rt][lda_L]
  int Rt, R2, D;
  static constexpr bool kHasJvp = false;
  static constexpr bool kScaledVjp = false;  // vjp returns J^T w; the caller scales by h
  static constexpr int kCombineBatch = 4;    // stage loads in flight per ordered sum (registers)
  static constexpr bool kOwnsStep = false;   // the adapter runs whole RK steps itself
  OB_DEV void finish(T*) {}   // flush device-resident parameter cotangents (none here)
  OB_DEV void release() {}    // free per-CTA hardware resources (none here)

  OB_DEV CnfAdapter(const RkParams<T>& p_, const Weights<T>& W, MlpSmem<T>& ms, T* sm, int row0,
                    int Rv)
      : p(p_), mt(p_.d, W, ms, 4 * LR) {
    Rt = p.Rt;
    R2 = 2 * Rt;
    D = p.d.N - 1;
    P = p.cnf_pre + blockIdx.x * p.cnf_pre_stride;
    aux = sm + p.sm.aux;
    // Hutchinson probes into the tangent half of the input (time tangent 0)
    const int ld0 = p.d.lda[0];
    for (int i = threadIdx.x; i < Rv * D; i += blockDim.x) {
      const int r = i / D, j = i % D;
      mt.s.x0[(Rt + r) * ld0 + j] = p.eps[(long long)(row0 + r) * D + j];
    }
    __syncthreads();
  }
  OB_DEV T* x0() { return mt.s.x0; }
  OB_DEV int nin() const { return p.d.N - 1; }
  OB_DEV void put(int r, int j, T v) { mt.s.x0[r * p.d.lda[0] + j] = v; }
  OB_DEV void put_time(double t) {
    for (int r = threadIdx.x; r < Rt; r += blockDim.x) mt.s.x0[r * p.d.lda[0] + D] = T(t);
  }
  OB_DEV void set_scratch(T*, int) {}
  OB_DEV void jvp(const T*, T*) {}

  OB_DEV T* Pl(int l) {
    long long o = 0;
    for (int k = 0; k < l; ++k) o += (long long)R2 * p.d.lda[k + 1];
    return P + o;
  }

  // hidden layers [0, L-1): forward + tangent rows, pre-activations to P_l
  OB_DEV void hidden_forward() {
    const Dims& d = p.d;
    for (int l = 0; l < d.L - 1; ++l) {
      const int ldh = d.lda[l + 1], N = d.w[l + 1], act = d.act, rt = Rt;
      T* H = mt.s.hid[l];
      T* Pp = Pl(l);
      const T* b = mt.W.bias[l];
      mt.nt(mt.in(l), d.lda[l], l, 1, Warps::all(), [&](int r, int n, T acc, int) {
        if (r < rt) {
          const T z = Num<T>::add(acc, b[n]);
          Pp[r * ldh + n] = z;
          H[r * ldh + n] = act_fn(z, act);
        } else {
          Pp[r * ldh + n] = acc;
        }
      });
      __syncthreads();
      for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
        const int r = i / N, n = i % N;
        H[(Rt + r) * ldh + n] = Num<T>::mul(act_prime(Pp[r * ldh + n], act), Pp[(Rt + r) * ldh + n]);
      }
      __syncthreads();
    }
  }

  // f_aug(x0) -> out [Rt][ldn]: columns [0, D) = f, column D = -eps^T J eps
  OB_DEV void eval(T* out) {
    const Dims& d = p.d;
    hidden_forward();
    const int l = d.L - 1, lda = d.lda[d.L], ldn = d.ldn, rt = Rt;
    const T* b = mt.W.bias[l];
    T* ax = aux;
    mt.nt(mt.in(l), d.lda[l], l, 1, Warps::all(), [&](int r, int n, T acc, int) {
      if (r < rt) out[r * ldn + n] = Num<T>::add(acc, b[n]);
      else ax[(r - rt) * lda + n] = acc;
    });
    __syncthreads();
    const int ld0 = d.lda[0];
    for (int r = warp_id(); r < Rt; r += n_warps()) {
      const T jv = warp_dot(aux + r * lda, mt.s.x0 + (Rt + r) * ld0, D);
      if (lane_id() == 0) out[r * ldn + D] = -jv;
    }
    __syncthreads();
  }

  // (J_aug^T w, mu += h * P_aug^T w) at x0; w: [Rt][ldn] with columns [0, D) the
  // cotangent of f and column D that of Delta' (f_aug does not depend on Delta)
  OB_DEV void vjp(const T* w, T* jtv, T* mu, double h, int Rv) {
    const Dims& d = p.d;
    const int ldn = d.ldn, ld0 = d.lda[0], act = d.act, rt = Rt;
    const T hs = T(h);
    hidden_forward();
    // output-layer cotangents: [v_z ; -v_Delta * eps]
    const int lo = d.lda[d.L];
    for (int i = threadIdx.x; i < Rt * D; i += blockDim.x) {
      const int r = i / D, n = i % D;
      aux[r * lo + n] = w[r * ldn + n];
      aux[(Rt + r) * lo + n] = Num<T>::mul(-w[r * ldn + D], mt.s.x0[(Rt + r) * ld0 + n]);
    }
    __syncthreads();
    {
      const int l = d.L - 1;
      if (mu) {
        gemm_tn_accum<T>(aux, lo, mt.in(l), d.lda[l], R2, d.w[l + 1], d.w[l], hs, mu + d.mwoff[l],
                         d.ldm[l], mu + d.mboff[l], Warps::all(), Rt);
        __syncthreads();
      }
      T* H = mt.s.hid[l - 1];
      const int ldh = d.lda[l];
      mt.nn(aux, lo, l, d.w[l], Warps::all(), [&](int r, int k, T acc, int) { H[r * ldh + k] = acc; });
      __syncthreads();
    }
    for (int l = d.L - 2; l >= 0; --l) {
      const int ldh = d.lda[l + 1], N = d.w[l + 1];
      T* H = mt.s.hid[l];
      const T* Pp = Pl(l);
      for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
        const int r = i / N, n = i % N;
        const T z = Pp[r * ldh + n], sr = Pp[(Rt + r) * ldh + n];
        const T ab = H[r * ldh + n], ub = H[(Rt + r) * ldh + n];
        const T sp = act_prime(z, act), spp = act_second(z, act);
        H[(Rt + r) * ldh + n] = Num<T>::mul(sp, ub);
        H[r * ldh + n] = Num<T>::add(Num<T>::mul(Num<T>::mul(spp, sr), ub), Num<T>::mul(sp, ab));
      }
      __syncthreads();
      if (l > 0) {
        if (mu) {
          gemm_tn_accum<T>(H, ldh, mt.in(l), d.lda[l], R2, N, d.w[l], hs, mu + d.mwoff[l],
                           d.ldm[l], mu + d.mboff[l], Warps::all(), Rt);
          __syncthreads();
        }
        T* Hn = mt.s.hid[l - 1];
        const int ldn2 = d.lda[l];
        mt.nn(H, ldh, l, d.w[l], Warps::all(), [&](int r, int k, T acc, int) { Hn[r * ldn2 + k] = acc; });
        __syncthreads();
      } else {
        const int nw = n_warps();
        const bool both = mu && jtv;
        const Warps wn = both ? Warps{0, nw / 2} : Warps::all();
        const Warps wa = both ? Warps{nw / 2, nw - nw / 2} : Warps::all();
        if (jtv)
          mt.nn(H, ldh, 0, D, wn, [&](int r, int k, T acc, int) { if (r < rt) jtv[r * ldn + k] = acc; });
        if (mu)
          gemm_tn_accum<T>(H, ldh, mt.s.x0, ld0, R2, N, d.w[0], hs, mu + d.mwoff[0], d.ldm[0],
                           mu + d.mboff[0], wa, Rt);
        __syncthreads();
      }
    }
    if (jtv)
      for (int r = threadIdx.x; r < Rt; r += blockDim.x) jtv[r * ldn + D] = T(0);
    __syncthreads();
  }
};

template <typename T, int LR>
static cudaError_t launch_cnf_lr(const RkParams<T>& p, int tiles, size_t smem, cudaStream_t st,
                                 bool forward) {
  using F = CnfAdapter<T, LR>;
  return forward ? launch_smem(rk_forward_kernel<T, F>, tiles, smem, st, p)
                 : launch_smem(rk_reverse_kernel<T, F>, tiles, smem, st, p);
}

template <typename T>
cudaError_t launch_cnf(const RkParams<T>& p, int lr, int tiles, size_t smem, cudaStream_t st,
                       bool forward) {
  switch (lr) {
    case 2: return launch_cnf_lr<T, 2>(p, tiles, smem, st, forward);
    case 4: return launch_cnf_lr<T, 4>(p, tiles, smem, st, forward);
    default: return launch_cnf_lr<T, 8>(p, tiles, smem, st, forward);
  }
}

template <typename T>
cudaError_t launch_cnf_field(const RkParams<T>& p, int lr, int tiles, size_t smem, int mode,
                             double t, const T* u, const T* w, T* out, cudaStream_t st) {
  switch (lr) {
    case 2: return launch_smem(field_op_kernel<T, CnfAdapter<T, 2>>, tiles, smem, st, p, mode, t, u, w, out);
    case 4: return launch_smem(field_op_kernel<T, CnfAdapter<T, 4>>, tiles, smem, st, p, mode, t, u, w, out);
    default: return launch_smem(field_op_kernel<T, CnfAdapter<T, 8>>, tiles, smem, st, p, mode, t, u, w, out);
  }
}

}  // namespace ob
