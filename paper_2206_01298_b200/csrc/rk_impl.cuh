// rk_impl.cuh -- persistent explicit Runge-Kutta forward / discrete-adjoint
// reverse kernels (one CTA = one fixed tile of samples for the whole sweep).
//
// Forward: integrate (integrators.py:252-292) -> explicit_rk_step
// (:196-222) with FSAL carry, writing the checkpoint records the policy asks
// for (checkpointing.py:242-269).  Reverse: executes a host-compiled program
// of REPLAY / REVERSE ops (checkpointing.py:286-340 + replay_step,
// integrators.py:352-368) and the stage-wise transpose rk_adjoint_step
// (adjoint.py:67-94).  Stage sums ascend in j with the scalar (h*a_ij) formed
// first and exact zeros skipped, with round-to-nearest mul/add (no FMA
// contraction), reproducing the reference combination bit-for-bit in fp64.
#pragma once
#include <algorithm>
#include <type_traits>

#include "rk.cuh"

namespace ob {

OB_DEV void set_status(int* status, int code, int info) {
  if (atomicCAS(status, 0, code) == 0) status[1] = info;
}

// Adapters whose CTAs cooperate across a thread-block cluster (multicast weight
// streams) must not leave the sweep early: a CTA that hits an error records it and
// keeps stepping with its cluster (its results are discarded by the host).
// threads per CTA of the kernels instantiated with adapter F (default kThreads)
template <class F, class = void> struct BlockThreads { static constexpr int value = kThreads; };
template <class F>
struct BlockThreads<F, std::void_t<decltype(F::kBlockThreads)>> { static constexpr int value = F::kBlockThreads; };
template <class F, class = void> struct NoEarlyExit { static constexpr bool value = false; };
template <class F>
struct NoEarlyExit<F, std::void_t<decltype(F::kNoEarlyExit)>> { static constexpr bool value = F::kNoEarlyExit; };

template <typename T>
OB_DEV void zero_smem(T* sm, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = T(0);
  __syncthreads();
}

// carve the MLP tile out of shared memory; stage packed weights into smem when
// the layout reserved room for them (one L2 read per CTA per launch)
template <typename T>
OB_DEV void setup_tile(const RkParams<T>& p, T* sm, MlpSmem<T>& ms, Weights<T>& W) {
  const SmemLayout& L = p.sm;
  ms.x0 = sm + L.x0;
  for (int l = 0; l < OB_MAX_LAYERS; ++l) {
    ms.hid[l] = L.hid[l] >= 0 ? sm + L.hid[l] : nullptr;
    ms.pre[l] = L.pre[l] >= 0 ? sm + L.pre[l] : nullptr;
  }
  ms.tA = L.tA >= 0 ? sm + L.tA : nullptr;
  ms.tB = L.tB >= 0 ? sm + L.tB : nullptr;
  ms.ring = L.ring >= 0 ? sm + L.ring : nullptr;
  ms.ring_elems = L.ring >= 0 ? L.ring_elems : 0;
  const T* base = p.packed;
  if (L.wts >= 0) {
    T* dst = sm + L.wts;
    const long long n16 = p.d.n_packed * (long long)sizeof(T) / 16;  // packed length is a multiple of 4
    const float4* src4 = reinterpret_cast<const float4*>(p.packed);
    float4* dst4 = reinterpret_cast<float4*>(dst);
    for (long long i = threadIdx.x; i < n16; i += blockDim.x) dst4[i] = src4[i];
    base = dst;
  }
  for (int l = 0; l < p.d.L; ++l) {
    W.W[l] = base + p.d.pwoff[l];
    W.bias[l] = p.W.bias[l];
  }
  __syncthreads();
}

// ------------------------------------------------------------ field adapters
// The RK kernels are generic over the right-hand side: an adapter exposes the
// tile's input buffer (x0, rows [0, Rt), state columns [0, nin) then time),
// eval (f(x0) -> out [Rt][ldn]) and vjp (cotangent w -> jtv, mu).

// MlpField / the stiff a*u + s*MLP(u) field (integrators.py:76-141)
template <typename T, int LR, bool WS>
struct MlpAdapter {
  const RkParams<T>& p;
  MlpTile<T, LR, WS> mt;
  OB_DEV MlpAdapter(const RkParams<T>& p_, const Weights<T>& W, MlpSmem<T>& ms, T* sm, int, int)
      : p(p_), mt(p_.d, W, ms, p_.Rt) {
    mt.prof_acc = p.prof ? p.phase : nullptr;
    if (p.sm.hscr >= 0) { mt.hscratch = sm + p.sm.hscr; mt.hscratch_elems = p.sm.hscr_elems; }
  }
  OB_DEV MlpAdapter(const RkParams<T>& p_, const MlpTile<T, LR, WS>& m) : p(p_), mt(m) {}
  OB_DEV T* x0() { return mt.s.x0; }
  OB_DEV int nin() const { return p.d.N; }
  // field input: state element j of row r, and the time column (CTA-wide)
  OB_DEV void put(int r, int j, T v) { mt.s.x0[r * p.d.lda[0] + j] = v; }
  OB_DEV void put_time(double t) {
    if (p.d.time_input)
      for (int r = threadIdx.x; r < p.Rt; r += blockDim.x) mt.s.x0[r * p.d.lda[0] + p.d.N] = T(t);
  }
  OB_DEV void put_time_row(int r, double t) {   // per-row time (adaptive stepping)
    if (p.d.time_input) mt.s.x0[r * p.d.lda[0] + p.d.N] = T(t);
  }
  OB_DEV void set_scratch(T* s, int n) { mt.scratch = s; mt.scratch_elems = n; }
  static constexpr bool kHasJvp = true;
  static constexpr bool kScaledVjp = false;  // vjp returns J^T w; the caller scales by h
  static constexpr int kCombineBatch = 4;    // stage loads in flight per ordered sum (registers)
  static constexpr bool kOwnsStep = false;   // the adapter runs whole RK steps itself
  OB_DEV void finish(T*) {}   // flush device-resident parameter cotangents (none here)
  OB_DEV void release() {}    // free per-CTA hardware resources (none here)

  // (df/du) w at x0 (integrators.py:88-92)
  OB_DEV void jvp(const T* w, T* out) {
    const int N = p.d.N, ldn = p.d.ldn;
    mt.forward(nullptr, 0, p.d.L - 1);
    mt.jvp(w, ldn, out, ldn);
    if (p.field_kind == OB_FIELD_STIFF) {
      for (int i = threadIdx.x; i < p.Rt * N; i += blockDim.x) {
        const int o = (i / N) * ldn + i % N, j = i % N;
        out[o] = Num<T>::add(Num<T>::mul(p.diag[j], w[o]), Num<T>::mul(p.out_scale, out[o]));
      }
      __syncthreads();
    }
  }

  // f(x0) -> out ([Rt][ldn]; columns >= N untouched)
  OB_DEV void eval(T* out) {
    const int N = p.d.N, ldn = p.d.ldn;
    mt.forward(out, ldn, p.d.L);
    if (p.field_kind == OB_FIELD_STIFF) {  // a*u + s*mlp(u)
      const int ld0 = p.d.lda[0];
      for (int i = threadIdx.x; i < p.Rt * N; i += blockDim.x) {
        const int r = i / N, j = i % N;
        out[r * ldn + j] = Num<T>::add(Num<T>::mul(p.diag[j], mt.s.x0[r * ld0 + j]),
                                       Num<T>::mul(p.out_scale, out[r * ldn + j]));
      }
      __syncthreads();
    }
  }

  // ((df/du)^T w, mu += h * (df/dtheta)^T w) at the state in x0
  OB_DEV void vjp(const T* w, T* jtv, T* mu, double h, int Rv) {
    PhaseTimer pt(p.prof ? p.phase : nullptr);
    mt.forward(nullptr, 0, p.d.L - 1);  // hidden layers only: the output value is not needed
    pt.mark(kPhRecompute);
    const int ldn = p.d.ldn;
    if (p.field_kind == OB_FIELD_STIFF) {
      mt.vjp(w, ldn, Rv, jtv, ldn, mu, T(h * double(p.out_scale)));
      const int N = p.d.N;
      for (int i = threadIdx.x; i < p.Rt * N; i += blockDim.x) {
        const int r = i / N, j = i % N;
        jtv[r * ldn + j] = Num<T>::add(Num<T>::mul(p.diag[j], w[r * ldn + j]),
                                       Num<T>::mul(p.out_scale, jtv[r * ldn + j]));
      }
      __syncthreads();
    } else {
      mt.vjp(w, ldn, Rv, jtv, ldn, mu, T(h));
    }
  }
};

// One explicit RK step of the tile from the state in `u` (smem [Rt][ldn]).
// ks: this tile's stage-derivative scratch [s][Rt][ldn].  rec (nullable):
// record base for this step ([s+1][B][N]).  On return `u` holds u_next.
// Returns false (block-uniform) if u_next has a non-finite entry.
// keep_last: k_{s-1} feeds the next step (FSAL carry); otherwise stages whose
// derivative nothing uses (p.skip_vjp: b_i = 0 and a_ji = 0 for j > i) are not
// evaluated (their stage state is still recorded).
template <typename T, class F>
OB_DEV bool rk_step_tile(const RkParams<T>& p, F& f, T* u, T* ks, double t, double h, bool carry,
                         T* rec, int row0, int Rv, bool keep_last = false) {
  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt, s = p.s, nin = f.nin();
  const long long kst = (long long)Rt * ldn;
  const long long vec = (long long)p.B * N;
  PhaseTimer pt(p.prof ? p.phase : nullptr);
  for (int i = 0; i < s; ++i) {
    // stage coefficients T(h a_iq), formed once per stage (exact zeros skipped)
    T cq[OB_MAX_STAGES];
    unsigned nzq = 0;
#pragma unroll
    for (int q = 0; q < OB_MAX_STAGES; ++q) {
      const double aiq = q < i ? p.a[i * OB_MAX_STAGES + q] : 0.0;
      cq[q] = T(h * aiq);
      if (aiq != 0.0) nzq |= 1u << q;
    }
    for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
      const int r = idx / N, j = idx % N;
      // issue every stage-derivative load (L2-resident scratch) before the dependent
      // sum so they overlap; the sum keeps the reference order
      T v = u[r * ldn + j];
#pragma unroll
      for (int q0 = 0; q0 < OB_MAX_STAGES; q0 += F::kCombineBatch) {
        T kv[F::kCombineBatch];
#pragma unroll
        for (int t = 0; t < F::kCombineBatch; ++t)
          kv[t] = q0 + t < i ? ks[(q0 + t) * kst + r * ldn + j] : T(0);
#pragma unroll
        for (int t = 0; t < F::kCombineBatch; ++t)
          if ((nzq >> (q0 + t)) & 1u) v = Num<T>::add(v, Num<T>::mul(cq[q0 + t], kv[t]));
      }
      if (j < nin) f.put(r, j, v);
      if (rec && r < Rv) rec[i * vec + (long long)(row0 + r) * N + j] = v;
    }
    f.put_time(t + p.c[i] * h);
    __syncthreads();
    pt.mark(8);   // stage combination + record write
    if (i == 0 && carry) {  // FSAL: k_0 of this step is k_{s-1} of the previous one
      for (int idx = threadIdx.x; idx < kst; idx += blockDim.x) ks[idx] = ks[(s - 1) * kst + idx];
      __syncthreads();
    } else if (!((p.skip_vjp >> i) & 1u) || (keep_last && i == s - 1)) {
      f.eval(ks + i * kst);
    }
    pt.mark(9);   // field eval
  }
  int bad = 0;
  T cb[OB_MAX_STAGES];
  unsigned nzb = 0;
#pragma unroll
  for (int q = 0; q < OB_MAX_STAGES; ++q) {
    const double bq = q < s ? p.b[q] : 0.0;
    cb[q] = T(h * bq);
    if (bq != 0.0) nzb |= 1u << q;
  }
  for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
    const int r = idx / N, j = idx % N;
    T v = u[r * ldn + j];
#pragma unroll
    for (int i0 = 0; i0 < OB_MAX_STAGES; i0 += F::kCombineBatch) {
      T kv[F::kCombineBatch];
#pragma unroll
      for (int t = 0; t < F::kCombineBatch; ++t)
        kv[t] = i0 + t < s ? ks[(i0 + t) * kst + r * ldn + j] : T(0);
#pragma unroll
      for (int t = 0; t < F::kCombineBatch; ++t)
        if ((nzb >> (i0 + t)) & 1u) v = Num<T>::add(v, Num<T>::mul(cb[i0 + t], kv[t]));
    }
    u[r * ldn + j] = v;
    if (r < Rv) {
      if (!Num<T>::finite(v)) bad = 1;
      if (rec) rec[s * vec + (long long)(row0 + r) * N + j] = v;
    }
  }
  return __syncthreads_or(bad) == 0;
}

template <typename T>
OB_DEV void load_rows(T* dst, int ldd, const T* src, int N, int row0, int Rv) {
  for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
    const int r = idx / N, j = idx % N;
    dst[r * ldd + j] = src[(long long)(row0 + r) * N + j];
  }
}

template <typename T>
OB_DEV void store_rows(T* dst, int N, const T* src, int lds, int row0, int Rv) {
  for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
    const int r = idx / N, j = idx % N;
    dst[(long long)(row0 + r) * N + j] = src[r * lds + j];
  }
}

// state-shaped buffers (0 u, 1 lam, 2 lamn, 3 w, 4 jtv): shared memory, or a
// per-tile global scratch for states too large for it (C3: 16384 per sample)
template <typename T>
OB_DEV T* state_buf(const RkParams<T>& p, T* sm, int k) {
  if (p.sm.u >= 0) {
    const int off[5] = {p.sm.u, p.sm.lam, p.sm.lamn, p.sm.w, p.sm.jtv};
    return sm + off[k];
  }
  return p.state_glob + blockIdx.x * p.state_stride + (long long)k * p.Rt * p.d.ldn;
}

// --------------------------------------------------------------- observation losses
// Reference LossSpec mse/mae over K observations with optional min-max scaling
// (losses.py:10-107), batched as the mean over samples: states captured at the
// observed boundaries in the forward (adjoint.py:196-210), seeds injected into
// lambda before reversing the step that ends at each observed boundary and at
// boundary 0 last (backward_sweep, adjoint.py:235-253).
template <typename T>
OB_DEV bool is_obs_loss(const RkParams<T>& p) {
  return p.loss_kind == OB_LOSS_OBS_MSE || p.loss_kind == OB_LOSS_OBS_MAE;
}



// rows of boundary n -> predictions[k] when boundary n is observed
template <typename T>
OB_DEV void obs_capture(const RkParams<T>& p, const T* u, int n, int row0, int Rv) {
  if (!p.obs_k) return;
  const int k = p.obs_k[n];
  if (k < 0) return;
  store_rows(p.preds + (long long)k * p.B * p.d.N, p.d.N, u, p.d.ldn, row0, Rv);
  __syncthreads();
}

// r = scale(pred) - obs for one element, and the scaling span (1 when unscaled
// or degenerate: MinMaxScaling.apply / .chain, losses.py:26-37)
template <typename T>
OB_DEV double obs_residual(const RkParams<T>& p, int k, int row, int j, double& span) {
  const long long g = ((long long)k * p.B + row) * p.d.N + j;
  double v = double(p.preds[g]);
  span = 1.0;
  if (p.scale_lo) {
    const double lo = double(p.scale_lo[j]), hi = double(p.scale_hi[j]);
    if (hi > lo) {
      span = hi - lo;
      v = (v - lo) / span;
    }
  }
  return v - double(p.obs_values[g]);
}

// seed added to lambda at an observed boundary: the built-in observation losses form
// {sign r | 2r} / (K N), chained through the min-max span, / B (loss_and_grad_seed,
// losses.py:78-107); OB_LOSS_SEED takes the caller's injection as given
template <typename T>
OB_DEV double obs_seed(const RkParams<T>& p, int k, int row, int j) {
  if (p.loss_kind == OB_LOSS_SEED) return double(p.obs_values[((long long)k * p.B + row) * p.d.N + j]);
  double span;
  const double rr = obs_residual(p, k, row, j, span);
  const double denom = double(p.n_obs) * p.d.N;
  const double sd = p.loss_kind == OB_LOSS_OBS_MAE ? double((rr > 0.0) - (rr < 0.0)) / denom
                                                    : 2.0 * rr / denom;
  return sd / span / p.batch_global;
}

// deterministic block sum (fixed shuffle tree, then warps in order); result on thread 0
OB_DEV double block_sum_fixed(double v) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < n_warps(); ++w) s += red[w];
  __syncthreads();
  return s;
}

// per-tile sum over samples of the per-sample loss mean over K*N (losses.py:94-107)
template <typename T>
OB_DEV void obs_loss_partial(const RkParams<T>& p, int row0, int Rv, int tile) {
  const int N = p.d.N;
  const int per = Rv * N;
  double acc = 0.0;
  for (int k = 0; k < p.n_obs; ++k)
    for (int i = threadIdx.x; i < per; i += blockDim.x) {
      double span;
      const double r = obs_residual(p, k, row0 + i / N, i % N, span);
      acc += p.loss_kind == OB_LOSS_OBS_MAE ? fabs(r) : r * r;
    }
  acc = block_sum_fixed(acc);
  if (threadIdx.x == 0) p.loss_part[tile] = acc / (double(p.n_obs) * N);
}

// lambda += dL/du at boundary n (inject_observation, adjoint.py:135-140):
// seed = {sign(r) | 2r} / (K N), chained through the scaling, / B
template <typename T>
OB_DEV void obs_inject(const RkParams<T>& p, T* lam, int n, int row0, int Rv) {
  if (!p.obs_k) return;
  const int k = p.obs_k[n];
  if (k < 0) return;
  const int N = p.d.N, ldn = p.d.ldn;
  for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
    const int r = idx / N, j = idx % N;
    lam[r * ldn + j] = T(double(lam[r * ldn + j]) + obs_seed(p, k, row0 + r, j));
  }
  __syncthreads();
}

// --------------------------------------------------------------- losses
// Terminal losses (losses.py:78-107 with the batch mean; BASELINE configs):
// per-tile fp64 partial sums in fixed order, and the seed lambda_N = dL/du(T).
constexpr double kLog2Pi = 1.8378770664093454836;

// Classification head (config C3): global average pool over the 16x16 pixels,
// logits = Wh gap + bh, softmax cross-entropy.  Row r's gap/logits/dlogits are
// computed by warp r; returns nothing, fills g[C], dl[n_classes] (smem).
template <typename T>
OB_DEV void ce_head_row(const RkParams<T>& p, const T* urow, int label, double* gap, double* dl,
                        double* loss) {
  const int C = p.d.w[2], K = p.n_classes, P = p.d.N / C;
  for (int c = lane_id(); c < C; c += 32) {
    double s = 0.0;
    for (int q = 0; q < P; ++q) s += double(urow[q * C + c]);
    gap[c] = s / P;
  }
  __syncwarp();
  if (lane_id() == 0) {
    double mx = -1e300;
    for (int k = 0; k < K; ++k) {
      double z = double(p.head[K * C + k]);
      for (int c = 0; c < C; ++c) z += double(p.head[k * C + c]) * gap[c];
      dl[k] = z;
      mx = z > mx ? z : mx;
    }
    double se = 0.0;
    for (int k = 0; k < K; ++k) se += exp(dl[k] - mx);
    *loss = mx + log(se) - dl[label];
    for (int k = 0; k < K; ++k) dl[k] = exp(dl[k] - mx) / se - (k == label ? 1.0 : 0.0);
  }
  __syncwarp();
}

template <typename T>
OB_DEV void loss_partial(const RkParams<T>& p, const T* u, int row0, int Rv, int tile) {
  if (p.loss_kind == OB_LOSS_SEED) {   // the caller forms the loss from u_final / predictions
    if (threadIdx.x == 0) p.loss_part[tile] = 0.0;
    return;
  }
  if (is_obs_loss(p)) {
    obs_loss_partial(p, row0, Rv, tile);
    return;
  }
  if (p.loss_kind == OB_LOSS_CE_HEAD) {
    // per-tile loss sum and head-gradient partial (dWh = dl gap^T / B, dbh = dl / B);
    // scratch rows (gap | dl | loss, fp64) live after this tile's head partial
    const int C = p.d.w[2], K = p.n_classes;
    const int ldn = p.d.ldn;
    double* scr = reinterpret_cast<double*>(p.head_part + (long long)p.tiles_total * (K * C + K)) +
                  (long long)tile * 8 * (64 + 16 + 1);
    auto gap = [&](int r) { return scr + r * 81; };
    auto dl = [&](int r) { return scr + r * 81 + 64; };
    for (int r = warp_id(); r < Rv && r < 8; r += n_warps())
      ce_head_row(p, u + r * ldn, p.labels[row0 + r], gap(r), dl(r), scr + r * 81 + 80);
    __syncthreads();
    T* hp = p.head_part + (long long)tile * (K * C + K);
    const double ib = 1.0 / p.batch_global;
    for (int i = threadIdx.x; i < K * C + K; i += blockDim.x) {
      double acc = 0.0;
      for (int r = 0; r < Rv; ++r) acc += (i < K * C ? dl(r)[i / C] * gap(r)[i % C] : dl(r)[i - K * C]);
      hp[i] = T(acc * ib);
    }
    if (threadIdx.x == 0) {
      double acc = 0.0;
      for (int r = 0; r < Rv; ++r) acc += scr[r * 81 + 80];
      p.loss_part[tile] = acc;
    }
    return;
  }
  if (threadIdx.x != 0) return;
  const int N = p.d.N, ldn = p.d.ldn;
  double acc = 0.0;
  for (int r = 0; r < Rv; ++r) {
    double sr = 0.0;
    if (p.loss_kind == OB_LOSS_CNF_NLL) {  // NLL = 0.5|z|^2 + D/2 log 2pi + Delta
      const int D = N - 1;
      for (int j = 0; j < D; ++j) {
        const double v = double(u[r * ldn + j]);
        sr += v * v;
      }
      acc += 0.5 * sr + 0.5 * D * kLog2Pi + double(u[r * ldn + D]);
      continue;
    }
    for (int j = 0; j < N; ++j) {
      double v = double(u[r * ldn + j]);
      if (p.loss_kind == OB_LOSS_MSE) v -= double(p.targets[(long long)(row0 + r) * N + j]);
      sr += v * v;
    }
    acc += (p.loss_kind == OB_LOSS_MSE) ? sr / N : 0.5 * sr;
  }
  p.loss_part[tile] = acc;
}

template <typename T>
OB_DEV void loss_seed(const RkParams<T>& p, T* lam, int row0, int Rv) {
  const int N = p.d.N, ldn = p.d.ldn;
  if (p.loss_kind == OB_LOSS_SEED) {   // adjoint_terminal (adjoint.py:47-52): lambda_N as given
    for (int i = threadIdx.x; i < p.Rt * ldn; i += blockDim.x) lam[i] = T(0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
      const int r = idx / N, j = idx % N;
      lam[r * ldn + j] = p.seed[(long long)(row0 + r) * N + j];
    }
    return;
  }
  if (is_obs_loss(p)) {  // lambda starts at zero; seeds arrive by injection
    for (int i = threadIdx.x; i < p.Rt * ldn; i += blockDim.x) lam[i] = T(0);
    return;
  }
  if (p.loss_kind == OB_LOSS_CE_HEAD) {
    // lambda = d CE / du(T) = (dl Wh) / (P * B) broadcast over the pixels
    const int C = p.d.w[2], K = p.n_classes, P = N / C;
    double* scr = reinterpret_cast<double*>(p.head_part + (long long)p.tiles_total * (K * C + K)) +
                  (long long)blockIdx.x * 8 * (64 + 16 + 1);
    double* dg = reinterpret_cast<double*>(p.head_part + (long long)p.tiles_total * (K * C + K)) +
                 (long long)p.tiles_total * 8 * 81 + (long long)blockIdx.x * 8 * 64;
    for (int r = warp_id(); r < Rv && r < 8; r += n_warps())
      ce_head_row(p, p.u_final + (long long)(row0 + r) * N, p.labels[row0 + r], scr + r * 81,
                  scr + r * 81 + 64, scr + r * 81 + 80);
    __syncthreads();
    for (int i = threadIdx.x; i < Rv * C; i += blockDim.x) {
      const int r = i / C, c = i % C;
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += scr[r * 81 + 64 + k] * double(p.head[k * C + c]);
      dg[r * 64 + c] = s / (double(P) * p.batch_global);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
      const int r = idx / N, j = idx % N;
      lam[(long long)r * ldn + j] = T(dg[r * 64 + j % C]);
    }
    return;
  }
  for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
    const int r = idx / N, j = idx % N;
    const long long g = (long long)(row0 + r) * N + j;
    T v = p.u_final[g];
    if (p.loss_kind == OB_LOSS_MSE) v = T(2) * (v - p.targets[g]) / T(N);
    if (p.loss_kind == OB_LOSS_CNF_NLL && j == N - 1) v = T(1);
    lam[r * ldn + j] = v / T(p.batch_global);
  }
}

// --------------------------------------------------------------- forward
template <typename T, class F>
__global__ void __launch_bounds__(BlockThreads<F>::value, 1) rk_forward_kernel(const __grid_constant__ RkParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  zero_smem(sm, p.sm.wts >= 0 ? p.sm.wts : p.sm.total);
  const int tile = blockIdx.x;
  const int row0 = tile * p.R;
  const int Rv = max(0, min(p.R, p.B - row0));   // 0 on cluster-padding tiles
  MlpSmem<T> ms;
  Weights<T> W;
  setup_tile(p, sm, ms, W);
  F f(p, W, ms, sm, row0, Rv);
  // split-K scratch: the same lamn | w | jtv region as the reverse kernel's
  // replays, so forward and replayed steps sum identically (bit-identical records)
  if (p.sm.u >= 0) f.set_scratch(sm + p.sm.lamn, p.sm.jtv + p.Rt * p.d.ldn - p.sm.lamn);
  T* u = state_buf(p, sm, 0);
  T* ks = p.sm.ks >= 0 ? sm + p.sm.ks : p.scratch + tile * p.scratch_stride;
  const int N = p.d.N, ldn = p.d.ldn;
  const long long vec = (long long)p.B * N;

  load_rows(u, ldn, p.u0, N, row0, Rv);
  __syncthreads();
  int bad = 0;  // as_state rejects non-finite inputs (nn.py:31-32)
  for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x)
    if (!Num<T>::finite(u[(idx / N) * ldn + idx % N])) bad = 1;
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) set_status(p.status, OB_ERR_VALUE, -1);
    if constexpr (!NoEarlyExit<F>::value) {
      f.release();
      return;
    }
  }
  for (int n = 0; n < p.n_steps; ++n) {
    const double t = p.ts[n], h = p.ts[n + 1] - p.ts[n];
    obs_capture(p, u, n, row0, Rv);
    if (p.fwd_sol[n] >= 0) {
      store_rows(p.sol + p.fwd_sol[n] * vec, N, u, ldn, row0, Rv);
      __syncthreads();
    }
    T* rec = p.fwd_rec[n] >= 0 ? p.rec + (long long)p.fwd_rec[n] * (p.s + 1) * vec : nullptr;
    PhaseTimer pt(p.prof ? p.phase : nullptr);
    bool ok;
    if constexpr (F::kOwnsStep)
      ok = f.step(u, t, h, p.fsal && n > 0, rec, row0, p.fsal && n + 1 < p.n_steps);
    else
      ok = rk_step_tile<T, F>(p, f, u, ks, t, h, p.fsal && n > 0, rec, row0, Rv,
                              p.fsal && n + 1 < p.n_steps);
    pt.mark(kPhFwdStep);
    if (!ok) {  // integrators.py:219-220
      if (threadIdx.x == 0) set_status(p.status, OB_ERR_INTEGRATION, n);
      if constexpr (!NoEarlyExit<F>::value) {
        f.release();
        return;
      }
    }
  }
  f.release();
  store_rows(p.u_final, N, u, ldn, row0, Rv);
  obs_capture(p, u, p.n_steps, row0, Rv);
  loss_partial(p, u, row0, Rv, tile);
}

// --------------------------------------------------------------- reverse
template <typename T, class F>
__global__ void __launch_bounds__(BlockThreads<F>::value, 1) rk_reverse_kernel(const __grid_constant__ RkParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  if (*(volatile int*)p.status != 0) return;  // forward failed
  zero_smem(sm, p.sm.wts >= 0 ? p.sm.wts : p.sm.total);
  const int tile = blockIdx.x;
  const int row0 = tile * p.R;
  const int Rv = max(0, min(p.R, p.B - row0));   // 0 on cluster-padding tiles
  MlpSmem<T> ms;
  Weights<T> W;
  setup_tile(p, sm, ms, W);
  F f(p, W, ms, sm, row0, Rv);
  if (p.sm.u >= 0)  // lamn | w | jtv are free during replays
    f.set_scratch(sm + p.sm.lamn, p.sm.jtv + p.Rt * p.d.ldn - p.sm.lamn);
  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt, s = p.s, nin = f.nin();
  const long long vec = (long long)p.B * N;
  const long long kst = (long long)Rt * ldn;
  T* u = state_buf(p, sm, 0);
  T* lam = state_buf(p, sm, 1);
  T* lamn = state_buf(p, sm, 2);
  T* w = state_buf(p, sm, 3);
  T* jtv = state_buf(p, sm, 4);
  T* ks = p.sm.ks >= 0 ? sm + p.sm.ks : p.scratch + tile * p.scratch_stride;
  T* Lam = ks + s * kst;
  T* mu = p.mu + tile * p.d.n_mu;

  loss_seed(p, lam, row0, Rv);
  __syncthreads();
  PhaseTimer pt(p.prof ? p.phase : nullptr);

  for (int pc = 0; pc < p.prog_len; ++pc) {
    const int4 op = p.prog[pc];
    const int n = op.y;
    const double t = p.ts[n], h = p.ts[n + 1] - p.ts[n];
    if (op.x == kOpReplay) {
      // start state: u0 | record u_next | stored solution  (restore semantics,
      // checkpointing.py:312-325); replay never reuses FSAL (integrators.py:363)
      const int src_kind = op.z >> 24, src = op.z & 0xffffff;
      const T* srcp = src_kind == kSrcU0 ? p.u0
                    : src_kind == kSrcSol ? p.sol + src * vec
                    : p.rec + ((long long)src * (s + 1) + s) * vec;
      load_rows(u, ldn, srcp, N, row0, Rv);
      __syncthreads();
      T* rec = p.rec + (long long)op.w * (s + 1) * vec;
      if constexpr (F::kOwnsStep)
        f.step(u, t, h, false, rec, row0, false);
      else
        rk_step_tile<T, F>(p, f, u, ks, t, h, false, rec, row0, Rv);
      pt.mark(kPhReplay);
      continue;
    }
    // REVERSE(n) from record buffer op.w: rk_adjoint_step (adjoint.py:67-94)
    obs_inject(p, lam, n + 1, row0, Rv);
    const T* rec = p.rec + (long long)op.w * (s + 1) * vec;
    if constexpr (F::kOwnsStep) {
      if (!f.reverse_step(lam, t, h, rec, row0, mu)) {
        if (threadIdx.x == 0) set_status(p.status, OB_ERR_GRADIENT_EXPLOSION, n);
        if constexpr (!NoEarlyExit<F>::value) {
          f.release();
          return;
        }
      }
      pt.mark(kPhVjp);
    } else {
      for (int idx = threadIdx.x; idx < kst; idx += blockDim.x) lamn[idx] = lam[idx];
      __syncthreads();
      for (int i = s - 1; i >= 0; --i) {
        if (p.skip_vjp & (1u << i)) {  // w_i == 0 exactly: Lam_i = 0 (still counted, B8)
          for (int idx = threadIdx.x; idx < kst; idx += blockDim.x) Lam[i * kst + idx] = T(0);
          continue;
        }
        // w_i = b_i lam_{n+1} + sum_{j>i, a_ji != 0} a_ji Lam_j   (pad rows stay 0)
        {
        for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
          const int o = (idx / N) * ldn + idx % N;
          T v = Num<T>::mul(T(p.b[i]), lam[o]);
  #pragma unroll
          for (int j0 = 0; j0 < OB_MAX_STAGES; j0 += F::kCombineBatch) {   // loads in flight first
            T lv[F::kCombineBatch];
  #pragma unroll
            for (int t = 0; t < F::kCombineBatch; ++t)
              lv[t] = (j0 + t > i && j0 + t < s) ? Lam[(j0 + t) * kst + o] : T(0);
  #pragma unroll
            for (int t = 0; t < F::kCombineBatch; ++t) {
              const double aji = (j0 + t > i && j0 + t < s) ? p.a[(j0 + t) * OB_MAX_STAGES + i] : 0.0;
              if (aji != 0.0) v = Num<T>::add(v, Num<T>::mul(T(aji), lv[t]));
            }
          }
          w[o] = v;
        }
        // stage state U_i into the field input (+ stage time)
        for (int idx = threadIdx.x; idx < Rv * nin; idx += blockDim.x) {
          const int r = idx / nin, j = idx % nin;
          f.put(r, j, rec[i * vec + (long long)(row0 + r) * N + j]);
        }
        }
        f.put_time(t + p.c[i] * h);
        __syncthreads();
        pt.mark(kPhElem);
        f.vjp(w, jtv, mu, h, Rv);
        pt.mark(kPhVjp);
        // Lam_i = h * jtv; lam_n += Lam_i  (scaled-VJP adapters return J^T (h w) directly)
        for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
          const int o = (idx / N) * ldn + idx % N;
          const T li = F::kScaledVjp ? jtv[o] : Num<T>::mul(T(h), jtv[o]);
          Lam[i * kst + o] = li;
          lamn[o] = Num<T>::add(lamn[o], li);
        }
        __syncthreads();
        pt.mark(kPhLam);
      }
      int bad = 0;
      for (int idx = threadIdx.x; idx < kst; idx += blockDim.x) {
        lam[idx] = lamn[idx];
        if (!Num<T>::finite(lamn[idx])) bad = 1;
      }
      if (__syncthreads_or(bad)) {  // AdjointState.check_finite (adjoint.py:42-44)
        if (threadIdx.x == 0) set_status(p.status, OB_ERR_GRADIENT_EXPLOSION, n);
        if constexpr (!NoEarlyExit<F>::value) {
          f.release();
          return;
        }
      }
    }
  }
  f.finish(mu);
  f.release();
  obs_inject(p, lam, 0, row0, Rv);
  store_rows(p.du0, N, lam, ldn, row0, Rv);
}

// Field protocol ops on a batch (integrators.py:53-102): eval / jvp / vjp / vjp_u.
// jvp needs the MLP tangent pass (MlpAdapter); other adapters reject mode 1 on the host.
template <typename T, class F>
__global__ void __launch_bounds__(kThreads, 1)
field_op_kernel(const __grid_constant__ RkParams<T> p, int mode, double t, const T* u,
                const T* w, T* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  zero_smem(sm, p.sm.wts >= 0 ? p.sm.wts : p.sm.total);
  const int tile = blockIdx.x;
  const int row0 = tile * p.R;
  const int Rv = max(0, min(p.R, p.B - row0));   // 0 on cluster-padding tiles
  MlpSmem<T> ms;
  Weights<T> W;
  setup_tile(p, sm, ms, W);
  F f(p, W, ms, sm, row0, Rv);
  const int N = p.d.N, ldn = p.d.ldn, nin = f.nin();
  T* wb = state_buf(p, sm, 3);
  T* res = state_buf(p, sm, 4);
  for (int idx = threadIdx.x; idx < Rv * nin; idx += blockDim.x) {
    const int r = idx / nin, j = idx % nin;
    f.put(r, j, u[(long long)(row0 + r) * N + j]);
  }
  f.put_time(t);
  if (mode != 0) load_rows(wb, ldn, w, N, row0, Rv);
  __syncthreads();
  if (mode == 0) {
    f.eval(res);
  } else if (mode == 1) {
    if constexpr (F::kHasJvp) f.jvp(wb, res);
  } else {
    T* mu = mode == 2 ? p.mu + tile * p.d.n_mu : nullptr;
    f.vjp(wb, res, mu, 1.0, Rv);
    f.finish(mu);   // adapters with device-resident / deferred parameter cotangents
  }
  f.release();
  store_rows(out, N, res, ldn, row0, Rv);
}

// ------------------------------------------------------ continuous adjoint
// Vanilla continuous-adjoint baseline (continuous_adjoint_solve, adjoint.py:294-331):
// the augmented reverse-time system y = (u, lambda, mu), dy/dtau = (-f, J^T lam,
// P^T lam) at t = tF - tau, integrated with the same explicit tableau and FSAL
// carry on the fixed tau grid p.ts.  mu never feeds back into the derivatives,
// so its stage derivatives go straight into the CTA's mu slot scaled by h b_i;
// with FSAL the reused stage's contribution is added when it is computed, with
// the next step's h b_0 folded into its scale.
template <typename T, class F>
__global__ void __launch_bounds__(kThreads, 1) cadj_kernel(const __grid_constant__ RkParams<T> p, double tF,
                                                           const T* dphi) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  zero_smem(sm, p.sm.wts >= 0 ? p.sm.wts : p.sm.total);
  const int tile = blockIdx.x;
  const int row0 = tile * p.R;
  const int Rv = max(0, min(p.R, p.B - row0));   // 0 on cluster-padding tiles
  MlpSmem<T> ms;
  Weights<T> W;
  setup_tile(p, sm, ms, W);
  F f(p, W, ms, sm, row0, Rv);
  // no split-K scratch here: the stage cotangent lives in the lamn slot

  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt, s = p.s, nin = f.nin();
  const long long kst = (long long)Rt * ldn;
  T* u = state_buf(p, sm, 0);
  T* lam = state_buf(p, sm, 1);
  T* li = state_buf(p, sm, 2);     // stage lambda (the VJP cotangent)
  T* jtv = state_buf(p, sm, 4);
  T* kU = p.sm.ks >= 0 ? sm + p.sm.ks : p.scratch + tile * p.scratch_stride;
  T* kL = kU + s * kst;
  T* mu = p.mu + tile * p.d.n_mu;
  load_rows(u, ldn, p.u_final, N, row0, Rv);
  load_rows(lam, ldn, dphi, N, row0, Rv);
  __syncthreads();
  for (int n = 0; n < p.n_steps; ++n) {
    const double tau = p.ts[n], h = p.ts[n + 1] - p.ts[n];
    const bool has_next = n + 1 < p.n_steps;
    const double hn = has_next ? p.ts[n + 2] - p.ts[n + 1] : 0.0;
    for (int i = 0; i < s; ++i) {
      if (i == 0 && p.fsal && n > 0) {   // k_first = k_last (integrators.py:210-211)
        for (int idx = threadIdx.x; idx < kst; idx += blockDim.x) {
          kU[idx] = kU[(s - 1) * kst + idx];
          kL[idx] = kL[(s - 1) * kst + idx];
        }
        __syncthreads();
        continue;
      }
      for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
        const int r = idx / N, j = idx % N, o = r * ldn + j;
        T vu = u[o], vl = lam[o];
        for (int q = 0; q < i; ++q) {
          const double aiq = p.a[i * OB_MAX_STAGES + q];
          if (aiq != 0.0) {
            vu = Num<T>::add(vu, Num<T>::mul(T(h * aiq), kU[q * kst + o]));
            vl = Num<T>::add(vl, Num<T>::mul(T(h * aiq), kL[q * kst + o]));
          }
        }
        if (j < nin) f.put(r, j, vu);
        li[o] = r < Rv ? vl : T(0);
      }
      f.put_time(tF - (tau + p.c[i] * h));
      __syncthreads();
      f.eval(kU + i * kst);                 // f(U_i); negated below
      double sc = h * p.b[i];
      if (i == s - 1 && p.fsal && has_next) sc += hn * p.b[0];
      f.vjp(li, jtv, sc != 0.0 ? mu : nullptr, sc, Rv);
      for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
        const int o = (idx / N) * ldn + idx % N;
        kU[i * kst + o] = -kU[i * kst + o];
        kL[i * kst + o] = jtv[o];
      }
      __syncthreads();
    }
    int bad = 0;
    for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
      const int r = idx / N, o = r * ldn + idx % N;
      T vu = u[o], vl = lam[o];
      for (int i = 0; i < s; ++i)
        if (p.b[i] != 0.0) {
          vu = Num<T>::add(vu, Num<T>::mul(T(h * p.b[i]), kU[i * kst + o]));
          vl = Num<T>::add(vl, Num<T>::mul(T(h * p.b[i]), kL[i * kst + o]));
        }
      u[o] = vu;
      lam[o] = vl;
      if (r < Rv && !(Num<T>::finite(vu) && Num<T>::finite(vl))) bad = 1;
    }
    if (__syncthreads_or(bad)) {   // explicit_rk_step overflow (integrators.py:219-220)
      if (threadIdx.x == 0) set_status(p.status, OB_ERR_INTEGRATION, n);
      return;
    }
  }
  store_rows(p.du0, N, lam, ldn, row0, Rv);
}

// --------------------------------------------------------------- helpers
// packed W_l: [nrow_l][ldw_l] row-major copy of theta's W_l, zero padded
template <typename T>
__global__ void pack_weights_kernel(const __grid_constant__ PackParams<T> p) {
  for (int l = 0; l < p.d.L; ++l) {
    const int nin = p.d.w[l], nout = p.d.w[l + 1], ldw = p.d.ldw[l];
    const T* Wl = p.theta + p.d.woff[l];
    T* dst = p.packed + p.d.pwoff[l];
    const long long n = (long long)p.d.nrow[l] * ldw;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
      const int r = (int)(i / ldw), k = (int)(i % ldw);
      dst[i] = (r < nout && k < nin) ? Wl[(long long)r * nin + k] : T(0);
    }
  }
}

// dtheta = sum over tiles of the padded mu slots, in tile order (deterministic),
// scattered back to the reference flat layout; loss likewise.
template <typename T>
__global__ void reduce_tiles_kernel(const __grid_constant__ Dims d, const T* mu, int tiles,
                                    long long np, T* dtheta, const double* loss_part,
                                    double inv_b, double* loss, const T* mu0) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < np;
       j += (long long)gridDim.x * blockDim.x) {
    int l = 0;
    while (l + 1 < d.L && j >= d.woff[l + 1]) ++l;
    long long src;
    if (j < d.boff[l] && d.conv) {   // theta [co][tap][cin] -> mu [co][tap][68]
      const long long q = j - d.woff[l];
      const int cin = d.conv_cin[l];
      const long long co = q / (9 * cin), r = q % (9 * cin);
      src = d.mwoff[l] + co * d.ldm[l] + (r / cin) * 68 + r % cin;
    } else if (j < d.boff[l]) {
      const long long q = j - d.woff[l];
      src = d.mwoff[l] + (q / d.w[l]) * d.ldm[l] + q % d.w[l];
    } else {
      src = d.mboff[l] + (j - d.boff[l]);
    }
    double acc = mu0 ? double(mu0[j]) : 0.0;   // terminal mu (adjoint_terminal), then the tiles
    for (int t = 0; t < tiles; ++t) acc += double(mu[t * d.n_mu + src]);
    dtheta[j] = T(acc);
  }
  if (loss && blockIdx.x == 0 && threadIdx.x == 0) {
    double acc = 0.0;
    for (int t = 0; t < tiles; ++t) acc += loss_part[t];
    *loss = acc * inv_b;
  }
}

// ------------------------------------------------------------ launchers
template <typename T>
cudaError_t launch_pack(const PackParams<T>& pp, cudaStream_t st) {
  pack_weights_kernel<T><<<148, 256, 0, st>>>(pp);
  return cudaGetLastError();
}

template <typename K, typename... A>
static cudaError_t launch_smem(K kf, int grid, size_t smem, cudaStream_t st, A... args) {
  cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kf<<<grid, kThreads, smem, st>>>(args...);
  return cudaGetLastError();
}

template <typename T, int LR, bool WS>
static cudaError_t launch_rk_lr(const RkParams<T>& p, int tiles, size_t smem, cudaStream_t st,
                                bool forward) {
  using F = MlpAdapter<T, LR, WS>;
  return forward ? launch_smem(rk_forward_kernel<T, F>, tiles, smem, st, p)
                 : launch_smem(rk_reverse_kernel<T, F>, tiles, smem, st, p);
}

// lane-row variants: LR 1 / 2 / 8 (tiles of <= 4, <= 8, <= 32 samples; fp64 tiles
// are capped at 8 rows by the planner)
template <typename T, bool WS>
cudaError_t launch_rk_ws(const RkParams<T>& p, int lr, int tiles, size_t smem, cudaStream_t st,
                         bool forward) {
  switch (lr) {
    case 1: return launch_rk_lr<T, 1, WS>(p, tiles, smem, st, forward);
    case 2: return launch_rk_lr<T, 2, WS>(p, tiles, smem, st, forward);
    default:
      if constexpr (sizeof(T) == 4) return launch_rk_lr<T, 8, WS>(p, tiles, smem, st, forward);
      return cudaErrorInvalidConfiguration;
  }
}

template <typename T, bool WS>
cudaError_t launch_cadj_ws(const RkParams<T>& p, int lr, int tiles, size_t smem, double tF,
                           const T* dphi, cudaStream_t st) {
  switch (lr) {
    case 1: return launch_smem(cadj_kernel<T, MlpAdapter<T, 1, WS>>, tiles, smem, st, p, tF, dphi);
    case 2: return launch_smem(cadj_kernel<T, MlpAdapter<T, 2, WS>>, tiles, smem, st, p, tF, dphi);
    default:
      if constexpr (sizeof(T) == 4)
        return launch_smem(cadj_kernel<T, MlpAdapter<T, 8, WS>>, tiles, smem, st, p, tF, dphi);
      return cudaErrorInvalidConfiguration;
  }
}

template <typename T, bool WS>
cudaError_t launch_field_ws(const RkParams<T>& p, int lr, int tiles, size_t smem, int mode,
                            double t, const T* u, const T* w, T* out, cudaStream_t st) {
  switch (lr) {
    case 1:
      return launch_smem(field_op_kernel<T, MlpAdapter<T, 1, WS>>, tiles, smem, st, p, mode, t, u, w, out);
    case 2:
      return launch_smem(field_op_kernel<T, MlpAdapter<T, 2, WS>>, tiles, smem, st, p, mode, t, u, w, out);
    default:
      if constexpr (sizeof(T) == 4)
        return launch_smem(field_op_kernel<T, MlpAdapter<T, 8, WS>>, tiles, smem, st, p, mode, t, u,
                           w, out);
      return cudaErrorInvalidConfiguration;
  }
}

template <typename T>
cudaError_t launch_reduce(const Dims& d, const T* mu, int tiles, long long np, T* dtheta,
                          const double* lp, double inv_b, double* loss, cudaStream_t st,
                          const T* mu0) {
  const int blocks = (int)std::min<long long>((np + 255) / 256, 148 * 4);
  reduce_tiles_kernel<T><<<blocks > 0 ? blocks : 1, 256, 0, st>>>(d, mu, tiles, np, dtheta, lp,
                                                                    inv_b, loss, mu0);
  return cudaGetLastError();
}

}  // namespace ob
