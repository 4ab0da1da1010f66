// adaptive_impl.cuh -- adaptive explicit stepping with per-sample step sizes
// (SURVEY 8f row 1): the adaptive branch of integrate (integrators.py:294-349)
// and of forward_pass (adjoint.py:162-186), then the discrete adjoint over each
// sample's frozen grid (backward_sweep, adjoint.py:235-253).
//
// One CTA keeps its tile of samples for the whole sweep, as the fixed-step
// kernels do, but every row runs its own controller: per-row t, h, previous
// error, FSAL carry (k_last after an accept, ks[0] after a reject), step
// counters and observation interval.  Trial steps run in lockstep over the
// rows still integrating, each with its own h and stage times; finished rows
// ride along with h = 0 and write nothing.  Accepted steps commit their record
// into slot n of the per-step record buffer (store_all: [cap][s+1][B][N];
// store_solutions: the step-start state into [cap][B][N] plus a two-slot
// ping-pong record holding the final step) and (t_n, h_n) into the grid.  The
// reverse kernel walks every row's own grid backwards in lockstep (row r
// reverses its step n_r-1-i at iteration i), replaying from stored solutions
// where the policy says so, with the per-row step size folded into the
// cotangent (J^T (h w) = h J^T w) so one tile-wide VJP serves rows with
// different h.
#pragma once

#include "rk_impl.cuh"

namespace ob {

constexpr int kAdMaxRows = 32;

struct AdRow {
  double t, h, errp, enorm, tstep, hstep;
  int carry;      // k_first for the next trial: 0 none, 1 ks[s-1] (accepted), 2 ks[0] (rejected)
  int seg, taken, nacc, rej, nfe, rec;
  int done, act, acc, fin, bad, slot, m;
};

// One lockstep trial step of the rows with act set, from u: stages with per-row
// (t_r, h_r) and the candidate un (integrators.py:196-222); with q, also
// q = (err / scale)^2 per element (err = sum_i (h d_i) k_i, d = b - b_emb,
// integrators.py:312-317, :247-249) and the overflow flag.  ks: [s][Rt][ldn];
// ktmp: [Rt][ldn].  rec_slot(r): record base ([s+1][B][N]) for row r or null.
template <typename T, class F, class Slot>
OB_DEV void ad_trial(const RkParams<T>& p, F& f, AdRow* rs, const T* u, T* un, T* q, T* ks,
                     T* ktmp, int row0, int Rv, Slot rec_slot) {
  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt, s = p.s, nin = f.nin();
  const long long kst = (long long)Rt * ldn, vec = (long long)p.B * N;
  for (int i = 0; i < s; ++i) {
    for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
      const int r = idx / N, j = idx % N;
      const bool a = r < Rv && rs[r].act;
      const double h = a ? rs[r].h : 0.0;
      T v = u[r * ldn + j];
      for (int qq = 0; qq < i; ++qq) {
        const double aiq = p.a[i * OB_MAX_STAGES + qq];
        if (aiq != 0.0) v = Num<T>::add(v, Num<T>::mul(T(h * aiq), ks[qq * kst + r * ldn + j]));
      }
      if (j < nin) f.put(r, j, v);
      if (a) {
        T* rec = rec_slot(r);
        if (rec) rec[i * vec + (long long)(row0 + r) * N + j] = v;
      }
    }
    for (int r = threadIdx.x; r < Rt; r += blockDim.x) {
      const bool a = r < Rv && rs[r].act;
      f.put_time_row(r, a ? rs[r].t + p.c[i] * rs[r].h : 0.0);
    }
    __syncthreads();
    if (i == 0) {
      // k_first reuse (integrators.py:210-211): evaluate only if some row has none
      bool need = false;
      for (int r = 0; r < Rv; ++r) need = need || (rs[r].act && rs[r].carry == 0);
      if (need) f.eval(ktmp);
      for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
        const int r = idx / N, j = idx % N, o = r * ldn + j;
        const int c = r < Rv ? rs[r].carry : 0;
        if (c == 1) ks[o] = ks[(s - 1) * kst + o];
        else if (c == 0) ks[o] = need ? ktmp[o] : T(0);
      }
      __syncthreads();
    } else {
      f.eval(ks + i * kst);
    }
  }
  for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
    const int r = idx / N, o = r * ldn + idx % N;
    const bool a = r < Rv && rs[r].act;
    const double h = a ? rs[r].h : 0.0;
    T v = u[o];
    for (int i = 0; i < s; ++i)
      if (p.b[i] != 0.0) v = Num<T>::add(v, Num<T>::mul(T(h * p.b[i]), ks[i * kst + o]));
    un[o] = v;
    if (q) {
      T e = T(0);
      for (int i = 0; i < s; ++i)
        if (p.ad_d[i] != 0.0) e = Num<T>::add(e, Num<T>::mul(T(h * p.ad_d[i]), ks[i * kst + o]));
      const double sc = p.ad_abstol + p.ad_reltol * fmax(fabs(double(u[o])), fabs(double(v)));
      const double z = double(e) / sc;
      q[o] = T(z * z);
      if (a && !Num<T>::finite(v)) atomicOr(&rs[r].bad, 1);
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------ forward
template <typename T, class F>
__global__ void __launch_bounds__(kThreads, 1) ad_forward_kernel(const __grid_constant__ RkParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ AdRow rs[kAdMaxRows];
  __shared__ int any_active;
  T* sm = reinterpret_cast<T*>(smem_raw);
  zero_smem(sm, p.sm.wts >= 0 ? p.sm.wts : p.sm.total);
  const int tile = blockIdx.x;
  const int row0 = tile * p.R;
  const int Rv = min(p.R, p.B - row0);
  MlpSmem<T> ms;
  Weights<T> W;
  setup_tile(p, sm, ms, W);
  F f(p, W, ms, sm, row0, Rv);
  if (p.sm.u >= 0) f.set_scratch(sm + p.sm.lamn, p.sm.jtv + p.Rt * p.d.ldn - p.sm.lamn);
  T* u = state_buf(p, sm, 0);
  T* un = state_buf(p, sm, 1);
  T* q = state_buf(p, sm, 3);
  T* ks = p.scratch + tile * p.scratch_stride;
  const int N = p.d.N, ldn = p.d.ldn, s = p.s;
  const long long kst = (long long)p.Rt * ldn, vec = (long long)p.B * N;
  T* ktmp = ks + s * kst;
  const bool store_all = p.ad_policy == 0;

  load_rows(u, ldn, p.u0, N, row0, Rv);
  __syncthreads();
  int bad = 0;
  for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x)
    if (!Num<T>::finite(u[(idx / N) * ldn + idx % N])) bad = 1;
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) set_status(p.status, OB_ERR_VALUE, -1);
    return;
  }
  if (threadIdx.x < kAdMaxRows) {
    AdRow R{};
    R.t = p.ad_pts[0];
    R.h = fmin(p.ad_hinit, p.ad_pts[1] - p.ad_pts[0]);
    R.errp = 1.0;
    R.done = threadIdx.x >= Rv;
    rs[threadIdx.x] = R;
  }
  if (p.obs_k && p.ad_obs0) {   // observation at t0: the initial state (adjoint.py:180)
    store_rows(p.preds, N, u, ldn, row0, Rv);
    for (int r = threadIdx.x; r < Rv; r += blockDim.x) p.obs_step[row0 + r] = 0;
  }
  __syncthreads();
  for (;;) {
    // ---- prologue (integrators.py:308-311)
    if (threadIdx.x == 0) any_active = 0;
    __syncthreads();
    if (threadIdx.x < Rv) {
      AdRow& R = rs[threadIdx.x];
      R.act = R.acc = R.bad = R.fin = 0;
      if (!R.done) {
        if (R.taken >= p.ad_max_steps) {
          set_status(p.status, OB_ERR_STIFFNESS, 2 * (row0 + threadIdx.x) + 1);
          R.done = 1;
        } else {
          R.h = fmin(R.h, p.ad_pts[R.seg + 1] - R.t);
          R.act = 1;
          atomicOr(&any_active, 1);
        }
      }
    }
    __syncthreads();
    if (!any_active || *(volatile int*)p.status != 0) break;
    // ---- trial: store_all records into the row's next slot, store_solutions
    // into the ping-pong slot (nacc & 1)
    ad_trial<T, F>(p, f, rs, u, un, q, ks, ktmp, row0, Rv, [&](int r) -> T* {
      const int slot = store_all ? rs[r].nacc : (rs[r].nacc & 1);
      return p.rec + (long long)slot * (s + 1) * vec;
    });
    // ---- per-row WRMS norm, max(., 1e-10) (warp per row, fixed reduction order)
    for (int r = warp_id(); r < Rv; r += n_warps()) {
      double acc = 0.0;
      for (int j = lane_id(); j < N; j += 32) acc += double(q[r * ldn + j]);
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane_id() == 0) rs[r].enorm = fmax(sqrt(acc / N), 1e-10);
    }
    __syncthreads();
    // ---- controller (integrators.py:312-349), one thread per row
    if (threadIdx.x < Rv && rs[threadIdx.x].act) {
      AdRow& R = rs[threadIdx.x];
      const int row = row0 + threadIdx.x;
      R.nfe += s - (R.carry != 0 ? 1 : 0);
      R.taken += 1;
      if (R.bad) {   // overflow inside the trial: rejection, h * 0.2 (:318-327)
        R.rej += 1;
        R.carry = 0;
        if (R.h <= p.ad_hmin * (1 + 1e-12)) {
          set_status(p.status, OB_ERR_STIFFNESS, 2 * row);
          R.done = 1;
        }
        R.h = fmax(R.h * 0.2, p.ad_hmin);
      } else {
        double factor;
        if (R.enorm <= 1.0) {
          if (R.nacc >= p.ad_cap) {
            set_status(p.status, OB_ERR_UNSUPPORTED, row);
            R.done = 1;
          }
          R.acc = 1;
          R.slot = R.nacc;
          R.tstep = R.t;
          R.hstep = R.h;
          R.nacc += 1;
          R.t = R.t + R.h;
          R.carry = p.fsal ? 1 : 0;
          factor = p.ad_safety * pow(R.enorm, -p.ad_alpha) * pow(R.errp, p.ad_beta);
          R.errp = R.enorm;
          const double b = p.ad_pts[R.seg + 1];
          R.fin = !(R.t < b - 1e-14 * fmax(1.0, fabs(b)));
        } else {
          R.rej += 1;
          R.carry = 2;
          if (R.h <= p.ad_hmin * (1 + 1e-12)) {
            set_status(p.status, OB_ERR_STIFFNESS, 2 * row);
            R.done = 1;
          }
          factor = fmin(p.ad_safety * pow(R.enorm, -p.ad_alpha), 1.0);
        }
        factor = fmin(5.0, fmax(0.2, factor));
        R.h = fmin(fmax(R.h * factor, p.ad_hmin), p.ad_hmax);
      }
    }
    __syncthreads();
    if (*(volatile int*)p.status != 0) break;
    // ---- commit accepted rows: records, solutions, grid, u <- u_next
    for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
      const int r = idx / N, j = idx % N, o = r * ldn + j;
      if (!rs[r].acc) continue;
      const int n = rs[r].slot;
      const long long g = (long long)(row0 + r) * N + j;
      if (store_all) {
        p.rec[((long long)n * (s + 1) + s) * vec + g] = un[o];
      } else {
        p.rec[((long long)(n & 1) * (s + 1) + s) * vec + g] = un[o];
        p.sol[(long long)n * vec + g] = u[o];
      }
      u[o] = un[o];
    }
    if (threadIdx.x < Rv && rs[threadIdx.x].acc) {
      const AdRow& R = rs[threadIdx.x];
      double* gr = p.ad_grid + ((long long)(row0 + threadIdx.x) * p.ad_cap + R.slot) * 2;
      gr[0] = R.tstep;
      gr[1] = R.hstep;
    }
    __syncthreads();
    // ---- interval ends: observation capture, next interval (adjoint.py:176-183)
    bool any_fin = false;
    for (int r = 0; r < Rv; ++r) any_fin = any_fin || rs[r].fin;
    if (any_fin) {
      for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
        const int r = idx / N, j = idx % N;
        if (!rs[r].fin) continue;
        const int k = p.obs_k ? p.ad_seg_obs[rs[r].seg] : -1;
        if (k >= 0) p.preds[((long long)k * p.B + row0 + r) * N + j] = u[r * ldn + j];
      }
      __syncthreads();
      if (threadIdx.x < Rv && rs[threadIdx.x].fin) {
        AdRow& R = rs[threadIdx.x];
        const int k = p.obs_k ? p.ad_seg_obs[R.seg] : -1;
        if (k >= 0) p.obs_step[(long long)k * p.B + row0 + threadIdx.x] = R.nacc;
        R.seg += 1;
        if (R.seg >= p.ad_nseg) {
          R.done = 1;
        } else {   // integrate restarts on the next interval (integrators.py:302-307)
          R.t = p.ad_pts[R.seg];
          R.h = fmin(p.ad_hinit, p.ad_pts[R.seg + 1] - p.ad_pts[R.seg]);
          R.errp = 1.0;
          R.carry = 0;
          R.taken = 0;
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x < Rv) {
    const AdRow& R = rs[threadIdx.x];
    const int row = row0 + threadIdx.x;
    p.ad_nacc[row] = R.nacc;
    int* st = p.sample_stats + (long long)row * OB_NSTATS;
    st[OB_STAT_NFE_F] = R.nfe;
    st[OB_STAT_ACCEPTED] = R.nacc;
    st[OB_STAT_REJECTED] = R.rej;
  }
  if (*(volatile int*)p.status != 0) return;
  store_rows(p.u_final, N, u, ldn, row0, Rv);
  __syncthreads();
  loss_partial(p, u, row0, Rv, tile);
}

// ------------------------------------------------------------------ reverse
// lambda += seeds of the observations at boundary m_r + 1 of each active row
// (m_r = -1: boundary 0 after the sweep)
template <typename T>
OB_DEV void ad_inject(const RkParams<T>& p, const AdRow* rs, T* lam, int row0, int Rv, bool final_) {
  if (!p.obs_k) return;
  const int N = p.d.N, ldn = p.d.ldn;
  for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
    const int r = idx / N, j = idx % N;
    if (!final_ && !rs[r].act) continue;
    const int bnd = final_ ? 0 : rs[r].m + 1;
    for (int k = 0; k < p.n_obs; ++k) {
      if (p.obs_step[(long long)k * p.B + row0 + r] != bnd) continue;
      lam[r * ldn + j] = T(double(lam[r * ldn + j]) + obs_seed(p, k, row0 + r, j));
    }
  }
  __syncthreads();
}

template <typename T, class F>
__global__ void __launch_bounds__(kThreads, 1) ad_reverse_kernel(const __grid_constant__ RkParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ AdRow rs[kAdMaxRows];
  __shared__ int maxn;
  T* sm = reinterpret_cast<T*>(smem_raw);
  if (*(volatile int*)p.status != 0) return;
  zero_smem(sm, p.sm.wts >= 0 ? p.sm.wts : p.sm.total);
  const int tile = blockIdx.x;
  const int row0 = tile * p.R;
  const int Rv = min(p.R, p.B - row0);
  MlpSmem<T> ms;
  Weights<T> W;
  setup_tile(p, sm, ms, W);
  F f(p, W, ms, sm, row0, Rv);
  if (p.sm.u >= 0) f.set_scratch(sm + p.sm.lamn, p.sm.jtv + p.Rt * p.d.ldn - p.sm.lamn);
  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt, s = p.s, nin = f.nin();
  const long long vec = (long long)p.B * N, kst = (long long)Rt * ldn;
  T* u = state_buf(p, sm, 0);
  T* lam = state_buf(p, sm, 1);
  T* lamn = state_buf(p, sm, 2);
  T* w = state_buf(p, sm, 3);
  T* jtv = state_buf(p, sm, 4);
  T* ks = p.scratch + tile * p.scratch_stride;
  T* Lam = ks + s * kst;
  T* mu = p.mu + tile * p.d.n_mu;
  const bool store_all = p.ad_policy == 0;

  if (threadIdx.x == 0) maxn = 0;
  __syncthreads();
  if (threadIdx.x < kAdMaxRows) {
    AdRow R{};
    if (threadIdx.x < Rv) {
      R.nacc = p.ad_nacc[row0 + threadIdx.x];
      atomicMax(&maxn, R.nacc);
    }
    rs[threadIdx.x] = R;
  }
  loss_seed(p, lam, row0, Rv);
  __syncthreads();
  const int iters = maxn;
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x < kAdMaxRows) {
      AdRow& R = rs[threadIdx.x];
      R.m = R.nacc - 1 - it;
      R.act = threadIdx.x < Rv && R.m >= 0;
      R.carry = 0;   // replay never reuses FSAL (integrators.py:363)
      if (R.act) {
        const double* gr = p.ad_grid + ((long long)(row0 + threadIdx.x) * p.ad_cap + R.m) * 2;
        R.t = gr[0];
        R.h = gr[1];
        R.rec = store_all ? R.m : (R.m == R.nacc - 1 ? (R.m & 1) : 2);
      } else {
        R.t = R.h = 0.0;
      }
    }
    __syncthreads();
    ad_inject(p, rs, lam, row0, Rv, false);
    if (!store_all) {
      // replay the rows whose step is not the held-out final record (integrators.py:352-368)
      bool any = false;
      for (int r = 0; r < Rv; ++r) any = any || (rs[r].act && rs[r].rec == 2);
      if (any) {
        __syncthreads();
        if (threadIdx.x < Rv) {
          AdRow& R = rs[threadIdx.x];
          R.acc = R.act;                    // park the adjoint participation flag
          R.act = R.act && R.rec == 2;
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
          const int r = idx / N, j = idx % N;
          u[r * ldn + j] = (r < Rv && rs[r].act)
                               ? p.sol[(long long)rs[r].m * vec + (long long)(row0 + r) * N + j]
                               : T(0);
        }
        __syncthreads();
        ad_trial<T, F>(p, f, rs, u, jtv, nullptr, ks, Lam, row0, Rv, [&](int) -> T* {
          return p.rec + 2LL * (s + 1) * vec;
        });
        if (threadIdx.x < Rv) {
          AdRow& R = rs[threadIdx.x];
          if (R.act) {
            R.nfe += s;
            R.rej += 1;   // steps recomputed
          }
          R.act = R.acc;
        }
        __syncthreads();
      }
    }
    // ---- rk_adjoint_step on every active row (adjoint.py:67-94)
    for (int idx = threadIdx.x; idx < kst; idx += blockDim.x) lamn[idx] = lam[idx];
    __syncthreads();
    for (int i = s - 1; i >= 0; --i) {
      if (p.skip_vjp & (1u << i)) {
        for (int idx = threadIdx.x; idx < kst; idx += blockDim.x) Lam[i * kst + idx] = T(0);
        continue;
      }
      for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
        const int r = idx / N, j = idx % N, o = r * ldn + j;
        const bool a = r < Rv && rs[r].act;
        T v = Num<T>::mul(T(p.b[i]), lam[o]);
        for (int jj = i + 1; jj < s; ++jj) {
          const double aji = p.a[jj * OB_MAX_STAGES + i];
          if (aji != 0.0) v = Num<T>::add(v, Num<T>::mul(T(aji), Lam[jj * kst + o]));
        }
        w[o] = a ? Num<T>::mul(T(rs[r].h), v) : T(0);   // h folded into the cotangent
        if (j < nin) {
          T x = T(0);
          if (a) {
            const T* rec = p.rec + (long long)rs[r].rec * (s + 1) * vec;
            x = rec[i * vec + (long long)(row0 + r) * N + j];
          }
          f.put(r, j, x);
        }
      }
      for (int r = threadIdx.x; r < Rt; r += blockDim.x) {
        const bool a = r < Rv && rs[r].act;
        f.put_time_row(r, a ? rs[r].t + p.c[i] * rs[r].h : 0.0);
      }
      __syncthreads();
      f.vjp(w, jtv, mu, 1.0, Rv);
      for (int idx = threadIdx.x; idx < Rt * N; idx += blockDim.x) {
        const int o = (idx / N) * ldn + idx % N;
        Lam[i * kst + o] = jtv[o];
        lamn[o] = Num<T>::add(lamn[o], jtv[o]);
      }
      __syncthreads();
    }
    int bad = 0;
    for (int idx = threadIdx.x; idx < kst; idx += blockDim.x) {
      lam[idx] = lamn[idx];
      if (!Num<T>::finite(lamn[idx])) bad = 1;
    }
    if (__syncthreads_or(bad)) {  // AdjointState.check_finite (adjoint.py:42-44)
      if (threadIdx.x == 0) set_status(p.status, OB_ERR_GRADIENT_EXPLOSION, it);
      return;
    }
  }
  ad_inject(p, rs, lam, row0, Rv, true);
  store_rows(p.du0, N, lam, ldn, row0, Rv);
  if (threadIdx.x < Rv) {
    const AdRow& R = rs[threadIdx.x];
    int* st = p.sample_stats + (long long)(row0 + threadIdx.x) * OB_NSTATS;
    st[OB_STAT_NFE_F] += R.nfe;
    st[OB_STAT_NFE_B] = s * R.nacc;
    st[OB_STAT_RECOMPUTED] = R.rej;
  }
}

template <typename T, int LR, bool WS>
static cudaError_t launch_ad_lr(const RkParams<T>& p, int tiles, size_t smem, cudaStream_t st,
                                bool forward) {
  using F = MlpAdapter<T, LR, WS>;
  return forward ? launch_smem(ad_forward_kernel<T, F>, tiles, smem, st, p)
                 : launch_smem(ad_reverse_kernel<T, F>, tiles, smem, st, p);
}

template <typename T, bool WS>
cudaError_t launch_adaptive_ws(const RkParams<T>& p, int lr, int tiles, size_t smem,
                               cudaStream_t st, bool forward) {
  switch (lr) {
    case 1: return launch_ad_lr<T, 1, WS>(p, tiles, smem, st, forward);
    case 2: return launch_ad_lr<T, 2, WS>(p, tiles, smem, st, forward);
    default:
      if constexpr (sizeof(T) == 4) return launch_ad_lr<T, 8, WS>(p, tiles, smem, st, forward);
      return cudaErrorInvalidConfiguration;
  }
}

}  // namespace ob
