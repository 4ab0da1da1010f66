// theta_impl.cuh -- persistent theta-method (backward Euler / Crank-Nicolson)
// forward and discrete-adjoint kernels with batched matrix-free Newton-GMRES.
//
// Every sample of a CTA tile runs its own Newton iteration and its own
// restarted GMRES(m) exactly as linalg.py:37-142 prescribes (x0 = 0, modified
// Gram-Schmidt Arnoldi, Givens rotations on the fly, ||r|| <= tol*||rhs||,
// maxit counting Arnoldi steps across restarts, final residual check).  The
// samples advance in lockstep, one operator application per lockstep
// iteration: each sample feeds the vector its own state machine needs
// (x at a cycle start or final check, Q_k inside a cycle) and finished samples
// feed zeros and stop counting.  Operator products go through the cached
// linearisation (JVP for the forward Newton system, transposed VJP for the
// adjoint system), computed once per Newton iterate instead of once per
// product as the reference's MlpField does (integrators.py:88-102).
// Dot products are warp butterfly reductions (deterministic).
#pragma once

#include "rk_impl.cuh"

namespace ob {

enum { kPhTop = 0, kPhCycle = 1, kPhFinal = 2, kPhDone = 3, kPhFail = 4 };
constexpr int kMaxTileRows = 32;
constexpr int kMgsV = 4;   // state elements per lane in the register MGS path (N <= 128)

struct SampleState {
  int phase, total, k, used, breakdown;
  double tol;
};

// per-tile theta-method context (shared memory vectors + per-sample state)
template <typename T>
struct ThetaCtx {
  T *base, *xk, *rv, *gx, *vin, *vout, *fb, *rhs;
  SampleState* st;        // [kMaxTileRows]
  int* cnt;               // [kMaxTileRows][OB_NSTATS]
  unsigned char* active;  // [kMaxTileRows]
  double* rn;             // [kMaxTileRows]
  int* flag;              // [1] block-wide scratch
};

// Operator A v = v - (h*theta) * J v  (forward Newton system, integrators.py:236-237)
// or A v = v - (h*theta) * J^T v  (adjoint system, adjoint.py:112-113), J from
// the linearisation cached in the tile.
template <typename T, int LR, bool WS>
struct ThetaOp {
  const RkParams<T>& p;
  MlpTile<T, LR, WS>& mt;
  T hth;
  bool transpose;
  T* tmp;
  OB_DEV void apply(const T* vin, T* vout) {
    const int N = p.d.N, ldn = p.d.ldn;
    if (transpose) mt.vjp_keep(vin, ldn, p.Rt, tmp, ldn, nullptr, T(0));
    else mt.jvp(vin, ldn, tmp, ldn);
    for (int i = threadIdx.x; i < p.Rt * N; i += blockDim.x) {
      const int o = (i / N) * ldn + i % N, j = i % N;
      T jv = tmp[o];
      if (p.field_kind == OB_FIELD_STIFF)
        jv = Num<T>::add(Num<T>::mul(p.diag[j], vin[o]), Num<T>::mul(p.out_scale, jv));
      vout[o] = Num<T>::add(vin[o], -Num<T>::mul(hth, jv));
    }
    __syncthreads();
  }
  template <class Vote>
  OB_DEV bool apply_any(int any, const T* vin, T* vout, Vote& vote) {
    if (!vote.any(any)) return false;
    apply(vin, vout);
    return true;
  }
};

// block-wide votes of the lockstep loops (the cluster kernels vote across their CTAs)
struct CtaVote {
  OB_DEV int any(int v) const { return __syncthreads_or(v); }
  OB_DEV int all(int v) const { return __syncthreads_and(v); }
};

// Batched restarted GMRES(m) on the tile: solves A x_r = rhs_r for every row r
// with active[r]; inactive rows are left untouched.  cnt_col: stats column to
// add the Arnoldi steps to; nfe_col: stats column counting operator calls.
// Returns false if some active sample failed (ConvergenceError).
template <typename T, class Op, class Vote = CtaVote>
OB_DEV bool gmres_tile(const RkParams<T>& p, Op& op, ThetaCtx<T>& c, const T* rhs, T* x,
                       int Rv, T* kry, int cnt_col, int nfe_col, Vote vote = Vote()) {
  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt;
  const int m = min(p.gmres_restart, N);
  const long long qs = (long long)(m + 1) * ldn, hs = (long long)(m + 1) * m;
  // per-sample Krylov workspace, one block per valid row (p.R rows per tile)
  const int Rk = p.R;
  T* Qb = kry;
  T* Hb = Qb + (long long)Rk * qs;
  T* csb = Hb + (long long)Rk * hs;
  T* snb = csb + (long long)Rk * m;
  T* gb = snb + (long long)Rk * m;
  T* yb = gb + (long long)Rk * (m + 1);
  const int w = warp_id();
  if (w < Rv) {
    // warp-uniform local copy of the sample state; lane 0 writes it back
    SampleState S = c.st[w];
    S.total = 0;
    S.k = S.used = S.breakdown = 0;
    if (!c.active[w]) {
      S.phase = kPhDone;
    } else {
      const T* b = rhs + w * ldn;
      const T bn = sqrt(warp_dot(b, b, N));        // ||rhs|| (linalg.py:45)
      for (int j = lane_id(); j < N; j += 32) x[w * ldn + j] = T(0);
      if (bn == T(0)) {
        S.phase = kPhDone;                             // (linalg.py:46-47)
      } else {
        S.tol = double(p.gmres_tol) * double(bn);
        S.phase = kPhTop;
      }
    }
    __syncwarp();
    if (lane_id() == 0) c.st[w] = S;
  }
  __syncthreads();
  bool ok = true;
  PhaseTimer pt(p.prof ? p.phase : nullptr);
  for (;;) {
    // operator input of every row from its own state machine
    int any = 0;
    for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
      const int r = i / N, j = i % N;
      const int ph = r < Rv ? c.st[r].phase : kPhDone;
      T v = T(0);
      if (ph == kPhTop || ph == kPhFinal) v = x[r * ldn + j];
      else if (ph == kPhCycle) v = Qb[r * qs + (long long)c.st[r].k * ldn + j];
      if (ph <= kPhFinal) any = 1;
      c.vin[r * ldn + j] = v;
    }
    pt.mark(14);   // operator-input assembly
    // "is any sample of the (cluster) tile still iterating?" and the operator product: the
    // cluster operator carries the vote on its all-gather barrier
    if (!op.apply_any(any, c.vin, c.vout, vote)) break;
    pt.mark(kPhGmres);   // operator products (JVP / transposed VJP)
    if (w < Rv) {
      SampleState S = c.st[w];           // warp-uniform copy, written back by lane 0
      const int lane = lane_id();
      const T* b = rhs + w * ldn;
      T* vo = c.vout + w * ldn;
      T* Q = Qb + w * qs;
      T* H = Hb + w * hs;
      T* cs = csb + w * m;
      T* sn = snb + w * m;
      T* g = gb + w * (m + 1);
      T* y = yb + w * m;
      if (S.phase <= kPhFinal && lane == 0) c.cnt[w * OB_NSTATS + nfe_col] += 1;
      if (S.phase == kPhTop || S.phase == kPhFinal) {
        // r = rhs - A x (linalg.py:52 / :107)
        for (int j = lane; j < N; j += 32) vo[j] = Num<T>::add(b[j], -vo[j]);
        __syncwarp();
        const T beta = sqrt(warp_dot(vo, vo, N));
        if (double(beta) <= S.tol) {
          S.phase = kPhDone;
        } else if (S.phase == kPhFinal) {
          S.phase = kPhFail;                            // linalg.py:111-114
        } else if (S.total >= p.gmres_maxit) {
          S.phase = kPhFinal;                           // linalg.py:56-57 -> final check
        } else {
          for (int j = lane; j < N; j += 32) Q[j] = vo[j] / beta;
          if (lane == 0) {
            g[0] = beta;
            for (int i = 1; i <= m; ++i) g[i] = T(0);
          }
          S.k = 0;
          S.used = 0;
          S.breakdown = 0;
          S.phase = kPhCycle;
        }
      } else if (S.phase == kPhCycle) {
        const int k = S.k;
        S.total += 1;
        // Column k of H, the rotations and (at a cycle end) y are worked on in this row's
        // slice of the operator-input buffer, which is dead until the next lockstep
        // iteration: the Krylov workspace lives in global memory (L2: ~800 cycles per
        // dependent access, and stores do not allocate in L1), and lane 0's serial Givens
        // chain read its own fresh stores back from there.  Needs 96 doubles per row.
        const bool fast = ldn >= 96 && m <= 31;
        T* scr = c.vin + w * ldn;
        // modified Gram-Schmidt (linalg.py:73-75).  The operator output stays in registers
        // (kMgsV elements per lane) and the next basis vector is loaded while the current
        // projection reduces (the basis lives in L2); same operation order as warp_dot.
        if (N <= 32 * kMgsV) {
          T v[kMgsV], q[kMgsV], qn[kMgsV];
#pragma unroll
          for (int e = 0; e < kMgsV; ++e) {
            const int j = lane + 32 * e;
            v[e] = j < N ? vo[j] : T(0);
            q[e] = j < N ? Q[j] : T(0);
          }
          for (int i = 0; i <= k; ++i) {
            if (i < k) {
              const T* qx = Q + (long long)(i + 1) * ldn;
#pragma unroll
              for (int e = 0; e < kMgsV; ++e) qn[e] = lane + 32 * e < N ? qx[lane + 32 * e] : T(0);
            }
            T sdot = T(0);
#pragma unroll
            for (int e = 0; e < kMgsV; ++e)
              if (lane + 32 * e < N) sdot = Num<T>::fma(v[e], q[e], sdot);
            const T hik = warp_sum(sdot);
#pragma unroll
            for (int e = 0; e < kMgsV; ++e)
              if (lane + 32 * e < N) v[e] = Num<T>::add(v[e], -Num<T>::mul(hik, q[e]));
            if (lane == 0) {
              if (fast) scr[i] = hik;
              else H[i * m + k] = hik;
            }
#pragma unroll
            for (int e = 0; e < kMgsV; ++e) q[e] = qn[e];
          }
#pragma unroll
          for (int e = 0; e < kMgsV; ++e)
            if (lane + 32 * e < N) vo[lane + 32 * e] = v[e];
          __syncwarp();
        } else {
          for (int i = 0; i <= k; ++i) {
            const T* qi = Q + (long long)i * ldn;
            const T hik = warp_dot(vo, qi, N);
            for (int j = lane; j < N; j += 32) vo[j] = Num<T>::add(vo[j], -Num<T>::mul(hik, qi[j]));
            __syncwarp();
            if (lane == 0) {
              if (fast) scr[i] = hik;
              else H[i * m + k] = hik;
            }
          }
        }
        const T hn = sqrt(warp_dot(vo, vo, N));
        if (lane == 0) {
          if (fast) scr[k + 1] = hn;
          else H[(k + 1) * m + k] = hn;
        }
        if (double(hn) > 1e-300) {
          T* qn = Q + (long long)(k + 1) * ldn;
          for (int j = lane; j < N; j += 32) qn[j] = vo[j] / hn;
        } else {
          S.breakdown = 1;                              // linalg.py:79-80
        }
        T gk1;   // g[k + 1] after this step's rotation (every lane)
        if (fast) {
          // Givens rotations on the fly (linalg.py:81-93): the k earlier rotations are
          // fetched by k lanes at once, the chain itself runs on lane 0 out of the scratch
          if (lane < k) {
            scr[32 + lane] = cs[lane];
            scr[64 + lane] = sn[lane];
          }
          T gk = lane == 0 ? g[k] : T(0);
          __syncwarp();
          T gn = T(0);
          if (lane == 0) {
            for (int i = 0; i < k; ++i) {
              const T a = scr[i], bb = scr[i + 1], ci = scr[32 + i], si = scr[64 + i];
              const T top = Num<T>::add(Num<T>::mul(ci, a), Num<T>::mul(si, bb));
              scr[i + 1] = Num<T>::add(Num<T>::mul(-si, a), Num<T>::mul(ci, bb));
              scr[i] = top;
            }
            const T hkk = scr[k], hk1 = scr[k + 1];
            const T den = hypot(hkk, hk1);
            T ck, sk;
            if (den == T(0)) { ck = T(1); sk = T(0); }
            else { ck = hkk / den; sk = hk1 / den; }
            cs[k] = ck;
            sn[k] = sk;
            scr[k] = Num<T>::add(Num<T>::mul(ck, hkk), Num<T>::mul(sk, hk1));
            scr[k + 1] = T(0);
            gn = Num<T>::mul(-sk, gk);
            g[k + 1] = gn;
            g[k] = Num<T>::mul(ck, gk);
          }
          gk1 = __shfl_sync(0xffffffffu, gn, 0);
          __syncwarp();
          if (lane <= k + 1) H[lane * m + k] = scr[lane];   // column k goes to the workspace once
        } else {
          if (lane == 0) {
            // Givens rotations on the fly (linalg.py:81-93)
            for (int i = 0; i < k; ++i) {
              const T a = H[i * m + k], bb = H[(i + 1) * m + k];
              const T top = Num<T>::add(Num<T>::mul(cs[i], a), Num<T>::mul(sn[i], bb));
              H[(i + 1) * m + k] = Num<T>::add(Num<T>::mul(-sn[i], a), Num<T>::mul(cs[i], bb));
              H[i * m + k] = top;
            }
            const T hkk = H[k * m + k], hk1 = H[(k + 1) * m + k];
            const T den = hypot(hkk, hk1);
            if (den == T(0)) { cs[k] = T(1); sn[k] = T(0); }
            else { cs[k] = hkk / den; sn[k] = hk1 / den; }
            H[k * m + k] = Num<T>::add(Num<T>::mul(cs[k], hkk), Num<T>::mul(sn[k], hk1));
            H[(k + 1) * m + k] = T(0);
            g[k + 1] = Num<T>::mul(-sn[k], g[k]);
            g[k] = Num<T>::mul(cs[k], g[k]);
          }
          __syncwarp();
          gk1 = g[k + 1];
        }
        S.used = k + 1;
        bool stop = double(fabs(gk1)) <= S.tol || S.breakdown;   // linalg.py:95-96
        if (!stop) {
          S.k = k + 1;
          if (S.k == m || S.total >= p.gmres_maxit) stop = true;      // loop end / :69-70
        }
        if (stop) {
          // y = H[:u,:u]^{-1} g[:u] (column-oriented back substitution, as
          // LAPACK trsm) and x += Q[:u]^T y (linalg.py:99-106)
          const int u = S.used;
          int singular = 0;
          if (fast) {
            // the same column-oriented substitution with lane i holding y[i]: after y[j] is
            // formed every y[i], i < j, takes its update at once (the serial loop spent
            // O(u^2) dependent accesses on the workspace); identical operations per element
            __syncwarp();   // column k of H written above
            T yi = lane < u ? g[lane] : T(0);
            T hnext = (u >= 1 && lane <= u - 1) ? H[lane * m + (u - 1)] : T(0);
            for (int j = u - 1; j >= 0; --j) {
              const T hcol = hnext;                       // H[lane][j] (lane <= j)
              if (j >= 1 && lane <= j - 1) hnext = H[lane * m + (j - 1)];
              const T d = __shfl_sync(0xffffffffu, hcol, j);
              if (d == T(0)) { singular = 1; break; }
              if (lane == j) yi = yi / d;
              const T yj = __shfl_sync(0xffffffffu, yi, j);
              if (lane < j) yi = Num<T>::add(yi, -Num<T>::mul(yj, hcol));
            }
            if (lane < u) scr[lane] = yi;
            __syncwarp();
          } else {
            if (lane == 0) {
              for (int i = 0; i < u; ++i) y[i] = g[i];
              for (int j = u - 1; j >= 0; --j) {
                const T d = H[j * m + j];
                if (d == T(0)) { singular = 1; break; }
                y[j] = y[j] / d;
                for (int i = 0; i < j; ++i) y[i] = Num<T>::add(y[i], -Num<T>::mul(y[j], H[i * m + j]));
              }
            }
            singular = __shfl_sync(0xffffffffu, singular, 0);
            __syncwarp();
          }
          if (singular) {
            S.phase = kPhFail;
          } else {
            const T* yv = fast ? scr : y;
            for (int j = lane; j < N; j += 32) {
              T acc = T(0);
              for (int i = 0; i < u; ++i) acc = Num<T>::fma(Q[(long long)i * ldn + j], yv[i], acc);
              x[w * ldn + j] = Num<T>::add(x[w * ldn + j], acc);
            }
            S.phase = kPhTop;
          }
        }
      }
      __syncwarp();
      if (lane == 0) c.st[w] = S;
      if (S.phase == kPhFail) ok = false;
    }
    __syncthreads();
    pt.mark(kPhOther);   // per-sample Arnoldi / Givens / update work
  }
  if (w < Rv && lane_id() == 0 && c.active[w]) c.cnt[w * OB_NSTATS + cnt_col] += c.st[w].total;
  return vote.all(ok) != 0;
}

// field eval at x0 (already loaded) into c.fb, counting one forward evaluation
// per active sample
template <typename T, int LR, bool WS>
OB_DEV void theta_eval(const RkParams<T>& p, MlpTile<T, LR, WS>& mt, ThetaCtx<T>& c, int Rv,
                       bool count_all) {
  MlpAdapter<T, LR, WS> f{p, mt};
  f.eval(c.fb);
  if (threadIdx.x < Rv && (count_all || c.active[threadIdx.x]))
    c.cnt[threadIdx.x * OB_NSTATS + OB_STAT_NFE_F] += 1;
}

template <typename T>
OB_DEV void set_x0(const RkParams<T>& p, T* x0, const T* src, int ld_src, double t) {
  const int N = p.d.N, ld0 = p.d.lda[0];
  for (int i = threadIdx.x; i < p.Rt * N; i += blockDim.x)
    x0[(i / N) * ld0 + i % N] = src[(i / N) * ld_src + i % N];
  if (p.d.time_input)
    for (int r = threadIdx.x; r < p.Rt; r += blockDim.x) x0[r * ld0 + N] = T(t);
  __syncthreads();
}

// residual F(x) = x - base - (h*theta) f(x, t1) for every row (integrators.py:233-234),
// its norms, and the linearisation at x left in the tile for the JVPs
template <typename T, int LR, bool WS>
OB_DEV void theta_residual(const RkParams<T>& p, MlpTile<T, LR, WS>& mt, ThetaCtx<T>& c, int Rv,
                           double t1, T hth) {
  const int N = p.d.N, ldn = p.d.ldn;
  set_x0(p, mt.s.x0, c.xk, ldn, t1);
  theta_eval<T, LR, WS>(p, mt, c, Rv, false);
  for (int i = threadIdx.x; i < p.Rt * N; i += blockDim.x) {
    const int o = (i / N) * ldn + i % N;
    c.rv[o] = Num<T>::add(Num<T>::add(c.xk[o], -c.base[o]), -Num<T>::mul(hth, c.fb[o]));
  }
  __syncthreads();
  if (warp_id() < Rv) {
    const T nr = sqrt(warp_dot(c.rv + warp_id() * ldn, c.rv + warp_id() * ldn, N));
    int fin = 1;
    for (int j = lane_id(); j < N; j += 32) fin &= Num<T>::finite(c.rv[warp_id() * ldn + j]) ? 1 : 0;
    fin = __all_sync(0xffffffffu, fin);
    if (lane_id() == 0) c.rn[warp_id()] = fin ? double(nr) : __longlong_as_double(0x7ff8000000000000LL);
  }
  __syncthreads();
}

// One theta step of the tile (theta_step, integrators.py:225-244 + newton_solve,
// linalg.py:117-142).  u: [Rt][ldn] state at t (replaced by u_{n+1}); rec
// (nullable): record [u_n, u_{n+1}, u_{n+1}] (s = 2 stages + u_next).
// Returns an OB status (OB_OK / OB_ERR_CONVERGENCE).
template <typename T, int LR, bool WS>
OB_DEV int theta_step_tile(const RkParams<T>& p, MlpTile<T, LR, WS>& mt, ThetaCtx<T>& c, T* u,
                           double t, double h, T* rec, int row0, int Rv, T* kry) {
  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt;
  const long long vec = (long long)p.B * N;
  const double th = p.theta, t1 = t + h;
  const T hth = T(h * th), h1 = T(h * (1.0 - th));
  // f0 = f(u, t); base = u + h(1-theta) f0
  set_x0(p, mt.s.x0, u, ldn, t);
  for (int r = threadIdx.x; r < Rv; r += blockDim.x) c.active[r] = 1;
  __syncthreads();
  theta_eval<T, LR, WS>(p, mt, c, Rv, true);
  for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
    const int o = (i / N) * ldn + i % N;
    c.base[o] = Num<T>::add(u[o], Num<T>::mul(h1, c.fb[o]));
    c.xk[o] = u[o];
    if (rec && i / N < Rv) rec[(long long)(row0 + i / N) * N + i % N] = u[o];
  }
  __syncthreads();
  theta_residual<T, LR, WS>(p, mt, c, Rv, t1, hth);
  ThetaOp<T, LR, WS> op{p, mt, hth, false, c.fb};
  int status = OB_OK;
  for (int it = 0; it < p.newton_maxit; ++it) {
    int any = 0, bad = 0;
    if (threadIdx.x < Rv) {
      const double rn = c.rn[threadIdx.x];
      const bool act = c.active[threadIdx.x] && !(rn <= p.newton_tol);
      if (act && !isfinite(rn)) bad = 1;                // linalg.py:130-131
      c.active[threadIdx.x] = act ? 1 : 0;
      any = act ? 1 : 0;
    }
    if (__syncthreads_or(bad)) return OB_ERR_CONVERGENCE;
    if (!__syncthreads_or(any)) break;
    for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
      const int o = (i / N) * ldn + i % N;
      c.rhs[o] = -c.rv[o];
    }
    __syncthreads();
    if (!gmres_tile<T>(p, op, c, c.rhs, c.gx, Rv, kry, OB_STAT_GMRES_F, OB_STAT_NFE_F))
      return OB_ERR_CONVERGENCE;
    for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
      const int r = i / N, o = r * ldn + i % N;
      if (r < Rv && c.active[r]) c.xk[o] = Num<T>::add(c.xk[o], c.gx[o]);
    }
    if (threadIdx.x < Rv && c.active[threadIdx.x]) c.cnt[threadIdx.x * OB_NSTATS + OB_STAT_NEWTON] += 1;
    __syncthreads();
    theta_residual<T, LR, WS>(p, mt, c, Rv, t1, hth);
  }
  int bad = 0;
  if (threadIdx.x < Rv && !(c.rn[threadIdx.x] <= p.newton_tol)) bad = 1;   // linalg.py:136-142
  if (__syncthreads_or(bad)) return OB_ERR_CONVERGENCE;
  for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
    const int r = i / N, o = r * ldn + i % N;
    u[o] = c.xk[o];
    if (rec && r < Rv) {
      const long long g = (long long)(row0 + r) * N + i % N;
      rec[vec + g] = u[o];
      rec[2 * vec + g] = u[o];
    }
  }
  __syncthreads();
  return status;
}

template <typename T>
OB_DEV ThetaCtx<T> theta_ctx(const RkParams<T>& p, T* sm) {
  __shared__ SampleState st[kMaxTileRows];
  __shared__ int cnt[kMaxTileRows * OB_NSTATS];
  __shared__ unsigned char active[kMaxTileRows];
  __shared__ double rn[kMaxTileRows];
  __shared__ int flag[1];
  ThetaCtx<T> c;
  c.base = sm + p.sm.vec[0];
  c.xk = sm + p.sm.vec[1];
  c.rv = sm + p.sm.vec[2];
  c.gx = sm + p.sm.vec[3];
  c.vin = sm + p.sm.vec[4];
  c.vout = sm + p.sm.vec[5];
  c.fb = sm + p.sm.vec[6];
  c.rhs = sm + p.sm.vec[7];
  c.st = st;
  c.cnt = cnt;
  c.active = active;
  c.rn = rn;
  c.flag = flag;
  for (int i = threadIdx.x; i < kMaxTileRows * OB_NSTATS; i += blockDim.x) cnt[i] = 0;
  for (int i = threadIdx.x; i < kMaxTileRows; i += blockDim.x) active[i] = 0;
  __syncthreads();
  return c;
}

template <typename T>
OB_DEV void flush_stats(const RkParams<T>& p, const ThetaCtx<T>& c, int row0, int Rv) {
  if (!p.sample_stats) return;
  for (int i = threadIdx.x; i < Rv * OB_NSTATS; i += blockDim.x)
    p.sample_stats[(long long)row0 * OB_NSTATS + i] += c.cnt[i];
}

// --------------------------------------------------------------- forward
template <typename T, int LR, bool WS>
__global__ void __launch_bounds__(kThreads, 1)
theta_forward_kernel(const __grid_constant__ RkParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  zero_smem(sm, p.sm.wts >= 0 ? p.sm.wts : p.sm.total);
  const int tile = blockIdx.x;
  const int row0 = tile * p.R;
  const int Rv = min(p.R, p.B - row0);
  MlpSmem<T> ms;
  Weights<T> W;
  setup_tile(p, sm, ms, W);
  MlpTile<T, LR, WS> mt(p.d, W, ms, p.Rt);
  if (p.sm.scr >= 0) { mt.scratch = sm + p.sm.scr; mt.scratch_elems = p.sm.scr_elems; }
  ThetaCtx<T> c = theta_ctx(p, sm);
  T* u = sm + p.sm.u;
  T* kry = p.sm.kry >= 0 ? sm + p.sm.kry : p.krylov + tile * p.krylov_stride;
  const int N = p.d.N, ldn = p.d.ldn;
  const long long vec = (long long)p.B * N;
  load_rows(u, ldn, p.u0, N, row0, Rv);
  __syncthreads();
  int bad = 0;  // as_state (nn.py:31-32)
  for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x)
    if (!Num<T>::finite(u[(idx / N) * ldn + idx % N])) bad = 1;
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) set_status(p.status, OB_ERR_VALUE, -1);
    return;
  }
  for (int n = 0; n < p.n_steps; ++n) {
    const double t = p.ts[n], h = p.ts[n + 1] - p.ts[n];
    obs_capture(p, u, n, row0, Rv);
    if (p.fwd_sol[n] >= 0) {
      store_rows(p.sol + p.fwd_sol[n] * vec, N, u, ldn, row0, Rv);
      __syncthreads();
    }
    T* rec = p.fwd_rec[n] >= 0 ? p.rec + (long long)p.fwd_rec[n] * 3 * vec : nullptr;
    const int st = theta_step_tile<T, LR, WS>(p, mt, c, u, t, h, rec, row0, Rv, kry);
    if (st != OB_OK) {
      if (threadIdx.x == 0) set_status(p.status, st, n);
      flush_stats(p, c, row0, Rv);
      return;
    }
  }
  store_rows(p.u_final, N, u, ldn, row0, Rv);
  obs_capture(p, u, p.n_steps, row0, Rv);
  flush_stats(p, c, row0, Rv);
  loss_partial(p, u, row0, Rv, tile);
}

// --------------------------------------------------------------- reverse
template <typename T, int LR, bool WS>
__global__ void __launch_bounds__(kThreads, 1)
theta_reverse_kernel(const __grid_constant__ RkParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  if (*(volatile int*)p.status != 0) return;
  zero_smem(sm, p.sm.wts >= 0 ? p.sm.wts : p.sm.total);
  const int tile = blockIdx.x;
  const int row0 = tile * p.R;
  const int Rv = min(p.R, p.B - row0);
  MlpSmem<T> ms;
  Weights<T> W;
  setup_tile(p, sm, ms, W);
  ms.ring = nullptr;   // the transposed adjoint products run faster from L1/L2 (measured, C5)
  MlpTile<T, LR, WS> mt(p.d, W, ms, p.Rt);
  if (p.sm.scr >= 0) { mt.scratch = sm + p.sm.scr; mt.scratch_elems = p.sm.scr_elems; }
  ThetaCtx<T> c = theta_ctx(p, sm);
  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt;
  const long long vec = (long long)p.B * N;
  T* u = sm + p.sm.u;
  T* lam = sm + p.sm.lam;
  T* jtv = sm + p.sm.jtv;
  T* kry = p.sm.kry >= 0 ? sm + p.sm.kry : p.krylov + tile * p.krylov_stride;
  T* mu = p.mu + tile * p.d.n_mu;
  const double th = p.theta;
  loss_seed(p, lam, row0, Rv);
  __syncthreads();
  for (int pc = 0; pc < p.prog_len; ++pc) {
    const int4 op = p.prog[pc];
    const int n = op.y;
    const double t = p.ts[n], h = p.ts[n + 1] - p.ts[n];
    if (op.x == kOpReplay) {
      const int src_kind = op.z >> 24, src = op.z & 0xffffff;
      const T* srcp = src_kind == kSrcU0 ? p.u0
                    : src_kind == kSrcSol ? p.sol + src * vec
                    : p.rec + ((long long)src * 3 + 2) * vec;
      load_rows(u, ldn, srcp, N, row0, Rv);
      __syncthreads();
      T* rec = p.rec + (long long)op.w * 3 * vec;
      const int st = theta_step_tile<T, LR, WS>(p, mt, c, u, t, h, rec, row0, Rv, kry);
      if (st != OB_OK) {
        if (threadIdx.x == 0) set_status(p.status, st, n);
        flush_stats(p, c, row0, Rv);
        return;
      }
      continue;
    }
    // theta_adjoint_step (adjoint.py:97-126)
    obs_inject(p, lam, n + 1, row0, Rv);
    const T* rec = p.rec + (long long)op.w * 3 * vec;
    const double t1 = t + h;
    const T hth = T(h * th), h1 = T(h * (1.0 - th));
    // linearisation at u1
    for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
      const int r = idx / N, j = idx % N;
      u[r * ldn + j] = rec[vec + (long long)(row0 + r) * N + j];
    }
    __syncthreads();
    set_x0(p, ms.x0, u, ldn, t1);
    mt.forward(nullptr, 0, p.d.L - 1);
    for (int r = threadIdx.x; r < Rv; r += blockDim.x) c.active[r] = 1;
    for (int i = threadIdx.x; i < Rt * ldn; i += blockDim.x) c.rhs[i] = lam[i];
    __syncthreads();
    ThetaOp<T, LR, WS> aop{p, mt, hth, true, jtv};
    if (!gmres_tile<T>(p, aop, c, c.rhs, c.gx, Rv, kry, OB_STAT_GMRES_B, OB_STAT_NFE_B)) {
      if (threadIdx.x == 0) set_status(p.status, OB_ERR_CONVERGENCE, n);
      flush_stats(p, c, row0, Rv);
      return;
    }
    // mu += h theta P(u1)^T lam_s  (one VJP pair at u1)
    const T sc = p.field_kind == OB_FIELD_STIFF ? p.out_scale : T(1);
    mt.vjp_keep(c.gx, ldn, Rv, jtv, ldn, mu, T(double(hth) * double(sc)));
    if (threadIdx.x < Rv) c.cnt[threadIdx.x * OB_NSTATS + OB_STAT_NFE_B] += 1;
    if (th < 1.0) {
      for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
        const int r = idx / N, j = idx % N;
        u[r * ldn + j] = rec[(long long)(row0 + r) * N + j];
      }
      __syncthreads();
      set_x0(p, ms.x0, u, ldn, t);
      mt.forward(nullptr, 0, p.d.L - 1);
      mt.vjp_keep(c.gx, ldn, Rv, jtv, ldn, mu, T(double(h1) * double(sc)));
      if (threadIdx.x < Rv) c.cnt[threadIdx.x * OB_NSTATS + OB_STAT_NFE_B] += 1;
      for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
        const int o = (i / N) * ldn + i % N, j = i % N;
        T jv = jtv[o];
        if (p.field_kind == OB_FIELD_STIFF)
          jv = Num<T>::add(Num<T>::mul(p.diag[j], c.gx[o]), Num<T>::mul(p.out_scale, jv));
        lam[o] = Num<T>::add(c.gx[o], Num<T>::mul(h1, jv));
      }
    } else {
      for (int i = threadIdx.x; i < Rt * ldn; i += blockDim.x) lam[i] = c.gx[i];
    }
    int bad = 0;
    for (int i = threadIdx.x; i < Rt * N; i += blockDim.x)
      if (!Num<T>::finite(lam[(i / N) * ldn + i % N])) bad = 1;
    if (__syncthreads_or(bad)) {
      if (threadIdx.x == 0) set_status(p.status, OB_ERR_GRADIENT_EXPLOSION, n);
      flush_stats(p, c, row0, Rv);
      return;
    }
  }
  obs_inject(p, lam, 0, row0, Rv);
  store_rows(p.du0, N, lam, ldn, row0, Rv);
  flush_stats(p, c, row0, Rv);
}

// one sweep direction per translation unit (theta_*_fwd.cu / theta_*_rev.cu compile in parallel)
template <typename T, bool kFwd, int LR>
static cudaError_t launch_theta_lr(const RkParams<T>& p, int tiles, size_t smem, cudaStream_t st) {
  if constexpr (kFwd) return launch_smem(theta_forward_kernel<T, LR, false>, tiles, smem, st, p);
  else return launch_smem(theta_reverse_kernel<T, LR, false>, tiles, smem, st, p);
}

template <typename T, bool kFwd>
cudaError_t launch_theta_dir(const RkParams<T>& p, int lr, int tiles, size_t smem, cudaStream_t st) {
  switch (lr) {
    case 1: return launch_theta_lr<T, kFwd, 1>(p, tiles, smem, st);
    case 2: return launch_theta_lr<T, kFwd, 2>(p, tiles, smem, st);
    default:
      if constexpr (sizeof(T) == 4) return launch_theta_lr<T, kFwd, 8>(p, tiles, smem, st);
      return cudaErrorInvalidConfiguration;
  }
}

}  // namespace ob
