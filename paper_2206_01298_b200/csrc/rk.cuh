// rk.cuh -- parameters shared by the persistent explicit-RK kernels and the
// host engine.
#pragma once

#include "tile.cuh"

namespace ob {

// reverse-program opcodes (host-compiled from the checkpoint policy)
enum { kOpReplay = 0, kOpReverse = 1 };
// replay start-state sources
enum { kSrcU0 = 0, kSrcRecNext = 1, kSrcSol = 2 };

struct SmemLayout {      // offsets in elements of T (-1: not allocated)
  int x0, hid[OB_MAX_LAYERS], pre[OB_MAX_LAYERS], tA, tB;
  int u, lam, lamn, w, jtv;
  int vec[8];             // theta-method work vectors [Rt][ldn] (-1 when unused)
  int aux;                // CNF: output-layer buffer [2Rt][lda_L]
  int scr, scr_elems;     // theta: split-K scratch for narrow JVP / VJP products
  int kry;                // theta: Krylov workspace in shared memory (or -1: global)
  int wts;                // packed weights staged in shared memory, or -1
  int ks;                 // per-tile stage scratch [2][s][Rt][ldn] in shared memory, or -1 (global)
  int ring, ring_elems;   // per-warp cp.async rings for L2-streamed weights, or -1
  int hscr, hscr_elems;   // hidden-layer split-K partials (MLP explicit-RK tiles), or -1
  int total;
};

template <typename T>
struct RkParams {
  Dims d;
  Weights<T> W;
  SmemLayout sm;
  // scheme (tableaux.py:14-56)
  int s, fsal;
  double a[OB_MAX_STAGES * OB_MAX_STAGES], b[OB_MAX_STAGES], c[OB_MAX_STAGES];
  unsigned skip_vjp;      // bit i: stage i cotangent is identically zero
  // field
  int field_kind;
  const T* diag;          // stiff: a
  T out_scale;            // stiff: s
  // problem
  int B, R, Rt, n_steps;
  const double* ts;       // [n_steps+1]
  int loss_kind;
  const T* targets;
  const T* seed;          // OB_LOSS_SEED: terminal lambda [B][N] (caller-formed)
  // observation losses (OB_LOSS_OBS_*): obs_k[n] = observation index at boundary n or -1
  const int* obs_k;
  int n_obs;
  const T* obs_values;             // [n_obs][B][N]
  const T* scale_lo;               // [N] or null
  const T* scale_hi;
  T* preds;                        // [n_obs][B][N]
  int* obs_step;                   // adaptive: [n_obs][B] boundary index of each observation
  // adaptive stepping (integrators.py:294-349)
  int ad_policy;                   // 0 store_all, 1 store_solutions
  double ad_abstol, ad_reltol, ad_hinit, ad_hmin, ad_hmax, ad_safety, ad_alpha, ad_beta;
  long long ad_max_steps;
  int ad_cap;                      // accepted-step capacity per sample
  double ad_d[OB_MAX_STAGES];      // b - b_emb
  const double* ad_pts;            // interval end points [ad_nseg + 1]
  int ad_nseg;
  const int* ad_seg_obs;           // observation index at the end of interval seg, or -1
  int ad_obs0;                     // observation 0 at t0 (initial state)
  double* ad_grid;                 // [B][cap][2] (t_n, h_n)
  int* ad_nacc;                    // [B]
  double inv_batch_global;
  double batch_global;
  // buffers
  const T* u0;
  T* u_final;
  T* du0;
  T* rec;                 // [nbuf][s+1][B][N]: stage states then u_next
  T* sol;                 // [nsol][B][N]
  const int* fwd_rec;     // [n_steps] record buffer written in the forward, or -1
  const int* fwd_sol;     // [n_steps] solution slot written in the forward, or -1
  const int4* prog;       // reverse program
  int prog_len;
  const T* packed;        // packed weights in global memory (n_packed elements)
  T* scratch;             // per tile [2][s][Rt][ldn]: ks (forward), Lam (reverse)
  long long scratch_stride;
  T* mu;                  // [tiles][n_mu] per-CTA padded parameter cotangent slots
  long long n_params;
  double* loss_part;      // [tiles]
  int* status;            // [2] first error code, step
  int prof;               // OB_FLAG_PHASE_TIMING
  unsigned long long* phase;  // [OB_NPHASES] cycle accumulators (prof only)
  // theta methods (integrators.py:225-244, linalg.py:37-142)
  double theta;
  double newton_tol, gmres_tol;
  int newton_maxit, gmres_maxit, gmres_restart;
  T* krylov;              // per tile: Q [R][m+1][ldn] | H [R][m+1][m] | cs, sn [R][m] | g [R][m+1] | y [R][m]
  long long krylov_stride;
  int* sample_stats;      // [B][OB_NSTATS] per-sample counters (nullable)
  // state buffers (u, lam, lamn, w, jtv) in global memory when sm.u < 0 (C3)
  T* state_glob;
  long long state_stride;
  // classification head (OB_LOSS_CE_HEAD, config C3)
  const T* head;
  const int* labels;
  int n_classes;
  T* head_part;           // [tiles][n_head] head-gradient partials, then fp64 scratch
  int tiles_total;
  // CNF (config C4)
  const T* eps;           // Hutchinson probes [B][D]
  T* cnf_pre;             // per tile [L-1][2Rt][lda] pre-activations (forward | raw tangent)
  long long cnf_pre_stride;
  // one launcher-set word for the specialised tiles.  tcgen05 conv tile: the shared-window
  // address of the kernel's dynamic shared memory (1 KB reserved + its static shared size; a
  // kernel-parameter value is uniform, so MMA descriptors built from it can stay on the
  // uniform datapath).  Cluster theta kernels: rows per cluster the layout is sized for.
  unsigned tile_aux;
};

template <typename T>
struct PackParams {
  Dims d;
  const T* theta;
  T* packed;
};

// per-phase SM-cycle counters (profiling aid, OB_FLAG_PHASE_TIMING)
enum { kPhElem = 0, kPhRecompute = 1, kPhVjp = 2, kPhLam = 3, kPhReplay = 4, kPhFwdStep = 5,
       kPhGmres = 6, kPhOther = 7 };


}  // namespace ob
