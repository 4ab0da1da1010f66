/*
 * odeblock.h -- C ABI of the B200-native discrete-adjoint ODE-block engine.
 *
 * Every entry point replaces one reference interface of the CPU package
 * `odegrad` (/root/reference/pkg/src/odegrad; cited file:line below).  The
 * reference is pure Python, so there is no reference FFI; these are the calls
 * its `Field` protocol and `grad()` would bind through ctypes.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "device" pointers are CUDA global memory
 *    (owned by the caller, e.g. torch tensors); "host" pointers are CPU memory.
 *  - Float arrays are float32 or float64 per the descriptor's dtype.
 *  - Every function returns an ob_status; detail text via ob_last_error()
 *    (thread-local).  Status codes map 1:1 onto the reference exception
 *    classes (nn.py:29-34 ValueError, integrators.py:20-25 IntegrationError,
 *    linalg.py:14-19 ConvergenceError, adjoint.py:33-34 GradientExplosionError).
 *  - Calls are reentrant per stream; no allocation inside the hot loop: all
 *    scratch lives in the caller's workspace (size from *_workspace_size).
 *  - Inputs are never mutated (reference ownership rule).
 */
#ifndef ODEBLOCK_H
#define ODEBLOCK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  OB_OK = 0,
  OB_ERR_VALUE = 1,              /* ValueError: shape / non-finite input (nn.py:26-35)       */
  OB_ERR_INTEGRATION = 2,        /* IntegrationError: state overflow (integrators.py:219-220) */
  OB_ERR_STIFFNESS = 3,          /* StiffnessError (adaptive only; unused by fixed stepping)  */
  OB_ERR_CONVERGENCE = 4,        /* ConvergenceError (linalg.py:101-142)                      */
  OB_ERR_GRADIENT_EXPLOSION = 5, /* GradientExplosionError (adjoint.py:42-44)                 */
  OB_ERR_CUDA = 6,               /* CUDA runtime failure / no device                          */
  OB_ERR_UNSUPPORTED = 7         /* configuration outside this build                          */
} ob_status;

enum { OB_F32 = 0, OB_F64 = 1 };
/* activation ids: nn.py:23 (identity/relu/tanh/gelu) + softplus (C4, new) */
enum { OB_ACT_IDENTITY = 0, OB_ACT_RELU = 1, OB_ACT_TANH = 2, OB_ACT_GELU = 3, OB_ACT_SOFTPLUS = 4 };
/* right-hand sides: MlpField (integrators.py:76-102); a*u + s*MLP(u) as a
   CallableField (integrators.py:105-141, config C5); CNF and conv are new */
enum { OB_FIELD_MLP = 0, OB_FIELD_STIFF = 1, OB_FIELD_CNF = 2, OB_FIELD_CONV = 3 };
/* OB_FIELD_CONV (config C3): state = 16x16 NHWC image with C = widths[2] channels;
   f = conv3x3(C+1 -> C)(cat(u, t)) -> relu -> conv3x3(C -> C), padding 1, i.e.
   n_layers = 2, widths = {C+1, C, C}, time_input = 1, activation = relu;
   theta = [W1 (C x 3 x 3 x (C+1)), b1, W2 (C x 3 x 3 x C), b2]. */
enum { OB_SCHEME_RK = 0, OB_SCHEME_THETA = 1 };
/* CheckpointPolicy kinds (checkpointing.py:173-190) */
enum { OB_POLICY_STORE_ALL = 0, OB_POLICY_STORE_SOLUTIONS = 1, OB_POLICY_REVOLVE = 2 };
/* losses: 0.5*mean||u||^2 (BASELINE C1/C2/C5), per-sample MSE vs terminal
   targets (losses.py:78-107, K=1), CE head (C3), CNF NLL (C4), and the
   reference's observation losses (LossSpec mse/mae over K observation times
   with optional min-max scaling, losses.py:10-107; seeds injected at step
   boundaries as in backward_sweep, adjoint.py:235-253) for MLP / stiff fields */
enum { OB_LOSS_HALF_SQNORM = 0, OB_LOSS_MSE = 1, OB_LOSS_CE_HEAD = 2, OB_LOSS_CNF_NLL = 3,
       OB_LOSS_OBS_MSE = 4, OB_LOSS_OBS_MAE = 5,
       /* caller-supplied seeds (backward_sweep with an arbitrary terminal AdjointState,
          adjoint.py:47-52, :235-253): lambda_N = ob_buffers.seed [B,N] as given (no batch
          scaling), injections ob_buffers.obs_values [n_obs,B,N] added to lambda at the
          boundaries obs_steps (inject_observation, adjoint.py:135-140), mu_N =
          ob_buffers.dtheta_seed [n_params] or 0; the loss is the caller's (ob loss = 0) */
       OB_LOSS_SEED = 6 };
/* revolve action kinds (checkpointing.py:70-80) */
enum { OB_ACT_ADVANCE = 0, OB_ACT_STORE = 1, OB_ACT_RESTORE = 2, OB_ACT_REVERSE = 3 };

#define OB_MAX_LAYERS 8
#define OB_MAX_STAGES 8

/* Vector field descriptor (MlpSpec, nn.py:38-76). widths[0..n_layers]. */
typedef struct {
  int32_t kind;        /* OB_FIELD_* */
  int32_t dtype;       /* OB_F32 | OB_F64 */
  int32_t n_layers;
  int32_t widths[OB_MAX_LAYERS + 1];
  int32_t activation;  /* OB_ACT_* for hidden layers; output layer is linear */
  int32_t time_input;  /* 1: time appended as the last input (nn.py:126-129) */
  double out_scale;    /* OB_FIELD_STIFF: s in a*u + s*MLP(u) */
  int64_t n_params;    /* sum_l w_{l+1}*w_l + w_{l+1} (nn.py:60-63) */
} ob_field_desc;

/* Scheme (tableaux.py:14-56): explicit Butcher tableau or theta method. */
typedef struct {
  int32_t kind;        /* OB_SCHEME_RK | OB_SCHEME_THETA */
  int32_t stages;
  int32_t fsal;
  int32_t _pad;
  double theta;        /* theta methods: 1 = beuler, 0.5 = cn */
  double a[OB_MAX_STAGES * OB_MAX_STAGES];  /* row-major s x s */
  double b[OB_MAX_STAGES];
  double c[OB_MAX_STAGES];
  double b_emb[OB_MAX_STAGES]; /* embedded weights (adaptive stepping), when has_emb */
  int32_t order;               /* order p of b: PI exponents 0.7/p, 0.4/p (integrators.py:300-302) */
  int32_t has_emb;
} ob_scheme_desc;

/* SolverConfig (linalg.py:22-34). */
typedef struct {
  double newton_tol;
  double gmres_tol;
  int32_t newton_maxit;
  int32_t gmres_maxit;
  int32_t gmres_restart;
  int32_t _pad;
} ob_solver_cfg;

/* One gradient problem: grad(field, scheme, loss, u0, t0, tF, ctrl, policy,
   solver_cfg) of adjoint.py:256-279, batched over `batch` samples. */
typedef struct {
  ob_field_desc field;
  ob_scheme_desc scheme;
  ob_solver_cfg solver;
  int64_t batch;          /* samples handled by this call (this rank's shard)   */
  int64_t batch_global;   /* samples across all ranks: loss = sum / batch_global */
  int32_t n_steps;        /* FixedController / FixedGridController step count   */
  int32_t policy;         /* OB_POLICY_*                                          */
  int32_t nc;             /* revolve slots                                         */
  int32_t loss;           /* OB_LOSS_*                                             */
  const double* times;    /* HOST array, n_steps+1 boundary times (integrators.py:276) */
  int32_t flags;          /* OB_FLAG_* */
  int32_t n_obs;          /* OB_LOSS_OBS_*: observation count K >= 1           */
  const int32_t* obs_steps; /* HOST [n_obs] boundary index of each observation, strictly
                             increasing in [0, n_steps] (_match_boundaries, adjoint.py:213) */
  /* AdaptiveController (integrators.py:178-193): adaptive = 1 replaces the fixed
     grid (times / n_steps unused) by per-sample error-controlled steps on [t0, tF],
     one integration per observation interval (adjoint.py:162-186) */
  int32_t adaptive;
  int32_t max_accepted;   /* per-sample capacity of accepted steps (workspace sizing) */
  double abstol, reltol, h_init, h_min, h_max, safety;
  int64_t max_steps;      /* per integrate() call, trials included               */
  double t0, tF;
  const double* obs_times; /* HOST [n_obs] observation times (adaptive + OB_LOSS_OBS_*) */
  /* samples per CTA tile: 0 = the planner's choice (ceil(B / #SM), capped per kernel
     family); > 0 forces it (capped the same way) -- selects the tile geometry a test
     or a benchmark exercises */
  int32_t tile_rows;
  int32_t _pad2;
} ob_problem;

/* flags: accumulate per-phase SM cycles of the persistent kernels (profiling aid;
   read with ob_debug_phase_cycles) */
enum { OB_FLAG_PHASE_TIMING = 1,
       /* force the baseline single-CTA SIMT kernels: no tcgen05 tensor-core tiles (MLP, CNF,
          conv) and no cluster-resident weights for the theta methods */
       OB_FLAG_NO_TENSOR_CORES = 2 };
#define OB_NPHASES 16

/* Device buffers of one gradient call. */
typedef struct {
  const void* theta;      /* [n_params]                                          */
  const void* aux;        /* STIFF: diag a [N]; CNF: probes eps [B,N]; else NULL */
  const void* u0;         /* [B, N]                                              */
  const void* targets;    /* OB_LOSS_MSE: [B, N]; else NULL                       */
  void* u_final;          /* out [B, N]                                          */
  void* du0;              /* out [B, N]     (lambda_0)                           */
  void* dtheta;           /* out [n_params] (mu_0, summed over this call's batch) */
  double* loss;           /* out [1] float64: this call's sum of per-sample loss / batch_global */
  void* workspace;        /* scratch, >= ob_grad_workspace_size bytes            */
  size_t workspace_bytes;
  int32_t* sample_stats;  /* optional out [B, OB_NSTATS] per-sample counters, or NULL */
  /* OB_LOSS_CE_HEAD (config C3): global-average-pool + linear + cross-entropy head */
  const void* head;       /* [n_classes*C + n_classes] head parameters (W row-major, b) */
  const int32_t* labels;  /* [B] class labels                                      */
  void* dhead;            /* out [n_classes*C + n_classes] head gradient (this batch) */
  int32_t n_classes;
  int32_t _pad;
  /* OB_LOSS_OBS_*: observations and the optional min-max scaling (losses.py:10-37) */
  const void* obs_values; /* [n_obs, B, N] observed states (scaled space when scaling) */
  const void* scale_lo;   /* [N] or NULL (no scaling); components with hi <= lo pass through */
  const void* scale_hi;   /* [N] or NULL                                          */
  void* predictions;      /* out [n_obs, B, N]: states at the observation boundaries */
  /* adaptive: optional outputs of the per-sample grids */
  double* grid;           /* out [B, max_accepted + 1] boundary times (NaN past the end) or NULL */
  int32_t* n_accepted;    /* out [B] accepted steps per sample, or NULL                 */
  /* OB_LOSS_SEED: terminal adjoint state (adjoint_terminal, adjoint.py:47-52) */
  const void* seed;        /* [B, N] lambda_N                                            */
  const void* dtheta_seed; /* [n_params] mu_N, or NULL (zero)                            */
} ob_buffers;

/* per-sample stats columns (implicit schemes; explicit: fixed by the schedule) */
enum { OB_STAT_NFE_F = 0, OB_STAT_NFE_B = 1, OB_STAT_NEWTON = 2, OB_STAT_GMRES_F = 3,
       OB_STAT_GMRES_B = 4, OB_STAT_ACCEPTED = 5, OB_STAT_REJECTED = 6, OB_STAT_RECOMPUTED = 7,
       OB_NSTATS = 8 };

/* NfeCounters (integrators.py:28-50) + StoreCounters (checkpointing.py:193-198),
   reference semantics per sample trajectory, plus what the device really ran. */
typedef struct {
  int64_t nfe_forward, nfe_backward, steps_accepted, steps_rejected, steps_recomputed;
  int64_t stored_states, stored_stage_vectors, max_live_slots, recomputed_steps;
  int64_t kernel_launches;       /* kernels this call launched                          */
  int64_t device_rhs_evals;      /* RHS evaluations the device executed (per sample)    */
  int64_t device_vjp_evals;      /* VJP pairs the device executed (zero cotangents skipped) */
  int64_t tile_rows;             /* samples per CTA tile                                 */
  int64_t tiles;                 /* CTAs per persistent launch                           */
  int64_t tensor_cores;          /* 1: the contractions ran on a tcgen05 tile (split fp32 products);
                                    2: fp64 cluster MLP (weights resident across a cluster of 2 or 8 CTAs,
                                       mma.sync f64) */
  double ms_pack, ms_forward, ms_reverse, ms_reduce;  /* CUDA-event device times of this call */
} ob_counters;

/* ---- library ----------------------------------------------------------- */
const char* ob_version(void);
const char* ob_last_error(void);
int ob_device_count(int32_t* count);

/* ---- host-only schedule math (checkpointing.py:32-170) ------------------- */
int ob_revolve_count(int32_t nt, int32_t nc, int64_t* out);
/* actions: capacity x 4 int32 (kind, step, start, stop) as in ScheduleAction */
int ob_revolve_schedule(int32_t nt, int32_t nc, int32_t* actions, int64_t capacity,
                        int64_t* n_actions);

/* ---- block gradient: forward integration + checkpoints + discrete adjoint --
   replaces grad() (adjoint.py:256-279) = forward_pass (:151-210) +
   loss_and_grad_seed (losses.py:78-107) + backward_sweep (:235-253). */
int ob_grad_workspace_size(const ob_problem* p, size_t* bytes);
int ob_grad(const ob_problem* p, const ob_buffers* b, ob_counters* out, void* stream);
/* The two halves of ob_grad on one workspace, for callers that form the terminal
   seed themselves (grad() split as forward_pass + loss + backward_sweep,
   adjoint.py:151-210 / :235-253):
   ob_forward_pass: weight packing + forward sweep: u_final, predictions at observed
     boundaries, checkpoints kept in b->workspace (and, for a built-in loss, b->loss);
   ob_backward_sweep: reverse sweep from those checkpoints -> du0 (lambda_0), dtheta
     (mu_0).  Same problem struct and workspace in both calls; theta and u0 must not
     change in between (the reference's ForwardSolution holds the same state). */
int ob_forward_pass(const ob_problem* p, const ob_buffers* b, ob_counters* out, void* stream);
int ob_backward_sweep(const ob_problem* p, const ob_buffers* b, ob_counters* out, void* stream);

/* ---- continuous-adjoint baseline (continuous_adjoint_solve, adjoint.py:294-331) ----
   Integrates the augmented reverse-time system (u, lambda, mu) with p's explicit
   scheme over the tau grid p->times (n_steps + 1 points from 0 to tF - t0; p->tF
   sets t = tF - tau) from u_final [B,N] and dphi_du [B,N]: lam0 [B,N] =
   lambda(t0), mu0 [n_params] = sum over samples of the integral of P^T lambda.
   Workspace: >= ob_grad_workspace_size(p).  Explicit schemes, MLP / stiff fields. */
int ob_continuous_adjoint(const ob_problem* p, const void* theta, const void* aux,
                          const void* u_final, const void* dphi_du, void* lam0, void* mu0,
                          void* workspace, size_t workspace_bytes, ob_counters* out, void* stream);

/* ---- training-loop optimizer (training.py:156-190, :276-277) ------------------
   ob_adamw_step: one AdamW update of device vectors theta/m/v (n params, dtype
   OB_F32|OB_F64) with gradient g; step = the new step count t >= 1.  Bit-identical
   to the reference's numpy update in fp64.  A non-finite g returns
   OB_ERR_GRADIENT_EXPLOSION and leaves theta/m/v untouched.
   ob_grad_norm: ||g||_2 in fp64 (fixed reduction order) into *norm (host).
   Errors of these two calls are reported by ob_optim_last_error(). */
int ob_adamw_step(int32_t dtype, void* theta, const void* g, void* m, void* v, int64_t n,
                  int64_t step, double lr, double beta1, double beta2, double eps,
                  double weight_decay, void* stream);
int ob_grad_norm(int32_t dtype, const void* g, int64_t n, double* norm, void* stream);
/* The training loop's per-epoch optimizer step with no host round trip (train,
   training.py:276-283): ||g|| into the device slot *norm_out, then a sticky device
   status (*status = 1: gradient explosion -- g non-finite or ||g|| > threshold, the
   reference's GradientExplosionError / explosion_threshold stop), then the AdamW
   update unless the status is set.  The host reads norms and status when it logs. */
int ob_adamw_step_gated(int32_t dtype, void* theta, const void* g, void* m, void* v, int64_t n,
                        int64_t step, double lr, double beta1, double beta2, double eps,
                        double weight_decay, double threshold, double* norm_out, int32_t* status,
                        void* stream);
const char* ob_optim_last_error(void);

/* ---- profiling aid: per-phase cycle totals summed over CTAs (reset: zero them) */
int ob_debug_phase_cycles(uint64_t* out, int32_t n, int32_t reset);

/* ---- the Field protocol, batched (integrators.py:53-102) -----------------
   eval: f(u,t); jvp: (df/du) w; vjp: ((df/du)^T v, sum_b (df/dtheta)^T v);
   vjp_u: (df/du)^T v.  t is one time for the whole batch; aux as in ob_buffers. */
int ob_field_eval(const ob_field_desc* f, int64_t batch, const void* theta, const void* aux,
                  const void* u, double t, void* out, void* stream);
int ob_field_jvp(const ob_field_desc* f, int64_t batch, const void* theta, const void* aux,
                 const void* u, double t, const void* w, void* out, void* stream);
int ob_field_vjp(const ob_field_desc* f, int64_t batch, const void* theta, const void* aux,
                 const void* u, double t, const void* v, void* jtv, void* ptv, void* stream);
int ob_field_vjp_u(const ob_field_desc* f, int64_t batch, const void* theta, const void* aux,
                   const void* u, double t, const void* v, void* jtv, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ODEBLOCK_H */
