// capi.cu -- the C ABI (include/odeblock.h) and the host engine behind it.
//
// The engine plans one gradient call (tile size, shared-memory layout,
// checkpoint buffers, the reverse program compiled from the checkpoint policy,
// reference-semantics counters), carves the caller's workspace, uploads one
// small control blob and launches: pack_weights -> forward (persistent) ->
// reverse (persistent) -> fixed-order tile reduction.  No allocation, no host
// round trip inside the integration; one stream synchronisation at the end to
// surface the reference's exceptions as status codes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <chrono>
#include <cstdio>

#include "../../include/odeblock.h"
#include "revolve.h"
#include "rk.cuh"

namespace ob {
template <typename T> cudaError_t launch_pack(const PackParams<T>&, cudaStream_t);
template <typename T, bool WS>
cudaError_t launch_rk_ws(const RkParams<T>&, int, int, size_t, cudaStream_t, bool);
template <typename T, bool WS>
cudaError_t launch_field_ws(const RkParams<T>&, int, int, size_t, int, double, const T*, const T*,
                            T*, cudaStream_t);
template <typename T> cudaError_t launch_reduce(const Dims&, const T*, int, long long, T*,
                                                const double*, double, double*, cudaStream_t,
                                                const T*);
template <typename T, bool kFwd>
cudaError_t launch_theta_dir(const RkParams<T>&, int, int, size_t, cudaStream_t);
template <typename T>
cudaError_t launch_theta(const RkParams<T>& p, int lr, int tiles, size_t smem, cudaStream_t st,
                         bool forward) {
  return forward ? launch_theta_dir<T, true>(p, lr, tiles, smem, st)
                 : launch_theta_dir<T, false>(p, lr, tiles, smem, st);
}
template <typename T>
cudaError_t launch_cnf(const RkParams<T>&, int, int, size_t, cudaStream_t, bool);
template <typename T>
cudaError_t launch_cnf_field(const RkParams<T>&, int, int, size_t, int, double, const T*, const T*,
                             T*, cudaStream_t);
template <typename T>
cudaError_t launch_conv(const RkParams<T>&, int, size_t, cudaStream_t, bool);
template <typename T>
cudaError_t launch_conv_field(const RkParams<T>&, int, size_t, int, double, const T*, const T*, T*,
                              cudaStream_t);
template <typename T> cudaError_t launch_pack_conv(const PackParams<T>&, cudaStream_t);
template <typename T, bool WS>
cudaError_t launch_adaptive_ws(const RkParams<T>&, int, int, size_t, cudaStream_t, bool);
template <typename T, bool WS>
cudaError_t launch_cadj_ws(const RkParams<T>&, int, int, size_t, double, const T*, cudaStream_t);
template <typename T>
cudaError_t launch_reduce_plain(const T*, int, long long, long long, T*, cudaStream_t);
// tcgen05 tensor-core MLP tile (rk_tc.cu)
void tc_sizes(int D0, int H, int D2, unsigned* packed_bytes, unsigned* total_bytes);
bool tc_shape_supported(int D0, int H, int D2);
cudaError_t launch_pack_tc(const Dims& d, const float* theta, float* packed, cudaStream_t st);
cudaError_t launch_rk_tc(const RkParams<float>& p, int tiles, size_t smem, cudaStream_t st,
                         bool forward);
// tcgen05 CNF tile (cnf_tc.cu)
bool tc_cnf_shape(int D, int H);
void tc_cnf_sizes(unsigned* packed_bytes, unsigned* smem_bytes, unsigned* log_record_bytes);
cudaError_t launch_pack_tc_cnf(const Dims& d, const float* theta, void* img, cudaStream_t st);
cudaError_t launch_cnf_tc(const RkParams<float>& p, int tiles, int cl, size_t smem, cudaStream_t st,
                          bool forward);
cudaError_t launch_cnf_tc_field(const RkParams<float>& p, int tiles, int cl, size_t smem, int mode,
                                double t, const float* u, const float* w, float* out, cudaStream_t st);

// cluster-resident-weights theta kernels (theta_cl_f64.cu)
void theta_cluster_geom(int N, int H, int R, int RC, bool second_x, int* region_doubles, int* cluster);
int theta_cluster_max_active(size_t smem);
cudaError_t launch_theta_cluster(const RkParams<double>& p, int tiles, size_t smem, cudaStream_t st, bool forward);
// explicit-RK kernels on the cluster MLP, clusters of 8 and of 2 CTAs (rk_cl_f64.cu, rk_cl2_f64.cu)
void rk_cluster8_geom(int N, int H, int R, int* region_doubles);
int rk_cluster8_max_active(size_t smem);
cudaError_t launch_rk_cluster8(const RkParams<double>& p, int tiles, size_t smem, cudaStream_t st, bool forward);
void rk_cluster2_geom(int N, int H, int R, int* region_doubles);
int rk_cluster2_max_active(size_t smem);
cudaError_t launch_rk_cluster2(const RkParams<double>& p, int tiles, size_t smem, cudaStream_t st, bool forward);
// tcgen05 conv tile (conv_tc.cu)
void tc_conv_sizes(unsigned* packed_bytes, unsigned* smem_bytes);
cudaError_t launch_pack_tc_conv(const Dims& d, const float* theta, void* img, cudaStream_t st);
cudaError_t launch_conv_tc(const RkParams<float>& p, int tiles, size_t smem, cudaStream_t st, bool forward);
cudaError_t launch_conv_tc_field(const RkParams<float>& p, int tiles, size_t smem, int mode, double t,
                                 const float* u, const float* w, float* out, cudaStream_t st);

// dispatch on where the weights live (fp32 only stages them in shared memory)
template <typename T>
cudaError_t launch_rk(const RkParams<T>& p, int lr, int tiles, size_t smem, cudaStream_t st,
                      bool forward) {
  if constexpr (sizeof(T) == 4)
    if (p.sm.wts >= 0) return launch_rk_ws<T, true>(p, lr, tiles, smem, st, forward);
  return launch_rk_ws<T, false>(p, lr, tiles, smem, st, forward);
}
template <typename T>
cudaError_t launch_adaptive(const RkParams<T>& p, int lr, int tiles, size_t smem, cudaStream_t st,
                            bool forward) {
  if constexpr (sizeof(T) == 4)
    if (p.sm.wts >= 0) return launch_adaptive_ws<T, true>(p, lr, tiles, smem, st, forward);
  return launch_adaptive_ws<T, false>(p, lr, tiles, smem, st, forward);
}
template <typename T>
cudaError_t launch_cadj(const RkParams<T>& p, int lr, int tiles, size_t smem, double tF, const T* dphi,
                        cudaStream_t st) {
  if constexpr (sizeof(T) == 4)
    if (p.sm.wts >= 0) return launch_cadj_ws<T, true>(p, lr, tiles, smem, tF, dphi, st);
  return launch_cadj_ws<T, false>(p, lr, tiles, smem, tF, dphi, st);
}
template <typename T>
cudaError_t launch_field_op(const RkParams<T>& p, int lr, int tiles, size_t smem, int mode,
                            double t, const T* u, const T* w, T* out, cudaStream_t st) {
  if constexpr (sizeof(T) == 4)
    if (p.sm.wts >= 0) return launch_field_ws<T, true>(p, lr, tiles, smem, mode, t, u, w, out, st);
  return launch_field_ws<T, false>(p, lr, tiles, smem, mode, t, u, w, out, st);
}
}  // namespace ob

using namespace ob;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(OB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
static int pad4i(int n) { return (n + 3) & ~3; }

// per-device [OB_NPHASES] cycle accumulators (profiling aid), created on first use
// on the device current at the call
constexpr int kMaxDevices = 64;
static unsigned long long* g_phase[kMaxDevices] = {};
static std::mutex g_phase_mu;

static int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = 0;
  }
  return dev < kMaxDevices ? dev : kMaxDevices - 1;
}

static unsigned long long* phase_buffer() {
  std::lock_guard<std::mutex> lk(g_phase_mu);
  unsigned long long*& buf = g_phase[current_device()];
  if (!buf) {
    if (cudaMalloc(&buf, sizeof(unsigned long long) * OB_NPHASES) != cudaSuccess) {
      buf = nullptr;
      return nullptr;
    }
    cudaMemset(buf, 0, sizeof(unsigned long long) * OB_NPHASES);
  }
  return buf;
}

extern "C" int ob_debug_phase_cycles(uint64_t* out, int32_t n, int32_t reset) {
  unsigned long long h[OB_NPHASES] = {};
  unsigned long long* d = phase_buffer();
  if (!d) return fail(OB_ERR_CUDA, "no device");
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(OB_ERR_CUDA, cudaGetErrorString(e));
  for (int i = 0; i < n && i < OB_NPHASES; ++i) out[i] = h[i];
  if (reset && (e = cudaMemset(d, 0, sizeof(h))) != cudaSuccess)
    return fail(OB_ERR_CUDA, cudaGetErrorString(e));
  return OB_OK;
}

extern "C" const char* ob_version(void) { return "odeblock-b200 0.1.0 (sm_100a)"; }
extern "C" const char* ob_last_error(void) { return g_err.c_str(); }

extern "C" int ob_device_count(int32_t* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
    return fail(OB_ERR_CUDA, cudaGetErrorString(e));
  }
  *count = n;
  return OB_OK;
}

extern "C" int ob_revolve_count(int32_t nt, int32_t nc, int64_t* out) {
  if (nt < 1 || nc < 1) return fail(OB_ERR_VALUE, "need nt >= 1 and nc >= 1");
  *out = ob::revolve_count(nt, nc);
  return OB_OK;
}

extern "C" int ob_revolve_schedule(int32_t nt, int32_t nc, int32_t* actions, int64_t capacity,
                                   int64_t* n_actions) {
  if (nt < 1 || nc < 1) return fail(OB_ERR_VALUE, "need nt >= 1 and nc >= 1");
  auto acts = ob::revolve_schedule(nt, nc);
  *n_actions = (int64_t)acts.size();
  if (actions == nullptr) return OB_OK;
  if ((int64_t)acts.size() > capacity) return fail(OB_ERR_VALUE, "action buffer too small");
  for (size_t i = 0; i < acts.size(); ++i) {
    actions[4 * i + 0] = acts[i].kind;
    actions[4 * i + 1] = acts[i].step;
    actions[4 * i + 2] = acts[i].start;
    actions[4 * i + 3] = acts[i].stop;
  }
  return OB_OK;
}

// ===================================================================== plan
namespace {

struct Plan {
  int dtype = 0;
  size_t esz = 8;
  Dims d{};
  int R = 1, Rt = 4, LR = 1, tiles = 1;
  int req_rows = 0;               // ob_problem.tile_rows (0: planner's choice)
  bool need_jvp = false;
  bool theta = false;
  bool tc = false;                // tcgen05 tensor-core MLP tile (rk_tc.cu)
  bool tc_cnf = false;            // tcgen05 CNF tile (cnf_tc.cu)
  bool tc_conv = false;           // tcgen05 conv tile (conv_tc.cu)
  bool theta_cluster = false;     // theta kernels with the weights resident across a cluster
  int rk_cluster = 0;             // explicit-RK kernels on the cluster MLP (fp64 two-layer MLP fields): CTAs per cluster
  int cluster_rows = 0;           // ... rows per cluster the shared-memory layout is sized for
  long long cnf_log_rec = 0;      // tcgen05 CNF tile: bytes of one VJP record of the dW log
  int cnf_cluster = 1;            // tcgen05 CNF tile: CTAs per cluster sharing the weight stream
  int s_stages = 0;               // scheme stages (stage scratch sizing)
  int gmres_m = 0;
  size_t off_kry = 0, off_stats = 0, off_cnf = 0, off_state = 0, off_head = 0;
  long long cnf_stride = 0;
  long long krylov_stride = 0;
  SmemLayout sm{};
  size_t smem_bytes = 0;
  // checkpoint program
  int nbuf = 0, nsol = 0;
  std::vector<int> fwd_rec, fwd_sol, obs_k;
  std::vector<int4> prog;
  unsigned skip_vjp = 0;
  ob_counters cnt{};
  // workspace layout (byte offsets)
  size_t o_ts = 0, o_fr = 0, o_fs = 0, o_pg = 0, o_stat = 0, o_obs = 0;
  size_t off_blob = 0, blob_bytes = 0, off_w = 0, off_rec = 0, off_sol = 0, off_scr = 0,
         off_mu = 0, off_lp = 0, total = 0;
  size_t off_pk = 0;
  long long scratch_stride = 0;
  size_t smem_reserve = 0;        // static shared memory of the kernel family
  // adaptive stepping
  bool adaptive = false;
  int cap = 0, nseg = 0, obs0 = 0;
  std::vector<double> pts;
  size_t off_grid = 0, off_nacc = 0, off_ostep = 0;
};

constexpr size_t kSmemLimit = 227 * 1024;
constexpr size_t kAdaptiveStaticSmem = 6 * 1024;   // per-row controller state + reductions
inline size_t smem_cap(const Plan& P) { return kSmemLimit - P.smem_reserve; }

int check_field(const ob_field_desc& f) {
  if (f.dtype != OB_F32 && f.dtype != OB_F64) return fail(OB_ERR_VALUE, "dtype must be f32 or f64");
  if (f.n_layers < 1 || f.n_layers > OB_MAX_LAYERS)
    return fail(OB_ERR_VALUE, "n_layers must be in [1, 8]");
  for (int l = 0; l <= f.n_layers; ++l)
    if (f.widths[l] <= 0) return fail(OB_ERR_VALUE, "layer widths must be positive");
  const int N = f.widths[f.n_layers];
  if (f.widths[0] != N + (f.time_input ? 1 : 0))  // MlpSpec.__post_init__ (nn.py:53-58)
    return fail(OB_ERR_VALUE, "input width inconsistent with state dim and time_input");
  if (f.activation < 0 || f.activation > OB_ACT_SOFTPLUS) return fail(OB_ERR_VALUE, "unknown activation");
  if (f.kind != OB_FIELD_MLP && f.kind != OB_FIELD_STIFF && f.kind != OB_FIELD_CNF &&
      f.kind != OB_FIELD_CONV)
    return fail(OB_ERR_UNSUPPORTED, "field kind not built into this library version");
  if (f.kind == OB_FIELD_CONV) {
    if (f.n_layers != 2 || f.widths[0] != 65 || f.widths[1] != 64 || f.widths[2] != 64 ||
        !f.time_input || f.activation != OB_ACT_RELU)
      return fail(OB_ERR_UNSUPPORTED, "conv kernels are built for the 16x16x64 C3 block");
    if (f.dtype != OB_F32) return fail(OB_ERR_UNSUPPORTED, "conv kernels are built for fp32");
    if (f.n_params != 64LL * 9 * 65 + 64 + 64LL * 9 * 64 + 64)
      return fail(OB_ERR_VALUE, "n_params does not match the conv block");
    return OB_OK;
  }
  if (f.kind == OB_FIELD_CNF) {
    if (!f.time_input) return fail(OB_ERR_VALUE, "CNF field takes time as an input");
    if (f.dtype != OB_F32) return fail(OB_ERR_UNSUPPORTED, "CNF kernels are built for fp32");
    if (f.n_layers < 2) return fail(OB_ERR_VALUE, "CNF field needs a hidden layer");
  }
  if (f.kind == OB_FIELD_STIFF && f.time_input) return fail(OB_ERR_VALUE, "stiff field is autonomous");
  long long np = 0;
  for (int l = 0; l < f.n_layers; ++l) np += (long long)f.widths[l + 1] * f.widths[l] + f.widths[l + 1];
  if (np != f.n_params) return fail(OB_ERR_VALUE, "n_params does not match widths");
  return OB_OK;
}

int ld_quad_odd(int x) {  // >= x, multiple of 4, (ld/4) odd: conflict-free strided rows
  int l = (x + 3) & ~3;
  if (((l / 4) & 1) == 0) l += 4;
  return l;
}
int round_up(int x, int m) { return (x + m - 1) / m * m; }

void make_conv_dims(const ob_field_desc& f, Dims& d) {
  d = Dims{};
  d.L = 2;
  d.conv = 1;
  for (int l = 0; l <= 2; ++l) d.w[l] = f.widths[l];
  d.N = d.nin = d.ldn = 256 * 64;
  d.conv_cin[0] = 65;
  d.conv_cin[1] = 64;
  long long off = 0, mo = 0;
  for (int l = 0; l < 2; ++l) {
    d.woff[l] = off;
    d.boff[l] = off + 64LL * 9 * d.conv_cin[l];
    off = d.boff[l] + 64;
    d.ldm[l] = 9 * 68;
    d.mwoff[l] = mo;
    mo += 64LL * d.ldm[l];
    d.mboff[l] = mo;
    mo += 64;
  }
  d.n_mu = mo;
  d.pwoff[0] = 0;
  d.pwoff[1] = 64LL * 9 * 68;
  d.pwoff[2] = 2 * 64LL * 9 * 68;
  d.pwoff[3] = d.pwoff[2] + 9LL * 64 * 68;
  d.n_packed = d.pwoff[3] + 9LL * 64 * 68;
  d.act = f.activation;
  d.time_input = 1;
}

void make_dims(const ob_field_desc& f, int LR, Dims& d) {
  if (f.kind == OB_FIELD_CONV) {
    make_conv_dims(f, d);
    return;
  }
  const int CT = 4 * (32 / LR);
  d = Dims{};
  d.L = f.n_layers;
  d.cnf = f.kind == OB_FIELD_CNF;
  d.nin = f.widths[f.n_layers];
  d.N = d.nin + (d.cnf ? 1 : 0);           // CNF state carries the log-density Delta
  d.maxw = 0;
  for (int l = 0; l <= d.L; ++l) {
    d.w[l] = f.widths[l];
    d.lda[l] = ld_quad_odd(f.widths[l]);
    d.maxw = std::max(d.maxw, d.w[l]);
  }
  long long off = 0, po = 0, mo = 0;
  for (int l = 0; l < d.L; ++l) {
    const int K = d.w[l], Nn = d.w[l + 1], Kout = l == 0 ? d.nin : K;
    d.woff[l] = off;
    d.boff[l] = off + (long long)Nn * K;
    off = d.boff[l] + Nn;
    d.nrow[l] = round_up(Nn, CT);
    d.ldw[l] = ld_quad_odd(std::max(round_up(K, 4), round_up(Kout, CT)));
    d.pwoff[l] = po;
    po += (long long)d.nrow[l] * d.ldw[l];
    d.ldm[l] = round_up(K, 4);
    d.mwoff[l] = mo;
    mo += (long long)Nn * d.ldm[l];
    d.mboff[l] = mo;
    mo += round_up(Nn, 4);
  }
  d.n_packed = po;
  d.n_mu = mo;
  d.ldn = ld_quad_odd(d.N);
  d.act = f.activation;
  d.time_input = f.time_input;
  d.need_pre = !d.cnf && (f.activation == OB_ACT_GELU || f.activation == OB_ACT_SOFTPLUS);
  d.ldt = ld_quad_odd(d.maxw);
}

// shared-memory layout for Rt rows; weights staged in smem when they fit
void layout_smem(Plan& P) {
  const Dims& d = P.d;
  if (P.theta) {   // Krylov workspace of the tile: Q | H | cs | sn | g | y per row
    const long long m = P.gmres_m;
    P.krylov_stride = (long long)P.R * ((m + 1) * d.ldn + (m + 1) * m + 2 * m + (m + 1) + m);
  }
  SmemLayout& s = P.sm;
  int o = 0;
  auto take = [&](long long n) { int r = o; o += (int)((n + 7) & ~7LL); return r; };  // 32 B aligned
  if (d.conv) {   // two zero-halo image tiles; state buffers live in global memory
    s = SmemLayout{};
    s.x0 = take(18 * 18 * 68);
    for (int l = 0; l < OB_MAX_LAYERS; ++l) s.hid[l] = s.pre[l] = -1;
    s.hid[0] = take(18 * 18 * 68);
    s.tA = s.tB = s.u = s.lam = s.lamn = s.w = s.jtv = s.aux = s.wts = s.ks = s.ring = s.hscr = -1;
    s.ring_elems = s.hscr_elems = 0;
    for (int i = 0; i < 8; ++i) s.vec[i] = -1;
    // double-buffered tap weights (2 x 64 x 68) for the staged conv GEMMs, when they fit
    if ((size_t)(o + 2 * 64 * 68) * P.esz <= smem_cap(P) && !getenv("OB_CONV_UNSTAGED")) s.tA = take(2 * 64 * 68);
    s.total = o;
    P.smem_bytes = (size_t)o * P.esz;
    return;
  }
  const int Rm = d.cnf ? 2 * P.Rt : P.Rt;   // MLP rows (CNF: forward + tangent rows)
  s.x0 = take((long long)Rm * d.lda[0]);
  for (int l = 0; l < OB_MAX_LAYERS; ++l) {
    s.hid[l] = (l < d.L - 1) ? take((long long)Rm * d.lda[l + 1]) : -1;
    s.pre[l] = (l < d.L - 1 && d.need_pre) ? take((long long)Rm * d.lda[l + 1]) : -1;
  }
  s.aux = d.cnf ? take((long long)Rm * d.lda[d.L]) : -1;
  s.tA = P.need_jvp ? take((long long)P.Rt * d.ldt) : -1;
  s.tB = P.need_jvp ? take((long long)P.Rt * d.ldt) : -1;
  s.u = take((long long)P.Rt * d.ldn);
  s.lam = take((long long)P.Rt * d.ldn);
  s.lamn = take((long long)P.Rt * d.ldn);
  s.w = take((long long)P.Rt * d.ldn);
  s.jtv = take((long long)P.Rt * d.ldn);
  for (int i = 0; i < 8; ++i) s.vec[i] = P.theta ? take((long long)P.Rt * d.ldn) : -1;
  s.scr = s.kry = -1;
  s.scr_elems = 0;
  if (P.theta) {
    s.scr_elems = 8 * P.Rt * d.ldn;     // up to 8 split-K partials of a state-wide product
    s.scr = take(s.scr_elems);
    // The Krylov basis stays in global memory by default: the L1 capacity it would
    // take caches the streamed weights, which matters more (measured on C5)
    if ((size_t)(o + P.krylov_stride) * P.esz <= smem_cap(P) && getenv("OB_KRYLOV_SMEM"))
      s.kry = take(P.krylov_stride);
  }
  s.total = o;
  s.wts = -1;
  // fp32 explicit-RK MLP / stiff weights are staged in shared memory when
  // they fit; fp64, theta-method and CNF kernels read L1/L2-resident weights
  // (only rk_f32s.cu instantiates the shared-memory-weight variants)
  const bool ws_variant = P.esz == 4 && !P.theta && !d.cnf && !d.conv;
  if (ws_variant && (size_t)(o + d.n_packed) * P.esz <= smem_cap(P) && !getenv("OB_NO_SMEM_WEIGHTS")) {
    s.wts = take(d.n_packed);
    s.total = o;
  }
  // hidden-layer split-K partials for tiny explicit-RK MLP tiles (4 slices of the widest layer)
  s.hscr = -1;
  s.hscr_elems = 0;
  if (!P.theta && !d.cnf && !getenv("OB_NO_HSPLIT")) {
    const long long n = 4LL * P.Rt * d.maxw;
    if ((size_t)(o + n) * P.esz + 4096 <= smem_cap(P)) {
      s.hscr = take(n);
      s.hscr_elems = (int)n;
      s.total = o;
    }
  }
  // per-warp cp.async rings for weights streamed from L2 (weights not staged in smem)
  s.ring = -1;
  s.ring_elems = 0;
  if (s.wts < 0 && !getenv("OB_NO_WRING")) {
    const long long ctw = 4LL * (32 / P.LR);                  // widest column tile
    const long long kd = P.esz == 4 ? 4 : 2;                  // RingDepth (gemm.cuh)
    const long long want = (kThreads / 32) * kd * ctw * 4;
    // leave 4 KB for the kernels' static shared memory (reductions, flags)
    const long long avail = (long long)((smem_cap(P) - 4096) / P.esz) - o;
    long long n = std::min(want, avail) / 64 * 64;
    if (n >= (kThreads / 32) * kd * 64) {
      s.ring = take(n);
      s.ring_elems = (int)n;
      s.total = o;
    }
  }
  // explicit-RK stage scratch (k_i forward, Lambda_i reverse) in shared memory when it
  // fits beside everything else: the stage sums then read it without L2 latency
  s.ks = -1;
  const long long kscr = 2LL * P.s_stages * P.Rt * d.ldn;
  if (!P.theta && P.s_stages > 0 && (size_t)(o + kscr) * P.esz <= smem_cap(P) && !getenv("OB_KS_GLOBAL")) {
    s.ks = take(kscr);
    s.total = o;
  }
  P.smem_bytes = (size_t)s.total * P.esz;
}

int pick_lr(int R) { return R <= 4 ? 1 : R <= 8 ? 2 : 8; }

void choose_tiles(Plan& P, const ob_field_desc& f, long long B, int sm_count) {
  int R = (int)std::max<long long>(1, (B + sm_count - 1) / sm_count);
  if (f.kind == OB_FIELD_CONV) {   // one sample (a 64 KB image) per CTA
    P.R = P.Rt = P.LR = 1;
    make_dims(f, 1, P.d);
    layout_smem(P);
    P.tiles = (int)B;
    return;
  }
  if (P.req_rows > 0) R = P.req_rows;
  if (f.kind == OB_FIELD_CNF) {  // stacked forward|tangent rows: 2*Rt = 4*LR
    for (R = std::min(R, 16);; R = std::max(1, R / 2)) {
      P.LR = R <= 4 ? 2 : R <= 8 ? 4 : 8;
      P.Rt = 2 * P.LR;
      P.R = std::min(R, P.Rt);
      make_dims(f, P.LR, P.d);
      layout_smem(P);
      if (P.smem_bytes <= smem_cap(P) || R == 1) break;
    }
    P.tiles = (int)((B + P.R - 1) / P.R);
    return;
  }
  R = std::min(R, P.esz == 8 ? 8 : 32);   // fp64 kernels are built for tiles of <= 8 rows
  for (;;) {
    P.R = R;
    P.LR = pick_lr(R);
    P.Rt = round_up(R, 4 * P.LR);
    make_dims(f, P.LR, P.d);
    layout_smem(P);
    if (P.smem_bytes <= smem_cap(P) || R == 1) break;
    R = std::max(1, R * 3 / 4);
  }
  P.tiles = (int)((B + P.R - 1) / P.R);
}

// Tensor-core tile: fp32 two-layer MLP field on an explicit fixed-step scheme.
// Tiles of <= 32 samples (the MMA N), generic state buffers then the tcgen05
// region (staged weights + operand tiles) in shared memory.
bool tc_eligible(const ob_problem& p, const Plan& P) {
  const ob_field_desc& f = p.field;
  if (P.esz != 4 || P.theta || P.adaptive || f.kind != OB_FIELD_MLP || f.n_layers != 2) return false;
  // smooth activations only: ReLU' jumps at 0 and the ~2^-16 split-product error moves
  // pre-activations across it (measured 3.7e-4 on du0), so ReLU keeps the fp32 SIMT tile
  if (f.activation != OB_ACT_TANH && f.activation != OB_ACT_IDENTITY) return false;
  if ((p.flags & OB_FLAG_NO_TENSOR_CORES) || getenv("OB_NO_TC")) return false;
  // stage derivatives live in TMEM slots 0..5 during reverse-sweep replays: stages >= 6
  // must be ones a replay never evaluates (b_i = 0 and a_ji = 0 for j > i; dopri5's 7th)
  const int s = p.scheme.stages;
  for (int i = 6; i < s; ++i) {
    bool unused = p.scheme.b[i] == 0.0;
    for (int j = i + 1; j < s && unused; ++j) unused = p.scheme.a[j * OB_MAX_STAGES + i] == 0.0;
    if (!unused) return false;
  }
  const int N = f.widths[2];
  return tc_shape_supported(N, f.widths[1], N);
}

bool plan_tc(Plan& P, const ob_field_desc& f, long long B, int sm_count) {
  Plan Q = P;
  int R = (int)std::max<long long>(1, (B + sm_count - 1) / sm_count);
  if (P.req_rows > 0) R = P.req_rows;
  R = std::min(R, 32);
  Q.R = Q.Rt = R;
  Q.LR = 8;
  make_dims(f, Q.LR, Q.d);
  unsigned packed = 0, total = 0;
  tc_sizes(Q.d.N, f.widths[1], Q.d.N, &packed, &total);
  Q.d.n_packed = packed / 4;
  for (int l = 0; l < OB_MAX_LAYERS; ++l) Q.d.pwoff[l] = 0;
  SmemLayout& s = Q.sm;
  s = SmemLayout{};
  int o = 0;
  auto take = [&](long long n) { int r = o; o += (int)((n + 7) & ~7LL); return r; };
  s.x0 = s.tA = s.tB = s.aux = s.scr = s.kry = s.ks = s.ring = s.hscr = -1;
  s.ring_elems = s.hscr_elems = 0;
  for (int l = 0; l < OB_MAX_LAYERS; ++l) s.hid[l] = s.pre[l] = -1;
  for (int i = 0; i < 8; ++i) s.vec[i] = -1;
  s.scr_elems = 0;
  s.wts = take(total / 4);   // the tcgen05 region first: constant operand addresses
  s.u = take((long long)Q.Rt * Q.d.ldn);
  s.lam = take((long long)Q.Rt * Q.d.ldn);
  s.lamn = take((long long)Q.Rt * Q.d.ldn);
  s.w = take((long long)Q.Rt * Q.d.ldn);
  s.jtv = take((long long)Q.Rt * Q.d.ldn);
  s.total = o;
  Q.smem_bytes = (size_t)o * 4;
  if (Q.smem_bytes > smem_cap(Q)) return false;
  Q.tiles = (int)((B + R - 1) / R);
  Q.tc = true;
  P = Q;
  return true;
}

// Tensor-core CNF tile: fp32 softplus CNF field of the C4 shape on an explicit scheme.
bool tc_cnf_eligible(const ob_field_desc& f, int flags) {
  if (f.kind != OB_FIELD_CNF || f.dtype != OB_F32 || f.n_layers != 3 || f.activation != OB_ACT_SOFTPLUS)
    return false;
  if ((flags & OB_FLAG_NO_TENSOR_CORES) || getenv("OB_NO_TC")) return false;
  const int D = f.widths[3], H = f.widths[1];
  return f.widths[0] == D + 1 && f.widths[2] == H && tc_cnf_shape(D, H);
}

// <= 8 samples per CTA (the tile's N = 16 stacks forward and tangent rows); generic
// state buffers after the tcgen05 region, stage scratch in global memory
bool plan_tc_cnf(Plan& P, const ob_field_desc& f, long long B, int sm_count) {
  Plan Q = P;
  int R = (int)std::max<long long>(1, (B + sm_count - 1) / sm_count);
  if (P.req_rows > 0) R = P.req_rows;
  R = std::min(R, 8);
  Q.R = R;
  Q.Rt = 8;
  Q.LR = 2;
  make_dims(f, Q.LR, Q.d);
  unsigned packed = 0, total = 0, rec = 0;
  tc_cnf_sizes(&packed, &total, &rec);
  Q.d.n_packed = packed / 4;
  for (int l = 0; l < OB_MAX_LAYERS; ++l) Q.d.pwoff[l] = 0;
  SmemLayout& s = Q.sm;
  s = SmemLayout{};
  int o = 0;
  auto take = [&](long long n) { int r = o; o += (int)((n + 7) & ~7LL); return r; };
  s.x0 = s.tA = s.tB = s.aux = s.scr = s.kry = s.ks = s.ring = s.hscr = s.wts = -1;
  s.ring_elems = s.hscr_elems = s.scr_elems = 0;
  for (int l = 0; l < OB_MAX_LAYERS; ++l) s.hid[l] = s.pre[l] = -1;
  for (int i = 0; i < 8; ++i) s.vec[i] = -1;
  take(total / 4);   // the tcgen05 region first (offset 0)
  s.u = take((long long)Q.Rt * Q.d.ldn);
  s.lam = take((long long)Q.Rt * Q.d.ldn);
  s.lamn = take((long long)Q.Rt * Q.d.ldn);
  s.w = take((long long)Q.Rt * Q.d.ldn);
  s.jtv = take((long long)Q.Rt * Q.d.ldn);
  s.total = o;
  Q.smem_bytes = (size_t)o * 4;
  if (Q.smem_bytes > smem_cap(Q)) return false;
  // clusters of CTAs share the weight stream (TMA multicast); pad to whole clusters
  int cl = 2;
  if (const char* e = getenv("OB_CNF_CLUSTER")) cl = atoi(e);   // experiments: 1, 2, 4
  if (cl != 1 && cl != 2 && cl != 4) cl = 2;
  Q.cnf_cluster = cl;
  Q.tiles = (int)(((B + R - 1) / R + cl - 1) / cl * cl);
  Q.tc_cnf = true;
  Q.cnf_log_rec = rec;
  P = Q;
  return true;
}

// Theta methods on fp64 two-layer MLP / stiff fields: clusters of 8 CTAs keep the weights
// in shared memory (hidden units split across the cluster) instead of streaming them from
// L2 for every Krylov operator product.  2 rows per CTA (16 per cluster).
bool theta_cluster_eligible(const ob_problem& p, const Plan& P) {
  const ob_field_desc& f = p.field;
  if (!P.theta || P.adaptive || P.esz != 8) return false;
  if (f.kind != OB_FIELD_MLP && f.kind != OB_FIELD_STIFF) return false;
  if (f.n_layers != 2 || f.time_input) return false;
  // act' from the activation value (tanh, identity, relu)
  if (f.activation != OB_ACT_TANH && f.activation != OB_ACT_IDENTITY && f.activation != OB_ACT_RELU) return false;
  const int N = f.widths[2], H = f.widths[1];
  // fp64 MMA tiles over swizzled rows: state dim and hidden slice multiples of 16, >= 32
  if (N % 16 || N < 32 || N > 128 || H % 128 || H < 256) return false;
  if (p.tile_rows != 0 && p.tile_rows != 2) return false;
  if (p.batch < 16) return false;   // a cluster holds 16 rows: tiny batches keep the single-CTA kernels
  if ((p.flags & OB_FLAG_NO_TENSOR_CORES) || getenv("OB_NO_THETA_CLUSTER")) return false;
  return true;
}

// Geometry: the batch is dealt evenly to ncl clusters and a cluster's rows evenly to its 8
// CTAs.  16 rows per cluster (2 per CTA) when that many clusters are resident at once;
// otherwise as many clusters as fit with up to 18 rows each (3 per CTA at most: the
// shared-memory budget), so the sweep still runs as ONE wave (C5: 256 rows on 15 clusters
// of 17-18); beyond that, waves of 16-row clusters.
bool plan_theta_cluster(Plan& P, const ob_field_desc& f, long long B) {
  auto layout = [&](Plan& Q, int R, int RC) {
    Q.R = Q.Rt = R;
    Q.LR = 1;
    make_dims(f, 1, Q.d);
    int region = 0, cl = 0;
    theta_cluster_geom(Q.d.N, f.widths[1], R, RC, false, &region, &cl);
    const long long m = Q.gmres_m;
    Q.krylov_stride = (long long)R * ((m + 1) * Q.d.ldn + (m + 1) * m + 2 * m + (m + 1) + m);
    SmemLayout& s = Q.sm;
    s = SmemLayout{};
    int o = 0;
    auto take = [&](long long n) { int r = o; o += (int)((n + 1) & ~1LL); return r; };
    s.x0 = s.tA = s.tB = s.aux = s.scr = s.kry = s.ks = s.ring = s.hscr = -1;
    s.lamn = s.w = -1;
    s.ring_elems = s.hscr_elems = s.scr_elems = 0;
    for (int l = 0; l < OB_MAX_LAYERS; ++l) s.hid[l] = s.pre[l] = -1;
    const long long v = (long long)Q.Rt * Q.d.ldn;
    s.u = take(v);
    s.lam = take(v);
    for (int i = 0; i < 8; ++i) s.vec[i] = take(v);
    s.jtv = s.vec[6];       // the adjoint sweep's product buffer shares the forward's f buffer
    s.wts = take(region);   // the cluster region (weight slices, exchange buffers)
    s.total = o;
    Q.smem_bytes = (size_t)o * 8;
    Q.smem_reserve = 3072;  // static shared memory of the theta context
    return Q.smem_bytes <= smem_cap(Q);
  };
  Plan Q = P;
  if (!layout(Q, 2, 16)) return false;
  const int max_active = theta_cluster_max_active(Q.smem_bytes);
  if (max_active < 1) return false;
  long long ncl = (B + 15) / 16;
  int rc = 16;
  if (ncl > max_active) {
    const long long per = (B + max_active - 1) / max_active;   // rows per cluster in one wave
    Plan Q2 = P;
    if (per <= 24 && layout(Q2, (int)((per + 7) / 8), (int)per) &&
        theta_cluster_max_active(Q2.smem_bytes) >= max_active) {
      Q = Q2;
      ncl = max_active;
      rc = (int)per;
    }
  }
  Q.tiles = (int)ncl * 8;
  Q.cluster_rows = rc;
  Q.theta_cluster = true;
  P = Q;
  return true;
}

// Explicit fixed-step schemes on fp64 two-layer MLP fields without a time input (C1): the
// generic RK kernels with the cluster MLP adapter -- the weights stay in the shared memory
// of 8 CTAs (hidden units split), and the batch is sized to ONE wave of resident clusters.
bool rk_cluster_eligible(const ob_problem& p, const Plan& P) {
  const ob_field_desc& f = p.field;
  if (P.theta || P.adaptive || P.esz != 8 || f.kind != OB_FIELD_MLP) return false;
  if (f.n_layers != 2 || f.time_input) return false;
  if (f.activation != OB_ACT_TANH && f.activation != OB_ACT_IDENTITY && f.activation != OB_ACT_RELU) return false;
  const int N = f.widths[2], H = f.widths[1];
  // fp64 MMA tiles over swizzled rows: state dim and hidden slice multiples of 16, >= 32
  if (N % 16 || N < 32 || N > 128 || H % 128 || H < 256) return false;
  if (p.tile_rows != 0) return false;
  if (p.batch < 32) return false;
  if (p.n_obs > 0) return false;   // (observation losses keep the single-CTA tiles)
  if ((p.flags & OB_FLAG_NO_TENSOR_CORES) || getenv("OB_NO_RK_CLUSTER")) return false;
  return true;
}

// Cluster size: two CTAs when half of both weight matrices fits one CTA's shared memory and its
// parameter-cotangent tiles fit the warps' registers (8 warps x 8 tiles of 8 x 16 per matrix:
// N H / 2 <= 8192) -- an eighth of the exchange traffic and no row-tile padding; else eight.
bool plan_rk_cluster(Plan& P, const ob_field_desc& f, long long B) {
  auto attempt = [&](int CL) {
    auto geom = CL == 2 ? rk_cluster2_geom : rk_cluster8_geom;
    auto max_act = CL == 2 ? rk_cluster2_max_active : rk_cluster8_max_active;
    auto layout = [&](Plan& Q, int R) {
      Q.R = Q.Rt = R;
      Q.LR = 1;
      make_dims(f, 1, Q.d);
      int region = 0;
      geom(Q.d.N, f.widths[1], R, &region);
      SmemLayout& s = Q.sm;
      s = SmemLayout{};
      int o = 0;
      auto take = [&](long long n) { int r = o; o += (int)((n + 1) & ~1LL); return r; };
      s.tA = s.tB = s.scr = s.kry = s.ring = s.hscr = s.wts = -1;
      s.ring_elems = s.hscr_elems = s.scr_elems = 0;
      for (int l = 0; l < OB_MAX_LAYERS; ++l) s.hid[l] = s.pre[l] = -1;
      for (int i = 0; i < 8; ++i) s.vec[i] = -1;
      const long long v = (long long)Q.Rt * Q.d.ldn;
      s.x0 = take((long long)Q.Rt * Q.d.lda[0]);
      s.u = take(v);
      s.lam = take(v);
      s.lamn = take(v);
      s.w = take(v);
      s.jtv = take(v);
      s.ks = take(2LL * Q.s_stages * v);
      s.aux = take(region);   // the cluster region (weight slices, exchange buffers)
      s.total = o;
      Q.smem_bytes = (size_t)o * 8;
      return Q.smem_bytes + 1024 <= smem_cap(Q);
    };
    Plan Q = P;
    if (!layout(Q, 2)) return false;
    const int max_active = max_act(Q.smem_bytes);
    if (max_active < 1) return false;
    // rows per CTA so that the batch is one wave of resident clusters (<= 6: the tiles' row groups)
    int R = (int)((B + (long long)CL * max_active - 1) / ((long long)CL * max_active));
    R = std::max(2, std::min(R, 6));
    Plan Q2 = P;
    if (!layout(Q2, R) || max_act(Q2.smem_bytes) < 1) return false;
    Q2.tiles = (int)(((B + R - 1) / R + CL - 1) / CL * CL);
    Q2.rk_cluster = CL;
    P = Q2;
    return true;
  };
  const long long N = f.widths[2], H = f.widths[1];
  if (!getenv("OB_RK_CLUSTER8") && H % 32 == 0 && N * H / 2 <= 8192 && attempt(2)) return true;
  return attempt(8);
}

// Tensor-core conv tile: the C3 block on an explicit fixed-step scheme, one image per CTA.
bool tc_conv_eligible(const ob_field_desc& f, int flags) {
  if (f.kind != OB_FIELD_CONV || f.dtype != OB_F32) return false;
  return !((flags & OB_FLAG_NO_TENSOR_CORES) || getenv("OB_NO_TC"));
}

bool plan_tc_conv(Plan& P, const ob_field_desc& f, long long B) {
  Plan Q = P;
  Q.R = Q.Rt = Q.LR = 1;
  make_dims(f, 1, Q.d);
  unsigned packed = 0, total = 0;
  tc_conv_sizes(&packed, &total);
  Q.d.n_packed = packed / 4;
  SmemLayout& s = Q.sm;
  s = SmemLayout{};
  s.x0 = s.tA = s.tB = s.aux = s.scr = s.kry = s.ks = s.ring = s.hscr = s.wts = -1;
  s.u = s.lam = s.lamn = s.w = s.jtv = -1;   // state buffers in global memory
  s.ring_elems = s.hscr_elems = s.scr_elems = 0;
  for (int l = 0; l < OB_MAX_LAYERS; ++l) s.hid[l] = s.pre[l] = -1;
  for (int i = 0; i < 8; ++i) s.vec[i] = -1;
  s.total = (int)(total / 4);
  Q.smem_bytes = total;
  if (Q.smem_bytes > smem_cap(Q)) return false;
  Q.tiles = (int)B;
  Q.tc_conv = true;
  P = Q;
  return true;
}

// compile the checkpoint policy into forward store directives + a reverse
// program (checkpointing.py:242-340), with reference-semantics counters.
int compile_policy(const ob_problem& p, Plan& P) {
  const int nt = p.n_steps, s = p.scheme.stages;
  P.fwd_rec.assign(nt, -1);
  P.fwd_sol.assign(nt, -1);
  P.prog.clear();
  ob_counters& c = P.cnt;
  auto replay = [&](int n, int src_kind, int src, int dst) {
    P.prog.push_back(make_int4(kOpReplay, n, (src_kind << 24) | src, dst));
    c.steps_recomputed += 1;
    c.recomputed_steps += 1;
  };
  auto reverse = [&](int n, int buf) { P.prog.push_back(make_int4(kOpReverse, n, 0, buf)); };

  if (p.policy == OB_POLICY_STORE_ALL) {
    P.nbuf = nt;
    for (int n = 0; n < nt; ++n) P.fwd_rec[n] = n;
    for (int n = nt - 1; n >= 0; --n) reverse(n, n);
    c.stored_states = nt - 1;
    c.stored_stage_vectors = (long long)(nt - 1) * s;
    c.max_live_slots = nt - 1;
  } else if (p.policy == OB_POLICY_STORE_SOLUTIONS) {
    P.nbuf = 1;
    P.nsol = std::max(nt - 1, 0);
    for (int n = 0; n < nt - 1; ++n) P.fwd_sol[n] = n;
    P.fwd_rec[nt - 1] = 0;
    reverse(nt - 1, 0);
    for (int n = nt - 2; n >= 0; --n) {
      replay(n, kSrcSol, n, 0);
      reverse(n, 0);
    }
    c.stored_states = nt - 1;
    c.max_live_slots = nt - 1;
  } else if (p.policy == OB_POLICY_REVOLVE) {
    if (p.nc < 1) return fail(OB_ERR_VALUE, "revolve requires nc >= 1");
    auto acts = ob::revolve_schedule(nt, p.nc);
    size_t first = 0;
    while (acts[first].kind != kReverse) ++first;
    // physical record buffers with reference counts (slots + the record in hand)
    std::vector<int> refc;
    auto alloc = [&]() {
      for (size_t i = 0; i < refc.size(); ++i)
        if (refc[i] == 0) { refc[i] = 1; return (int)i; }
      refc.push_back(1);
      return (int)refc.size() - 1;
    };
    std::map<int, int> slot;  // step -> buffer
    int live_peak = 0;
    for (size_t i = 0; i < first; ++i)
      if (acts[i].kind == kStore) {
        const int b = alloc();
        slot[acts[i].step] = b;
        P.fwd_rec[acts[i].step] = b;
        c.stored_states += 1;
        c.stored_stage_vectors += s;
        live_peak = std::max(live_peak, (int)slot.size());
      }
    int hand = -1, hand_step = nt - 1;
    if (P.fwd_rec[nt - 1] >= 0) { hand = P.fwd_rec[nt - 1]; refc[hand] += 1; }
    else { hand = alloc(); P.fwd_rec[nt - 1] = hand; }
    int src_kind = kSrcRecNext, src = hand;  // executor position after the forward sweep
    auto drop_hand = [&]() { if (hand >= 0) { refc[hand] -= 1; hand = -1; hand_step = -2; } };
    for (size_t i = first; i < acts.size(); ++i) {
      const Action& a = acts[i];
      if (a.kind == kRestore) {
        if (a.step == -1) { src_kind = kSrcU0; src = 0; }
        else { src_kind = kSrcRecNext; src = slot.at(a.step); }
        drop_hand();
      } else if (a.kind == kAdvance) {
        for (int n = a.start; n < a.stop; ++n) {
          int dst;
          if (hand >= 0 && refc[hand] == 1) dst = hand;  // only the hand holds it: reuse
          else { drop_hand(); dst = alloc(); }
          hand = dst;
          replay(n, src_kind, src, dst);
          hand_step = n;
          src_kind = kSrcRecNext;
          src = dst;
        }
      } else if (a.kind == kStore) {
        if (hand < 0 || hand_step != a.step) return fail(OB_ERR_VALUE, "schedule bug: no record in hand");
        slot[a.step] = hand;
        refc[hand] += 1;
        live_peak = std::max(live_peak, (int)slot.size());
      } else {  // reverse
        int buf;
        if (hand >= 0 && hand_step == a.step) buf = hand;
        else {
          auto it = slot.find(a.step);
          if (it == slot.end()) return fail(OB_ERR_VALUE, "schedule bug: record unavailable");
          buf = it->second;
          refc[buf] -= 1;
          slot.erase(it);
          // the buffer stays readable for this op; it can only be reused by a later replay
        }
        reverse(a.step, buf);
      }
    }
    P.nbuf = (int)refc.size();
    c.max_live_slots = live_peak;
  } else {
    return fail(OB_ERR_VALUE, "unknown checkpoint policy");
  }
  return OB_OK;
}

int plan_problem(const ob_problem& p, Plan& P, bool allow_tc = false) {
  int st = check_field(p.field);
  if (st) return st;
  P.theta = (p.scheme.kind == OB_SCHEME_THETA);
  if (P.theta) {
    if (!(p.scheme.theta > 0.0 && p.scheme.theta <= 1.0)) return fail(OB_ERR_VALUE, "theta must lie in (0, 1]");
    if (p.scheme.stages != 2) return fail(OB_ERR_VALUE, "theta schemes carry 2 stage states");
    const ob_solver_cfg& sc = p.solver;
    if (!(sc.newton_tol > 0 && sc.newton_tol < 1 && sc.gmres_tol > 0 && sc.gmres_tol < 1))
      return fail(OB_ERR_VALUE, "tolerances must lie in (0, 1)");
    if (sc.newton_maxit < 1 || sc.gmres_maxit < 1 || sc.gmres_restart < 1)
      return fail(OB_ERR_VALUE, "iteration caps must be >= 1");
    P.need_jvp = true;
  } else if (p.scheme.kind != OB_SCHEME_RK) {
    return fail(OB_ERR_VALUE, "unknown scheme kind");
  }
  if (p.scheme.stages < 1 || p.scheme.stages > OB_MAX_STAGES) return fail(OB_ERR_VALUE, "bad stage count");
  P.adaptive = p.adaptive != 0;
  if (p.batch < 1) return fail(OB_ERR_VALUE, "batch must be >= 1");
  if (p.tile_rows < 0) return fail(OB_ERR_VALUE, "tile_rows must be >= 0");
  P.req_rows = p.tile_rows;
  const bool seed = p.loss == OB_LOSS_SEED;
  const bool obs = p.loss == OB_LOSS_OBS_MSE || p.loss == OB_LOSS_OBS_MAE || (seed && p.n_obs > 0);
  const bool vec_field = p.field.kind == OB_FIELD_MLP || p.field.kind == OB_FIELD_STIFF;
  if (seed && p.n_obs > 0 && !vec_field && p.adaptive)
    return fail(OB_ERR_UNSUPPORTED, "adaptive stepping is built for MLP / stiff fields");
  if (p.loss != OB_LOSS_HALF_SQNORM && p.loss != OB_LOSS_MSE && !(obs && vec_field) && !seed &&
      !(p.loss == OB_LOSS_CNF_NLL && p.field.kind == OB_FIELD_CNF) &&
      !(p.loss == OB_LOSS_CE_HEAD && p.field.kind == OB_FIELD_CONV))
    return fail(OB_ERR_UNSUPPORTED, "loss kind not supported for this field");
  P.obs_k.clear();
  if (P.adaptive) {
    // AdaptiveController / integrate / forward_pass checks (integrators.py:187-193,
    // :297-299; adjoint.py:165-166; checkpointing.py:218-220)
    if (!(p.abstol > 0 && p.reltol > 0)) return fail(OB_ERR_VALUE, "tolerances must be positive");
    if (!(p.h_min <= p.h_init && p.h_init <= p.h_max))
      return fail(OB_ERR_VALUE, "need h_min <= h_init <= h_max");
    if (!(p.tF > p.t0)) return fail(OB_ERR_VALUE, "tF must exceed t0");
    if (p.policy == OB_POLICY_REVOLVE)
      return fail(OB_ERR_VALUE, "revolve checkpointing needs fixed stepping");
    if (P.theta || !p.scheme.has_emb || p.scheme.order < 1)
      return fail(OB_ERR_INTEGRATION, "adaptive mode needs an embedded explicit scheme");
    if (!vec_field) return fail(OB_ERR_UNSUPPORTED, "adaptive stepping is built for MLP / stiff fields");
    if (p.max_accepted < 1) return fail(OB_ERR_VALUE, "max_accepted must be >= 1");
    if (p.max_steps < 1) return fail(OB_ERR_VALUE, "max_steps must be >= 1");
    P.cap = p.max_accepted;
    // observation intervals: [t0] + obs > t0 (+ tF)
    std::vector<double> ot;
    if (obs) {
      if (p.n_obs < 1 || !p.obs_times) return fail(OB_ERR_VALUE, "need one observation vector per time");
      for (int k = 0; k < p.n_obs; ++k) {
        if (k > 0 && !(p.obs_times[k] > p.obs_times[k - 1]))
          return fail(OB_ERR_VALUE, "observation times must be strictly increasing");
        if (p.obs_times[k] > p.tF + 1e-9 * std::max(1.0, std::fabs(p.tF)))
          return fail(OB_ERR_VALUE, "observations extend past the final time");
        ot.push_back(p.obs_times[k]);
      }
    }
    P.pts.assign(1, p.t0);
    for (double t : ot)
      if (t > p.t0) P.pts.push_back(t);
    if (std::fabs(P.pts.back() - p.tF) > 1e-12 * std::max(1.0, std::fabs(p.tF))) P.pts.push_back(p.tF);
    P.nseg = (int)P.pts.size() - 1;
    P.obs0 = !ot.empty() && ot[0] == p.t0;
    if (obs) {
      P.obs_k.assign(P.nseg, -1);
      std::vector<int> seen(ot.size(), 0);
      if (P.obs0) seen[0] = 1;
      for (int sgm = 0; sgm < P.nseg; ++sgm) {
        const double b = P.pts[sgm + 1];
        for (size_t k = 0; k < ot.size(); ++k)
          if (std::fabs(b - ot[k]) <= 1e-9 * std::max(1.0, std::fabs(ot[k]))) {
            if (P.obs_k[sgm] < 0) P.obs_k[sgm] = (int)k;
            seen[k] = 1;
          }
      }
      for (int v : seen)   // loss_and_grad_seed (losses.py:85-86)
        if (!v) return fail(OB_ERR_VALUE, "one prediction per observation required");
    }
  } else {
    if (p.n_steps < 1) return fail(OB_ERR_VALUE, "fixed mode requires at least one step");
    if (!p.times) return fail(OB_ERR_VALUE, "times array is required");
    for (int i = 0; i < p.n_steps; ++i)
      if (!(p.times[i + 1] > p.times[i])) return fail(OB_ERR_VALUE, "step size must be positive");
    if (obs) {  // LossSpec validation (losses.py:54-69) on boundary indices
      if (p.n_obs < 1 || !p.obs_steps) return fail(OB_ERR_VALUE, "need one observation vector per time");
      P.obs_k.assign(p.n_steps + 1, -1);
      for (int k = 0; k < p.n_obs; ++k) {
        const int j = p.obs_steps[k];
        if (j < 0 || j > p.n_steps) return fail(OB_ERR_VALUE, "observation boundary out of range");
        if (k > 0 && j <= p.obs_steps[k - 1])
          return fail(OB_ERR_VALUE, "observation times must be strictly increasing");
        P.obs_k[j] = k;
      }
    }
  }
  if ((p.field.kind == OB_FIELD_CNF || p.field.kind == OB_FIELD_CONV) &&
      p.scheme.kind != OB_SCHEME_RK)
    return fail(OB_ERR_UNSUPPORTED, "CNF / conv fields are built for explicit schemes");
  P.dtype = p.field.dtype;
  P.esz = P.dtype == OB_F32 ? 4 : 8;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
  } else {
    cudaGetLastError();
  }
  P.gmres_m = P.theta ? std::min(p.solver.gmres_restart, p.field.widths[p.field.n_layers]) : 0;
  P.smem_reserve = P.adaptive ? kAdaptiveStaticSmem : 0;
  P.s_stages = (P.adaptive || P.theta) ? 0 : p.scheme.stages;   // fixed explicit: smem stage scratch
  choose_tiles(P, p.field, p.batch, sms);
  if (allow_tc && tc_eligible(p, P)) plan_tc(P, p.field, p.batch, sms);
  if (allow_tc && !P.adaptive && tc_cnf_eligible(p.field, p.flags)) plan_tc_cnf(P, p.field, p.batch, sms);
  if (allow_tc && !P.adaptive && tc_conv_eligible(p.field, p.flags)) plan_tc_conv(P, p.field, p.batch);
  if (allow_tc && theta_cluster_eligible(p, P)) plan_theta_cluster(P, p.field, p.batch);
  if (allow_tc && rk_cluster_eligible(p, P)) plan_rk_cluster(P, p.field, p.batch);
  if (P.smem_bytes > smem_cap(P)) return fail(OB_ERR_UNSUPPORTED, "layer widths exceed shared memory");
  if (P.adaptive) {
    P.prog.clear();
    P.fwd_rec.assign(P.nseg, -1);
    P.fwd_sol.assign(P.nseg, -1);
    if (p.policy == OB_POLICY_STORE_ALL) {
      P.nbuf = P.cap;
      P.nsol = 0;
    } else if (p.policy == OB_POLICY_STORE_SOLUTIONS) {
      P.nbuf = 3;          // final-record ping-pong + replay slot
      P.nsol = P.cap;
    } else {
      return fail(OB_ERR_VALUE, "unknown checkpoint policy");
    }
  } else {
    st = compile_policy(p, P);
    if (st) return st;
  }
  // zero-cotangent stages: b_i == 0 and a_ji == 0 for all j > i  (dopri5 stage 7)
  const int s = p.scheme.stages;
  P.skip_vjp = 0;
  for (int i = 0; i < s && !P.theta; ++i) {
    bool zero = p.scheme.b[i] == 0.0;
    for (int j = i + 1; j < s && zero; ++j) zero = p.scheme.a[j * OB_MAX_STAGES + i] == 0.0;
    if (zero) P.skip_vjp |= 1u << i;
  }
  // reference-semantics NFE counters, per trajectory (integrators.py:83-102)
  ob_counters& c = P.cnt;
  const long long nt = P.adaptive ? P.nseg : p.n_steps;   // blob: fixed grid | interval ends
  c.nfe_forward = s * nt - (p.scheme.fsal ? nt - 1 : 0) + c.steps_recomputed * s;
  c.nfe_backward = s * nt;
  c.steps_accepted = nt;
  c.device_rhs_evals = c.nfe_forward;
  if (!P.theta && !P.adaptive) {
    // stages whose derivative no later stage and no update uses are not evaluated on the
    // device (dopri5 stage 7 outside the FSAL carry: replays and the final forward step)
    const long long unused = __builtin_popcount(P.skip_vjp);
    const bool carried = p.scheme.fsal && (P.skip_vjp >> (s - 1) & 1u);
    c.device_rhs_evals -= c.steps_recomputed * unused + (nt - 1) * (unused - (carried ? 1 : 0)) +
                          (nt > 0 ? unused : 0);
  }
  c.device_vjp_evals = (s - __builtin_popcount(P.skip_vjp)) * nt;
  if (P.theta) {  // data dependent: filled from the per-sample device counters after the run
    c.nfe_forward = c.nfe_backward = c.device_rhs_evals = c.device_vjp_evals = 0;
  }
  if (P.adaptive) c = ob_counters{};   // per-sample grids: filled after the run
  c.tile_rows = P.R;
  c.tiles = P.tiles;
  c.tensor_cores = (P.tc || P.tc_cnf || P.tc_conv) ? 1 : (P.theta_cluster || P.rk_cluster) ? 2 : 0;
  c.kernel_launches = 4;
  // workspace
  const long long B = p.batch, N = P.d.N;
  size_t o = 0;
  P.off_blob = o;
  P.o_ts = 0;
  P.o_fr = P.o_ts + sizeof(double) * (nt + 1);
  P.o_fs = P.o_fr + sizeof(int) * nt;
  P.o_pg = align_up(P.o_fs + sizeof(int) * nt, 16);
  P.o_stat = P.o_pg + sizeof(int4) * P.prog.size();
  P.o_obs = P.o_stat + sizeof(int) * 4;
  P.blob_bytes = P.o_obs + sizeof(int) * P.obs_k.size();
  o = align_up(o + P.blob_bytes, 256);
  P.off_pk = o;
  o = align_up(o + P.esz * (size_t)P.d.n_packed, 256);
  P.off_rec = o;
  o = align_up(o + P.esz * (size_t)P.nbuf * (s + 1) * B * N, 256);
  P.off_sol = o;
  o = align_up(o + P.esz * (size_t)P.nsol * B * N, 256);
  P.off_scr = o;
  P.scratch_stride = 2LL * s * P.Rt * P.d.ldn;
  o = align_up(o + P.esz * (size_t)P.tiles * P.scratch_stride, 256);
  P.off_mu = o;
  o = align_up(o + P.esz * (size_t)P.tiles * P.d.n_mu, 256);
  P.off_kry = o;
  if (P.theta && P.sm.kry < 0) o = align_up(o + P.esz * (size_t)P.tiles * P.krylov_stride, 256);
  P.off_stats = o;
  o = align_up(o + sizeof(int) * (size_t)p.batch * OB_NSTATS, 256);
  P.off_cnf = o;
  P.cnf_stride = 0;
  if (P.tc_cnf) {   // per-tile log of the deferred parameter cotangents: one record per VJP
    P.cnf_stride = std::max<long long>(1, c.device_vjp_evals) * P.cnf_log_rec / 4;
  } else if (P.d.cnf) {
    for (int l = 0; l < P.d.L - 1; ++l) P.cnf_stride += 2LL * P.Rt * P.d.lda[l + 1];
  } else if (P.tc_conv) {
    P.cnf_stride = 256LL * 64;       // the tile's field input (fp32 image)
  } else if (P.d.conv) {
    P.cnf_stride = 18LL * 18 * 68;   // parked input tile
  }
  o = align_up(o + P.esz * (size_t)P.tiles * P.cnf_stride, 256);
  P.off_state = o;
  if (P.sm.u < 0) o = align_up(o + P.esz * (size_t)P.tiles * 5 * P.Rt * P.d.ldn, 256);
  P.off_head = o;
  if (p.loss == OB_LOSS_CE_HEAD)   // partials + fp64 scratch (gap|dl|loss rows, dgap rows)
    o = align_up(o + P.esz * (size_t)P.tiles * (10 * 64 + 10) + 16 +
                     sizeof(double) * (size_t)P.tiles * 8 * (81 + 64), 256);
  P.off_lp = o;
  o = align_up(o + sizeof(double) * P.tiles, 256);
  if (P.adaptive) {
    P.off_grid = o;
    o = align_up(o + sizeof(double) * 2 * (size_t)B * P.cap, 256);
    P.off_nacc = o;
    o = align_up(o + sizeof(int) * (size_t)B, 256);
    P.off_ostep = o;
    o = align_up(o + sizeof(int) * (size_t)B * std::max(p.n_obs, 1), 256);
  }
  P.total = o;
  return OB_OK;
}

thread_local std::chrono::steady_clock::time_point g_t_entry;   // OB_HOST_TIMING

// phases of one gradient problem on one workspace (ob_grad runs both)
enum { kPhaseForward = 1, kPhaseReverse = 2, kPhaseBoth = 3 };

// per-device CUDA events of the phase timeline (created on first use on each device)
static cudaError_t phase_events(cudaEvent_t*& ev) {
  static thread_local std::map<int, std::vector<cudaEvent_t>> evs;
  std::vector<cudaEvent_t>& v = evs[current_device()];
  if (v.empty()) {
    v.assign(5, nullptr);
    for (auto& e : v) {
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) {
        evs.erase(current_device());
        return r;
      }
    }
  }
  ev = v.data();
  return cudaSuccess;
}

template <typename T>
int run_grad(const ob_problem& p, const ob_buffers& b, Plan& P, cudaStream_t st,
             const void* cadj_dphi = nullptr, int phases = kPhaseBoth) {
  const bool do_fwd = phases & kPhaseForward, do_rev = phases & kPhaseReverse;
  char* ws = static_cast<char*>(b.workspace);
  const int nt = P.adaptive ? P.nseg : p.n_steps, s = p.scheme.stages;
  // ---- control blob: ts (adaptive: interval ends) | fwd_rec | fwd_sol | prog | status | obs
  std::vector<char> blob(P.blob_bytes, 0);
  std::memcpy(blob.data() + P.o_ts, P.adaptive ? P.pts.data() : p.times, sizeof(double) * (nt + 1));
  std::memcpy(blob.data() + P.o_fr, P.fwd_rec.data(), sizeof(int) * nt);
  std::memcpy(blob.data() + P.o_fs, P.fwd_sol.data(), sizeof(int) * nt);
  if (!P.prog.empty()) std::memcpy(blob.data() + P.o_pg, P.prog.data(), sizeof(int4) * P.prog.size());
  if (!P.obs_k.empty()) std::memcpy(blob.data() + P.o_obs, P.obs_k.data(), sizeof(int) * P.obs_k.size());
  const size_t o_ts = P.o_ts, o_fr = P.o_fr, o_fs = P.o_fs, o_pg = P.o_pg, o_stat = P.o_stat;
  CU(cudaMemcpyAsync(ws + P.off_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice, st));

  RkParams<T> rp{};
  rp.d = P.d;
  rp.sm = P.sm;
  PackParams<T> pp{};
  pp.d = P.d;
  pp.theta = static_cast<const T*>(b.theta);
  pp.packed = reinterpret_cast<T*>(ws + P.off_pk);
  rp.packed = pp.packed;
  for (int l = 0; l < P.d.L; ++l) rp.W.bias[l] = pp.theta + P.d.boff[l];
  rp.s = s;
  rp.fsal = p.scheme.fsal;
  std::memcpy(rp.a, p.scheme.a, sizeof(rp.a));
  std::memcpy(rp.b, p.scheme.b, sizeof(rp.b));
  std::memcpy(rp.c, p.scheme.c, sizeof(rp.c));
  rp.skip_vjp = P.skip_vjp;
  rp.field_kind = p.field.kind;
  rp.diag = static_cast<const T*>(b.aux);
  rp.out_scale = T(p.field.out_scale);
  rp.B = (int)p.batch;
  rp.R = P.R;
  rp.Rt = P.Rt;
  rp.n_steps = nt;
  rp.ts = reinterpret_cast<const double*>(ws + P.off_blob + o_ts);
  rp.loss_kind = p.loss;
  rp.targets = static_cast<const T*>(b.targets);
  rp.seed = static_cast<const T*>(b.seed);
  if (!P.obs_k.empty()) {
    rp.obs_k = reinterpret_cast<const int*>(ws + P.off_blob + P.o_obs);
    rp.n_obs = p.n_obs;
    rp.obs_values = static_cast<const T*>(b.obs_values);
    rp.scale_lo = static_cast<const T*>(b.scale_lo);
    rp.scale_hi = static_cast<const T*>(b.scale_hi);
    rp.preds = static_cast<T*>(b.predictions);
  }
  rp.batch_global = double(p.batch_global > 0 ? p.batch_global : p.batch);
  rp.inv_batch_global = 1.0 / rp.batch_global;
  rp.u0 = static_cast<const T*>(b.u0);
  rp.u_final = static_cast<T*>(b.u_final);
  rp.du0 = static_cast<T*>(b.du0);
  rp.rec = reinterpret_cast<T*>(ws + P.off_rec);
  rp.sol = reinterpret_cast<T*>(ws + P.off_sol);
  rp.fwd_rec = reinterpret_cast<const int*>(ws + P.off_blob + o_fr);
  rp.fwd_sol = reinterpret_cast<const int*>(ws + P.off_blob + o_fs);
  rp.prog = reinterpret_cast<const int4*>(ws + P.off_blob + o_pg);
  rp.prog_len = (int)P.prog.size();
  rp.scratch = reinterpret_cast<T*>(ws + P.off_scr);
  rp.scratch_stride = P.scratch_stride;
  rp.mu = reinterpret_cast<T*>(ws + P.off_mu);
  rp.n_params = p.field.n_params;
  rp.loss_part = reinterpret_cast<double*>(ws + P.off_lp);
  int* status = reinterpret_cast<int*>(ws + P.off_blob + o_stat);
  rp.status = status;
  rp.prof = (p.flags & OB_FLAG_PHASE_TIMING) ? 1 : 0;
  rp.phase = rp.prof ? phase_buffer() : nullptr;
  rp.theta = p.scheme.theta;
  rp.newton_tol = p.solver.newton_tol;
  rp.gmres_tol = p.solver.gmres_tol;
  rp.newton_maxit = p.solver.newton_maxit;
  rp.gmres_maxit = p.solver.gmres_maxit;
  rp.gmres_restart = p.solver.gmres_restart;
  rp.krylov = reinterpret_cast<T*>(ws + P.off_kry);
  rp.krylov_stride = P.krylov_stride;
  int* stats = reinterpret_cast<int*>(ws + P.off_stats);
  rp.sample_stats = stats;
  rp.eps = static_cast<const T*>(b.aux);
  rp.cnf_pre = reinterpret_cast<T*>(ws + P.off_cnf);
  rp.cnf_pre_stride = P.cnf_stride;
  rp.state_glob = reinterpret_cast<T*>(ws + P.off_state);
  rp.state_stride = 5LL * P.Rt * P.d.ldn;
  rp.head = static_cast<const T*>(b.head);
  rp.labels = b.labels;
  rp.n_classes = b.n_classes;
  rp.head_part = reinterpret_cast<T*>(ws + P.off_head);
  rp.tiles_total = P.tiles;
  if (P.adaptive) {
    rp.ad_policy = p.policy == OB_POLICY_STORE_ALL ? 0 : 1;
    rp.ad_abstol = p.abstol;
    rp.ad_reltol = p.reltol;
    rp.ad_hinit = p.h_init;
    rp.ad_hmin = p.h_min;
    rp.ad_hmax = p.h_max;
    rp.ad_safety = p.safety;
    rp.ad_alpha = 0.7 / p.scheme.order;   // PI exponents (integrators.py:300-302)
    rp.ad_beta = 0.4 / p.scheme.order;
    rp.ad_max_steps = p.max_steps;
    rp.ad_cap = P.cap;
    for (int i = 0; i < s; ++i) rp.ad_d[i] = p.scheme.b[i] - p.scheme.b_emb[i];
    rp.ad_pts = reinterpret_cast<const double*>(ws + P.off_blob + o_ts);
    rp.ad_nseg = P.nseg;
    rp.ad_seg_obs = rp.obs_k;
    rp.ad_obs0 = P.obs0;
    rp.ad_grid = reinterpret_cast<double*>(ws + P.off_grid);
    rp.ad_nacc = reinterpret_cast<int*>(ws + P.off_nacc);
    rp.obs_step = reinterpret_cast<int*>(ws + P.off_ostep);
    if (do_fwd)
      CU(cudaMemsetAsync(rp.obs_step, 0xff, sizeof(int) * (size_t)p.batch * std::max(p.n_obs, 1), st));
  }
  if (do_fwd) CU(cudaMemsetAsync(stats, 0, sizeof(int) * (size_t)p.batch * OB_NSTATS, st));

  // per-phase CUDA events on the launch stream (bench roofline timing)
  cudaEvent_t* ev = nullptr;
  CU(phase_events(ev));
  if (do_rev) CU(cudaMemsetAsync(rp.mu, 0, P.esz * (size_t)P.tiles * P.d.n_mu, st));
  CU(cudaEventRecord(ev[0], st));
  if (!do_fwd) {
    // packed weights of the forward call are still in the workspace
  } else if (P.tc_conv) {
    if constexpr (sizeof(T) == 4)
      CU(launch_pack_tc_conv(P.d, reinterpret_cast<const float*>(pp.theta), pp.packed, st));
  } else if (P.d.conv) {
    if constexpr (sizeof(T) == 4) CU(launch_pack_conv<T>(pp, st));
  } else if (P.tc) {
    if constexpr (sizeof(T) == 4)
      CU(launch_pack_tc(P.d, reinterpret_cast<const float*>(pp.theta),
                        reinterpret_cast<float*>(pp.packed), st));
  } else if (P.tc_cnf) {
    if constexpr (sizeof(T) == 4)
      CU(launch_pack_tc_cnf(P.d, reinterpret_cast<const float*>(pp.theta), pp.packed, st));
  } else {
    CU(launch_pack<T>(pp, st));
  }
  CU(cudaEventRecord(ev[1], st));
  auto sweep = [&](bool fwd) -> cudaError_t {
    if (P.adaptive) return launch_adaptive<T>(rp, P.LR, P.tiles, P.smem_bytes, st, fwd);
    if (P.theta_cluster) {
      if constexpr (sizeof(T) == 8) {
        RkParams<double> q = reinterpret_cast<const RkParams<double>&>(rp);
        q.tile_aux = (unsigned)P.cluster_rows;
        return launch_theta_cluster(q, P.tiles, P.smem_bytes, st, fwd);
      }
      return cudaErrorNotSupported;
    }
    if (P.rk_cluster) {
      if constexpr (sizeof(T) == 8)
        return (P.rk_cluster == 2 ? launch_rk_cluster2 : launch_rk_cluster8)(
            reinterpret_cast<const RkParams<double>&>(rp), P.tiles, P.smem_bytes, st, fwd);
      return cudaErrorNotSupported;
    }
    if (P.theta) return launch_theta<T>(rp, P.LR, P.tiles, P.smem_bytes, st, fwd);
    if (P.tc) {
      if constexpr (sizeof(T) == 4)
        return launch_rk_tc(reinterpret_cast<const RkParams<float>&>(rp), P.tiles, P.smem_bytes, st,
                            fwd);
      return cudaErrorNotSupported;
    }
    if (P.tc_cnf) {
      if constexpr (sizeof(T) == 4)
        return launch_cnf_tc(reinterpret_cast<const RkParams<float>&>(rp), P.tiles, P.cnf_cluster,
                             P.smem_bytes, st, fwd);
      return cudaErrorNotSupported;
    }
    if (P.tc_conv) {
      if constexpr (sizeof(T) == 4)
        return launch_conv_tc(reinterpret_cast<const RkParams<float>&>(rp), P.tiles, P.smem_bytes, st, fwd);
      return cudaErrorNotSupported;
    }
    if (P.d.cnf || P.d.conv) {
      if constexpr (sizeof(T) == 4) {
        if (P.d.conv) return launch_conv<T>(rp, P.tiles, P.smem_bytes, st, fwd);
        return launch_cnf<T>(rp, P.LR, P.tiles, P.smem_bytes, st, fwd);
      }
      return cudaErrorNotSupported;
    }
    return launch_rk<T>(rp, P.LR, P.tiles, P.smem_bytes, st, fwd);
  };
  if (cadj_dphi) {   // continuous-adjoint baseline: one augmented reverse-time sweep
    CU(launch_cadj<T>(rp, P.LR, P.tiles, P.smem_bytes, p.tF, static_cast<const T*>(cadj_dphi), st));
    CU(cudaEventRecord(ev[2], st));
  } else {
    if (do_fwd) CU(sweep(true));
    CU(cudaEventRecord(ev[2], st));
    if (do_rev) CU(sweep(false));
  }
  CU(cudaEventRecord(ev[3], st));
  // dtheta (reverse) and the loss (forward: per-tile partials of loss_partial)
  CU(launch_reduce<T>(P.d, rp.mu, P.tiles, do_rev ? p.field.n_params : 0, static_cast<T*>(b.dtheta),
                      rp.loss_part, rp.inv_batch_global, do_fwd ? b.loss : nullptr, st,
                      static_cast<const T*>(b.dtheta_seed)));
  if (do_fwd && p.loss == OB_LOSS_CE_HEAD && b.dhead) {
    if constexpr (sizeof(T) == 4)
      CU(launch_reduce_plain<T>(rp.head_part, P.tiles, 10 * 64 + 10, 10 * 64 + 10,
                                static_cast<T*>(b.dhead), st));
  }
  CU(cudaEventRecord(ev[4], st));
  const auto t_issued = std::chrono::steady_clock::now();
  int hs[2] = {0, 0};
  CU(cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st));
  std::vector<int> hstats;
  if (P.theta || P.adaptive) {
    hstats.resize((size_t)p.batch * OB_NSTATS);
    CU(cudaMemcpyAsync(hstats.data(), stats, sizeof(int) * hstats.size(), cudaMemcpyDeviceToHost, st));
  }
  if (b.sample_stats)
    CU(cudaMemcpyAsync(b.sample_stats, stats, sizeof(int) * (size_t)p.batch * OB_NSTATS,
                       cudaMemcpyDeviceToDevice, st));
  CU(cudaStreamSynchronize(st));
  if (getenv("OB_HOST_TIMING")) {
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "ob_grad host: issue %.1f us, sync wait %.1f us\n",
            std::chrono::duration<double, std::micro>(t_issued - g_t_entry).count(),
            std::chrono::duration<double, std::micro>(now - t_issued).count());
  }
  if (P.theta || P.adaptive) {  // reference-semantics counters of the critical-path trajectory
    long long mf = 0, mb = 0, ma = 0, mr = 0, mc = 0;
    for (long long i = 0; i < p.batch; ++i) {
      const int* r = &hstats[i * OB_NSTATS];
      mf = std::max<long long>(mf, r[OB_STAT_NFE_F]);
      mb = std::max<long long>(mb, r[OB_STAT_NFE_B]);
      ma = std::max<long long>(ma, r[OB_STAT_ACCEPTED]);
      mr = std::max<long long>(mr, r[OB_STAT_REJECTED]);
      mc = std::max<long long>(mc, r[OB_STAT_RECOMPUTED]);
    }
    P.cnt.nfe_forward = P.cnt.device_rhs_evals = mf;
    P.cnt.nfe_backward = P.cnt.device_vjp_evals = mb;
    if (P.adaptive) {   // per trajectory, max over samples (checkpointing.py:193-198, :272-284)
      P.cnt.steps_accepted = ma;
      P.cnt.steps_rejected = mr;
      P.cnt.steps_recomputed = P.cnt.recomputed_steps = mc;
      P.cnt.stored_states = ma > 0 ? ma - 1 : 0;
      P.cnt.stored_stage_vectors = p.policy == OB_POLICY_STORE_ALL ? (ma > 0 ? ma - 1 : 0) * s : 0;
      P.cnt.max_live_slots = P.cnt.stored_states;
      P.cnt.tile_rows = P.R;
      P.cnt.tiles = P.tiles;
      P.cnt.kernel_launches = 4;
    }
  }
  if (do_fwd && P.adaptive && hs[0] == 0 && (b.grid || b.n_accepted)) {
    // per-sample boundary times t_0, t_n + h_n (adjoint.py:171-173)
    std::vector<double> g((size_t)p.batch * P.cap * 2);
    std::vector<int> na((size_t)p.batch);
    CU(cudaMemcpy(g.data(), rp.ad_grid, sizeof(double) * g.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(na.data(), rp.ad_nacc, sizeof(int) * na.size(), cudaMemcpyDeviceToHost));
    if (b.n_accepted)
      CU(cudaMemcpyAsync(b.n_accepted, na.data(), sizeof(int) * na.size(), cudaMemcpyHostToDevice, st));
    if (b.grid) {
      const size_t w = (size_t)P.cap + 1;
      std::vector<double> bt((size_t)p.batch * w, std::nan(""));
      for (long long i = 0; i < p.batch; ++i) {
        bt[i * w] = p.t0;
        for (int n = 0; n < na[i]; ++n)
          bt[i * w + n + 1] = g[((size_t)i * P.cap + n) * 2] + g[((size_t)i * P.cap + n) * 2 + 1];
      }
      CU(cudaMemcpyAsync(b.grid, bt.data(), sizeof(double) * bt.size(), cudaMemcpyHostToDevice, st));
    }
    CU(cudaStreamSynchronize(st));
  }
  float ms[4] = {0, 0, 0, 0};
  for (int i = 0; i < 4; ++i) CU(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
  if (!do_fwd) ms[0] = ms[1] = 0.f;
  if (!do_rev) ms[2] = 0.f;
  P.cnt.ms_pack = ms[0];
  P.cnt.ms_forward = ms[1];
  P.cnt.ms_reverse = ms[2];
  P.cnt.ms_reduce = ms[3];
  if (hs[0] != 0) {
    char msg[256];
    if (hs[0] == OB_ERR_INTEGRATION) {
      const double t = p.times[hs[1]], h = p.times[hs[1] + 1] - p.times[hs[1]];
      snprintf(msg, sizeof msg, "state overflowed at t=%.17g (h=%.17g)", t, h);
    } else if (hs[0] == OB_ERR_GRADIENT_EXPLOSION) {
      snprintf(msg, sizeof msg, "non-finite adjoint state in reverse sweep (step %d)", hs[1]);
    } else if (hs[0] == OB_ERR_CONVERGENCE) {
      const double t = p.times[hs[1]];
      snprintf(msg, sizeof msg, "implicit step at t=%.17g failed: Newton/GMRES did not converge", t);
    } else if (hs[0] == OB_ERR_VALUE) {
      snprintf(msg, sizeof msg, "vector contains non-finite entries");
    } else if (hs[0] == OB_ERR_STIFFNESS) {   // integrators.py:309-311, :322-323, :342-343
      if (hs[1] & 1)
        snprintf(msg, sizeof msg, "adaptive integration exceeded %lld steps (sample %d)",
                 (long long)p.max_steps, hs[1] >> 1);
      else
        snprintf(msg, sizeof msg, "step size underflow (sample %d): stiffness suspected", hs[1] >> 1);
    } else if (hs[0] == OB_ERR_UNSUPPORTED && P.adaptive) {
      snprintf(msg, sizeof msg, "sample %d needs more than max_accepted = %d accepted steps", hs[1],
               P.cap);
    } else {
      snprintf(msg, sizeof msg, "device status %d (%d)", hs[0], hs[1]);
    }
    return fail(hs[0], msg);
  }
  return OB_OK;
}

}  // namespace

// The plan of the last gradient problem, reused while the problem (struct and the host
// arrays it points to) and the device are unchanged: ob_grad_workspace_size + ob_grad
// on a training / benchmark loop then plan once.
namespace {
std::vector<char> plan_key(const ob_problem& p) {
  ob_problem q = p;
  q.times = nullptr;
  q.obs_steps = nullptr;
  q.obs_times = nullptr;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) cudaGetLastError();
  std::vector<char> k(sizeof(q) + sizeof(dev));
  std::memcpy(k.data(), &q, sizeof(q));
  std::memcpy(k.data() + sizeof(q), &dev, sizeof(dev));
  auto app = [&](const void* src, size_t n) {
    if (!src || !n) return;
    const size_t o = k.size();
    k.resize(o + n);
    std::memcpy(k.data() + o, src, n);
  };
  if (!p.adaptive && p.n_steps >= 0) app(p.times, sizeof(double) * (size_t)(p.n_steps + 1));
  if (p.n_obs > 0) {
    app(p.obs_steps, sizeof(int32_t) * (size_t)p.n_obs);
    app(p.obs_times, sizeof(double) * (size_t)p.n_obs);
  }
  return k;
}

int cached_plan(const ob_problem& p, Plan& P) {
  static thread_local std::vector<char> key;
  static thread_local Plan plan;
  static thread_local bool valid = false;
  std::vector<char> k = plan_key(p);
  if (valid && k == key) {
    P = plan;
    return OB_OK;
  }
  valid = false;
  int st = plan_problem(p, P, true);
  if (st) return st;
  key = std::move(k);
  plan = P;
  valid = true;
  return OB_OK;
}
}  // namespace

extern "C" int ob_grad_workspace_size(const ob_problem* p, size_t* bytes) {
  if (!p || !bytes) return fail(OB_ERR_VALUE, "null argument");
  Plan P;
  int st = cached_plan(*p, P);
  if (st) return st;
  *bytes = P.total;
  return OB_OK;
}

static int grad_phases(const ob_problem* p, const ob_buffers* b, ob_counters* out, void* stream,
                       int phases) {
  g_t_entry = std::chrono::steady_clock::now();
  if (!p || !b) return fail(OB_ERR_VALUE, "null argument");
  Plan P;
  int st = cached_plan(*p, P);
  if (st) return st;
  if (!b->workspace || b->workspace_bytes < P.total)
    return fail(OB_ERR_VALUE, "workspace too small (need " + std::to_string(P.total) + " bytes)");
  const bool fwd = phases & kPhaseForward, rev = phases & kPhaseReverse;
  if (!b->theta || !b->u0 || !b->u_final || (rev && (!b->du0 || !b->dtheta)) || (fwd && !b->loss))
    return fail(OB_ERR_VALUE, "null device buffer");
  if (p->loss == OB_LOSS_SEED && rev && !b->seed)
    return fail(OB_ERR_VALUE, "seeded sweep needs the terminal seed lambda_N");
  if (p->loss == OB_LOSS_SEED && p->n_obs > 0 && (!b->predictions || (rev && !b->obs_values)))
    return fail(OB_ERR_VALUE, "seeded sweep with observations needs a predictions buffer and "
                              "one injection per observation");
  if (p->field.kind == OB_FIELD_STIFF && !b->aux) return fail(OB_ERR_VALUE, "stiff field needs diag");
  if (p->field.kind == OB_FIELD_CNF && !b->aux) return fail(OB_ERR_VALUE, "CNF field needs probes");
  if (p->loss == OB_LOSS_CE_HEAD && (!b->head || !b->labels || b->n_classes != 10))
    return fail(OB_ERR_VALUE, "cross-entropy head needs head parameters, labels and 10 classes");
  if (p->loss == OB_LOSS_MSE && !b->targets) return fail(OB_ERR_VALUE, "mse loss needs targets");
  if ((p->loss == OB_LOSS_OBS_MSE || p->loss == OB_LOSS_OBS_MAE) &&
      (!b->obs_values || !b->predictions || (!b->scale_lo) != (!b->scale_hi)))
    return fail(OB_ERR_VALUE, "observation loss needs observations, a predictions buffer and "
                              "both or neither scaling bounds");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = P.dtype == OB_F32 ? run_grad<float>(*p, *b, P, s, nullptr, phases)
                         : run_grad<double>(*p, *b, P, s, nullptr, phases);
  if (out) {
    *out = P.cnt;
    if (!rev) out->nfe_backward = out->device_vjp_evals = 0;
    if (!fwd) out->nfe_forward = out->device_rhs_evals = out->steps_accepted = 0;
    out->kernel_launches = phases == kPhaseBoth ? 4 : (fwd ? 3 : 2);
  }
  return st;
}

extern "C" int ob_grad(const ob_problem* p, const ob_buffers* b, ob_counters* out, void* stream) {
  return grad_phases(p, b, out, stream, kPhaseBoth);
}

extern "C" int ob_forward_pass(const ob_problem* p, const ob_buffers* b, ob_counters* out,
                               void* stream) {
  return grad_phases(p, b, out, stream, kPhaseForward);
}

extern "C" int ob_backward_sweep(const ob_problem* p, const ob_buffers* b, ob_counters* out,
                                 void* stream) {
  return grad_phases(p, b, out, stream, kPhaseReverse);
}

// Continuous-adjoint baseline (continuous_adjoint_solve, adjoint.py:314-331):
// lambda(t0) and the integral of P^T lambda from the terminal state u(tF) and
// seed dphi/du, integrating the augmented reverse-time system with the
// problem's explicit scheme over p->times (the tau grid, 0 .. tF - t0).
extern "C" int ob_continuous_adjoint(const ob_problem* p, const void* theta, const void* aux,
                                     const void* u_final, const void* dphi_du, void* lam0,
                                     void* mu0, void* workspace, size_t workspace_bytes,
                                     ob_counters* out, void* stream) {
  if (!p || !theta || !u_final || !dphi_du || !lam0 || !mu0) return fail(OB_ERR_VALUE, "null argument");
  if (p->scheme.kind != OB_SCHEME_RK)
    return fail(OB_ERR_VALUE, "the continuous-adjoint baseline supports explicit schemes");
  if (p->field.kind != OB_FIELD_MLP && p->field.kind != OB_FIELD_STIFF)
    return fail(OB_ERR_UNSUPPORTED, "the continuous-adjoint baseline is built for MLP / stiff fields");
  if (p->field.kind == OB_FIELD_STIFF && !aux) return fail(OB_ERR_VALUE, "stiff field needs diag");
  ob_problem q = *p;
  q.policy = OB_POLICY_STORE_SOLUTIONS;
  q.loss = OB_LOSS_HALF_SQNORM;
  q.n_obs = 0;
  q.adaptive = 0;
  q.flags |= OB_FLAG_NO_TENSOR_CORES;   // the SIMT tile runs the augmented sweep
  Plan P;
  int st = plan_problem(q, P);
  if (st) return st;
  if (!workspace || workspace_bytes < P.total)
    return fail(OB_ERR_VALUE, "workspace too small (need " + std::to_string(P.total) + " bytes)");
  ob_buffers b{};
  b.theta = theta;
  b.aux = aux;
  b.u0 = u_final;
  b.u_final = const_cast<void*>(u_final);
  b.du0 = lam0;
  b.dtheta = mu0;
  b.loss = nullptr;
  b.workspace = workspace;
  b.workspace_bytes = workspace_bytes;
  const long long s = q.scheme.stages, n = q.n_steps;
  P.cnt = ob_counters{};
  P.cnt.nfe_forward = P.cnt.nfe_backward = s * n - (q.scheme.fsal ? n - 1 : 0);
  P.cnt.steps_accepted = n;
  P.cnt.tile_rows = P.R;
  P.cnt.tiles = P.tiles;
  P.cnt.kernel_launches = 3;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  st = P.dtype == OB_F32 ? run_grad<float>(q, b, P, cs, dphi_du) : run_grad<double>(q, b, P, cs, dphi_du);
  if (out) *out = P.cnt;
  return st;
}

// ============================================================ field ops
namespace {

enum { kEval = 0, kJvp = 1, kVjp = 2, kVjpU = 3 };

template <typename T>
int run_field_op(const ob_field_desc& f, int64_t batch, const void* theta, const void* aux,
                 const void* u, double t, const void* w, void* out, void* ptv, int mode,
                 cudaStream_t st) {
  Plan P;
  P.dtype = f.dtype;
  P.esz = sizeof(T);
  P.need_jvp = (mode == kJvp);
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  choose_tiles(P, f, batch, sms);
  if (mode != kJvp && tc_cnf_eligible(f, 0)) plan_tc_cnf(P, f, batch, sms);
  if (mode != kJvp && tc_conv_eligible(f, 0)) plan_tc_conv(P, f, batch);
  if (P.smem_bytes > kSmemLimit) return fail(OB_ERR_UNSUPPORTED, "layer widths exceed shared memory");
  const size_t pk_bytes = align_up(P.esz * (size_t)P.d.n_packed, 256);
  const size_t mu_bytes = mode == kVjp ? P.esz * (size_t)P.tiles * P.d.n_mu : 0;
  long long cnf_stride = 0;
  for (int l = 0; P.d.cnf && !P.tc_cnf && l < P.d.L - 1; ++l) cnf_stride += 2LL * P.Rt * P.d.lda[l + 1];
  if (P.tc_cnf) cnf_stride = P.cnf_log_rec / 4;   // one VJP record per tile
  if (P.d.conv) cnf_stride = P.tc_conv ? 256LL * 64 : 18LL * 18 * 68;
  const size_t cnf_bytes = align_up(P.esz * (size_t)P.tiles * cnf_stride, 256);
  const size_t st_bytes = P.sm.u < 0 ? align_up(P.esz * (size_t)P.tiles * 5 * P.Rt * P.d.ldn, 256) : 0;
  char* ws = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void**>(&ws), pk_bytes + mu_bytes + cnf_bytes + st_bytes + 256,
                     st));
  RkParams<T> rp{};
  rp.d = P.d;
  rp.sm = P.sm;
  PackParams<T> pp{};
  pp.d = P.d;
  pp.theta = static_cast<const T*>(theta);
  pp.packed = reinterpret_cast<T*>(ws);
  rp.packed = pp.packed;
  for (int l = 0; l < P.d.L; ++l) rp.W.bias[l] = pp.theta + P.d.boff[l];
  rp.field_kind = f.kind;
  rp.diag = static_cast<const T*>(aux);
  rp.out_scale = T(f.out_scale);
  rp.B = (int)batch;
  rp.R = P.R;
  rp.Rt = P.Rt;
  rp.n_params = f.n_params;
  rp.mu = mode == kVjp ? reinterpret_cast<T*>(ws + pk_bytes) : nullptr;
  rp.eps = static_cast<const T*>(aux);
  rp.cnf_pre = reinterpret_cast<T*>(ws + pk_bytes + align_up(mu_bytes, 256));
  rp.cnf_pre_stride = cnf_stride;
  rp.state_glob = reinterpret_cast<T*>(ws + pk_bytes + align_up(mu_bytes, 256) + cnf_bytes);
  rp.state_stride = 5LL * P.Rt * P.d.ldn;
  int rc = OB_OK;
  cudaError_t e = cudaSuccess;
  if (mu_bytes) e = cudaMemsetAsync(rp.mu, 0, mu_bytes, st);
  if (e == cudaSuccess) {
    if (P.tc_conv) {
      if constexpr (sizeof(T) == 4) e = launch_pack_tc_conv(P.d, reinterpret_cast<const float*>(theta), ws, st);
    } else if (P.d.conv) {
      if constexpr (sizeof(T) == 4) e = launch_pack_conv<T>(pp, st);
    } else if (P.tc_cnf) {
      if constexpr (sizeof(T) == 4) e = launch_pack_tc_cnf(P.d, reinterpret_cast<const float*>(theta), ws, st);
    } else {
      e = launch_pack<T>(pp, st);
    }
  }
  if (e == cudaSuccess) {
    if (P.tc_conv) {
      if constexpr (sizeof(T) == 4)
        e = launch_conv_tc_field(reinterpret_cast<const RkParams<float>&>(rp), P.tiles, P.smem_bytes, mode, t,
                                 reinterpret_cast<const float*>(u), reinterpret_cast<const float*>(w),
                                 reinterpret_cast<float*>(out), st);
    } else if (P.d.conv) {
      if constexpr (sizeof(T) == 4)
        e = launch_conv_field<T>(rp, P.tiles, P.smem_bytes, mode, t, static_cast<const T*>(u),
                                 static_cast<const T*>(w), static_cast<T*>(out), st);
    } else if (P.tc_cnf) {
      if constexpr (sizeof(T) == 4)
        e = launch_cnf_tc_field(reinterpret_cast<const RkParams<float>&>(rp), P.tiles, P.cnf_cluster,
                                P.smem_bytes, mode,
                                t, reinterpret_cast<const float*>(u), reinterpret_cast<const float*>(w),
                                reinterpret_cast<float*>(out), st);
    } else if (P.d.cnf) {
      if constexpr (sizeof(T) == 4)
        e = launch_cnf_field<T>(rp, P.LR, P.tiles, P.smem_bytes, mode, t, static_cast<const T*>(u),
                                static_cast<const T*>(w), static_cast<T*>(out), st);
    } else {
      e = launch_field_op<T>(rp, P.LR, P.tiles, P.smem_bytes, mode, t, static_cast<const T*>(u),
                             static_cast<const T*>(w), static_cast<T*>(out), st);
    }
  }
  if (e == cudaSuccess && mode == kVjp)
    e = launch_reduce<T>(P.d, rp.mu, P.tiles, f.n_params, static_cast<T*>(ptv), nullptr, 0.0,
                         nullptr, st, static_cast<const T*>(nullptr));
  cudaFreeAsync(ws, st);
  if (e != cudaSuccess) rc = fail(OB_ERR_CUDA, cudaGetErrorString(e));
  return rc;
}

int field_op(const ob_field_desc* f, int64_t batch, const void* theta, const void* aux,
             const void* u, double t, const void* w, void* out, void* ptv, int mode, void* stream) {
  if (!f || !theta || !u || !out) return fail(OB_ERR_VALUE, "null argument");
  int st = check_field(*f);
  if (st) return st;
  if (batch < 1) return fail(OB_ERR_VALUE, "batch must be >= 1");
  if ((mode != kEval) && !w) return fail(OB_ERR_VALUE, "null tangent/cotangent");
  if (mode == kVjp && !ptv) return fail(OB_ERR_VALUE, "null ptv");
  if ((f->kind == OB_FIELD_STIFF || f->kind == OB_FIELD_CNF) && !aux)
    return fail(OB_ERR_VALUE, "field needs its auxiliary array");
  if ((f->kind == OB_FIELD_CNF || f->kind == OB_FIELD_CONV) && mode == kJvp)
    return fail(OB_ERR_UNSUPPORTED, "CNF field has no JVP (explicit schemes only)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return f->dtype == OB_F32 ? run_field_op<float>(*f, batch, theta, aux, u, t, w, out, ptv, mode, s)
                            : run_field_op<double>(*f, batch, theta, aux, u, t, w, out, ptv, mode, s);
}

}  // namespace

extern "C" int ob_field_eval(const ob_field_desc* f, int64_t batch, const void* theta,
                             const void* aux, const void* u, double t, void* out, void* stream) {
  return field_op(f, batch, theta, aux, u, t, nullptr, out, nullptr, kEval, stream);
}
extern "C" int ob_field_jvp(const ob_field_desc* f, int64_t batch, const void* theta,
                            const void* aux, const void* u, double t, const void* w, void* out,
                            void* stream) {
  return field_op(f, batch, theta, aux, u, t, w, out, nullptr, kJvp, stream);
}
extern "C" int ob_field_vjp(const ob_field_desc* f, int64_t batch, const void* theta,
                            const void* aux, const void* u, double t, const void* v, void* jtv,
                            void* ptv, void* stream) {
  return field_op(f, batch, theta, aux, u, t, v, jtv, ptv, kVjp, stream);
}
extern "C" int ob_field_vjp_u(const ob_field_desc* f, int64_t batch, const void* theta,
                              const void* aux, const void* u, double t, const void* v, void* jtv,
                              void* stream) {
  return field_op(f, batch, theta, aux, u, t, v, jtv, nullptr, kVjpU, stream);
}
