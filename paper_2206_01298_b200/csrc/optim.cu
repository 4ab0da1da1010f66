// optim.cu -- device side of the training loop's optimizer:
// the decoupled-weight-decay Adam update adamw_step (training.py:175-190) and
// the gradient 2-norm the loop records (training.py:276-277).
//
// adamw_step follows numpy's evaluation order exactly with round-to-nearest
// mul/add/div/sqrt and no FMA contraction, so fp64 results are bit-identical
// to the reference; the bias corrections (1 - beta^t) are formed on the host
// with the same pow the reference uses.  The norm is a fixed-order two-pass
// reduction (per-block partial sums in a fixed tree, then blocks in order).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <map>
#include <string>

#include "../../include/odeblock.h"

namespace {

constexpr int kBlock = 256;
constexpr int kMaxBlocks = 1024;

template <typename T> struct Op;
template <> struct Op<double> {
  static __device__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ double sqrt_(double a) { return __dsqrt_rn(a); }
};
template <> struct Op<float> {
  static __device__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ float sqrt_(float a) { return __fsqrt_rn(a); }
};

struct AdamScalars {
  double decay;      // 1 - lr * weight_decay
  double b1, omb1;   // beta1, 1 - beta1
  double b2, omb2;   // beta2, 1 - beta2
  double bc1, bc2;   // 1 - beta1^t, 1 - beta2^t
  double lr, eps;
};

// partial sums of g^2 (fp64) and a non-finite flag per block
template <typename T>
__global__ void sumsq_kernel(const T* g, long long n, double* part, int* bad) {
  __shared__ double red[kBlock];
  double acc = 0.0;
  int nf = 0;
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock) {
    const double x = double(g[i]);
    if (!isfinite(x)) nf = 1;
    acc = __dadd_rn(acc, __dmul_rn(x, x));
  }
  red[threadIdx.x] = acc;
  if (nf) atomicOr(bad, 1);
  __syncthreads();
  for (int s = kBlock / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void finish_norm_kernel(const double* part, int nb, double* out) {
  double acc = 0.0;
  for (int b = 0; b < nb; ++b) acc = __dadd_rn(acc, part[b]);
  *out = __dsqrt_rn(acc);
}

// training-loop gate (training.py:276-283): record ||g|| into the caller's history slot and
// raise the sticky status (1: gradient explosion) when g is non-finite or ||g|| exceeds the
// threshold; the update that follows is skipped once the status is set
__global__ void gate_kernel(const double* norm, int* bad, double threshold, double* norm_out,
                            int* status) {
  const double nv = *norm;
  if (norm_out) *norm_out = nv;
  if (*status == 0 && (*bad || !(nv <= threshold))) *status = 1;
  if (*status != 0) *bad = 1;
}

// theta = theta * decay; m = b1 m + (1-b1) g; v = b2 v + ((1-b2) g) g;
// theta = theta - (lr * (m / bc1)) / (sqrt(v / bc2) + eps)   (training.py:184-189)
template <typename T>
__global__ void adamw_kernel(T* theta, const T* g, T* m, T* v, long long n, AdamScalars s,
                             const int* bad) {
  if (*bad) return;   // GradientExplosionError: nothing is updated (training.py:178-179)
  using O = Op<T>;
  const T decay = T(s.decay), b1 = T(s.b1), omb1 = T(s.omb1), b2 = T(s.b2), omb2 = T(s.omb2);
  const T bc1 = T(s.bc1), bc2 = T(s.bc2), lr = T(s.lr), eps = T(s.eps);
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock) {
    const T gi = g[i];
    T th = O::mul(theta[i], decay);
    const T mi = O::add(O::mul(b1, m[i]), O::mul(omb1, gi));
    const T vi = O::add(O::mul(b2, v[i]), O::mul(O::mul(omb2, gi), gi));
    const T mh = O::div(mi, bc1);
    const T vh = O::div(vi, bc2);
    th = O::sub(th, O::div(O::mul(lr, mh), O::add(O::sqrt_(vh), eps)));
    theta[i] = th;
    m[i] = mi;
    v[i] = vi;
  }
}

thread_local std::string g_err;

int set_err(int code, const char* msg) {
  g_err = msg;
  return code;
}

struct Scratch {
  double* part = nullptr;
  int* bad = nullptr;
  double* norm = nullptr;
  ~Scratch() {}
};

// one scratch set per device (created on first use on the device current at the call)
int scratch(Scratch& s, cudaStream_t st) {
  static thread_local std::map<int, Scratch> per_device;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return OB_ERR_CUDA;
  Scratch& cached = per_device[dev];
  if (!cached.part) {
    if (cudaMalloc(&cached.part, sizeof(double) * kMaxBlocks) != cudaSuccess ||
        cudaMalloc(&cached.bad, sizeof(int)) != cudaSuccess ||
        cudaMalloc(&cached.norm, sizeof(double)) != cudaSuccess)
      return OB_ERR_CUDA;
  }
  s = cached;
  (void)st;
  return OB_OK;
}

template <typename T>
int run_norm(const T* g, long long n, Scratch& sc, cudaStream_t st, int& nb) {
  nb = (int)std::min<long long>(kMaxBlocks, std::max<long long>(1, (n + kBlock - 1) / kBlock));
  if (cudaMemsetAsync(sc.bad, 0, sizeof(int), st) != cudaSuccess) return OB_ERR_CUDA;
  sumsq_kernel<T><<<nb, kBlock, 0, st>>>(g, n, sc.part, sc.bad);
  finish_norm_kernel<<<1, 1, 0, st>>>(sc.part, nb, sc.norm);
  return cudaGetLastError() == cudaSuccess ? OB_OK : OB_ERR_CUDA;
}

}  // namespace

extern "C" const char* ob_optim_last_error(void) { return g_err.c_str(); }

// ||g||_2 in fp64 (fixed reduction order); non-finite entries -> *norm = inf|nan
extern "C" int ob_grad_norm(int32_t dtype, const void* g, int64_t n, double* norm_host, void* stream) {
  if (!g || !norm_host || n < 0) return set_err(OB_ERR_VALUE, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Scratch sc;
  if (scratch(sc, st)) return set_err(OB_ERR_CUDA, "cudaMalloc failed");
  int nb = 0;
  const int rc = dtype == OB_F64 ? run_norm(static_cast<const double*>(g), n, sc, st, nb)
                                 : run_norm(static_cast<const float*>(g), n, sc, st, nb);
  if (rc) return set_err(rc, cudaGetErrorString(cudaGetLastError()));
  if (cudaMemcpyAsync(norm_host, sc.norm, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return set_err(OB_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  return OB_OK;
}

// One training-loop step without a host round trip: ||g|| -> norm_out (device), the
// explosion gate -> *status (device, sticky), then AdamW unless the gate tripped.
extern "C" int ob_adamw_step_gated(int32_t dtype, void* theta, const void* g, void* m, void* v,
                                   int64_t n, int64_t step, double lr, double beta1, double beta2,
                                   double eps, double weight_decay, double threshold,
                                   double* norm_out, int32_t* status, void* stream) {
  if (!theta || !g || !m || !v || !status || n < 0) return set_err(OB_ERR_VALUE, "null argument");
  if (step < 1) return set_err(OB_ERR_VALUE, "step counts from 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Scratch sc;
  if (scratch(sc, st)) return set_err(OB_ERR_CUDA, "cudaMalloc failed");
  AdamScalars s;
  s.decay = 1.0 - lr * weight_decay;
  s.b1 = beta1;
  s.omb1 = 1.0 - beta1;
  s.b2 = beta2;
  s.omb2 = 1.0 - beta2;
  s.bc1 = 1.0 - std::pow(beta1, (double)step);
  s.bc2 = 1.0 - std::pow(beta2, (double)step);
  s.lr = lr;
  s.eps = eps;
  int nb = 0;
  int rc = dtype == OB_F64 ? run_norm(static_cast<const double*>(g), n, sc, st, nb)
                           : run_norm(static_cast<const float*>(g), n, sc, st, nb);
  if (rc) return set_err(rc, "norm kernel failed");
  gate_kernel<<<1, 1, 0, st>>>(sc.norm, sc.bad, threshold, norm_out, status);
  const int blocks = (int)std::min<long long>(148 * 8, std::max<long long>(1, (n + kBlock - 1) / kBlock));
  if (dtype == OB_F64)
    adamw_kernel<double><<<blocks, kBlock, 0, st>>>(static_cast<double*>(theta), static_cast<const double*>(g),
                                                    static_cast<double*>(m), static_cast<double*>(v), n, s, sc.bad);
  else
    adamw_kernel<float><<<blocks, kBlock, 0, st>>>(static_cast<float*>(theta), static_cast<const float*>(g),
                                                   static_cast<float*>(m), static_cast<float*>(v), n, s, sc.bad);
  return cudaGetLastError() == cudaSuccess ? OB_OK : set_err(OB_ERR_CUDA, "launch failed");
}

// One AdamW step on device vectors of n parameters; step = the new step count t.
extern "C" int ob_adamw_step(int32_t dtype, void* theta, const void* g, void* m, void* v, int64_t n,
                             int64_t step, double lr, double beta1, double beta2, double eps,
                             double weight_decay, void* stream) {
  if (!theta || !g || !m || !v || n < 0) return set_err(OB_ERR_VALUE, "null argument");
  if (step < 1) return set_err(OB_ERR_VALUE, "step counts from 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Scratch sc;
  if (scratch(sc, st)) return set_err(OB_ERR_CUDA, "cudaMalloc failed");
  AdamScalars s;
  s.decay = 1.0 - lr * weight_decay;
  s.b1 = beta1;
  s.omb1 = 1.0 - beta1;
  s.b2 = beta2;
  s.omb2 = 1.0 - beta2;
  s.bc1 = 1.0 - std::pow(beta1, (double)step);
  s.bc2 = 1.0 - std::pow(beta2, (double)step);
  s.lr = lr;
  s.eps = eps;
  int nb = 0;
  int rc = dtype == OB_F64 ? run_norm(static_cast<const double*>(g), n, sc, st, nb)
                           : run_norm(static_cast<const float*>(g), n, sc, st, nb);
  if (rc) return set_err(rc, "norm kernel failed");
  const int blocks = (int)std::min<long long>(148 * 8, std::max<long long>(1, (n + kBlock - 1) / kBlock));
  if (dtype == OB_F64)
    adamw_kernel<double><<<blocks, kBlock, 0, st>>>(static_cast<double*>(theta), static_cast<const double*>(g),
                                                    static_cast<double*>(m), static_cast<double*>(v), n, s, sc.bad);
  else
    adamw_kernel<float><<<blocks, kBlock, 0, st>>>(static_cast<float*>(theta), static_cast<const float*>(g),
                                                   static_cast<float*>(m), static_cast<float*>(v), n, s, sc.bad);
  int bad = 0;
  if (cudaMemcpyAsync(&bad, sc.bad, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return set_err(OB_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  if (bad) return set_err(OB_ERR_GRADIENT_EXPLOSION, "non-finite gradient passed to the optimizer");
  return OB_OK;
}
