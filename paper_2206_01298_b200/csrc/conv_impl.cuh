// conv_impl.cuh -- the image-classifier ODE block (config C3) for the
// persistent RK kernels: f(u, t) = conv3x3(65 -> 64)(cat(u, t)) -> relu ->
// conv3x3(64 -> 64), padding 1, on a 16x16x64 NHWC state, one sample per CTA.
// The input (state + time channel) and the hidden activation sit in shared
// memory as zero-halo tiles; weights are packed once per call into forward
// ([Cout][tap][Cin]) and transposed ([tap][Cout][Cin]) layouts in global
// memory.  The VJP reuses the input tile for the incoming cotangent (the input
// is parked in a per-tile global buffer and restored for the conv1 weight
// gradient), keeping the footprint at two 88 KB tiles.
// No reference counterpart; fp64 restatement in oracle/fields_ext.py.
#pragma once

#include "conv.cuh"
#include "rk_impl.cuh"

namespace ob {

template <typename T>
struct ConvAdapter {
  const RkParams<T>& p;
  T* A;        // input / cotangent halo tile [18*18][68]
  T* Bh;       // hidden halo tile
  T* xsave;    // global parking slot for A
  const T *W1f, *W2f, *W1b, *W2b, *b1, *b2;
  T* stage;    // double-buffered tap weights in shared memory (nullptr: read through L1/L2)
  static constexpr bool kHasJvp = false;
  static constexpr bool kScaledVjp = false;  // vjp returns J^T w; the caller scales by h
  static constexpr int kCombineBatch = 4;    // stage loads in flight per ordered sum (registers)
  static constexpr bool kOwnsStep = false;   // the adapter runs whole RK steps itself
  OB_DEV void finish(T*) {}   // flush device-resident parameter cotangents (none here)
  OB_DEV void release() {}    // free per-CTA hardware resources (none here)

  OB_DEV ConvAdapter(const RkParams<T>& p_, const Weights<T>& W, MlpSmem<T>&, T* sm, int, int)
      : p(p_) {
    A = sm + p.sm.x0;
    Bh = sm + p.sm.hid[0];
    xsave = p.cnf_pre + blockIdx.x * p.cnf_pre_stride;
    W1f = p.packed + p.d.pwoff[0];
    W2f = p.packed + p.d.pwoff[1];
    W1b = p.packed + p.d.pwoff[2];
    W2b = p.packed + p.d.pwoff[3];
    b1 = W.bias[0];
    b2 = W.bias[1];
    stage = p.sm.tA >= 0 ? sm + p.sm.tA : nullptr;
  }
  template <class Epi>
  OB_DEV void fwd(const T* X, const T* Wf, int Kc, Warps ws, Epi epi) {
    if (stage) conv_staged<T, false>(X, Wf, 9 * kCP, kCP, 64, Kc, ws, stage, epi);
    else conv_fwd<T>(X, Wf, 64, Kc, ws, epi);
  }
  template <class Epi>
  OB_DEV void bwd(const T* D, const T* Wb, Warps ws, Epi epi) {
    if (stage) conv_staged<T, true>(D, Wb, kCP, 64LL * kCP, 64, 64, ws, stage, epi);
    else conv_bwd<T>(D, Wb, kCP, 64, ws, epi);
  }
  OB_DEV T* x0() { return A; }
  OB_DEV int nin() const { return p.d.N; }
  OB_DEV void set_scratch(T*, int) {}
  OB_DEV void jvp(const T*, T*) {}
  OB_DEV void put(int, int j, T v) { A[halo_idx(j >> 6, 1, 1) * kCP + (j & 63)] = v; }
  OB_DEV void put_time(double t) {
    for (int q = threadIdx.x; q < kPix; q += blockDim.x) A[halo_idx(q, 1, 1) * kCP + 64] = T(t);
  }

  OB_DEV void hidden() {   // Bh = relu(conv1(A) + b1)
    T* H = Bh;
    const T* bb = b1;
    fwd(A, W1f, kCP, Warps::all(), [&](int q, int co, T acc) {
      const T z = Num<T>::add(acc, bb[co]);
      H[halo_idx(q, 1, 1) * kCP + co] = z > T(0) ? z : T(0);
    });
    __syncthreads();
  }

  OB_DEV void eval(T* out) {
    hidden();
    const T* bb = b2;
    fwd(Bh, W2f, 64, Warps::all(),
        [&](int q, int co, T acc) { out[q * 64 + co] = Num<T>::add(acc, bb[co]); });
    __syncthreads();
  }

  OB_DEV void vjp(const T* w, T* jtv, T* mu, double h, int) {
    const T hs = T(h);
    hidden();
    // park the input, load the cotangent into the same tile
    for (int i = threadIdx.x; i < kHalo * kHalo * kCP; i += blockDim.x) xsave[i] = A[i];
    __syncthreads();
    for (int i = threadIdx.x; i < kPix * 68; i += blockDim.x) {
      const int q = i / 68, c = i % 68;
      A[halo_idx(q, 1, 1) * kCP + c] = c < 64 ? w[q * 64 + c] : T(0);
    }
    __syncthreads();
    if (mu) {   // dW2 += v (x) h1, db2 += v
      conv_wgrad<T>(A, Bh, 64, hs, mu + p.d.mwoff[1], mu + p.d.mboff[1], Warps::all());
      __syncthreads();
    }
    T* H = Bh;
    bwd(A, W2b, Warps::all(), [&](int q, int ci, T acc) {   // dz1 in place
      const int o = halo_idx(q, 1, 1) * kCP + ci;
      H[o] = H[o] > T(0) ? acc : T(0);
    });
    __syncthreads();
    for (int i = threadIdx.x; i < kHalo * kHalo * kCP; i += blockDim.x) A[i] = xsave[i];
    __syncthreads();
    const int nw = n_warps();
    const bool both = mu && jtv;
    const Warps wn = both ? Warps{0, nw / 2} : Warps::all();
    const Warps wa = both ? Warps{nw / 2, nw - nw / 2} : Warps::all();
    if (jtv)
      bwd(Bh, W1b, wn, [&](int q, int ci, T acc) { jtv[q * 64 + ci] = acc; });
    if (mu) conv_wgrad<T>(Bh, A, kCP, hs, mu + p.d.mwoff[0], mu + p.d.mboff[0], wa);
    __syncthreads();
  }
};

// packed conv weights: W1f/W2f [64][9*68] (tap-major, Cin padded), W1b/W2b
// [9*64][68] (transposed per tap), zero padded
template <typename T>
__global__ void pack_conv_kernel(const __grid_constant__ PackParams<T> p) {
  for (int l = 0; l < 2; ++l) {
    const int cin = p.d.conv_cin[l];
    const T* Wl = p.theta + p.d.woff[l];
    T* f = p.packed + p.d.pwoff[l];
    T* b = p.packed + p.d.pwoff[2 + l];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 64 * 9 * kCP; i += gridDim.x * blockDim.x) {
      const int co = i / (9 * kCP), s = (i / kCP) % 9, ci = i % kCP;
      const T v = ci < cin ? Wl[(co * 9 + s) * cin + ci] : T(0);
      f[i] = v;                                   // [co][s][ci]
      b[(s * 64 + co) * kCP + ci] = v;            // [s][co][ci]
    }
  }
}

template <typename T>
cudaError_t launch_conv(const RkParams<T>& p, int tiles, size_t smem, cudaStream_t st,
                        bool forward) {
  using F = ConvAdapter<T>;
  return forward ? launch_smem(rk_forward_kernel<T, F>, tiles, smem, st, p)
                 : launch_smem(rk_reverse_kernel<T, F>, tiles, smem, st, p);
}

template <typename T>
cudaError_t launch_conv_field(const RkParams<T>& p, int tiles, size_t smem, int mode, double t,
                              const T* u, const T* w, T* out, cudaStream_t st) {
  return launch_smem(field_op_kernel<T, ConvAdapter<T>>, tiles, smem, st, p, mode, t, u, w, out);
}

template <typename T>
cudaError_t launch_pack_conv(const PackParams<T>& pp, cudaStream_t st) {
  pack_conv_kernel<T><<<148, 256, 0, st>>>(pp);
  return cudaGetLastError();
}

// out[j] = sum_t in[t * stride + j] in tile order (deterministic)
template <typename T>
__global__ void reduce_plain_kernel(const T* in, int tiles, long long stride, long long n, T* out) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < tiles; ++t) acc += double(in[t * stride + j]);
    out[j] = T(acc);
  }
}

template <typename T>
cudaError_t launch_reduce_plain(const T* in, int tiles, long long stride, long long n, T* out,
                                cudaStream_t st) {
  reduce_plain_kernel<T><<<std::max<long long>(1, std::min<long long>((n + 255) / 256, 592)), 256, 0,
                           st>>>(in, tiles, stride, n, out);
  return cudaGetLastError();
}

}  // namespace ob
