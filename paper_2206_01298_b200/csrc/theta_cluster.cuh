// theta_cluster.cuh -- theta-method (Crank-Nicolson / backward Euler) forward and
// discrete-adjoint kernels for fp64 two-layer MLP / stiff fields with the WEIGHTS RESIDENT
// ON CHIP across a thread-block cluster (config C5: a*u + s*MLP(u), 128 -> 512 -> 128).
//
// The single-CTA theta kernels (theta_impl.cuh) stream the 1 MB of fp64 weights from L2
// for every Krylov operator product of a 2-row tile: 65 % of the C5 sweep, at 53k cycles
// per product.  Here a cluster of CL = 8 CTAs splits the HIDDEN units: CTA c keeps rows
// [c H/8, (c+1) H/8) of W1 and the matching columns of W2 in shared memory (2 x 64 KB)
// and evaluates its slice for ALL 8 x R rows of the cluster, so a product needs no weight
// traffic at all:
//   1. all-gather: every CTA writes its R input rows into every CTA's X (distributed
//      shared memory stores), cluster barrier;
//   2. slice products: Z = X W1_c^T, T = act'(.) o Z, partial O = T W2_c^T;
//   3. reduce-scatter: the partial rows go straight into the owning CTA's receive buffer
//      [source rank][row], cluster barrier, and the owner sums the eight partials in rank
//      order (deterministic).
// Everything per sample -- Newton iterates, GMRES(m) state machines, Arnoldi, Givens --
// stays with the CTA that owns the row, exactly as in theta_impl.cuh (gmres_tile is shared);
// the lockstep loops vote across the cluster so that all eight CTAs apply the operator the
// same number of times.  Parameter cotangents need no exchange: CTA c accumulates dW for its
// own hidden slice over all 16 rows.
// Reference: theta_step / newton_solve / gmres (integrators.py:225-244, linalg.py:37-142),
// theta_adjoint_step (adjoint.py:97-126); same per-sample semantics as theta_impl.cuh.
#pragma once

#include "theta_impl.cuh"

// CTAs per cluster: 8 (the portable maximum) unless the including translation unit asks for
// another size.  Everything below lives in an inline namespace named after the size, so the
// builds of different sizes are distinct entities at link time.
#ifndef OB_THCL_CL
#define OB_THCL_CL 8
#endif
#define OB_THCL_NS2(n) thcl_cl##n
#define OB_THCL_NS(n) OB_THCL_NS2(n)

namespace ob {
inline namespace OB_THCL_NS(OB_THCL_CL) {

namespace thcl {
constexpr int kCL = OB_THCL_CL;
// parameter cotangents of the explicit-RK adapter accumulate in registers over the whole sweep
// (clusters of two: a CTA's slice is half of every weight matrix, far too much to
// read-modify-write through L2 per VJP); kMuSlots output tiles per warp and matrix
constexpr bool kRegMu = kCL == 2;
constexpr int kMuSlots = 8;
constexpr int kRkThreads = kCL == 2 ? 256 : kThreads;

OB_DEV uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
OB_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the same shared-memory location in CTA `rank` of the cluster
OB_DEV uint32_t remote(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
OB_DEV void st_remote(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
OB_DEV void st_remote(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Element (row, col) of a row-major [rows][ld] fp64 array whose 32-byte chunks are XOR-swizzled
// with the row (ld / 4 >= 8 chunks): the 8 x 4 and 4 x 8 operand fragments of the fp64 MMA then
// touch every bank once, with no padding.
OB_DEV int sw(int row, int col, int ld) { return row * ld + ((((col >> 2) ^ (row & 7)) << 2) | (col & 3)); }
// fp64 tensor-core MMA, D (8 x 8) += A (8 x 4, row) B (4 x 8, col): lane l holds A[l/4][l%4],
// B[l%4][l/4] and D[l/4][2 (l%4) .. + 1]
OB_DEV void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
}  // namespace thcl

// Geometry of one cluster tile (host and device)
struct ThclGeom {
  int N, H, HS, R, RC;      // state dim, hidden, hidden slice, max rows per CTA, max rows per cluster (even)
  int ld1, ld2;             // leading dims of the W1 slice [HS][ld1] and the W2 slice [N][ld2]
  // offsets in doubles from the start of the cluster region
  int w1, w2, b1, b2, x, hs, ts, recv, flags, total;
  int x2;   // second row buffer (the VJP's cotangent rows beside the linearisation rows), or -1
  int mb;   // bias-cotangent accumulators of the sweep (db2 [N] | db1 slice [HS]), or -1
};
__host__ __device__ inline ThclGeom thcl_geom(int N, int H, int R, int RC, bool second_x = false) {
  ThclGeom g{};
  g.N = N; g.H = H; g.HS = H / thcl::kCL; g.R = R;
  // the MMA row tiles read whole groups of 8 rows: the fixed-rows geometry (whose last buffer is
  // a row buffer) allocates them; the theta geometry's row buffers are followed by others
  g.RC = second_x ? (RC + 7) & ~7 : (RC + 1) & ~1;
  g.ld1 = N;                // rows are XOR-swizzled in 32-byte chunks (thcl::sw), not padded
  g.ld2 = g.HS;
  int o = 0;
  auto take = [&](int n) { int r = o; o += (n + 1) & ~1; return r; };
  g.w1 = take(g.HS * g.ld1);
  g.w2 = take(N * g.ld2);
  g.b1 = take(g.HS);
  g.b2 = take(N);
  g.x = take(g.RC * N);
  g.hs = take(g.RC * g.HS);
  g.ts = take(g.RC * g.HS);
  g.recv = take(thcl::kCL * R * N);
  g.flags = take(2 * thcl::kCL);   // int pairs inside doubles: 2 x kCL ints fit
  g.mb = second_x ? take(N + g.HS) : -1;
  g.x2 = second_x ? take(g.RC * N) : -1;
  g.total = o;
  return g;
}

// The MLP of the field on the cluster (two affine layers, no time input).
struct ClusterNet {
  const RkParams<double>& p;
  ThclGeom g;
  double *w1, *w2, *b1, *b2, *X, *Hs, *Ts, *recv, *X2, *mb;
  int* flags;
  uint32_t rank, vpar;
  // rows of the batch are dealt evenly to the clusters, and a cluster's rows evenly
  // (contiguous ranges) to its CTAs: nk rows in this cluster, q or q + 1 per CTA
  int nk, q, e;
  int row0, Rv;   // this CTA's global rows [row0, row0 + Rv)
  int off;        // its first row within the cluster
  double mu2[thcl::kMuSlots][2][2], mu1[thcl::kMuSlots][2][2];   // kRegMu: dW2 / dW1 slice tiles of this warp

  OB_DEV ClusterNet(const RkParams<double>& p_, double* region, bool fixed_rows = false)
      : p(p_), g(thcl_geom(p_.d.N, p_.d.w[1], p_.R, fixed_rows ? thcl::kCL * p_.R : (int)p_.tile_aux, fixed_rows)),
        vpar(0) {
    w1 = region + g.w1; w2 = region + g.w2; b1 = region + g.b1; b2 = region + g.b2;
    X = region + g.x; Hs = region + g.hs; Ts = region + g.ts; recv = region + g.recv;
    X2 = g.x2 >= 0 ? region + g.x2 : nullptr;
    mb = g.mb >= 0 ? region + g.mb : nullptr;
    flags = reinterpret_cast<int*>(region + g.flags);
    rank = thcl::cta_rank();
    if (fixed_rows) {   // the generic RK kernels' mapping: tile t holds rows [t R, t R + R)
      const int base = (int)(blockIdx.x - rank) * p.R;
      nk = max(0, min(thcl::kCL * p.R, p.B - base));
      q = p.R;
      e = 0;
      off = (int)rank * p.R;
      row0 = base + off;
      Rv = max(0, min(p.R, p.B - row0));
    } else {
      const int ncl = (int)gridDim.x / thcl::kCL, k = (int)blockIdx.x / thcl::kCL;
      nk = p.B / ncl + (k < p.B % ncl ? 1 : 0);
      const int base = k * (p.B / ncl) + min(k, p.B % ncl);
      q = nk / thcl::kCL;
      e = nk % thcl::kCL;
      Rv = q + ((int)rank < e ? 1 : 0);
      off = (int)rank * q + min((int)rank, e);
      row0 = base + off;
    }
    // weight slices from the packed (zero padded) copies: W1 [H][ldw0], W2 [N][ldw1]
    const double* W1 = p.packed + p.d.pwoff[0];
    const double* W2 = p.packed + p.d.pwoff[1];
    const int N = g.N, HS = g.HS, k0 = (int)rank * HS;
    for (int i = threadIdx.x; i < HS * N; i += blockDim.x) {
      const int k = i / N, c = i % N;
      w1[thcl::sw(k, c, N)] = W1[(long long)(k0 + k) * p.d.ldw[0] + c];
    }
    for (int i = threadIdx.x; i < N * HS; i += blockDim.x) {
      const int j = i / HS, k = i % HS;
      w2[thcl::sw(j, k, HS)] = W2[(long long)j * p.d.ldw[1] + k0 + k];
    }
    for (int i = threadIdx.x; i < HS; i += blockDim.x) b1[i] = p.W.bias[0][k0 + i];
    for (int i = threadIdx.x; i < N; i += blockDim.x) b2[i] = p.W.bias[1][i];
    for (int i = threadIdx.x; i < 2 * thcl::kCL; i += blockDim.x) flags[i] = 0;
    if constexpr (thcl::kRegMu) {
      for (int i = threadIdx.x; i < g.N + g.HS; i += blockDim.x) mb[i] = 0.0;
#pragma unroll
      for (int s = 0; s < thcl::kMuSlots; ++s)
        mu2[s][0][0] = mu2[s][0][1] = mu2[s][1][0] = mu2[s][1][1] = mu1[s][0][0] = mu1[s][0][1] = mu1[s][1][0] =
            mu1[s][1][1] = 0.0;
    }
    __syncthreads();
    thcl::cluster_sync();   // every CTA's buffers exist before anyone writes into them
  }

  // ---- cluster-wide votes (double-buffered flags: one cluster barrier per vote)
  OB_DEV int vote_any(int v) {
    const int loc = __syncthreads_or(v);
    int* f = flags + thcl::kCL * vpar;
    if (threadIdx.x < thcl::kCL) thcl::st_remote(thcl::remote(f + rank, threadIdx.x), loc);
    thcl::cluster_sync();
    int r = 0;
#pragma unroll
    for (int c = 0; c < thcl::kCL; ++c) r |= f[c];
    vpar ^= 1u;
    return r;
  }
  OB_DEV int vote_all(int v) { return !vote_any(!v); }

  // ---- step 1: this CTA's rows (src [Rv][ld]) -> every CTA's X at the cluster row index.
  // any_io (nullable): a cluster-wide "any" vote carried on the same barrier.
  OB_DEV void gather(const double* src, int ld, int, int* any_io = nullptr, double* Xd = nullptr) {
    const int N = g.N;
    if (!Xd) Xd = X;
    int* f = flags + thcl::kCL * vpar;
    if (any_io) {
      const int loc = __syncthreads_or(*any_io);
      if (threadIdx.x < thcl::kCL) thcl::st_remote(thcl::remote(f + rank, threadIdx.x), loc);
    }
    for (int i = threadIdx.x; i < Rv * N * thcl::kCL; i += blockDim.x) {
      const int c = i / (Rv * N), el = i % (Rv * N), r = el / N, j = el % N;
      thcl::st_remote(thcl::remote(Xd + thcl::sw(off + r, j, N), c), src[r * ld + j]);
    }
    thcl::cluster_sync();
    if (any_io) {
      int r = 0;
#pragma unroll
      for (int c = 0; c < thcl::kCL; ++c) r |= f[c];
      vpar ^= 1u;
      *any_io = r;
    }
  }
  // two row sets in one exchange (the VJP's linearisation rows -> X and cotangent rows -> X2)
  OB_DEV void gather_pair(const double* s1, int ld1, const double* s2, int ld2) {
    const int N = g.N;
    for (int i = threadIdx.x; i < Rv * N * thcl::kCL; i += blockDim.x) {
      const int c = i / (Rv * N), el = i % (Rv * N), r = el / N, j = el % N;
      const int o = thcl::sw(off + r, j, N);
      thcl::st_remote(thcl::remote(X + o, c), s1[r * ld1 + j]);
      thcl::st_remote(thcl::remote(X2 + o, c), s2[r * ld2 + j]);
    }
    thcl::cluster_sync();
  }
  // ---- step 3: owner side of the reduce-scatter: out[r][j] = sum over ranks (+ bias)
  OB_DEV void reduce(double* out, int ldo, const double* bias) {
    thcl::cluster_sync();
    const int N = g.N, R = g.R;
    for (int i = threadIdx.x; i < Rv * N; i += blockDim.x) {
      const int r = i / N, j = i % N;
      double acc = recv[(0 * R + r) * N + j];
#pragma unroll
      for (int c = 1; c < thcl::kCL; ++c) acc = Num<double>::add(acc, recv[(c * R + r) * N + j]);
      out[r * ldo + j] = bias ? Num<double>::add(acc, bias[j]) : acc;
    }
    __syncthreads();
  }
  // cluster row r (< nk) -> the remote address of its slot in the owner's receive buffer
  // (column 0); partial outputs are stored at + 8 j
  OB_DEV uint32_t scatter_row(int r) const {
    const int big = e * (q + 1);   // rows held by the CTAs with q + 1 rows
    const int c = r < big ? r / (q + 1) : e + (r - big) / max(q, 1);
    const int loc = r < big ? r % (q + 1) : (r - big) % max(q, 1);
    return thcl::remote(recv + ((int)rank * g.R + loc) * g.N, (uint32_t)c);
  }

  // ---- slice products on the fp64 tensor cores (mma.sync m8n8k4).  With FMAs on the vector
  // pipe the products ran at a fifth of its rate (10.7k cycles for 147 k FMAs): every FMA
  // needs a shared-memory operand, and a warp-wide broadcast operand costs as many wavefronts
  // as a distinct one.  An MMA takes 32 + 32 distinct operand values for 256 FMAs, and the A
  // fragment is reused across the N tiles of a task.  (The pipes' rates are equal: 64
  // FMA/clk/SM for DMMA, tools/dmma_probe.cu.)
  // D[r][n] = sum_k A[r][k] Bm[n][k]   (A: [rows][KD], Bm: [ncols][KD], both swizzled).
  // Task = (group of MTG row tiles, pair of column tiles), one per warp.
  template <int MTG, class Out>
  OB_DEV void mma_nt(const double* A, int RC, const double* Bm, int ncols, int KD, Out out) {
    const int lane = lane_id(), lr = lane >> 2, lc = lane & 3;
    const int MT = (RC + 7) / 8, mgroups = (MT + MTG - 1) / MTG, npairs = ncols / 16;
    for (int task = warp_id(); task < mgroups * npairs; task += n_warps()) {
      const int np = task % npairs, mg = task / npairs;
      double c[MTG][2][2];
#pragma unroll
      for (int m = 0; m < MTG; ++m) c[m][0][0] = c[m][0][1] = c[m][1][0] = c[m][1][1] = 0.0;
      const int n0 = 16 * np + lr, n1 = n0 + 8;
#pragma unroll 4
      for (int ks = 0; ks < KD / 4; ++ks) {
        const double b0 = Bm[n0 * KD + (((ks ^ (n0 & 7)) << 2) | lc)];
        const double b1 = Bm[n1 * KD + (((ks ^ (n1 & 7)) << 2) | lc)];
#pragma unroll
        for (int m = 0; m < MTG; ++m) {
          const int r = 8 * (mg * MTG + m) + lr;   // (rows past RC: finite shared memory, discarded)
          const double a = A[r * KD + (((ks ^ (r & 7)) << 2) | lc)];
          thcl::dmma(c[m][0][0], c[m][0][1], a, b0);
          thcl::dmma(c[m][1][0], c[m][1][1], a, b1);
        }
      }
#pragma unroll
      for (int m = 0; m < MTG; ++m) {
        const int r = 8 * (mg * MTG + m) + lr;
        if (r < RC) {
          auto ro = out(r);   // per-row output (the scatter resolves the row's owner once)
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            ro(16 * np + 8 * t + 2 * lc, c[m][t][0]);
            ro(16 * np + 8 * t + 2 * lc + 1, c[m][t][1]);
          }
        }
      }
    }
  }
  // D[r][n] = sum_k A[r][k] Bt[k][n]   (Bt: [KD][ncols], swizzled by its rows k)
  template <int MTG, class Out>
  OB_DEV void mma_tn(const double* A, int RC, const double* Bt, int ncols, int KD, Out out) {
    const int lane = lane_id(), lr = lane >> 2, lc = lane & 3;
    const int MT = (RC + 7) / 8, mgroups = (MT + MTG - 1) / MTG, npairs = ncols / 16;
    for (int task = warp_id(); task < mgroups * npairs; task += n_warps()) {
      const int np = task % npairs, mg = task / npairs;
      double c[MTG][2][2];
#pragma unroll
      for (int m = 0; m < MTG; ++m) c[m][0][0] = c[m][0][1] = c[m][1][0] = c[m][1][1] = 0.0;
      const int n0 = 16 * np + lr, n1 = n0 + 8;
#pragma unroll 4
      for (int ks = 0; ks < KD / 4; ++ks) {
        const int kr = 4 * ks + lc;   // B fragment: row k = 4 ks + l % 4, column n = l / 4
        const double b0 = Bt[thcl::sw(kr, n0, ncols)];
        const double b1 = Bt[thcl::sw(kr, n1, ncols)];
#pragma unroll
        for (int m = 0; m < MTG; ++m) {
          const int r = 8 * (mg * MTG + m) + lr;
          const double a = A[r * KD + (((ks ^ (r & 7)) << 2) | lc)];
          thcl::dmma(c[m][0][0], c[m][0][1], a, b0);
          thcl::dmma(c[m][1][0], c[m][1][1], a, b1);
        }
      }
#pragma unroll
      for (int m = 0; m < MTG; ++m) {
        const int r = 8 * (mg * MTG + m) + lr;
        if (r < RC) {
          auto ro = out(r);   // per-row output (the scatter resolves the row's owner once)
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            ro(16 * np + 8 * t + 2 * lc, c[m][t][0]);
            ro(16 * np + 8 * t + 2 * lc + 1, c[m][t][1]);
          }
        }
      }
    }
  }
  // A: Z[r][k] = sum_i In[r][i] W1s[k][i]
  template <class Epi>
  OB_DEV void prod_a(const double* In, Epi epi) {
    mma_nt<1>(In, nk, w1, g.HS, g.N, [&](int r) { return [=](int k, double v) { epi(r, k, v); }; });
  }
  // B: O[r][j] = sum_k Tin[r][k] W2s[j][k]  (partial over this slice) -> scatter
  OB_DEV void prod_b(const double* Tin) {
    auto out = [&](int r) {
      const uint32_t base = scatter_row(r);
      return [=](int j, double v) { thcl::st_remote(base + 8u * (uint32_t)j, v); };
    };
    if constexpr (thcl::kCL == 2) {   // at most 12 rows per cluster: one or two row tiles
      if (nk <= 8) mma_nt<1>(Tin, nk, w2, g.N, g.HS, out);
      else mma_nt<2>(Tin, nk, w2, g.N, g.HS, out);
    } else {
      mma_nt<3>(Tin, nk, w2, g.N, g.HS, out);
    }
  }
  // C: G[r][k] = sum_j V[r][j] W2s[j][k]
  template <class Epi>
  OB_DEV void prod_c(const double* V, Epi epi) {
    mma_tn<1>(V, nk, w2, g.HS, g.N, [&](int r) { return [=](int k, double v) { epi(r, k, v); }; });
  }
  // D: O[r][i] = sum_k Tin[r][k] W1s[k][i]  (partial over this slice) -> scatter
  OB_DEV void prod_d(const double* Tin) {
    auto out = [&](int r) {
      const uint32_t base = scatter_row(r);
      return [=](int i, double v) { thcl::st_remote(base + 8u * (uint32_t)i, v); };
    };
    if constexpr (thcl::kCL == 2) {
      if (nk <= 8) mma_tn<1>(Tin, nk, w1, g.N, g.HS, out);
      else mma_tn<2>(Tin, nk, w1, g.N, g.HS, out);
    } else {
      mma_tn<3>(Tin, nk, w1, g.N, g.HS, out);
    }
  }
  // parameter cotangents of a slice on the MMA as well: M[a][b] += scale sum_{r < nk} P[r][a] Q[r][b]
  // (P: [rows][pa], Q: [rows][qb], swizzled; rows past nk masked), added to mu at
  // dst[a * ldm + b].  One 8 x 16 output tile per task.
  OB_DEV void outer_acc(const double* P, int pa, const double* Q, int qb, double scale, double* dst, long long ldm) {
    const int lane = lane_id(), lr = lane >> 2, lc = lane & 3;
    const int npairs = qb / 16, mtiles = pa / 8;
    for (int task = warp_id(); task < mtiles * npairs; task += n_warps()) {
      const int np = task % npairs, mt = task / npairs;
      double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      const int a0 = 8 * mt + lr, n0 = 16 * np + lr, n1 = n0 + 8;
      for (int rs = 0; rs < nk; rs += 4) {
        const int r = rs + lc;   // A fragment: A[a][r] = P[r][a]; B fragment: B[r][n] = Q[r][n]
        const bool ok = r < nk;
        const double a = ok ? P[thcl::sw(r, a0, pa)] : 0.0;
        const double b0 = ok ? Q[thcl::sw(r, n0, qb)] : 0.0;
        const double b1 = ok ? Q[thcl::sw(r, n1, qb)] : 0.0;
        thcl::dmma(c[0][0], c[0][1], a, b0);
        thcl::dmma(c[1][0], c[1][1], a, b1);
      }
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          double* m = dst + (long long)a0 * ldm + 16 * np + 8 * t + 2 * lc + u;
          *m = Num<double>::fma(scale, c[t][u], *m);
        }
    }
  }

  // the same product into this warp's register tiles (kRegMu): acc[s] is output tile
  // warp + s * n_warps; the scale goes on the P fragment
  // register tile s of this warp: output tile (row tile mt, column pair np).  When the warps
  // divide evenly over the column pairs a warp keeps ONE column pair for all its tiles (its B
  // fragments are then loaded once per k-step for all of them); else tiles are dealt round robin.
  OB_DEV bool mu_tile(int s, int mtiles, int npairs, int& mt, int& np) const {
    const int w = warp_id(), nw = n_warps();
    if (nw % npairs == 0) {
      np = w % npairs;
      mt = w / npairs + s * (nw / npairs);
      return mt < mtiles;
    }
    const int task = w + s * nw;
    np = task % npairs;
    mt = task / npairs;
    return task < mtiles * npairs;
  }
  template <bool SHARED_B>
  OB_DEV void outer_reg_impl(const double* P, int pa, const double* Q, int qb, double scale,
                             double (&acc)[thcl::kMuSlots][2][2]) {
    const int lane = lane_id(), lr = lane >> 2, lc = lane & 3;
    const int npairs = qb / 16, mtiles = pa / 8;
    int oa[thcl::kMuSlots], o0[thcl::kMuSlots];   // operand columns per tile (no branches: the
    bool live[thcl::kMuSlots];                    // tiles' loads and MMAs interleave)
#pragma unroll
    for (int s = 0; s < thcl::kMuSlots; ++s) {
      int mt, np;
      live[s] = mu_tile(s, mtiles, npairs, mt, np);
      oa[s] = 8 * (live[s] ? mt : 0) + lr;
      o0[s] = 16 * (live[s] ? np : 0) + lr;
    }
    for (int rs = 0; rs < nk; rs += 4) {
      const bool ok = rs + lc < nk;
      const int r = ok ? rs + lc : 0;
      double a[thcl::kMuSlots], b0[thcl::kMuSlots], b1[thcl::kMuSlots];
#pragma unroll
      for (int s = 0; s < thcl::kMuSlots; ++s) {
        // unconditional loads from clamped (valid) addresses: a conditional load compiles to a
        // branch per operand (the dead fragments are finite values of row 0 / tile 0 times a
        // zero scale)
        a[s] = Num<double>::mul((ok && live[s]) ? scale : 0.0, P[thcl::sw(r, oa[s], pa)]);
        if (!SHARED_B || s == 0) {
          b0[s] = Q[thcl::sw(r, o0[s], qb)];
          b1[s] = Q[thcl::sw(r, o0[s] + 8, qb)];
        } else {
          b0[s] = b0[0];
          b1[s] = b1[0];
        }
      }
#pragma unroll
      for (int s = 0; s < thcl::kMuSlots; ++s) {
        thcl::dmma(acc[s][0][0], acc[s][0][1], a[s], b0[s]);
        thcl::dmma(acc[s][1][0], acc[s][1][1], a[s], b1[s]);
      }
    }
  }
  OB_DEV void outer_reg(const double* P, int pa, const double* Q, int qb, double scale,
                        double (&acc)[thcl::kMuSlots][2][2]) {
    if (n_warps() % (qb / 16) == 0) outer_reg_impl<true>(P, pa, Q, qb, scale, acc);
    else outer_reg_impl<false>(P, pa, Q, qb, scale, acc);
  }
  OB_DEV void flush_reg(int pa, int qb, const double (&acc)[thcl::kMuSlots][2][2], double* dst, long long ldm) {
    const int lane = lane_id(), lr = lane >> 2, lc = lane & 3;
    const int npairs = qb / 16, mtiles = pa / 8;
#pragma unroll
    for (int s = 0; s < thcl::kMuSlots; ++s) {
      int mt, np;
      if (mu_tile(s, mtiles, npairs, mt, np)) {
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            double* m = dst + (long long)(8 * mt + lr) * ldm + 16 * np + 8 * t + 2 * lc + u;
            *m = Num<double>::add(*m, acc[s][t][u]);
          }
      }
    }
  }
  // end of the sweep: the register tiles join the CTA's mu slot
  OB_DEV void finish_mu(double* mu) {
    if constexpr (thcl::kRegMu) {
      const int k0 = (int)rank * g.HS;
      flush_reg(g.N, g.HS, mu2, mu + p.d.mwoff[1] + k0, p.d.ldm[1]);
      flush_reg(g.HS, g.N, mu1, mu + p.d.mwoff[0] + (long long)k0 * p.d.ldm[0], p.d.ldm[0]);
      for (int j = threadIdx.x; j < g.N; j += blockDim.x) {
        double* m = mu + p.d.mboff[1] + j;
        *m = Num<double>::add(*m, mb[j]);
      }
      for (int k = threadIdx.x; k < g.HS; k += blockDim.x) {
        double* m = mu + p.d.mboff[0] + k0 + k;
        *m = Num<double>::add(*m, mb[g.N + k]);
      }
    }
  }

  // hidden activations of the rows in `src` (cached for the tangent / cotangent passes);
  // with out: the MLP value W2 act(W1 x + b1) + b2 for this CTA's rows
  // (no_sync: the caller's next exchange does not write X -- a VJP that gathers its cotangent
  // rows into the second row buffer -- so the closing barrier is not needed)
  // pre_gathered: X already holds the cluster's rows (gather_pair).
  OB_DEV void forward(const double* src, int ld, int Rv, double* out, int ldo, bool no_sync = false,
                      bool pre_gathered = false) {
    // (profiling slots of tools/profile_step.py --phases: 10 all-gather, 11 hidden product +
    // activation, 12 output product + scatter, 13 reduce / barrier; in vjp(): 14 all-gather,
    // 15 W2^T product, 6 parameter cotangents, 7 W1^T product + scatter, 4 reduce)
    PhaseTimer pt(p.prof ? p.phase : nullptr);
    if (!pre_gathered) gather(src, ld, Rv);
    pt.mark(10);
    const int HS = g.HS, act = p.d.act;
    double* H = Hs;
    const double* bb = b1;
    prod_a(X, [&](int r, int k, double z) { H[thcl::sw(r, k, HS)] = act_fn(Num<double>::add(z, bb[k]), act); });
    __syncthreads();
    pt.mark(11);
    if (out) {
      prod_b(Hs);
      if (p.prof) __syncthreads();
      pt.mark(12);
      reduce(out, ldo, b2);
      pt.mark(13);
    } else if (!no_sync) {
      thcl::cluster_sync();   // X is rewritten by the next gather of any CTA
      pt.mark(13);
    }
  }
  // (dMLP/du) v at the cached linearisation (tanh / identity / relu: act' from the value)
  OB_DEV void jvp(const double* v, int ld, int Rv, double* out, int ldo, int* any_io = nullptr) {
    PhaseTimer pt(p.prof ? p.phase : nullptr);
    gather(v, ld, Rv, any_io);
    if (any_io && !*any_io) return;   // (cluster-uniform) nobody iterates: no product
    pt.mark(0);   // all-gather (remote stores + cluster barrier)
    const int HS = g.HS, act = p.d.act;
    const double* H = Hs;
    double* Tt = Ts;
    prod_a(X, [&](int r, int k, double z) {
      const double a = H[thcl::sw(r, k, HS)];
      Tt[thcl::sw(r, k, HS)] = Num<double>::mul(z, act_prime_from(a, a, act));
    });
    __syncthreads();
    pt.mark(1);   // first slice product
    prod_b(Ts);
    __syncthreads();
    pt.mark(2);   // second slice product + scatter stores
    reduce(out, ldo, nullptr);
    pt.mark(3);   // cluster barrier + owner sum
  }
  // (dMLP/du)^T v -> jtv; with mu: mu += scale (dMLP/dtheta)^T v over the valid rows.  xin:
  // the rows the linearisation was taken at (for dW1), gathered again when mu is given.
  OB_DEV void vjp(const double* v, int ld, int Rv, double* jtv, int ldo, double* mu, double scale,
                  const double* xin, int ldx, int* any_io = nullptr, bool pre_gathered = false) {
    const int N = g.N, HS = g.HS, act = p.d.act;
    const double* H = Hs;
    double* Tt = Ts;
    // With a second row buffer the cotangent rows go beside the linearisation rows X (still
    // there from forward()), so dW1 needs no second all-gather and every use of X precedes
    // the reduce barrier: two cluster barriers per VJP instead of four.
    const bool keep_x = mu && X2 != nullptr;
    double* V = keep_x ? X2 : X;
    PhaseTimer pt(p.prof ? p.phase : nullptr);
    if (!pre_gathered) gather(v, ld, Rv, any_io, V);   // all cotangent rows of the cluster
    if (any_io && !*any_io) return;
    pt.mark(14);
    prod_c(V, [&](int r, int k, double gk) {
      const double a = H[thcl::sw(r, k, HS)];
      Tt[thcl::sw(r, k, HS)] = Num<double>::mul(gk, act_prime_from(a, a, act));
    });
    __syncthreads();
    pt.mark(15);
    const int k0 = (int)rank * HS;
    if (mu) {   // dW2 slice, db2 (own rows), db1 slice
      if (thcl::kRegMu && keep_x) outer_reg(V, N, H, HS, scale, mu2);
      else outer_acc(V, N, H, HS, scale, mu + p.d.mwoff[1] + k0, p.d.ldm[1]);   // dW2[j][k0 + k] += v^T a
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        double acc = 0.0;
        for (int r = 0; r < Rv; ++r) acc = Num<double>::add(acc, V[thcl::sw(off + r, j, N)]);
        double* m = (thcl::kRegMu && keep_x) ? mb + j : mu + p.d.mboff[1] + j;
        *m = Num<double>::fma(scale, acc, *m);
      }
      for (int k = threadIdx.x; k < HS; k += blockDim.x) {
        double acc = 0.0;
        for (int r = 0; r < nk; ++r) acc = Num<double>::add(acc, Tt[thcl::sw(r, k, HS)]);
        double* m = (thcl::kRegMu && keep_x) ? mb + N + k : mu + p.d.mboff[0] + k0 + k;
        *m = Num<double>::fma(scale, acc, *m);
      }
      if (thcl::kRegMu && keep_x) outer_reg(Tt, HS, X, N, scale, mu1);
      else if (keep_x)   // dW1[k0 + k][i] += (act' o W2^T v)^T x
        outer_acc(Tt, HS, X, N, scale, mu + p.d.mwoff[0] + (long long)k0 * p.d.ldm[0], p.d.ldm[0]);
    }
    if (p.prof) __syncthreads();   // (phase boundaries only: nothing below depends on the cotangent sums)
    pt.mark(6);
    prod_d(Ts);
    if (p.prof) __syncthreads();
    pt.mark(7);
    reduce(jtv, ldo, nullptr);   // (cluster barrier: X / X2 may be overwritten below)
    pt.mark(4);
    if (mu && !keep_x) {   // dW1 slice needs the layer input of every row: gather it again
      gather(xin, ldx, Rv);
      outer_acc(Tt, HS, X, N, scale, mu + p.d.mwoff[0] + (long long)k0 * p.d.ldm[0], p.d.ldm[0]);
      __syncthreads();
      thcl::cluster_sync();   // X is rewritten by the next gather of any CTA
    }
  }
};

// Field adapter of the generic explicit-RK kernels (rk_impl.cuh) over the cluster MLP:
// fp64 two-layer MlpField without a time input (config C1).  Tiles keep the generic row
// mapping (tile t = rows [t R, t R + R)); eval / vjp are the cluster products.
struct ClusterMlpAdapter {
  static constexpr bool kHasJvp = false;
  static constexpr bool kScaledVjp = false;   // vjp returns J^T w; mu += h P^T w
  static constexpr int kCombineBatch = 4;
  static constexpr bool kOwnsStep = false;
  static constexpr bool kNoEarlyExit = true;  // the cluster applies its products together
  static constexpr int kBlockThreads = thcl::kRkThreads;
  const RkParams<double>& p;
  ClusterNet net;
  double* xin;   // field input rows [Rt][lda0]
  OB_DEV ClusterMlpAdapter(const RkParams<double>& p_, const Weights<double>&, MlpSmem<double>& ms, double* sm, int, int)
      : p(p_), net(p_, sm + p_.sm.aux, true), xin(ms.x0) {}
  OB_DEV double* x0() { return xin; }
  OB_DEV int nin() const { return p.d.N; }
  OB_DEV void put(int r, int j, double v) { xin[r * p.d.lda[0] + j] = v; }
  OB_DEV void put_time(double) {}
  OB_DEV void set_scratch(double*, int) {}
  OB_DEV void jvp(const double*, double*) {}
  OB_DEV void finish(double* mu) { net.finish_mu(mu); }
  OB_DEV void release() { thcl::cluster_sync(); }   // no CTA leaves while a partner may still write into it
  OB_DEV void eval(double* out) { net.forward(xin, p.d.lda[0], net.Rv, out, p.d.ldn); }
  OB_DEV void vjp(const double* w, double* jtv, double* mu, double h, int) {
    if (mu != nullptr && net.X2 != nullptr) {
      // stage-state rows and cotangent rows in ONE exchange (both buffers are free: every read
      // of the previous VJP precedes its reduce barrier), then the hidden activations at the
      // stage state and the VJP without further gathers
      net.gather_pair(xin, p.d.lda[0], w, p.d.ldn);
      net.forward(xin, p.d.lda[0], net.Rv, nullptr, 0, true, true);
      net.vjp(w, p.d.ldn, net.Rv, jtv, p.d.ldn, mu, h, xin, p.d.lda[0], nullptr, true);
      return;
    }
    net.forward(xin, p.d.lda[0], net.Rv, nullptr, 0);   // hidden activations at the stage state
    net.vjp(w, p.d.ldn, net.Rv, jtv, p.d.ldn, mu, h, xin, p.d.lda[0]);
  }
};

struct ClVote {
  ClusterNet* net;
  OB_DEV int any(int v) const { return net->vote_any(v); }
  OB_DEV int all(int v) const { return net->vote_all(v); }
};

// Operator A v = v - (h theta) J v / J^T v on the cluster (see ThetaOp)
struct ThclOp {
  const RkParams<double>& p;
  ClusterNet& net;
  double hth;
  bool transpose;
  double* tmp;
  int Rv;
  template <class Vote>
  OB_DEV bool apply_any(int any, const double* vin, double* vout, Vote&) {
    const int N = p.d.N, ldn = p.d.ldn;
    if (transpose) net.vjp(vin, ldn, Rv, tmp, ldn, nullptr, 0.0, nullptr, 0, &any);
    else net.jvp(vin, ldn, Rv, tmp, ldn, &any);
    if (!any) return false;
    for (int i = threadIdx.x; i < p.Rt * N; i += blockDim.x) {
      const int o = (i / N) * ldn + i % N, j = i % N;
      double jv = tmp[o];
      if (p.field_kind == OB_FIELD_STIFF)
        jv = Num<double>::add(Num<double>::mul(p.diag[j], vin[o]), Num<double>::mul(p.out_scale, jv));
      vout[o] = Num<double>::add(vin[o], -Num<double>::mul(hth, jv));
    }
    __syncthreads();
    return true;
  }
};

// f(x) for this CTA's rows into c.fb (MlpAdapter::eval semantics), linearisation cached
OB_DEV void thcl_eval(const RkParams<double>& p, ClusterNet& net, ThetaCtx<double>& c, const double* x, int Rv,
                      bool count_all) {
  const int N = p.d.N, ldn = p.d.ldn;
  net.forward(x, ldn, Rv, c.fb, ldn);
  if (p.field_kind == OB_FIELD_STIFF) {
    for (int i = threadIdx.x; i < p.Rt * N; i += blockDim.x) {
      const int o = (i / N) * ldn + i % N, j = i % N;
      c.fb[o] = Num<double>::add(Num<double>::mul(p.diag[j], x[o]), Num<double>::mul(p.out_scale, c.fb[o]));
    }
    __syncthreads();
  }
  if (threadIdx.x < Rv && (count_all || c.active[threadIdx.x])) c.cnt[threadIdx.x * OB_NSTATS + OB_STAT_NFE_F] += 1;
}

OB_DEV void thcl_residual(const RkParams<double>& p, ClusterNet& net, ThetaCtx<double>& c, int Rv, double hth) {
  const int N = p.d.N, ldn = p.d.ldn;
  thcl_eval(p, net, c, c.xk, Rv, false);
  for (int i = threadIdx.x; i < p.Rt * N; i += blockDim.x) {
    const int o = (i / N) * ldn + i % N;
    c.rv[o] = Num<double>::add(Num<double>::add(c.xk[o], -c.base[o]), -Num<double>::mul(hth, c.fb[o]));
  }
  __syncthreads();
  if (warp_id() < Rv) {
    const double nr = sqrt(warp_dot(c.rv + warp_id() * ldn, c.rv + warp_id() * ldn, N));
    int fin = 1;
    for (int j = lane_id(); j < N; j += 32) fin &= Num<double>::finite(c.rv[warp_id() * ldn + j]) ? 1 : 0;
    fin = __all_sync(0xffffffffu, fin);
    if (lane_id() == 0) c.rn[warp_id()] = fin ? nr : __longlong_as_double(0x7ff8000000000000LL);
  }
  __syncthreads();
}

// theta_step_tile on the cluster: identical per-sample logic, cluster-wide loop votes
OB_DEV int thcl_step(const RkParams<double>& p, ClusterNet& net, ThetaCtx<double>& c, double* u, double t,
                     double h, double* rec, int row0, int Rv, double* kry) {
  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt;
  const long long vec = (long long)p.B * N;
  const double th = p.theta;
  const double hth = h * th, h1 = h * (1.0 - th);
  for (int r = threadIdx.x; r < Rv; r += blockDim.x) c.active[r] = 1;
  __syncthreads();
  thcl_eval(p, net, c, u, Rv, true);
  for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
    const int o = (i / N) * ldn + i % N;
    c.base[o] = Num<double>::add(u[o], Num<double>::mul(h1, c.fb[o]));
    c.xk[o] = u[o];
    if (rec && i / N < Rv) rec[(long long)(row0 + i / N) * N + i % N] = u[o];
  }
  __syncthreads();
  thcl_residual(p, net, c, Rv, hth);
  ThclOp op{p, net, hth, false, c.fb, Rv};
  ClVote vote{&net};
  for (int it = 0; it < p.newton_maxit; ++it) {
    int any = 0, bad = 0;
    if (threadIdx.x < Rv) {
      const double rn = c.rn[threadIdx.x];
      const bool act = c.active[threadIdx.x] && !(rn <= p.newton_tol);
      if (act && !isfinite(rn)) bad = 1;
      c.active[threadIdx.x] = act ? 1 : 0;
      any = act ? 1 : 0;
    }
    if (net.vote_any(bad)) return OB_ERR_CONVERGENCE;
    if (!net.vote_any(any)) break;
    for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
      const int o = (i / N) * ldn + i % N;
      c.rhs[o] = -c.rv[o];
    }
    __syncthreads();
    if (!gmres_tile<double>(p, op, c, c.rhs, c.gx, Rv, kry, OB_STAT_GMRES_F, OB_STAT_NFE_F, vote))
      return OB_ERR_CONVERGENCE;
    for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
      const int r = i / N, o = r * ldn + i % N;
      if (r < Rv && c.active[r]) c.xk[o] = Num<double>::add(c.xk[o], c.gx[o]);
    }
    if (threadIdx.x < Rv && c.active[threadIdx.x]) c.cnt[threadIdx.x * OB_NSTATS + OB_STAT_NEWTON] += 1;
    __syncthreads();
    thcl_residual(p, net, c, Rv, hth);
  }
  int bad = 0;
  if (threadIdx.x < Rv && !(c.rn[threadIdx.x] <= p.newton_tol)) bad = 1;
  if (net.vote_any(bad)) return OB_ERR_CONVERGENCE;
  for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
    const int r = i / N, o = r * ldn + i % N;
    u[o] = c.xk[o];
    if (rec && r < Rv) {
      const long long gi = (long long)(row0 + r) * N + i % N;
      rec[vec + gi] = u[o];
      rec[2 * vec + gi] = u[o];
    }
  }
  __syncthreads();
  return OB_OK;
}

#ifdef OB_THCL_KERNELS   // the theta kernels are emitted by theta_cl_f64.cu only
// --------------------------------------------------------------- forward
__global__ void __launch_bounds__(kThreads, 1) thcl_forward_kernel(const __grid_constant__ RkParams<double> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  zero_smem(sm, p.sm.total);
  const int tile = blockIdx.x;
  ClusterNet net(p, sm + p.sm.wts);
  const int row0 = net.row0, Rv = net.Rv;
  ThetaCtx<double> c = theta_ctx(p, sm);
  double* u = sm + p.sm.u;
  double* kry = p.krylov + tile * p.krylov_stride;
  const int N = p.d.N, ldn = p.d.ldn;
  const long long vec = (long long)p.B * N;
  load_rows(u, ldn, p.u0, N, row0, Rv);
  __syncthreads();
  int bad = 0;  // as_state (nn.py:31-32)
  for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x)
    if (!Num<double>::finite(u[(idx / N) * ldn + idx % N])) bad = 1;
  bad = __syncthreads_or(bad);   // this CTA's rows
  if (net.vote_any(bad)) {
    if (threadIdx.x == 0 && bad) set_status(p.status, OB_ERR_VALUE, -1);
    thcl::cluster_sync();
    return;
  }
  for (int n = 0; n < p.n_steps; ++n) {
    const double t = p.ts[n], h = p.ts[n + 1] - p.ts[n];
    obs_capture(p, u, n, row0, Rv);
    if (p.fwd_sol[n] >= 0) {
      store_rows(p.sol + p.fwd_sol[n] * vec, N, u, ldn, row0, Rv);
      __syncthreads();
    }
    double* rec = p.fwd_rec[n] >= 0 ? p.rec + (long long)p.fwd_rec[n] * 3 * vec : nullptr;
    const int st = thcl_step(p, net, c, u, t, h, rec, row0, Rv, kry);
    if (st != OB_OK) {   // cluster-uniform (voted)
      if (threadIdx.x == 0) set_status(p.status, st, n);
      flush_stats(p, c, row0, Rv);
      thcl::cluster_sync();
      return;
    }
  }
  store_rows(p.u_final, N, u, ldn, row0, Rv);
  obs_capture(p, u, p.n_steps, row0, Rv);
  flush_stats(p, c, row0, Rv);
  loss_partial(p, u, row0, Rv, tile);
  thcl::cluster_sync();   // no CTA leaves while a partner may still write into it
}

// --------------------------------------------------------------- reverse
__global__ void __launch_bounds__(kThreads, 1) thcl_reverse_kernel(const __grid_constant__ RkParams<double> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  if (*(volatile int*)p.status != 0) return;   // grid-uniform: the forward finished before
  zero_smem(sm, p.sm.total);
  const int tile = blockIdx.x;
  ClusterNet net(p, sm + p.sm.wts);
  const int row0 = net.row0, Rv = net.Rv;
  ThetaCtx<double> c = theta_ctx(p, sm);
  const int N = p.d.N, ldn = p.d.ldn, Rt = p.Rt;
  const long long vec = (long long)p.B * N;
  double* u = sm + p.sm.u;
  double* lam = sm + p.sm.lam;
  double* jtv = sm + p.sm.jtv;
  double* kry = p.krylov + tile * p.krylov_stride;
  double* mu = p.mu + tile * p.d.n_mu;
  const double th = p.theta;
  ClVote vote{&net};
  loss_seed(p, lam, row0, Rv);
  __syncthreads();
  for (int pc = 0; pc < p.prog_len; ++pc) {
    const int4 op = p.prog[pc];
    const int n = op.y;
    const double t = p.ts[n], h = p.ts[n + 1] - p.ts[n];
    if (op.x == kOpReplay) {
      const int src_kind = op.z >> 24, src = op.z & 0xffffff;
      const double* srcp = src_kind == kSrcU0 ? p.u0
                         : src_kind == kSrcSol ? p.sol + src * vec
                         : p.rec + ((long long)src * 3 + 2) * vec;
      load_rows(u, ldn, srcp, N, row0, Rv);
      __syncthreads();
      double* rec = p.rec + (long long)op.w * 3 * vec;
      const int st = thcl_step(p, net, c, u, t, h, rec, row0, Rv, kry);
      if (st != OB_OK) {
        if (threadIdx.x == 0) set_status(p.status, st, n);
        flush_stats(p, c, row0, Rv);
        thcl::cluster_sync();
        return;
      }
      continue;
    }
    // theta_adjoint_step (adjoint.py:97-126)
    obs_inject(p, lam, n + 1, row0, Rv);
    const double* rec = p.rec + (long long)op.w * 3 * vec;
    const double hth = h * th, h1 = h * (1.0 - th);
    for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
      const int r = idx / N, j = idx % N;
      u[r * ldn + j] = rec[vec + (long long)(row0 + r) * N + j];
    }
    __syncthreads();
    net.forward(u, ldn, Rv, nullptr, 0);   // linearisation at u1
    for (int r = threadIdx.x; r < Rv; r += blockDim.x) c.active[r] = 1;
    for (int i = threadIdx.x; i < Rt * ldn; i += blockDim.x) c.rhs[i] = lam[i];
    __syncthreads();
    ThclOp aop{p, net, hth, true, jtv, Rv};
    if (!gmres_tile<double>(p, aop, c, c.rhs, c.gx, Rv, kry, OB_STAT_GMRES_B, OB_STAT_NFE_B, vote)) {
      if (threadIdx.x == 0) set_status(p.status, OB_ERR_CONVERGENCE, n);
      flush_stats(p, c, row0, Rv);
      thcl::cluster_sync();
      return;
    }
    // mu += h theta P(u1)^T lam_s  (one VJP pair at u1)
    const double sc = p.field_kind == OB_FIELD_STIFF ? p.out_scale : 1.0;
    net.vjp(c.gx, ldn, Rv, jtv, ldn, mu, hth * sc, u, ldn);
    if (threadIdx.x < Rv) c.cnt[threadIdx.x * OB_NSTATS + OB_STAT_NFE_B] += 1;
    if (th < 1.0) {
      for (int idx = threadIdx.x; idx < Rv * N; idx += blockDim.x) {
        const int r = idx / N, j = idx % N;
        u[r * ldn + j] = rec[(long long)(row0 + r) * N + j];
      }
      __syncthreads();
      net.forward(u, ldn, Rv, nullptr, 0);
      net.vjp(c.gx, ldn, Rv, jtv, ldn, mu, h1 * sc, u, ldn);
      if (threadIdx.x < Rv) c.cnt[threadIdx.x * OB_NSTATS + OB_STAT_NFE_B] += 1;
      for (int i = threadIdx.x; i < Rt * N; i += blockDim.x) {
        const int o = (i / N) * ldn + i % N, j = i % N;
        double jv = jtv[o];
        if (p.field_kind == OB_FIELD_STIFF)
          jv = Num<double>::add(Num<double>::mul(p.diag[j], c.gx[o]), Num<double>::mul(p.out_scale, jv));
        lam[o] = Num<double>::add(c.gx[o], Num<double>::mul(h1, jv));
      }
    } else {
      for (int i = threadIdx.x; i < Rt * ldn; i += blockDim.x) lam[i] = c.gx[i];
    }
    int bad = 0;
    for (int i = threadIdx.x; i < Rt * N; i += blockDim.x)
      if (!Num<double>::finite(lam[(i / N) * ldn + i % N])) bad = 1;
    bad = __syncthreads_or(bad);
    if (net.vote_any(bad)) {
      if (threadIdx.x == 0 && bad) set_status(p.status, OB_ERR_GRADIENT_EXPLOSION, n);
      flush_stats(p, c, row0, Rv);
      thcl::cluster_sync();
      return;
    }
  }
  obs_inject(p, lam, 0, row0, Rv);
  store_rows(p.du0, N, lam, ldn, row0, Rv);
  flush_stats(p, c, row0, Rv);
  thcl::cluster_sync();
}

#endif  // OB_THCL_KERNELS

// ------------------------------------------------------------ launchers
template <typename K>
static cudaError_t thcl_launch(K kf, int grid, size_t smem, cudaStream_t st, const RkParams<double>& p,
                               int threads = kThreads) {
  cudaError_t e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = thcl::kCL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kf, p);
}

}  // inline namespace
}  // namespace ob
