// kernels_fast.cuh — fused sm_100a Block-CG kernels (BKG_NUMERICS_FAST).
//
// One Block-CG iteration (solver.hpp:157-201, M = I) is three fused kernels:
//   K1  Q = A P (CSR SpMM, kernels.hpp:129-157) with the Gram epilogue
//       alpha = <<P,Q>>, rho_prev = <<P,R>> (kernels.hpp:59-88); the last CTA
//       reduces the grid partials and solves lambda = alpha^-1 rho_prev
//       (kernels.hpp:231-240) on device.
//   K2  X += P lambda, R -= Q lambda (kernels.hpp:94-125), then rho = <<R,R>>
//       and the k column norms of the new R (block_vector.hpp:59-70); the last
//       CTA solves beta = rho_prev^-1 rho, records history and the stop test.
//   K3  P = R + P beta in place (Z = M^-1 R = R, solver.hpp:176-190).
//
// Layout: block vectors are row-major n x K doubles (block_vector.hpp:20-21).
// A row is served by TPR = K/CPT threads, each owning CPT consecutive lanes
// read/written as one 8- or 16-byte access, so a warp touches whole 128-byte
// lines.  The p-group of a lane (P consecutive lanes, subalgebra.hpp:104-109)
// lives in GT = P/CPT consecutive threads of one warp; the Gram tile is built
// from warp shuffles inside the group (no shared memory in the row loop).
// Reductions are deterministic: per-thread accumulators -> warp shuffles over
// row slots -> fixed-order shared-memory sum over warps -> per-CTA partial in
// global memory -> fixed-order group sums -> fixed-order total in the last
// CTA (ticket counters, no floating-point atomics).
#pragma once

#include "bsolve.cuh"
#include "common.cuh"

namespace bkg {

constexpr int kThreads = 256;
constexpr unsigned kFull = 0xffffffffu;

template <int K, int P, int CPT>
struct Layout {
  static constexpr int TPR = K / CPT;  // threads per row
  static constexpr int GT = P / CPT;   // threads per p-group
  static constexpr int RPC = kThreads / TPR;  // rows per CTA pass
  static constexpr int Q = K / P;
  static_assert(K % CPT == 0 && P % CPT == 0, "lane split");
  static_assert(TPR <= kThreads && kThreads % TPR == 0, "row split");
  static_assert(GT <= 32 && 32 % GT == 0, "p-group must sit inside a warp");
};

// CPT lanes/thread: 1 (8-byte) or 2 (16-byte) accesses.
template <int CPT>
__device__ __forceinline__ void ld_nc(double (&d)[CPT], const double* p) {
  if constexpr (CPT == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    d[0] = t.x;
    d[1] = t.y;
  } else {
    d[0] = __ldg(p);
  }
}
template <int CPT>
__device__ __forceinline__ void ld_rw(double (&d)[CPT], const double* p) {
  if constexpr (CPT == 2) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    d[0] = t.x;
    d[1] = t.y;
  } else {
    d[0] = *p;
  }
}
template <int CPT>
__device__ __forceinline__ void st(double* p, const double (&d)[CPT]) {
  if constexpr (CPT == 2) {
    *reinterpret_cast<double2*>(p) = make_double2(d[0], d[1]);
  } else {
    *p = d[0];
  }
}

// Deterministic grid-wide sum of per-thread accumulators acc[NACC] over all
// threads sharing pos = tid % TPR.  Returns true in exactly one CTA (the last
// to arrive); there red[pos*NACC + e] holds the grid totals.
template <int TPR, int NACC>
__device__ bool grid_reduce(double (&acc)[NACC], double* red, double* partials, double* gpart,
                            uint32_t* tickets, int group) {
  constexpr int E = TPR * NACC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pos = tid % TPR;
  if constexpr (TPR < 32) {
#pragma unroll
    for (int off = TPR; off < 32; off <<= 1)
#pragma unroll
      for (int e = 0; e < NACC; ++e) acc[e] += __shfl_xor_sync(kFull, acc[e], off);
  }
  const bool rep = (TPR >= 32) || (lane < TPR);
  for (int i = tid; i < E; i += kThreads) red[i] = 0.0;
  __syncthreads();
#pragma unroll 1
  for (int w = 0; w < kThreads / 32; ++w) {
    if (warp == w && rep) {
#pragma unroll
      for (int e = 0; e < NACC; ++e) red[pos * NACC + e] += acc[e];
    }
    __syncthreads();
  }
  double* mine = partials + (size_t)blockIdx.x * E;
  for (int i = tid; i < E; i += kThreads) mine[i] = red[i];
  __threadfence();
  __syncthreads();
  __shared__ int s_flag;
  const int nblk = gridDim.x;
  // groups of >= 16 CTAs, at most kMaxTicketGroups groups
  group = max(16, (nblk + kMaxTicketGroups - 1) / kMaxTicketGroups);
  const int ngroups = (nblk + group - 1) / group;
  const int g = blockIdx.x / group;
  if (tid == 0) {
    const int gsize = min(group, nblk - g * group);
    const uint32_t t = atomicAdd(&tickets[g], 1u);
    s_flag = (t == (uint32_t)(gsize - 1));
  }
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  const int c0 = g * group, c1 = min(c0 + group, nblk);
  for (int i = tid; i < E; i += kThreads) {
    double s = 0.0;
    for (int c = c0; c < c1; ++c) s += __ldcg(partials + (size_t)c * E + i);
    gpart[(size_t)g * E + i] = s;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    tickets[g] = 0;
    const uint32_t t = atomicAdd(&tickets[kMaxTicketGroups], 1u);
    s_flag = (t == (uint32_t)(ngroups - 1));
  }
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  for (int i = tid; i < E; i += kThreads) {
    double s = 0.0;
    for (int gg = 0; gg < ngroups; ++gg) s += __ldcg(gpart + (size_t)gg * E + i);
    red[i] = s;
  }
  if (tid == 0) tickets[kMaxTicketGroups] = 0;
  __syncthreads();
  return true;
}

// Gather the grid totals of a Gram accumulator (layout acc[(a*CPT)+j] at
// offset `off` inside each pos's NACC slice) into row-major p x p blocks.
template <int K, int P, int CPT, bool GLOBAL, int NACC>
__device__ void gather_gram(const double* red, int off, double* blocks) {
  using L = Layout<K, P, CPT>;
  constexpr int NB = GLOBAL ? 1 : L::Q;
  for (int idx = threadIdx.x; idx < NB * P * P; idx += kThreads) {
    const int blk = idx / (P * P), a = (idx / P) % P, b = idx % P;
    double s = 0.0;
    const int g0 = GLOBAL ? 0 : blk, g1 = GLOBAL ? L::Q : blk + 1;
    for (int g = g0; g < g1; ++g) {
      const int babs = g * P + b;
      const int pos = babs / CPT, j = babs % CPT;
      s += red[pos * NACC + off + a * CPT + j];
    }
    blocks[idx] = s;
  }
}

struct IterArgs {
  int64_t n;
  const int64_t* rowptr;
  const int32_t* cols;
  const double* vals;
  double* X;
  double* R;
  double* P;
  double* Q;
  double* partials;
  double* gpart;
  double* coef;  // [0,cs) lambda, [cs,2cs) rho_prev, [2cs,3cs) beta, [3cs,4cs) rho
  const double* limits;
  double* hist;  // ring of hist_ring rows x K
  int hist_ring;
  int group;
  Ctrl* ctrl;
};

// Last-CTA epilogue shared by both numerics modes: norms[k] are the column
// norms of R^i (already square-rooted).  Records history, runs all_below
// (solver.hpp:81-85, NaN => not converged) and the max_iter cap.
__device__ inline void finish_iteration(Ctrl* ctrl, const double* norms, const double* limits,
                                        double* hist, int ring, int k) {
  bool ok = true;
  const uint64_t it = ctrl->iterations + 1;
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    const double v = norms[c];
    if (!(v <= limits[c])) ok = false;
    if (hist) hist[(size_t)(it % ring) * k + c] = v;
  }
  const int all_ok = __syncthreads_and(ok);
  if (threadIdx.x == 0) {
    ctrl->iterations = it;
    if (all_ok) ctrl->converged = 1;
    if (all_ok || it >= ctrl->max_iter) ctrl->done = 1;
  }
}

__device__ inline void record_breakdown(Ctrl* ctrl, int bad, int stage) {
  if (threadIdx.x == 0) {
    ctrl->breakdown = 1;
    ctrl->breakdown_iteration = ctrl->iterations + 1;
    ctrl->breakdown_block = (uint64_t)bad;
    ctrl->stage = stage;
    ctrl->done = 1;
  }
}

template <int K, int P, int CPT, bool GLOBAL>
struct FastSmem {
  static constexpr int NB = GLOBAL ? 1 : K / P;
  static constexpr int CS = NB * P * P;
  static constexpr int RED1 = 2 * K * P;         // K1: TPR * 2*P*CPT
  static constexpr int RED2 = K * P + K;         // K2: TPR * (P*CPT + CPT)
  static constexpr int RED = RED1 > RED2 ? RED1 : RED2;
  static int bytes() {
    return (int)sizeof(double) * (RED + 2 * CS + CS + bsolve_ws_doubles(P, kThreads) + K);
  }
};

// ---------------------------------------------------------------- K1 ----
template <int K, int P, int CPT, bool GLOBAL>
__global__ void __launch_bounds__(kThreads) k1_spmm_gram(IterArgs a) {
  using L = Layout<K, P, CPT>;
  using S = FastSmem<K, P, CPT, GLOBAL>;
  if (stopped(a.ctrl)) return;
  constexpr int NACC = 2 * P * CPT;
  double acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.0;
  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT;
  const int gbase = (lane / L::GT) * L::GT;
  const int64_t stride = (int64_t)gridDim.x * L::RPC;
  for (int64_t base = (int64_t)blockIdx.x * L::RPC; base < a.n; base += stride) {
    const int64_t row = base + slot;
    double q[CPT], pv[CPT], rv[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) q[j] = pv[j] = rv[j] = 0.0;
    if (row < a.n) {
      const int64_t beg = __ldg(a.rowptr + row), end = __ldg(a.rowptr + row + 1);
      int64_t i = beg;
      for (; i + 4 <= end; i += 4) {
        double v[4], x[4][CPT];
        int c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u] = __ldg(a.vals + i + u);
          c[u] = __ldg(a.cols + i + u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) ld_nc<CPT>(x[u], a.P + (int64_t)c[u] * K + col0);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < CPT; ++j) q[j] = fma(v[u], x[u][j], q[j]);
      }
      for (; i < end; ++i) {
        const double v = __ldg(a.vals + i);
        const int c = __ldg(a.cols + i);
        double x[CPT];
        ld_nc<CPT>(x, a.P + (int64_t)c * K + col0);
#pragma unroll
        for (int j = 0; j < CPT; ++j) q[j] = fma(v, x[j], q[j]);
      }
      ld_nc<CPT>(pv, a.P + row * K + col0);
      ld_nc<CPT>(rv, a.R + row * K + col0);
      st<CPT>(a.Q + row * K + col0, q);
    }
#pragma unroll
    for (int s = 0; s < L::GT; ++s) {
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) {
        const double ps = __shfl_sync(kFull, pv[jj], gbase + s);
        const int aa = s * CPT + jj;
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
          acc[aa * CPT + j] = fma(ps, q[j], acc[aa * CPT + j]);
          acc[P * CPT + aa * CPT + j] = fma(ps, rv[j], acc[P * CPT + aa * CPT + j]);
        }
      }
    }
  }
  extern __shared__ double sm[];
  double* red = sm;
  if (!grid_reduce<L::TPR, NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  double* alpha = sm + S::RED;
  double* rho_prev = alpha + S::CS;
  double* ws = rho_prev + S::CS + S::CS;
  gather_gram<K, P, CPT, GLOBAL, NACC>(red, 0, alpha);
  gather_gram<K, P, CPT, GLOBAL, NACC>(red, P * CPT, rho_prev);
  __syncthreads();
  for (int i = threadIdx.x; i < S::CS; i += kThreads) a.coef[S::CS + i] = rho_prev[i];
  const int bad = cta_bsolve<P>(S::NB, P, alpha, rho_prev, a.coef, ws);  // lambda
  if (bad >= 0) record_breakdown(a.ctrl, bad, 1);
}

// ---------------------------------------------------------------- K2 ----
template <int K, int P, int CPT, bool GLOBAL>
__global__ void __launch_bounds__(kThreads) k2_update_gram(IterArgs a) {
  using L = Layout<K, P, CPT>;
  using S = FastSmem<K, P, CPT, GLOBAL>;
  if (stopped(a.ctrl)) return;
  extern __shared__ double sm[];
  double* lam = sm + S::RED;
  for (int i = threadIdx.x; i < S::CS; i += kThreads) lam[i] = a.coef[i];
  __syncthreads();
  constexpr int NACC = P * CPT + CPT;
  double acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.0;
  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT;
  const int gbase = (lane / L::GT) * L::GT;
  const int grp = col0 / P;
  const double* lg = lam + (GLOBAL ? 0 : grp) * P * P;
  const int64_t stride = (int64_t)gridDim.x * L::RPC;
  for (int64_t base = (int64_t)blockIdx.x * L::RPC; base < a.n; base += stride) {
    const int64_t row = base + slot;
    const bool valid = row < a.n;
    double pv[CPT], qv[CPT], xv[CPT], rv[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) pv[j] = qv[j] = xv[j] = rv[j] = 0.0;
    if (valid) {
      ld_nc<CPT>(pv, a.P + row * K + col0);
      ld_nc<CPT>(qv, a.Q + row * K + col0);
      ld_rw<CPT>(xv, a.X + row * K + col0);
      ld_rw<CPT>(rv, a.R + row * K + col0);
    }
#pragma unroll
    for (int s = 0; s < L::GT; ++s) {
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) {
        const double ps = __shfl_sync(kFull, pv[jj], gbase + s);
        const double qs = __shfl_sync(kFull, qv[jj], gbase + s);
        const int b = s * CPT + jj;
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
          const double l = lg[b * P + (col0 + j) % P];
          xv[j] = fma(ps, l, xv[j]);
          rv[j] = fma(-qs, l, rv[j]);
        }
      }
    }
    if (valid) {
      st<CPT>(a.X + row * K + col0, xv);
      st<CPT>(a.R + row * K + col0, rv);
    }
#pragma unroll
    for (int s = 0; s < L::GT; ++s) {
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) {
        const double rs = __shfl_sync(kFull, rv[jj], gbase + s);
        const int aa = s * CPT + jj;
#pragma unroll
        for (int j = 0; j < CPT; ++j) acc[aa * CPT + j] = fma(rs, rv[j], acc[aa * CPT + j]);
      }
    }
#pragma unroll
    for (int j = 0; j < CPT; ++j) acc[P * CPT + j] = fma(rv[j], rv[j], acc[P * CPT + j]);
  }
  double* red = sm;
  if (!grid_reduce<L::TPR, NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  double* rho = lam;  // lambda no longer needed
  double* norms = rho + S::CS;
  double* beta_s = norms + K;
  double* ws = beta_s + S::CS;
  gather_gram<K, P, CPT, GLOBAL, NACC>(red, 0, rho);
  for (int c = threadIdx.x; c < K; c += kThreads)
    norms[c] = sqrt(red[(c / CPT) * NACC + P * CPT + (c % CPT)]);
  __syncthreads();
  const int bad = cta_bsolve<P>(S::NB, P, a.coef + S::CS, rho, beta_s, ws);  // beta
  if (bad >= 0) {
    record_breakdown(a.ctrl, bad, 2);
    return;
  }
  for (int i = threadIdx.x; i < S::CS; i += kThreads) {
    a.coef[2 * S::CS + i] = beta_s[i];
    a.coef[3 * S::CS + i] = rho[i];
  }
  finish_iteration(a.ctrl, norms, a.limits, a.hist, a.hist_ring, K);
}

// ---------------------------------------------------------------- K3 ----
template <int K, int P, int CPT, bool GLOBAL>
__global__ void __launch_bounds__(kThreads) k3_update_p(IterArgs a) {
  using L = Layout<K, P, CPT>;
  using S = FastSmem<K, P, CPT, GLOBAL>;
  if (stopped(a.ctrl)) return;
  __shared__ double beta[S::CS];
  for (int i = threadIdx.x; i < S::CS; i += kThreads) beta[i] = a.coef[2 * S::CS + i];
  __syncthreads();
  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT;
  const int gbase = (lane / L::GT) * L::GT;
  const double* bg = beta + (GLOBAL ? 0 : col0 / P) * P * P;
  const int64_t stride = (int64_t)gridDim.x * L::RPC;
  for (int64_t base = (int64_t)blockIdx.x * L::RPC; base < a.n; base += stride) {
    const int64_t row = base + slot;
    const bool valid = row < a.n;
    double pv[CPT], pn[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) pv[j] = pn[j] = 0.0;
    if (valid) {
      ld_rw<CPT>(pv, a.P + row * K + col0);
      ld_nc<CPT>(pn, a.R + row * K + col0);
    }
#pragma unroll
    for (int s = 0; s < L::GT; ++s) {
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) {
        const double ps = __shfl_sync(kFull, pv[jj], gbase + s);
        const int b = s * CPT + jj;
#pragma unroll
        for (int j = 0; j < CPT; ++j) pn[j] = fma(ps, bg[b * P + (col0 + j) % P], pn[j]);
      }
    }
    if (valid) st<CPT>(a.P + row * K + col0, pn);
  }
}

// ------------------------------------------------ standalone fast kernels ----
struct VecArgs {
  int64_t n;
  const int64_t* rowptr;
  const int32_t* cols;
  const double* vals;
  const double* x;
  const double* y;
  double* out;        // Y (spmm) / X (baxpy, in place) / coefficient or norms
  const double* coef; // baxpy gamma
  double* partials;
  double* gpart;
  uint32_t* tickets;
  int group;
};

// Y = A X (kernels.hpp:129-157), FMA, CSR order.
template <int K, int CPT>
__global__ void __launch_bounds__(kThreads) k_spmm_fast(VecArgs a) {
  constexpr int TPR = K / CPT, RPC = kThreads / TPR;
  const int pos = threadIdx.x % TPR, slot = threadIdx.x / TPR, col0 = pos * CPT;
  for (int64_t row = (int64_t)blockIdx.x * RPC + slot; row < a.n; row += (int64_t)gridDim.x * RPC) {
    double q[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) q[j] = 0.0;
    const int64_t end = __ldg(a.rowptr + row + 1);
    for (int64_t i = __ldg(a.rowptr + row); i < end; ++i) {
      const double v = __ldg(a.vals + i);
      double x[CPT];
      ld_nc<CPT>(x, a.x + (int64_t)__ldg(a.cols + i) * K + col0);
#pragma unroll
      for (int j = 0; j < CPT; ++j) q[j] = fma(v, x[j], q[j]);
    }
    st<CPT>(a.out + row * K + col0, q);
  }
}

// BDOT (kernels.hpp:59-88) with deterministic grid reduction; the last CTA
// writes the block coefficient to a.out.
template <int K, int P, int CPT, bool GLOBAL>
__global__ void __launch_bounds__(kThreads) k_gram_fast(VecArgs a) {
  using L = Layout<K, P, CPT>;
  constexpr int NACC = P * CPT;
  double acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.0;
  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT, gbase = (lane / L::GT) * L::GT;
  for (int64_t base = (int64_t)blockIdx.x * L::RPC; base < a.n; base += (int64_t)gridDim.x * L::RPC) {
    const int64_t row = base + slot;
    double xv[CPT], yv[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) xv[j] = yv[j] = 0.0;
    if (row < a.n) {
      ld_nc<CPT>(xv, a.x + row * K + col0);
      ld_nc<CPT>(yv, a.y + row * K + col0);
    }
#pragma unroll
    for (int s = 0; s < L::GT; ++s)
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) {
        const double xs = __shfl_sync(kFull, xv[jj], gbase + s);
#pragma unroll
        for (int j = 0; j < CPT; ++j)
          acc[(s * CPT + jj) * CPT + j] = fma(xs, yv[j], acc[(s * CPT + jj) * CPT + j]);
      }
  }
  extern __shared__ double sm[];
  if (!grid_reduce<L::TPR, NACC>(acc, sm, a.partials, a.gpart, a.tickets, a.group)) return;
  gather_gram<K, P, CPT, GLOBAL, NACC>(sm, 0, a.out);
}

// Column norms (block_vector.hpp:59-70), deterministic grid reduction.
template <int K, int CPT>
__global__ void __launch_bounds__(kThreads) k_norms_fast(VecArgs a) {
  constexpr int TPR = K / CPT, RPC = kThreads / TPR;
  double acc[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) acc[j] = 0.0;
  const int pos = threadIdx.x % TPR, slot = threadIdx.x / TPR, col0 = pos * CPT;
  for (int64_t row = (int64_t)blockIdx.x * RPC + slot; row < a.n; row += (int64_t)gridDim.x * RPC) {
    double xv[CPT];
    ld_nc<CPT>(xv, a.x + row * K + col0);
#pragma unroll
    for (int j = 0; j < CPT; ++j) acc[j] = fma(xv[j], xv[j], acc[j]);
  }
  extern __shared__ double sm[];
  if (!grid_reduce<TPR, CPT>(acc, sm, a.partials, a.gpart, a.tickets, a.group)) return;
  for (int c = threadIdx.x; c < K; c += kThreads) a.out[c] = sqrt(sm[c]);
}

// BAXPY (kernels.hpp:94-125): X += Y embed(gamma), FMA chain in b order.
template <int K, int P, int CPT, bool GLOBAL>
__global__ void __launch_bounds__(kThreads) k_baxpy_fast(VecArgs a) {
  using L = Layout<K, P, CPT>;
  constexpr int CS = (GLOBAL ? 1 : K / P) * P * P;
  __shared__ double gam[CS];
  for (int i = threadIdx.x; i < CS; i += kThreads) gam[i] = a.coef[i];
  __syncthreads();
  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT, gbase = (lane / L::GT) * L::GT;
  const double* gg = gam + (GLOBAL ? 0 : col0 / P) * P * P;
  for (int64_t base = (int64_t)blockIdx.x * L::RPC; base < a.n; base += (int64_t)gridDim.x * L::RPC) {
    const int64_t row = base + slot;
    const bool valid = row < a.n;
    double yv[CPT], xv[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) yv[j] = xv[j] = 0.0;
    if (valid) {
      ld_nc<CPT>(yv, a.y + row * K + col0);
      ld_rw<CPT>(xv, a.out + row * K + col0);
    }
#pragma unroll
    for (int s = 0; s < L::GT; ++s)
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) {
        const double ys = __shfl_sync(kFull, yv[jj], gbase + s);
        const int b = s * CPT + jj;
#pragma unroll
        for (int j = 0; j < CPT; ++j) xv[j] = fma(ys, gg[b * P + (col0 + j) % P], xv[j]);
      }
    if (valid) st<CPT>(a.out + row * K + col0, xv);
  }
}

}  // namespace bkg
