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
// to arrive); there red[pos*NACC + e] holds the grid totals.  NTHR = threads
// per CTA (k1_stage runs 16 warps).
template <int TPR, int NACC, int NTHR = kThreads>
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
  for (int i = tid; i < E; i += NTHR) red[i] = 0.0;
  __syncthreads();
#pragma unroll 1
  for (int w = 0; w < NTHR / 32; ++w) {
    if (warp == w && rep) {
#pragma unroll
      for (int e = 0; e < NACC; ++e) red[pos * NACC + e] += acc[e];
    }
    __syncthreads();
  }
  double* mine = partials + (size_t)blockIdx.x * E;
  for (int i = tid; i < E; i += NTHR) mine[i] = red[i];
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
  for (int i = tid; i < E; i += NTHR) {
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
  for (int i = tid; i < E; i += NTHR) {
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
  // Row-partitioned solver (psolver.cu): the last CTA only publishes this
  // part's totals -- red1 = [alpha | rho_prev], red2 = [rho | ||R_s||^2] --
  // and the p x p solves run after the cross-part allreduce.
  int dist;
  double* red1;
  double* red2;
  // Jacobi in the fused loop: Z = zscale (.) R row-wise (zscale = D^-1,
  // preconditioners.hpp:109-129); nullptr for M = I.
  const double* zscale;
  // ILU(0) in the fused loop: Z = M^-1 R from the sync-free sweeps (K3's
  // P' = Z + P beta source); nullptr otherwise.
  const double* zsrc;
  // Sliced-ELL copy of the CSR (k1_wide; slice height = its tile rows)
  const int64_t* sptr;
  const int32_t* scols;
  const double* svals;
  const double* stri;  // line variant (k1_line): tri-diagonal entries per slice row
  // Deferred X update (K3 template XM): K3 writes P' to Pn; in a flush
  // launch X += Pold lambda_old + P lambda (lambda_old at coef + 4 cs).
  double* Pn;
  const double* Pold;
  // k1_stage (kernels_stage.cuh): the staged-block copy (common.cuh
  // StageCsr), the ring depth, and the blocks of this launch -- all stg_cnt
  // blocks in order, or stg_map[0 .. stg_cnt) (the partitioned solver
  // launches interior and boundary blocks separately).
  const StageHdr* stg_hdr;
  const int2* stg_segs;
  const double* stg_vals;
  const uint16_t* stg_lidx;
  const int32_t* stg_rowid;
  int stg_nstage, stg_cap, stg_wmax, stg_smax, stg_R;
  int stg_debug;  // tuning only (BKG_STAGE_DEBUG): 1 skip the tile compute, 2 skip the row copies
  int64_t stg_cnt;
  const int64_t* stg_map;  // non-null: block j of the launch is stg_map[j]
  // dist: add this launch's alpha to red1 instead of overwriting it
  int dist_acc;
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
  // largest TPR * NACC over the scalar K1..K3 and the DMMA K2/K3 (P >= 8)
  static constexpr int RED_SCALAR = K * P + K;
  static constexpr int PE = P < 8 ? 8 : P;  // DMMA group width (kernels_mma.cuh MmaLayout)
  static constexpr int RED_MMA =
      (K % 8 == 0) ? 32 * (K / PE) * (2 * (PE / 8) * (PE / 8) + 2 * (PE / 8)) : 0;
  // K1 warp-tile kernel (kernels_mma.cuh k1_tile): 32*QW positions x 2*NPAIR
  static constexpr int W1 = K >= 16 ? 16 : 8;
  static constexpr int RED_K1 =
      (K % 8 == 0) ? 32 * (K / W1) * 2 * ((P >= 8) ? (W1 / 8) * (P / 8) : (W1 / 8)) : 0;
  static constexpr int RED_A = RED_SCALAR > RED_MMA ? RED_SCALAR : RED_MMA;
  static constexpr int RED = RED_A > RED_K1 ? RED_A : RED_K1;
  static int bytes() {
    return (int)sizeof(double) * (RED + 3 * CS + bsolve_ws_doubles(P, kThreads) + K);
  }
};

// Minimum resident CTAs per SM for the row-streaming kernels: 4 caps
// registers at 64/thread so enough rows are in flight to cover DRAM latency;
// kernels carrying a p x p Gram tile of >= 16 doubles per thread get 85.
#ifndef BKG_MINB_BIG
#define BKG_MINB_BIG 3
#endif
#ifndef BKG_MINB_SMALL
#define BKG_MINB_SMALL 4
#endif
template <int P, int CPT>
constexpr int min_blocks() {
  return P * CPT >= 16 ? BKG_MINB_BIG : BKG_MINB_SMALL;
}

// One CSR row of Q = A P for the CPT lanes of this thread, in CSR order.
// Chunks of 8 nonzeros are loaded with predication so that every index and
// operand load of a stencil row is in flight at once (no serial tail loop).
template <int K, int CPT>
__device__ __forceinline__ void spmm_row(const IterArgs& a, int64_t beg, int64_t end, int col0,
                                         double (&q)[CPT]) {
  constexpr int CH = 8;
#pragma unroll 1
  for (int64_t i = beg; i < end; i += CH) {
    double v[CH], x[CH][CPT];
    int c[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const bool on = i + u < end;
      v[u] = on ? __ldg(a.vals + i + u) : 0.0;
      c[u] = on ? __ldg(a.cols + i + u) : kNoCol;
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if (c[u] != kNoCol) {
        ld_nc<CPT>(x[u], a.P + (int64_t)c[u] * K + col0);
      } else {
#pragma unroll
        for (int j = 0; j < CPT; ++j) x[u][j] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u)
      if (c[u] != kNoCol) {
#pragma unroll
        for (int j = 0; j < CPT; ++j) q[j] = fma(v[u], x[u][j], q[j]);
      }
  }
}

// Rows interleaved per thread in the streaming kernels (bytes in flight) and
// how K2/K3 read the p x p coefficients: `const double*` lets the compiler
// keep them in registers, `const volatile double*` re-reads shared memory per
// row.  Defaults from the tools/kernel_sweep.py measurements on B200 (C2):
// K2 2 rows/thread + register coefficients (0.34 ms, 73% of HBM peak); K3 one
// row/thread (two spill).
#ifndef BKG_K2_ROWS
#define BKG_K2_ROWS 2
#endif
#ifndef BKG_K3_ROWS
#define BKG_K3_ROWS 1
#endif
#ifndef BKG_K2_COEF_PTR
#define BKG_K2_COEF_PTR const double*
#endif
#ifndef BKG_K3_COEF_PTR
#define BKG_K3_COEF_PTR const double*
#endif

// ---------------------------------------------------------------- K1 ----
// Q = A P; alpha = <<P, Q>>; last CTA: lambda = alpha^-1 rho_prev.
// rho_prev = <<P^i, R^{i-1}>> (solver.hpp:168) was produced by K3 of the
// previous iteration (R is not modified between that K3 and this K1), so K1
// does not read R at all.
template <int K, int P, int CPT, bool GLOBAL>
__global__ void __launch_bounds__(kThreads, (min_blocks<P, CPT>())) k1_spmm_gram(IterArgs a) {
  using L = Layout<K, P, CPT>;
  using S = FastSmem<K, P, CPT, GLOBAL>;
  if (stopped(a.ctrl)) return;
  constexpr int NACC = P * CPT;
  static_assert(L::TPR * NACC <= S::RED, "grid_reduce buffer");
  double acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.0;
  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT;
  const int gbase = (lane / L::GT) * L::GT;
  const int64_t stride = (int64_t)gridDim.x * L::RPC;
  int64_t row = (int64_t)blockIdx.x * L::RPC + slot;
  int64_t beg = 0, end = 0;
  if (row < a.n) {
    beg = __ldg(a.rowptr + row);
    end = __ldg(a.rowptr + row + 1);
  }
  for (int64_t base = (int64_t)blockIdx.x * L::RPC; base < a.n; base += stride) {
    // prefetch the next row's extent while this row's loads are in flight
    const int64_t nrow = row + stride;
    int64_t nbeg = 0, nend = 0;
    if (nrow < a.n) {
      nbeg = __ldg(a.rowptr + nrow);
      nend = __ldg(a.rowptr + nrow + 1);
    }
    double q[CPT], pv[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) q[j] = pv[j] = 0.0;
    if (row < a.n) {
      ld_nc<CPT>(pv, a.P + row * K + col0);
      spmm_row<K, CPT>(a, beg, end, col0, q);
      st<CPT>(a.Q + row * K + col0, q);
    }
#pragma unroll
    for (int s = 0; s < L::GT; ++s) {
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) {
        const double ps = __shfl_sync(kFull, pv[jj], gbase + s);
        const int aa = s * CPT + jj;
#pragma unroll
        for (int j = 0; j < CPT; ++j) acc[aa * CPT + j] = fma(ps, q[j], acc[aa * CPT + j]);
      }
    }
    row = nrow;
    beg = nbeg;
    end = nend;
  }
  extern __shared__ double sm[];
  double* red = sm;
  if (!grid_reduce<L::TPR, NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  double* alpha = sm + S::RED;
  double* ws = alpha + 3 * S::CS;
  gather_gram<K, P, CPT, GLOBAL, NACC>(red, 0, alpha);
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.red1[i] = alpha[i];
    return;
  }
  const int bad = fast_bsolve<P>(S::NB, P, alpha, a.coef + S::CS, a.coef, ws);  // lambda
  if (bad >= 0) record_breakdown(a.ctrl, bad, 1);
}

// ---------------------------------------------------------------- K2 ----
// R -= Q lambda; rho = <<Z, R>> (Z = M^-1 R: R, or D^-1 R for Jacobi) and
// ||R_s||^2; last CTA:
// beta = rho_prev^-1 rho, history, stop test.  X += P lambda is deferred to
// K3, which reads P anyway (nothing reads X before K3).
template <int K, int P, int CPT, bool GLOBAL, bool JAC = false>
__global__ void __launch_bounds__(kThreads, (min_blocks<P, CPT>())) k2_update_gram(IterArgs a) {
  using L = Layout<K, P, CPT>;
  using S = FastSmem<K, P, CPT, GLOBAL>;
  constexpr int U = BKG_K2_ROWS;
  if (stopped(a.ctrl)) return;
  extern __shared__ double sm[];
  double* lam = sm + S::RED;
  for (int i = threadIdx.x; i < S::CS; i += kThreads) lam[i] = a.coef[i];
  __syncthreads();
  constexpr int NACC = P * CPT + CPT;
  static_assert(L::TPR * NACC <= S::RED, "grid_reduce buffer");
  double acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.0;
  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT;
  const int gbase = (lane / L::GT) * L::GT;
  BKG_K2_COEF_PTR lg = lam + (GLOBAL ? 0 : col0 / P) * P * P;
  const int64_t r1 = a.n;
  for (int64_t base = (int64_t)blockIdx.x * L::RPC * U; base < r1;
       base += (int64_t)gridDim.x * L::RPC * U) {
    double qv[U][CPT], rv[U][CPT], dz[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = base + u * L::RPC + slot;
#pragma unroll
      for (int j = 0; j < CPT; ++j) qv[u][j] = rv[u][j] = 0.0;
      dz[u] = 1.0;
      if (row < r1) {
        ld_nc<CPT>(qv[u], a.Q + row * K + col0);
        ld_rw<CPT>(rv[u], a.R + row * K + col0);
        if constexpr (JAC) dz[u] = __ldg(a.zscale + row);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int s = 0; s < L::GT; ++s) {
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj) {
          const double qs = __shfl_sync(kFull, qv[u][jj], gbase + s);
          const int b = s * CPT + jj;
#pragma unroll
          for (int j = 0; j < CPT; ++j)
            rv[u][j] = fma(-qs, lg[b * P + (col0 + j) % P], rv[u][j]);
        }
      }
      const int64_t row = base + u * L::RPC + slot;
      if (row < r1) st<CPT>(a.R + row * K + col0, rv[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int s = 0; s < L::GT; ++s) {
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj) {
          // rho = <<Z, R>>: Z = D^-1 R for Jacobi, R for M = I
          double zs = __shfl_sync(kFull, rv[u][jj], gbase + s);
          if constexpr (JAC) zs *= dz[u];
          const int aa = s * CPT + jj;
#pragma unroll
          for (int j = 0; j < CPT; ++j) acc[aa * CPT + j] = fma(zs, rv[u][j], acc[aa * CPT + j]);
        }
      }
#pragma unroll
      for (int j = 0; j < CPT; ++j) acc[P * CPT + j] = fma(rv[u][j], rv[u][j], acc[P * CPT + j]);
    }
  }
  double* red = sm;
  if (!grid_reduce<L::TPR, NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  double* rho = lam;  // lambda no longer needed in smem
  double* beta_s = rho + S::CS;
  double* norms = beta_s + S::CS;
  double* ws = sm + S::RED + 3 * S::CS + K;
  gather_gram<K, P, CPT, GLOBAL, NACC>(red, 0, rho);
  for (int c = threadIdx.x; c < K; c += kThreads) {
    const double ss = red[(c / CPT) * NACC + P * CPT + (c % CPT)];
    norms[c] = a.dist ? ss : sqrt(ss);
  }
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.red2[i] = rho[i];
    for (int c = threadIdx.x; c < K; c += kThreads) a.red2[S::CS + c] = norms[c];
    return;
  }
  const int bad = fast_bsolve<P>(S::NB, P, a.coef + S::CS, rho, beta_s, ws);  // beta
  if (threadIdx.x == 0) a.ctrl->xpending = 1;  // K3 still owes X += P lambda
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
// X += P lambda (always, once K2 ran: solver.hpp:171-175 precede the beta
// solve and the stop test); unless the solve stopped: P = Z + P beta in
// place (solver.hpp:186-190) and rho_prev' = <<P', R>> for the next K1.
template <int K, int P, int CPT, bool GLOBAL, bool JAC = false, bool ZS = false, int XM = 0>
__device__ __forceinline__ void k3_update_xp_body(const IterArgs& a) {
  using L = Layout<K, P, CPT>;
  using S = FastSmem<K, P, CPT, GLOBAL>;
  // XM: deferred X update, see kernels_mma.cuh k3_mma; the skip launch
  // streams only P and R, so it takes two rows per thread step where the
  // per-row coefficient work is small (P * CPT <= 2; measured on B200)
  constexpr int U = (XM == 1 && P * CPT <= 2) ? 2 : BKG_K3_ROWS;
  const bool cur = *reinterpret_cast<const volatile int32_t*>(&a.ctrl->xpending) != 0;
  const bool old = XM == 2 && *reinterpret_cast<const volatile int32_t*>(&a.ctrl->xold) != 0;
  if (!cur && !old) return;
  const bool fin = stopped(a.ctrl);  // uniform: nothing writes `done` during K3
  const bool upd = cur && !fin;
  const bool dox = XM != 1 || fin;
  extern __shared__ double sm[];
  double* lam = sm + S::RED;
  double* beta = lam + S::CS;
  double* lamo = beta + S::CS;  // FastSmem reserves 3 coefficient blocks past RED
  for (int i = threadIdx.x; i < S::CS; i += kThreads) {
    lam[i] = a.coef[i];
    beta[i] = a.coef[2 * S::CS + i];
    if (XM == 2) lamo[i] = a.coef[4 * S::CS + i];
  }
  __syncthreads();
  constexpr int NACC = P * CPT;
  static_assert(L::TPR * NACC <= S::RED, "grid_reduce buffer");
  double acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.0;
  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT;
  const int gbase = (lane / L::GT) * L::GT;
  const int goff = (GLOBAL ? 0 : col0 / P) * P * P;
  BKG_K3_COEF_PTR lg = lam + goff;
  BKG_K3_COEF_PTR bg = beta + goff;
  BKG_K3_COEF_PTR og = lamo + goff;
  double* Pout = XM == 0 ? a.P : a.Pn;
  const int64_t r1 = a.n;
  for (int64_t base = (int64_t)blockIdx.x * L::RPC * U; base < r1;
       base += (int64_t)gridDim.x * L::RPC * U) {
    double pv[U][CPT], ov[U][CPT], xv[U][CPT], rv[U][CPT], zv[U][CPT], dz[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = base + u * L::RPC + slot;
#pragma unroll
      for (int j = 0; j < CPT; ++j) pv[u][j] = ov[u][j] = xv[u][j] = rv[u][j] = zv[u][j] = 0.0;
      dz[u] = 1.0;
      if (row < r1) {
        if (cur) ld_rw<CPT>(pv[u], a.P + row * K + col0);
        if constexpr (XM == 2)
          if (old) ld_nc<CPT>(ov[u], a.Pold + row * K + col0);
        if (dox) ld_rw<CPT>(xv[u], a.X + row * K + col0);
        if (upd) ld_nc<CPT>(rv[u], a.R + row * K + col0);
        if constexpr (ZS)
          if (upd) ld_nc<CPT>(zv[u], a.zsrc + row * K + col0);
        if constexpr (JAC)
          if (upd) dz[u] = __ldg(a.zscale + row);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double pn[CPT];  // Z = M^-1 R: D^-1 R (Jacobi), the ILU sweeps' Z, or R
#pragma unroll
      for (int j = 0; j < CPT; ++j) pn[j] = ZS ? zv[u][j] : (JAC ? rv[u][j] * dz[u] : rv[u][j]);
#pragma unroll
      for (int s = 0; s < L::GT; ++s) {
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj) {
          const double ps = __shfl_sync(kFull, pv[u][jj], gbase + s);
          double os = 0.0;
          if constexpr (XM == 2) os = __shfl_sync(kFull, ov[u][jj], gbase + s);
          const int b = s * CPT + jj;
#pragma unroll
          for (int j = 0; j < CPT; ++j) {
            const int e = b * P + (col0 + j) % P;
            if constexpr (XM == 2)
              if (old) xv[u][j] = fma(os, og[e], xv[u][j]);
            // after a lambda breakdown (cur = 0) lg / bg hold stale values
            // (an Inf there must not reach X): skip, as k3_mma does
            if (cur) {
              xv[u][j] = fma(ps, lg[e], xv[u][j]);
              pn[j] = fma(ps, bg[e], pn[j]);
            }
          }
        }
      }
      const int64_t row = base + u * L::RPC + slot;
      if (row < r1) {
        if (dox) st<CPT>(a.X + row * K + col0, xv[u]);
        if (upd) st<CPT>(Pout + row * K + col0, pn);
      }
      if (upd) {
#pragma unroll
        for (int s = 0; s < L::GT; ++s) {
#pragma unroll
          for (int jj = 0; jj < CPT; ++jj) {
            const double ps = __shfl_sync(kFull, pn[jj], gbase + s);
            const int aa = s * CPT + jj;
#pragma unroll
            for (int j = 0; j < CPT; ++j)
              acc[aa * CPT + j] = fma(ps, rv[u][j], acc[aa * CPT + j]);
          }
        }
      }
    }
  }
  double* red = sm;
  if (!grid_reduce<L::TPR, NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  if (upd) gather_gram<K, P, CPT, GLOBAL, NACC>(red, 0, (a.dist ? a.red1 : a.coef) + S::CS);
  if (XM == 1 && upd)
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.coef[4 * S::CS + i] = a.coef[i];
  __syncthreads();
  if (threadIdx.x == 0) {  // every CTA has read the flags (we are last)
    if (XM == 1) a.ctrl->xold = upd ? 1 : 0;
    if (XM == 2) a.ctrl->xold = 0;
    a.ctrl->xpending = 0;
  }
}
template <int K, int P, int CPT, bool GLOBAL, bool JAC = false, bool ZS = false, int XM = 0>
__global__ void __launch_bounds__(kThreads, (min_blocks<P, CPT>())) k3_update_xp(IterArgs a) {
  k3_update_xp_body<K, P, CPT, GLOBAL, JAC, ZS, XM>(a);
}

// ------------------------------------------------------- K2 (ILU(0)) ---
// ILU(0) in the fused loop, first half of K2: R -= Q lambda and ||R_s||^2.
// The Gram rho = <<Z, R>> needs Z = M^-1 R of the whole new R, so it runs
// after the sync-free sweeps (k_gram_fast), then k_ilu_finish (beta, history,
// stop test).  The last CTA writes the column sums of squares to a.red2.
template <int K, int P, int CPT, bool GLOBAL>
__global__ void __launch_bounds__(kThreads, (min_blocks<P, CPT>())) k2_ilu(IterArgs a) {
  using L = Layout<K, P, CPT>;
  using S = FastSmem<K, P, CPT, GLOBAL>;
  if (stopped(a.ctrl)) return;
  extern __shared__ double sm[];
  double* lam = sm + S::RED;
  for (int i = threadIdx.x; i < S::CS; i += kThreads) lam[i] = a.coef[i];
  __syncthreads();
  double acc[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) acc[j] = 0.0;
  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT;
  const int gbase = (lane / L::GT) * L::GT;
  const double* lg = lam + (GLOBAL ? 0 : col0 / P) * P * P;
  for (int64_t row = (int64_t)blockIdx.x * L::RPC + slot; row - slot < a.n;
       row += (int64_t)gridDim.x * L::RPC) {
    const bool ok = row < a.n;
    double qv[CPT], rv[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) qv[j] = rv[j] = 0.0;
    if (ok) {
      ld_nc<CPT>(qv, a.Q + row * K + col0);
      ld_rw<CPT>(rv, a.R + row * K + col0);
    }
#pragma unroll
    for (int s = 0; s < L::GT; ++s)
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) {
        const double qs = __shfl_sync(kFull, qv[jj], gbase + s);
        const int b = s * CPT + jj;
#pragma unroll
        for (int j = 0; j < CPT; ++j) rv[j] = fma(-qs, lg[b * P + (col0 + j) % P], rv[j]);
      }
    if (ok) st<CPT>(a.R + row * K + col0, rv);
#pragma unroll
    for (int j = 0; j < CPT; ++j) acc[j] = fma(rv[j], rv[j], acc[j]);
  }
  if (!grid_reduce<L::TPR, CPT>(acc, sm, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  for (int c = threadIdx.x; c < K; c += kThreads) a.red2[c] = sm[c];
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
  const Ctrl* ctrl;  // solver loop: skip once the device stop flag is set
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
  if (stopped(a.ctrl)) return;
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
