// kernels_mma.cuh — FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) versions of
// the row-streaming Block-CG updates for block widths P in {8, 16}.
//
// For P >= 8 the update X += Y gamma (kernels.hpp:94-125) is a real dense
// contraction (P multiply-adds per element) and the Gram tile
// (kernels.hpp:59-88) is P^2 per row.  With scalar FMAs every thread needs
// the whole p-group of its row (warp shuffles) and P*CPT coefficients in
// registers, which made the scalar K2/K3 shuffle/L1-bound (ncu: L1/TEX 97%).
// Here a warp owns an 8-row x P-column tile of one p-group:
//   * the p x p coefficient block lives in B fragments: P^2/32 doubles/lane;
//   * Y enters as A fragments (8 B per lane per k-chunk, 32 B row segments);
//   * X / R enter and leave in the C/D layout (16 B per lane);
//   * the Gram tile G = U^T V over the 8 rows is two more k=4 MMAs per
//     8x8 output tile after an in-register D->T relayout (2 shuffles).
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64):
//   A (8x4, row): lane holds A[lane>>2][lane&3]
//   B (4x8, col): lane holds B[lane&3][lane>>2]
//   C/D (8x8):    lane holds D[lane>>2][2*(lane&3) + i], i = 0, 1
#pragma once

#include "kernels_fast.cuh"

namespace bkg {

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// D-layout 8x8 tile -> the two T-layout 4x8 chunks (rows 4c..4c+3):
// t[c] = tile[4c + (lane&3)][lane>>2], the A/B operand layout of a Gram
// product over rows.
__device__ __forceinline__ void d_to_t(const double (&d)[2], double (&t)[2], int lane) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int src = 16 * c + 4 * (lane & 3) + (lane >> 3);
    const double v0 = __shfl_sync(kFull, d[0], src);
    const double v1 = __shfl_sync(kFull, d[1], src);
    t[c] = ((lane >> 2) & 1) ? v1 : v0;
  }
}

// A warp works on PE = max(P, 8) columns of a row block ("tile group"): one
// p-group for P >= 8, or 8/P whole p-groups for P < 8, whose coefficient
// blocks then form a block-diagonal 8 x 8 B operand (the zero blocks cost
// DMMA issue slots only, which are idle in these HBM-bound kernels).
template <int K, int P, bool GLOBAL>
struct MmaLayout {
  static constexpr int PE = P < 8 ? 8 : P;
  static constexpr int Q = K / PE;    // tile groups per row
  static constexpr int NT = PE / 8;   // 8-column output tiles per tile group
  static constexpr int KC = PE / 4;   // 4-column k-chunks per tile group
  static constexpr int TPR = 32 * Q;  // grid_reduce positions: (warp % Q, lane)
  static constexpr int NB = GLOBAL ? 1 : K / P;  // coefficient blocks
  static constexpr int CS = NB * P * P;
  static_assert(K % 8 == 0 && P <= 16, "DMMA path: K a multiple of 8, P <= 16");
  static_assert(8 % Q == 0, "the 8 warps of a CTA must cover whole rows of tile groups");
};

// B fragments of tile group g: frag[kc][nt] = sign * B[kc*4 + (lane&3)][nt*8 +
// (lane>>2)] where B is the group's coefficient block (row-major c[b][a],
// kernels.hpp:94-125 right-multiplication) for P >= 8, or the block-diagonal
// embedding of its 8/P blocks for P < 8 (global: block 0 everywhere).
template <int K, int P, bool GLOBAL>
__device__ __forceinline__ void load_bfrag(const double* coef, int g, double sign,
                                           double (&f)[MmaLayout<K, P, GLOBAL>::KC]
                                                      [MmaLayout<K, P, GLOBAL>::NT],
                                           int lane) {
  using L = MmaLayout<K, P, GLOBAL>;
#pragma unroll
  for (int kc = 0; kc < L::KC; ++kc)
#pragma unroll
    for (int nt = 0; nt < L::NT; ++nt) {
      const int b = kc * 4 + (lane & 3), a = nt * 8 + (lane >> 2);
      if constexpr (P >= 8) {
        f[kc][nt] = sign * coef[(GLOBAL ? 0 : g) * P * P + b * P + a];
      } else {
        const int blk = GLOBAL ? 0 : (g * 8 + b) / P;
        f[kc][nt] = (b / P == a / P) ? sign * coef[blk * P * P + (b % P) * P + a % P] : 0.0;
      }
    }
}

// Grid totals of a Gram accumulator in D layout (per (group, lane) position
// of grid_reduce) gathered into row-major p x p blocks.
template <int K, int P, bool GLOBAL, int NACC>
__device__ void gather_gram_mma(const double* red, int off, double* blocks) {
  using L = MmaLayout<K, P, GLOBAL>;
  for (int idx = threadIdx.x; idx < L::NB * P * P; idx += kThreads) {
    const int blk = idx / (P * P), a = (idx / P) % P, b = idx % P;
    double s = 0.0;
    // p-groups summed into this block (global: all of them, in order)
    const int g0 = GLOBAL ? 0 : blk, g1 = GLOBAL ? K / P : blk + 1;
    for (int g = g0; g < g1; ++g) {
      const int tg = g * P / L::PE, o = g * P % L::PE;  // tile group, column offset
      const int ca = o + a, cb = o + b;
      const int lane = ((ca & 7) << 2) | ((cb & 7) >> 1), i = cb & 1;
      const int e = off + ((ca >> 3) * L::NT + (cb >> 3)) * 2 + i;
      s += red[(tg * 32 + lane) * NACC + e];
    }
    blocks[idx] = s;
  }
}

// Column sums of squares held per lane in D layout (entry off + nt*2 + i is
// column nt*8 + 2*(lane&3) + i of the lane's group), summed over the 8 row
// lanes and square-rooted.
template <int K, int P, bool GLOBAL, int NACC>
__device__ void gather_norms_mma(const double* red, int off, double* norms, bool squares) {
  using L = MmaLayout<K, P, GLOBAL>;
  for (int c = threadIdx.x; c < K; c += kThreads) {
    const int g = c / L::PE, cc = c % L::PE, nt = cc >> 3, i = cc & 1, l4 = (cc & 7) >> 1;
    double s = 0.0;
    for (int r = 0; r < 8; ++r) s += red[(g * 32 + (r << 2) + l4) * NACC + off + nt * 2 + i];
    norms[c] = squares ? s : sqrt(s);
  }
}

// ------------------------------------------------------------ K2 (DMMA) --
// R -= Q lambda; rho = <<Z, R>> (Z = D^-1 R for Jacobi, R for M = I);
// ||R_s||^2; last CTA: beta, history, stop.
// Resident CTAs per SM (register cap) for the DMMA K2/K3, measured on B200
// (tools/kernel_sweep.py): P = 8 K3 tiles are small enough for 4 CTAs (64
// regs), the two-block-unrolled P <= 8 K2 runs 3; at P = 16, K2 peaks at 3
// and K3 (two coefficient blocks) at 2.
// K2 with P <= 8 processes two row blocks per warp step (3 CTAs/SM): C2 K2
// 0.281 -> 0.265 ms; at P = 16 the doubled tile costs more than it hides.
#ifndef BKG_K2_U8
#define BKG_K2_U8 2
#endif
#ifndef BKG_K2_MINB8
#define BKG_K2_MINB8 3
#endif
#ifndef BKG_K3_MINB8
#define BKG_K3_MINB8 4
#endif
template <int P>
constexpr int k2_unroll() {
  return P <= 8 ? BKG_K2_U8 : 1;
}
// L2 bulk prefetch distance of K2 / K3 in warp steps (0: off): the warp that
// owns column group 0 of a row block asks the copy engine to pull the whole
// 8-row block (8 K doubles, contiguous) of every operand stream BKG_MMA_PF
// steps ahead into L2 (cp.async.bulk.prefetch.L2: no register, no L1 miss
// slot), so the fragment loads that follow find their lines in L2.
#ifndef BKG_MMA_PF
#define BKG_MMA_PF 0
#endif
__device__ __forceinline__ void mma_prefetch_block(const double* base, int64_t rb, int64_t nrb,
                                                   int64_t n, int K) {
  if (rb < nrb && rb * 8 + 8 <= n)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + rb * 8 * K),
                 "r"((uint32_t)(8 * K * 8))
                 : "memory");
}

// Tuning: the P = 16 skip launch (XM 1: P, R in, P' out -- K2's byte mix) at
// K2's shape, one row block per step and 3 CTAs per SM, instead of two row
// blocks at 2 CTAs per SM.
#ifndef BKG_K3_SKIP3
#define BKG_K3_SKIP3 0
#endif
template <int P, int KERNEL>
constexpr int mma_minb() {
  return P <= 8 ? (KERNEL == 2 ? BKG_K2_MINB8 : BKG_K3_MINB8) : (KERNEL == 2 ? 3 : 2);
}
template <int K, int P, bool GLOBAL, bool JAC = false>
__global__ void __launch_bounds__(kThreads, (mma_minb<P, 2>())) k2_mma(IterArgs a) {
  using L = MmaLayout<K, P, GLOBAL>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  if (stopped(a.ctrl)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp % L::Q;
  double nlam[L::KC][L::NT];
  load_bfrag<K, P, GLOBAL>(a.coef, g, -1.0, nlam, lane);
  constexpr int NG = L::NT * L::NT * 2;  // Gram accumulators
  constexpr int NACC = NG + L::NT * 2;   // + column sums of squares
  static_assert(L::TPR * NACC <= S::RED, "grid_reduce buffer");
  double acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.0;
  const int64_t nrb = (a.n + 7) >> 3;
  const int64_t wstride = (int64_t)gridDim.x * (kThreads / 32) / L::Q;
  const int col_a = g * L::PE + (lane & 3);            // A-fragment column base
  const int col_c = g * L::PE + 2 * (lane & 3);        // C-fragment column base
  // U row blocks per warp step: all their loads are issued before any DMMA
  // (bytes in flight per warp x U; K2 is latency-bound at U = 1)
  constexpr int U = k2_unroll<P>();
  for (int64_t rb0 = ((int64_t)blockIdx.x * (kThreads / 32) + warp) / L::Q; rb0 < nrb;
       rb0 += U * wstride) {
    double qa[U][L::KC], rc[U][L::NT][2], dt[U][2];
    if constexpr (BKG_MMA_PF > 0) {
      if (g == 0 && lane == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t rbp = rb0 + (BKG_MMA_PF * U + u) * wstride;
          mma_prefetch_block(a.Q, rbp, nrb, a.n, K);
          mma_prefetch_block(a.R, rbp, nrb, a.n, K);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t rb = rb0 + u * wstride;
      const int64_t row = rb * 8 + (lane >> 2);
      const bool ok = rb < nrb && row < a.n;
      dt[u][0] = dt[u][1] = 1.0;
#pragma unroll
      for (int kc = 0; kc < L::KC; ++kc)
        qa[u][kc] = ok ? __ldg(a.Q + row * K + col_a + kc * 4) : 0.0;
      if constexpr (JAC) {  // Jacobi scale of the T-layout rows 4c + (lane & 3)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int64_t rt = rb * 8 + 4 * c + (lane & 3);
          dt[u][c] = (rb < nrb && rt < a.n) ? __ldg(a.zscale + rt) : 0.0;
        }
      }
#pragma unroll
      for (int nt = 0; nt < L::NT; ++nt) {
        double t[2] = {0.0, 0.0};
        if (ok) ld_rw<2>(t, a.R + row * K + col_c + nt * 8);
        rc[u][nt][0] = t[0];
        rc[u][nt][1] = t[1];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t rb = rb0 + u * wstride;
      const int64_t row = rb * 8 + (lane >> 2);
      const bool ok = rb < nrb && row < a.n;
#pragma unroll
      for (int nt = 0; nt < L::NT; ++nt)
#pragma unroll
        for (int kc = 0; kc < L::KC; ++kc) dmma(rc[u][nt], qa[u][kc], nlam[kc][nt]);
#pragma unroll
      for (int nt = 0; nt < L::NT; ++nt) {
        if (ok) st<2>(a.R + row * K + col_c + nt * 8, rc[u][nt]);
        acc[NG + nt * 2] = fma(rc[u][nt][0], rc[u][nt][0], acc[NG + nt * 2]);
        acc[NG + nt * 2 + 1] = fma(rc[u][nt][1], rc[u][nt][1], acc[NG + nt * 2 + 1]);
      }
      double tr[L::NT][2], tz[L::NT][2];
#pragma unroll
      for (int nt = 0; nt < L::NT; ++nt) {
        d_to_t(rc[u][nt], tr[nt], lane);
        tz[nt][0] = JAC ? tr[nt][0] * dt[u][0] : tr[nt][0];  // rho = <<Z, R>>
        tz[nt][1] = JAC ? tr[nt][1] * dt[u][1] : tr[nt][1];
      }
#pragma unroll
      for (int at = 0; at < L::NT; ++at)
#pragma unroll
        for (int bt = 0; bt < L::NT; ++bt) {
          double* gacc = acc + (at * L::NT + bt) * 2;
          double d[2] = {gacc[0], gacc[1]};
          dmma(d, tz[at][0], tr[bt][0]);
          dmma(d, tz[at][1], tr[bt][1]);
          gacc[0] = d[0];
          gacc[1] = d[1];
        }
    }
  }
  extern __shared__ double sm[];
  double* red = sm;
  if (!grid_reduce<L::TPR, NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  double* rho = sm + S::RED;
  double* beta_s = rho + S::CS;
  double* norms = beta_s + S::CS;
  double* ws = sm + S::RED + 3 * S::CS + K;
  gather_gram_mma<K, P, GLOBAL, NACC>(red, 0, rho);
  gather_norms_mma<K, P, GLOBAL, NACC>(red, NG, norms, a.dist != 0);
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.red2[i] = rho[i];
    for (int c = threadIdx.x; c < K; c += kThreads) a.red2[S::CS + c] = norms[c];
    return;
  }
  const int bad = fast_bsolve<P>(L::NB, P, a.coef + S::CS, rho, beta_s, ws);  // beta
  if (threadIdx.x == 0) a.ctrl->xpending = 1;
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

// ------------------------------------------------------------ K3 (DMMA) --
// X += P lambda; unless stopped: P' = Z + P beta (Z = R, D^-1 R or the ILU
// sweeps' Z) into a.Pn, rho_prev' = <<P', R>>.
// XM (deferred X update, the solver alternates 1 / 2 per iteration): 0 = X
// every iteration; 1 = skip: X untouched (unless the solve ends here), lambda
// saved to coef + 4 cs, ctrl->xold set, P' written to the other P buffer;
// 2 = flush: X += Pold lambda_old + P lambda in one pass.  X is then read and
// written every other iteration (K3 traffic 5nk -> 3nk / 6nk alternating).
template <int K, int P, bool GLOBAL, bool JAC = false, bool ZS = false, int XM = 0>
__device__ __forceinline__ void k3_mma_body(const IterArgs& a) {
  using L = MmaLayout<K, P, GLOBAL>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  const bool cur = *reinterpret_cast<const volatile int32_t*>(&a.ctrl->xpending) != 0;
  const bool old = XM == 2 && *reinterpret_cast<const volatile int32_t*>(&a.ctrl->xold) != 0;
  if (!cur && !old) return;
  const bool fin = stopped(a.ctrl);
  const bool upd = cur && !fin;           // P' and the Gram
  const bool dox = XM != 1 || fin;        // X written by this launch
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp % L::Q;
  double lam[L::KC][L::NT], bet[L::KC][L::NT], lamo[L::KC][L::NT];
  load_bfrag<K, P, GLOBAL>(a.coef, g, 1.0, lam, lane);
  load_bfrag<K, P, GLOBAL>(a.coef + 2 * S::CS, g, 1.0, bet, lane);
  if constexpr (XM == 2) load_bfrag<K, P, GLOBAL>(a.coef + 4 * S::CS, g, 1.0, lamo, lane);
  constexpr int NACC = L::NT * L::NT * 2;
  static_assert(L::TPR * NACC <= S::RED, "grid_reduce buffer");
  double acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.0;
  const int64_t nrb = (a.n + 7) >> 3;
  const int64_t wstride = (int64_t)gridDim.x * (kThreads / 32) / L::Q;
  const int col_a = g * L::PE + (lane & 3);
  const int col_c = g * L::PE + 2 * (lane & 3);
  double* Pout = XM == 0 ? a.P : a.Pn;
  // U row blocks per warp step, all loads issued before any DMMA: the skip
  // launch (XM 1) streams only P and R, too few bytes in flight at one block
  constexpr int U = (XM == 1 && (P <= 8 || K == 64) && !(BKG_K3_SKIP3 && P > 8)) ? 2 : 1;  // C4 p = 16: slower
  for (int64_t rb0 = ((int64_t)blockIdx.x * (kThreads / 32) + warp) / L::Q; rb0 < nrb;
       rb0 += U * wstride) {
    double pa[U][L::KC], po[U][L::KC], xc[U][L::NT][2], pn[U][L::NT][2], zz[U][L::NT][2];
    if constexpr (BKG_MMA_PF > 0) {
      if (g == 0 && lane == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t rbp = rb0 + (BKG_MMA_PF * U + u) * wstride;
          if (cur) mma_prefetch_block(a.P, rbp, nrb, a.n, K);
          if (upd) mma_prefetch_block(a.R, rbp, nrb, a.n, K);
          if (dox) mma_prefetch_block(a.X, rbp, nrb, a.n, K);
          if constexpr (XM == 2)
            if (old) mma_prefetch_block(a.Pold, rbp, nrb, a.n, K);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t rb = rb0 + u * wstride;
      const int64_t row = rb * 8 + (lane >> 2);
      const bool ok = rb < nrb && row < a.n;
#pragma unroll
      for (int kc = 0; kc < L::KC; ++kc) {
        pa[u][kc] = ok && cur ? a.P[row * K + col_a + kc * 4] : 0.0;
        po[u][kc] = 0.0;
        if constexpr (XM == 2) po[u][kc] = ok && old ? a.Pold[row * K + col_a + kc * 4] : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < L::NT; ++nt) {
        double t[2] = {0.0, 0.0}, r[2] = {0.0, 0.0}, zt[2] = {0.0, 0.0};
        if (ok) {
          if (dox) ld_rw<2>(t, a.X + row * K + col_c + nt * 8);
          if (upd) ld_nc<2>(r, a.R + row * K + col_c + nt * 8);
          if constexpr (ZS)
            if (upd) ld_nc<2>(zt, a.zsrc + row * K + col_c + nt * 8);
        }
        xc[u][nt][0] = t[0];
        xc[u][nt][1] = t[1];
        pn[u][nt][0] = r[0];
        pn[u][nt][1] = r[1];
        zz[u][nt][0] = zt[0];
        zz[u][nt][1] = zt[1];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t rb = rb0 + u * wstride;
      const int64_t row = rb * 8 + (lane >> 2);
      const bool ok = rb < nrb && row < a.n;
      double tr[L::NT][2];
      if (upd) {
#pragma unroll
        for (int nt = 0; nt < L::NT; ++nt) d_to_t(pn[u][nt], tr[nt], lane);  // R, T layout
        if constexpr (ZS) {  // P' = Z + P beta with Z from the ILU(0) sweeps
#pragma unroll
          for (int nt = 0; nt < L::NT; ++nt) {
            pn[u][nt][0] = zz[u][nt][0];
            pn[u][nt][1] = zz[u][nt][1];
          }
        }
        if constexpr (JAC) {  // P' = Z + P beta with Z = D^-1 R (Jacobi)
          const double dz = ok ? __ldg(a.zscale + row) : 0.0;
#pragma unroll
          for (int nt = 0; nt < L::NT; ++nt) {
            pn[u][nt][0] *= dz;
            pn[u][nt][1] *= dz;
          }
        }
      }
#pragma unroll
      for (int nt = 0; nt < L::NT; ++nt)
#pragma unroll
        for (int kc = 0; kc < L::KC; ++kc) {
          if constexpr (XM == 2)
            if (old) dmma(xc[u][nt], po[u][kc], lamo[kc][nt]);
          if (dox && cur) dmma(xc[u][nt], pa[u][kc], lam[kc][nt]);
          if (upd) dmma(pn[u][nt], pa[u][kc], bet[kc][nt]);
        }
      __syncwarp();
#pragma unroll
      for (int nt = 0; nt < L::NT; ++nt) {
        if (ok) {
          if (dox) st<2>(a.X + row * K + col_c + nt * 8, xc[u][nt]);
          if (upd) st<2>(Pout + row * K + col_c + nt * 8, pn[u][nt]);
        }
      }
      if (upd) {
        double tp[L::NT][2];
#pragma unroll
        for (int nt = 0; nt < L::NT; ++nt) d_to_t(pn[u][nt], tp[nt], lane);
#pragma unroll
        for (int at = 0; at < L::NT; ++at)
#pragma unroll
          for (int bt = 0; bt < L::NT; ++bt) {
            double* gacc = acc + (at * L::NT + bt) * 2;
            double d[2] = {gacc[0], gacc[1]};
            dmma(d, tp[at][0], tr[bt][0]);
            dmma(d, tp[at][1], tr[bt][1]);
            gacc[0] = d[0];
            gacc[1] = d[1];
          }
      }
    }
  }
  extern __shared__ double sm[];
  double* red = sm;
  if (!grid_reduce<L::TPR, NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  if (upd) gather_gram_mma<K, P, GLOBAL, NACC>(red, 0, (a.dist ? a.red1 : a.coef) + S::CS);
  if (XM == 1 && upd)
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.coef[4 * S::CS + i] = a.coef[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    if (XM == 1) a.ctrl->xold = upd ? 1 : 0;
    if (XM == 2) a.ctrl->xold = 0;
    a.ctrl->xpending = 0;
  }
}
template <int K, int P, bool GLOBAL, bool JAC = false, bool ZS = false, int XM = 0>
__global__ void __launch_bounds__(kThreads, (BKG_K3_SKIP3 && XM == 1 && P > 8 ? 3 : mma_minb<P, 3>()))
    k3_mma(IterArgs a) {
  k3_mma_body<K, P, GLOBAL, JAC, ZS, XM>(a);
}

}  // namespace bkg

namespace bkg {

// ------------------------------------------------------------ K1 (tile) --
// Q = A P and alpha = <<P, Q>> with the warp as the unit of work: a warp owns
// an 8-row x W-column tile (W = 16, or K when K < 16); lane (lane>>2) is its
// row and it accumulates W/4 columns of Q in the DMMA C/D layout (16-byte
// operand loads, one CSR stream per row shared by its 4 lanes).  The Gram
// tile P^T Q over the 8 rows is then DMMA work: P is read in the T layout
// (its rows are L1-resident: they were just read as diagonal operands) and Q
// is relaid D->T in registers.  Only the (at, bt) 8x8 tile pairs inside one
// p-group are formed (block-diagonal for P < 8).
template <int K, int P, int W>
struct TileLayout {
  static constexpr int QW = K / W;     // warps per 8-row block
  static constexpr int NTW = W / 8;    // 8-column tiles per warp
  static constexpr int PT = P >= 8 ? P / 8 : 1;  // tiles per p-group side
  // Gram tile pairs kept per warp: within-group pairs of its NTW tiles
  static constexpr int NPAIR = (P >= 8) ? NTW * PT : NTW;
  static constexpr int TPR = 32 * QW;
  static_assert(K % W == 0 && W % 8 == 0, "tile width");
  static_assert(P < 8 || W % P == 0, "a p-group must not straddle warps");
};

template <int K, int P, int W>
__device__ __forceinline__ void tile_pair(int idx, int& at, int& bt) {
  using T = TileLayout<K, P, W>;
  if (P >= 8) {  // idx = tile * PT + j: partner j inside the tile's group
    const int t = idx / T::PT, j = idx % T::PT;
    at = t;
    bt = (t / T::PT) * T::PT + j;
  } else {
    at = bt = idx;
  }
}

// Grid totals of the tile-pair Gram accumulators -> row-major p x p blocks.
template <int K, int P, int W, bool GLOBAL, int NACC>
__device__ void gather_gram_tile(const double* red, double* blocks) {
  using T = TileLayout<K, P, W>;
  constexpr int NB = GLOBAL ? 1 : K / P;
  constexpr int Qg = K / P;
  for (int idx = threadIdx.x; idx < NB * P * P; idx += kThreads) {
    const int blk = idx / (P * P), a = (idx / P) % P, b = idx % P;
    double s = 0.0;
    const int g0 = GLOBAL ? 0 : blk, g1 = GLOBAL ? Qg : blk + 1;
    for (int g = g0; g < g1; ++g) {
      const int ca = g * P + a, cb = g * P + b;
      const int w = ca / W, aw = ca % W, bw = cb % W;
      const int at = aw >> 3, bt = bw >> 3;
      int pi = 0;
      if (P >= 8) pi = at * T::PT + (bt % T::PT);
      else pi = at;
      const int lane = ((aw & 7) << 2) | ((bw & 7) >> 1), i = bw & 1;
      s += red[(w * 32 + lane) * NACC + pi * 2 + i];
    }
    blocks[idx] = s;
  }
}

#ifndef BKG_K1_MINB
#define BKG_K1_MINB 2
#endif
// K1 with the SpMM laid out for whole cache lines: LPR = W/2 lanes x 16 bytes
// cover a row's W-column segment (128 bytes when W = 16), so a warp tile is
// RPW = 64/W rows.  The Gram P^T Q over those rows is k = 4 rows per DMMA
// (m8n8k4), RPW/4 MMAs per tile pair; both operands are relaid from the row
// layout into the T layout with shuffles.  Software pipeline: the CSR chunk
// (values + columns) of tile t+1 and the row extents of tile t+2 are loaded
// while tile t's operand loads are in flight, so a tile costs one dependent
// memory round trip instead of three.
template <int K, int P, int W, bool GLOBAL>
__global__ void __launch_bounds__(kThreads, BKG_K1_MINB) k1_tile(IterArgs a) {
  using T = TileLayout<K, P, W>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  if (stopped(a.ctrl)) return;
  constexpr int LPR = W / 2, RPW = 32 / LPR, CHK = RPW / 4;
  constexpr int CH = 8;  // CSR entries per lane per chunk (a 7-point row in one)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = warp % T::QW;
  const int rr = lane / LPR, cl = lane % LPR;
  const int col = w * W + 2 * cl;
  const double* Pc = a.P + col;
  constexpr int NACC = T::NPAIR * 2;
  static_assert(T::TPR * NACC <= S::RED, "grid_reduce buffer");
  double acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.0;
  const int64_t ntile = (a.n + RPW - 1) / RPW;
  const int64_t wstride = (int64_t)gridDim.x * (kThreads / 32) / T::QW;
  const int64_t rstride = wstride * RPW;
  int64_t tile = ((int64_t)blockIdx.x * (kThreads / 32) + warp) / T::QW;
  int64_t row = tile * RPW + rr;

  auto extent = [&](int64_t r, int64_t& b, int& len) {
    b = 0;
    len = 0;
    if (r < a.n) {
      b = __ldg(a.rowptr + r);
      len = (int)(__ldg(a.rowptr + r + 1) - b);
    }
  };
  auto load_chunk = [&](int64_t b, int len, double (&v)[CH], int (&c)[CH]) {
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      v[u] = u < len ? __ldg(a.vals + b + u) : 0.0;
      c[u] = u < len ? __ldg(a.cols + b + u) : kNoCol;
    }
  };
  // FMAs of one chunk: inactive slots carry v = 0, x = 0.
  auto fma_chunk = [&](const double (&v)[CH], const int (&c)[CH], double (&q)[2]) {
    double x[CH][2];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if (c[u] != kNoCol) {
        ld_nc<2>(x[u], Pc + (int64_t)c[u] * K);
      } else {
        x[u][0] = x[u][1] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      q[0] = fma(v[u], x[u][0], q[0]);
      q[1] = fma(v[u], x[u][1], q[1]);
    }
  };

  int64_t b0, b1;
  int len0, len1;
  double v[CH];
  int c[CH];
  extent(row, b0, len0);
  extent(row + rstride, b1, len1);
  load_chunk(b0, len0, v, c);
  for (; tile < ntile; tile += wstride) {
    // prefetch: extents of tile t+2, CSR chunk of tile t+1
    int64_t b2;
    int len2;
    extent(row + 2 * rstride, b2, len2);
    double nv[CH];
    int nc[CH];
    load_chunk(b1, len1, nv, nc);
    double q[2] = {0.0, 0.0}, pd[2] = {0.0, 0.0};
    if (row < a.n) ld_nc<2>(pd, Pc + row * K);
    fma_chunk(v, c, q);
    for (int off = CH; off < len0; off += CH) {  // rows longer than one chunk
      double v2[CH];
      int c2[CH];
      load_chunk(b0 + off, len0 - off, v2, c2);
      fma_chunk(v2, c2, q);
    }
    __syncwarp();
    if (row < a.n) st<2>(a.Q + row * K + col, q);
    // T layout of the tile's 4-row chunks: t[nt][c] = tile[4c + (lane&3)][nt*8 + (lane>>2)]
    double pt[T::NTW][CHK], qt[T::NTW][CHK];
#pragma unroll
    for (int nt = 0; nt < T::NTW; ++nt)
#pragma unroll
      for (int cc = 0; cc < CHK; ++cc) {
        const int src = (4 * cc + (lane & 3)) * LPR + nt * 4 + (lane >> 3);
        const bool hi = (lane >> 2) & 1;
        const double q0 = __shfl_sync(kFull, q[0], src), q1 = __shfl_sync(kFull, q[1], src);
        const double p0 = __shfl_sync(kFull, pd[0], src), p1 = __shfl_sync(kFull, pd[1], src);
        qt[nt][cc] = hi ? q1 : q0;
        pt[nt][cc] = hi ? p1 : p0;
      }
#pragma unroll
    for (int pi = 0; pi < T::NPAIR; ++pi) {
      int at, bt;
      tile_pair<K, P, W>(pi, at, bt);
      double d[2] = {acc[2 * pi], acc[2 * pi + 1]};
#pragma unroll
      for (int cc = 0; cc < CHK; ++cc) dmma(d, pt[at][cc], qt[bt][cc]);
      acc[2 * pi] = d[0];
      acc[2 * pi + 1] = d[1];
    }
    row += rstride;
    b0 = b1;
    len0 = len1;
    b1 = b2;
    len1 = len2;
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      v[u] = nv[u];
      c[u] = nc[u];
    }
  }
  extern __shared__ double sm[];
  double* red = sm;
  if (!grid_reduce<T::TPR, NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  double* alpha = sm + S::RED;
  double* ws = alpha + 3 * S::CS;
  gather_gram_tile<K, P, W, GLOBAL, NACC>(red, alpha);
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.red1[i] = alpha[i];
    return;
  }
  const int bad = fast_bsolve<P>(S::NB, P, alpha, a.coef + S::CS, a.coef, ws);  // lambda
  if (bad >= 0) record_breakdown(a.ctrl, bad, 1);
}

}  // namespace bkg
