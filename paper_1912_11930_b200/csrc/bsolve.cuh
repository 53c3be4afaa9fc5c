// bsolve.cuh — on-device batched BSOLVE (kernels.hpp:166-240).
//
// gamma_b^{-1} delta_b for every p x p block, by LU with partial pivoting in
// exactly the reference's operation order (detail::solve_block,
// kernels.hpp:171-224): same max-norm / 1e-14 breakdown test, same
// "first strictly larger" pivot rule, same elimination and permuted
// forward/backward substitution, all with unfused IEEE double ops.  Results
// are therefore bit-identical to the reference for bit-identical inputs.
//
// Parallelisation keeps each element's operation sequence unchanged: during
// elimination thread (r,c) owns lu[r][c]; during substitution thread c owns
// result column c.  Blocks are solved concurrently, `par` at a time, by one
// CTA.  No host round-trip: the fused solver calls this from the last CTA of
// its grid reduction.
#pragma once

#include <climits>

#include "common.cuh"

namespace bkg {

__host__ __device__ inline int bsolve_par(int p, int nthreads) {
  const int pp = p * p;
  const int grp = pp < nthreads ? pp : nthreads;
  const int par = nthreads / grp;
  return par < 1 ? 1 : par;
}

// Shared-memory workspace (in doubles) needed by cta_bsolve.
__host__ __device__ inline int bsolve_ws_doubles(int p, int nthreads) {
  const int par = bsolve_par(p, nthreads);
  const int pp = p * p;
  const int ints = par * p + 2 * par + 1;
  return par * (2 * pp + 1 + p) + (ints + 1) / 2 + 1;
}

// Returns (to every thread) the smallest failing block index, or -1.
// gamma, delta: nblk*p*p row-major blocks (global or shared memory).
// out: nblk*p*p (global or shared; may alias neither input).
// ws: bsolve_ws_doubles(p, blockDim.x) doubles of shared memory.
template <int P>
__device__ int cta_bsolve(int nblk, int p_rt, const double* gamma, const double* delta,
                          double* out, double* ws) {
  const int p = P > 0 ? P : p_rt;
  const int pp = p * p;
  const int T = blockDim.x, tid = threadIdx.x;
  const int grp = pp < T ? pp : T;
  const int par = bsolve_par(p, T);
  const int gi = tid / grp;       // concurrent block slot served by this thread
  const int gt = tid - gi * grp;  // thread index inside the slot
  const bool in_grp = gi < par;

  double* lu_all = ws;
  double* res_all = ws + par * pp;
  double* maxn_all = ws + 2 * par * pp;
  // 1 / pivot of every elimination step, computed once by the pivot thread
  // (the same __ddiv_rn the reference applies to the same value, so bits are
  // unchanged) and reused by the elimination and the back substitution
  double* inv_all = maxn_all + par;
  int* perm_all = reinterpret_cast<int*>(ws + par * (2 * pp + 1 + p));
  int* piv_all = perm_all + par * p;
  int* brk_all = piv_all + par;
  int* bad_s = brk_all + par;

  if (tid == 0) *bad_s = INT_MAX;
  __syncthreads();

  for (int base = 0; base < nblk; base += par) {
    const int blk = base + gi;
    const bool live = in_grp && blk < nblk;
    double* lu = lu_all + gi * pp;
    double* res = res_all + gi * pp;
    double* invp = inv_all + gi * p;
    int* perm = perm_all + gi * p;
    if (live) {
      for (int el = gt; el < pp; el += grp) lu[el] = gamma[(size_t)blk * pp + el];
      for (int el = gt; el < p; el += grp) perm[el] = el;
      if (gt == 0) brk_all[gi] = 0;
    }
    __syncthreads();
    // max-norm (kernels.hpp:177-179); std::max(m, NaN) keeps m.
    if (live && gt == 0) {
      double m = 0.0;
      for (int el = 0; el < pp; ++el) {
        const double v = fabs(lu[el]);
        m = (m < v) ? v : m;
      }
      maxn_all[gi] = m;
    }
    __syncthreads();
    const double max_norm = live ? maxn_all[gi] : 0.0;
    const double tiny = __dmul_rn(1e-14, max_norm);
#pragma unroll 1
    for (int col = 0; col < p; ++col) {
      // pivot search + breakdown test (kernels.hpp:182-195), reference order.
      if (live && gt == 0 && !brk_all[gi]) {
        int pivot_row = col;
        double pivot = fabs(lu[col * p + col]);
        for (int r = col + 1; r < p; ++r) {
          const double cand = fabs(lu[r * p + col]);
          if (cand > pivot) {
            pivot = cand;
            pivot_row = r;
          }
        }
        if (pivot < tiny || max_norm == 0.0) brk_all[gi] = 1;
        piv_all[gi] = pivot_row;
        // lu[col][col] after the row swap
        invp[col] = __ddiv_rn(1.0, lu[pivot_row * p + col]);
      }
      __syncthreads();
      const bool go = live && !brk_all[gi];
      // row swap (kernels.hpp:196-199)
      if (go) {
        const int prow = piv_all[gi];
        if (prow != col) {
          for (int c = gt; c < p; c += grp) {
            const double t = lu[col * p + c];
            lu[col * p + c] = lu[prow * p + c];
            lu[prow * p + c] = t;
          }
          if (gt == 0) {
            const int t = perm[col];
            perm[col] = perm[prow];
            perm[prow] = t;
          }
        }
      }
      __syncthreads();
      // elimination (kernels.hpp:200-205).  Phase 1 updates the trailing
      // block (reads lu[r][col], untouched here); phase 2 stores f.
      if (go) {
        const double inv = invp[col];
        for (int el = gt; el < pp; el += grp) {
          const int r = el / p, c = el - r * p;
          if (r > col && c > col) {
            const double f = __dmul_rn(lu[r * p + col], inv);
            lu[r * p + c] = __dsub_rn(lu[r * p + c], __dmul_rn(f, lu[col * p + c]));
          }
        }
      }
      __syncthreads();
      if (go) {
        const double inv = invp[col];
        for (int r = col + 1 + gt; r < p; r += grp) lu[r * p + col] = __dmul_rn(lu[r * p + col], inv);
      }
      __syncthreads();
    }
    // permuted forward then backward substitution (kernels.hpp:208-223).
    if (live && !brk_all[gi]) {
      const double* dl = delta + (size_t)blk * pp;
      for (int c = gt; c < p; c += grp) {
        for (int r = 0; r < p; ++r) res[r * p + c] = dl[perm[r] * p + c];
        for (int r = 0; r < p; ++r) {
          double acc = res[r * p + c];
          for (int j = 0; j < r; ++j) acc = __dsub_rn(acc, __dmul_rn(lu[r * p + j], res[j * p + c]));
          res[r * p + c] = acc;
        }
        for (int r = p; r-- > 0;) {
          double acc = res[r * p + c];
          for (int j = r + 1; j < p; ++j)
            acc = __dsub_rn(acc, __dmul_rn(lu[r * p + j], res[j * p + c]));
          res[r * p + c] = __dmul_rn(acc, invp[r]);  // = __ddiv_rn(1.0, lu[r][r])
        }
      }
    }
    __syncthreads();
    if (live) {
      if (brk_all[gi]) {
        if (gt == 0) atomicMin(bad_s, blk);
      } else {
        for (int el = gt; el < pp; el += grp) out[(size_t)blk * pp + el] = res[el];
      }
    }
    __syncthreads();
  }
  const int bad = *bad_s;
  __syncthreads();
  return bad == INT_MAX ? -1 : bad;
}

// gamma_b^-1 delta_b for every p x p block with one warp per block, in the
// operation order of detail::solve_block (kernels.hpp:171-224), as cta_bsolve
// (bsolve.cuh) -- same max-norm / 1e-14 breakdown test, same "first strictly
// larger" pivot rule, unfused multiply / subtract per element in the same
// sequence -- but without a CTA barrier per elimination step: lane c < P owns
// column c of the block, lane P + c column c of the right-hand side, both in
// registers; multipliers and pivots travel by shuffles.  cta_bsolve's 4
// barriers and single-thread pivot search per column made the two solves 47%
// of a C1 iteration.  Returns the smallest failing block or -1 to every thread.
// gamma, delta, out: shared or global memory; bad_s: one int of shared memory.
// Every thread of the CTA must call it (CTA barriers around the flag).
template <int P>
__device__ int warp_bsolve(int nblk, const double* gamma, const double* delta, double* out,
                           int* bad_s) {
  static_assert(P >= 1 && P <= 16, "one warp holds [A | B]");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) *bad_s = INT_MAX;
  __syncthreads();
  for (int blk = warp; blk < nblk; blk += (int)(blockDim.x >> 5)) {
    const bool isa = lane < P, isb = lane >= P && lane < 2 * P;
    const int cidx = isa ? lane : lane - P;
    const double* src = (isa ? gamma : delta) + (size_t)blk * P * P;
    double col[P], inv[P];
#pragma unroll
    for (int r = 0; r < P; ++r) col[r] = (isa || isb) ? src[r * P + cidx] : 0.0;
    // max-norm of the block (kernels.hpp:177-179)
    double m = 0.0;
    if (isa) {
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const double v = fabs(col[r]);
        m = (m < v) ? v : m;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v = __shfl_xor_sync(0xffffffffu, m, o);
      m = (m < v) ? v : m;
    }
    const double tiny = __dmul_rn(1e-14, m);
    bool broke = false;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      // pivot search in column k by its owner, reference order (kernels.hpp:182-195)
      int prow = k;
      double pv = fabs(col[k]);
#pragma unroll
      for (int r = k + 1; r < P; ++r) {
        const double cand = fabs(col[r]);
        if (cand > pv) {
          pv = cand;
          prow = r;
        }
      }
      prow = __shfl_sync(0xffffffffu, prow, k);
      pv = __shfl_sync(0xffffffffu, pv, k);
      if (pv < tiny || m == 0.0) {
        broke = true;
        break;
      }
      // row swap (every column, right-hand sides included: the permuted delta)
#pragma unroll
      for (int r = k + 1; r < P; ++r)
        if (r == prow) {
          const double t = col[k];
          col[k] = col[r];
          col[r] = t;
        }
      inv[k] = __ddiv_rn(1.0, __shfl_sync(0xffffffffu, col[k], k));
      // elimination: f = lu[r][k] * inv; lu[r][c] -= f * lu[k][c] for c > k and
      // every right-hand side (the forward substitution, same order in k)
#pragma unroll
      for (int r = k + 1; r < P; ++r) {
        const double f = __dmul_rn(__shfl_sync(0xffffffffu, col[r], k), inv[k]);
        if (lane > k) col[r] = __dsub_rn(col[r], __dmul_rn(f, col[k]));
      }
    }
    if (broke) {
      if (lane == 0) atomicMin(bad_s, blk);
      continue;
    }
    // backward substitution (kernels.hpp:216-223): right-hand-side lanes
#pragma unroll
    for (int r = P - 1; r >= 0; --r) {
      double accv = col[r];
#pragma unroll
      for (int j = r + 1; j < P; ++j) {
        const double u = __shfl_sync(0xffffffffu, col[r], j);  // lu[r][j], column j's lane
        if (isb) accv = __dsub_rn(accv, __dmul_rn(u, col[j]));
      }
      if (isb) col[r] = __dmul_rn(accv, inv[r]);
    }
    if (isb) {
#pragma unroll
      for (int r = 0; r < P; ++r) out[(size_t)blk * P * P + r * P + cidx] = col[r];
    }
  }
  __syncthreads();
  const int bad = *bad_s;
  __syncthreads();
  return bad == INT_MAX ? -1 : bad;
}

// The fused fast kernels' solves: one warp per block for the tabulated block
// widths (same results as cta_bsolve: same operations per element), else the
// CTA-wide solver.  ws: bsolve_ws_doubles(p, blockDim.x) doubles of shared memory.
template <int P>
__device__ int fast_bsolve(int nblk, int p_rt, const double* gamma, const double* delta,
                           double* out, double* ws) {
  int* flag = reinterpret_cast<int*>(ws);
  if constexpr (P >= 1 && P <= 16) {
    return warp_bsolve<P>(nblk, gamma, delta, out, flag);
  } else {
    switch (P > 0 ? P : p_rt) {
      case 1: return warp_bsolve<1>(nblk, gamma, delta, out, flag);
      case 2: return warp_bsolve<2>(nblk, gamma, delta, out, flag);
      case 4: return warp_bsolve<4>(nblk, gamma, delta, out, flag);
      case 8: return warp_bsolve<8>(nblk, gamma, delta, out, flag);
      case 16: return warp_bsolve<16>(nblk, gamma, delta, out, flag);
      default: return cta_bsolve<P>(nblk, p_rt, gamma, delta, out, ws);
    }
  }
}

// Standalone BSOLVE launch (one CTA).  status[0] = failing block or -1.
template <int P>
__global__ void k_bsolve(int nblk, int p, const double* gamma, const double* delta, double* out,
                         int* status) {
  extern __shared__ double ws[];
  const int bad = cta_bsolve<P>(nblk, p, gamma, delta, out, ws);
  if (threadIdx.x == 0) status[0] = bad;
}

}  // namespace bkg
