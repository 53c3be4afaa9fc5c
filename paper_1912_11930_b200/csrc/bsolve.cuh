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

// Standalone BSOLVE launch (one CTA).  status[0] = failing block or -1.
template <int P>
__global__ void k_bsolve(int nblk, int p, const double* gamma, const double* delta, double* out,
                         int* status) {
  extern __shared__ double ws[];
  const int bad = cta_bsolve<P>(nblk, p, gamma, delta, out, ws);
  if (threadIdx.x == 0) status[0] = bad;
}

}  // namespace bkg
