// precond.cuh — Preconditioner on device (preconditioners.hpp:66-196).
//
// identity: Z = R.  Jacobi: Z = D^-1 R, D^-1 = 1/diag(A) (preconditioners.hpp:48-59).
// ILU(0): factor (ilu0_factor, :153-196) and apply (forward L, backward U
// sweeps, :95-127), level-scheduled: a row is processed once every row it
// depends on is done, and each row runs exactly the reference's operation
// sequence (CSR order, unfused mul/sub), so results are bit-identical to the
// reference.  Levels come from a host pass over the pattern (setup only).
#pragma once

#include <algorithm>
#include <climits>
#include <vector>

#include "common.cuh"

namespace bkg {

int elem_grid(const bkg_ctx* c, int64_t total);
void launch(bkg_ctx* c, const void* fn, int grid, int block, size_t smem, void** args);

// ------------------------------------------------------------ Jacobi -----
// inv_diag[r] = 1 / A(r,r); bad_row = first row whose diagonal is not > 0.
__global__ void k_jacobi_setup(int64_t n, const int64_t* __restrict__ rowptr,
                               const int32_t* __restrict__ cols, const double* __restrict__ vals,
                               double* __restrict__ inv_diag, unsigned long long* bad_row) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;  // SparseMatrix::at: 0 when (r,r) is not stored
    for (int64_t i = rowptr[r]; i < rowptr[r + 1]; ++i)
      if (cols[i] == r) d = vals[i];
    if (!(d > 0.0)) atomicMin(bad_row, (unsigned long long)r);
    inv_diag[r] = __ddiv_rn(1.0, d);
  }
}

__global__ void k_jacobi_apply(const Ctrl* ctrl, int64_t n, int k,
                               const double* __restrict__ inv_diag, const double* __restrict__ r,
                               double* __restrict__ z) {
  if (stopped(ctrl)) return;
  const int64_t total = n * (int64_t)k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    z[idx] = __dmul_rn(inv_diag[idx / k], r[idx]);
}

// ------------------------------------------------------------- ILU(0) ----
// One dependency level of the factorization (preconditioners.hpp:167-193).
__global__ void k_ilu_factor_level(const int32_t* __restrict__ rows, int count,
                                   const int64_t* __restrict__ rowptr,
                                   const int32_t* __restrict__ cols, double* lu,
                                   double* inv_diag, int64_t* diag_pos,
                                   unsigned long long* bad_row) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x) {
    const int64_t row = rows[t];
    const int64_t end = rowptr[row + 1];
    for (int64_t i = rowptr[row]; i < end && cols[i] < row; ++i) {
      const int64_t j = cols[i];
      const double factor = __dmul_rn(lu[i], inv_diag[j]);
      lu[i] = factor;
      int64_t target = i + 1;
      for (int64_t ju = diag_pos[j] + 1; ju < rowptr[j + 1]; ++ju) {
        const int32_t c = cols[ju];
        while (target < end && cols[target] < c) ++target;
        if (target == end) break;
        if (cols[target] == c) lu[target] = __dsub_rn(lu[target], __dmul_rn(factor, lu[ju]));
      }
    }
    int64_t dp = -1;  // std::lower_bound(row): first column >= row
    for (int64_t i = rowptr[row]; i < end; ++i)
      if (cols[i] >= row) {
        if (cols[i] == row) dp = i;
        break;
      }
    if (dp < 0 || lu[dp] == 0.0) {
      atomicMin(bad_row, (unsigned long long)row);
      diag_pos[row] = dp < 0 ? rowptr[row] : dp;
      inv_diag[row] = 0.0;
      continue;
    }
    diag_pos[row] = dp;
    inv_diag[row] = __ddiv_rn(1.0, lu[dp]);
  }
}

// Forward sweep L y = r (unit diagonal), one level (preconditioners.hpp:98-108).
__global__ void k_ilu_fwd_level(const Ctrl* ctrl, const int32_t* __restrict__ rows, int count,
                                int k, const int64_t* __restrict__ rowptr,
                                const int32_t* __restrict__ cols, const double* __restrict__ lu,
                                double* z) {
  if (stopped(ctrl)) return;
  const int64_t total = (int64_t)count * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = rows[idx / k];
    const int c = (int)(idx % k);
    double acc = z[row * k + c];
    for (int64_t i = rowptr[row]; i < rowptr[row + 1] && cols[i] < row; ++i)
      acc = __dsub_rn(acc, __dmul_rn(lu[i], z[(int64_t)cols[i] * k + c]));
    z[row * k + c] = acc;
  }
}

// Backward sweep U z = y, one level (preconditioners.hpp:109-123).
__global__ void k_ilu_bwd_level(const Ctrl* ctrl, const int32_t* __restrict__ rows, int count,
                                int k, const int64_t* __restrict__ rowptr,
                                const int32_t* __restrict__ cols, const double* __restrict__ lu,
                                const double* __restrict__ inv_diag, double* z) {
  if (stopped(ctrl)) return;
  const int64_t total = (int64_t)count * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = rows[idx / k];
    const int c = (int)(idx % k);
    double acc = z[row * k + c];
    for (int64_t i = rowptr[row + 1]; i-- > rowptr[row];) {
      const int64_t col = cols[i];
      if (col <= row) break;
      acc = __dsub_rn(acc, __dmul_rn(lu[i], z[col * k + c]));
    }
    z[row * k + c] = __dmul_rn(acc, inv_diag[row]);
  }
}

// ---------------------------------------------- ILU(0), sync-free sweeps --
// One persistent launch per triangular sweep instead of one launch per
// dependency level (C2: 382 + 382 levels, launch-bound at ~8 ms per apply).
// Rows are cut into segments of S consecutive rows, handed to warps by an
// atomic ticket in processing order (forward: ascending rows, backward:
// descending); a warp sweeps its segment row by row.  Completion is carried
// by the data itself: the output buffer is filled with a NaN sentinel before
// the sweep, and a dependency is ready once its element is no longer the
// sentinel (each element is one 8-byte store, read back with L2 loads), so
// there are no fences or flags; the previous row of the segment (the x
// neighbour of a lexicographic stencil) is taken from registers.  Every
// dependency of the lowest unfinished row is finished and its segment's warp
// is running, so the sweep cannot deadlock.  Lanes own columns (lane, lane +
// 32); each element runs exactly the reference's operation sequence (CSR
// order, unfused mul/sub), so the result is bit-identical to
// preconditioners.hpp:95-127 (a result whose bits equal the sentinel -- a
// NaN -- is stored as the canonical NaN).
#ifndef BKG_ILU_ELL
#define BKG_ILU_ELL 1
#endif
// Lanes per segment for 16 < k <= 32 in the ELL sweep (16 would run two
// segments per warp with two columns per lane: C2 apply 2.46 -> 3.56 ms)
#ifndef BKG_ILU_W32
#define BKG_ILU_W32 32
#endif
// Longest sync-free sweep segment (rows per ticket).
#ifndef BKG_ILU_SEG
#define BKG_ILU_SEG 256
#endif
constexpr unsigned long long kIluSentinel = 0x7FF4DEAD7FF4DEADull;

__device__ __forceinline__ double ld_ready(const double* p) {
  unsigned long long v;
  do {
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  } while (v == kIluSentinel);
  return __longlong_as_double((long long)v);
}
__device__ __forceinline__ double not_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) == kIluSentinel ? __longlong_as_double(0x7FF8000000000000ll) : v;
}

__global__ void k_ilu_fill(const Ctrl* ctrl, int64_t total, double* a, double* b,
                           unsigned long long* tickets) {
  if (stopped(ctrl)) return;
  const double s = __longlong_as_double((long long)kIluSentinel);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    a[i] = s;
    b[i] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x < 2) tickets[threadIdx.x] = 0;
}

// FWD: out = L^-1 src (unit lower); BWD: out = U^-1 src over the CSR (rows
// with more than 16 triangle entries); out must hold the sentinel everywhere
// on entry; src and out must not alias.
template <bool FWD>
__global__ void __launch_bounds__(256) k_ilu_sweep_csr(const Ctrl* ctrl, int64_t n, int k, int64_t nseg,
                                                      const int64_t* __restrict__ segs,
                                                      const int64_t* __restrict__ rowptr,
                                                      const int32_t* __restrict__ cols,
                                                      const double* __restrict__ lu,
                                                      const double* __restrict__ inv_diag,
                                                      const double* __restrict__ src, double* out,
                                                      unsigned long long* ticket) {
  if (stopped(ctrl)) return;
  const int lane = threadIdx.x & 31;
  const bool c0 = lane < k, c1 = lane + 32 < k;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    const int64_t s = (int64_t)__shfl_sync(0xffffffffu, t, 0);
    if (s >= nseg) return;
    // segment s: positions [segs[s], segs[s+1]) in processing order (row =
    // position forward, n - 1 - position backward)
    const int64_t pb = segs[s];
    const int64_t first = FWD ? pb : n - 1 - pb;  // first row in processing order
    const int cnt = (int)(segs[s + 1] - pb);
    double p0 = 0.0, p1 = 0.0;  // previous row of the segment (registers)
    for (int i = 0; i < cnt; ++i) {
      const int64_t row = FWD ? first + i : first - i;
      const int64_t prev = FWD ? row - 1 : row + 1;
      double a0 = 0.0, a1 = 0.0;
      if (c0) a0 = src[row * k + lane];
      if (c1) a1 = src[row * k + lane + 32];
      const int64_t rb = rowptr[row], re = rowptr[row + 1];
      for (int64_t e = FWD ? rb : re - 1; FWD ? e < re : e >= rb; FWD ? ++e : --e) {
        const int64_t col = cols[e];
        if (FWD ? col >= row : col <= row) break;
        const double v = lu[e];
        double x0 = 0.0, x1 = 0.0;
        if (col == prev && i > 0) {
          x0 = p0;
          x1 = p1;
        } else {
          if (c0) x0 = ld_ready(out + col * k + lane);
          if (c1) x1 = ld_ready(out + col * k + lane + 32);
        }
        a0 = __dsub_rn(a0, __dmul_rn(v, x0));
        a1 = __dsub_rn(a1, __dmul_rn(v, x1));
      }
      if (!FWD) {
        const double d = inv_diag[row];
        a0 = __dmul_rn(a0, d);
        a1 = __dmul_rn(a1, d);
      }
      if (c0) out[row * k + lane] = not_sentinel(a0);
      if (c1) out[row * k + lane + 32] = not_sentinel(a1);
      p0 = a0;
      p1 = a1;
    }
  }
}

// Sweep over a padded row-major copy of the triangle (ELL: D entries per row
// in the reference's processing order, column -1 = padding): entry addresses
// need no row-offset load, and row i+1's entries and source element are
// loaded while row i is computed, so a row costs one dependent load round
// trip (its dependencies) instead of three.  Few registers: occupancy (the
// number of segments in flight) sets the sweep's speed.
template <bool FWD, int D>
__global__ void __launch_bounds__(256, (D <= 8 ? 4 : 3)) k_ilu_sweep_ell(const Ctrl* ctrl, int64_t n, int k, int64_t nseg,
                                                       const int64_t* __restrict__ segs,
                                                       const int32_t* __restrict__ ecols,
                                                       const double* __restrict__ evals,
                                                       const double* __restrict__ inv_diag,
                                                       const double* __restrict__ src,
                                                       double* out, unsigned long long* ticket) {
  if (stopped(ctrl)) return;
  // k <= 16: the warp splits into 32 / W lane groups of W = 8 or 16 lanes,
  // each sweeping its own segment (more segments in flight per register)
  // lane groups of W lanes, two columns per lane (lane, lane + W) when k > W:
  // k <= 8: W = 8, k <= 16: 16, k <= 64: 32
  const int W = k <= 8 ? 8 : (k <= 16 ? 16 : (k <= 32 ? BKG_ILU_W32 : 32));
  const int wl = threadIdx.x & 31, g = wl / W;
  const int lane = wl % W;  // column index within the group
  const unsigned gmask = W == 32 ? 0xffffffffu : (((1u << W) - 1u) << (g * W));
  const bool c0 = lane < k, c1 = lane + W < k;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    const int64_t s = (int64_t)__shfl_sync(gmask, t, g * W);
    if (s >= nseg) return;
    const int64_t pb = segs[s];
    const int64_t first = FWD ? pb : n - 1 - pb;
    const int cnt = (int)(segs[s + 1] - pb);
    int cc[D];
    double vv[D], s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int u = 0; u < D; ++u) {
      cc[u] = ecols[first * D + u];
      vv[u] = evals[first * D + u];
    }
    if (c0) s0 = src[first * k + lane];
    if (c1) s1 = src[first * k + lane + W];
    double p0 = 0.0, p1 = 0.0;
    for (int i = 0; i < cnt; ++i) {
      const int64_t row = FWD ? first + i : first - i;
      const int64_t prev = FWD ? row - 1 : row + 1;
      int nc[D];
      double nv[D], n0 = 0.0, n1 = 0.0;
      if (i + 1 < cnt) {  // next row's entries and source element
        const int64_t nr = FWD ? row + 1 : row - 1;
#pragma unroll
        for (int u = 0; u < D; ++u) {
          nc[u] = ecols[nr * D + u];
          nv[u] = evals[nr * D + u];
        }
        if (c0) n0 = src[nr * k + lane];
        if (c1) n1 = src[nr * k + lane + W];
      }
      double a0 = s0, a1 = s1;
#pragma unroll
      for (int u = 0; u < D; ++u) {
        if (cc[u] < 0) break;
        double x0 = 0.0, x1 = 0.0;
        if (cc[u] == prev && i > 0) {
          x0 = p0;
          x1 = p1;
        } else {
          if (c0) x0 = ld_ready(out + (int64_t)cc[u] * k + lane);
          if (c1) x1 = ld_ready(out + (int64_t)cc[u] * k + lane + W);
        }
        a0 = __dsub_rn(a0, __dmul_rn(vv[u], x0));
        a1 = __dsub_rn(a1, __dmul_rn(vv[u], x1));
      }
      if (!FWD) {
        const double d = inv_diag[row];
        a0 = __dmul_rn(a0, d);
        a1 = __dmul_rn(a1, d);
      }
      if (c0) out[row * k + lane] = not_sentinel(a0);
      if (c1) out[row * k + lane + W] = not_sentinel(a1);
      p0 = a0;
      p1 = a1;
#pragma unroll
      for (int u = 0; u < D; ++u) {
        cc[u] = nc[u];
        vv[u] = nv[u];
      }
      s0 = n0;
      s1 = n1;
    }
  }
}

// ELL copy of the strict lower (FWD, CSR order) or upper (BWD, reverse CSR
// order) part of the ILU factors: D entries per row, column -1 = padding.
__global__ void k_ilu_ell_build(int64_t n, int D, bool fwd, const int64_t* __restrict__ rowptr,
                                const int32_t* __restrict__ cols, const double* __restrict__ lu,
                                int32_t* __restrict__ ecols, double* __restrict__ evals) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int u = 0;
    const int64_t rb = rowptr[r], re = rowptr[r + 1];
    if (fwd) {
      for (int64_t e = rb; e < re && cols[e] < r && u < D; ++e, ++u) {
        ecols[r * D + u] = cols[e];
        evals[r * D + u] = lu[e];
      }
    } else {
      for (int64_t e = re - 1; e >= rb && cols[e] > r && u < D; --e, ++u) {
        ecols[r * D + u] = cols[e];
        evals[r * D + u] = lu[e];
      }
    }
    for (; u < D; ++u) {
      ecols[r * D + u] = -1;
      evals[r * D + u] = 0.0;
    }
  }
}

__global__ void k_copy_ctrl(const Ctrl* ctrl, int64_t total, const double* __restrict__ src,
                            double* __restrict__ dst) {
  if (stopped(ctrl)) return;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    dst[idx] = src[idx];
}

// Level sets (rows grouped by dependency depth) of the lower (forward) or
// upper (backward) triangle of the pattern, from the device CSR.
inline void build_levels(bkg_ctx* c, bkg_matrix* a) {
  const int64_t n = (int64_t)a->n;
  std::vector<int64_t> rp(n + 1);
  std::vector<int32_t> cl(a->nnz);
  BKG_CUDA_CHECK(cudaMemcpyAsync(rp.data(), a->rowptr.ptr, sizeof(int64_t) * (n + 1),
                                 cudaMemcpyDeviceToHost, c->stream));
  if (a->nnz)
    BKG_CUDA_CHECK(cudaMemcpyAsync(cl.data(), a->cols.ptr, sizeof(int32_t) * a->nnz,
                                   cudaMemcpyDeviceToHost, c->stream));
  BKG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  auto make = [&](bool fwd, DevBuf<int32_t>& rows_out, std::vector<int64_t>& ptr) {
    std::vector<int32_t> lev(n, 0);
    int32_t maxl = 0;
    if (fwd) {
      for (int64_t r = 0; r < n; ++r) {
        int32_t l = 0;
        for (int64_t i = rp[r]; i < rp[r + 1] && cl[i] < r; ++i) l = std::max(l, lev[cl[i]] + 1);
        lev[r] = l;
        maxl = std::max(maxl, l);
      }
    } else {
      for (int64_t r = n - 1; r >= 0; --r) {
        int32_t l = 0;
        for (int64_t i = rp[r + 1]; i-- > rp[r];) {
          if (cl[i] <= r) break;
          l = std::max(l, lev[cl[i]] + 1);
        }
        lev[r] = l;
        maxl = std::max(maxl, l);
      }
    }
    ptr.assign(maxl + 2, 0);
    for (int64_t r = 0; r < n; ++r) ptr[lev[r] + 1]++;
    for (int32_t l = 0; l <= maxl; ++l) ptr[l + 1] += ptr[l];
    std::vector<int32_t> rows(n);
    std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
    for (int64_t r = 0; r < n; ++r) rows[fill[lev[r]]++] = (int32_t)r;
    rows_out.alloc(n);
    BKG_CUDA_CHECK(cudaMemcpyAsync(rows_out.ptr, rows.data(), sizeof(int32_t) * n,
                                   cudaMemcpyHostToDevice, c->stream));
    BKG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  };
  make(true, a->level_rows, a->level_ptr_fwd);
  make(false, a->level_rows_bwd, a->level_ptr_bwd);
  // ILU multiply-add count per apply (preconditioners.hpp:123-125) and the
  // longest strictly lower / upper row parts (sync-free sweep pipeline depth)
  uint64_t off = 0;
  int lmax = 0, umax = 0;
  for (int64_t r = 0; r < n; ++r) {
    int lo = 0, up = 0;
    for (int64_t i = rp[r]; i < rp[r + 1]; ++i) {
      if (cl[i] != r) ++off;
      if (cl[i] < r) ++lo;
      if (cl[i] > r) ++up;
    }
    lmax = std::max(lmax, lo);
    umax = std::max(umax, up);
  }
  a->ilu_offdiag = off;
  a->ilu_lower_max = lmax;
  a->ilu_upper_max = umax;
  // Sync-free sweep segments: maximal runs of rows chained by the previous
  // row (forward: row r depends on r-1; backward: on r+1), split every
  // BKG_ILU_SEG rows, so a segment's first row never waits for the end of the
  // segment before it (stencil x-lines become segments).
  auto segs = [&](bool fwd, DevBuf<int64_t>& out, int64_t& count) {
    std::vector<int64_t> b;
    int64_t run = 0;
    for (int64_t q = 0; q < n; ++q) {  // q: position in processing order
      const int64_t r = fwd ? q : n - 1 - q;
      bool chained = false;
      if (q > 0) {
        const int64_t want = fwd ? r - 1 : r + 1;
        for (int64_t i = rp[r]; i < rp[r + 1]; ++i)
          if (cl[i] == want) chained = true;
      }
      if (!chained || run >= BKG_ILU_SEG) {
        b.push_back(q);
        run = 0;
      }
      ++run;
    }
    b.push_back(n);
    count = (int64_t)b.size() - 1;
    out.alloc(b.size());
    BKG_CUDA_CHECK(cudaMemcpyAsync(out.ptr, b.data(), sizeof(int64_t) * b.size(),
                                   cudaMemcpyHostToDevice, c->stream));
    BKG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  };
  segs(true, a->ilu_seg_f, a->ilu_nseg_f);
  segs(false, a->ilu_seg_b, a->ilu_nseg_b);
}

inline int grid_for(const bkg_ctx* c, int64_t total) { return elem_grid(c, total); }

inline void jacobi_ready(bkg_ctx* c, bkg_matrix* a) {
  if (a->precond_ready == BKG_PRECOND_JACOBI) return;
  const int64_t n = (int64_t)a->n;
  a->inv_diag.alloc(n);
  DevBuf<unsigned long long> bad(1);
  const unsigned long long none = ~0ull;
  BKG_CUDA_CHECK(cudaMemcpyAsync(bad.ptr, &none, sizeof(none), cudaMemcpyHostToDevice, c->stream));
  const int64_t* rp = a->rowptr.ptr;
  const int32_t* cl = a->cols.ptr;
  const double* vl = a->vals.ptr;
  double* inv = a->inv_diag.ptr;
  unsigned long long* b = bad.ptr;
  int64_t nn = n;
  void* args[] = {&nn, &rp, &cl, &vl, &inv, &b};
  launch(c, (const void*)&k_jacobi_setup, elem_grid(c, n), 256, 0, args);
  unsigned long long h = 0;
  BKG_CUDA_CHECK(cudaMemcpyAsync(&h, bad.ptr, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  BKG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (h != none) {
    a->bad_row = (int64_t)h;
    throw Error(BKG_FACTORIZATION,
                "jacobi: diagonal entry " + std::to_string(h) + " is not strictly positive");
  }
  a->precond_ready = BKG_PRECOND_JACOBI;
}

inline void ilu_ready(bkg_ctx* c, bkg_matrix* a) {
  if (a->precond_ready == BKG_PRECOND_ILU0) return;
  const int64_t n = (int64_t)a->n;
  if (a->level_ptr_fwd.empty()) build_levels(c, a);
  a->inv_diag.alloc(n);
  a->lu.alloc(std::max<uint64_t>(a->nnz, 1));
  a->diag_pos.alloc(n);
  BKG_CUDA_CHECK(cudaMemcpyAsync(a->lu.ptr, a->vals.ptr, sizeof(double) * a->nnz,
                                 cudaMemcpyDeviceToDevice, c->stream));
  DevBuf<unsigned long long> bad(1);
  const unsigned long long none = ~0ull;
  BKG_CUDA_CHECK(cudaMemcpyAsync(bad.ptr, &none, sizeof(none), cudaMemcpyHostToDevice, c->stream));
  const int64_t* rp = a->rowptr.ptr;
  const int32_t* cl = a->cols.ptr;
  double* lu = a->lu.ptr;
  double* inv = a->inv_diag.ptr;
  int64_t* dpos = a->diag_pos.ptr;
  unsigned long long* b = bad.ptr;
  for (size_t l = 0; l + 1 < a->level_ptr_fwd.size(); ++l) {
    const int32_t* rows = a->level_rows.ptr + a->level_ptr_fwd[l];
    int cnt = (int)(a->level_ptr_fwd[l + 1] - a->level_ptr_fwd[l]);
    if (!cnt) continue;
    void* args[] = {&rows, &cnt, &rp, &cl, &lu, &inv, &dpos, &b};
    launch(c, (const void*)&k_ilu_factor_level, grid_for(c, cnt), 128, 0, args);
  }
  unsigned long long h = 0;
  BKG_CUDA_CHECK(cudaMemcpyAsync(&h, bad.ptr, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  BKG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  if (h != none) {
    a->bad_row = (int64_t)h;
    throw Error(BKG_FACTORIZATION, "ilu0: zero pivot or missing diagonal in row " +
                                       std::to_string(h));
  }
  // ELL copies of the factors' strict triangles for the sync-free sweeps
  a->ilu_ell_dl = a->ilu_ell_du = 0;
  if (BKG_ILU_ELL && a->ilu_lower_max <= 16 && a->ilu_upper_max <= 16) {
    auto round = [](int d) { return d <= 4 ? 4 : d <= 8 ? 8 : 16; };
    int dl = round(a->ilu_lower_max), du = round(a->ilu_upper_max);
    a->ilu_ell_lc.ensure((size_t)n * dl);
    a->ilu_ell_lv.ensure((size_t)n * dl);
    a->ilu_ell_uc.ensure((size_t)n * du);
    a->ilu_ell_uv.ensure((size_t)n * du);
    for (int pass = 0; pass < 2; ++pass) {
      bool fw = pass == 0;
      int d = fw ? dl : du;
      int32_t* ec = fw ? a->ilu_ell_lc.ptr : a->ilu_ell_uc.ptr;
      double* ev = fw ? a->ilu_ell_lv.ptr : a->ilu_ell_uv.ptr;
      int64_t nn = n;
      const double* luc = a->lu.ptr;
      void* args[] = {&nn, &d, &fw, &rp, &cl, &luc, &ec, &ev};
      launch(c, (const void*)&k_ilu_ell_build, elem_grid(c, n), 256, 0, args);
    }
    a->ilu_ell_dl = dl;
    a->ilu_ell_du = du;
  }
  a->precond_ready = BKG_PRECOND_ILU0;
}

// FlopCounter increment of one apply (preconditioners.hpp:91,124-125).
inline uint64_t precond_flops(const bkg_matrix* a, int kind, int k) {
  if (kind == BKG_PRECOND_JACOBI) return a->n * (uint64_t)k;
  if (kind == BKG_PRECOND_ILU0) return 2ull * k * a->ilu_offdiag + a->n * (uint64_t)k;
  return 0;
}

// Factor / validate the preconditioner of `kind` for matrix a (setup).
inline void precond_ready(bkg_ctx* c, bkg_matrix* a, int kind) {
  if (kind == BKG_PRECOND_JACOBI) jacobi_ready(c, a);
  if (kind == BKG_PRECOND_ILU0) ilu_ready(c, a);
}

// Lanes per segment for 16 < k <= 32 in the ELL sweep (16 would run two
// segments per warp with two columns per lane: C2 apply 2.46 -> 3.56 ms)
#ifndef BKG_ILU_W32
#define BKG_ILU_W32 32
#endif
// Longest sync-free sweep segment (rows per ticket).
#ifndef BKG_ILU_WARPS
#define BKG_ILU_WARPS 0  // cap on concurrent sweep warps (0: one full wave)
#endif
#ifndef BKG_ILU_SEG
#define BKG_ILU_SEG 256
#endif

// ILU(0) apply z = U^-1 L^-1 r with the sync-free sweeps (k <= 64); y is an
// n x k scratch for L^-1 r (the fused loop passes Q, free between K2 and K1).
inline void ilu_apply_sf(bkg_ctx* c, bkg_matrix* a, int k, const double* r, double* y, double* z,
                         const Ctrl* ctrl) {
  const int64_t n = (int64_t)a->n;
  a->ilu_state.ensure(2);
  const int64_t nseg = std::max(a->ilu_nseg_f, a->ilu_nseg_b);
  int dev = 0, nsm = 0;
  BKG_CUDA_CHECK(cudaGetDevice(&dev));
  BKG_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // as many resident warps as fit: a sweep is latency-bound per row, so the
  // number of segments in flight sets its speed
  auto grid_of = [&](const void* fn) {
    int per = 0;
    BKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, 0));
    int64_t cap = (int64_t)nsm * std::max(per, 1);
    if (BKG_ILU_WARPS > 0) cap = std::min<int64_t>(cap, BKG_ILU_WARPS / 8);
    return (int)std::max<int64_t>(1, std::min<int64_t>(cap, (nseg + 7) / 8));
  };
  const bool ell = a->ilu_ell_dl > 0 && a->ilu_ell_du > 0;
  auto ell_fn = [](bool fw, int d) -> const void* {
    if (fw) return d <= 4 ? (const void*)&k_ilu_sweep_ell<true, 4>
                 : d <= 8 ? (const void*)&k_ilu_sweep_ell<true, 8>
                          : (const void*)&k_ilu_sweep_ell<true, 16>;
    return d <= 4 ? (const void*)&k_ilu_sweep_ell<false, 4>
         : d <= 8 ? (const void*)&k_ilu_sweep_ell<false, 8>
                  : (const void*)&k_ilu_sweep_ell<false, 16>;
  };
  const void* fwd = ell ? ell_fn(true, a->ilu_ell_dl) : (const void*)&k_ilu_sweep_csr<true>;
  const void* bwd = ell ? ell_fn(false, a->ilu_ell_du) : (const void*)&k_ilu_sweep_csr<false>;
  const int64_t* rp = a->rowptr.ptr;
  const int32_t* cl = a->cols.ptr;
  const double* lu = a->lu.ptr;
  const double* inv = a->inv_diag.ptr;
  unsigned long long* st = a->ilu_state.ptr;
  int64_t nn = n, tot = n * (int64_t)k;
  int kk = k;
  {
    void* args[] = {&ctrl, &tot, &y, &z, &st};
    launch(c, (const void*)&k_ilu_fill, elem_grid(c, tot), 256, 0, args);
  }
  for (int pass = 0; pass < 2; ++pass) {
    const bool fw = pass == 0;
    const double* srcp = fw ? r : y;
    double* outp = fw ? y : z;
    unsigned long long* tk = st + pass;
    int64_t ns = fw ? a->ilu_nseg_f : a->ilu_nseg_b;
    const int64_t* sg = fw ? a->ilu_seg_f.ptr : a->ilu_seg_b.ptr;
    if (ell) {
      const int32_t* ec = fw ? a->ilu_ell_lc.ptr : a->ilu_ell_uc.ptr;
      const double* ev = fw ? a->ilu_ell_lv.ptr : a->ilu_ell_uv.ptr;
      void* args[] = {&ctrl, &nn, &kk, &ns, &sg, &ec, &ev, &inv, &srcp, &outp, &tk};
      launch(c, fw ? fwd : bwd, grid_of(fw ? fwd : bwd), 256, 0, args);
    } else {
      void* args[] = {&ctrl, &nn, &kk, &ns, &sg, &rp, &cl, &lu, &inv, &srcp, &outp, &tk};
      launch(c, fw ? fwd : bwd, grid_of(fw ? fwd : bwd), 256, 0, args);
    }
  }
}

// Z = M^-1 R on device (ctrl-gated inside the solver loop); returns the
// FlopCounter increment.  r and z must not alias.
inline uint64_t precond_apply_dev(bkg_ctx* c, bkg_matrix* a, int kind, int k, const double* r,
                                  double* z, const Ctrl* ctrl) {
  const int64_t n = (int64_t)a->n;
  int64_t tot = n * k;
  if (kind == BKG_PRECOND_IDENTITY || (kind == BKG_PRECOND_ILU0 && k > 64)) {
    void* args[] = {&ctrl, &tot, &r, &z};
    launch(c, (const void*)&k_copy_ctrl, elem_grid(c, tot), 256, 0, args);
  }
  if (kind == BKG_PRECOND_IDENTITY) return 0;
  precond_ready(c, a, kind);
  if (kind == BKG_PRECOND_JACOBI) {
    const double* inv = a->inv_diag.ptr;
    int kk = k;
    int64_t nn = n;
    void* args[] = {&ctrl, &nn, &kk, &inv, &r, &z};
    launch(c, (const void*)&k_jacobi_apply, elem_grid(c, tot), 256, 0, args);
    return precond_flops(a, kind, k);
  }
  if (k <= 64) {
    a->ilu_y.ensure((size_t)n * k);
    ilu_apply_sf(c, a, k, r, a->ilu_y.ptr, z, ctrl);
    return precond_flops(a, kind, k);
  }
  const int64_t* rp = a->rowptr.ptr;
  const int32_t* cl = a->cols.ptr;
  const double* lu = a->lu.ptr;
  const double* inv = a->inv_diag.ptr;
  int kk = k;
  for (size_t l = 0; l + 1 < a->level_ptr_fwd.size(); ++l) {
    const int32_t* rows = a->level_rows.ptr + a->level_ptr_fwd[l];
    int cnt = (int)(a->level_ptr_fwd[l + 1] - a->level_ptr_fwd[l]);
    if (!cnt) continue;
    void* args[] = {&ctrl, &rows, &cnt, &kk, &rp, &cl, &lu, &z};
    launch(c, (const void*)&k_ilu_fwd_level, elem_grid(c, (int64_t)cnt * k), 256, 0, args);
  }
  for (size_t l = 0; l + 1 < a->level_ptr_bwd.size(); ++l) {
    const int32_t* rows = a->level_rows_bwd.ptr + a->level_ptr_bwd[l];
    int cnt = (int)(a->level_ptr_bwd[l + 1] - a->level_ptr_bwd[l]);
    if (!cnt) continue;
    void* args[] = {&ctrl, &rows, &cnt, &kk, &rp, &cl, &lu, &inv, &z};
    launch(c, (const void*)&k_ilu_bwd_level, elem_grid(c, (int64_t)cnt * k), 256, 0, args);
  }
  return precond_flops(a, kind, k);
}

}  // namespace bkg
