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

// FWD: out = L^-1 src (unit lower); BWD: out = U^-1 src.  out must hold the
// sentinel everywhere on entry; src and out must not alias.
template <bool FWD>
__global__ void __launch_bounds__(256) k_ilu_sweep_sf(const Ctrl* ctrl, int64_t n, int k, int S,
                                                      const int64_t* __restrict__ rowptr,
                                                      const int32_t* __restrict__ cols,
                                                      const double* __restrict__ lu,
                                                      const double* __restrict__ inv_diag,
                                                      const double* __restrict__ src, double* out,
                                                      unsigned long long* ticket) {
  if (stopped(ctrl)) return;
  const int lane = threadIdx.x & 31;
  const int64_t nseg = (n + S - 1) / S;
  const bool c0 = lane < k, c1 = lane + 32 < k;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    const int64_t s = (int64_t)__shfl_sync(0xffffffffu, t, 0);
    if (s >= nseg) return;
    const int64_t first = FWD ? s * S : n - 1 - s * S;  // first row in processing order
    const int cnt = (int)(n - s * S < (int64_t)S ? n - s * S : (int64_t)S);
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
  // ILU multiply-add count per apply (preconditioners.hpp:123-125)
  uint64_t off = 0;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t i = rp[r]; i < rp[r + 1]; ++i)
      if (cl[i] != r) ++off;
  a->ilu_offdiag = off;
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

// Segment length of the sync-free sweeps (rows per ticket).
#ifndef BKG_ILU_SEG
#define BKG_ILU_SEG 128
#endif

// ILU(0) apply z = U^-1 L^-1 r with the sync-free sweeps (k <= 64); y is an
// n x k scratch for L^-1 r (the fused loop passes Q, free between K2 and K1).
inline void ilu_apply_sf(bkg_ctx* c, bkg_matrix* a, int k, const double* r, double* y, double* z,
                         const Ctrl* ctrl) {
  const int64_t n = (int64_t)a->n;
  const int S = BKG_ILU_SEG;
  const int64_t nseg = (n + S - 1) / S;
  a->ilu_state.ensure(2);
  int dev = 0, nsm = 0, per = 0;
  BKG_CUDA_CHECK(cudaGetDevice(&dev));
  BKG_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  BKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per, (const void*)&k_ilu_sweep_sf<true>, 256, 0));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * std::max(per, 1),
                                                               (nseg + 7) / 8));
  const int64_t* rp = a->rowptr.ptr;
  const int32_t* cl = a->cols.ptr;
  const double* lu = a->lu.ptr;
  const double* inv = a->inv_diag.ptr;
  unsigned long long* st = a->ilu_state.ptr;
  int64_t nn = n, tot = n * (int64_t)k;
  int kk = k, ss = S;
  {
    void* args[] = {&ctrl, &tot, &y, &z, &st};
    launch(c, (const void*)&k_ilu_fill, elem_grid(c, tot), 256, 0, args);
  }
  {
    const double* srcp = r;
    double* outp = y;
    unsigned long long* tk = st;
    void* args[] = {&ctrl, &nn, &kk, &ss, &rp, &cl, &lu, &inv, &srcp, &outp, &tk};
    launch(c, (const void*)&k_ilu_sweep_sf<true>, grid, 256, 0, args);
  }
  {
    const double* srcp = y;
    double* outp = z;
    unsigned long long* tk = st + 1;
    void* args[] = {&ctrl, &nn, &kk, &ss, &rp, &cl, &lu, &inv, &srcp, &outp, &tk};
    launch(c, (const void*)&k_ilu_sweep_sf<false>, grid, 256, 0, args);
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
