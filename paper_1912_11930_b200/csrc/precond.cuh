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

// Z = M^-1 R on device (ctrl-gated inside the solver loop); returns the
// FlopCounter increment.  r and z must not alias.
inline uint64_t precond_apply_dev(bkg_ctx* c, bkg_matrix* a, int kind, int k, const double* r,
                                  double* z, const Ctrl* ctrl) {
  const int64_t n = (int64_t)a->n;
  int64_t tot = n * k;
  if (kind == BKG_PRECOND_IDENTITY || kind == BKG_PRECOND_ILU0) {
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
