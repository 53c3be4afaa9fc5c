// precond.cuh — Preconditioner::apply on device (preconditioners.hpp:73-129).
//
// identity: Z = R.  jacobi: Z = D^-1 R with D^-1 = 1/diag(A) computed on
// device (preconditioners.hpp:48-59).  Both are exact (one rounding per entry,
// same as the reference).  ILU(0) is rejected here until its level-scheduled
// sweeps land.
#pragma once

#include "common.cuh"

namespace bkg {

// inv_diag[r] = 1 / A(r,r); flag[0] = first row whose diagonal is not > 0.
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

__global__ void k_jacobi_apply(int64_t n, int k, const double* __restrict__ inv_diag,
                               const double* __restrict__ r, double* __restrict__ z) {
  const int64_t total = n * (int64_t)k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    z[idx] = __dmul_rn(inv_diag[idx / k], r[idx]);
}

int elem_grid(const bkg_ctx* c, int64_t total);
void launch(bkg_ctx* c, const void* fn, int grid, int block, size_t smem, void** args);

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
  BKG_REQUIRE(h == none, BKG_FACTORIZATION,
              "jacobi: diagonal entry " + std::to_string(h) + " is not strictly positive");
  a->precond_ready = BKG_PRECOND_JACOBI;
}

// Z = M^-1 R on device; returns the FlopCounter increment
// (preconditioners.hpp:91,124-125).
inline uint64_t precond_apply_dev(bkg_ctx* c, bkg_matrix* a, int kind, int k, const double* r,
                                  double* z, const Ctrl* ctrl) {
  (void)ctrl;
  const int64_t n = (int64_t)a->n;
  if (kind == BKG_PRECOND_IDENTITY) {
    BKG_CUDA_CHECK(cudaMemcpyAsync(z, r, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, c->stream));
    return 0;
  }
  if (kind == BKG_PRECOND_JACOBI) {
    jacobi_ready(c, a);
    const double* inv = a->inv_diag.ptr;
    int kk = k;
    int64_t nn = n;
    void* args[] = {&nn, &kk, &inv, &r, &z};
    launch(c, (const void*)&k_jacobi_apply, elem_grid(c, n * k), 256, 0, args);
    return (uint64_t)n * k;
  }
  throw Error(BKG_CONFIG, "ilu0: device ILU(0) sweeps are not available in this build");
}

}  // namespace bkg
