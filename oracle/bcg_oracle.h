/*
 * bcg_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, single-threaded, -ffp-contract=off) of the
 * reference blockkrylov hot path: BDOT / BAXPY / BOP / BSOLVE / column
 * norms / preconditioner apply / the stabilised Block-CG loop, plus the
 * input generators.  Every function cites the reference file:line it
 * restates.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * (paper_1912_11930_b200/) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks this restatement bit-for-bit
 * against (a) the reference's frozen RNG golden values
 * (proj/tests/test_problems.cpp:67-78) and (b) the reference itself compiled
 * from /root/reference into oracle/_ref/libbkref.so (oracle/Makefile), via
 * the committed fixtures in tests/golden/ (tests/golden/make_golden.py).
 */
#ifndef BCG_ORACLE_H
#define BCG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes shared with the product ABI (include/bkg.h). */
#define ORC_OK 0
#define ORC_DIMENSION 1
#define ORC_CONFIG 2
#define ORC_BREAKDOWN 3

/* Matrix kinds for orc_stencil_*. */
#define ORC_POISSON2D_CONST 0   /* problems.hpp:74-124 with PoissonSpec::constant            */
#define ORC_POISSON2D_LOGUNI 1  /* problems.hpp:74-124 with PoissonSpec::heterogeneous       */
#define ORC_DIFFUSION2D_LOGNORMAL 2 /* C3: cell coeff exp(N(0,1)), harmonic faces (new, frozen) */
#define ORC_LAPLACE3D_7PT 3     /* C2/C5: diag 6, off -1, Dirichlet eliminated (new, frozen) */
#define ORC_STENCIL3D_27PT 4    /* C4: centre 26, off -1, Dirichlet eliminated (new, frozen) */

/* Preconditioner kinds (preconditioners.hpp:317). */
#define ORC_PRECOND_IDENTITY 0
#define ORC_PRECOND_JACOBI 1
#define ORC_PRECOND_ILU0 2

typedef struct {
  uint64_t iterations;
  int32_t converged;
  int32_t breakdown; /* 1 when report.breakdown has a value */
  uint64_t breakdown_iteration;
  uint64_t breakdown_block;
  uint64_t flops_bdot, flops_baxpy, flops_bop, flops_precond;
  double seconds_bdot, seconds_baxpy, seconds_bop, seconds_precond;
  uint64_t history_rows; /* rows produced (may exceed the caller's capacity) */
} orc_report;

/* --- RNG + generators (problems.hpp) -------------------------------- */
uint64_t orc_rng_seed_state(uint64_t seed);
/* n draws of next_symmetric() from Xorshift64Star(seed). */
void orc_rng_symmetric(uint64_t seed, size_t count, double* out);
void orc_random_block_rhs(size_t n, size_t k, uint64_t seed, double* out);
void orc_normal_block_rhs(size_t n, size_t k, uint64_t seed, double* out);
size_t orc_stencil_rows(int kind, size_t nx, size_t ny, size_t nz);
size_t orc_stencil_nnz(int kind, size_t nx, size_t ny, size_t nz);
int orc_stencil_fill(int kind, size_t nx, size_t ny, size_t nz, uint64_t seed, double contrast,
                     uint64_t* rowptr, uint64_t* cols, double* vals);

/* --- kernels (kernels.hpp) ------------------------------------------- */
void orc_bdot(size_t n, size_t k, size_t p, int global, const double* x, const double* y,
              double* out);
void orc_baxpy(size_t n, size_t k, size_t p, int global, double* x, const double* y,
               const double* gamma);
void orc_bop(size_t n, const uint64_t* rowptr, const uint64_t* cols, const double* vals,
             size_t k, const double* x, double* y);
/* returns ORC_OK or ORC_BREAKDOWN (bad_block set) */
int orc_bsolve(size_t k, size_t p, int global, const double* gamma, const double* delta,
               double* out, uint64_t* bad_block);
void orc_column_norms(size_t n, size_t k, const double* x, double* out);

/* --- preconditioners (preconditioners.hpp) -------------------------- */
/* Builds the factor arrays for kind (jacobi: inv_diag only; ilu0: lu + inv_diag).
 * lu_vals may be NULL for identity/jacobi.  Returns ORC_OK or -1-row on a
 * FactorizationError at `row`. */
int64_t orc_precond_setup(int kind, size_t n, const uint64_t* rowptr, const uint64_t* cols,
                          const double* vals, double* inv_diag, double* lu_vals);
void orc_precond_apply(int kind, size_t n, const uint64_t* rowptr, const uint64_t* cols,
                       const double* inv_diag, const double* lu_vals, size_t k, const double* r,
                       double* z, uint64_t* flops);

/* --- solver (solver.hpp:106-216) ------------------------------------ */
int orc_bcg_solve(size_t n, const uint64_t* rowptr, const uint64_t* cols, const double* vals,
                  int precond_kind, size_t k, size_t p, int global, const double* b,
                  const double* x0 /* nullable: zero */, double tol, uint64_t max_iter,
                  int record_history, double* history, uint64_t history_cap_rows,
                  double* x_out, double* final_norms, orc_report* rep);

/* --- CPU baseline: `threads` independent solves of the same system, one
 * per thread, each capped at max_iter.  Returns wall seconds; *iterations is
 * the sum of the iteration counts. */
double orc_bench_solve(int threads, size_t n, const uint64_t* rowptr, const uint64_t* cols,
                       const double* vals, size_t k, size_t p, int global, const double* b,
                       double tol, uint64_t max_iter, uint64_t* iterations);

#ifdef __cplusplus
}
#endif
#endif
