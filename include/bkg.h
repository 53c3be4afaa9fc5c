/*
 * bkg.h — C ABI of the B200-native Block-CG hot path (libbkgpu.so).
 *
 * This is the drop-in boundary for the reference's header-only C++ API
 * (namespace blockkrylov, /root/reference/proj/include/blockkrylov).  Each
 * entry point names the reference interface it replaces.  Plain pointers and
 * sizes only: every *host* pointer argument is ordinary (pageable or pinned)
 * host memory; the library owns all device memory.  No exceptions cross the
 * ABI: every call returns a bkg_status and bkg_last_error() holds the
 * message of the last failing call on the calling thread.
 *
 * Numerics: every context runs in one of two modes.
 *   BKG_NUMERICS_EXACT — reproduces the reference's operation order and
 *     rounding (unfused mul/add, row-ordered Gram/norm chains), so results are
 *     bit-identical to the reference CPU build (-O3 -ffp-contract=off).
 *   BKG_NUMERICS_FAST (default) — fused sm_100a kernels (FMA, deterministic
 *     two-stage grid reductions).  Run-to-run bit-reproducible on a given
 *     GPU/grid; differs from the reference only by summation order.
 * There is no CPU fallback: without a CUDA device every compute call fails
 * with BKG_CUDA.
 */
#ifndef BKG_H
#define BKG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BKG_OK = 0,
  BKG_DIMENSION = 1, /* blockkrylov::DimensionError (errors.hpp:13-16)        */
  BKG_CONFIG = 2,    /* blockkrylov::ConfigError    (errors.hpp:19-22)        */
  BKG_BREAKDOWN = 3, /* blockkrylov::BreakdownError (errors.hpp:31-40)        */
  BKG_CUDA = 4,      /* device / driver failure (no reference counterpart)    */
  BKG_NCCL = 5,      /* collective failure (multi-GPU only)                   */
  BKG_FACTORIZATION = 6, /* blockkrylov::FactorizationError (errors.hpp:43-52) */
  BKG_INTERNAL = 7
} bkg_status;

/* SubalgebraMode (subalgebra.hpp:19) */
enum { BKG_HYBRID = 0, BKG_GLOBAL = 1 };
/* PreconditionerKind (preconditioners.hpp:317) */
enum { BKG_PRECOND_IDENTITY = 0, BKG_PRECOND_JACOBI = 1, BKG_PRECOND_ILU0 = 2 };
enum { BKG_NUMERICS_FAST = 0, BKG_NUMERICS_EXACT = 1 };

typedef struct bkg_ctx bkg_ctx;
typedef struct bkg_matrix bkg_matrix;
typedef struct bkg_solver bkg_solver;

/* ---- context ---------------------------------------------------------- */
const char* bkg_last_error(void);
const char* bkg_version(void);
int bkg_device_count(int* count);
int bkg_ctx_create(int device, bkg_ctx** out);
int bkg_ctx_destroy(bkg_ctx* ctx);
int bkg_ctx_set_numerics(bkg_ctx* ctx, int numerics);
int bkg_ctx_get_numerics(const bkg_ctx* ctx, int* numerics);
/* The cudaStream_t every launch of ctx is queued on (for event timing). */
int bkg_ctx_stream(const bkg_ctx* ctx, void** stream);
/* Number of kernels this library launched on ctx so far (evidence counter). */
int bkg_ctx_launch_count(const bkg_ctx* ctx, uint64_t* launches);

/* ---- sparse operator (SparseMatrix, sparse_matrix.hpp:27-131) ----------- */
/* Uploads a CSR matrix with the reference's size_t (uint64) offsets/columns.
 * Structure is validated on the host (sparse_matrix.hpp:89-105); value
 * symmetry is the host API's job (the SparseMatrix constructor).          */
int bkg_matrix_create(bkg_ctx* ctx, uint64_t n, const uint64_t* row_offsets,
                      const uint64_t* col_indices, const double* values, bkg_matrix** out);
int bkg_matrix_destroy(bkg_matrix* m);
int bkg_matrix_info(const bkg_matrix* m, uint64_t* n, uint64_t* nnz);

/* ---- kernels (kernels.hpp) ---------------------------------------------- */
/* BDOT   kernels.hpp:59-88.  out: block_count*p*p doubles, row-major blocks. */
int bkg_bdot(bkg_ctx* ctx, uint64_t n, uint64_t k, uint64_t p, int mode, const double* x,
             const double* y, double* out, uint64_t* flops_bdot /* nullable, += */);
/* BAXPY  kernels.hpp:94-125.  x <- x + y * embed(gamma).                     */
int bkg_baxpy(bkg_ctx* ctx, uint64_t n, uint64_t k, uint64_t p, int mode, double* x,
              const double* y, const double* gamma, uint64_t* flops_baxpy);
/* BOP    kernels.hpp:129-164.  y <- A x.                                      */
int bkg_bop(bkg_ctx* ctx, const bkg_matrix* a, uint64_t k, const double* x, double* y,
            uint64_t* flops_bop);
/* BSOLVE kernels.hpp:166-240.  On BKG_BREAKDOWN *bad_block holds the first
 * singular block (BreakdownError::block_index).                             */
int bkg_bsolve(bkg_ctx* ctx, uint64_t k, uint64_t p, int mode, const double* gamma,
               const double* delta, double* out, uint64_t* bad_block);
/* column_norms  block_vector.hpp:59-70.  out: k doubles.                     */
int bkg_column_norms(bkg_ctx* ctx, uint64_t n, uint64_t k, const double* x, double* out);
/* Preconditioner::apply  preconditioners.hpp:73-129 (identity / Jacobi /
 * ILU(0) factored on device from `a`; ilu0_factor preconditioners.hpp:153-196). */
int bkg_precond_apply(bkg_ctx* ctx, const bkg_matrix* a, int precond, uint64_t k,
                      const double* r, double* z, uint64_t* flops_precond);

/* Factor / validate a preconditioner for `a` on the device (Jacobi: diagonal
 * > 0, preconditioners.hpp:48-59; ILU(0): ilu0_factor :153-196).  On
 * BKG_FACTORIZATION *bad_row is the FactorizationError row.                */
int bkg_precond_setup(bkg_ctx* ctx, bkg_matrix* a, int precond, int64_t* bad_row);

/* ---- solver (solver.hpp:21-216) ----------------------------------------- */
/* SolveReport (solver.hpp:48-59) flattened.  defect_history is returned via
 * the caller's buffer (history_cap rows of k doubles).                      */
typedef struct {
  uint64_t iterations;
  int32_t converged;
  int32_t breakdown; /* 1 when report.breakdown has a value */
  uint64_t breakdown_iteration;
  uint64_t breakdown_block;
  uint64_t flops_bdot, flops_baxpy, flops_bop, flops_precond; /* FlopCounter   */
  double seconds_bdot, seconds_baxpy, seconds_bop, seconds_precond; /* KernelSeconds */
  uint64_t history_rows; /* rows produced (may exceed history_cap)          */
  double loop_seconds;   /* device time of the iteration loop (CUDA events)  */
} bkg_report;

/* SolveOptions::on_iterate (solver.hpp:29-31): x and r are HOST copies of
 * X^i, R^i (n*k row-major), valid during the call only.  Setting it makes the
 * loop copy X and R back every iteration (the reference semantics).        */
typedef void (*bkg_iterate_fn)(uint64_t iteration, const double* x, const double* r,
                               uint64_t n, uint64_t k, void* user);

typedef struct {
  double tol;          /* SolveOptions::tol       (solver.hpp:24)   */
  uint64_t max_iter;   /* SolveOptions::max_iter  (0 -> 10 n)       */
  int32_t record_history;
  int32_t precond;     /* BKG_PRECOND_*                               */
  bkg_iterate_fn on_iterate; /* nullable */
  void* user;
  /* Per-kernel-class device seconds into bkg_report.seconds_* (KernelSeconds,
   * solver.hpp:41-46): the loop runs launch by launch with CUDA events at the
   * class boundaries instead of as a captured graph.  Fast mode times its
   * fused kernels: K1 (SpMM + alpha) as bop, K2 + K3 as baxpy; their Grams
   * are fused, so seconds_bdot stays 0.  0: not timed (all zeros).         */
  int32_t time_kernels;
} bkg_solve_options;

/* bcg_solve (solver.hpp:106-209, X0 = 0 overload :212-216 when x0 == NULL).
 * Host buffers in, host buffers out; breakdown is reported in *rep, not as a
 * status (solver.hpp:191-194).                                              */
int bkg_solve(bkg_ctx* ctx, const bkg_matrix* a, uint64_t k, uint64_t p, int mode,
              const double* b, const double* x0, const bkg_solve_options* opts, double* x_out,
              double* history, uint64_t history_cap, double* final_norms, bkg_report* rep);

/* Defect history of the context's last bkg_solve (rows x k doubles): the
 * reference grows defect_history one row per iteration (solver.hpp:146,198),
 * so callers size their buffer after the solve from *rows instead of from
 * max_iter.  Copies min(cap, rows) rows; history may be NULL to query.      */
int bkg_solve_history(bkg_ctx* ctx, double* history, uint64_t cap, uint64_t* rows);

/* Which K1 (SpMM + alpha Gram) the context's last bkg_solve ran: -1 exact /
 * unfused kernels, 0 k1_wide (sliced ELL), 1 k1_line (line-window sliced
 * ELL), 2 k1_stage (TMA-staged row blocks), 3 the whole loop in the
 * persistent cooperative kernel for small systems (k_resident), 4 k1_grid /
 * k1_grid2 (grid stencils from TMA-tiled operand planes / lines).  Tests
 * assert the headline configs run the kernel the bench measures.            */
int bkg_solve_k1_variant(bkg_ctx* ctx, int* variant);

/* ---- device-resident solver (bench / repeated solves) ------------------- */
/* Keeps A, B, X and the work block vectors resident in HBM.                */
int bkg_solver_create(bkg_ctx* ctx, const bkg_matrix* a, uint64_t k, uint64_t p, int mode,
                      bkg_solver** out);
int bkg_solver_destroy(bkg_solver* s);
int bkg_solver_set_rhs(bkg_solver* s, const double* b_host);
/* Runs a whole solve from X0 = 0 on the resident B.  Host is touched only
 * every `chunk` iterations to read the stop flag.                          */
int bkg_solver_run(bkg_solver* s, double tol, uint64_t max_iter, int record_history,
                   bkg_report* rep);
int bkg_solver_get_x(bkg_solver* s, double* x_host);
int bkg_solver_history(bkg_solver* s, double* history, uint64_t cap, uint64_t* rows);
/* K1 variant of a resident solver (same codes as bkg_solve_k1_variant).     */
int bkg_solver_k1_variant(const bkg_solver* s, int* variant);
/* Device time (ms, CUDA events on the solver stream) of each fused kernel
 * class averaged over `iterations` iterations of an untimed profiling pass:
 * out_ms[0]=SpMM+Gram (K1), [1]=update+Gram (K2), [2]=P update (K3),
 * [3]=whole iteration.  Launches are not graph-captured in this pass.      */
int bkg_solver_profile(bkg_solver* s, uint64_t iterations, double* out_ms);
/* Test hook: set up a solve from X0 = 0 and run only the first SpMM+Gram
 * step (K1); returns Q = A P^1 (n*k) and [lambda^1 | rho_prev^1] (2*cs).   */
int bkg_solver_debug_first_step(bkg_solver* s, double* q_out, double* coef_out);
/* Algorithmic bytes one launch of each fused kernel class must move
 * (DESIGN.md §Roofline): out[0..2] as above, out[3] = per iteration.       */
int bkg_solver_kernel_bytes(const bkg_solver* s, double* out);

/* ---- row-partitioned solver (multi-GPU) --------------------- */
/* Rows are split into contiguous blocks ("parts"); each part keeps its rows
 * of X, R, Q and a ghost-extended P.  Per iteration: halo exchange of P,
 * SpMM + local Gram partials, allreduce of [alpha|rho_prev] and
 * [rho|col norms^2], replicated p x p solves.  Fast numerics only.         */
typedef struct bkg_psolver bkg_psolver;
/* Halo plan for nparts contiguous row blocks row_begin[0..nparts]: part r
 * needs operand rows [need_lo[r], need_hi[r]).  Writes `count` copies
 * (dst, src, first row, rows) into out (4 int64 each, up to cap).          */
int bkg_halo_plan(int nparts, const int64_t* row_begin, const int64_t* need_lo,
                  const int64_t* need_hi, int64_t* out, uint64_t cap, uint64_t* count);
/* Work plan of the grid-stencil K1 (k1_grid / k1_grid2) for an
 * nx x ny x nz grid (nz = 1: 2-D), k right-hand sides, sm_count SMs: pure host
 * logic, no device needed.  Rows produced are planes (2-D: lines) [zbeg, zend)
 * of a part whose plane 0 is plane zoff of an operand tensor of nzt planes
 * (one solver: 0, nz, 0, nz).  out (12 values): tiles_x, tiles_y, planes per
 * item, items per (tile, slice), slices, items, CTAs, first / last existing
 * tensor plane in part coordinates, plane stride between items, pacing segment
 * (0: off), pacing lead.                                                    */
int bkg_grid_plan(int64_t nx, int64_t ny, int64_t nz, uint64_t k, int sm_count, int zbeg, int zend,
                  int zoff, int nzt, int64_t* out);
/* NCCL unique id (128 bytes) for bkg_psolver_create_nccl, made on rank 0.  */
int bkg_nccl_unique_id(void* id_out);
/* All parts on this context's device (single-GPU emulation of nparts ranks;
 * halo = device copies, allreduce = fixed-order sum).  Global CSR in.      */
int bkg_psolver_create_virtual(bkg_ctx* ctx, uint64_t n, const uint64_t* row_offsets,
                               const uint64_t* cols, const double* vals, int nparts, uint64_t k,
                               uint64_t p, int mode, bkg_psolver** out);
/* One part per process (rank), NCCL over NVLink.  local_row_offsets has
 * row_end-row_begin+1 entries starting at 0; cols are GLOBAL indices.      */
int bkg_psolver_create_nccl(bkg_ctx* ctx, uint64_t n_global, uint64_t row_begin,
                            uint64_t row_end, const uint64_t* local_row_offsets,
                            const uint64_t* cols, const double* vals, uint64_t k, uint64_t p,
                            int mode, int rank, int nranks, const void* nccl_id,
                            bkg_psolver** out);
/* Same, with this rank's rows [row_begin, row_end) of a stencil matrix
 * (kinds and seeds of bkg_matrix_generate) generated on its own device: no
 * host CSR, no global assembly (C5 at 384^3: 6.2 GB of CSR, 29 GB per block
 * vector).                                                                  */
int bkg_psolver_create_nccl_generated(bkg_ctx* ctx, int kind, uint64_t nx, uint64_t ny,
                                      uint64_t nz, uint64_t seed, double contrast,
                                      uint64_t row_begin, uint64_t row_end, uint64_t k,
                                      uint64_t p, int mode, int rank, int nranks,
                                      const void* nccl_id, bkg_psolver** out);
/* Fill each part's B with its rows of the generated block (distribution as
 * bkg_solver_generate_rhs); bkg_psolver_get_rhs reads it back (virtual:
 * global n*k; NCCL: this rank's rows).                                      */
int bkg_psolver_generate_rhs(bkg_psolver* s, int distribution, uint64_t seed);
int bkg_psolver_get_rhs(bkg_psolver* s, double* b);
/* Part `part` (virtual: 0..nparts-1; NCCL: 0 = this rank): out[0] = K1
 * variant (bkg_solve_k1_variant codes), out[1] / out[2] = k1_stage blocks
 * launched before / after the halo (interior / boundary), out[3] / out[4] =
 * the part's global rows [r0, r1), out[5] = row slots per k1_stage block,
 * out[6..8] = its grid box bx, by, bz (0: consecutive rows).  out: 9 values. */
int bkg_psolver_part_info(const bkg_psolver* s, int part, int64_t* out);
int bkg_psolver_destroy(bkg_psolver* s);
/* virtual: global B (n*k); NCCL: this rank's rows.                         */
int bkg_psolver_set_rhs(bkg_psolver* s, const double* b);
int bkg_psolver_run(bkg_psolver* s, double tol, uint64_t max_iter, int record_history,
                    double* final_norms /* nullable, k */, bkg_report* rep);
int bkg_psolver_get_x(bkg_psolver* s, double* x);
int bkg_psolver_history(bkg_psolver* s, double* history, uint64_t cap, uint64_t* rows);

/* ---- problem generators (problems.hpp + frozen new generators) ---------- */
/* kinds: 0 poisson2d constant, 1 poisson2d log-uniform(seed, contrast),
 * 2 lognormal 2D diffusion (seed), 3 3D 7-point, 4 3D 27-point.            */
int bkg_stencil_size(int kind, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t* n,
                     uint64_t* nnz);
int bkg_stencil_fill(int kind, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed,
                     double contrast, uint64_t* row_offsets, uint64_t* cols, double* vals);
/* random_block_rhs (problems.hpp:128-134) and the frozen N(0,1) stream.   */
int bkg_random_block_rhs(uint64_t n, uint64_t k, uint64_t seed, double* out);
int bkg_normal_block_rhs(uint64_t n, uint64_t k, uint64_t seed, double* out);

/* Device-side generation (csrc/generate.cu).  The stencil
 * is assembled straight into a device matrix on ctx (bit-identical to
 * bkg_stencil_fill); bkg_matrix_download copies any device matrix back.
 * bkg_solver_generate_rhs fills the resident B: distribution 0 =
 * random_block_rhs (bit-identical), 1 = the N(0,1) stream (Box-Muller with
 * CUDA libm: within a few ulp of bkg_normal_block_rhs).                     */
int bkg_matrix_generate(bkg_ctx* ctx, int kind, uint64_t nx, uint64_t ny, uint64_t nz,
                        uint64_t seed, double contrast, bkg_matrix** out);
int bkg_matrix_download(const bkg_matrix* m, uint64_t* row_offsets, uint64_t* cols,
                        double* vals);
int bkg_solver_generate_rhs(bkg_solver* s, int distribution, uint64_t seed);
int bkg_solver_get_rhs(bkg_solver* s, double* b_host); /* the resident B    */

#ifdef __cplusplus
}
#endif
#endif
