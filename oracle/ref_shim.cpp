// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference blockkrylov headers,
// compiled straight from /root/reference/proj/include by oracle/Makefile into
// oracle/_ref/libbkref.so.  Used (a) to pin the C restatement in
// oracle/bcg_oracle.c bit-for-bit, (b) to generate tests/golden fixtures and
// (c) as the `kind: "reference"` CPU baseline in bench.py.  Nothing here is a
// copy of reference source: it only #includes the reference headers.
#include <blockkrylov/blockkrylov.hpp>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

using namespace blockkrylov;

namespace {

SubalgebraConfig make_cfg(size_t k, size_t p, int global) {
  return SubalgebraConfig(k, p, global ? SubalgebraMode::global : SubalgebraMode::hybrid);
}

BlockVector to_bv(size_t n, size_t k, const double* d) {
  BlockVector v(n, k);
  std::memcpy(v.data(), d, n * k * sizeof(double));
  return v;
}

SparseMatrix to_csr(size_t n, const uint64_t* rowptr, const uint64_t* cols, const double* vals) {
  const size_t nnz = rowptr[n];
  return SparseMatrix(n, std::vector<std::size_t>(rowptr, rowptr + n + 1),
                      std::vector<std::size_t>(cols, cols + nnz),
                      std::vector<double>(vals, vals + nnz));
}

Preconditioner make_precond(int kind, const SparseMatrix& a) {
  if (kind == 1) return Preconditioner::jacobi(a);
  if (kind == 2) return ilu0_factor(a);
  return Preconditioner::identity(a.n());
}

struct Report {  // same layout as orc_report (bcg_oracle.h)
  uint64_t iterations;
  int32_t converged;
  int32_t breakdown;
  uint64_t breakdown_iteration;
  uint64_t breakdown_block;
  uint64_t flops_bdot, flops_baxpy, flops_bop, flops_precond;
  double seconds_bdot, seconds_baxpy, seconds_bop, seconds_precond;
  uint64_t history_rows;
};

}  // namespace

extern "C" {

void bkref_rng_symmetric(uint64_t seed, size_t count, double* out) {
  Xorshift64Star g(seed);
  for (size_t i = 0; i < count; ++i) out[i] = g.next_symmetric();
}

void bkref_random_block_rhs(size_t n, size_t k, uint64_t seed, double* out) {
  const BlockVector b = random_block_rhs(n, k, seed);
  std::memcpy(out, b.data(), n * k * sizeof(double));
}

// poisson2d (constant when contrast < 0, heterogeneous otherwise); returns nnz.
size_t bkref_poisson2d(size_t nx, size_t ny, uint64_t seed, double contrast, uint64_t* rowptr,
                       uint64_t* cols, double* vals) {
  const SparseMatrix a = contrast < 0 ? poisson2d(PoissonSpec::constant(nx, ny))
                                      : poisson2d(PoissonSpec::heterogeneous(nx, ny, seed, contrast));
  if (rowptr) {
    for (size_t i = 0; i <= a.n(); ++i) rowptr[i] = a.row_offsets()[i];
    for (size_t i = 0; i < a.nnz(); ++i) {
      cols[i] = a.col_indices()[i];
      vals[i] = a.values()[i];
    }
  }
  return a.nnz();
}

void bkref_bdot(size_t n, size_t k, size_t p, int global, const double* x, const double* y,
                double* out) {
  const SubalgebraConfig cfg = make_cfg(k, p, global);
  const BlockCoefficient g = bdot(to_bv(n, k, x), to_bv(n, k, y), cfg);
  for (size_t b = 0; b < g.block_count(); ++b)
    std::memcpy(out + b * p * p, g.block(b).data(), p * p * sizeof(double));
}

void bkref_baxpy(size_t n, size_t k, size_t p, int global, double* x, const double* y,
                 const double* gamma) {
  const SubalgebraConfig cfg = make_cfg(k, p, global);
  BlockCoefficient g(cfg);
  for (size_t b = 0; b < g.block_count(); ++b)
    std::memcpy(g.block(b).data(), gamma + b * p * p, p * p * sizeof(double));
  BlockVector xv = to_bv(n, k, x);
  baxpy(xv, to_bv(n, k, y), g);
  std::memcpy(x, xv.data(), n * k * sizeof(double));
}

void bkref_bop(size_t n, const uint64_t* rowptr, const uint64_t* cols, const double* vals,
               size_t k, const double* x, double* y) {
  const BlockVector out = bop(to_csr(n, rowptr, cols, vals), to_bv(n, k, x));
  std::memcpy(y, out.data(), n * k * sizeof(double));
}

int bkref_bsolve(size_t k, size_t p, int global, const double* gamma, const double* delta,
                 double* out, uint64_t* bad_block) {
  const SubalgebraConfig cfg = make_cfg(k, p, global);
  BlockCoefficient g(cfg), d(cfg);
  for (size_t b = 0; b < g.block_count(); ++b) {
    std::memcpy(g.block(b).data(), gamma + b * p * p, p * p * sizeof(double));
    std::memcpy(d.block(b).data(), delta + b * p * p, p * p * sizeof(double));
  }
  try {
    const BlockCoefficient r = bsolve(g, d);
    for (size_t b = 0; b < r.block_count(); ++b)
      std::memcpy(out + b * p * p, r.block(b).data(), p * p * sizeof(double));
    return 0;
  } catch (const BreakdownError& e) {
    if (bad_block) *bad_block = e.block_index();
    return 3;
  }
}

void bkref_column_norms(size_t n, size_t k, const double* x, double* out) {
  const std::vector<double> v = column_norms(to_bv(n, k, x));
  std::memcpy(out, v.data(), k * sizeof(double));
}

int bkref_bcg_solve(size_t n, const uint64_t* rowptr, const uint64_t* cols, const double* vals,
                    int precond_kind, size_t k, size_t p, int global, const double* b,
                    const double* x0, double tol, uint64_t max_iter, int record_history,
                    double* history, uint64_t history_cap, double* x_out, double* final_norms,
                    Report* rep) {
  const SparseMatrix a = to_csr(n, rowptr, cols, vals);
  const SubalgebraConfig cfg = make_cfg(k, p, global);
  SolveOptions opts;
  opts.tol = tol;
  opts.max_iter = max_iter;
  opts.record_history = record_history != 0;
  const Preconditioner m = make_precond(precond_kind, a);
  const BlockVector bv = to_bv(n, k, b);
  const SolveResult res = x0 ? bcg_solve(a, bv, to_bv(n, k, x0), m, cfg, opts)
                             : bcg_solve(a, bv, m, cfg, opts);
  std::memcpy(x_out, res.x.data(), n * k * sizeof(double));
  if (final_norms)
    std::memcpy(final_norms, res.report.final_defect_norms.data(), k * sizeof(double));
  std::memset(rep, 0, sizeof(*rep));
  rep->iterations = res.report.iterations;
  rep->converged = res.report.converged;
  rep->breakdown = res.report.breakdown.has_value();
  if (res.report.breakdown) {
    rep->breakdown_iteration = res.report.breakdown->iteration;
    rep->breakdown_block = res.report.breakdown->block_index;
  }
  rep->flops_bdot = res.report.flops.multiply_adds_bdot;
  rep->flops_baxpy = res.report.flops.multiply_adds_baxpy;
  rep->flops_bop = res.report.flops.multiply_adds_bop;
  rep->flops_precond = res.report.flops.multiply_adds_precond;
  rep->seconds_bdot = res.report.seconds.bdot;
  rep->seconds_baxpy = res.report.seconds.baxpy;
  rep->seconds_bop = res.report.seconds.bop;
  rep->seconds_precond = res.report.seconds.precond;
  rep->history_rows = res.report.defect_history.size();
  for (size_t i = 0; i < res.report.defect_history.size() && i < history_cap; ++i)
    std::memcpy(history + i * k, res.report.defect_history[i].data(), k * sizeof(double));
  return 0;
}

// CPU baseline: `threads` independent reference solves (one per thread) of the
// same system, each capped at max_iter.  Returns wall seconds of the solves.
double bkref_bench_solve(int threads, size_t n, const uint64_t* rowptr, const uint64_t* cols,
                         const double* vals, size_t k, size_t p, int global, const double* b,
                         double tol, uint64_t max_iter, uint64_t* iterations) {
  const SparseMatrix a = to_csr(n, rowptr, cols, vals);
  const SubalgebraConfig cfg = make_cfg(k, p, global);
  const BlockVector bv = to_bv(n, k, b);
  const Preconditioner m = Preconditioner::identity(n);
  SolveOptions opts;
  opts.tol = tol;
  opts.max_iter = max_iter;
  if (threads < 1) threads = 1;
  std::vector<uint64_t> its(threads, 0);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] { its[t] = bcg_solve(a, bv, m, cfg, opts).report.iterations; });
  for (auto& th : pool) th.join();
  const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  uint64_t total = 0;
  for (auto v : its) total += v;
  if (iterations) *iterations = total;
  return dt;
}

// CPU baseline with the loop isolated: `threads` concurrent reference solves
// of the same system, max_iter = iters, tol tiny.  The reference calls
// SolveOptions::on_iterate at i = 0 after its setup (solver.hpp:147) and after
// every iteration (:199); the observer holds every thread at i = 0 until all
// threads are there, so the window [release, last thread's i = iters] is
// `threads` x `iters` concurrent reference iterations -- no per-solve setup,
// no final residual.  Returns the window in seconds.
double bkref_bench_iterations(int threads, size_t n, const uint64_t* rowptr, const uint64_t* cols,
                              const double* vals, size_t k, size_t p, int global,
                              const double* b, uint64_t iters, uint64_t* iterations) {
  const SparseMatrix a = to_csr(n, rowptr, cols, vals);
  const SubalgebraConfig cfg = make_cfg(k, p, global);
  const BlockVector bv = to_bv(n, k, b);
  const Preconditioner m = Preconditioner::identity(n);
  if (threads < 1) threads = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  std::chrono::steady_clock::time_point start;
  std::vector<std::chrono::steady_clock::time_point> end(threads);
  std::vector<uint64_t> its(threads, 0);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      SolveOptions opts;
      opts.tol = 1e-300;
      opts.max_iter = iters;
      opts.on_iterate = [&, t](std::size_t i, const BlockVector&, const BlockVector&) {
        if (i == 0) {
          std::unique_lock<std::mutex> lk(mu);
          if (++arrived == threads) {
            start = std::chrono::steady_clock::now();
            cv.notify_all();
          } else {
            cv.wait(lk, [&] { return arrived == threads; });
          }
        }
        if (i == iters) end[t] = std::chrono::steady_clock::now();
      };
      its[t] = bcg_solve(a, bv, m, cfg, opts).report.iterations;
    });
  for (auto& th : pool) th.join();
  double dt = 0.0;
  uint64_t total = 0;
  for (int t = 0; t < threads; ++t) {
    dt = std::max(dt, std::chrono::duration<double>(end[t] - start).count());
    total += its[t];
  }
  if (iterations) *iterations = total;
  return dt;
}

// ---- host-side modules (perf_model.hpp, theory.hpp, text formats) -------
// out = {omega, beta, tau}; returns 0, or -1 on ConfigError.
int bkref_characteristics(int kernel, size_t n, size_t k, size_t p, size_t z, uint64_t* out) {
  try {
    const KernelCharacteristics c = characteristics(static_cast<Kernel>(kernel), n, k, p, z);
    out[0] = c.omega;
    out[1] = c.beta;
    out[2] = c.tau;
    return 0;
  } catch (const Error&) {
    return -1;
  }
}

// out = {t_comp, t_mem, t_reg, t}; *bound = Bound enum value.
int bkref_predict(int kernel, size_t n, size_t k, size_t p, size_t z, double peak, double mem,
                  double reg, double bps, double* out, int* bound) {
  try {
    const MachineProfile m{peak, mem, reg, bps};
    const Prediction pr = predict(characteristics(static_cast<Kernel>(kernel), n, k, p, z), m);
    out[0] = pr.t_comp;
    out[1] = pr.t_mem;
    out[2] = pr.t_reg;
    out[3] = pr.t;
    *bound = static_cast<int>(pr.bound);
    return 0;
  } catch (const Error&) {
    return -1;
  }
}

double bkref_rate(int global, size_t count, const double* ev, size_t p, size_t q) {
  const Spectrum s(std::vector<double>(ev, ev + count));
  return global ? rate_global(s, p, q) : rate_classical(s, p);
}

void bkref_spectrum_of(size_t n, const uint64_t* rowptr, const uint64_t* cols, const double* vals,
                       double* out) {
  const Spectrum s = spectrum_of(to_csr(n, rowptr, cols, vals));
  std::copy(s.values().begin(), s.values().end(), out);
}

void bkref_save_matrix_market(const char* path, size_t n, const uint64_t* rowptr,
                              const uint64_t* cols, const double* vals) {
  save_matrix_market(path, to_csr(n, rowptr, cols, vals));
}

void bkref_save_block_vector(const char* path, size_t n, size_t k, const double* x) {
  save_block_vector(path, to_bv(n, k, x));
}

// Reads a Matrix Market file and writes it back in the reference's canonical
// form (the read semantics: mirroring, duplicate summation, validation).
// Returns 0, 1 on IoError, 2 on another blockkrylov error.
int bkref_mm_roundtrip(const char* in, const char* out) {
  try {
    save_matrix_market(out, load_matrix_market(in));
    return 0;
  } catch (const IoError&) {
    return 1;
  } catch (const Error&) {
    return 2;
  }
}

int bkref_bv_roundtrip(const char* in, const char* out) {
  try {
    save_block_vector(out, load_block_vector(in));
    return 0;
  } catch (const IoError&) {
    return 1;
  } catch (const Error&) {
    return 2;
  }
}

}  // extern "C"
