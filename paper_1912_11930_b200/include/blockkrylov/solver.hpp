// blockkrylov/solver.hpp — drop-in for bcg_solve and its report types
// (proj/include/blockkrylov/solver.hpp:21-216).  The whole iteration loop
// runs device-resident behind bkg_solve; this header only validates
// arguments (same exceptions as the reference), marshals the observer and
// unpacks the report.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "bkg.h"
#include "blockkrylov/block_vector.hpp"
#include "blockkrylov/device.hpp"
#include "blockkrylov/errors.hpp"
#include "blockkrylov/kernels.hpp"
#include "blockkrylov/preconditioners.hpp"
#include "blockkrylov/sparse_matrix.hpp"
#include "blockkrylov/subalgebra.hpp"

namespace blockkrylov {

struct SolveOptions {
  double tol = 1e-8;
  std::size_t max_iter = 0;
  bool record_history = false;
  std::function<void(std::size_t, const BlockVector&, const BlockVector&)> on_iterate;
  /// Extension: fill SolveReport::seconds with device time per kernel class
  /// (bkg.h time_kernels; the reference always wall-clocks its kernels).
  bool time_kernels = false;
};

struct BreakdownInfo {
  std::size_t iteration;
  std::size_t block_index;
};

struct KernelSeconds {
  double bdot = 0.0, baxpy = 0.0, bop = 0.0, precond = 0.0;
};

struct SolveReport {
  std::size_t iterations = 0;
  bool converged = false;
  std::vector<std::vector<double>> defect_history;
  FlopCounter flops;
  std::optional<BreakdownInfo> breakdown;
  std::vector<double> final_defect_norms;
  KernelSeconds seconds;
  double loop_seconds = 0.0;  // device time of the iteration loop (extension)
};

struct SolveResult {
  BlockVector x;
  SolveReport report;
};

namespace detail {
struct ObserverBridge {
  const SolveOptions* opts;
  BlockVector x, r;
  static void call(uint64_t it, const double* xp, const double* rp, uint64_t n, uint64_t k,
                   void* user) {
    auto* self = static_cast<ObserverBridge*>(user);
    if (self->x.rows() != n || self->x.cols() != k) {
      self->x = BlockVector(n, k);
      self->r = BlockVector(n, k);
    }
    std::copy(xp, xp + n * k, self->x.data());
    std::copy(rp, rp + n * k, self->r.data());
    self->opts->on_iterate(static_cast<std::size_t>(it), self->x, self->r);
  }
};
}  // namespace detail

/// Preconditioned Block CG, stabilised variant (solver.hpp:106-209).
inline SolveResult bcg_solve(const SparseMatrix& a, const BlockVector& b, const BlockVector& x0,
                             const Preconditioner& m, const SubalgebraConfig& cfg,
                             const SolveOptions& opts = {}) {
  if (a.n() != b.rows())
    throw DimensionError("bcg_solve: matrix dimension " + std::to_string(a.n()) +
                         " does not match right hand side rows " + std::to_string(b.rows()));
  if (b.cols() != cfg.k())
    throw DimensionError("bcg_solve: right hand side has k=" + std::to_string(b.cols()) +
                         " but configuration expects k=" + std::to_string(cfg.k()));
  if (x0.rows() != b.rows() || x0.cols() != b.cols())
    throw DimensionError("bcg_solve: initial guess shape does not match right hand side");
  if (m.n() != a.n())
    throw DimensionError("bcg_solve: preconditioner dimension does not match matrix");
  if (!(opts.tol > 0.0)) throw ConfigError("bcg_solve: tol must be positive");

  const std::size_t n = b.rows(), k = b.cols();
  SolveResult res{BlockVector(n, k), {}};
  res.report.final_defect_norms.assign(k, 0.0);
  detail::ObserverBridge bridge{&opts, {}, {}};
  bkg_solve_options o{};
  o.tol = opts.tol;
  o.max_iter = opts.max_iter;
  o.record_history = opts.record_history ? 1 : 0;
  o.precond = static_cast<int32_t>(m.kind());
  o.time_kernels = opts.time_kernels ? 1 : 0;
  if (opts.on_iterate) {
    o.on_iterate = &detail::ObserverBridge::call;
    o.user = &bridge;
  }
  bkg_report rep{};
  detail::check(bkg_solve(gpu::context(), a.device(), cfg.k(), cfg.p(), cfg.abi_mode(), b.data(),
                          x0.data(), &o, res.x.data(), nullptr, 0,
                          res.report.final_defect_norms.data(), &rep));
  SolveReport& r = res.report;
  r.iterations = rep.iterations;
  r.converged = rep.converged != 0;
  r.flops = {rep.flops_bdot, rep.flops_baxpy, rep.flops_bop, rep.flops_precond};
  r.seconds = {rep.seconds_bdot, rep.seconds_baxpy, rep.seconds_bop, rep.seconds_precond};
  r.loop_seconds = rep.loop_seconds;
  if (rep.breakdown) r.breakdown = BreakdownInfo{rep.breakdown_iteration, rep.breakdown_block};
  if (opts.record_history) {  // sized from the rows the solve produced, not max_iter
    const std::size_t rows = rep.history_rows;
    std::vector<double> hist(rows * k);
    uint64_t got = 0;
    detail::check(bkg_solve_history(gpu::context(), hist.data(), rows, &got));
    for (std::size_t i = 0; i < rows && i < got; ++i)
      r.defect_history.emplace_back(hist.begin() + i * k, hist.begin() + (i + 1) * k);
  }
  return res;
}

/// X0 = 0 overload (solver.hpp:212-216).
inline SolveResult bcg_solve(const SparseMatrix& a, const BlockVector& b, const Preconditioner& m,
                             const SubalgebraConfig& cfg, const SolveOptions& opts = {}) {
  return bcg_solve(a, b, BlockVector(b.rows(), b.cols()), m, cfg, opts);
}

}  // namespace blockkrylov
