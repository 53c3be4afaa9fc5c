// blockkrylov/kernels.hpp — drop-in for BDOT / BAXPY / BOP / BSOLVE and
// FlopCounter (proj/include/blockkrylov/kernels.hpp:22-240).  Shape checks
// and exceptions happen here on the host, before any launch; the arithmetic
// runs in the sm_100a kernels behind the C ABI (include/bkg.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "bkg.h"
#include "blockkrylov/block_vector.hpp"
#include "blockkrylov/device.hpp"
#include "blockkrylov/errors.hpp"
#include "blockkrylov/sparse_matrix.hpp"
#include "blockkrylov/subalgebra.hpp"

namespace blockkrylov {

struct FlopCounter {
  std::uint64_t multiply_adds_bdot = 0;
  std::uint64_t multiply_adds_baxpy = 0;
  std::uint64_t multiply_adds_bop = 0;
  std::uint64_t multiply_adds_precond = 0;
  std::uint64_t total() const noexcept {
    return multiply_adds_bdot + multiply_adds_baxpy + multiply_adds_bop + multiply_adds_precond;
  }
};

namespace detail {
inline void require_same_shape(const BlockVector& x, const BlockVector& y, const char* kernel) {
  if (x.rows() != y.rows() || x.cols() != y.cols())
    throw DimensionError(std::string(kernel) + ": block vectors have shapes " +
                         std::to_string(x.rows()) + "x" + std::to_string(x.cols()) + " and " +
                         std::to_string(y.rows()) + "x" + std::to_string(y.cols()));
}
inline void require_config_cols(const BlockVector& x, const SubalgebraConfig& cfg,
                                const char* kernel) {
  if (x.cols() != cfg.k())
    throw DimensionError(std::string(kernel) + ": block vector has k=" + std::to_string(x.cols()) +
                         " but configuration expects k=" + std::to_string(cfg.k()));
}
}  // namespace detail

/// BDOT <<X, Y>> in the configured subalgebra (kernels.hpp:59-88).
inline BlockCoefficient bdot(const BlockVector& x, const BlockVector& y,
                             const SubalgebraConfig& cfg, FlopCounter* flops = nullptr) {
  detail::require_same_shape(x, y, "bdot");
  detail::require_config_cols(x, cfg, "bdot");
  BlockCoefficient out(cfg);
  std::uint64_t f = 0;
  detail::check(bkg_bdot(gpu::context(), x.rows(), cfg.k(), cfg.p(), cfg.abi_mode(), x.data(),
                         y.data(), out.data(), &f));
  if (flops) flops->multiply_adds_bdot += f;
  return out;
}

/// BAXPY X <- X + Y embed(gamma) (kernels.hpp:94-125).
inline void baxpy(BlockVector& x, const BlockVector& y, const BlockCoefficient& gamma,
                  FlopCounter* flops = nullptr) {
  detail::require_same_shape(x, y, "baxpy");
  detail::require_config_cols(x, gamma.config(), "baxpy");
  if (&x == &y) throw DimensionError("baxpy: X and Y must be distinct");
  const SubalgebraConfig& cfg = gamma.config();
  std::uint64_t f = 0;
  detail::check(bkg_baxpy(gpu::context(), x.rows(), cfg.k(), cfg.p(), cfg.abi_mode(), x.data(),
                          y.data(), gamma.data(), &f));
  if (flops) flops->multiply_adds_baxpy += f;
}

/// BOP Y = A X (kernels.hpp:129-157).
inline void bop(const SparseMatrix& a, const BlockVector& x, BlockVector& y,
                FlopCounter* flops = nullptr) {
  if (a.n() != x.rows())
    throw DimensionError("bop: matrix is " + std::to_string(a.n()) +
                         "-dimensional but block vector has " + std::to_string(x.rows()) + " rows");
  if (y.rows() != x.rows() || y.cols() != x.cols()) y = BlockVector(x.rows(), x.cols());
  if (&x == &y) throw DimensionError("bop: X and Y must be distinct");
  std::uint64_t f = 0;
  detail::check(bkg_bop(gpu::context(), a.device(), x.cols(), x.data(), y.data(), &f));
  if (flops) flops->multiply_adds_bop += f;
}

inline BlockVector bop(const SparseMatrix& a, const BlockVector& x, FlopCounter* flops = nullptr) {
  BlockVector y(x.rows(), x.cols());
  bop(a, x, y, flops);
  return y;
}

/// BSOLVE gamma^-1 delta blockwise (kernels.hpp:231-240): same LU, pivot rule
/// and 1e-14 breakdown test, on the device.
inline BlockCoefficient bsolve(const BlockCoefficient& gamma, const BlockCoefficient& delta) {
  if (!(gamma.config() == delta.config()))
    throw DimensionError("bsolve: gamma and delta use different subalgebra configurations");
  const SubalgebraConfig& cfg = gamma.config();
  BlockCoefficient out(cfg);
  std::uint64_t bad = 0;
  const int st = bkg_bsolve(gpu::context(), cfg.k(), cfg.p(), cfg.abi_mode(), gamma.data(),
                            delta.data(), out.data(), &bad);
  detail::check(st, static_cast<std::size_t>(bad));
  return out;
}

}  // namespace blockkrylov
