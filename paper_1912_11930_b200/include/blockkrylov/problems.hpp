// blockkrylov/problems.hpp — input generators: the reference's
// Xorshift64Star / PoissonSpec / poisson2d / random_block_rhs
// (proj/include/blockkrylov/problems.hpp:19-134) plus the frozen synthetic
// inputs of the BASELINE configs.  The matrix and block
// generators run in libbkgpu.so (bkg_stencil_fill, bkg_*_block_rhs).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "bkg.h"
#include "blockkrylov/block_vector.hpp"
#include "blockkrylov/errors.hpp"
#include "blockkrylov/sparse_matrix.hpp"

namespace blockkrylov {

/// xorshift64* with a splitmix64 seeding step (bit-identical stream).
class Xorshift64Star {
 public:
  explicit Xorshift64Star(std::uint64_t seed) {
    std::uint64_t z = seed + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    state_ = z ^ (z >> 31);
    if (state_ == 0) state_ = 0x9E3779B97F4A7C15ull;
  }
  std::uint64_t next() {
    state_ ^= state_ >> 12;
    state_ ^= state_ << 25;
    state_ ^= state_ >> 27;
    return state_ * 0x2545F4914F6CDD1Dull;
  }
  double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double next_symmetric() { return 2.0 * next_unit() - 1.0; }

 private:
  std::uint64_t state_;
};

struct PoissonSpec {
  std::size_t nx = 32;
  std::size_t ny = 32;
  enum class Coefficients { constant, log_uniform };
  Coefficients coefficients = Coefficients::constant;
  double contrast = 2.0;
  std::uint64_t seed = 0;

  static PoissonSpec constant(std::size_t nx, std::size_t ny) {
    return {nx, ny, Coefficients::constant, 0.0, 0};
  }
  static PoissonSpec heterogeneous(std::size_t nx, std::size_t ny, std::uint64_t seed,
                                   double contrast = 2.0) {
    return {nx, ny, Coefficients::log_uniform, contrast, seed};
  }
};

/// Stencil generator kinds of bkg_stencil_fill.
enum class StencilKind { poisson2d_constant = 0, poisson2d_log_uniform = 1,
                         diffusion2d_lognormal = 2, laplace3d_7pt = 3, stencil3d_27pt = 4 };

inline SparseMatrix stencil(StencilKind kind, std::size_t nx, std::size_t ny, std::size_t nz,
                            std::uint64_t seed = 0, double contrast = 2.0) {
  uint64_t n = 0, nnz = 0;
  detail::check(bkg_stencil_size(static_cast<int>(kind), nx, ny, nz, &n, &nnz));
  std::vector<std::size_t> off(n + 1), cols(nnz);
  std::vector<double> vals(nnz);
  const int st = bkg_stencil_fill(static_cast<int>(kind), nx, ny, nz, seed, contrast,
                                  reinterpret_cast<uint64_t*>(off.data()),
                                  reinterpret_cast<uint64_t*>(cols.data()), vals.data());
  if (st == BKG_CONFIG) throw ConfigError("stencil: grid must be at least 2 cells per axis");
  detail::check(st);
  return SparseMatrix(n, std::move(off), std::move(cols), std::move(vals));
}

/// problems.hpp:74-124: SPD 5-point heterogeneous Poisson matrix.
inline SparseMatrix poisson2d(const PoissonSpec& spec) {
  if (spec.nx < 2 || spec.ny < 2) throw ConfigError("poisson2d: grid must be at least 2 x 2 cells");
  if (spec.coefficients == PoissonSpec::Coefficients::log_uniform && !(spec.contrast >= 0.0))
    throw ConfigError("poisson2d: contrast exponent must be non-negative");
  return stencil(spec.coefficients == PoissonSpec::Coefficients::constant
                     ? StencilKind::poisson2d_constant
                     : StencilKind::poisson2d_log_uniform,
                 spec.nx, spec.ny, 1, spec.seed, spec.contrast);
}

/// problems.hpp:128-134: U(-1,1) entries, one stream, row-major.
inline BlockVector random_block_rhs(std::size_t n, std::size_t k, std::uint64_t seed) {
  BlockVector b(n, k);
  detail::check(bkg_random_block_rhs(n, k, seed, b.data()));
  return b;
}

/// Frozen N(0,1) block.
inline BlockVector normal_block_rhs(std::size_t n, std::size_t k, std::uint64_t seed) {
  BlockVector b(n, k);
  detail::check(bkg_normal_block_rhs(n, k, seed, b.data()));
  return b;
}

}  // namespace blockkrylov
