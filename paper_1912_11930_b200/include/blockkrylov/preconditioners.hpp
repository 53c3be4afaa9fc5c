// blockkrylov/preconditioners.hpp — drop-in for Preconditioner
// (proj/include/blockkrylov/preconditioners.hpp:66-147).  identity is a copy;
// Jacobi is applied on the device (bkg_precond_apply); the device solver loop
// currently runs M = I (Jacobi / ILU(0) in the loop are the
// next rows of the scope table).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <string_view>

#include "bkg.h"
#include "blockkrylov/block_vector.hpp"
#include "blockkrylov/device.hpp"
#include "blockkrylov/errors.hpp"
#include "blockkrylov/kernels.hpp"
#include "blockkrylov/sparse_matrix.hpp"

namespace blockkrylov {

enum class PreconditionerKind { identity, jacobi, ilu0 };

inline const char* to_string(PreconditionerKind k) {
  switch (k) {
    case PreconditionerKind::identity: return "identity";
    case PreconditionerKind::jacobi: return "jacobi";
    default: return "ilu0";
  }
}

inline PreconditionerKind parse_preconditioner_kind(std::string_view name) {
  if (name == "identity") return PreconditionerKind::identity;
  if (name == "jacobi") return PreconditionerKind::jacobi;
  if (name == "ilu0") return PreconditionerKind::ilu0;
  throw ConfigError("unknown preconditioner '" + std::string(name) +
                    "' (expected identity, jacobi or ilu0)");
}

class Preconditioner {
 public:
  static Preconditioner identity(std::size_t n) {
    Preconditioner m;
    m.n_ = n;
    return m;
  }
  static Preconditioner jacobi(const SparseMatrix& a) {
    for (std::size_t r = 0; r < a.n(); ++r)
      if (!(a.at(r, r) > 0.0))
        throw FactorizationError(r, "jacobi: diagonal entry " + std::to_string(r) +
                                        " is not strictly positive");
    Preconditioner m;
    m.kind_ = PreconditionerKind::jacobi;
    m.n_ = a.n();
    m.a_ = &a;
    return m;
  }

  /// ILU(0) factored on the device now (FactorizationError on a zero or
  /// missing pivot, preconditioners.hpp:153-196).
  static Preconditioner ilu0(const SparseMatrix& a) {
    int64_t bad = -1;
    const int st = bkg_precond_setup(gpu::context(), const_cast<bkg_matrix*>(a.device()),
                                     BKG_PRECOND_ILU0, &bad);
    detail::check(st, bad < 0 ? 0 : static_cast<std::size_t>(bad));
    Preconditioner m;
    m.kind_ = PreconditionerKind::ilu0;
    m.n_ = a.n();
    m.a_ = &a;
    return m;
  }

  PreconditionerKind kind() const noexcept { return kind_; }
  std::size_t n() const noexcept { return n_; }
  const SparseMatrix* matrix() const noexcept { return a_; }

  void apply(const BlockVector& r, BlockVector& z, FlopCounter* flops = nullptr) const {
    if (r.rows() != n_)
      throw DimensionError("preconditioner: expected " + std::to_string(n_) + " rows, got " +
                           std::to_string(r.rows()));
    if (z.rows() != r.rows() || z.cols() != r.cols()) z = BlockVector(r.rows(), r.cols());
    if (kind_ == PreconditionerKind::identity) {
      std::copy(r.data(), r.data() + r.size(), z.data());
      return;
    }
    std::uint64_t f = 0;
    detail::check(bkg_precond_apply(gpu::context(), a_->device(), static_cast<int>(kind_),
                                    r.cols(), r.data(), z.data(), &f));
    if (flops) flops->multiply_adds_precond += f;
  }

  BlockVector apply(const BlockVector& r, FlopCounter* flops = nullptr) const {
    BlockVector z(r.rows(), r.cols());
    apply(r, z, flops);
    return z;
  }

 private:
  Preconditioner() = default;
  PreconditionerKind kind_ = PreconditionerKind::identity;
  std::size_t n_ = 0;
  const SparseMatrix* a_ = nullptr;
};

inline Preconditioner ilu0_factor(const SparseMatrix& a) { return Preconditioner::ilu0(a); }

inline BlockVector precond_apply(const Preconditioner& m, const BlockVector& r,
                                 FlopCounter* flops = nullptr) {
  return m.apply(r, flops);
}

}  // namespace blockkrylov
