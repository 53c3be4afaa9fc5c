// blockkrylov/sparse_matrix.hpp — drop-in for SparseMatrix
// (proj/include/blockkrylov/sparse_matrix.hpp:27-131).  Same construction
// checks (CSR structure, 1e-14 value symmetry) and accessors; the device copy
// (int32 columns / int64 offsets) is uploaded once on first use and cached.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <memory>
#include <span>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "bkg.h"
#include "blockkrylov/device.hpp"
#include "blockkrylov/errors.hpp"

namespace blockkrylov {

class SparseMatrix {
 public:
  SparseMatrix(std::size_t n, std::vector<std::size_t> row_offsets,
               std::vector<std::size_t> col_indices, std::vector<double> values)
      : n_(n),
        off_(std::move(row_offsets)),
        cols_(std::move(col_indices)),
        vals_(std::move(values)) {
    validate();
  }

  /// Assembles from (row, col, value) triplets; duplicates are summed.
  static SparseMatrix from_triplets(std::size_t n,
                                    std::vector<std::tuple<std::size_t, std::size_t, double>> t) {
    std::sort(t.begin(), t.end(), [](const auto& a, const auto& b) {
      return std::tie(std::get<0>(a), std::get<1>(a)) < std::tie(std::get<0>(b), std::get<1>(b));
    });
    std::vector<std::size_t> count(n, 0), cols;
    std::vector<double> vals;
    for (const auto& [r, c, v] : t) {
      if (r >= n || c >= n) throw ConfigError("triplet index out of range");
      if (count[r] > 0 && cols.back() == c) {
        vals.back() += v;
        continue;
      }
      ++count[r];
      cols.push_back(c);
      vals.push_back(v);
    }
    std::vector<std::size_t> off(n + 1, 0);
    for (std::size_t r = 0; r < n; ++r) off[r + 1] = off[r] + count[r];
    return {n, std::move(off), std::move(cols), std::move(vals)};
  }

  std::size_t n() const noexcept { return n_; }
  std::size_t nnz() const noexcept { return vals_.size(); }
  std::span<const std::size_t> row_offsets() const noexcept { return off_; }
  std::span<const std::size_t> col_indices() const noexcept { return cols_; }
  std::span<const double> values() const noexcept { return vals_; }

  double at(std::size_t row, std::size_t col) const {
    const auto lo = cols_.begin() + static_cast<std::ptrdiff_t>(off_[row]);
    const auto hi = cols_.begin() + static_cast<std::ptrdiff_t>(off_[row + 1]);
    const auto it = std::lower_bound(lo, hi, col);
    return (it == hi || *it != col) ? 0.0 : vals_[static_cast<std::size_t>(it - cols_.begin())];
  }

  friend bool operator==(const SparseMatrix& a, const SparseMatrix& b) {
    return a.n_ == b.n_ && a.off_ == b.off_ && a.cols_ == b.cols_ && a.vals_ == b.vals_;
  }

  /// The device-resident copy (uploaded on first use; immutable afterwards).
  const bkg_matrix* device() const {
    if (!dev_) {
      static_assert(sizeof(std::size_t) == sizeof(uint64_t), "size_t must be 64-bit");
      bkg_matrix* m = nullptr;
      detail::check(bkg_matrix_create(gpu::context(), n_,
                                      reinterpret_cast<const uint64_t*>(off_.data()),
                                      reinterpret_cast<const uint64_t*>(cols_.data()),
                                      vals_.data(), &m));
      dev_ = std::shared_ptr<bkg_matrix>(m, [](bkg_matrix* p) { bkg_matrix_destroy(p); });
    }
    return dev_.get();
  }

 private:
  void validate() const {  // sparse_matrix.hpp:89-125
    if (n_ == 0) throw ConfigError("sparse matrix: dimension must be positive");
    if (off_.size() != n_ + 1) throw ConfigError("sparse matrix: row_offsets must have n+1 entries");
    if (off_.front() != 0 || off_.back() != vals_.size() || cols_.size() != vals_.size())
      throw ConfigError("sparse matrix: offsets inconsistent with stored entries");
    for (std::size_t r = 0; r < n_; ++r) {
      if (off_[r] > off_[r + 1]) throw ConfigError("sparse matrix: row_offsets must be non-decreasing");
      for (std::size_t i = off_[r]; i < off_[r + 1]; ++i) {
        if (cols_[i] >= n_) throw ConfigError("sparse matrix: column index out of range");
        if (i > off_[r] && cols_[i] <= cols_[i - 1])
          throw ConfigError("sparse matrix: columns must be strictly ascending per row");
      }
    }
    for (std::size_t r = 0; r < n_; ++r)
      for (std::size_t i = off_[r]; i < off_[r + 1]; ++i) {
        const std::size_t c = cols_[i];
        if (c == r) continue;
        const auto lo = cols_.begin() + static_cast<std::ptrdiff_t>(off_[c]);
        const auto hi = cols_.begin() + static_cast<std::ptrdiff_t>(off_[c + 1]);
        const auto it = std::lower_bound(lo, hi, r);
        if (it == hi || *it != r)
          throw ConfigError("sparse matrix: entry (" + std::to_string(r) + "," +
                            std::to_string(c) + ") has no symmetric counterpart");
        const double v = vals_[i], w = vals_[static_cast<std::size_t>(it - cols_.begin())];
        if (std::abs(v - w) > 1e-14 * std::max(std::abs(v), std::abs(w)))
          throw ConfigError("sparse matrix: values not symmetric at (" + std::to_string(r) +
                            "," + std::to_string(c) + ")");
      }
  }

  std::size_t n_;
  std::vector<std::size_t> off_, cols_;
  std::vector<double> vals_;
  mutable std::shared_ptr<bkg_matrix> dev_;
};

}  // namespace blockkrylov
