// blockkrylov/block_vector.hpp — drop-in for the reference BlockVector
// (proj/include/blockkrylov/block_vector.hpp:23-70): an n x k host block,
// lane-interleaved (data[row * k + col]); column_norms runs on the GPU.
#pragma once

#include <algorithm>
#include <cstddef>
#include <span>
#include <vector>

#include "bkg.h"
#include "blockkrylov/device.hpp"
#include "blockkrylov/errors.hpp"

namespace blockkrylov {

class BlockVector {
 public:
  BlockVector() = default;
  BlockVector(std::size_t n, std::size_t k, double value = 0.0)
      : n_(n), k_(k), data_(n * k, value) {
    if (k == 0) throw ConfigError("BlockVector: column count must be positive");
  }

  std::size_t rows() const noexcept { return n_; }
  std::size_t cols() const noexcept { return k_; }
  double& operator()(std::size_t r, std::size_t c) { return data_[r * k_ + c]; }
  double operator()(std::size_t r, std::size_t c) const { return data_[r * k_ + c]; }
  std::span<double> row(std::size_t r) { return {data_.data() + r * k_, k_}; }
  std::span<const double> row(std::size_t r) const { return {data_.data() + r * k_, k_}; }
  double* data() noexcept { return data_.data(); }
  const double* data() const noexcept { return data_.data(); }
  std::size_t size() const noexcept { return data_.size(); }
  void fill(double v) { std::fill(data_.begin(), data_.end(), v); }

  friend bool operator==(const BlockVector& a, const BlockVector& b) {
    return a.n_ == b.n_ && a.k_ == b.k_ && a.data_ == b.data_;
  }

 private:
  std::size_t n_ = 0, k_ = 0;
  std::vector<double> data_;
};

/// Euclidean norm of each column (block_vector.hpp:59-70) — on the device.
inline std::vector<double> column_norms(const BlockVector& x) {
  std::vector<double> out(x.cols());
  detail::check(bkg_column_norms(gpu::context(), x.rows(), x.cols(), x.data(), out.data()));
  return out;
}

}  // namespace blockkrylov
