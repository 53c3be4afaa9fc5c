// blockkrylov/errors.hpp — drop-in for the reference exception hierarchy
// (proj/include/blockkrylov/errors.hpp:10-61), plus the mapping from C-ABI
// status codes (include/bkg.h) back to exceptions.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

#include "bkg.h"

namespace blockkrylov {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class DimensionError : public Error {
 public:
  using Error::Error;
};

class ConfigError : public Error {
 public:
  using Error::Error;
};

class SizeError : public Error {
 public:
  using Error::Error;
};

class BreakdownError : public Error {
 public:
  BreakdownError(std::size_t block_index, const std::string& what)
      : Error(what), block_index_(block_index) {}
  std::size_t block_index() const noexcept { return block_index_; }

 private:
  std::size_t block_index_;
};

class FactorizationError : public Error {
 public:
  FactorizationError(std::size_t row, const std::string& what) : Error(what), row_(row) {}
  std::size_t row() const noexcept { return row_; }

 private:
  std::size_t row_;
};

class IoError : public Error {
 public:
  using Error::Error;
};

/// Device / driver failure (no reference counterpart: the reference is CPU-only).
class DeviceError : public Error {
 public:
  using Error::Error;
};

namespace detail {

/// Rethrow a failing C-ABI status as the reference's exception type.
inline void check(int status, std::size_t index = 0) {
  if (status == BKG_OK) return;
  const std::string msg = bkg_last_error();
  switch (status) {
    case BKG_DIMENSION: throw DimensionError(msg);
    case BKG_CONFIG: throw ConfigError(msg);
    case BKG_BREAKDOWN: throw BreakdownError(index, msg);
    case BKG_FACTORIZATION: throw FactorizationError(index, msg);
    case BKG_CUDA: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

}  // namespace detail
}  // namespace blockkrylov
