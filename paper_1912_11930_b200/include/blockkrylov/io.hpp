// blockkrylov/io.hpp — the reference's text formats, host side:
//   * Matrix Market coordinate (sparse_matrix.hpp:133-205): written as
//     "real symmetric" with the lower triangle, 1-based, %.17g values; read
//     as symmetric (mirrored) or general, then assembled through
//     SparseMatrix::from_triplets and its symmetry validation;
//   * the dense block-vector text format (block_vector.hpp:72-112): an
//     "n k" header and n lines of k %.17g values.
// Failures throw IoError, as in the reference.
#pragma once

#include <cstddef>
#include <cstdio>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "blockkrylov/block_vector.hpp"
#include "blockkrylov/errors.hpp"
#include "blockkrylov/sparse_matrix.hpp"

namespace blockkrylov {

namespace detail {
inline std::string g17(double v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}
}  // namespace detail

inline void write_matrix_market(std::ostream& out, const SparseMatrix& a) {
  const auto off = a.row_offsets();
  const auto col = a.col_indices();
  const auto val = a.values();
  std::size_t lower = 0;  // entries with col <= row
  for (std::size_t r = 0; r < a.n(); ++r)
    for (std::size_t i = off[r]; i < off[r + 1] && col[i] <= r; ++i) ++lower;
  out << "%%MatrixMarket matrix coordinate real symmetric\n"
      << a.n() << ' ' << a.n() << ' ' << lower << '\n';
  for (std::size_t r = 0; r < a.n(); ++r)
    for (std::size_t i = off[r]; i < off[r + 1] && col[i] <= r; ++i)
      out << r + 1 << ' ' << col[i] + 1 << ' ' << detail::g17(val[i]) << '\n';
}

inline SparseMatrix read_matrix_market(std::istream& in) {
  std::string line;
  if (!std::getline(in, line)) throw IoError("matrix market: empty file");
  std::string banner, object, format, field, symmetry;
  std::istringstream(line) >> banner >> object >> format >> field >> symmetry;
  if (banner != "%%MatrixMarket" || object != "matrix" || format != "coordinate")
    throw IoError("matrix market: expected '%%MatrixMarket matrix coordinate' header");
  if (field != "real") throw IoError("matrix market: only real matrices are supported");
  if (symmetry != "symmetric" && symmetry != "general")
    throw IoError("matrix market: unsupported symmetry '" + symmetry + "'");
  const bool mirror = symmetry == "symmetric";
  do {  // skip comment lines up to the size line
    if (!std::getline(in, line)) throw IoError("matrix market: missing size line");
  } while (line.empty() || line[0] == '%');
  std::size_t rows = 0, cols = 0, entries = 0;
  if (!(std::istringstream(line) >> rows >> cols >> entries))
    throw IoError("matrix market: missing size line");
  if (rows != cols) throw IoError("matrix market: matrix must be square");
  std::vector<std::tuple<std::size_t, std::size_t, double>> t;
  t.reserve(mirror ? 2 * entries : entries);
  for (std::size_t e = 0; e < entries; ++e) {
    std::size_t r = 0, c = 0;
    double v = 0.0;
    if (!(in >> r >> c >> v)) throw IoError("matrix market: truncated entry list");
    if (r < 1 || c < 1 || r > rows || c > cols)
      throw IoError("matrix market: entry index out of range");
    t.emplace_back(r - 1, c - 1, v);
    if (mirror && r != c) t.emplace_back(c - 1, r - 1, v);
  }
  return SparseMatrix::from_triplets(rows, std::move(t));
}

inline void save_matrix_market(const std::string& path, const SparseMatrix& a) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot open '" + path + "' for writing");
  write_matrix_market(out, a);
  if (!out) throw IoError("error while writing '" + path + "'");
}

inline SparseMatrix load_matrix_market(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open '" + path + "'");
  return read_matrix_market(in);
}

inline void write_block_vector(std::ostream& out, const BlockVector& x) {
  out << x.rows() << ' ' << x.cols() << '\n';
  for (std::size_t r = 0; r < x.rows(); ++r) {
    std::string line;
    for (std::size_t c = 0; c < x.cols(); ++c) {
      if (c) line += ' ';
      line += detail::g17(x(r, c));
    }
    out << line << '\n';
  }
}

inline BlockVector read_block_vector(std::istream& in) {
  std::size_t n = 0, k = 0;
  if (!(in >> n >> k)) throw IoError("block vector file: missing 'n k' header");
  if (k == 0) throw IoError("block vector file: column count must be positive");
  BlockVector x(n, k);
  double* d = x.data();
  for (std::size_t i = 0; i < n * k; ++i)
    if (!(in >> d[i]))
      throw IoError("block vector file: expected " + std::to_string(n * k) +
                    " entries, file ended early");
  return x;
}

inline void save_block_vector(const std::string& path, const BlockVector& x) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot open '" + path + "' for writing");
  write_block_vector(out, x);
  if (!out) throw IoError("error while writing '" + path + "'");
}

inline BlockVector load_block_vector(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open '" + path + "'");
  return read_block_vector(in);
}

}  // namespace blockkrylov
