// problems.cpp — input generators exported through the C ABI.
//
// poisson2d (problems.hpp:74-124) and random_block_rhs (problems.hpp:128-134)
// reproduce the reference generators bit-for-bit; the N(0,1) RHS, the
// exp(N(0,1)) diffusion field and the 3D 7/27-point stencils are the frozen
// synthetic inputs defined in DESIGN.md §Inputs.  Compiled with
// -ffp-contract=off so libm-based values match the oracle's.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "bkg.h"
#include "rng.h"

namespace {

using namespace bkg;

// Stream position -> state, shared by all generator threads.
const uint64_t* jump_table() {
  static const std::vector<uint64_t> t = [] {
    std::vector<uint64_t> v(64 * 64);
    rng::jump_table(v.data());
    return v;
  }();
  return t.data();
}

// Runs body(begin, end, state_at_begin_draw) over [0, units) in parallel
// chunks; `draws` draws per unit.  Chunks start from the jumped state, so the
// result is the serial stream's bit for bit.
template <class F>
void parallel_stream(uint64_t seed, uint64_t units, uint64_t draws, F body) {
  const uint64_t s0 = rng::seed_state(seed);
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const uint64_t per = std::max<uint64_t>(1u << 18, (units + hw - 1) / hw);
  std::vector<std::thread> pool;
  for (uint64_t b = 0; b < units; b += per) {
    const uint64_t e = std::min(units, b + per);
    const uint64_t s = rng::jump(jump_table(), s0, b * draws);
    if (e == units && pool.empty()) {  // one chunk: no thread
      body(b, e, s);
      return;
    }
    pool.emplace_back([=] { body(b, e, s); });
  }
  for (auto& t : pool) t.join();
}

// Box-Muller pairs over Xorshift64Star, both outputs used, storage order:
// pair j consumes draws 2j, 2j+1 and writes values 2j, 2j+1.
void normal_fill(uint64_t seed, uint64_t count, double* out) {
  parallel_stream(seed, (count + 1) / 2, 2, [=](uint64_t b, uint64_t e, uint64_t s) {
    for (uint64_t j = b; j < e; ++j) {
      const double u1 = rng::unit(s);
      const double u2 = rng::unit(s);
      const double rad = std::sqrt(-2.0 * std::log(1.0 - u1));
      const double th = 6.283185307179586 * u2;
      out[2 * j] = rad * std::cos(th);
      if (2 * j + 1 < count) out[2 * j + 1] = rad * std::sin(th);
    }
  });
}

inline double harmonic(double a, double b) { return 2.0 * a * b / (a + b); }

uint64_t pairs(uint64_t m) { return m > 0 ? m - 1 : 0; }

void assemble2d(uint64_t nx, uint64_t ny, const double* coeff, uint64_t* off, uint64_t* cols,
                double* vals) {
  uint64_t nnz = 0;
  off[0] = 0;
  for (uint64_t j = 0; j < ny; ++j)
    for (uint64_t i = 0; i < nx; ++i) {
      const uint64_t row = j * nx + i;
      double diag = 0.0, south = 0.0, west = 0.0, east = 0.0, north = 0.0;
      if (j > 0) diag += south = harmonic(coeff[row], coeff[row - nx]);
      else diag += coeff[row];
      if (i > 0) diag += west = harmonic(coeff[row], coeff[row - 1]);
      else diag += coeff[row];
      if (i + 1 < nx) diag += east = harmonic(coeff[row], coeff[row + 1]);
      else diag += coeff[row];
      if (j + 1 < ny) diag += north = harmonic(coeff[row], coeff[row + nx]);
      else diag += coeff[row];
      if (j > 0) { cols[nnz] = row - nx; vals[nnz++] = -south; }
      if (i > 0) { cols[nnz] = row - 1; vals[nnz++] = -west; }
      cols[nnz] = row; vals[nnz++] = diag;
      if (i + 1 < nx) { cols[nnz] = row + 1; vals[nnz++] = -east; }
      if (j + 1 < ny) { cols[nnz] = row + nx; vals[nnz++] = -north; }
      off[row + 1] = nnz;
    }
}

void assemble3d(uint64_t nx, uint64_t ny, uint64_t nz, bool full27, uint64_t* off,
                uint64_t* cols, double* vals) {
  const double centre = full27 ? 26.0 : 6.0;
  uint64_t nnz = 0;
  off[0] = 0;
  for (uint64_t l = 0; l < nz; ++l)
    for (uint64_t j = 0; j < ny; ++j)
      for (uint64_t i = 0; i < nx; ++i) {
        const uint64_t row = (l * ny + j) * nx + i;
        for (int dl = -1; dl <= 1; ++dl)
          for (int dj = -1; dj <= 1; ++dj)
            for (int di = -1; di <= 1; ++di) {
              if (!full27 && (di != 0) + (dj != 0) + (dl != 0) > 1) continue;
              const int64_t ii = (int64_t)i + di, jj = (int64_t)j + dj, ll = (int64_t)l + dl;
              if (ii < 0 || jj < 0 || ll < 0 || ii >= (int64_t)nx || jj >= (int64_t)ny ||
                  ll >= (int64_t)nz)
                continue;
              const uint64_t c = ((uint64_t)ll * ny + (uint64_t)jj) * nx + (uint64_t)ii;
              cols[nnz] = c;
              vals[nnz++] = c == row ? centre : -1.0;
            }
        off[row + 1] = nnz;
      }
}

}  // namespace

namespace bkg {
// Cell coefficients of the 2D generators: kind 1 = 10^(contrast * U(-1,1))
// (problems.hpp:90-99), kind 2 = exp(N(0,1)).  Host libm,
// so the device assembler (generate.cu) uses these same bits.
void coefficient_field(int kind, uint64_t seed, double contrast, uint64_t n, double* coeff) {
  if (kind == 1) {
    parallel_stream(seed, n, 1, [=](uint64_t b, uint64_t e, uint64_t s) {
      for (uint64_t i = b; i < e; ++i) coeff[i] = std::pow(10.0, contrast * rng::symmetric(s));
    });
  } else {
    normal_fill(seed, n, coeff);
    for (uint64_t i = 0; i < n; ++i) coeff[i] = std::exp(coeff[i]);
  }
}
}  // namespace bkg

extern "C" {

int bkg_stencil_size(int kind, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t* n,
                     uint64_t* nnz) {
  switch (kind) {
    case 0:
    case 1:
    case 2:
      *n = nx * ny;
      *nnz = nx * ny + 2 * (pairs(nx) * ny + nx * pairs(ny));
      return BKG_OK;
    case 3:
      *n = nx * ny * nz;
      *nnz = nx * ny * nz + 2 * (pairs(nx) * ny * nz + nx * pairs(ny) * nz + nx * ny * pairs(nz));
      return BKG_OK;
    case 4:
      *n = nx * ny * nz;
      *nnz = (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2);
      return BKG_OK;
    default: return BKG_CONFIG;
  }
}

int bkg_stencil_fill(int kind, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t seed,
                     double contrast, uint64_t* off, uint64_t* cols, double* vals) {
  if (kind == 3 || kind == 4) {
    if (nx < 2 || ny < 2 || nz < 2) return BKG_CONFIG;
    assemble3d(nx, ny, nz, kind == 4, off, cols, vals);
    return BKG_OK;
  }
  if (kind < 0 || kind > 2) return BKG_CONFIG;
  if (nx < 2 || ny < 2) return BKG_CONFIG;
  const uint64_t n = nx * ny;
  std::vector<double> coeff(n, 1.0);
  if (kind == 1 || kind == 2) {
    if (kind == 1 && !(contrast >= 0.0)) return BKG_CONFIG;
    coefficient_field(kind, seed, contrast, n, coeff.data());
  }
  assemble2d(nx, ny, coeff.data(), off, cols, vals);
  return BKG_OK;
}

int bkg_random_block_rhs(uint64_t n, uint64_t k, uint64_t seed, double* out) {
  parallel_stream(seed, n * k, 1, [=](uint64_t b, uint64_t e, uint64_t s) {
    for (uint64_t i = b; i < e; ++i) out[i] = rng::symmetric(s);
  });
  return BKG_OK;
}

int bkg_normal_block_rhs(uint64_t n, uint64_t k, uint64_t seed, double* out) {
  normal_fill(seed, n * k, out);
  return BKG_OK;
}

}  // extern "C"
