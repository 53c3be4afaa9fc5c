/*
 * bcg_oracle.c — TEST INFRASTRUCTURE ONLY (see bcg_oracle.h).
 *
 * Plain-C restatement of the reference blockkrylov hot path, operation for
 * operation in the reference's order so that, compiled with
 * -O3 -ffp-contract=off, it is bit-identical to the reference's own Release
 * build (SURVEY.md §0 finding 5).  Never shipped, never called by the product.
 */
#include "bcg_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ */
/* Xorshift64Star: problems.hpp:19-46                                   */
/* ------------------------------------------------------------------ */
typedef struct {
  uint64_t s;
} orc_rng;

uint64_t orc_rng_seed_state(uint64_t seed) {
  /* splitmix64 step, problems.hpp:22-28 */
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  if (z == 0) z = 0x9E3779B97F4A7C15ull;
  return z;
}

static inline uint64_t rng_next(orc_rng* g) { /* problems.hpp:31-36 */
  g->s ^= g->s >> 12;
  g->s ^= g->s << 25;
  g->s ^= g->s >> 27;
  return g->s * 0x2545F4914F6CDD1Dull;
}
static inline double rng_unit(orc_rng* g) { /* problems.hpp:39 */
  return (double)(rng_next(g) >> 11) * 0x1.0p-53;
}
static inline double rng_symmetric(orc_rng* g) { /* problems.hpp:42 */
  return 2.0 * rng_unit(g) - 1.0;
}

void orc_rng_symmetric(uint64_t seed, size_t count, double* out) {
  orc_rng g = {orc_rng_seed_state(seed)};
  for (size_t i = 0; i < count; ++i) out[i] = rng_symmetric(&g);
}

/* random_block_rhs: problems.hpp:128-134 (row-major fill, one stream) */
void orc_random_block_rhs(size_t n, size_t k, uint64_t seed, double* out) {
  orc_rng g = {orc_rng_seed_state(seed)};
  for (size_t i = 0; i < n * k; ++i) out[i] = rng_symmetric(&g);
}

/* Frozen N(0,1) stream (new; defined in DESIGN.md §Inputs): Box-Muller over
 * Xorshift64Star, both outputs used, filled in storage order like
 * random_block_rhs. */
static void normal_fill(orc_rng* g, size_t count, double* out) {
  for (size_t i = 0; i < count; i += 2) {
    const double u1 = rng_unit(g);
    const double u2 = rng_unit(g);
    const double rad = sqrt(-2.0 * log(1.0 - u1));
    const double th = 6.283185307179586 * u2;
    out[i] = rad * cos(th);
    if (i + 1 < count) out[i + 1] = rad * sin(th);
  }
}

void orc_normal_block_rhs(size_t n, size_t k, uint64_t seed, double* out) {
  orc_rng g = {orc_rng_seed_state(seed)};
  normal_fill(&g, n * k, out);
}

/* ------------------------------------------------------------------ */
/* Matrix generators                                                    */
/* ------------------------------------------------------------------ */
size_t orc_stencil_rows(int kind, size_t nx, size_t ny, size_t nz) {
  switch (kind) {
    case ORC_POISSON2D_CONST:
    case ORC_POISSON2D_LOGUNI:
    case ORC_DIFFUSION2D_LOGNORMAL: return nx * ny;
    default: return nx * ny * nz;
  }
}

static size_t axis_pairs(size_t m) { return m > 0 ? m - 1 : 0; }

size_t orc_stencil_nnz(int kind, size_t nx, size_t ny, size_t nz) {
  switch (kind) {
    case ORC_POISSON2D_CONST:
    case ORC_POISSON2D_LOGUNI:
    case ORC_DIFFUSION2D_LOGNORMAL:
      return nx * ny + 2 * (axis_pairs(nx) * ny + nx * axis_pairs(ny));
    case ORC_LAPLACE3D_7PT:
      return nx * ny * nz + 2 * (axis_pairs(nx) * ny * nz + nx * axis_pairs(ny) * nz +
                                 nx * ny * axis_pairs(nz));
    case ORC_STENCIL3D_27PT:
      /* (3nx-2)(3ny-2)(3nz-2) neighbour pairs incl. self */
      return (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2);
    default: return 0;
  }
}

static inline double harmonic(double a, double b) { return 2.0 * a * b / (a + b); }

/* poisson2d: problems.hpp:74-124, generalised to a caller-given cell
 * coefficient array (the C3 lognormal field uses the same assembly). */
static void assemble2d(size_t nx, size_t ny, const double* coeff, uint64_t* offsets,
                       uint64_t* cols, double* vals) {
  size_t nnz = 0;
  offsets[0] = 0;
  for (size_t j = 0; j < ny; ++j) {
    for (size_t i = 0; i < nx; ++i) {
      const size_t row = j * nx + i;
      double diag = 0.0;
      double south = 0.0, west = 0.0, east = 0.0, north = 0.0;
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
      offsets[row + 1] = nnz;
    }
  }
}

static void assemble3d(size_t nx, size_t ny, size_t nz, int full27, uint64_t* offsets,
                       uint64_t* cols, double* vals) {
  const double centre = full27 ? 26.0 : 6.0;
  size_t nnz = 0;
  offsets[0] = 0;
  for (size_t l = 0; l < nz; ++l)
    for (size_t j = 0; j < ny; ++j)
      for (size_t i = 0; i < nx; ++i) {
        const size_t row = (l * ny + j) * nx + i;
        for (int dl = -1; dl <= 1; ++dl)
          for (int dj = -1; dj <= 1; ++dj)
            for (int di = -1; di <= 1; ++di) {
              const int off = (di != 0) + (dj != 0) + (dl != 0);
              if (!full27 && off > 1) continue;
              const long ii = (long)i + di, jj = (long)j + dj, ll = (long)l + dl;
              if (ii < 0 || jj < 0 || ll < 0 || ii >= (long)nx || jj >= (long)ny ||
                  ll >= (long)nz)
                continue;
              const size_t c = ((size_t)ll * ny + (size_t)jj) * nx + (size_t)ii;
              cols[nnz] = c;
              vals[nnz++] = c == row ? centre : -1.0;
            }
        offsets[row + 1] = nnz;
      }
}

int orc_stencil_fill(int kind, size_t nx, size_t ny, size_t nz, uint64_t seed, double contrast,
                     uint64_t* rowptr, uint64_t* cols, double* vals) {
  if (kind == ORC_LAPLACE3D_7PT || kind == ORC_STENCIL3D_27PT) {
    if (nx < 2 || ny < 2 || nz < 2) return ORC_CONFIG;
    assemble3d(nx, ny, nz, kind == ORC_STENCIL3D_27PT, rowptr, cols, vals);
    return ORC_OK;
  }
  if (nx < 2 || ny < 2) return ORC_CONFIG; /* problems.hpp:75-76 */
  const size_t n = nx * ny;
  double* coeff = (double*)malloc(n * sizeof(double));
  for (size_t i = 0; i < n; ++i) coeff[i] = 1.0;
  if (kind == ORC_POISSON2D_LOGUNI) { /* problems.hpp:84-88 */
    if (!(contrast >= 0.0)) { free(coeff); return ORC_CONFIG; }
    orc_rng g = {orc_rng_seed_state(seed)};
    for (size_t i = 0; i < n; ++i) coeff[i] = pow(10.0, contrast * rng_symmetric(&g));
  } else if (kind == ORC_DIFFUSION2D_LOGNORMAL) {
    orc_rng g = {orc_rng_seed_state(seed)};
    normal_fill(&g, n, coeff);
    for (size_t i = 0; i < n; ++i) coeff[i] = exp(coeff[i]);
  }
  assemble2d(nx, ny, coeff, rowptr, cols, vals);
  free(coeff);
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Kernels                                                              */
/* ------------------------------------------------------------------ */

/* bdot: kernels.hpp:59-88 — row loop, group loop, p x p outer product. */
void orc_bdot(size_t n, size_t k, size_t p, int global, const double* x, const double* y,
              double* out) {
  const size_t q = k / p;
  const size_t blocks = global ? 1 : q;
  memset(out, 0, blocks * p * p * sizeof(double));
  for (size_t r = 0; r < n; ++r) {
    const double* xr = x + r * k;
    const double* yr = y + r * k;
    for (size_t g = 0; g < q; ++g) {
      double* blk = out + (global ? 0 : g) * p * p;
      const double* xg = xr + g * p;
      const double* yg = yr + g * p;
      for (size_t a = 0; a < p; ++a)
        for (size_t b = 0; b < p; ++b) blk[a * p + b] += xg[a] * yg[b];
    }
  }
}

/* baxpy: kernels.hpp:94-125 — X <- X + Y * embed(gamma). */
void orc_baxpy(size_t n, size_t k, size_t p, int global, double* x, const double* y,
               const double* gamma) {
  const size_t q = k / p;
  for (size_t r = 0; r < n; ++r) {
    double* xr = x + r * k;
    const double* yr = y + r * k;
    for (size_t g = 0; g < q; ++g) {
      const double* blk = gamma + (global ? 0 : g) * p * p;
      double* xg = xr + g * p;
      const double* yg = yr + g * p;
      for (size_t a = 0; a < p; ++a) {
        double acc = xg[a];
        for (size_t b = 0; b < p; ++b) acc += yg[b] * blk[b * p + a];
        xg[a] = acc;
      }
    }
  }
}

/* bop: kernels.hpp:129-157 — Y = A X, all k lanes per nonzero. */
void orc_bop(size_t n, const uint64_t* rowptr, const uint64_t* cols, const double* vals,
             size_t k, const double* x, double* y) {
  for (size_t r = 0; r < n; ++r) {
    double* yr = y + r * k;
    for (size_t c = 0; c < k; ++c) yr[c] = 0.0;
    for (uint64_t i = rowptr[r]; i < rowptr[r + 1]; ++i) {
      const double v = vals[i];
      const double* xc = x + cols[i] * k;
      for (size_t c = 0; c < k; ++c) yr[c] += v * xc[c];
    }
  }
}

/* detail::solve_block: kernels.hpp:171-224 — LU with partial pivoting. */
static int solve_block(size_t p, const double* gamma, const double* delta, double* result,
                       double* lu, size_t* perm) {
  memcpy(lu, gamma, p * p * sizeof(double));
  for (size_t i = 0; i < p; ++i) perm[i] = i;
  double max_norm = 0.0;
  for (size_t i = 0; i < p * p; ++i) {
    const double v = fabs(lu[i]);
    max_norm = (max_norm < v) ? v : max_norm; /* std::max(max_norm, v) */
  }
  const double tiny = 1e-14 * max_norm;
  for (size_t col = 0; col < p; ++col) {
    size_t pivot_row = col;
    double pivot = fabs(lu[col * p + col]);
    for (size_t r = col + 1; r < p; ++r) {
      const double cand = fabs(lu[r * p + col]);
      if (cand > pivot) {
        pivot = cand;
        pivot_row = r;
      }
    }
    if (pivot < tiny || max_norm == 0.0) return 1;
    if (pivot_row != col) {
      for (size_t c = 0; c < p; ++c) {
        const double t = lu[col * p + c];
        lu[col * p + c] = lu[pivot_row * p + c];
        lu[pivot_row * p + c] = t;
      }
      const size_t t = perm[col];
      perm[col] = perm[pivot_row];
      perm[pivot_row] = t;
    }
    const double inv = 1.0 / lu[col * p + col];
    for (size_t r = col + 1; r < p; ++r) {
      const double f = lu[r * p + col] * inv;
      lu[r * p + col] = f;
      for (size_t c = col + 1; c < p; ++c) lu[r * p + c] -= f * lu[col * p + c];
    }
  }
  for (size_t r = 0; r < p; ++r)
    for (size_t c = 0; c < p; ++c) result[r * p + c] = delta[perm[r] * p + c];
  for (size_t r = 0; r < p; ++r)
    for (size_t j = 0; j < r; ++j) {
      const double f = lu[r * p + j];
      for (size_t c = 0; c < p; ++c) result[r * p + c] -= f * result[j * p + c];
    }
  for (size_t r = p; r-- > 0;) {
    for (size_t j = r + 1; j < p; ++j) {
      const double f = lu[r * p + j];
      for (size_t c = 0; c < p; ++c) result[r * p + c] -= f * result[j * p + c];
    }
    const double inv = 1.0 / lu[r * p + r];
    for (size_t c = 0; c < p; ++c) result[r * p + c] *= inv;
  }
  return 0;
}

/* bsolve: kernels.hpp:231-240 — blocks in order, first singular block wins. */
int orc_bsolve(size_t k, size_t p, int global, const double* gamma, const double* delta,
               double* out, uint64_t* bad_block) {
  const size_t blocks = global ? 1 : k / p;
  double* lu = (double*)malloc(p * p * sizeof(double));
  size_t* perm = (size_t*)malloc(p * sizeof(size_t));
  int status = ORC_OK;
  for (size_t b = 0; b < blocks; ++b) {
    if (solve_block(p, gamma + b * p * p, delta + b * p * p, out + b * p * p, lu, perm)) {
      if (bad_block) *bad_block = b;
      status = ORC_BREAKDOWN;
      break;
    }
  }
  free(lu);
  free(perm);
  return status;
}

/* column_norms: block_vector.hpp:59-70 */
void orc_column_norms(size_t n, size_t k, const double* x, double* out) {
  for (size_t c = 0; c < k; ++c) out[c] = 0.0;
  for (size_t r = 0; r < n; ++r) {
    const double* xr = x + r * k;
    for (size_t c = 0; c < k; ++c) out[c] += xr[c] * xr[c];
  }
  for (size_t c = 0; c < k; ++c) out[c] = sqrt(out[c]);
}

/* ------------------------------------------------------------------ */
/* Preconditioners: preconditioners.hpp                                 */
/* ------------------------------------------------------------------ */
static uint64_t find_col(const uint64_t* rowptr, const uint64_t* cols, size_t row, size_t col,
                         int* found) {
  /* std::lower_bound over the row's columns (sparse_matrix.hpp:75-81) */
  uint64_t lo = rowptr[row], hi = rowptr[row + 1];
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (cols[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  *found = lo < rowptr[row + 1] && cols[lo] == col;
  return lo;
}

int64_t orc_precond_setup(int kind, size_t n, const uint64_t* rowptr, const uint64_t* cols,
                          const double* vals, double* inv_diag, double* lu) {
  if (kind == ORC_PRECOND_IDENTITY) return ORC_OK;
  if (kind == ORC_PRECOND_JACOBI) { /* preconditioners.hpp:48-59 */
    for (size_t r = 0; r < n; ++r) {
      int found;
      const uint64_t pos = find_col(rowptr, cols, r, r, &found);
      const double d = found ? vals[pos] : 0.0;
      if (!(d > 0.0)) return -1 - (int64_t)r;
      inv_diag[r] = 1.0 / d;
    }
    return ORC_OK;
  }
  /* ilu0_factor: preconditioners.hpp:153-196 */
  const uint64_t nnz = rowptr[n];
  memcpy(lu, vals, nnz * sizeof(double));
  uint64_t* diag_pos = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
  for (size_t r = 0; r < n; ++r) inv_diag[r] = 0.0;
  for (size_t row = 0; row < n; ++row) {
    for (uint64_t i = rowptr[row]; i < rowptr[row + 1] && cols[i] < row; ++i) {
      const size_t j = cols[i];
      const double factor = lu[i] * inv_diag[j];
      lu[i] = factor;
      uint64_t target = i + 1;
      for (uint64_t ju = diag_pos[j] + 1; ju < rowptr[j + 1]; ++ju) {
        const uint64_t c = cols[ju];
        while (target < rowptr[row + 1] && cols[target] < c) ++target;
        if (target == rowptr[row + 1]) break;
        if (cols[target] == c) lu[target] -= factor * lu[ju];
      }
    }
    int found;
    const uint64_t pos = find_col(rowptr, cols, row, row, &found);
    if (!found) { free(diag_pos); return -1 - (int64_t)row; }
    diag_pos[row] = pos;
    const double pivot = lu[pos];
    if (pivot == 0.0) { free(diag_pos); return -1 - (int64_t)row; }
    inv_diag[row] = 1.0 / pivot;
  }
  free(diag_pos);
  return ORC_OK;
}

/* Preconditioner::apply: preconditioners.hpp:73-129 */
void orc_precond_apply(int kind, size_t n, const uint64_t* rowptr, const uint64_t* cols,
                       const double* inv_diag, const double* lu, size_t k, const double* r,
                       double* z, uint64_t* flops) {
  if (kind == ORC_PRECOND_IDENTITY) {
    memcpy(z, r, n * k * sizeof(double));
    return;
  }
  if (kind == ORC_PRECOND_JACOBI) {
    for (size_t row = 0; row < n; ++row) {
      const double d = inv_diag[row];
      for (size_t c = 0; c < k; ++c) z[row * k + c] = d * r[row * k + c];
    }
    if (flops) *flops += (uint64_t)n * k;
    return;
  }
  memcpy(z, r, n * k * sizeof(double));
  uint64_t madds = 0;
  for (size_t row = 0; row < n; ++row) {
    double* zr = z + row * k;
    uint64_t i = rowptr[row];
    for (; i < rowptr[row + 1] && cols[i] < row; ++i) {
      const double v = lu[i];
      const double* zc = z + cols[i] * k;
      for (size_t c = 0; c < k; ++c) zr[c] -= v * zc[c];
      madds += k;
    }
  }
  for (size_t row = n; row-- > 0;) {
    double* zr = z + row * k;
    for (uint64_t i = rowptr[row + 1]; i-- > rowptr[row];) {
      const uint64_t c = cols[i];
      if (c <= row) break;
      const double v = lu[i];
      const double* zc = z + c * k;
      for (size_t lane = 0; lane < k; ++lane) zr[lane] -= v * zc[lane];
      madds += k;
    }
    const double inv = inv_diag[row];
    for (size_t lane = 0; lane < k; ++lane) zr[lane] *= inv;
  }
  if (flops) *flops += 2 * madds + (uint64_t)n * k;
}

/* ------------------------------------------------------------------ */
/* bcg_solve: solver.hpp:106-209                                        */
/* ------------------------------------------------------------------ */
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int all_below(size_t k, const double* norms, const double* limits) { /* :81-85 */
  for (size_t s = 0; s < k; ++s)
    if (!(norms[s] <= limits[s])) return 0;
  return 1;
}

int orc_bcg_solve(size_t n, const uint64_t* rowptr, const uint64_t* cols, const double* vals,
                  int precond_kind, size_t k, size_t p, int global, const double* b,
                  const double* x0, double tol, uint64_t max_iter_opt, int record_history,
                  double* history, uint64_t history_cap, double* x, double* final_norms,
                  orc_report* rep) {
  if (k == 0 || p == 0 || k % p != 0) return ORC_CONFIG;
  if (!(tol > 0.0)) return ORC_CONFIG; /* :120 */
  memset(rep, 0, sizeof(*rep));
  const uint64_t max_iter = max_iter_opt ? max_iter_opt : 10 * (uint64_t)n; /* :121 */
  const size_t q = k / p;
  const size_t blocks = global ? 1 : q;
  const size_t cs = blocks * p * p;
  const size_t nk = n * k;
  const uint64_t bdot_flops = 2ull * n * p * p * q;
  const uint64_t baxpy_flops = bdot_flops;
  const uint64_t bop_flops = 2ull * k * rowptr[n];

  double* inv_diag = (double*)calloc(n ? n : 1, sizeof(double));
  double* lu = precond_kind == ORC_PRECOND_ILU0 ? (double*)malloc(rowptr[n] * sizeof(double))
                                                : NULL;
  if (orc_precond_setup(precond_kind, n, rowptr, cols, vals, inv_diag, lu) != ORC_OK) {
    free(inv_diag);
    free(lu);
    return ORC_CONFIG;
  }

  double* r = (double*)malloc(nk * sizeof(double));
  double* qv = (double*)calloc(nk, sizeof(double));
  double* pv = (double*)calloc(nk, sizeof(double));
  double* z = (double*)calloc(nk, sizeof(double));
  double* limits = (double*)malloc(k * sizeof(double));
  double* defect = (double*)malloc(k * sizeof(double));
  double* alpha = (double*)malloc(cs * sizeof(double));
  double* rho_prev = (double*)malloc(cs * sizeof(double));
  double* rho = (double*)malloc(cs * sizeof(double));
  double* lambda = (double*)malloc(cs * sizeof(double));
  double* neg = (double*)malloc(cs * sizeof(double));
  double* beta = (double*)malloc(cs * sizeof(double));

  /* :125-139 — X = X0; R = B - A X0 when X0 has a nonzero entry */
  int x0_zero = 1;
  if (x0) {
    memcpy(x, x0, nk * sizeof(double));
    for (size_t i = 0; i < nk && x0_zero; ++i) x0_zero = x0[i] == 0.0;
  } else {
    memset(x, 0, nk * sizeof(double));
  }
  memcpy(r, b, nk * sizeof(double));
  if (!x0_zero) {
    double t0 = now_s();
    orc_bop(n, rowptr, cols, vals, k, x, qv);
    rep->flops_bop += bop_flops;
    double t1 = now_s();
    rep->seconds_bop += t1 - t0;
    for (size_t i = 0; i < cs; ++i) neg[i] = -0.0; /* identity(cfg).negated() */
    for (size_t blk = 0; blk < blocks; ++blk)
      for (size_t i = 0; i < p; ++i) neg[blk * p * p + i * p + i] = -1.0;
    orc_baxpy(n, k, p, global, r, qv, neg);
    rep->flops_baxpy += baxpy_flops;
    rep->seconds_baxpy += now_s() - t1;
  }

  /* :141-148 */
  orc_column_norms(n, k, b, limits);
  for (size_t s = 0; s < k; ++s) limits[s] = limits[s] > 0.0 ? tol * limits[s] : tol;
  orc_column_norms(n, k, r, defect);
  if (record_history) {
    if (rep->history_rows < history_cap) memcpy(history, defect, k * sizeof(double));
    rep->history_rows++;
  }
  rep->converged = all_below(k, defect, limits);

  if (!rep->converged) { /* :150-155 */
    double t0 = now_s();
    orc_precond_apply(precond_kind, n, rowptr, cols, inv_diag, lu, k, r, pv,
                      &rep->flops_precond);
    rep->seconds_precond += now_s() - t0;
  }

  while (!rep->converged && rep->iterations < max_iter) { /* :157-201 */
    const uint64_t i = rep->iterations + 1;
    uint64_t bad = 0;
    double t0 = now_s();
    orc_bop(n, rowptr, cols, vals, k, pv, qv);
    rep->flops_bop += bop_flops;
    double t1 = now_s();
    rep->seconds_bop += t1 - t0;
    orc_bdot(n, k, p, global, pv, qv, alpha);
    rep->flops_bdot += bdot_flops;
    orc_bdot(n, k, p, global, pv, r, rho_prev); /* recompute */
    rep->flops_bdot += bdot_flops;
    double t2 = now_s();
    rep->seconds_bdot += t2 - t1;
    if (orc_bsolve(k, p, global, alpha, rho_prev, lambda, &bad) != ORC_OK) {
      rep->breakdown = 1;
      rep->breakdown_iteration = i;
      rep->breakdown_block = bad;
      break;
    }
    t2 = now_s();
    orc_baxpy(n, k, p, global, x, pv, lambda);
    rep->flops_baxpy += baxpy_flops;
    for (size_t e = 0; e < cs; ++e) neg[e] = -lambda[e]; /* lambda.negated() */
    orc_baxpy(n, k, p, global, r, qv, neg);
    rep->flops_baxpy += baxpy_flops;
    double t3 = now_s();
    rep->seconds_baxpy += t3 - t2;
    orc_precond_apply(precond_kind, n, rowptr, cols, inv_diag, lu, k, r, z,
                      &rep->flops_precond);
    double t4 = now_s();
    rep->seconds_precond += t4 - t3;
    orc_bdot(n, k, p, global, z, r, rho);
    rep->flops_bdot += bdot_flops;
    double t5 = now_s();
    rep->seconds_bdot += t5 - t4;
    if (orc_bsolve(k, p, global, rho_prev, rho, beta, &bad) != ORC_OK) {
      rep->breakdown = 1;
      rep->breakdown_iteration = i;
      rep->breakdown_block = bad;
      break;
    }
    t5 = now_s();
    orc_baxpy(n, k, p, global, z, pv, beta);
    rep->flops_baxpy += baxpy_flops;
    rep->seconds_baxpy += now_s() - t5;
    double* tmp = pv; /* std::swap(p, z) */
    pv = z;
    z = tmp;

    rep->iterations = i;
    orc_column_norms(n, k, r, defect);
    if (record_history) {
      if (rep->history_rows < history_cap)
        memcpy(history + rep->history_rows * k, defect, k * sizeof(double));
      rep->history_rows++;
    }
    rep->converged = all_below(k, defect, limits);
  }

  /* :203-207 explicit residual, not instrumented */
  orc_bop(n, rowptr, cols, vals, k, x, qv);
  for (size_t e = 0; e < nk; ++e) qv[e] = b[e] - qv[e];
  if (final_norms) orc_column_norms(n, k, qv, final_norms);

  free(r); free(qv); free(pv); free(z); free(limits); free(defect); free(alpha);
  free(rho_prev); free(rho); free(lambda); free(neg); free(beta); free(inv_diag); free(lu);
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* CPU baseline harness                                                 */
/* ------------------------------------------------------------------ */
typedef struct {
  size_t n, k, p;
  int global;
  const uint64_t *rowptr, *cols;
  const double *vals, *b;
  double tol;
  uint64_t max_iter;
  uint64_t iterations;
} bench_job;

static void* bench_thread(void* arg) {
  bench_job* j = (bench_job*)arg;
  double* x = (double*)malloc(j->n * j->k * sizeof(double));
  orc_report rep;
  orc_bcg_solve(j->n, j->rowptr, j->cols, j->vals, ORC_PRECOND_IDENTITY, j->k, j->p, j->global,
                j->b, NULL, j->tol, j->max_iter, 0, NULL, 0, x, NULL, &rep);
  j->iterations = rep.iterations;
  free(x);
  return NULL;
}

double orc_bench_solve(int threads, size_t n, const uint64_t* rowptr, const uint64_t* cols,
                       const double* vals, size_t k, size_t p, int global, const double* b,
                       double tol, uint64_t max_iter, uint64_t* iterations) {
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  bench_job* jobs = (bench_job*)malloc(sizeof(bench_job) * threads);
  const double t0 = now_s();
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (bench_job){n, k, p, global, rowptr, cols, vals, b, tol, max_iter, 0};
    pthread_create(&th[t], NULL, bench_thread, &jobs[t]);
  }
  uint64_t total = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    total += jobs[t].iterations;
  }
  const double dt = now_s() - t0;
  if (iterations) *iterations = total;
  free(th);
  free(jobs);
  return dt;
}
