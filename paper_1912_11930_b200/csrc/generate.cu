// generate.cu — device-side problem generation: the
// stencil matrices straight into the device CSR and the block right hand
// sides straight into HBM, so large configurations (C4, C5: GB-sized CSR and
// RHS) skip host assembly and the PCIe upload.
//
//   * Stencils: one thread per row; the row's first entry comes from a closed
//     form of the per-axis neighbour counts (no scan), entries in ascending
//     column order as problems.cpp / problems.hpp:74-124 emit them.  Kinds 0,
//     3, 4 use only exactly rounded arithmetic; kinds 1, 2 take their cell
//     coefficients (n host pow/exp values, problems.cpp coefficient_field)
//     and assemble the harmonic faces with __dmul_rn/__ddiv_rn/__dadd_rn in
//     the host's order — every kind is bit-identical to bkg_stencil_fill.
//   * random_block_rhs (U(-1,1)): each thread jumps the Xorshift64Star stream
//     to its first draw (rng.h) and continues serially: bit-identical.
//   * normal_block_rhs: the same draws; Box-Muller uses CUDA's log / sqrt /
//     cos / sin, so values agree with the host generator to a few ulp, not
//     bit for bit (documented in DESIGN.md §Inputs).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bkg.h"
#include "common.cuh"
#include "host.cuh"
#include "rng.h"

namespace bkg {

void coefficient_field(int kind, uint64_t seed, double contrast, uint64_t n, double* coeff);

namespace {

__host__ __device__ __forceinline__ int64_t nb(int64_t c, int64_t N) {
  return (c > 0) + (c < N - 1);
}
// sum of nb(c') over c' < c, for c <= N - 1
__host__ __device__ __forceinline__ int64_t nb_prefix(int64_t c) { return c == 0 ? 0 : 2 * c - 1; }

// Entries of the rows before row r (closed form over the per-axis neighbour
// counts; the CSR row offset of r without a scan).
__host__ __device__ __forceinline__ int64_t first_entry_7pt(int64_t nx, int64_t ny, int64_t nz,
                                                            int64_t r) {
  const int64_t i = r % nx, j = (r / nx) % ny, l = r / (nx * ny);
  int64_t e = r;
  e += (l * ny + j) * 2 * (nx - 1) + nb_prefix(i);
  e += l * nx * 2 * (ny - 1) + nx * nb_prefix(j) + i * nb(j, ny);
  if (nz > 1) e += nx * ny * nb_prefix(l) + (j * nx + i) * nb(l, nz);
  return e;
}
__host__ __device__ __forceinline__ int64_t first_entry_27pt(int64_t nx, int64_t ny, int64_t nz,
                                                             int64_t r) {
  const int64_t Cx = 3 * nx - 2, Cy = 3 * ny - 2;
  const int64_t i = r % nx, j = (r / nx) % ny, l = r / (nx * ny);
  const int64_t cx = 1 + nb(i, nx), cy = 1 + nb(j, ny), cz = 1 + nb(l, nz);
  const int64_t tx = i + nb_prefix(i), ty = j + nb_prefix(j), tz = l + nb_prefix(l);
  return Cx * Cy * tz + cz * (Cx * ty + cy * tx);
}

__device__ __forceinline__ double harmonic(double a, double b) {
  return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, a), b), __dadd_rn(a, b));
}

// 7-point 3D (kind 3) and 5-point 2D (kinds 0-2, nz = 1, coeff != nullptr).
// Rows [r0, r1) of the global matrix: row offsets relative to row r0's first
// entry e0, columns stored as (global column - cshift) -- the whole matrix for
// r0 = 0, r1 = n, e0 = cshift = 0; one rank's slab of a row partition
// otherwise (psolver local columns).
__global__ void k_gen_7pt(int64_t nx, int64_t ny, int64_t nz, const double* __restrict__ coeff,
                          int64_t* __restrict__ rowptr, int32_t* __restrict__ cols,
                          double* __restrict__ vals, int64_t r0, int64_t r1, int64_t e0,
                          int64_t cshift) {
  for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = r % nx, j = (r / nx) % ny, l = r / (nx * ny);
    // entries before row r: one diagonal per row + the axis links of rows < r
    int64_t e = first_entry_7pt(nx, ny, nz, r) - e0;
    if (r == r0) rowptr[0] = 0;
    const int64_t count = 1 + nb(i, nx) + nb(j, ny) + (nz > 1 ? nb(l, nz) : 0);
    rowptr[r - r0 + 1] = e + count;
    if (coeff) {  // 2D heterogeneous Poisson (problems.hpp:100-120 assembly order)
      const double cr = coeff[r];
      double diag = 0.0, s = 0.0, w = 0.0, ea = 0.0, no = 0.0;
      diag = __dadd_rn(diag, j > 0 ? (s = harmonic(cr, coeff[r - nx])) : cr);
      diag = __dadd_rn(diag, i > 0 ? (w = harmonic(cr, coeff[r - 1])) : cr);
      diag = __dadd_rn(diag, i + 1 < nx ? (ea = harmonic(cr, coeff[r + 1])) : cr);
      diag = __dadd_rn(diag, j + 1 < ny ? (no = harmonic(cr, coeff[r + nx])) : cr);
      if (j > 0) { cols[e] = (int32_t)(r - nx - cshift); vals[e++] = -s; }
      if (i > 0) { cols[e] = (int32_t)(r - 1 - cshift); vals[e++] = -w; }
      cols[e] = (int32_t)(r - cshift);
      vals[e++] = diag;
      if (i + 1 < nx) { cols[e] = (int32_t)(r + 1 - cshift); vals[e++] = -ea; }
      if (j + 1 < ny) { cols[e] = (int32_t)(r + nx - cshift); vals[e++] = -no; }
    } else {  // 3D 7-point Laplacian: diag 6, off -1
      const int64_t plane = nx * ny;
      if (l > 0) { cols[e] = (int32_t)(r - plane - cshift); vals[e++] = -1.0; }
      if (j > 0) { cols[e] = (int32_t)(r - nx - cshift); vals[e++] = -1.0; }
      if (i > 0) { cols[e] = (int32_t)(r - 1 - cshift); vals[e++] = -1.0; }
      cols[e] = (int32_t)(r - cshift);
      vals[e++] = 6.0;
      if (i + 1 < nx) { cols[e] = (int32_t)(r + 1 - cshift); vals[e++] = -1.0; }
      if (j + 1 < ny) { cols[e] = (int32_t)(r + nx - cshift); vals[e++] = -1.0; }
      if (l + 1 < nz) { cols[e] = (int32_t)(r + plane - cshift); vals[e++] = -1.0; }
    }
  }
}

// 27-point 3D (kind 4): count = cx cy cz with c = 1 + nb per axis.
__global__ void k_gen_27pt(int64_t nx, int64_t ny, int64_t nz, int64_t* __restrict__ rowptr,
                           int32_t* __restrict__ cols, double* __restrict__ vals, int64_t r0,
                           int64_t r1, int64_t e0, int64_t cshift) {
  for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = r % nx, j = (r / nx) % ny, l = r / (nx * ny);
    const int64_t cx = 1 + nb(i, nx), cy = 1 + nb(j, ny), cz = 1 + nb(l, nz);
    int64_t e = first_entry_27pt(nx, ny, nz, r) - e0;
    if (r == r0) rowptr[0] = 0;
    rowptr[r - r0 + 1] = e + cx * cy * cz;
    for (int dl = -1; dl <= 1; ++dl)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          const int64_t ii = i + di, jj = j + dj, ll = l + dl;
          if (ii < 0 || jj < 0 || ll < 0 || ii >= nx || jj >= ny || ll >= nz) continue;
          const int64_t c = (ll * ny + jj) * nx + ii;
          cols[e] = (int32_t)(c - cshift);
          vals[e++] = c == r ? 26.0 : -1.0;
        }
  }
}

// values [b, e) of one generator thread: U(-1,1) draws, or Box-Muller pairs.
// The stream starts `skip` draws in (a slab of rows of a larger block).
__global__ void k_gen_rhs(int normal, int64_t count, int64_t per, uint64_t s0,
                          const uint64_t* __restrict__ table, double* __restrict__ out,
                          uint64_t skip) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (normal) {
    const int64_t pairs = (count + 1) / 2, b = t * per, e = min(pairs, b + per);
    if (b >= e) return;
    uint64_t s = rng::jump(table, s0, skip + 2 * (uint64_t)b);
    for (int64_t j = b; j < e; ++j) {
      const double u1 = rng::unit(s), u2 = rng::unit(s);
      const double rad = sqrt(__dmul_rn(-2.0, log(__dadd_rn(1.0, -u1))));
      const double th = __dmul_rn(6.283185307179586, u2);
      out[2 * j] = __dmul_rn(rad, cos(th));
      if (2 * j + 1 < count) out[2 * j + 1] = __dmul_rn(rad, sin(th));
    }
  } else {
    const int64_t b = t * per, e = min(count, b + per);
    if (b >= e) return;
    uint64_t s = rng::jump(table, s0, skip + (uint64_t)b);
    for (int64_t i = b; i < e; ++i) out[i] = rng::symmetric(s);
  }
}

const uint64_t* device_jump_table(bkg_ctx* c) {
  static thread_local std::vector<std::pair<int, DevBuf<uint64_t>*>> cache;
  for (auto& [dev, buf] : cache)
    if (dev == c->device) return buf->ptr;
  std::vector<uint64_t> h(64 * 64);
  rng::jump_table(h.data());
  auto* buf = new DevBuf<uint64_t>(h.size());  // lives for the process
  BKG_CUDA_CHECK(cudaMemcpy(buf->ptr, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
  cache.push_back({c->device, buf});
  return buf->ptr;
}

}  // namespace

// Rows [row0, row0 + n) of the n_total x k block (row0 = 0: the whole block).
void dev_generate_rhs(bkg_ctx* c, int normal, int64_t n, int k, uint64_t seed, double* dst,
                      int64_t row0) {
  const int64_t count = n * k;
  if (count == 0) return;
  BKG_REQUIRE(!normal || (row0 * k) % 2 == 0, BKG_CONFIG,
              "normal_block_rhs slab must start on a Box-Muller pair");
  uint64_t skip = (uint64_t)(row0 * k);
  const uint64_t* table = device_jump_table(c);
  const int64_t units = normal ? (count + 1) / 2 : count;
  const int64_t threads = std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)c->sm_count * 1024));
  int64_t per = (units + threads - 1) / threads;
  const int blocks = (int)((units + per * 256 - 1) / (per * 256));
  uint64_t s0 = rng::seed_state(seed);
  void* args[] = {&normal, const_cast<int64_t*>(&count), &per, &s0, &table, &dst, &skip};
  launch(c, (const void*)&k_gen_rhs, std::max(1, blocks), 256, 0, args);
}

// Rows [r0, r1) of a stencil matrix into rowptr (r1 - r0 + 1, from 0), cols
// (global column - cshift) and vals, which hold stencil_rows_nnz() entries.
void dev_generate_stencil_rows(bkg_ctx* c, int kind, int64_t nx, int64_t ny, int64_t nz,
                               uint64_t seed, double contrast, int64_t r0, int64_t r1,
                               int64_t cshift, int64_t* rowptr, int32_t* cols, double* vals) {
  const int64_t n = nx * ny * nz;
  DevBuf<double> coeff;
  const int64_t rows = r1 - r0;
  if (kind <= 2) {  // 2D: cell coefficients (ones for the constant field)
    std::vector<double> h(n, 1.0);
    if (kind != 0) coefficient_field(kind, seed, contrast, (uint64_t)n, h.data());
    coeff.alloc(n);
    h2d(c, coeff.ptr, h.data(), n);
    int64_t one = 1;
    const double* cp = coeff.ptr;
    int64_t e0 = first_entry_7pt(nx, ny, 1, r0);
    void* args[] = {&nx, &ny, &one, &cp, &rowptr, &cols, &vals, &r0, &r1, &e0, &cshift};
    launch(c, (const void*)&k_gen_7pt, elem_grid(c, rows), 256, 0, args);
  } else if (kind == 3) {
    const double* cp = nullptr;
    int64_t e0 = first_entry_7pt(nx, ny, nz, r0);
    void* args[] = {&nx, &ny, &nz, &cp, &rowptr, &cols, &vals, &r0, &r1, &e0, &cshift};
    launch(c, (const void*)&k_gen_7pt, elem_grid(c, rows), 256, 0, args);
  } else {
    int64_t e0 = first_entry_27pt(nx, ny, nz, r0);
    void* args[] = {&nx, &ny, &nz, &rowptr, &cols, &vals, &r0, &r1, &e0, &cshift};
    launch(c, (const void*)&k_gen_27pt, elem_grid(c, rows), 256, 0, args);
  }
  sync(c);  // coeff is released on return
}

int64_t stencil_rows_nnz(int kind, int64_t nx, int64_t ny, int64_t nz, int64_t r0, int64_t r1) {
  if (kind == 4) {  // first_entry_27pt holds for r < n; r == n: all (3nx-2)(3ny-2)(3nz-2)
    auto at = [&](int64_t r) {
      return r < nx * ny * nz ? first_entry_27pt(nx, ny, nz, r)
                              : (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2);
    };
    return at(r1) - at(r0);
  }
  const int64_t z = kind == 3 ? nz : 1;
  auto at = [&](int64_t r) {  // entries before row r; r == n: all of them
    const int64_t n = nx * ny * z;
    if (r < n) return first_entry_7pt(nx, ny, z, r);
    return first_entry_7pt(nx, ny, z, n - 1) + 1 + nb(nx - 1, nx) + nb(ny - 1, ny) +
           (z > 1 ? nb(z - 1, z) : 0);
  };
  return at(r1) - at(r0);
}

void dev_generate_stencil(bkg_ctx* c, int kind, int64_t nx, int64_t ny, int64_t nz,
                          uint64_t seed, double contrast, bkg_matrix* m) {
  dev_generate_stencil_rows(c, kind, nx, ny, nz, seed, contrast, 0, (int64_t)m->n, 0,
                            m->rowptr.ptr, m->cols.ptr, m->vals.ptr);
}

}  // namespace bkg
