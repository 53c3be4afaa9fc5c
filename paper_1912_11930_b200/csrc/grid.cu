// grid.cu — host side of k1_grid (kernels_grid.cuh): exact detection of a
// constant-coefficient grid stencil in a device CSR matrix, the work plan and
// the TMA tensor map of a block vector.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "bkg.h"
#include "common.cuh"
#include "host.cuh"
#include "kernels_grid.cuh"
#include "kernels_grid2.cuh"

namespace bkg {

namespace {

struct Coef27 {
  double c[27];
};

// Every row must hold exactly the in-grid offsets with a nonzero coefficient,
// in ascending column order, each with the stencil's value bit for bit.
// Rows are global rows r0 .. r0 + n - 1 of an nx x ny x nz grid and the stored
// columns are global - r0 (a z-slab part of psolver.cu; r0 = 0: a whole matrix).
__global__ void k_grid_check(int64_t n, int64_t r0, int nx, int ny, int nz,
                             const int64_t* __restrict__ rowptr,
                             const int32_t* __restrict__ cols, const double* __restrict__ vals,
                             Coef27 cf, int* __restrict__ bad) {
  const int64_t ng = (int64_t)nx * ny * nz;
  for (int64_t rl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; rl < n;
       rl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rl + r0;
    const int x = (int)(r % nx), y = (int)((r / nx) % ny), z = (int)(r / ((int64_t)nx * ny));
    int expect = 0;
    for (int o = 0; o < 27; ++o) {
      const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
      if (cf.c[o] != 0.0 && x + dx >= 0 && x + dx < nx && y + dy >= 0 && y + dy < ny &&
          z + dz >= 0 && z + dz < nz)
        ++expect;
    }
    const int64_t e0 = rowptr[rl], e1 = rowptr[rl + 1];
    bool ok = e1 - e0 == expect;
    int64_t prev = -1;
    for (int64_t e = e0; ok && e < e1; ++e) {
      const int64_t c = (int64_t)cols[e] + r0;
      if (c <= prev || c < 0 || c >= ng) {
        ok = false;
        break;
      }
      prev = c;
      const int dx = (int)(c % nx) - x, dy = (int)((c / nx) % ny) - y,
                dz = (int)(c / ((int64_t)nx * ny)) - z;
      if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) {
        ok = false;
        break;
      }
      const double want = cf.c[(dz + 1) * 9 + (dy + 1) * 3 + dx + 1];
      if (want == 0.0 || __double_as_longlong(want) != __double_as_longlong(vals[e])) ok = false;
    }
    if (!ok) *bad = 1;
  }
}

// Variable coefficients: every entry must sit on the 5 / 7-point star of its
// row (columns ascending); its value goes to V[slot * n + row] (V zeroed before).
__global__ void k_grid_dia(int64_t n, int nx, int ny, int nz, const int64_t* __restrict__ rowptr,
                           const int32_t* __restrict__ cols, const double* __restrict__ vals,
                           double* __restrict__ V, int* __restrict__ bad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(r % nx), y = (int)((r / nx) % ny), z = (int)(r / ((int64_t)nx * ny));
    int64_t prev = -1;
    bool ok = true;
    for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
      const int64_t c = cols[e];
      if (c <= prev || c < 0 || c >= n) {
        ok = false;
        break;
      }
      prev = c;
      const int dx = (int)(c % nx) - x, dy = (int)((c / nx) % ny) - y,
                dz = (int)(c / ((int64_t)nx * ny)) - z;
      const int ad = (dx < 0 ? -dx : dx) + (dy < 0 ? -dy : dy) + (dz < 0 ? -dz : dz);
      if (ad > 1) {
        ok = false;
        break;
      }
      const int slot = dz ? (dz < 0 ? 0 : 6) : dy ? (dy < 0 ? 1 : 5) : dx ? (dx < 0 ? 2 : 4) : 3;
      V[(int64_t)slot * n + r] = vals[e];
    }
    if (!ok) *bad = 1;
  }
}

}  // namespace

// Rows [r0, r0 + n) of a global matrix of `nglobal` rows, stored with columns
// global - r0: grid shape from the column offsets (grid_detect), coefficients
// from one interior row, then the exact check of every row.  st.nz / st.zs are
// the part's planes and its first global plane (whole matrix: r0 = 0).
void grid_stencil_rows(bkg_ctx* c, int64_t n, const int64_t* rowptr, const int32_t* cols,
                       const double* vals, int64_t r0, int64_t nglobal, GridStencil& st) {
  st = GridStencil{};
  st.checked = true;
  st.n = n;
  int64_t grid[3];
  if (nglobal >= (int64_t)1 << 31 || !grid_detect(c, n, rowptr, cols, grid)) return;
  if (grid[0] < 3 || grid[1] < 3 || grid[2] < 1) return;
  if (grid[0] > (1 << 20) || grid[1] > (1 << 20)) return;
  const int nx = (int)grid[0], ny = (int)grid[1];
  const int64_t plane = (int64_t)nx * ny;
  if (r0 % plane != 0 || nglobal % plane != 0 || n % plane != 0) return;  // whole planes only
  if (nglobal / plane > (1 << 20) || nglobal / plane == 2) return;  // 2-D (one plane) or 3-D
  const int nz = (int)(n / plane), nzg = (int)(nglobal / plane), zs = (int)(r0 / plane);
  // a row away from every face of the global grid
  int zm = nz / 2;
  if (nzg > 1) {
    if (zs + zm < 1) zm = 1 - zs;
    if (zs + zm > nzg - 2) zm = nzg - 2 - zs;
  }
  if (zm < 0 || zm >= nz) return;
  const int64_t mid = ((int64_t)zm * ny + ny / 2) * nx + nx / 2;
  int64_t rp[2];
  d2h(c, rp, rowptr + mid, 2);
  sync(c);
  const int64_t cnt = rp[1] - rp[0];
  if (cnt <= 0 || cnt > 27) return;
  std::vector<int32_t> cl(cnt);
  std::vector<double> vl(cnt);
  d2h(c, cl.data(), cols + rp[0], cnt);
  d2h(c, vl.data(), vals + rp[0], cnt);
  sync(c);
  Coef27 cf{};
  for (int64_t e = 0; e < cnt; ++e) {
    const int64_t d = (int64_t)cl[e] - mid;  // column offset of an interior row
    // d = dz plane + dy nx + dx with |dx|, |dy|, |dz| <= 1
    int dz = 0, dy = 0;
    int64_t rem = d;
    if (rem > plane / 2) dz = 1;
    if (rem < -(plane / 2)) dz = -1;
    rem -= dz * plane;
    if (rem > nx / 2) dy = 1;
    if (rem < -(nx / 2)) dy = -1;
    rem -= (int64_t)dy * nx;
    if (rem < -1 || rem > 1) return;
    if (vl[e] == 0.0) return;
    cf.c[(dz + 1) * 9 + (dy + 1) * 3 + (int)rem + 1] = vl[e];
  }
  DevBuf<int> bad(1);
  BKG_CUDA_CHECK(cudaMemsetAsync(bad.ptr, 0, sizeof(int), c->stream));
  {
    int64_t nn = n, rr = r0;
    int ax = nx, ay = ny, az = nzg;
    int* bp = bad.ptr;
    void* args[] = {&nn, &rr, &ax, &ay, &az, &rowptr, &cols, &vals, &cf, &bp};
    launch(c, (const void*)&k_grid_check, elem_grid(c, n), 256, 0, args);
  }
  int hbad = 1;
  d2h(c, &hbad, bad.ptr, 1);
  sync(c);
  st.nx = nx;
  st.ny = ny;
  st.nz = nz;
  st.zs = zs;
  st.nzg = nzg;
  if (hbad) {
    // not one value per offset: variable coefficients on a 5 / 7-point star?
    // (whole matrices; TMA strides need an even nx)
    // BKG_GRID_VAR=0 turns it off.  B200: C3 (2-D) K1 0.313 -> 0.215 ms; 3-D
    // D A D of the 7-point stencil, 128^3 k = 32: 0.351 -> 0.244 ms, 160^3 k = 64:
    // 1.82 -> 0.86 ms (tools/var3d_probe.py).
    const char* ev = std::getenv("BKG_GRID_VAR");
    const bool want = !(ev && ev[0] == '0');
    if (r0 != 0 || nglobal != n || (nx & 1) || !want) return;
    st.dia.alloc((size_t)7 * n);
    BKG_CUDA_CHECK(cudaMemsetAsync(st.dia.ptr, 0, st.dia.bytes(), c->stream));
    BKG_CUDA_CHECK(cudaMemsetAsync(bad.ptr, 0, sizeof(int), c->stream));
    int64_t nn = n;
    int ax = nx, ay = ny, az = nz;
    double* vp = st.dia.ptr;
    int* bp = bad.ptr;
    void* args[] = {&nn, &ax, &ay, &az, &rowptr, &cols, &vals, &vp, &bp};
    launch(c, (const void*)&k_grid_dia, elem_grid(c, n), 256, 0, args);
    d2h(c, &hbad, bad.ptr, 1);
    sync(c);
    if (hbad)
      st.dia.release();
    else
      st.var = true;
    return;
  }
  st.ok = true;
  for (int o = 0; o < 27; ++o) {
    st.c[o / 9][o % 9] = cf.c[o];
    const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
    if (cf.c[o] != 0.0 && (dx != 0) + (dy != 0) + (dz != 0) > 1) st.full27 = true;
  }
  // isotropic: the coefficient depends only on the number of nonzero offsets
  st.iso27 = st.full27;
  for (int o = 0; o < 27 && st.iso27; ++o) {
    const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
    const int cls = (dx != 0) + (dy != 0) + (dz != 0);
    const double want = cls == 0 ? cf.c[13] : cls == 1 ? cf.c[12] : cls == 2 ? cf.c[9] : cf.c[0];
    if (cf.c[o] != want) st.iso27 = false;
  }
  const char* ei = std::getenv("BKG_GRID_ISO");
  if (ei && ei[0] == '0') st.iso27 = false;
}

// A->gridst, cached per matrix.
const GridStencil& grid_stencil(bkg_ctx* c, const bkg_matrix* A) {
  GridStencil& st = A->gridst;
  const int64_t n = (int64_t)A->n;
  if (st.checked && st.n == n) return st;
  grid_stencil_rows(c, n, A->rowptr.ptr, A->cols.ptr, A->vals.ptr, 0, n, st);
  return st;
}

// Work plan: z-chunk length that maximises (CTA utilisation) / (1 + 2 / chunk)
// -- each item reads two extra planes -- for a persistent grid of `ctas` CTAs
// (a multiple of the K / 16 slices, so a CTA keeps one slice).
// Rows produced: planes [zbeg, zend) of the part; zoff = the part's plane 0 in
// the operand tensor.
void grid_plan(const GridStencil& st, int K, int sm_count, int ns, int zbeg, int zend, int zoff,
               int nzt, GridArgs* g, int* ctas) {
  const int nsl = K / kGridW;
  const int nzr = zend - zbeg;
  std::memset(g, 0, sizeof(*g));
  g->nx = st.nx;
  g->ny = st.ny;
  g->nz = st.nz;
  g->zbeg = zbeg;
  g->zend = zend;
  g->zoff = zoff;
  g->tmin = -zoff;            // planes of the operand tensor, in part coordinates
  g->tmax = nzt - 1 - zoff;
  g->tx = (st.nx + kGridBX - 1) / kGridBX;
  g->ty = (st.ny + kGridBY - 1) / kGridBY;
  g->ns = ns;
  std::memcpy(g->c, st.c, sizeof(g->c));
  const int64_t T = (int64_t)g->tx * g->ty * nsl;
  const int64_t G = std::max<int64_t>(nsl, (int64_t)(sm_count / nsl) * nsl);
  double best = -1.0;
  int best_chunk = nzr;
  for (int nzc = 1; nzc <= std::max(1, nzr / 4); ++nzc) {
    const int chunk = (nzr + nzc - 1) / nzc;
    const int real = (nzr + chunk - 1) / chunk;
    const int64_t items = T * real;
    const int64_t grid = std::min(G, items);
    const int64_t rounds = (items + grid - 1) / grid;
    const double util = (double)items / (double)(rounds * grid) * ((double)grid / (double)G);
    const double score = util / (1.0 + 2.0 / chunk);
    if (score > best * 1.0001) {
      best = score;
      best_chunk = chunk;
    }
  }
  const char* ez = std::getenv("BKG_GRID_ZCHUNK");
  if (ez && std::atoi(ez) > 0) best_chunk = std::min(nzr, std::atoi(ez));
  g->zchunk = best_chunk;
  g->zstride = best_chunk;
  g->nzc = (nzr + best_chunk - 1) / best_chunk;
  g->nitems = T * g->nzc;
  *ctas = (int)std::min(G, g->nitems);
  // Lockstep pacing pays over long launches only (B200 sweeps, DESIGN.md §5:
  // C5, 28 rounds of 66 planes per CTA, 3.23 -> 3.05 ms with loose pacing; C2,
  // 7 rounds of 18, loses 3%; one round starts in step by itself)
  const char* es = std::getenv("BKG_GRID_SYNC");
  const char* el = std::getenv("BKG_GRID_LEAD");
  const int64_t rounds = (g->nitems + *ctas - 1) / *ctas;
  g->sync_every = es ? std::atoi(es) : (rounds * (g->zchunk + 2) >= 512 ? 16 : 0);
  g->sync_lead = el ? std::max(0, std::atoi(el)) : 1;
}

// 2-D grids (k1_grid2, kernels_grid2.cuh): items = (y-chunk, 128-point x tile,
// slice) for a persistent grid of 2 CTAs per SM; y-chunk by the same score.
void grid2_plan(const GridStencil& st, int K, int sm_count, int ns, GridArgs* g, int* ctas) {
  const int nsl = K / kGridW;
  std::memset(g, 0, sizeof(*g));
  g->nx = st.nx;
  g->ny = st.ny;
  g->nz = 1;
  g->tx = (st.nx + kG2BX - 1) / kG2BX;
  g->ty = 1;
  g->ns = ns;
  g->zbeg = 0;
  g->zend = st.ny;
  g->zoff = 0;
  g->tmin = 0;
  g->tmax = st.ny - 1;
  std::memcpy(g->c, st.c, sizeof(g->c));
  const int64_t T = (int64_t)g->tx * nsl;
  const int64_t G = std::max<int64_t>(nsl, (int64_t)(2 * sm_count / nsl) * nsl);
  double best = -1.0;
  int best_chunk = st.ny;
  for (int nyc = 1; nyc <= std::max(1, st.ny / 8); ++nyc) {
    const int chunk = (st.ny + nyc - 1) / nyc;
    const int real = (st.ny + chunk - 1) / chunk;
    const int64_t items = T * real;
    const int64_t grid = std::min(G, items);
    const int64_t rounds = (items + grid - 1) / grid;
    const double util = (double)items / (double)(rounds * grid) * ((double)grid / (double)G);
    const double score = util / (1.0 + 2.0 / chunk);
    if (score > best * 1.0001) {
      best = score;
      best_chunk = chunk;
    }
  }
  const char* ez = std::getenv("BKG_GRID_ZCHUNK");
  if (ez && std::atoi(ez) > 0) best_chunk = std::min(st.ny, std::atoi(ez));
  g->zchunk = best_chunk;
  g->zstride = best_chunk;
  g->nzc = (st.ny + best_chunk - 1) / best_chunk;
  g->nitems = T * g->nzc;
  *ctas = (int)std::min(G, g->nitems);
}

// The two single-plane items per (tile, slice) at the ends of a z-slab part:
// planes 0 and nz - 1 (the rows that read the neighbours' ghost planes).
void grid_plan_ends(const GridStencil& st, int K, int sm_count, int ns, bool lower, bool upper,
                    int zoff, int nzt, GridArgs* g, int* ctas) {
  const int first = lower ? 0 : st.nz - 1;
  grid_plan(st, K, sm_count, ns, first, first + 1, zoff, nzt, g, ctas);
  if (lower && upper && st.nz > 1) {
    g->zend = st.nz;
    g->zstride = st.nz - 1;
    g->nzc = 2;
    g->nitems *= 2;
    const int nsl = K / kGridW;
    *ctas = (int)std::min<int64_t>(std::max<int64_t>(nsl, (int64_t)(sm_count / nsl) * nsl),
                                   g->nitems);
  }
  g->sync_every = 0;
}

// TMA tensor map of a row-major n x K block vector seen as (column, x, y, z),
// box = one 16-column plane tile with its halo, 128-byte swizzle, zero fill.
namespace {
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn tensor_map_encoder() {
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qres;
    BKG_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres));
    BKG_REQUIRE(fn && qres == cudaDriverEntryPointSuccess, BKG_CUDA,
                "cuTensorMapEncodeTiled is not available from the driver");
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  return encode;
}
}  // namespace

// 2-D tensor map of a row-major n x K block vector (column, row), box = one
// 16-column x `rows`-row tile, 128-byte swizzle; rows past n read as zero and
// are not written (kernels_tma.cuh).
void tile_tensor_map(const double* P, int K, int64_t n, int rows, void* out) {
  EncodeFn encode = tensor_map_encoder();
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 8};
  const cuuint32_t box[2] = {kGridW, (cuuint32_t)rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = encode(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                             2, const_cast<double*>(P), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BKG_REQUIRE(rc == CUDA_SUCCESS, BKG_CUDA,
              "cuTensorMapEncodeTiled (2-D) failed (" + std::to_string((int)rc) + ")");
}

// Tensor maps of the DIA copy V seen as (x, y, z, slot): boxes of one 16 x 16
// tile x `slots` slots (5: the in-plane slots, 1: a dz slot); zero fill.
void grid_dia_tensor_map(const double* V, int nx, int ny, int nz, int slots, void* out) {
  EncodeFn encode = tensor_map_encoder();
  const cuuint64_t dims[4] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz, 7};
  const cuuint64_t strides[3] = {(cuuint64_t)8 * nx, (cuuint64_t)8 * nx * ny,
                                 (cuuint64_t)8 * nx * ny * nz};
  const cuuint32_t box[4] = {kGridBX, kGridBY, 1, (cuuint32_t)slots};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult rc = encode(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                             4, const_cast<double*>(V), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BKG_REQUIRE(rc == CUDA_SUCCESS, BKG_CUDA,
              "cuTensorMapEncodeTiled (DIA) failed (" + std::to_string((int)rc) + ")");
}

// k1_grid2: a row-major n x K block vector of a 2-D grid as (column, x, y), box =
// 16 columns x one 128-point line tile with its two x neighbours; and its DIA
// copy as (x, y, slot), boxes of `slots` slots.
void grid2_tensor_map(const double* P, int K, int nx, int ny, void* out) {
  EncodeFn encode = tensor_map_encoder();
  const cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)nx, (cuuint64_t)ny};
  const cuuint64_t strides[2] = {(cuuint64_t)K * 8, (cuuint64_t)K * 8 * nx};
  const cuuint32_t box[3] = {kGridW, kG2BX + 2, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult rc = encode(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                             3, const_cast<double*>(P), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BKG_REQUIRE(rc == CUDA_SUCCESS, BKG_CUDA,
              "cuTensorMapEncodeTiled (2-D grid) failed (" + std::to_string((int)rc) + ")");
}
void grid2_dia_tensor_map(const double* V, int nx, int ny, int slots, void* out) {
  EncodeFn encode = tensor_map_encoder();
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, 7};
  const cuuint64_t strides[2] = {(cuuint64_t)8 * nx, (cuuint64_t)8 * nx * ny};
  const cuuint32_t box[3] = {kG2BX, 1, (cuuint32_t)slots};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult rc = encode(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                             3, const_cast<double*>(V), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BKG_REQUIRE(rc == CUDA_SUCCESS, BKG_CUDA,
              "cuTensorMapEncodeTiled (2-D DIA) failed (" + std::to_string((int)rc) + ")");
}

void grid_tensor_map(const double* P, int K, int nx, int ny, int nz, void* out) {
  EncodeFn encode = tensor_map_encoder();
  const cuuint64_t dims[4] = {(cuuint64_t)K, (cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  const cuuint64_t strides[3] = {(cuuint64_t)K * 8, (cuuint64_t)K * 8 * nx,
                                 (cuuint64_t)K * 8 * nx * ny};
  const cuuint32_t box[4] = {kGridW, kGridBX + 2, kGridBY + 2, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult rc = encode(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                             4, const_cast<double*>(P), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BKG_REQUIRE(rc == CUDA_SUCCESS, BKG_CUDA,
              "cuTensorMapEncodeTiled failed (" + std::to_string((int)rc) + ")");
}

}  // namespace bkg
