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

namespace bkg {

namespace {

struct Coef27 {
  double c[27];
};

// Every row must hold exactly the in-grid offsets with a nonzero coefficient,
// in ascending column order, each with the stencil's value bit for bit.
__global__ void k_grid_check(int64_t n, int nx, int ny, int nz, const int64_t* __restrict__ rowptr,
                             const int32_t* __restrict__ cols, const double* __restrict__ vals,
                             Coef27 cf, int* __restrict__ bad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(r % nx), y = (int)((r / nx) % ny), z = (int)(r / ((int64_t)nx * ny));
    int expect = 0;
    for (int o = 0; o < 27; ++o) {
      const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
      if (cf.c[o] != 0.0 && x + dx >= 0 && x + dx < nx && y + dy >= 0 && y + dy < ny &&
          z + dz >= 0 && z + dz < nz)
        ++expect;
    }
    const int64_t e0 = rowptr[r], e1 = rowptr[r + 1];
    bool ok = e1 - e0 == expect;
    int64_t prev = -1;
    for (int64_t e = e0; ok && e < e1; ++e) {
      const int64_t c = cols[e];
      if (c <= prev || c < 0 || c >= n) {
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

}  // namespace

// Fills A->gridst (cached per matrix): grid shape from the column offsets
// (grid_detect), coefficients from one interior row, then the exact check.
const GridStencil& grid_stencil(bkg_ctx* c, const bkg_matrix* A) {
  GridStencil& st = A->gridst;
  const int64_t n = (int64_t)A->n;
  if (st.checked && st.n == n) return st;
  st = GridStencil{};
  st.checked = true;
  st.n = n;
  int64_t grid[3];
  if (n >= (int64_t)1 << 31 || !grid_detect(c, n, A->rowptr.ptr, A->cols.ptr, grid)) return st;
  if (grid[0] < 3 || grid[1] < 3 || grid[2] < 3) return st;  // 3-D only
  if (grid[0] > (1 << 20) || grid[1] > (1 << 20) || grid[2] > (1 << 20)) return st;
  const int nx = (int)grid[0], ny = (int)grid[1], nz = (int)grid[2];
  const int64_t mid = ((int64_t)(nz / 2) * ny + ny / 2) * nx + nx / 2;
  int64_t rp[2];
  d2h(c, rp, A->rowptr.ptr + mid, 2);
  sync(c);
  const int64_t cnt = rp[1] - rp[0];
  if (cnt <= 0 || cnt > 27) return st;
  std::vector<int32_t> cl(cnt);
  std::vector<double> vl(cnt);
  d2h(c, cl.data(), A->cols.ptr + rp[0], cnt);
  d2h(c, vl.data(), A->vals.ptr + rp[0], cnt);
  sync(c);
  Coef27 cf{};
  for (int64_t e = 0; e < cnt; ++e) {
    const int64_t col = cl[e];
    const int dx = (int)(col % nx) - nx / 2, dy = (int)((col / nx) % ny) - ny / 2,
              dz = (int)(col / ((int64_t)nx * ny)) - nz / 2;
    if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) return st;
    if (vl[e] == 0.0) return st;
    cf.c[(dz + 1) * 9 + (dy + 1) * 3 + dx + 1] = vl[e];
  }
  DevBuf<int> bad(1);
  BKG_CUDA_CHECK(cudaMemsetAsync(bad.ptr, 0, sizeof(int), c->stream));
  {
    int64_t nn = n;
    int ax = nx, ay = ny, az = nz;
    const int64_t* rpp = A->rowptr.ptr;
    const int32_t* cp = A->cols.ptr;
    const double* vp = A->vals.ptr;
    int* bp = bad.ptr;
    void* args[] = {&nn, &ax, &ay, &az, &rpp, &cp, &vp, &cf, &bp};
    launch(c, (const void*)&k_grid_check, elem_grid(c, n), 256, 0, args);
  }
  int hbad = 1;
  d2h(c, &hbad, bad.ptr, 1);
  sync(c);
  if (hbad) return st;
  st.ok = true;
  st.nx = nx;
  st.ny = ny;
  st.nz = nz;
  for (int o = 0; o < 27; ++o) {
    st.c[o / 9][o % 9] = cf.c[o];
    const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
    if (cf.c[o] != 0.0 && (dx != 0) + (dy != 0) + (dz != 0) > 1) st.full27 = true;
  }
  return st;
}

// Work plan: z-chunk length that maximises (CTA utilisation) / (1 + 2 / chunk)
// -- each item reads two extra planes -- for a persistent grid of `ctas` CTAs
// (a multiple of the K / 16 slices, so a CTA keeps one slice).
void grid_plan(const GridStencil& st, int K, int sm_count, int ns, GridArgs* g, int* ctas) {
  const int nsl = K / kGridW;
  std::memset(g, 0, sizeof(*g));
  g->nx = st.nx;
  g->ny = st.ny;
  g->nz = st.nz;
  g->tx = (st.nx + kGridBX - 1) / kGridBX;
  g->ty = (st.ny + kGridBY - 1) / kGridBY;
  g->ns = ns;
  std::memcpy(g->c, st.c, sizeof(g->c));
  const int64_t T = (int64_t)g->tx * g->ty * nsl;
  const int64_t G = std::max<int64_t>(nsl, (int64_t)(sm_count / nsl) * nsl);
  double best = -1.0;
  int best_chunk = st.nz;
  for (int nzc = 1; nzc <= std::max(1, st.nz / 4); ++nzc) {
    const int chunk = (st.nz + nzc - 1) / nzc;
    const int real = (st.nz + chunk - 1) / chunk;
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
  if (ez && std::atoi(ez) > 0) best_chunk = std::min(st.nz, std::atoi(ez));
  g->zchunk = best_chunk;
  g->nzc = (st.nz + best_chunk - 1) / best_chunk;
  g->nitems = T * g->nzc;
  *ctas = (int)std::min(G, g->nitems);
}

// TMA tensor map of a row-major n x K block vector seen as (column, x, y, z),
// box = one 16-column plane tile with its halo, 128-byte swizzle, zero fill.
void grid_tensor_map(const double* P, int K, const GridStencil& st, void* out) {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qres;
    BKG_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres));
    BKG_REQUIRE(fn && qres == cudaDriverEntryPointSuccess, BKG_CUDA,
                "cuTensorMapEncodeTiled is not available from the driver");
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t dims[4] = {(cuuint64_t)K, (cuuint64_t)st.nx, (cuuint64_t)st.ny,
                              (cuuint64_t)st.nz};
  const cuuint64_t strides[3] = {(cuuint64_t)K * 8, (cuuint64_t)K * 8 * st.nx,
                                 (cuuint64_t)K * 8 * st.nx * st.ny};
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
