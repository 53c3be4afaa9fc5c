// host.cuh — host-side helpers shared by api.cu (single device solver and
// the C ABI) and psolver.cu (row-partitioned solver).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "fast_table.cuh"

namespace bkg {

void activate(bkg_ctx* c);
int elem_grid(const bkg_ctx* c, int64_t total);
void launch(bkg_ctx* c, const void* fn, int grid, int block, size_t smem, void** args);
void allow_smem(const void* fn, int bytes);
int occupancy_grid(const bkg_ctx* c, const void* fn, int smem, int64_t rows, int rpc,
                   int threads = 256);
bool use_fast(const bkg_ctx* c, int k, int p, bool global, FastTable* t);
// per-matrix K1 choices (api.cu): k1_stage (ring depth, smem out), k1_line
bool use_stage(bkg_ctx* c, const bkg_matrix* A, const FastTable& ft, int K, int* ns, int* smem);
bool use_line(bkg_ctx* c, const bkg_matrix* A, const FastTable& ft);
bool use_grid(bkg_ctx* c, const bkg_matrix* A, const FastTable& ft, int K, GridArgs* g, int* ctas,
              int* smem, bool* two_d);
// grid.cu: constant-coefficient grid stencil detection, k1_grid plan and tensor map
const GridStencil& grid_stencil(bkg_ctx* c, const bkg_matrix* A);
void grid_stencil_rows(bkg_ctx* c, int64_t n, const int64_t* rowptr, const int32_t* cols,
                       const double* vals, int64_t r0, int64_t nglobal, GridStencil& st);
void grid_plan(const GridStencil& st, int K, int sm_count, int ns, int zbeg, int zend, int zoff,
               int nzt, GridArgs* g, int* ctas);
void grid_plan_ends(const GridStencil& st, int K, int sm_count, int ns, bool lower, bool upper,
                    int zoff, int nzt, GridArgs* g, int* ctas);
void grid_tensor_map(const double* P, int K, int nx, int ny, int nz, void* out);
void grid_dia_tensor_map(const double* V, int nx, int ny, int nz, int slots, void* out);
// 2-D grids (k1_grid2)
void grid2_plan(const GridStencil& st, int K, int sm_count, int ns, GridArgs* g, int* ctas);
void grid2_tensor_map(const double* P, int K, int nx, int ny, void* out);
void grid2_dia_tensor_map(const double* V, int nx, int ny, int slots, void* out);
int grid_ring_depth(const FastTable& ft, int K, int per_cta);
// 2-D tensor map of a row-major n x K block vector, box = 16 columns x `rows` rows
void tile_tensor_map(const double* P, int K, int64_t n, int rows, void* out);
// generate.cu: device-side problem generation
void dev_generate_rhs(bkg_ctx* c, int normal, int64_t n, int k, uint64_t seed, double* dst,
                      int64_t row0 = 0);
void dev_generate_stencil_rows(bkg_ctx* c, int kind, int64_t nx, int64_t ny, int64_t nz,
                               uint64_t seed, double contrast, int64_t r0, int64_t r1,
                               int64_t cshift, int64_t* rowptr, int32_t* cols, double* vals);
// stage.cu: staged-block copy for k1_stage (grid boxes or consecutive rows)
bool grid_detect(bkg_ctx* c, int64_t n, const int64_t* rowptr, const int32_t* cols,
                 int64_t grid[3], std::vector<int64_t>* offsets = nullptr);
bool stage_build(bkg_ctx* c, int64_t n, const int64_t* rowptr, const int32_t* cols,
                 const double* vals, int R, const int box[3], const int64_t grid[3], int strip,
                 int max_segs, StageCsr& out);
// k1_stage arguments of a built StageCsr (all blocks in order; ring depth ns)
inline void stage_args(IterArgs& a, const StageCsr& st, int ns) {
  a.stg_hdr = st.hdr.ptr;
  a.stg_segs = st.segs.ptr;
  a.stg_vals = st.vals.ptr;
  a.stg_lidx = st.lidx.ptr;
  a.stg_rowid = st.rowid.ptr;
  a.stg_nstage = ns;
  a.stg_cap = st.cap;
  a.stg_wmax = st.wmax;
  a.stg_smax = st.smax;
  a.stg_R = st.R;
  a.stg_cnt = st.nblk;
  a.stg_map = nullptr;
  const char* dbg = std::getenv("BKG_STAGE_DEBUG");
  a.stg_debug = dbg ? std::atoi(dbg) : 0;
}
int64_t stencil_rows_nnz(int kind, int64_t nx, int64_t ny, int64_t nz, int64_t r0, int64_t r1);
void dev_generate_stencil(bkg_ctx* c, int kind, int64_t nx, int64_t ny, int64_t nz,
                          uint64_t seed, double contrast, bkg_matrix* m);
void check_cfg(uint64_t k, uint64_t p, int mode);
void dev_gram(bkg_ctx* c, int64_t n, int k, int p, bool global, const double* x, const double* y,
              double* out, bool force_exact);
// Build (or rebuild) `out` as the sliced-ELL copy of a device CSR with slice
// height R; buffers are reused when large enough (spare: donor buffers).
void sell_build(bkg_ctx* c, int64_t n, const int64_t* rowptr, const int32_t* cols,
                const double* vals, int R, SellCsr& out, SellCsr* spare = nullptr, int run = 0);
void dev_spmm(bkg_ctx* c, const bkg_matrix* A, int k, const double* x, double* y, const Ctrl* ctrl,
              bool force_exact);

// Reduction scratch (partials, group partials, tickets) owned by a context.
struct Scratch {
  double* partials;
  double* gpart;
  Ctrl* ctrl;
};

template <class T>
void h2d(bkg_ctx* c, T* dst, const T* src, size_t count) {
  if (count)
    BKG_CUDA_CHECK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
}
template <class T>
void d2h(bkg_ctx* c, T* dst, const T* src, size_t count) {
  if (count)
    BKG_CUDA_CHECK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
}
template <class T>
void d2d(bkg_ctx* c, T* dst, const T* src, size_t count) {
  if (count)
    BKG_CUDA_CHECK(
        cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
}
inline void sync(bkg_ctx* c) { BKG_CUDA_CHECK(cudaStreamSynchronize(c->stream)); }

}  // namespace bkg
