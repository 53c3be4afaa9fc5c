// common.cuh — shared host/device plumbing for libbkgpu.so.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <set>

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "bkg.h"

namespace bkg {

// ---- error handling (thread-local last error, status codes) ------------
void set_error(const std::string& msg);
const char* last_error();

struct Status {
  int code;
  std::string msg;
};

class Error {
 public:
  Error(int code, std::string msg) : code_(code), msg_(std::move(msg)) {}
  int code() const { return code_; }
  const std::string& msg() const { return msg_; }

 private:
  int code_;
  std::string msg_;
};

#define BKG_CUDA_CHECK(expr)                                                          \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      throw ::bkg::Error(BKG_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define BKG_REQUIRE(cond, code, msg)            \
  do {                                          \
    if (!(cond)) throw ::bkg::Error(code, msg); \
  } while (0)

// ---- device ownership ---------------------------------------------------
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  void* base = nullptr;  // the allocation (ptr = base + a skew, alloc_skewed)
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count), base(o.base) {
    o.ptr = nullptr;
    o.base = nullptr;
    o.count = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      count = o.count;
      base = o.base;
      o.ptr = nullptr;
      o.base = nullptr;
      o.count = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t n) { alloc_skewed(n, 0); }
  // n elements starting skew_bytes (a multiple of 256) into the allocation:
  // block vectors whose size is a power of two would otherwise sit exactly
  // 2^m bytes apart and send the same row of every stream of a kernel to the
  // same L2 slice / DRAM bank (vec_skew, api.cu)
  void alloc_skewed(size_t n, size_t skew_bytes) {
    release();
    if (n == 0) return;
    BKG_CUDA_CHECK(cudaMalloc(&base, n * sizeof(T) + skew_bytes));
    ptr = reinterpret_cast<T*>(static_cast<char*>(base) + skew_bytes);
    count = n;
  }
  void ensure(size_t n) {
    if (n > count) alloc(n);
  }
  void release() {
    if (base) cudaFree(base);
    ptr = nullptr;
    base = nullptr;
    count = 0;
  }
  size_t bytes() const { return count * sizeof(T); }
};

// Per-solve device control block: stop flags, counters, grid-reduction
// tickets.  Lives in device memory; mirrored to the host each chunk.
struct Ctrl {
  int32_t done;        // 1 once converged / breakdown / max_iter
  int32_t converged;
  int32_t breakdown;
  int32_t stage;       // 0 normal; 1 lambda-breakdown; 2 beta-breakdown
  int32_t xpending;    // fast mode: K2 ran, K3 still owes X += P lambda
  int32_t xold;        // deferred X: the previous iteration's X += P lambda is pending
  uint64_t iterations; // completed iterations
  uint64_t max_iter;
  uint64_t breakdown_iteration;
  uint64_t breakdown_block;
  uint32_t tickets[64];  // [0..62] group tickets, [63] top ticket
  // k1_grid: plane copies issued by all CTAs of the running launch (lockstep
  // pacing, kernels_grid.cuh); zero between launches
  unsigned long long grid_sync;
};

constexpr int kMaxTicketGroups = 63;
// Column sentinel for inactive CSR slots: local column indices may be
// negative in the row-partitioned solver (ghost rows below the own block).
constexpr int kNoCol = -2147483647 - 1;

// Every iteration kernel returns immediately once the device stop flag is set
// (null ctrl: standalone kernel call, never stopped).
__device__ __forceinline__ bool stopped(const Ctrl* c) {
  return c != nullptr && *reinterpret_cast<const volatile int32_t*>(&c->done) != 0;
}

// Sliced-ELL copy of a CSR matrix for the fused K1 (kernels_k1.cuh): slices
// of R consecutive rows, each padded to its longest row and stored slot-major
// (entry (slot u, row i) of slice s at sptr[s] + u * R + i; padding: value 0,
// column kNoCol), so the R rows of a K1 warp tile read each slot's values and
// columns as one contiguous segment.  Built on device from the CSR.
//
// Line variant (run > 0, k1_line): slice s holds rows
// (s / run) * R * run + i * run + s % run, i < R -- each of the R rows of a
// warp step starts its own run of `run` consecutive rows -- and the entries in
// columns r - 1, r, r + 1 of row r are taken out of the slots into
// tri[(s * R + i) * 4 + {0, 1, 2}] (0 where absent), because k1_line keeps
// P[r - 1], P[r], P[r + 1] of its run in registers.
struct SellCsr {
  int rows = 0;  // slice height R (0: not built)
  int run = 0;   // line variant: rows per run (0: slices of R consecutive rows)
  int64_t n = 0;
  DevBuf<double> tri;    // line variant: 4 doubles per slice row
  DevBuf<int64_t> sptr;  // nslices + 1 entry offsets
  DevBuf<int32_t> cols;
  DevBuf<double> vals;
};

// Staged-block copy of a CSR matrix for k1_stage (kernels_stage.cuh, built by
// stage.cu).  The rows are cut into blocks of R row slots: rowid[b R + i] is
// the row in slot i of block b (-1: empty slot).  On matrices whose pattern is
// a lexicographic grid stencil (detected from the column offsets) a block is
// a bx x by x bz box of grid points, visited in an order that keeps the
// neighbouring planes in L2; otherwise R consecutive rows.  Block b stages
// the operand row runs segs[b smax .. b smax + hdr[b].nseg) = {first row,
// rows} into shared memory; entry (slot u, row slot i) at hdr[b].ebeg + u R +
// i holds the value (vals) of the row's u-th CSR entry and, in lidx at
// hdr[b].ebeg + b R + u R + i, the staged index of its column (padding: value
// 0 at the row's own staged index); lidx slot u = hdr[b].w holds the staged
// index of the row itself (the Gram's P row).
struct StageHdr {   // 32 bytes, one per block
  int64_t ebeg;     // first entry of the block in vals (lidx: ebeg + b R)
  int32_t nseg;     // operand row runs
  int32_t w;        // slots = longest row of the block, rounded up to 4
  int32_t nstaged;  // staged operand rows (sum of the run lengths)
  int32_t pad[3];
};
struct StageCsr {
  int R = 0;  // row slots per block (0: not built)
  int64_t n = 0, nblk = 0;
  int cap = 0, smax = 0, wmax = 0;  // max staged rows / segments / slots per block
  int K = 0;                        // block-vector width the shape was chosen for
  int box[3] = {0, 0, 0};           // grid box of a block (0: consecutive rows)
  int64_t grid[3] = {0, 0, 0};      // grid the boxes were cut from
  int failed_R = 0, failed_K = 0;   // a build for (R0, n, K) did not fit
  int64_t failed_n = 0;
  // grid_detect result for this matrix (host side, stage.cu)
  bool grid_checked = false, has_grid = false;
  int64_t grid_n = 0;
  int64_t grid_found[3] = {0, 0, 0};
  std::vector<int64_t> offs;        // sampled column offsets c - r (all signs, no 0)
  DevBuf<StageHdr> hdr;
  DevBuf<int2> segs;
  DevBuf<uint16_t> lidx;
  DevBuf<double> vals;
  DevBuf<int32_t> rowid;
};

// Constant-coefficient grid stencil found in a CSR matrix (grid.cu): the
// matrix is exactly c[dz+1][(dy+1)*3 + dx+1] on offset (dx, dy, dz) of a
// lexicographic nx x ny x nz grid with the rows at the faces truncated.
// k1_grid (kernels_grid.cuh) applies it from TMA-tiled operand planes.
struct GridStencil {
  bool checked = false, ok = false;
  int64_t n = 0;
  int nx = 0, ny = 0, nz = 0;  // nz: planes of these rows (a z-slab part: its own)
  int zs = 0, nzg = 0;         // first global plane of the rows, planes of the global grid
  bool full27 = false;  // entries off the 7-point star
  bool iso27 = false;   // 27-point, one coefficient each for centre / faces / edges / corners
  double c[3][9] = {};
  // Variable coefficients (ok stays false): the pattern is a 5 / 7-point star
  // on the grid and dia holds its DIA copy V[slot * n + row], slots dz-1 |
  // dy-1 dx-1 0 dx+1 dy+1 | dz+1, zero where a row has no such entry.
  bool var = false;
  DevBuf<double> dia;
};

}  // namespace bkg

struct bkg_matrix;

struct bkg_ctx {
  int device = 0;
  int numerics = BKG_NUMERICS_FAST;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  // scratch (reused across calls on this ctx)
  bkg::DevBuf<double> scratch;
  bkg::DevBuf<char> ctrl;  // one bkg::Ctrl for standalone kernels
  bkg::DevBuf<char> upload_tmp;  // staging for size_t column uploads
  // operands of the kernel-level entry points (bkg_bdot, bkg_baxpy, bkg_bop,
  // bkg_bsolve, bkg_column_norms, bkg_precond_apply): grow-only, so a loop of
  // such calls does not pay a synchronising cudaMalloc + cudaFree per call
  bkg::DevBuf<double> kbuf[3];
  bkg::DevBuf<int> kstatus;
  // CSR buffers of the last destroyed matrix, reused by the next upload
  // (stream-ordered; saves a synchronising cudaFree + cudaMalloc per call)
  bkg::DevBuf<int64_t> spare_rowptr;
  bkg::DevBuf<int32_t> spare_cols;
  bkg::DevBuf<double> spare_vals;
  bkg::SellCsr spare_sell;  // sliced-ELL buffers of the last destroyed matrix
  // live matrices created on this ctx (orphaned, ctx = nullptr, when the ctx
  // is destroyed first; their buffers stay valid until bkg_matrix_destroy)
  std::set<bkg_matrix*> matrices;
  // device workspace of the last bkg_solve call (reused when shapes match)
  void* solver_cache = nullptr;
  void (*solver_cache_free)(void*) = nullptr;
};

struct bkg_matrix {
  bkg_ctx* ctx = nullptr;
  // Unique per object: a cached solver workspace compares serials, not
  // addresses (a destroyed matrix's address is reused by the next create).
  uint64_t serial = next_serial();
  static uint64_t next_serial() {
    static std::atomic<uint64_t> counter{0};
    return ++counter;
  }
  uint64_t n = 0, nnz = 0;
  bkg::DevBuf<int64_t> rowptr;
  bkg::DevBuf<int32_t> cols;
  bkg::DevBuf<double> vals;
  // sliced-ELL copy for the fused K1 (built lazily by the first fast solve)
  mutable bkg::SellCsr sell;
  // staged-block copy for k1_stage (built lazily by the first fast solve)
  mutable bkg::StageCsr stage;
  mutable bkg::GridStencil gridst;  // k1_grid: verified stencil structure (lazily)
  mutable int64_t tri_nnz = -1;  // entries in columns r - 1 .. r + 1 (counted lazily)
  // preconditioner data (built lazily on device)
  bkg::DevBuf<double> inv_diag;  // jacobi scaling or ILU 1/U(r,r)
  bkg::DevBuf<double> lu;        // ILU(0) factors on A's pattern
  int precond_ready = -1;        // kind whose factors are resident
  bkg::DevBuf<int64_t> diag_pos;  // ILU: position of A(r,r) in the CSR
  uint64_t ilu_offdiag = 0;       // ILU: stored off-diagonal entries
  int64_t bad_row = -1;           // row of the last FactorizationError
  // ILU level schedule
  bkg::DevBuf<int32_t> level_rows;  // rows ordered by level
  std::vector<int64_t> level_ptr_fwd, level_ptr_bwd;
  bkg::DevBuf<int32_t> level_rows_bwd;
  // sync-free ILU sweeps: the two sweeps' tickets, L^-1 r scratch (standalone
  // applies; the fused loop uses Q)
  bkg::DevBuf<unsigned long long> ilu_state;
  bkg::DevBuf<double> ilu_y;
  int ilu_lower_max = 0, ilu_upper_max = 0;  // longest strictly lower / upper row part
  // ELL copies (D entries per row, processing order) of the factors' strict
  // lower / upper parts; D = 0: not built (rows longer than 16: CSR sweeps)
  bkg::DevBuf<int32_t> ilu_ell_lc, ilu_ell_uc;
  bkg::DevBuf<double> ilu_ell_lv, ilu_ell_uv;
  int ilu_ell_dl = 0, ilu_ell_du = 0;
  // sync-free sweep segments (processing-order position boundaries)
  bkg::DevBuf<int64_t> ilu_seg_f, ilu_seg_b;
  int64_t ilu_nseg_f = 0, ilu_nseg_b = 0;
};
