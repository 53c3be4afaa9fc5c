// psolver.cu — row-partitioned Block-CG: the matrix rows are
// split into contiguous blocks ("parts"); each part owns its rows of X, R, Q
// and an extended P with ghost rows below/above its block.  Per iteration:
//   halo(P) -> K1 (SpMM + local alpha) -> allreduce [alpha | rho_prev]
//   -> lambda solve (replicated) -> K2 (local rho, ||R||^2) -> allreduce
//   -> beta solve + stop test (replicated) -> K3 (X, P, local rho_prev).
// Two transports: "virtual" parts all live on one device of this process
// (halo = device copies, allreduce = fixed-order sum kernel) — the single-GPU
// emulation the tests use; NCCL: one part per process/GPU, halo with
// ncclSend/ncclRecv of contiguous row blocks, ncclAllReduce of the Gram
// partials (NCCL is dlopen'ed on first use).  Fast numerics only.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "bkg.h"
#include "bsolve.cuh"
#include "common.cuh"
#include "host.cuh"
#include "kernels_fast.cuh"

// Deferred X update in the partitioned loop (P ping-pong, as api.cu).
#ifndef BKG_PSOLVER_DEFER_X
#define BKG_PSOLVER_DEFER_X 1
#endif

namespace bkg {

// ------------------------------------------------------------- NCCL ---
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (!api.h) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    BKG_REQUIRE(h, BKG_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      BKG_REQUIRE(f, BKG_NCCL, std::string("libnccl.so.2 lacks ") + name);
      return f;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.h = h;
  }
  return api;
}

#define BKG_NCCL_CHECK(expr)                                                         \
  do {                                                                               \
    ncclResult_t _r = (expr);                                                        \
    if (_r != ncclSuccess)                                                           \
      throw ::bkg::Error(BKG_NCCL, std::string(#expr) + ": " + nccl().GetErrorString(_r)); \
  } while (0)

// ----------------------------------------------------------- kernels ---
// lambda = alpha^-1 rho_prev from the allreduced red1 = [alpha | rho_prev].
__global__ void k_dist_lambda(Ctrl* ctrl, int nblk, int p, const double* red1, double* coef,
                              int cs) {
  if (stopped(ctrl)) return;
  extern __shared__ double ws[];
  for (int i = threadIdx.x; i < cs; i += blockDim.x) coef[cs + i] = red1[cs + i];
  const int bad = fast_bsolve<0>(nblk, p, red1, red1 + cs, coef, ws);
  if (bad >= 0) record_breakdown(ctrl, bad, 1);
}

// beta = rho_prev^-1 rho, history and stop test from red2 = [rho | ||R||^2].
__global__ void k_dist_beta(Ctrl* ctrl, int nblk, int p, int k, const double* red2, double* coef,
                            int cs, const double* limits, double* hist, int ring) {
  if (stopped(ctrl)) return;
  extern __shared__ double ws[];
  double* norms = ws + bsolve_ws_doubles(p, blockDim.x);
  const int bad = fast_bsolve<0>(nblk, p, coef + cs, red2, coef + 2 * cs, ws);
  if (threadIdx.x == 0) ctrl->xpending = 1;
  if (bad >= 0) {
    record_breakdown(ctrl, bad, 2);
    return;
  }
  for (int c = threadIdx.x; c < k; c += blockDim.x) norms[c] = sqrt(red2[cs + c]);
  __syncthreads();
  finish_iteration(ctrl, norms, limits, hist, ring, k);
}

// Virtual-part allreduce: fixed part order, result written back to every part.
__global__ void k_sum_parts(int nparts, int count, double* const* bufs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nparts; ++q) s += bufs[q][i];
    for (int q = 0; q < nparts; ++q) bufs[q][i] = s;
  }
}

__global__ void k_residual_sub(int64_t total, const double* __restrict__ b, double* __restrict__ ax) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    ax[i] = b[i] - ax[i];
}

// [min, max] of the local columns (atomics on an int2 initialised to
// {INT_MAX, INT_MIN}).
__global__ void k_col_range(int64_t nnz, const int32_t* __restrict__ cols, int* mm) {
  int lo = 0x7fffffff, hi = (int)0x80000000;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    lo = min(lo, cols[i]);
    hi = max(hi, cols[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

// ---------------------------------------------------------- halo plan ---
// Pure host logic (also exported for the multi-process CPU tests): part r
// needs rows [need_lo[r], need_hi[r]) of the operand; it owns [row_begin[r],
// row_begin[r+1]).  Every row of the need range owned by another part s
// becomes one contiguous copy (dst r, src s, first global row, count).
struct HaloCopy {
  int dst, src;
  int64_t row, count;
};

std::vector<HaloCopy> halo_plan(int nparts, const int64_t* row_begin, const int64_t* need_lo,
                                const int64_t* need_hi) {
  std::vector<HaloCopy> plan;
  for (int r = 0; r < nparts; ++r)
    for (int s = 0; s < nparts; ++s) {
      if (s == r) continue;
      const int64_t lo = std::max(need_lo[r], row_begin[s]);
      const int64_t hi = std::min(need_hi[r], row_begin[s + 1]);
      if (hi > lo) plan.push_back({r, s, lo, hi - lo});
    }
  return plan;
}

// ---------------------------------------------------------------- part ---
struct Part {
  int64_t r0 = 0, r1 = 0, nloc = 0;  // owned global rows [r0, r1)
  int64_t lo = 0, hi = 0;            // extended operand rows [lo, hi) (lo <= r0, hi >= r1)
  int64_t nnz = 0;
  // local CSR (columns: global - r0, negative for ghost rows below) with its
  // lazily built K1 copies (sliced ELL / staged blocks); ctx stays null
  bkg_matrix A;
  DevBuf<double> B, X, R, Q, coef, limits, hist, red1, red2, partials, gpart, tmp;
  DevBuf<double> Pext[2];  // P ping-pong (deferred X), each with its ghost rows
  double* P[2] = {nullptr, nullptr};  // own rows inside Pext[i]
  DevBuf<char> ctrl_buf;
  // K1 of this part: 2 k1_stage (interior / boundary block lists), 1 k1_line,
  // 0 k1_wide
  int k1_kind = 0, k1_run = 0, stage_ns = 0, smem_k1 = 0;
  const void* k1 = nullptr;
  DevBuf<int64_t> map_in, map_bd;  // k1_stage blocks without / with ghost rows
  int64_t nin = 0, nbd = 0;
  int g1 = 1, g1i = 1, g1b = 1, g2 = 1, g3 = 1;
  // k1_grid (k1_kind 4, kernels_grid.cuh): the part is a z-slab of a constant
  // grid stencil; interior planes (no ghost plane read) and the end planes
  // are separate launches over the ghost-extended P seen as a tensor
  GridStencil gst;
  GridArgs ga_in{}, ga_bd{};
  struct alignas(64) TensorMap {  // GridMaps of kernels_grid.cuh: p (v5, v1 unused)
    unsigned char bytes[3 * 128];
  } tmap[2];
  Ctrl* ctrl() { return reinterpret_cast<Ctrl*>(ctrl_buf.ptr); }
};

// 1 for staged blocks that read a ghost row (a segment outside [0, nloc)).
__global__ void k_block_ghost(int64_t nblk, int64_t nloc, const StageHdr* __restrict__ hdr,
                              int smax, const int2* __restrict__ segs,
                              unsigned char* __restrict__ flag) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblk;
       b += (int64_t)gridDim.x * blockDim.x) {
    unsigned char f = 0;
    const int ns = hdr[b].nseg;
    for (int i = 0; i < ns; ++i) {
      const int2 sg = segs[b * smax + i];
      if (sg.x < 0 || (int64_t)sg.x + sg.y > nloc) f = 1;
    }
    flag[b] = f;
  }
}

}  // namespace bkg

using namespace bkg;

struct bkg_psolver {
  bkg_ctx* ctx = nullptr;
  int64_t n = 0;
  int k = 0, p = 0;
  bool global = false;
  int nblk = 0, cs = 0;
  FastTable ft;
  std::vector<Part> parts;
  bool use_nccl = false;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t z_global = 0;
  std::vector<HaloCopy> plan;  // NCCL: copies with dst == rank or src == rank
  std::vector<int64_t> row_begin;  // global part boundaries (nranks + 1)
  DevBuf<double*> red1_ptrs, red2_ptrs, tmp_ptrs;
  int ring = 66, chunk = 32;
  Ctrl* h_ctrl = nullptr;
  double* h_ring = nullptr;
  std::vector<double> history;
  uint64_t history_rows = 0;
  bool have_b = false;
  bool defer = BKG_PSOLVER_DEFER_X;  // deferred X update, P ping-pong (api.cu k3_for)
  uint64_t iter_launched = 0;
  // halo on a side stream, overlapped with the interior blocks of K1
  cudaStream_t hstream = nullptr;
  cudaEvent_t ev_p = nullptr, ev_h = nullptr;

  ~bkg_psolver() {
    if (h_ctrl) cudaFreeHost(h_ctrl);
    if (h_ring) cudaFreeHost(h_ring);
    if (ev_p) cudaEventDestroy(ev_p);
    if (ev_h) cudaEventDestroy(ev_h);
    if (hstream) cudaStreamDestroy(hstream);
    if (comm) nccl().CommDestroy(comm);
  }

  // -- construction ------------------------------------------------------
  void add_part(int64_t r0, int64_t r1, const uint64_t* lrowptr, const uint64_t* gcols,
                const double* vals) {
    Part pt;
    pt.r0 = r0;
    pt.r1 = r1;
    pt.nloc = r1 - r0;
    const uint64_t nnz = lrowptr[pt.nloc];
    pt.nnz = (int64_t)nnz;
    int64_t mn = r0, mx = r1;  // extended range covers own rows
    std::vector<int32_t> lc(std::max<uint64_t>(nnz, 1));
    for (uint64_t i = 0; i < nnz; ++i) {
      const int64_t c = (int64_t)gcols[i];
      BKG_REQUIRE(c >= 0 && c < n, BKG_CONFIG, "psolver: column index out of range");
      mn = std::min(mn, c);
      mx = std::max(mx, c + 1);
      lc[i] = (int32_t)(c - r0);
    }
    pt.lo = mn;
    pt.hi = mx;
    pt.A.n = (uint64_t)pt.nloc;
    pt.A.nnz = nnz;
    pt.A.rowptr.alloc(pt.nloc + 1);
    pt.A.cols.alloc(lc.size());
    pt.A.vals.alloc(std::max<uint64_t>(nnz, 1));
    h2d(ctx, reinterpret_cast<uint64_t*>(pt.A.rowptr.ptr), lrowptr, pt.nloc + 1);
    h2d(ctx, pt.A.cols.ptr, lc.data(), nnz);
    h2d(ctx, pt.A.vals.ptr, vals, nnz);
    sync(ctx);
    parts.push_back(std::move(pt));
  }

  // Rows [r0, r1) of a stencil matrix generated straight into this part's
  // device CSR (local columns), no host CSR (SURVEY §8f row 3 at 384^3).
  void add_part_generated(int kind, int64_t nx, int64_t ny, int64_t nz, uint64_t seed,
                          double contrast, int64_t r0, int64_t r1) {
    Part pt;
    pt.r0 = r0;
    pt.r1 = r1;
    pt.nloc = r1 - r0;
    pt.nnz = stencil_rows_nnz(kind, nx, ny, nz, r0, r1);
    pt.A.n = (uint64_t)pt.nloc;
    pt.A.nnz = (uint64_t)pt.nnz;
    pt.A.rowptr.alloc(pt.nloc + 1);
    pt.A.cols.alloc(std::max<int64_t>(pt.nnz, 1));
    pt.A.vals.alloc(std::max<int64_t>(pt.nnz, 1));
    dev_generate_stencil_rows(ctx, kind, nx, ny, nz, seed, contrast, r0, r1, r0,
                              pt.A.rowptr.ptr, pt.A.cols.ptr, pt.A.vals.ptr);
    DevBuf<int> mm(2);
    const int init[2] = {0x7fffffff, (int)0x80000000};
    h2d(ctx, mm.ptr, init, 2);
    int64_t nz_ = pt.nnz;
    const int32_t* cp = pt.A.cols.ptr;
    int* mp = mm.ptr;
    void* args[] = {&nz_, &cp, &mp};
    launch(ctx, (const void*)&k_col_range, elem_grid(ctx, pt.nnz), 256, 0, args);
    int h[2];
    d2h(ctx, h, mm.ptr, 2);
    sync(ctx);
    pt.lo = std::min(r0, r0 + (int64_t)h[0]);
    pt.hi = std::max(r1, r0 + (int64_t)h[1] + 1);
    parts.push_back(std::move(pt));
  }

  // k1_grid for a part that is whole z-planes of a constant-coefficient grid
  // stencil (grid.cu checks every row): the ghost-extended P buffers are
  // tensors (column, x, y, plane) whose first plane is the lower ghost plane
  // when there is one; planes that read no ghost plane run while the halo is
  // in flight, the one or two end planes after it.  BKG_K1_GRID=0/1 forces it
  // off/on (default: parts of >= 2^16 rows).
  bool use_grid_part(Part& pt) {
    if (!ft.k1_grid[0] || pt.nloc == 0) return false;
    const char* env = std::getenv("BKG_K1_GRID");
    if (env && env[0] == '0') return false;
    if (!env && (!ft.grid_auto || pt.nloc < (1 << 16))) return false;
    const char* st_env = std::getenv("BKG_K1_STAGE");
    const char* ln_env = std::getenv("BKG_K1_LINE");
    if (!env && ((st_env && st_env[0] == '1') || (ln_env && ln_env[0] == '1'))) return false;
    grid_stencil_rows(ctx, pt.nloc, pt.A.rowptr.ptr, pt.A.cols.ptr, pt.A.vals.ptr, pt.r0, n,
                      pt.gst);
    const GridStencil& st = pt.gst;
    if (!st.ok) return false;  // (variable coefficients: whole matrices only)
    const int64_t plane = (int64_t)st.nx * st.ny;
    const bool lower = st.zs > 0, upper = st.zs + st.nz < st.nzg;
    if (pt.lo != pt.r0 - (lower ? plane : 0) || pt.hi != pt.r1 + (upper ? plane : 0)) return false;
    int optin = 0;
    BKG_CUDA_CHECK(
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    const int ns = grid_ring_depth(ft, k, std::min(optin, 227 * 1024));
    if (ns < 2) return false;
    pt.k1_kind = 4;
    pt.k1 = ft.k1_grid[st.full27 ? 1 : 0];  // + 2: paced (interior launch, chosen per launch)
    pt.smem_k1 = ft.grid_smem(ns, false);
    for (int v = 0; v < 8; ++v) allow_smem(ft.k1_grid[v], pt.smem_k1);
    const int zoff = lower ? 1 : 0;
    const int zb = lower ? 1 : 0, ze = upper ? st.nz - 1 : st.nz;
    const char* hs = std::getenv("BKG_HALO_SMS");
    const int reserve = use_nccl && nranks > 1 ? (hs ? std::atoi(hs) : 4) : 0;
    pt.nin = pt.nbd = 0;
    pt.g1i = pt.g1b = 1;
    const int nzt = (int)((pt.hi - pt.lo) / plane);
    if (ze > zb) {
      grid_plan(st, k, std::max(1, ctx->sm_count - reserve), ns, zb, ze, zoff, nzt, &pt.ga_in,
                &pt.g1i);
      pt.nin = pt.ga_in.nitems;
    }
    if (lower || upper) {
      const bool lo_end = lower, up_end = upper && !(lower && st.nz == 1);
      grid_plan_ends(st, k, ctx->sm_count, ns, lo_end, up_end, zoff, nzt, &pt.ga_bd, &pt.g1b);
      pt.nbd = pt.ga_bd.nitems;
    }
    pt.g1 = std::max(pt.g1i, pt.g1b);
    for (int i = 0; i < (defer ? 2 : 1); ++i)
      grid_tensor_map(pt.Pext[i].ptr, k, st.nx, st.ny, nzt, pt.tmap[i].bytes);
    return true;
  }

  // K1 of a part: k1_stage with its blocks split into those that read ghost
  // rows (boundary: launched after the halo) and the rest (interior:
  // launched while the halo is in flight); else k1_line / k1_wide after the
  // halo.  BKG_HALO_SMS (default 4 with NCCL) SMs are left to NCCL's kernels
  // during the interior launch.
  void choose_k1(Part& pt) {
    FastTable base;
    use_fast(ctx, k, p, global, &base);
    pt.k1 = base.k1;
    pt.smem_k1 = base.smem_k1;
    pt.k1_kind = 0;
    pt.k1_run = 0;
    int rpc = base.rpc_k1;
    if (use_grid_part(pt)) return;
    if (use_stage(ctx, &pt.A, ft, k, &pt.stage_ns, &pt.smem_k1)) {
      pt.k1_kind = 2;
      pt.k1 = ft.k1_stage;
      const StageCsr& st = pt.A.stage;
      DevBuf<unsigned char> flag(std::max<int64_t>(st.nblk, 1));
      int64_t nb = st.nblk, nl = pt.nloc;
      const StageHdr* hd = st.hdr.ptr;
      int sm = st.smax;
      const int2* sg = st.segs.ptr;
      unsigned char* fp = flag.ptr;
      void* args[] = {&nb, &nl, &hd, &sm, &sg, &fp};
      launch(ctx, (const void*)&k_block_ghost, elem_grid(ctx, nb), 256, 0, args);
      std::vector<unsigned char> hf(st.nblk);
      d2h(ctx, hf.data(), flag.ptr, st.nblk);
      sync(ctx);
      std::vector<int64_t> in, bd;
      for (int64_t b = 0; b < st.nblk; ++b) (hf[b] ? bd : in).push_back(b);
      pt.nin = (int64_t)in.size();
      pt.nbd = (int64_t)bd.size();
      pt.map_in.alloc(std::max<int64_t>(pt.nin, 1));
      pt.map_bd.alloc(std::max<int64_t>(pt.nbd, 1));
      h2d(ctx, pt.map_in.ptr, in.data(), in.size());
      h2d(ctx, pt.map_bd.ptr, bd.data(), bd.size());
      int occ = 1;
      allow_smem(pt.k1, pt.smem_k1);
      BKG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pt.k1, kStageThreads,
                                                                   pt.smem_k1));
      occ = std::max(occ, 1);
      const char* hs = std::getenv("BKG_HALO_SMS");
      const int reserve = use_nccl && nranks > 1 ? (hs ? std::atoi(hs) : 4) : 0;
      const int full = occ * ctx->sm_count;
      pt.g1i = (int)std::max<int64_t>(1, std::min<int64_t>(full - occ * reserve, pt.nin));
      pt.g1b = (int)std::max<int64_t>(1, std::min<int64_t>(full, pt.nbd));
      pt.g1 = std::max(pt.g1i, pt.g1b);
      return;
    }
    if (use_line(ctx, &pt.A, ft)) {
      pt.k1_kind = 1;
      pt.k1 = ft.k1_line;
      pt.k1_run = ft.line_run;
      rpc = ft.rpc_k1_line;
    }
    if (ft.sell_rows)
      sell_build(ctx, pt.nloc, pt.A.rowptr.ptr, pt.A.cols.ptr, pt.A.vals.ptr, ft.sell_rows,
                 pt.A.sell, nullptr, pt.k1_run);
    pt.g1 = occupancy_grid(ctx, pt.k1, pt.smem_k1, pt.nloc, rpc);
  }

  void finish_setup() {
    global = global && p != k;
    nblk = global ? 1 : k / p;
    cs = nblk * p * p;
    BKG_REQUIRE(use_fast(ctx, k, p, global, &ft), BKG_CONFIG,
                "psolver: (k, p) needs the tuned fast kernels (k in {4,8,16,32,64,128}, p <= 16)");
    for (Part& pt : parts) {
      const size_t nk = (size_t)pt.nloc * k;
      pt.B.alloc(nk);
      pt.X.alloc(nk);
      pt.R.alloc(nk);
      pt.Q.alloc(nk);
      for (int i = 0; i < (defer ? 2 : 1); ++i) {
        pt.Pext[i].alloc((size_t)(pt.hi - pt.lo) * k);
        BKG_CUDA_CHECK(cudaMemsetAsync(pt.Pext[i].ptr, 0, pt.Pext[i].bytes(), ctx->stream));
        pt.P[i] = pt.Pext[i].ptr + (size_t)(pt.r0 - pt.lo) * k;
      }
      pt.coef.alloc((size_t)6 * cs);
      pt.limits.alloc(k);
      pt.hist.alloc((size_t)ring * k);
      pt.red1.alloc((size_t)2 * cs);
      pt.red2.alloc((size_t)cs + k);
      pt.tmp.alloc((size_t)cs + k);
      pt.ctrl_buf.alloc(sizeof(Ctrl));
      BKG_CUDA_CHECK(cudaMemsetAsync(pt.ctrl_buf.ptr, 0, sizeof(Ctrl), ctx->stream));
      choose_k1(pt);
      pt.g2 = occupancy_grid(ctx, ft.k2, ft.smem_iter, pt.nloc, ft.rpc_k2);
      pt.g3 = std::min(occupancy_grid(ctx, ft.k3x[0][1], ft.smem_iter, pt.nloc, ft.rpc_k3),
                       occupancy_grid(ctx, ft.k3x[0][2], ft.smem_iter, pt.nloc, ft.rpc_k3));
      allow_smem(ft.k3x[0][0], ft.smem_iter);  // observer path (no deferral)
      const int gmax = std::max(std::max(pt.g1, pt.g2), pt.g3);
      pt.partials.alloc((size_t)gmax * ft.e_iter);
      pt.gpart.alloc((size_t)kMaxTicketGroups * ft.e_iter);
    }
    if (!use_nccl) {
      std::vector<double*> r1, r2, t;
      for (Part& pt : parts) {
        r1.push_back(pt.red1.ptr);
        r2.push_back(pt.red2.ptr);
        t.push_back(pt.tmp.ptr);
      }
      red1_ptrs.alloc(parts.size());
      red2_ptrs.alloc(parts.size());
      tmp_ptrs.alloc(parts.size());
      h2d(ctx, red1_ptrs.ptr, r1.data(), r1.size());
      h2d(ctx, red2_ptrs.ptr, r2.data(), r2.size());
      h2d(ctx, tmp_ptrs.ptr, t.data(), t.size());
    }
    BKG_CUDA_CHECK(cudaStreamCreateWithFlags(&hstream, cudaStreamNonBlocking));
    BKG_CUDA_CHECK(cudaEventCreateWithFlags(&ev_p, cudaEventDisableTiming));
    BKG_CUDA_CHECK(cudaEventCreateWithFlags(&ev_h, cudaEventDisableTiming));
    BKG_CUDA_CHECK(cudaHostAlloc(&h_ctrl, sizeof(Ctrl), cudaHostAllocDefault));
    BKG_CUDA_CHECK(cudaHostAlloc(&h_ring, sizeof(double) * ring * k, cudaHostAllocDefault));
    sync(ctx);
  }

  // -- communication -----------------------------------------------------
  // Copy the owned rows of P[buf] of every part into the ghost rows of the
  // parts that read them, on stream `st` (virtual: device copies; NCCL:
  // grouped send/recv of contiguous row blocks over NVLink).
  void halo(int buf, cudaStream_t st) {
    if (!use_nccl) {
      for (const HaloCopy& h : plan) {
        Part& d = parts[h.dst];
        Part& s = parts[h.src];
        BKG_CUDA_CHECK(cudaMemcpyAsync(d.Pext[buf].ptr + (size_t)(h.row - d.lo) * k,
                                       s.P[buf] + (size_t)(h.row - s.r0) * k,
                                       (size_t)h.count * k * sizeof(double),
                                       cudaMemcpyDeviceToDevice, st));
      }
      return;
    }
    if (plan.empty()) return;
    Part& me = parts[0];
    BKG_NCCL_CHECK(nccl().GroupStart());
    for (const HaloCopy& h : plan) {
      if (h.src == rank)
        BKG_NCCL_CHECK(nccl().Send(me.P[buf] + (size_t)(h.row - me.r0) * k, (size_t)h.count * k,
                                   ncclDouble, h.dst, comm, st));
      if (h.dst == rank)
        BKG_NCCL_CHECK(nccl().Recv(me.Pext[buf].ptr + (size_t)(h.row - me.lo) * k,
                                   (size_t)h.count * k, ncclDouble, h.src, comm, st));
    }
    BKG_NCCL_CHECK(nccl().GroupEnd());
  }

  // Sum a per-part vector across parts; every part gets the total.
  void allreduce(DevBuf<double>& (*sel)(Part&), DevBuf<double*>& ptrs, int count) {
    if (use_nccl) {
      double* b = sel(parts[0]).ptr;
      BKG_NCCL_CHECK(nccl().AllReduce(b, b, count, ncclDouble, ncclSum, comm, ctx->stream));
      return;
    }
    int np = (int)parts.size();
    double* const* pp = ptrs.ptr;
    void* args[] = {&np, &count, &pp};
    launch(ctx, (const void*)&k_sum_parts, std::max(1, std::min(64, (count + 255) / 256)), 256,
           0, args);
  }

  IterArgs args_of(Part& pt, bool with_hist, int cur) {
    IterArgs a{};
    a.n = pt.nloc;
    a.rowptr = pt.A.rowptr.ptr;
    a.cols = pt.A.cols.ptr;
    a.vals = pt.A.vals.ptr;
    a.X = pt.X.ptr;
    a.R = pt.R.ptr;
    a.P = pt.P[cur];
    a.Pn = pt.P[cur];
    a.Q = pt.Q.ptr;
    a.partials = pt.partials.ptr;
    a.gpart = pt.gpart.ptr;
    a.coef = pt.coef.ptr;
    a.limits = pt.limits.ptr;
    a.hist = with_hist ? pt.hist.ptr : nullptr;
    a.hist_ring = ring;
    a.group = 16;
    a.ctrl = pt.ctrl();
    a.dist = 1;
    a.red1 = pt.red1.ptr;
    a.red2 = pt.red2.ptr;
    a.sptr = pt.A.sell.sptr.ptr;
    a.scols = pt.A.sell.cols.ptr;
    a.svals = pt.A.sell.vals.ptr;
    a.stri = pt.k1_run ? pt.A.sell.tri.ptr : nullptr;
    if (pt.k1_kind == 2) stage_args(a, pt.A.stage, pt.stage_ns);
    return a;
  }

  // K1 of part pt over its interior (interior = true) or boundary blocks
  // (k1_stage), or the whole K1 (interior = false, other kernels).
  void launch_k1(Part& pt, IterArgs a, bool interior, bool acc) {
    a.dist_acc = acc ? 1 : 0;
    int grid = pt.g1;
    if (pt.k1_kind == 2) {
      a.stg_map = interior ? pt.map_in.ptr : pt.map_bd.ptr;
      a.stg_cnt = interior ? pt.nin : pt.nbd;
      grid = interior ? pt.g1i : pt.g1b;
    }
    if (pt.k1_kind == 4) {
      GridArgs ga = interior ? pt.ga_in : pt.ga_bd;
      const int cur = a.P == pt.P[1] ? 1 : 0;
      void* gargs[] = {&a, &ga, pt.tmap[cur].bytes};
      const void* fn = pt.gst.iso27
                           ? ft.k1_grid[6 + (ga.sync_every > 0 ? 1 : 0)]
                           : ft.k1_grid[(pt.gst.full27 ? 1 : 0) + (ga.sync_every > 0 ? 2 : 0)];
      launch(ctx, fn, interior ? pt.g1i : pt.g1b, kGridThreads, pt.smem_k1, gargs);
      return;
    }
    void* args[] = {&a};
    launch(ctx, pt.k1, grid, pt.k1_kind == 2 ? kStageThreads : kThreads, pt.smem_k1, args);
  }

  void iteration(bool with_hist) {
    const bool odd = defer && (iter_launched++ & 1) != 0;
    const int cur = odd ? 1 : 0;
    // halo of P[cur] on the side stream once the previous K3 wrote it
    BKG_CUDA_CHECK(cudaEventRecord(ev_p, ctx->stream));
    BKG_CUDA_CHECK(cudaStreamWaitEvent(hstream, ev_p, 0));
    halo(cur, hstream);
    BKG_CUDA_CHECK(cudaEventRecord(ev_h, hstream));
    // K1 interior blocks overlap the halo; boundary blocks (and the other
    // K1 kernels) after it
    auto split = [](const Part& pt) { return pt.k1_kind == 2 || pt.k1_kind == 4; };
    for (Part& pt : parts)
      if (split(pt) && pt.nin > 0) launch_k1(pt, args_of(pt, with_hist, cur), true, false);
    BKG_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, ev_h, 0));
    for (Part& pt : parts) {
      if (!split(pt))
        launch_k1(pt, args_of(pt, with_hist, cur), false, false);
      else if (pt.nbd > 0)
        launch_k1(pt, args_of(pt, with_hist, cur), false, pt.nin > 0);
    }
    allreduce([](Part& q) -> DevBuf<double>& { return q.red1; }, red1_ptrs, 2 * cs);
    const int smem = (int)sizeof(double) * (bsolve_ws_doubles(p, 256) + k);
    allow_smem((const void*)&k_dist_lambda, smem);
    allow_smem((const void*)&k_dist_beta, smem);
    for (Part& pt : parts) {
      Ctrl* c = pt.ctrl();
      int nb = nblk, pp = p, c_s = cs;
      const double* r1 = pt.red1.ptr;
      double* cf = pt.coef.ptr;
      void* args[] = {&c, &nb, &pp, &r1, &cf, &c_s};
      launch(ctx, (const void*)&k_dist_lambda, 1, 256, smem, args);
    }
    for (Part& pt : parts) {
      IterArgs a = args_of(pt, with_hist, cur);
      void* args[] = {&a};
      launch(ctx, ft.k2, pt.g2, kThreads, ft.smem_iter, args);
    }
    allreduce([](Part& q) -> DevBuf<double>& { return q.red2; }, red2_ptrs, cs + k);
    for (Part& pt : parts) {
      Ctrl* c = pt.ctrl();
      int nb = nblk, pp = p, kk = k, c_s = cs, rg = ring;
      const double* r2 = pt.red2.ptr;
      double* cf = pt.coef.ptr;
      const double* lm = pt.limits.ptr;
      double* hs = with_hist ? pt.hist.ptr : nullptr;
      void* args[] = {&c, &nb, &pp, &kk, &r2, &cf, &c_s, &lm, &hs, &rg};
      launch(ctx, (const void*)&k_dist_beta, 1, 256, smem, args);
    }
    // K3: deferred X (api.cu k3_for): even iterations read P[0] and write
    // P' to P[1] leaving X (XM 1); odd ones read P[1], flush X with P[0]
    // and lambda_old, write P' over P[0] (XM 2)
    for (Part& pt : parts) {
      IterArgs a = args_of(pt, with_hist, cur);
      const void* k3 = ft.k3x[0][0];
      if (defer) {
        a.Pn = pt.P[1 - cur];
        a.Pold = odd ? pt.P[0] : nullptr;
        k3 = ft.k3x[0][odd ? 2 : 1];
      }
      void* args[] = {&a};
      launch(ctx, k3, pt.g3, kThreads, ft.smem_iter, args);
    }
  }

  // column sums of squares of a per-part block vector, allreduced, on host
  std::vector<double> global_sq_norms(double* (*sel)(Part&)) {
    for (Part& pt : parts)
      dev_gram(ctx, pt.nloc, k, 1, false, sel(pt), sel(pt), pt.tmp.ptr, false);
    allreduce([](Part& q) -> DevBuf<double>& { return q.tmp; }, tmp_ptrs, k);
    std::vector<double> out(k);
    d2h(ctx, out.data(), parts[0].tmp.ptr, k);
    sync(ctx);
    return out;
  }

  void run(double tol, uint64_t max_iter_opt, bool record, bkg_report* rep) {
    BKG_REQUIRE(have_b, BKG_CONFIG, "psolver: right hand side not set");
    BKG_REQUIRE(tol > 0.0, BKG_CONFIG, "bcg_solve: tol must be positive");
    std::memset(rep, 0, sizeof(*rep));
    const uint64_t max_iter = max_iter_opt ? max_iter_opt : 10ull * (uint64_t)n;
    for (Part& pt : parts) {
      BKG_CUDA_CHECK(cudaMemsetAsync(pt.X.ptr, 0, pt.X.bytes(), ctx->stream));
      d2d(ctx, pt.R.ptr, pt.B.ptr, (size_t)pt.nloc * k);
    }
    const std::vector<double> bn = global_sq_norms([](Part& q) { return q.B.ptr; });
    std::vector<double> lim(k);
    for (int s = 0; s < k; ++s) {
      const double v = std::sqrt(bn[s]);
      lim[s] = v > 0.0 ? tol * v : tol;
    }
    const std::vector<double> rn = global_sq_norms([](Part& q) { return q.R.ptr; });
    history.clear();
    history_rows = 0;
    bool conv = true;
    for (int s = 0; s < k; ++s) {
      const double v = std::sqrt(rn[s]);
      if (record) history.push_back(v);
      if (!(v <= lim[s])) conv = false;
    }
    if (record) history_rows = 1;
    Ctrl h{};
    h.done = conv ? 1 : 0;
    h.converged = conv ? 1 : 0;
    h.max_iter = max_iter;
    iter_launched = 0;
    for (Part& pt : parts) {
      h2d(ctx, pt.limits.ptr, lim.data(), k);
      h2d(ctx, pt.ctrl_buf.ptr, reinterpret_cast<const char*>(&h), sizeof(Ctrl));
      if (!conv) d2d(ctx, pt.P[0], pt.R.ptr, (size_t)pt.nloc * k);
    }
    if (!conv) {  // rho_prev^1 = <<P^1, R^0>> (local partials; reduced after K1)
      for (Part& pt : parts)
        dev_gram(ctx, pt.nloc, k, p, global, pt.P[0], pt.R.ptr, pt.red1.ptr + cs, false);
    }
    cudaEvent_t e0, e1;
    BKG_CUDA_CHECK(cudaEventCreate(&e0));
    BKG_CUDA_CHECK(cudaEventCreate(&e1));
    BKG_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
    uint64_t seen = 0;
    bool done = conv;
    while (!done) {
      // never queue iterations (and their collectives) past max_iter
      const uint64_t left = max_iter > seen ? max_iter - seen : 1;
      const int nq = (int)std::min<uint64_t>((uint64_t)chunk, left);
      for (int i = 0; i < nq; ++i) iteration(record);
      d2h(ctx, reinterpret_cast<char*>(h_ctrl), parts[0].ctrl_buf.ptr, sizeof(Ctrl));
      if (record) d2h(ctx, h_ring, parts[0].hist.ptr, (size_t)ring * k);
      sync(ctx);
      const uint64_t it = h_ctrl->iterations;
      if (record)
        for (uint64_t i = seen + 1; i <= it; ++i) {
          const double* row = h_ring + (size_t)(i % ring) * k;
          history.insert(history.end(), row, row + k);
          ++history_rows;
        }
      seen = it;
      done = h_ctrl->done != 0;
    }
    BKG_CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
    BKG_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    BKG_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (conv) {
      d2h(ctx, reinterpret_cast<char*>(h_ctrl), parts[0].ctrl_buf.ptr, sizeof(Ctrl));
      sync(ctx);
    }
    rep->loop_seconds = 1e-3 * ms;
    const Ctrl& c = *h_ctrl;
    rep->iterations = c.iterations;
    rep->converged = c.converged;
    rep->breakdown = c.breakdown;
    rep->breakdown_iteration = c.breakdown_iteration;
    rep->breakdown_block = c.breakdown_block;
    const uint64_t it = c.iterations;
    const uint64_t bdot1 = 2ull * (uint64_t)n * p * p * (k / p);
    uint64_t bops = it, bdots = 3 * it, baxpys = 3 * it;
    if (c.breakdown) {
      bops += 1;
      bdots += c.stage == 1 ? 2 : 3;
      baxpys += c.stage == 1 ? 0 : 2;
    }
    rep->flops_bdot = bdots * bdot1;
    rep->flops_baxpy = baxpys * bdot1;
    rep->flops_bop = bops * 2ull * k * (uint64_t)z_global;
    rep->history_rows = history_rows;
  }

  // Explicit residual ||B - A X|| per column (solver.hpp:203-207).
  std::vector<double> final_norms() {
    for (Part& pt : parts) d2d(ctx, pt.P[0], pt.X.ptr, (size_t)pt.nloc * k);
    halo(0, ctx->stream);
    for (Part& pt : parts) {
      dev_spmm(ctx, &pt.A, k, pt.P[0], pt.Q.ptr, nullptr, false);
      int64_t tot = pt.nloc * (int64_t)k;
      const double* b = pt.B.ptr;
      double* q = pt.Q.ptr;
      void* args[] = {&tot, &b, &q};
      launch(ctx, (const void*)&k_residual_sub, elem_grid(ctx, tot), 256, 0, args);
    }
    std::vector<double> sq = global_sq_norms([](Part& q) { return q.Q.ptr; });
    for (double& v : sq) v = std::sqrt(v);
    return sq;
  }
};

namespace bkg {
template <class F>
int pguard(F&& f) {
  try {
    f();
    return BKG_OK;
  } catch (const Error& e) {
    set_error(e.msg());
    return e.code();
  } catch (const std::exception& e) {
    set_error(e.what());
    return BKG_INTERNAL;
  }
}
}  // namespace bkg

extern "C" {

int bkg_halo_plan(int nparts, const int64_t* row_begin, const int64_t* need_lo,
                  const int64_t* need_hi, int64_t* out, uint64_t cap, uint64_t* count) {
  return pguard([&] {
    const auto plan = halo_plan(nparts, row_begin, need_lo, need_hi);
    *count = plan.size();
    for (size_t i = 0; i < plan.size() && i < cap; ++i) {
      out[4 * i + 0] = plan[i].dst;
      out[4 * i + 1] = plan[i].src;
      out[4 * i + 2] = plan[i].row;
      out[4 * i + 3] = plan[i].count;
    }
  });
}

int bkg_grid_plan(int64_t nx, int64_t ny, int64_t nz, uint64_t k, int sm_count, int zbeg, int zend,
                  int zoff, int nzt, int64_t* out) {
  return pguard([&] {
    BKG_REQUIRE(nx > 0 && ny > 0 && nz > 0 && k > 0 && k % kGridW == 0 && sm_count > 0 &&
                    zbeg >= 0 && zend > zbeg && zend <= nz,
                BKG_CONFIG, "grid plan: bad shape");
    GridStencil st;
    st.nx = (int)nx;
    st.ny = (int)ny;
    st.nz = (int)nz;
    GridArgs g{};
    int ctas = 0;
    if (nz == 1)
      grid2_plan(st, (int)k, sm_count, 3, &g, &ctas);
    else
      grid_plan(st, (int)k, sm_count, 3, zbeg, zend, zoff, nzt, &g, &ctas);
    const int64_t v[12] = {g.tx, g.ty, g.zchunk, g.nzc, (int64_t)(k / kGridW), g.nitems, ctas,
                           g.tmin, g.tmax, g.zstride, g.sync_every, g.sync_lead};
    for (int i = 0; i < 12; ++i) out[i] = v[i];
  });
}

int bkg_nccl_unique_id(void* id_out) {
  return pguard([&] {
    ncclUniqueId id;
    BKG_NCCL_CHECK(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int bkg_psolver_create_virtual(bkg_ctx* ctx, uint64_t n, const uint64_t* rowptr,
                               const uint64_t* cols, const double* vals, int nparts, uint64_t k,
                               uint64_t p, int mode, bkg_psolver** out) {
  return pguard([&] {
    *out = nullptr;
    check_cfg(k, p, mode);
    BKG_REQUIRE(nparts >= 1 && (uint64_t)nparts <= n, BKG_CONFIG, "psolver: bad part count");
    activate(ctx);
    auto* s = new bkg_psolver();
    try {
      s->ctx = ctx;
      s->n = (int64_t)n;
      s->k = (int)k;
      s->p = (int)p;
      s->global = mode == BKG_GLOBAL;
      s->z_global = (int64_t)rowptr[n];
      std::vector<int64_t> rb(nparts + 1), lo(nparts), hi(nparts);
      for (int r = 0; r <= nparts; ++r) rb[r] = (int64_t)(n * (uint64_t)r / nparts);
      for (int r = 0; r < nparts; ++r) {
        std::vector<uint64_t> lrp(rb[r + 1] - rb[r] + 1);
        const uint64_t base = rowptr[rb[r]];
        for (size_t i = 0; i < lrp.size(); ++i) lrp[i] = rowptr[rb[r] + i] - base;
        s->add_part(rb[r], rb[r + 1], lrp.data(), cols + base, vals + base);
        lo[r] = s->parts.back().lo;
        hi[r] = s->parts.back().hi;
      }
      s->row_begin = rb;
      s->plan = halo_plan(nparts, rb.data(), lo.data(), hi.data());
      s->finish_setup();
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

}  // extern "C"

namespace {
// One part per process over NCCL; `add` builds this rank's part.
template <class Add>
int create_nccl(bkg_ctx* ctx, uint64_t n_global, uint64_t row_begin, uint64_t row_end, uint64_t k,
                uint64_t p, int mode, int rank, int nranks, const void* nccl_id,
                bkg_psolver** out, Add&& add) {
  return pguard([&] {
    *out = nullptr;
    check_cfg(k, p, mode);
    BKG_REQUIRE(rank >= 0 && rank < nranks && row_begin < row_end && row_end <= n_global,
                BKG_CONFIG, "psolver: bad rank / row range");
    activate(ctx);
    auto* s = new bkg_psolver();
    try {
      s->ctx = ctx;
      s->n = (int64_t)n_global;
      s->k = (int)k;
      s->p = (int)p;
      s->global = mode == BKG_GLOBAL;
      s->use_nccl = true;
      s->rank = rank;
      s->nranks = nranks;
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      BKG_NCCL_CHECK(nccl().CommInitRank(&s->comm, nranks, id, rank));
      add(s);
      // exchange [row_begin, row_end, need_lo, need_hi, nnz] of every rank
      DevBuf<int64_t> mine(5), all((size_t)5 * nranks);
      const Part& me = s->parts[0];
      const int64_t info[5] = {me.r0, me.r1, me.lo, me.hi, me.nnz};
      h2d(ctx, mine.ptr, info, 5);
      BKG_NCCL_CHECK(nccl().AllGather(mine.ptr, all.ptr, 5, ncclInt64, s->comm, ctx->stream));
      std::vector<int64_t> h((size_t)5 * nranks);
      d2h(ctx, h.data(), all.ptr, h.size());
      sync(ctx);
      std::vector<int64_t> rb(nranks + 1), lo(nranks), hi(nranks);
      int64_t z = 0;
      for (int r = 0; r < nranks; ++r) {
        rb[r] = h[5 * r];
        lo[r] = h[5 * r + 2];
        hi[r] = h[5 * r + 3];
        z += h[5 * r + 4];
        if (r > 0) BKG_REQUIRE(h[5 * r] == h[5 * (r - 1) + 1], BKG_CONFIG, "psolver: row blocks must tile [0, n) in rank order");
      }
      rb[nranks] = h[5 * (nranks - 1) + 1];
      BKG_REQUIRE(rb[0] == 0 && rb[nranks] == (int64_t)n_global, BKG_CONFIG,
                  "psolver: row blocks must cover [0, n)");
      s->z_global = z;
      s->row_begin = rb;
      for (const HaloCopy& c : halo_plan(nranks, rb.data(), lo.data(), hi.data()))
        if (c.dst == rank || c.src == rank) s->plan.push_back(c);
      s->finish_setup();
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}
}  // namespace

extern "C" {

int bkg_psolver_create_nccl(bkg_ctx* ctx, uint64_t n_global, uint64_t row_begin,
                            uint64_t row_end, const uint64_t* local_rowptr, const uint64_t* cols,
                            const double* vals, uint64_t k, uint64_t p, int mode, int rank,
                            int nranks, const void* nccl_id, bkg_psolver** out) {
  return create_nccl(ctx, n_global, row_begin, row_end, k, p, mode, rank, nranks, nccl_id, out,
                     [&](bkg_psolver* s) {
                       s->add_part((int64_t)row_begin, (int64_t)row_end, local_rowptr, cols,
                                   vals);
                     });
}

int bkg_psolver_create_nccl_generated(bkg_ctx* ctx, int kind, uint64_t nx, uint64_t ny,
                                      uint64_t nz, uint64_t seed, double contrast,
                                      uint64_t row_begin, uint64_t row_end, uint64_t k,
                                      uint64_t p, int mode, int rank, int nranks,
                                      const void* nccl_id, bkg_psolver** out) {
  if (kind < 0 || kind > 4) {
    set_error("stencil: unknown kind");
    return BKG_CONFIG;
  }
  if (kind <= 2) nz = 1;
  uint64_t n = 0, nnz = 0;
  bkg_stencil_size(kind, nx, ny, nz, &n, &nnz);
  return create_nccl(ctx, n, row_begin, row_end, k, p, mode, rank, nranks, nccl_id, out,
                     [&](bkg_psolver* s) {
                       s->add_part_generated(kind, (int64_t)nx, (int64_t)ny, (int64_t)nz, seed,
                                             contrast, (int64_t)row_begin, (int64_t)row_end);
                     });
}

int bkg_psolver_generate_rhs(bkg_psolver* s, int distribution, uint64_t seed) {
  return pguard([&] {
    BKG_REQUIRE(distribution == 0 || distribution == 1, BKG_CONFIG, "unknown RHS distribution");
    activate(s->ctx);
    for (Part& pt : s->parts)
      dev_generate_rhs(s->ctx, distribution, pt.nloc, s->k, seed, pt.B.ptr, pt.r0);
    sync(s->ctx);
    s->have_b = true;
  });
}

int bkg_psolver_get_rhs(bkg_psolver* s, double* b) {
  return pguard([&] {
    activate(s->ctx);
    for (Part& pt : s->parts) {
      const int64_t off = s->use_nccl ? 0 : pt.r0;
      d2h(s->ctx, b + (size_t)off * s->k, pt.B.ptr, (size_t)pt.nloc * s->k);
    }
    sync(s->ctx);
  });
}

int bkg_psolver_part_info(const bkg_psolver* s, int part, int64_t* out) {
  return pguard([&] {
    BKG_REQUIRE(part >= 0 && part < (int)s->parts.size(), BKG_CONFIG, "psolver: no such part");
    const Part& pt = s->parts[part];
    out[0] = pt.k1_kind;
    out[1] = pt.k1_kind == 2 || pt.k1_kind == 4 ? pt.nin : 0;
    out[2] = pt.k1_kind == 2 || pt.k1_kind == 4 ? pt.nbd : 0;
    out[3] = pt.r0;
    out[4] = pt.r1;
    const StageCsr& st = pt.A.stage;
    out[5] = pt.k1_kind == 2 ? st.R : 0;
    for (int d = 0; d < 3; ++d) out[6 + d] = pt.k1_kind == 2 ? st.box[d] : 0;
  });
}

int bkg_psolver_destroy(bkg_psolver* s) {
  return pguard([&] {
    if (!s) return;
    cudaSetDevice(s->ctx->device);
    cudaStreamSynchronize(s->ctx->stream);
    delete s;
  });
}

int bkg_psolver_set_rhs(bkg_psolver* s, const double* b) {
  return pguard([&] {
    activate(s->ctx);
    for (Part& pt : s->parts) {
      const int64_t off = s->use_nccl ? 0 : pt.r0;
      h2d(s->ctx, pt.B.ptr, b + (size_t)off * s->k, (size_t)pt.nloc * s->k);
    }
    sync(s->ctx);
    s->have_b = true;
  });
}

int bkg_psolver_run(bkg_psolver* s, double tol, uint64_t max_iter, int record_history,
                    double* final_norms, bkg_report* rep) {
  return pguard([&] {
    activate(s->ctx);
    s->run(tol, max_iter, record_history != 0, rep);
    if (final_norms) {
      const std::vector<double> f = s->final_norms();
      std::memcpy(final_norms, f.data(), sizeof(double) * s->k);
    }
  });
}

int bkg_psolver_get_x(bkg_psolver* s, double* x) {
  return pguard([&] {
    activate(s->ctx);
    for (Part& pt : s->parts) {
      const int64_t off = s->use_nccl ? 0 : pt.r0;
      d2h(s->ctx, x + (size_t)off * s->k, pt.X.ptr, (size_t)pt.nloc * s->k);
    }
    sync(s->ctx);
  });
}

int bkg_psolver_history(bkg_psolver* s, double* hist, uint64_t cap, uint64_t* rows) {
  return pguard([&] {
    const uint64_t r = std::min<uint64_t>(cap, s->history_rows);
    std::memcpy(hist, s->history.data(), r * s->k * sizeof(double));
    *rows = s->history_rows;
  });
}

}  // extern "C"
