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
  const int bad = cta_bsolve<0>(nblk, p, red1, red1 + cs, coef, ws);
  if (bad >= 0) record_breakdown(ctrl, bad, 1);
}

// beta = rho_prev^-1 rho, history and stop test from red2 = [rho | ||R||^2].
__global__ void k_dist_beta(Ctrl* ctrl, int nblk, int p, int k, const double* red2, double* coef,
                            int cs, const double* limits, double* hist, int ring) {
  if (stopped(ctrl)) return;
  extern __shared__ double ws[];
  double* norms = ws + bsolve_ws_doubles(p, blockDim.x);
  const int bad = cta_bsolve<0>(nblk, p, coef + cs, red2, coef + 2 * cs, ws);
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
  DevBuf<int64_t> rowptr;
  DevBuf<int32_t> cols;  // local columns: global - r0 (negative for ghost rows below)
  DevBuf<double> vals;
  SellCsr sell;          // sliced-ELL copy for k1_wide (built at setup)
  DevBuf<double> B, X, R, Q, Pext, coef, limits, hist, red1, red2, partials, gpart, tmp;
  DevBuf<char> ctrl_buf;
  double* P = nullptr;  // own rows inside Pext
  int g1 = 1, g2 = 1, g3 = 1;
  Ctrl* ctrl() { return reinterpret_cast<Ctrl*>(ctrl_buf.ptr); }
};

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

  ~bkg_psolver() {
    if (h_ctrl) cudaFreeHost(h_ctrl);
    if (h_ring) cudaFreeHost(h_ring);
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
    pt.rowptr.alloc(pt.nloc + 1);
    pt.cols.alloc(lc.size());
    pt.vals.alloc(std::max<uint64_t>(nnz, 1));
    h2d(ctx, reinterpret_cast<uint64_t*>(pt.rowptr.ptr), lrowptr, pt.nloc + 1);
    h2d(ctx, pt.cols.ptr, lc.data(), nnz);
    h2d(ctx, pt.vals.ptr, vals, nnz);
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
    pt.rowptr.alloc(pt.nloc + 1);
    pt.cols.alloc(std::max<int64_t>(pt.nnz, 1));
    pt.vals.alloc(std::max<int64_t>(pt.nnz, 1));
    dev_generate_stencil_rows(ctx, kind, nx, ny, nz, seed, contrast, r0, r1, r0, pt.rowptr.ptr,
                              pt.cols.ptr, pt.vals.ptr);
    DevBuf<int> mm(2);
    const int init[2] = {0x7fffffff, (int)0x80000000};
    h2d(ctx, mm.ptr, init, 2);
    int64_t nz_ = pt.nnz;
    const int32_t* cp = pt.cols.ptr;
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

  void finish_setup() {
    global = global && p != k;
    nblk = global ? 1 : k / p;
    cs = nblk * p * p;
    BKG_REQUIRE(use_fast(ctx, k, p, global, &ft), BKG_CONFIG,
                "psolver: (k, p) needs the tuned fast kernels (k in {4,8,16,32,64}, p <= 16)");
    for (Part& pt : parts) {
      const size_t nk = (size_t)pt.nloc * k;
      pt.B.alloc(nk);
      pt.X.alloc(nk);
      pt.R.alloc(nk);
      pt.Q.alloc(nk);
      pt.Pext.alloc((size_t)(pt.hi - pt.lo) * k);
      BKG_CUDA_CHECK(cudaMemsetAsync(pt.Pext.ptr, 0, pt.Pext.bytes(), ctx->stream));
      pt.P = pt.Pext.ptr + (size_t)(pt.r0 - pt.lo) * k;
      pt.coef.alloc((size_t)6 * cs);
      pt.limits.alloc(k);
      pt.hist.alloc((size_t)ring * k);
      pt.red1.alloc((size_t)2 * cs);
      pt.red2.alloc((size_t)cs + k);
      pt.tmp.alloc((size_t)cs + k);
      pt.ctrl_buf.alloc(sizeof(Ctrl));
      BKG_CUDA_CHECK(cudaMemsetAsync(pt.ctrl_buf.ptr, 0, sizeof(Ctrl), ctx->stream));
      pt.g1 = occupancy_grid(ctx, ft.k1, ft.smem_k1, pt.nloc, ft.rpc_k1);
      pt.g2 = occupancy_grid(ctx, ft.k2, ft.smem_iter, pt.nloc, ft.rpc_k2);
      pt.g3 = occupancy_grid(ctx, ft.k3, ft.smem_iter, pt.nloc, ft.rpc_k3);
      const int gmax = std::max(std::max(pt.g1, pt.g2), pt.g3);
      pt.partials.alloc((size_t)gmax * ft.e_iter);
      pt.gpart.alloc((size_t)kMaxTicketGroups * ft.e_iter);
      if (ft.sell_rows)
        sell_build(ctx, pt.nloc, pt.rowptr.ptr, pt.cols.ptr, pt.vals.ptr, ft.sell_rows, pt.sell);
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
    BKG_CUDA_CHECK(cudaHostAlloc(&h_ctrl, sizeof(Ctrl), cudaHostAllocDefault));
    BKG_CUDA_CHECK(cudaHostAlloc(&h_ring, sizeof(double) * ring * k, cudaHostAllocDefault));
    sync(ctx);
  }

  // -- communication -----------------------------------------------------
  // Copy the owned rows of `own(part)` into the ghost rows of `ext(part)`.
  template <class Own, class Ext>
  void halo(Own own, Ext ext) {
    if (!use_nccl) {
      for (const HaloCopy& h : plan) {
        Part& d = parts[h.dst];
        Part& s = parts[h.src];
        d2d(ctx, ext(d) + (size_t)(h.row - d.lo) * k, own(s) + (size_t)(h.row - s.r0) * k,
            (size_t)h.count * k);
      }
      return;
    }
    if (plan.empty()) return;
    Part& me = parts[0];
    BKG_NCCL_CHECK(nccl().GroupStart());
    for (const HaloCopy& h : plan) {
      if (h.src == rank)
        BKG_NCCL_CHECK(nccl().Send(own(me) + (size_t)(h.row - me.r0) * k, (size_t)h.count * k,
                                   ncclDouble, h.dst, comm, ctx->stream));
      if (h.dst == rank)
        BKG_NCCL_CHECK(nccl().Recv(ext(me) + (size_t)(h.row - me.lo) * k, (size_t)h.count * k,
                                   ncclDouble, h.src, comm, ctx->stream));
    }
    BKG_NCCL_CHECK(nccl().GroupEnd());
  }

  void halo_p() {
    halo([](Part& q) { return q.P; }, [](Part& q) { return q.Pext.ptr; });
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

  IterArgs args_of(Part& pt, bool with_hist) {
    IterArgs a{};
    a.n = pt.nloc;
    a.rowptr = pt.rowptr.ptr;
    a.cols = pt.cols.ptr;
    a.vals = pt.vals.ptr;
    a.X = pt.X.ptr;
    a.R = pt.R.ptr;
    a.P = pt.P;
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
    a.sptr = pt.sell.sptr.ptr;
    a.scols = pt.sell.cols.ptr;
    a.svals = pt.sell.vals.ptr;
    return a;
  }

  void iteration(bool with_hist) {
    halo_p();
    for (Part& pt : parts) {
      IterArgs a = args_of(pt, with_hist);
      void* args[] = {&a};
      launch(ctx, ft.k1, pt.g1, kThreads, ft.smem_k1, args);
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
      IterArgs a = args_of(pt, with_hist);
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
    for (Part& pt : parts) {
      IterArgs a = args_of(pt, with_hist);
      void* args[] = {&a};
      launch(ctx, ft.k3, pt.g3, kThreads, ft.smem_iter, args);
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
    for (Part& pt : parts) {
      h2d(ctx, pt.limits.ptr, lim.data(), k);
      h2d(ctx, pt.ctrl_buf.ptr, reinterpret_cast<const char*>(&h), sizeof(Ctrl));
      if (!conv) d2d(ctx, pt.P, pt.R.ptr, (size_t)pt.nloc * k);
    }
    if (!conv) {  // rho_prev^1 = <<P^1, R^0>> (local partials; reduced after K1)
      for (Part& pt : parts)
        dev_gram(ctx, pt.nloc, k, p, global, pt.P, pt.R.ptr, pt.red1.ptr + cs, false);
    }
    cudaEvent_t e0, e1;
    BKG_CUDA_CHECK(cudaEventCreate(&e0));
    BKG_CUDA_CHECK(cudaEventCreate(&e1));
    BKG_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
    uint64_t seen = 0;
    bool done = conv;
    while (!done) {
      for (int i = 0; i < chunk; ++i) iteration(record);
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
    for (Part& pt : parts) d2d(ctx, pt.P, pt.X.ptr, (size_t)pt.nloc * k);
    halo_p();
    for (Part& pt : parts) {
      bkg_matrix m;  // non-owning view of the part's local CSR
      m.n = pt.nloc;
      m.nnz = pt.nnz;
      m.rowptr.ptr = pt.rowptr.ptr;
      m.cols.ptr = pt.cols.ptr;
      m.vals.ptr = pt.vals.ptr;
      dev_spmm(ctx, &m, k, pt.P, pt.Q.ptr, nullptr, false);
      m.rowptr.ptr = nullptr;
      m.cols.ptr = nullptr;
      m.vals.ptr = nullptr;
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
