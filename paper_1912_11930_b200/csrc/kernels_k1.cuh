// kernels_k1.cuh — K1 with 256-bit operand gathers: Q = A P (kernels.hpp:129-157)
// and alpha = <<P, Q>> (kernels.hpp:59-88), last CTA: lambda = alpha^-1 rho_prev
// (kernels.hpp:231-240).
//
// Row layout: a lane owns CPL = 4 consecutive columns of one row and reads
// each operand row segment as one 32-byte LDG.256, so LPR = W / 4 lanes cover
// the warp's W columns of a row and a warp tile is RPW = 32 / LPR rows.
// Compared with the 16-byte k1_tile this halves the number of lanes that
// replicate each row's (value, column) stream (~40% of K1's L1->register
// traffic on B200, ncu) and halves the gather instructions.  The matrix is
// read from its sliced-ELL copy (common.cuh SellCsr, slice height = RPW).
// The Gram P^T Q over the tile is FP64 DMMA (m8n8k4, k = 4 rows per MMA): the
// tile's P and Q rows go through a per-warp shared-memory scratch into the T
// (operand) layout.  Rows of a tile past n contribute zeros.
#pragma once

#include "kernels_mma.cuh"

namespace bkg {

// Cache operator of the operand gathers (tools/kernel_sweep.py variants): 0
// .nc (default, best), 1 .cg, 2 .nc.L1::no_allocate, 3 .nc.L1::evict_last.
#ifndef BKG_K1W_LD
#define BKG_K1W_LD 0
#endif
__device__ __forceinline__ void ldg4(double (&d)[4], const double* p) {
#if BKG_K1W_LD == 1
  asm("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
#elif BKG_K1W_LD == 2
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
#elif BKG_K1W_LD == 3
  asm("ld.global.nc.L1::evict_last.v4.f64 {%0, %1, %2, %3}, [%4];"
#else
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
#endif
      : "=d"(d[0]), "=d"(d[1]), "=d"(d[2]), "=d"(d[3])
      : "l"(p));
}
// L2 prefetch of the operand row segment a later step of this warp will
// gather.  K1's gathers miss L2 two times out of three (ncu on C5: L2 hit rate
// 35%) and a warp has about one step of gathers in flight, so a step costs a
// DRAM round trip; but a warp's next step reads the same pattern shifted by a
// constant number of rows on any shift-invariant (stencil) matrix -- the next
// row of its run (k1_line) or the tile one grid stride ahead (k1_wide) -- so
// each gather also prefetches "its address + that shift" into L2, and the next
// step's gathers hit L2.  On other matrices the prefetch is a harmless guess.
// BKG_K1_PF: 0 off; k1_line looks BKG_K1_PF rows ahead.
#ifndef BKG_K1_PF
#define BKG_K1_PF 0
#endif
#ifndef BKG_K1W_PF
#define BKG_K1W_PF 0  // k1_wide: prefetch one grid stride ahead (costs registers: spills)
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// Bulk L2 prefetch by the async copy engine (no L1 / LSU miss resources): one
// lane asks for `bytes` starting at p.  k1_line: every BKG_K1_BPF rows of a run
// the first lane of each lane group prefetches the next BKG_K1_BPF operand rows
// of each of its gather streams (the run's own rows and each slot's column +
// BKG_K1_BPF: exact on shift-invariant patterns, a harmless guess otherwise).
#ifndef BKG_K1_BPF
#define BKG_K1_BPF 0
#endif
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
template <int BYTES>  // the gather's own address register + an immediate
__device__ __forceinline__ void prefetch_l2_at(const void* p) {
  asm volatile("prefetch.global.L2 [%0+%1];" ::"l"(p), "n"(BYTES));
}
__device__ __forceinline__ void stg4(double* p, const double* d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(d[0]), "d"(d[1]),
               "d"(d[2]), "d"(d[3])
               : "memory");
}

// A warp owns W columns (W = K, or 32 when K = 64: QW = K / W warps share a
// row block) of RPW rows.
template <int K, int P, int W, int CPL>
struct WideLayout {
  static constexpr int QW = K / W;                // warps per row block
  static constexpr int LPR = W / CPL;             // lanes per row
  static constexpr int RPW = 32 / LPR;            // rows per warp tile
  static constexpr int H = W / 2 + 2;             // scratch: second-half column base
  static constexpr int SS = W + 4;                // scratch row stride (doubles)
  static constexpr int SCR = 2 * RPW * SS;        // scratch doubles per warp (P and Q)
  static constexpr int PT = P >= 8 ? P / 8 : 1;   // 8-col tiles per p-group side
  static constexpr int NPAIR = P >= 8 ? (W / 8) * PT : W / 8;  // Gram tile pairs per warp
  static constexpr int NACC = 2 * NPAIR;
  static constexpr int TPR = 32 * QW;             // grid_reduce positions
  static constexpr int RED = TPR * NACC;
  static_assert(CPL == 4 && K % W == 0 && 8 % QW == 0, "column split");
  static_assert(LPR >= 1 && 32 % LPR == 0 && RPW % 4 == 0, "row split");
  static_assert(W % 8 == 0 && P <= 16 && (P < 8 || W % P == 0), "DMMA Gram tiles");
};

// Scratch column of logical column c (0 <= c < W): each lane's two 16-byte
// halves go to [0, W/2) and [H, H + W/2), so a quarter-warp's stores are
// contiguous and the T-layout operand reads of 4 rows hit distinct banks.
#ifndef BKG_K1W_SWZ
#define BKG_K1W_SWZ 1
#endif
template <int W>
__device__ __forceinline__ int scr_col(int c) {
  if constexpr (BKG_K1W_SWZ) return ((c & 2) ? W / 2 + 2 : 0) + (c >> 2) * 2 + (c & 1);
  return c;
}

template <int K, int P, int W, int CPL>
__device__ __forceinline__ void wide_pair(int pi, int& at, int& bt) {
  using L = WideLayout<K, P, W, CPL>;
  if constexpr (P >= 8) {  // pi = tile * PT + j: partner j inside the tile's p-group
    const int t = pi / L::PT, j = pi % L::PT;
    at = t;
    bt = (t / L::PT) * L::PT + j;
  } else {  // block-diagonal 8 x 8 tiles (8/P whole p-groups each)
    at = bt = pi;
  }
}

// Grid totals (red[(w * 32 + lane) * NACC + pi * 2 + i], D layout) -> row-major
// p x p blocks.
template <int K, int P, int W, int CPL, bool GLOBAL>
__device__ void gather_gram_wide(const double* red, double* blocks) {
  using L = WideLayout<K, P, W, CPL>;
  constexpr int NB = GLOBAL ? 1 : K / P;
  for (int idx = threadIdx.x; idx < NB * P * P; idx += blockDim.x) {
    const int blk = idx / (P * P), a = (idx / P) % P, b = idx % P;
    double s = 0.0;
    const int g0 = GLOBAL ? 0 : blk, g1 = GLOBAL ? K / P : blk + 1;
    for (int g = g0; g < g1; ++g) {
      const int ca = g * P + a, cb = g * P + b;
      const int w = ca / W, at = (ca % W) >> 3, bt = (cb % W) >> 3;
      const int pi = P >= 8 ? at * L::PT + (bt % L::PT) : at;
      const int lane = ((ca & 7) << 2) | ((cb & 7) >> 1), i = cb & 1;
      s += red[(w * 32 + lane) * L::NACC + pi * 2 + i];
    }
    blocks[idx] = s;
  }
}

#ifndef BKG_K1W_MINB
#define BKG_K1W_MINB 2
#endif

// SCHED (chosen per (K, P) from B200 measurements, fast_table.cuh):
//   0  per tile; the diagonal operand row of tile t+1 is loaded at the end of tile t
//   1  per tile; the diagonal operand row is loaded with the tile's gathers
//   2  flat (tile, chunk) stream (below)
template <int K, int P, int W, int CPL, int CH, int SCHED, bool GLOBAL>
__global__ void __launch_bounds__(kThreads, BKG_K1W_MINB) k1_wide(IterArgs a) {
  using L = WideLayout<K, P, W, CPL>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  if (stopped(a.ctrl)) return;
  constexpr int LPR = L::LPR, RPW = L::RPW, SS = L::SS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rr = lane / LPR, cl = lane % LPR;
  const int col = (warp % L::QW) * W + cl * CPL;
  const double* Pc = a.P + col;
  extern __shared__ double sm[];
  double* sp = sm + warp * L::SCR;  // P rows of the tile (T-layout source)
  double* sq = sp + RPW * SS;       // Q rows
  double acc[L::NACC];
#pragma unroll
  for (int e = 0; e < L::NACC; ++e) acc[e] = 0.0;
  const int64_t ntile = (a.n + RPW - 1) / RPW;
  const int64_t wstride = (int64_t)gridDim.x * (kThreads / 32) / L::QW;
  const int64_t rstride = wstride * RPW;
  int64_t tile = ((int64_t)blockIdx.x * (kThreads / 32) + warp) / L::QW;
  int64_t row = tile * RPW + rr;

  // Sliced-ELL stream (common.cuh SellCsr, slice height RPW = the tile):
  // slice t spans entries [sptr[t], sptr[t+1]), slot-major, so the RPW rows
  // of a slot are one contiguous segment; the slot count is warp-uniform.
  auto extent = [&](int64_t t, int64_t& b, int& w) {
    b = 0;
    w = 0;
    if (t < ntile) {
      b = __ldg(a.sptr + t);
      w = (int)((__ldg(a.sptr + t + 1) - b) / RPW);
    }
  };
  auto load_chunk = [&](int64_t b, int off, int w, double (&v)[CH], int (&c)[CH]) {
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const bool in = off + u < w;
      const int64_t e = b + (int64_t)(off + u) * RPW + rr;
      v[u] = in ? __ldg(a.svals + e) : 0.0;
      c[u] = in ? __ldg(a.scols + e) : kNoCol;
    }
  };

  // gathers + FMAs of one CSR chunk; inactive slots: v = 0, x = 0
  // this warp's next tile is one grid stride ahead: prefetch offset in doubles,
  // and the last column whose shifted row still exists
  const int64_t pf_off = rstride * K;
  const int pf_lim = (int)max((int64_t)-1, min(a.n - rstride, (int64_t)0x7fffffff));
  auto gather_fma = [&](const double (&v)[CH], const int (&c)[CH], double (&q)[CPL]) {
    double x[CH][CPL];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if (c[u] != kNoCol) {
        const double* g = Pc + (int64_t)c[u] * K;
        ldg4(x[u], g);
        if (BKG_K1W_PF && c[u] < pf_lim) prefetch_l2(g + pf_off);
      } else {
#pragma unroll
        for (int t = 0; t < CPL; ++t) x[u][t] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u)
#pragma unroll
      for (int t = 0; t < CPL; ++t) q[t] = fma(v[u], x[u][t], q[t]);
  };
  // tile epilogue: store Q, Gram P^T Q over the tile rows (rows -> scratch ->
  // T-layout fragments -> DMMA)
  auto epilogue = [&](int64_t r, const double (&q)[CPL], const double (&pd)[CPL]) {
    if (r < a.n) stg4(a.Q + r * K + col, q);
    const int c0 = cl * CPL;
    *reinterpret_cast<double2*>(sp + rr * SS + scr_col<W>(c0)) = make_double2(pd[0], pd[1]);
    *reinterpret_cast<double2*>(sp + rr * SS + scr_col<W>(c0 + 2)) = make_double2(pd[2], pd[3]);
    *reinterpret_cast<double2*>(sq + rr * SS + scr_col<W>(c0)) = make_double2(q[0], q[1]);
    *reinterpret_cast<double2*>(sq + rr * SS + scr_col<W>(c0 + 2)) = make_double2(q[2], q[3]);
    __syncwarp();
#pragma unroll
    for (int cc = 0; cc < RPW / 4; ++cc) {
      const int sr = (4 * cc + (lane & 3)) * SS;
#pragma unroll
      for (int pi = 0; pi < L::NPAIR; ++pi) {
        int at, bt;
        wide_pair<K, P, W, CPL>(pi, at, bt);
        double d[2] = {acc[2 * pi], acc[2 * pi + 1]};
        dmma(d, sp[sr + scr_col<W>(at * 8 + (lane >> 2))],
             sq[sr + scr_col<W>(bt * 8 + (lane >> 2))]);
        acc[2 * pi] = d[0];
        acc[2 * pi + 1] = d[1];
      }
    }
    __syncwarp();
  };

  int64_t b0, b1, b2;
  int w0, w1, w2;
  double v[CH], q[CPL], pd[CPL];
  int c[CH];
  extent(tile, b0, w0);
  extent(tile + wstride, b1, w1);
  load_chunk(b0, 0, w0, v, c);
#pragma unroll
  for (int t = 0; t < CPL; ++t) q[t] = pd[t] = 0.0;
  if (SCHED != 1 && row < a.n) ldg4(pd, Pc + row * K);
  if constexpr (SCHED == 2) {
    // Flat stream of (tile, chunk) items: the chunk of item i+1 -- the next
    // slots of the same slice, or the first chunk of the next tile -- is in
    // flight while item i's gathers are, so wide slices (27-point rows) cost
    // one memory round trip per chunk.
    extent(tile + 2 * wstride, b2, w2);
    int64_t cb = b0;
    int coff = 0, cw = w0;
    while (tile < ntile) {
      const bool last = coff + CH >= cw;
      const int64_t nb = last ? b1 : cb;
      const int noff = last ? 0 : coff + CH, nw = last ? w1 : cw;
      double nv[CH];
      int nc[CH];
      load_chunk(nb, noff, nw, nv, nc);
      gather_fma(v, c, q);
      if (last) {
        epilogue(row, q, pd);
        tile += wstride;
        row += rstride;
        b0 = b1;
        w0 = w1;
        b1 = b2;
        w1 = w2;
        extent(tile + 2 * wstride, b2, w2);
#pragma unroll
        for (int t = 0; t < CPL; ++t) q[t] = pd[t] = 0.0;
        if (row < a.n) ldg4(pd, Pc + row * K);
      }
      cb = nb;
      coff = noff;
      cw = nw;
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        v[u] = nv[u];
        c[u] = nc[u];
      }
    }
  } else {
    // Per tile: the first chunk of tile t+1 and the slice extent of tile t+2
    // are in flight while tile t's gathers are.
    for (; tile < ntile; tile += wstride) {
      extent(tile + 2 * wstride, b2, w2);
      double nv[CH];
      int nc[CH];
      load_chunk(b1, 0, w1, nv, nc);
      if (SCHED == 1 && row < a.n) ldg4(pd, Pc + row * K);
      gather_fma(v, c, q);
      for (int off = CH; off < w0; off += CH) {  // slices wider than one chunk
        double v2[CH];
        int c2[CH];
        load_chunk(b0, off, w0, v2, c2);
        gather_fma(v2, c2, q);
      }
      epilogue(row, q, pd);
      row += rstride;
      b0 = b1;
      w0 = w1;
      b1 = b2;
      w1 = w2;
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        v[u] = nv[u];
        c[u] = nc[u];
      }
#pragma unroll
      for (int t = 0; t < CPL; ++t) q[t] = pd[t] = 0.0;
      if (SCHED == 0 && row < a.n) ldg4(pd, Pc + row * K);
    }
  }
  __syncthreads();  // the scratch is reused as the reduction buffer
  double* red = sm;
  if (!grid_reduce<L::TPR, L::NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group))
    return;
  double* alpha = sm + L::RED;
  double* ws = alpha + 3 * S::CS;
  gather_gram_wide<K, P, W, CPL, GLOBAL>(red, alpha);
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.red1[i] = alpha[i];
    return;
  }
  const int bad = fast_bsolve<P>(S::NB, P, alpha, a.coef + S::CS, a.coef, ws);  // lambda
  if (bad >= 0) record_breakdown(a.ctrl, bad, 1);
}

// k1_line — k1_wide over the line variant of the sliced-ELL copy (common.cuh
// SellCsr, run = LR): lane group rr of a warp walks LR consecutive rows
// r = base + t, so P[r - 1], P[r], P[r + 1] stay in registers as a sliding
// window -- one operand load per row (P[r + 1]) replaces the gathers of the
// entries in columns r - 1, r, r + 1 AND the separate diagonal load of the
// Gram (P[r] is the window centre).  On a 7-point stencil that is 5 instead of
// 8 operand row loads per row (5-point: 3 instead of 6).  Same epilogue,
// Gram, grid reduction and lambda solve as k1_wide; the products of a row are
// summed as slots first, then the three window terms (fast-mode order).
template <int K, int P, int W, int CPL, int CH, int LR, bool GLOBAL>
__global__ void __launch_bounds__(kThreads, BKG_K1W_MINB) k1_line(IterArgs a) {
  using L = WideLayout<K, P, W, CPL>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  if (stopped(a.ctrl)) return;
  constexpr int LPR = L::LPR, RPW = L::RPW, SS = L::SS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rr = lane / LPR, cl = lane % LPR;
  const int col = (warp % L::QW) * W + cl * CPL;
  const double* Pc = a.P + col;
  extern __shared__ double sm[];
  double* sp = sm + warp * L::SCR;
  double* sq = sp + RPW * SS;
  double acc[L::NACC];
#pragma unroll
  for (int e = 0; e < L::NACC; ++e) acc[e] = 0.0;
  const int64_t nsup = (a.n + RPW * LR - 1) / (RPW * LR);
  const int64_t nslice = nsup * LR;
  const int64_t wstride = (int64_t)gridDim.x * (kThreads / 32) / L::QW;
  int64_t sup = ((int64_t)blockIdx.x * (kThreads / 32) + warp) / L::QW;

  auto extent = [&](int64_t s, int64_t& b, int& w) {
    b = 0;
    w = 0;
    if (s < nslice) {
      b = __ldg(a.sptr + s);
      w = (int)((__ldg(a.sptr + s + 1) - b) / RPW);
    }
  };
  auto load_chunk = [&](int64_t b, int off, int w, double (&v)[CH], int (&c)[CH]) {
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const bool in = off + u < w;
      const int64_t e = b + (int64_t)(off + u) * RPW + rr;
      v[u] = in ? __ldg(a.svals + e) : 0.0;
      c[u] = in ? __ldg(a.scols + e) : kNoCol;
    }
  };
  const int pf_lim = (int)max((int64_t)-1, min(a.n - BKG_K1_PF, (int64_t)0x7fffffff));
  auto load_tri = [&](int64_t s, double (&d)[4]) {
    if (s < nslice) {
      ldg4(d, a.stri + (s * RPW + rr) * 4);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) d[t] = 0.0;
    }
  };
  auto gather_fma = [&](const double (&v)[CH], const int (&c)[CH], double (&q)[CPL]) {
    double x[CH][CPL];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if (c[u] != kNoCol) {
        const double* g = Pc + (int64_t)c[u] * K;
        ldg4(x[u], g);
        if (BKG_K1_PF && c[u] < pf_lim) prefetch_l2_at<BKG_K1_PF * K * 8>(g);  // the run's row + PF
      } else {
#pragma unroll
        for (int t = 0; t < CPL; ++t) x[u][t] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u)
#pragma unroll
      for (int t = 0; t < CPL; ++t) q[t] = fma(v[u], x[u][t], q[t]);
  };
  auto load_row = [&](int64_t r, double (&d)[CPL]) {
    if (r >= 0 && r < a.n) {
      ldg4(d, Pc + r * K);
      if (BKG_K1_PF && r < pf_lim) prefetch_l2_at<BKG_K1_PF * K * 8>(Pc + r * K);
    } else {
#pragma unroll
      for (int t = 0; t < CPL; ++t) d[t] = 0.0;
    }
  };
  auto epilogue = [&](int64_t r, const double (&q)[CPL], const double (&pd)[CPL]) {
    if (r < a.n) stg4(a.Q + r * K + col, q);
    const int c0 = cl * CPL;
    *reinterpret_cast<double2*>(sp + rr * SS + scr_col<W>(c0)) = make_double2(pd[0], pd[1]);
    *reinterpret_cast<double2*>(sp + rr * SS + scr_col<W>(c0 + 2)) = make_double2(pd[2], pd[3]);
    *reinterpret_cast<double2*>(sq + rr * SS + scr_col<W>(c0)) = make_double2(q[0], q[1]);
    *reinterpret_cast<double2*>(sq + rr * SS + scr_col<W>(c0 + 2)) = make_double2(q[2], q[3]);
    __syncwarp();
#pragma unroll
    for (int cc = 0; cc < RPW / 4; ++cc) {
      const int sr = (4 * cc + (lane & 3)) * SS;
#pragma unroll
      for (int pi = 0; pi < L::NPAIR; ++pi) {
        int at, bt;
        wide_pair<K, P, W, CPL>(pi, at, bt);
        double d[2] = {acc[2 * pi], acc[2 * pi + 1]};
        dmma(d, sp[sr + scr_col<W>(at * 8 + (lane >> 2))],
             sq[sr + scr_col<W>(bt * 8 + (lane >> 2))]);
        acc[2 * pi] = d[0];
        acc[2 * pi + 1] = d[1];
      }
    }
    __syncwarp();
  };

  // Pipeline: slice s (chunk + tri loaded), s1 (extent loaded); the slice
  // after a run's last one is the first of the warp's next super tile.
  auto next_of = [&](int64_t s) { return (s % LR) + 1 < LR ? s + 1 : s + 1 - LR + wstride * LR; };
  int64_t s = sup * LR;
  int64_t s1 = next_of(s);
  int64_t b0, b1;
  int w0, w1;
  double v[CH], td[4], xm[CPL], xc[CPL];
  int c[CH];
  extent(s, b0, w0);
  extent(s1, b1, w1);
  load_chunk(b0, 0, w0, v, c);
  load_tri(s, td);
#pragma unroll
  for (int t = 0; t < CPL; ++t) xm[t] = xc[t] = 0.0;
#pragma unroll 1
  for (; sup < nsup; sup += wstride) {
    const int64_t base = sup * (RPW * LR) + rr * LR;
#pragma unroll 1
    for (int t = 0; t < LR; ++t) {
      const int64_t row = base + t;
      if (t == 0) {  // run start: window P[row - 1], P[row]
        load_row(row - 1, xm);
        load_row(row, xc);
      }
      double xp[CPL];
      load_row(row + 1, xp);
      if (BKG_K1_BPF && (t % (BKG_K1_BPF ? BKG_K1_BPF : 1)) == 0 && cl == 0 && warp % L::QW == 0) {
        constexpr int64_t D = BKG_K1_BPF;
        const uint32_t bytes = (uint32_t)(D * K * 8);
        if (row + 1 + 2 * D <= a.n) bulk_prefetch_l2(a.P + (row + 1 + D) * K, bytes);
#pragma unroll
        for (int u = 0; u < CH; ++u)
          if (c[u] != kNoCol && (int64_t)c[u] + 2 * D <= a.n)
            bulk_prefetch_l2(a.P + ((int64_t)c[u] + D) * K, bytes);
      }
      const int64_t s2 = next_of(s1);
      int64_t b2;
      int w2;
      extent(s2, b2, w2);
      double nv[CH], nt[4];
      int nc[CH];
      load_chunk(b1, 0, w1, nv, nc);
      load_tri(s1, nt);
      double q[CPL];
#pragma unroll
      for (int e = 0; e < CPL; ++e) q[e] = 0.0;
      gather_fma(v, c, q);
      for (int off = CH; off < w0; off += CH) {  // slices wider than one chunk
        double v2[CH];
        int c2[CH];
        load_chunk(b0, off, w0, v2, c2);
        gather_fma(v2, c2, q);
      }
#pragma unroll
      for (int e = 0; e < CPL; ++e) {
        q[e] = fma(td[0], xm[e], q[e]);
        q[e] = fma(td[1], xc[e], q[e]);
        q[e] = fma(td[2], xp[e], q[e]);
      }
      epilogue(row, q, xc);
#pragma unroll
      for (int e = 0; e < CPL; ++e) {
        xm[e] = xc[e];
        xc[e] = xp[e];
      }
      s = s1;
      s1 = s2;
      b0 = b1;
      w0 = w1;
      b1 = b2;
      w1 = w2;
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        v[u] = nv[u];
        c[u] = nc[u];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) td[e] = nt[e];
    }
  }
  __syncthreads();  // the scratch is reused as the reduction buffer
  double* red = sm;
  if (!grid_reduce<L::TPR, L::NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group))
    return;
  double* alpha = sm + L::RED;
  double* ws = alpha + 3 * S::CS;
  gather_gram_wide<K, P, W, CPL, GLOBAL>(red, alpha);
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.red1[i] = alpha[i];
    return;
  }
  const int bad = fast_bsolve<P>(S::NB, P, alpha, a.coef + S::CS, a.coef, ws);  // lambda
  if (bad >= 0) record_breakdown(a.ctrl, bad, 1);
}

// Dynamic shared memory of k1_wide: max(warp scratch, reduction epilogue).
template <int K, int P, int W, int CPL, bool GLOBAL>
int k1_wide_smem() {
  using L = WideLayout<K, P, W, CPL>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  const int scratch = (kThreads / 32) * L::SCR;
  const int epi = L::RED + 3 * S::CS + bsolve_ws_doubles(P, kThreads) + K;
  return (int)sizeof(double) * (scratch > epi ? scratch : epi);
}

}  // namespace bkg
