// fast_table.cuh — instantiation table for the tuned fast kernels.
//
// The fused kernels are templated on (K lanes, P block width, CPT lanes per
// thread, GLOBAL).  Each K gets its own translation unit (fast_k*.cu) so the
// build parallelises; dispatch is a plain function-pointer table.
#pragma once

#include "kernels_fast.cuh"
#include "kernels_k1.cuh"
#include "kernels_resident.cuh"
#include "kernels_stage.cuh"
#include "kernels_grid.cuh"
#include "kernels_grid2.cuh"
#include "kernels_tma.cuh"

// K1 implementation: 1 = k1_wide (kernels_k1.cuh, 256-bit gathers), 0 = k1_tile.
#ifndef BKG_K1_IMPL
#define BKG_K1_IMPL 1
#endif

namespace bkg {

// k1_wide schedule and CSR chunk per (K, P), the measured winners on B200
// (tools/kernel_sweep.py): C2 (32, 8) per-tile/diagonal row
// with the gathers; C4 classical (16, 16) flat stream; C4 p = 4 and C3
// (64, <= 4) per-tile; C5 (64, 16) per-tile, 8-slot chunks.
#ifdef BKG_K1W_SCHED
template <int K, int P> constexpr int k1w_sched() { return BKG_K1W_SCHED; }
#else
template <int K, int P>
constexpr int k1w_sched() {
  return (K == 16 && P == 16) ? 2 : (K == 32 || (K == 64 && P >= 8)) ? 1 : 0;
}
#endif
#ifdef BKG_K1W_CH
template <int K, int P> constexpr int k1w_chunk() { return BKG_K1W_CH; }
#else
template <int K, int P>
constexpr int k1w_chunk() {
  return (K == 64 && P < 8) ? 4 : 8;
}
#endif

// k1_line (line-variant sliced ELL, kernels_k1.cuh): rows per run and CSR
// chunk (slots left after the r-1, r, r+1 entries are taken out: 4 on a
// 7-point stencil, 2 on a 5-point one).
#ifndef BKG_K1L_RUN
#define BKG_K1L_RUN 64
#endif
#ifndef BKG_K1L_CH
#define BKG_K1L_CH 4
#endif

struct FastTable {
  const void* k1 = nullptr;
  const void* k2 = nullptr;
  const void* k3 = nullptr;
  const void* k2_jac = nullptr;  // K2 / K3 with Jacobi folded in (Z = D^-1 R)
  const void* k3_jac = nullptr;
  const void* k2_ilu = nullptr;  // ILU(0) loop: R -= Q lambda + norms (Gram after the sweeps)
  const void* k3_ilu = nullptr;  // K3 with P' = Z + P beta from the sweeps' Z
  // K3 by [preconditioner: identity, Jacobi, ILU(0)][deferred-X mode 0/1/2]
  const void* k3x[3][3] = {};
  const void* spmm = nullptr;
  const void* gram = nullptr;
  const void* norms = nullptr;
  const void* baxpy = nullptr;
  int smem_iter = 0;   // dynamic smem of k2 / k3 (and the scalar k1)
  int smem_k1 = 0;     // dynamic smem of k1
  int smem_gram = 0;   // dynamic smem of gram
  int smem_norms = 0;  // dynamic smem of norms
  int cpt = 1;
  int rpc = 1;         // rows per CTA pass
  int e_iter = 0;      // partial entries per CTA (max of k1, k2)
  int e_gram = 0;
  int e_norms = 0;
  int rpc_k2 = 1;     // rows per CTA pass of K2 / K3 (grid sizing)
  int rpc_k3 = 1;
  int rpc_k1 = 1;     // rows per CTA pass of K1
  int sell_rows = 0;  // K1 reads a sliced-ELL copy with this slice height (0: CSR)
  // k1_line alternative (picked per matrix by the solver, api.cu use_line)
  const void* k1_line = nullptr;
  int rpc_k1_line = 1;  // rows per CTA pass (RPW x run per warp group)
  int line_run = 0;
  bool line_auto = false;  // the solver may pick it (measured winner for this (K, P))
  // k1_stage alternative (TMA-staged blocks, kernels_stage.cuh): row slots per
  // block are a multiple of stage_R0; its dynamic shared memory for (R, cap,
  // wmax, stages)
  const void* k1_stage = nullptr;
  bool stage_auto = false;  // the solver may pick it without BKG_K1_STAGE=1
  int stage_R0 = 0;
  int (*stage_smem)(int R, int cap, int wmax, int ns) = nullptr;
  // k1_grid alternative (constant-coefficient grid stencils from TMA-tiled
  // planes, kernels_grid.cuh): [0] 7-point, [1] 27-point; [+2] with the
  // lockstep pacing compiled in (long launches); [4], [5]: 5 / 7-point with
  // variable coefficients (DIA tiles), unpaced / paced
  // [6], [7]: isotropic 27-point (class sums), unpaced / paced
  const void* k1_grid[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  bool grid_auto = false;  // the solver may pick it without BKG_K1_GRID=1
  int (*grid_smem)(int ns, bool var) = nullptr;
  // 2-D grids (kernels_grid2.cuh): [0] 5-point, [1] 9-point, [2] 5-point variable
  const void* k1_grid2[3] = {nullptr, nullptr, nullptr};
  int (*grid2_smem)(int ns, bool var) = nullptr;
  // K2 / K3 with TMA-staged operand tiles (kernels_tma.cuh; M = I loop with
  // the deferred X update): k3_tma[0] skip, [1] flush
  const void* k2_tma = nullptr;
  const void* k3_tma[2] = {nullptr, nullptr};
  int tma_smem = 0;
  bool tma23_auto = false;  // the solver may pick them without BKG_TMA23=1
  // latency path for small systems (kernels_resident.cuh): the whole loop as
  // one cooperative kernel with 1 or 4 row passes per CTA
  const void* resident[2] = {nullptr, nullptr};
  int resident_rows[2] = {0, 0};  // rows per CTA
  int resident_smem = 0, resident_eb1 = 0, resident_eb2 = 0;
};

// Lanes per thread: 16-byte accesses where the Gram tile stays small enough
// to keep in registers (P <= 8), 8-byte otherwise.
template <int P>
constexpr int cpt_for() {
  return (P >= 2 && P <= 8) ? 2 : 1;
}

template <int K, int P, bool G>
void fill_table(FastTable* t) {
  constexpr int CPT = cpt_for<P>();
  using S = FastSmem<K, P, CPT, G>;
  t->smem_iter = S::bytes();
  t->smem_k1 = t->smem_iter;
  t->e_iter = S::RED;
  if constexpr (K % 8 == 0 && P <= 16 && BKG_K1_IMPL == 1) {  // 256-bit gathers + DMMA Gram
    constexpr int W = K > 32 ? 32 : K;
    constexpr int CH = k1w_chunk<K, P>();
    using WL = WideLayout<K, P, W, 4>;
    t->k1 = (const void*)&k1_wide<K, P, W, 4, CH, k1w_sched<K, P>(), G>;
    t->rpc_k1 = WL::RPW * (kThreads / 32) / WL::QW;
    t->smem_k1 = k1_wide_smem<K, P, W, 4, G>();
    t->sell_rows = WL::RPW;
    if (WL::RED > t->e_iter) t->e_iter = WL::RED;
    t->k1_line = (const void*)&k1_line<K, P, W, 4, BKG_K1L_CH, BKG_K1L_RUN, G>;
    t->rpc_k1_line = t->rpc_k1 * BKG_K1L_RUN;
    t->line_run = BKG_K1L_RUN;
    // B200 sweeps: k1_line wins only at K = 64, P >= 8 (C5
    // 7.42 -> 7.16 ms); at K <= 32 and K = 64, P < 8 it is 2-19% slower.
    t->line_auto = K == 64 && P >= 8;
    t->k1_stage = (const void*)&k1_stage<K, P, W, G>;
    t->stage_R0 = StageLayout<K, P, W>::R0;
    t->stage_smem = &k1_stage_smem<K, P, W, G>;
    if constexpr (K % kGridW == 0 && K <= 128) {
      t->k1_grid[0] = (const void*)&k1_grid<K, P, G, false, false>;
      t->k1_grid[1] = (const void*)&k1_grid<K, P, G, true, false>;
      t->k1_grid[2] = (const void*)&k1_grid<K, P, G, false, true>;
      t->k1_grid[3] = (const void*)&k1_grid<K, P, G, true, true>;
      t->k1_grid[4] = (const void*)&k1_grid<K, P, G, false, false, true>;
      t->k1_grid[5] = (const void*)&k1_grid<K, P, G, false, true, true>;
      t->k1_grid[6] = (const void*)&k1_grid<K, P, G, true, false, false, true>;
      t->k1_grid[7] = (const void*)&k1_grid<K, P, G, true, true, false, true>;
      t->k1_grid2[0] = (const void*)&k1_grid2<K, P, G, false, false>;
      t->k1_grid2[1] = (const void*)&k1_grid2<K, P, G, true, false>;
      t->k1_grid2[2] = (const void*)&k1_grid2<K, P, G, false, true>;
      t->grid2_smem = &k1_grid2_smem<K, P, G>;
      t->grid_smem = &k1_grid_smem<K, P, G>;
      // B200: C5 K1 6.93 -> 3.07 ms, C2 0.354 -> 0.207, C4 1.87 -> 0.44
      t->grid_auto = true;
      t->k2_tma = (const void*)&k2_tma<K, P, G>;
      t->k3_tma[0] = (const void*)&k3_tma<K, P, G, 1>;
      t->k3_tma[1] = (const void*)&k3_tma<K, P, G, 2>;
      t->tma_smem = k23_tma_smem<K, P, G>();
      if (32 * 8 * (K / kGridW) > t->e_iter) t->e_iter = 32 * 8 * (K / kGridW);
    }
  } else if constexpr (K % 8 == 0 && P <= 16) {  // warp-tile SpMM + DMMA Gram
    constexpr int W = K >= 16 ? 16 : 8;
    t->k1 = (const void*)&k1_tile<K, P, W, G>;
    t->rpc_k1 = (64 / W) * (8 * W / K);  // (rows per warp tile) x (row tiles per CTA)
  } else {
    t->k1 = (const void*)&k1_spmm_gram<K, P, CPT, G>;
    t->rpc_k1 = Layout<K, P, CPT>::RPC;
  }
  // K2 / K3: p x p contraction on FP64 DMMA (P < 8: block-diagonal tiles) or
  // the scalar kernels, per kernel as measured on B200 (tools/kernel_sweep.py,
  // DESIGN.md §5): DMMA always for P >= 8; for P < 8 the DMMA K3 wins for
  // K <= 32 (up to 1.55x) and the DMMA K2 only at P = 4; at K = 64 the scalar
  // kernels' full-line row accesses win.
  // (a CTA's 8 warps must cover whole rows of tile groups: K / max(P, 8) <= 8;
  // k = 128 with p <= 8 has 16 groups per row and takes the scalar kernels)
  constexpr bool MMA_OK = K % 8 == 0 && P <= 16 && K / (P < 8 ? 8 : P) <= 8;
  constexpr bool K2_MMA = MMA_OK && (P >= 8 || (P == 4 && K <= 32));
  constexpr bool K3_MMA = MMA_OK && (P >= 8 || K <= 32);
  constexpr int RPC_MMA = 64 * (P < 8 ? 8 : P) / K;  // 8 rows x (8 warps / tile groups per row)
  if constexpr (K2_MMA) {
    t->k2 = (const void*)&k2_mma<K, P, G>;
    t->k2_jac = (const void*)&k2_mma<K, P, G, true>;
    t->rpc_k2 = RPC_MMA;
  } else {
    t->k2 = (const void*)&k2_update_gram<K, P, CPT, G>;
    t->k2_jac = (const void*)&k2_update_gram<K, P, CPT, G, true>;
    t->rpc_k2 = Layout<K, P, CPT>::RPC;
  }
  if constexpr (K3_MMA) {
    t->k3x[0][0] = (const void*)&k3_mma<K, P, G>;
    t->k3x[0][1] = (const void*)&k3_mma<K, P, G, false, false, 1>;
    t->k3x[0][2] = (const void*)&k3_mma<K, P, G, false, false, 2>;
    t->k3x[1][0] = (const void*)&k3_mma<K, P, G, true>;
    t->k3x[1][1] = (const void*)&k3_mma<K, P, G, true, false, 1>;
    t->k3x[1][2] = (const void*)&k3_mma<K, P, G, true, false, 2>;
    t->k3x[2][0] = (const void*)&k3_mma<K, P, G, false, true>;
    t->k3x[2][1] = (const void*)&k3_mma<K, P, G, false, true, 1>;
    t->k3x[2][2] = (const void*)&k3_mma<K, P, G, false, true, 2>;
    t->rpc_k3 = RPC_MMA;
  } else {
    t->k3x[0][0] = (const void*)&k3_update_xp<K, P, CPT, G>;
    t->k3x[0][1] = (const void*)&k3_update_xp<K, P, CPT, G, false, false, 1>;
    t->k3x[0][2] = (const void*)&k3_update_xp<K, P, CPT, G, false, false, 2>;
    t->k3x[1][0] = (const void*)&k3_update_xp<K, P, CPT, G, true>;
    t->k3x[1][1] = (const void*)&k3_update_xp<K, P, CPT, G, true, false, 1>;
    t->k3x[1][2] = (const void*)&k3_update_xp<K, P, CPT, G, true, false, 2>;
    t->k3x[2][0] = (const void*)&k3_update_xp<K, P, CPT, G, false, true>;
    t->k3x[2][1] = (const void*)&k3_update_xp<K, P, CPT, G, false, true, 1>;
    t->k3x[2][2] = (const void*)&k3_update_xp<K, P, CPT, G, false, true, 2>;
    t->rpc_k3 = Layout<K, P, CPT>::RPC;
  }
  if constexpr (K <= 16) {
    using RS = ResidentSmem<K, P, CPT, G>;
    t->resident[0] = (const void*)&k_resident<K, P, CPT, G, 1>;
    t->resident[1] = (const void*)&k_resident<K, P, CPT, G, 4>;
    t->resident_rows[0] = Layout<K, P, CPT>::RPC;
    t->resident_rows[1] = Layout<K, P, CPT>::RPC * 4;
    t->resident_smem = RS::bytes();
    t->resident_eb1 = RS::EB1;
    t->resident_eb2 = RS::EB2;
  }
  t->k2_ilu = (const void*)&k2_ilu<K, P, CPT, G>;
  t->k3 = t->k3x[0][0];
  t->k3_jac = t->k3x[1][0];
  t->k3_ilu = t->k3x[2][0];
  t->spmm = (const void*)&k_spmm_fast<K, CPT>;
  t->gram = (const void*)&k_gram_fast<K, P, CPT, G>;
  t->norms = (const void*)&k_norms_fast<K, CPT>;
  t->baxpy = (const void*)&k_baxpy_fast<K, P, CPT, G>;
  t->smem_gram = (int)sizeof(double) * K * P;
  t->smem_norms = (int)sizeof(double) * K;
  t->cpt = CPT;
  t->rpc = Layout<K, P, CPT>::RPC;
  t->e_gram = K * P;
  t->e_norms = K;
}

template <int K, int P>
bool fill_p(bool global, FastTable* t) {
  if (global && P != K)
    fill_table<K, P, true>(t);
  else
    fill_table<K, P, false>(t);
  return true;
}

template <int K>
bool fast_lookup_k(int p, bool global, FastTable* t);

// Defined in fast_dispatch.cu: true when (k, p) has a tuned instantiation.
bool fast_lookup(int k, int p, bool global, FastTable* t);

}  // namespace bkg
