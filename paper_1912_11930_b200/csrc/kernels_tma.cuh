// kernels_tma.cuh — K2 and K3 with their operand tiles streamed through shared
// memory by TMA tensor copies (M = I loop, deferred X update):
//   k2_tma  R -= Q lambda (kernels.hpp:94-125), rho = <<R, R>> (:59-88) and the
//           column norms of R (block_vector.hpp:59-70, the Gram's diagonal);
//           last CTA: beta, history, stop test (solver.hpp:176-190)
//   k3_tma  XM 1 (skip):  P' = R + P beta, rho_prev' = <<P', R>>
//           XM 2 (flush): also X += Pold lambda_old + P lambda
//
// Why: the register-operand kernels (kernels_mma.cuh) read their A fragments
// as 8-byte loads, 32 bytes per row per instruction (ncu, C5: L1 data pipe
// 62-66%, long-scoreboard stalls 43-80%, K2 0.88 / K3 0.83 of the HBM peak),
// and at 79-128 registers hold about one row block of loads in flight per warp.
// Here a block vector is a 2-D tensor (column, row) and a warp owns a private
// ring of NST stages: each stage holds one TR-row x 16-column tile (128-byte
// rows, SWIZZLE_128B) of every operand, filled by one cp.async.bulk.tensor.2d
// per operand and completed on a per-warp mbarrier -- bytes in flight are set
// by shared memory (8 warps x 2 stages x 8 KB), not registers, every global
// access is a whole 128-byte row segment, and rows past n are zero-filled on
// load and clipped on store by the TMA unit.  Results are written back into
// the stage (P' over the P tile, R' over R, X' over X) and leave by one
// cp.async.bulk.tensor store per tile; a stage is refilled one step later,
// after its store group has drained (wait_group.read).
//
// Fragments come from the swizzled tile without bank conflicts: the 8 rows of
// a DMMA row block sit in tile rows 8b + rho(M), rho = (0,4,2,6,1,5,3,7), so
// the 8-byte A-fragment reads of a half-warp and the 16-byte C/D-fragment
// accesses of a quarter-warp each cover all 32 banks once; the Gram reads its
// operands in the k1_grid layout (lane (r, m): columns {2m, 2m+1} of row
// 8b + 2r + c), four DMMAs per four rows over "even" / "odd" column blocks.
//
// Rare launches (the solve stops in this K3, a lambda breakdown flush) take
// the register-operand kernel's body instead (k3_mma_body).
//
// Measured on B200: parity green, but level with the
// register-operand kernels (C5 K2 4.52 vs 4.47 ms, K3 7.09 vs 7.16) -- at p = 16
// the DMMA work, not the access pattern, is what keeps K2 / K3 below the
// roofline -- so the solver takes these only with BKG_TMA23=1.
#pragma once

#include <cuda.h>

#include "kernels_grid.cuh"
#include "kernels_fast.cuh"
#include "kernels_mma.cuh"

namespace bkg {

constexpr int kTmaStages = 3;
constexpr int kTmaWarps = kThreads / 32;

struct TmaMaps {  // K2: [0] Q, [1] R;  K3: [0] P, [1] R, [2] Pn, [3] X, [4] Pold
  CUtensorMap m[5];
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int c0, int c1,
                                             const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::
                   "l"(tm),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tma_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tma_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// tile row of fragment row M (0..7) of a DMMA row block
__device__ __forceinline__ int tma_rho(int M) { return ((M & 1) << 2) | (M & 2) | (M >> 2); }

// B fragments of the 16-column slice g: f[kc][nt] = sign * C[4kc + (lane&3)][8nt + (lane>>2)],
// C = the slice's 16 x 16 block-diagonal coefficient matrix (row-major c[b][a]
// p x p blocks, kernels.hpp:94-125; global: block 0 everywhere).
template <int K, int P, bool GLOBAL>
__device__ __forceinline__ void tma_bfrag(const double* coef, int g, double sign, double (&f)[4][2],
                                          int lane) {
#pragma unroll
  for (int kc = 0; kc < 4; ++kc)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int b = kc * 4 + (lane & 3), a = nt * 8 + (lane >> 2);
      const int blk = GLOBAL ? 0 : (g * kGridW + b) / P;
      f[kc][nt] = (b / P == a / P) ? sign * coef[blk * P * P + (b % P) * P + a % P] : 0.0;
    }
}
template <int P>
__device__ __forceinline__ constexpr bool tma_bnz(int kc, int nt) {  // block (kc, nt) can be nonzero
  return P == 16 || (kc >> 1) == nt;
}

// Grid totals red[(g * 32 + lane) * 8 + (i * 2 + j) * 2 + e] (slice g, D layout
// of the even/odd Gram DMMAs) -> row-major p x p blocks; diag != nullptr: also
// the K diagonal entries (column sums of squares).
template <int K, int P, bool GLOBAL>
__device__ void gather_gram_tma(const double* red, double* blocks, double* diag) {
  constexpr int NB = GLOBAL ? 1 : K / P;
  auto at = [&](int ca, int cb) {  // entry (ca, cb), same slice
    const int sl = ca / kGridW, a = ca % kGridW, b = cb % kGridW;
    const int lane = ((a >> 1) << 2) | (b >> 2), e = (b >> 1) & 1;
    return red[(sl * 32 + lane) * 8 + ((a & 1) * 2 + (b & 1)) * 2 + e];
  };
  for (int idx = threadIdx.x; idx < NB * P * P; idx += blockDim.x) {
    const int blk = idx / (P * P), pa = (idx / P) % P, pb = idx % P;
    double s = 0.0;
    const int g0 = GLOBAL ? 0 : blk, g1 = GLOBAL ? K / P : blk + 1;
    for (int g = g0; g < g1; ++g) s += at(g * P + pa, g * P + pb);
    blocks[idx] = s;
  }
  if (diag)
    for (int c = threadIdx.x; c < K; c += blockDim.x) diag[c] = at(c, c);
}

// Per-warp ring bookkeeping shared by k2_tma / k3_tma.
template <int K, int TR, int NOP>
struct TmaRing {
  static constexpr int NSL = K / kGridW;           // 16-column slices
  static constexpr int RW = kTmaWarps / NSL;       // row tiles per CTA step
  static constexpr int SLOT = TR * 128;            // one operand tile
  static constexpr int STAGE = NOP * SLOT;
  static constexpr int WARP = kTmaStages * STAGE;
  static constexpr int BYTES = kTmaWarps * WARP + kTmaWarps * kTmaStages * 8 + 1024;
  static_assert(kTmaWarps % NSL == 0 && SLOT % 1024 == 0, "ring layout");
};

// The Gram of a tile: rows 8b + 2r + c of tiles ta (A operand) and tb (B operand).
template <int TR>
__device__ __forceinline__ void tma_gram(const unsigned char* ta, const unsigned char* tb,
                                         double (&gram)[8], int lane) {
  const int r = lane & 3, m = lane >> 2;
#pragma unroll
  for (int q = 0; q < TR / 4; ++q) {
    const int row = 8 * (q >> 1) + 2 * r + (q & 1);
    const int off = row * 128 + ((m ^ (row & 7)) << 4);
    const double2 va = *reinterpret_cast<const double2*>(ta + off);
    const double2 vb = *reinterpret_cast<const double2*>(tb + off);
    const double pa[2] = {va.x, va.y}, pb[2] = {vb.x, vb.y};
#pragma unroll
    for (int ii = 0; ii < 2; ++ii)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        double d[2] = {gram[(ii * 2 + jj) * 2], gram[(ii * 2 + jj) * 2 + 1]};
        dmma(d, pa[ii], pb[jj]);
        gram[(ii * 2 + jj) * 2] = d[0];
        gram[(ii * 2 + jj) * 2 + 1] = d[1];
      }
  }
}

// ------------------------------------------------------------------ K3 ---
template <int K, int P, bool GLOBAL, int XM>
__global__ void __launch_bounds__(kThreads, 1)
    k3_tma(IterArgs a, const __grid_constant__ TmaMaps tm) {
  static_assert(XM == 1 || XM == 2, "deferred-X launches only");
  using S = FastSmem<K, P, 1, GLOBAL>;
  constexpr int TR = XM == 1 ? 32 : 16;
  constexpr int NOP = XM == 1 ? 2 : 4;  // P, R (, Pold, X)
  using RG = TmaRing<K, TR, NOP>;
  constexpr int NSL = RG::NSL, NB8 = TR / 8;
  const bool cur = *reinterpret_cast<const volatile int32_t*>(&a.ctrl->xpending) != 0;
  const bool old = XM == 2 && *reinterpret_cast<const volatile int32_t*>(&a.ctrl->xold) != 0;
  if (!cur && !old) return;
  const bool fin = stopped(a.ctrl);
  if (fin || !cur || (XM == 2 && !old)) {  // rare: the register-operand kernel's body
    constexpr bool MMA_OK = K / (P < 8 ? 8 : P) <= 8 && (P >= 8 || K <= 32);  // fast_table.cuh K3_MMA
    if constexpr (MMA_OK)
      k3_mma_body<K, P, GLOBAL, false, false, XM>(a);
    else
      k3_update_xp_body<K, P, (P >= 2 && P <= 8) ? 2 : 1, GLOBAL, false, false, XM>(a);
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp % NSL, wr = warp / NSL;
  extern __shared__ unsigned char smdyn[];
  unsigned char* smraw = smdyn + ((1024u - (smem_u32(smdyn) & 1023u)) & 1023u);
  unsigned char* ring = smraw + warp * RG::WARP;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + kTmaWarps * RG::WARP) + warp * kTmaStages;
  if (lane == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(full + s, 1);
    mbar_fence_init();
  }
  __syncwarp();

  double bet[4][2], lam[4][2], lamo[4][2];
  tma_bfrag<K, P, GLOBAL>(a.coef + 2 * S::CS, g, 1.0, bet, lane);
  if constexpr (XM == 2) {
    tma_bfrag<K, P, GLOBAL>(a.coef, g, 1.0, lam, lane);
    tma_bfrag<K, P, GLOBAL>(a.coef + 4 * S::CS, g, 1.0, lamo, lane);
  }
  double gram[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) gram[e] = 0.0;

  const int64_t ntile = (a.n + TR - 1) / TR;
  const int64_t t0 = (int64_t)blockIdx.x * RG::RW + wr, tstep = (int64_t)gridDim.x * RG::RW;
  const int64_t nmine = ntile > t0 ? (ntile - t0 + tstep - 1) / tstep : 0;
  auto issue = [&](int64_t i) {  // lane 0: the operand tiles of this warp's i-th tile
    const int s = (int)(i % kTmaStages);
    const int row0 = (int)((t0 + i * tstep) * TR);
    unsigned char* st = ring + s * RG::STAGE;
    mbar_expect_tx(full + s, RG::STAGE);
    tma_load_2d(st, &tm.m[0], g * kGridW, row0, full + s);
    tma_load_2d(st + RG::SLOT, &tm.m[1], g * kGridW, row0, full + s);
    if constexpr (XM == 2) {
      tma_load_2d(st + 2 * RG::SLOT, &tm.m[4], g * kGridW, row0, full + s);
      tma_load_2d(st + 3 * RG::SLOT, &tm.m[3], g * kGridW, row0, full + s);
    }
  };
  if (lane == 0)
    for (int64_t i = 0; i < kTmaStages && i < nmine; ++i) issue(i);

  const int M = lane >> 2, j = lane & 3, rho = tma_rho(M);
#pragma unroll 1
  for (int64_t i = 0; i < nmine; ++i) {
    const int s = (int)(i % kTmaStages);
    mbar_wait(full + s, (uint32_t)((i / kTmaStages) & 1));
    unsigned char* tp = ring + s * RG::STAGE;  // P tile -> P' tile
    unsigned char* tr = tp + RG::SLOT;         // R tile
    double pn[NB8][2][2], xn[NB8][2][2];
#pragma unroll
    for (int b = 0; b < NB8; ++b) {
      const int row = 8 * b + rho;
      double pa[4], po[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        const int off = row * 128 + (((2 * kc + (j >> 1)) ^ rho) << 4) + (j & 1) * 8;
        pa[kc] = *reinterpret_cast<const double*>(tp + off);
        if constexpr (XM == 2) po[kc] = *reinterpret_cast<const double*>(tp + 2 * RG::SLOT + off);
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int off = row * 128 + (((4 * nt + j) ^ rho) << 4);
        const double2 rv = *reinterpret_cast<const double2*>(tr + off);
        pn[b][nt][0] = rv.x;
        pn[b][nt][1] = rv.y;
        if constexpr (XM == 2) {
          const double2 xv = *reinterpret_cast<const double2*>(tp + 3 * RG::SLOT + off);
          xn[b][nt][0] = xv.x;
          xn[b][nt][1] = xv.y;
        }
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          if (!tma_bnz<P>(kc, nt)) continue;
          if constexpr (XM == 2) {
            dmma(xn[b][nt], po[kc], lamo[kc][nt]);
            dmma(xn[b][nt], pa[kc], lam[kc][nt]);
          }
          dmma(pn[b][nt], pa[kc], bet[kc][nt]);
        }
    }
    __syncwarp();  // every lane has read its P (and X) fragments: overwrite in place
#pragma unroll
    for (int b = 0; b < NB8; ++b)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int off = (8 * b + rho) * 128 + (((4 * nt + j) ^ rho) << 4);
        *reinterpret_cast<double2*>(tp + off) = make_double2(pn[b][nt][0], pn[b][nt][1]);
        if constexpr (XM == 2)
          *reinterpret_cast<double2*>(tp + 3 * RG::SLOT + off) =
              make_double2(xn[b][nt][0], xn[b][nt][1]);
      }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      const int row0 = (int)((t0 + i * tstep) * TR);
      tma_store_2d(&tm.m[2], g * kGridW, row0, tp);
      if constexpr (XM == 2) tma_store_2d(&tm.m[3], g * kGridW, row0, tp + 3 * RG::SLOT);
      tma_commit();
    }
    tma_gram<TR>(tp, tr, gram, lane);  // rho_prev' += P'^T R
    __syncwarp();
    // refill the stage of the previous step: its store has had this step to drain
    if (lane == 0 && i >= 1 && i - 1 + kTmaStages < nmine) {
      tma_wait_read<1>();
      issue(i - 1 + kTmaStages);
    }
  }
  if (lane == 0) tma_wait_all();
  __syncthreads();  // the rings are reused as the reduction buffer
  double* red = reinterpret_cast<double*>(smraw);
  if (!grid_reduce<32 * NSL, 8>(gram, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  double* blocks = red + 32 * NSL * 8;
  gather_gram_tma<K, P, GLOBAL>(red, blocks, nullptr);
  __syncthreads();
  double* out = (a.dist ? a.red1 : a.coef) + S::CS;
  for (int i = threadIdx.x; i < S::CS; i += kThreads) out[i] = blocks[i];
  if (XM == 1)
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.coef[4 * S::CS + i] = a.coef[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    a.ctrl->xold = XM == 1 ? 1 : 0;
    a.ctrl->xpending = 0;
  }
}

// ------------------------------------------------------------------ K2 ---
template <int K, int P, bool GLOBAL>
__global__ void __launch_bounds__(kThreads, 1)
    k2_tma(IterArgs a, const __grid_constant__ TmaMaps tm) {
  using S = FastSmem<K, P, 1, GLOBAL>;
  constexpr int TR = 32, NOP = 2;  // Q, R
  using RG = TmaRing<K, TR, NOP>;
  constexpr int NSL = RG::NSL, NB8 = TR / 8;
  if (stopped(a.ctrl)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = warp % NSL, wr = warp / NSL;
  extern __shared__ unsigned char smdyn[];
  unsigned char* smraw = smdyn + ((1024u - (smem_u32(smdyn) & 1023u)) & 1023u);
  unsigned char* ring = smraw + warp * RG::WARP;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + kTmaWarps * RG::WARP) + warp * kTmaStages;
  if (lane == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(full + s, 1);
    mbar_fence_init();
  }
  __syncwarp();
  double nlam[4][2];
  tma_bfrag<K, P, GLOBAL>(a.coef, g, -1.0, nlam, lane);
  double gram[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) gram[e] = 0.0;
  const int64_t ntile = (a.n + TR - 1) / TR;
  const int64_t t0 = (int64_t)blockIdx.x * RG::RW + wr, tstep = (int64_t)gridDim.x * RG::RW;
  const int64_t nmine = ntile > t0 ? (ntile - t0 + tstep - 1) / tstep : 0;
  auto issue = [&](int64_t i) {
    const int s = (int)(i % kTmaStages);
    const int row0 = (int)((t0 + i * tstep) * TR);
    unsigned char* st = ring + s * RG::STAGE;
    mbar_expect_tx(full + s, RG::STAGE);
    tma_load_2d(st, &tm.m[0], g * kGridW, row0, full + s);
    tma_load_2d(st + RG::SLOT, &tm.m[1], g * kGridW, row0, full + s);
  };
  if (lane == 0)
    for (int64_t i = 0; i < kTmaStages && i < nmine; ++i) issue(i);
  const int M = lane >> 2, j = lane & 3, rho = tma_rho(M);
#pragma unroll 1
  for (int64_t i = 0; i < nmine; ++i) {
    const int s = (int)(i % kTmaStages);
    mbar_wait(full + s, (uint32_t)((i / kTmaStages) & 1));
    unsigned char* tq = ring + s * RG::STAGE;  // Q tile
    unsigned char* tr = tq + RG::SLOT;         // R tile -> R' tile
    double rn[NB8][2][2];
#pragma unroll
    for (int b = 0; b < NB8; ++b) {
      const int row = 8 * b + rho;
      double qa[4];
#pragma unroll
      for (int kc = 0; kc < 4; ++kc)
        qa[kc] = *reinterpret_cast<const double*>(
            tq + row * 128 + (((2 * kc + (j >> 1)) ^ rho) << 4) + (j & 1) * 8);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const double2 rv =
            *reinterpret_cast<const double2*>(tr + row * 128 + (((4 * nt + j) ^ rho) << 4));
        rn[b][nt][0] = rv.x;
        rn[b][nt][1] = rv.y;
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int kc = 0; kc < 4; ++kc)
          if (tma_bnz<P>(kc, nt)) dmma(rn[b][nt], qa[kc], nlam[kc][nt]);
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < NB8; ++b)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
        *reinterpret_cast<double2*>(tr + (8 * b + rho) * 128 + (((4 * nt + j) ^ rho) << 4)) =
            make_double2(rn[b][nt][0], rn[b][nt][1]);
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&tm.m[1], g * kGridW, (int)((t0 + i * tstep) * TR), tr);
      tma_commit();
    }
    tma_gram<TR>(tr, tr, gram, lane);  // rho += R'^T R'
    __syncwarp();
    if (lane == 0 && i >= 1 && i - 1 + kTmaStages < nmine) {
      tma_wait_read<1>();
      issue(i - 1 + kTmaStages);
    }
  }
  if (lane == 0) tma_wait_all();
  __syncthreads();
  double* red = reinterpret_cast<double*>(smraw);
  if (!grid_reduce<32 * NSL, 8>(gram, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  double* rho_s = red + 32 * NSL * 8;
  double* beta_s = rho_s + S::CS;
  double* norms = beta_s + S::CS;
  double* ws = norms + K;
  gather_gram_tma<K, P, GLOBAL>(red, rho_s, norms);
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kThreads) a.red2[i] = rho_s[i];
    for (int c = threadIdx.x; c < K; c += kThreads) a.red2[S::CS + c] = norms[c];
    return;
  }
  for (int c = threadIdx.x; c < K; c += kThreads) norms[c] = sqrt(norms[c]);
  __syncthreads();
  const int bad = fast_bsolve<P>(S::NB, P, a.coef + S::CS, rho_s, beta_s, ws);  // beta
  if (threadIdx.x == 0) a.ctrl->xpending = 1;
  if (bad >= 0) {
    record_breakdown(a.ctrl, bad, 2);
    return;
  }
  for (int i = threadIdx.x; i < S::CS; i += kThreads) {
    a.coef[2 * S::CS + i] = beta_s[i];
    a.coef[3 * S::CS + i] = rho_s[i];
  }
  finish_iteration(a.ctrl, norms, a.limits, a.hist, a.hist_ring, K);
}

// Dynamic shared memory: the rings, or the last CTA's reduction + solve scratch.
template <int K, int P, bool GLOBAL>
int k23_tma_smem() {
  using S = FastSmem<K, P, 1, GLOBAL>;
  const int ring = TmaRing<K, 32, 2>::BYTES;  // = the flush launch's (16 rows x 4 operands)
  const int epi = (int)sizeof(double) * (32 * (K / kGridW) * 8 + 3 * S::CS + K +
                                         bsolve_ws_doubles(P, kThreads)) + 1024;
  const int mma = S::bytes();  // k3_mma_body
  return ring > epi ? (ring > mma ? ring : mma) : (epi > mma ? epi : mma);
}

}  // namespace bkg
