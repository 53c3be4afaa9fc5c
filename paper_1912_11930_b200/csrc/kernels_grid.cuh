// kernels_grid.cuh — K1 for grid stencils (3-D; 2-D grids: kernels_grid2.cuh), the
// operand planes tiled through shared memory by TMA tensor copies: Q = A P
// (kernels.hpp:129-157), alpha = <<P, Q>> (kernels.hpp:59-88), last CTA:
// lambda = alpha^-1 rho_prev (kernels.hpp:231-240).
//
// When the CSR matrix is *exactly* a 7- or 27-point stencil with one value per
// offset on a lexicographic nx x ny x nz grid, boundary rows truncated
// (verified entry by entry on device, grid.cu: BASELINE configs C2, C4, C5),
// row (x, y, z) of A P is sum_o c[o] P[(x, y, z) + o] with P = 0 outside the
// grid.  P (n x K row-major) is then a 4-D tensor (column, x, y, z) and a
// 16 x 16 tile of one z-plane plus its one-point halo, 16 columns wide, is ONE
// cp.async.bulk.tensor.4d copy (box 16 x 18 x 18 x 1, SWIZZLE_128B; the halo
// outside the grid is zero-filled by the TMA unit, which is exactly the
// truncated row).  No CSR index or value is read in the loop.  (VAR: the
// values differ from row to row on a 5 / 7-point star; the stage then also
// receives the tile's coefficients from a DIA copy, three more tensor copies.)
// Planes outside the tensor are neither copied nor computed.
//
// Work item = (z-chunk, tile, 16-column slice); CTA j of a persistent grid
// takes items j, j + grid, ... (slice fastest, then x tiles: concurrently
// running CTAs share their halos in L2).  The item's planes z0-1 .. z1 stream
// through a ring of NS stages (one mbarrier each); the last of the 16 warps to
// finish a stage (a shared-memory counter) issues the copy of the plane NS
// steps ahead into it, so no warp ever waits for a free stage and there is no
// CTA-wide barrier in the loop.  Warp w owns 8 x 2 points (x half w & 1, tile
// rows 2 (w >> 1) + {0, 1}) x 16 columns as four "row groups" of 4 points
// (x = 8 (w & 1) + (g & 1) + 2 r, y = 2 (w >> 1) + (g >> 1)) -- the groups'
// neighbourhoods overlap in x and y, so a warp step reads 12 (7-point) or 16
// (27-point) operand points per lane for its 4 rows, not 20 / 36 -- whose
// lane (r = lane & 3, m = lane >> 2) holds columns {2m, 2m+1} of point r --
// one LDS.128 per operand point, conflict-free under the 128-byte swizzle
// because the four points sit two box rows apart -- and which is at the same
// time the FP64 DMMA m8n8k4 operand layout (A[m][r], B[r][m]) of the Gram
// P^T Q over "even" / "odd" column blocks: no relayout, no scratch.
//
// March in z, scatter form: the 5 (7-point) or 9 (27-point) in-plane values
// of plane t are read once and feed rows t-1 (their dz = +1 terms: the row is
// complete, stored and added to the Gram), t and t+1, so an operand point is
// read from shared memory 5 / 9 times instead of 7 / 27.  A row's products
// are summed plane by plane (dz = -1, 0, +1), a different order from the CSR
// kernels: fast-mode parity bars only.
//
// Long launches pace their persistent CTAs against a grid-wide counter (PACE,
// GridArgs::sync_every) so that neighbouring tiles stay within a few planes of
// each other and find their shared halo rows in L2.
#pragma once

#include <cuda.h>

#include "kernels_stage.cuh"

namespace bkg {

constexpr int kGridBX = 16, kGridBY = 16;  // tile of grid points per plane
constexpr int kGridWarps = kGridBY;        // compute warps: one per tile row
constexpr int kGridThreads = kGridWarps * 32;  // 4 warps per scheduler: 128 registers
constexpr int kGridW = 16;                 // columns per slice (128-byte box rows)
constexpr int kGridPitch = kGridBX + 2;    // box rows per tile row
constexpr int kGridBoxRows = kGridPitch * (kGridBY + 2);
constexpr int kGridBoxBytes = kGridBoxRows * 128;
constexpr int kGridStageBytes = (kGridBoxBytes + 1023) / 1024 * 1024;
// Variable coefficients (VAR): the stage also holds the tile's coefficients from
// the DIA copy of the matrix (grid.cu: V[slot][row], slots dz-1 | dy-1 dx-1 0
// dx+1 dy+1 | dz+1): the 5 in-plane slots of plane t, slot dz+1 of plane t-1
// and slot dz-1 of plane t+1, 16 x 16 doubles each.
constexpr int kGridTile = kGridBX * kGridBY;
constexpr int kGridValBytes = 7 * kGridTile * 8;
constexpr int kGridStageBytesVar = kGridStageBytes + kGridValBytes;

struct GridMaps {  // p: the operand block vector; v5 / v1: the DIA copy, boxes of 5 / 1 slots
  CUtensorMap p, v5, v1;
};

// Row groups of a warp (tuning, B200 sweeps in DESIGN.md §5):
//   1  8 x 2 points: x = 8 (w & 1) + (g & 1) + 2 r, y = 2 (w >> 1) + (g >> 1)
//   0  16 x 1 points: x = 8 (g >> 1) + (g & 1) + 2 r, y = w
#ifndef BKG_GRID_ARR
#define BKG_GRID_ARR 1
#endif
__host__ __device__ constexpr int grid_gx(int q) {
  return BKG_GRID_ARR ? (q & 1) : 8 * (q >> 1) + (q & 1);
}
__host__ __device__ constexpr int grid_gy(int q) { return BKG_GRID_ARR ? (q >> 1) : 0; }
constexpr int kGridWinX = BKG_GRID_ARR ? 4 : 12;  // window of a lane's four points + halo
constexpr int kGridWinY = BKG_GRID_ARR ? 4 : 3;

struct GridArgs {
  int nx, ny, nz;
  int tx, ty;       // tiles per axis
  int zchunk, nzc;  // planes per item, items per (tile, slice)
  // Rows produced: planes [z0, min(z0 + zchunk, zend)) for z0 = zbeg + c zstride,
  // c < nzc (one solver: zbeg 0, zstride = zchunk, zend = nz).  The operand
  // tensor may start zoff planes below plane 0 (a z-slab part with its ghost
  // plane, psolver.cu): plane t is tensor plane t + zoff, and planes outside
  // the tensor read as zero.
  int zbeg, zend, zstride, zoff;
  // planes that exist in the operand tensor: [tmin, tmax] (part coordinates).
  // A plane outside is all zero: it is neither copied nor computed, and a row
  // whose dz = +1 plane does not exist is finished by a tail step.
  int tmin, tmax;
  int ns;           // ring depth
  // Lockstep pacing (0: off): before issuing the copy of its step j, j a
  // multiple of sync_every, a CTA waits until the grid as a whole has issued
  // (j / sync_every - sync_lead) segments per CTA, so neighbouring tiles stay
  // within a few planes of each other and read their shared halo rows from L2
  // (without it CTAs drift apart over a launch's rounds: ncu, C5, 1.31x the
  // operand bytes from DRAM).  Performance only: the wait times out.
  int sync_every, sync_lead;
  int64_t nitems;   // nzc * ty * tx * (K / 16)
  // coefficient of offset (dx, dy, dz) at [dz + 1][(dy + 1) * 3 + (dx + 1)]
  double c[3][9];
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// one plane tile: box (16 columns, 18 x, 18 y, 1 z) at (c0, x, y, z) -> dst
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int c0, int x, int y,
                                            int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// Grid totals (red[lane * NACC + slice * 8 + (i * 2 + j) * 2 + e] = D_ij of the
// slice, D layout) -> row-major p x p blocks.  Column c of a slice is element
// c & 1 of column pair c >> 1.
template <int K, int P, bool GLOBAL>
__device__ void gather_gram_grid(const double* red, double* blocks) {
  constexpr int NACC = 8 * (K / kGridW);
  constexpr int NB = GLOBAL ? 1 : K / P;
  for (int idx = threadIdx.x; idx < NB * P * P; idx += blockDim.x) {
    const int blk = idx / (P * P), pa = (idx / P) % P, pb = idx % P;
    double s = 0.0;
    const int g0 = GLOBAL ? 0 : blk, g1 = GLOBAL ? K / P : blk + 1;
    for (int g = g0; g < g1; ++g) {
      const int ca = g * P + pa, cb = g * P + pb;  // same slice: P divides 16
      const int sl = ca / kGridW, a = ca % kGridW, b = cb % kGridW;
      const int lane = ((a >> 1) << 2) | (b >> 2), e = (b >> 1) & 1;
      s += red[lane * NACC + sl * 8 + ((a & 1) * 2 + (b & 1)) * 2 + e];
    }
    blocks[idx] = s;
  }
}

// PACE: the lockstep pacing compiled in (GridArgs::sync_every > 0 launches;
// its live state costs the 27-point loop 14% when merely present).
template <int K, int P, bool GLOBAL, bool FULL27, bool PACE, bool VAR = false, bool ISO = false>
__global__ void __launch_bounds__(kGridThreads, 1)
    k1_grid(IterArgs a, GridArgs g, const __grid_constant__ GridMaps tm) {
  static_assert(!(VAR && FULL27), "variable coefficients: 5 / 7-point stencils");
  static_assert(!ISO || (FULL27 && BKG_GRID_ARR == 1), "isotropic form: 27-point, 8 x 2 groups");
  constexpr int STAGE = VAR ? kGridStageBytesVar : kGridStageBytes;
  using S = FastSmem<K, P, 1, GLOBAL>;
  constexpr int NSL = K / kGridW;
  constexpr int NACC = 8 * NSL;
  static_assert(K % kGridW == 0 && P <= kGridW && kGridW % P == 0, "16-column slices");
  if (stopped(a.ctrl)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  extern __shared__ unsigned char smdyn[];
  // SWIZZLE_128B works on shared-memory address bits: 1024-byte aligned stages
  unsigned char* smraw = smdyn + ((1024u - (smem_u32(smdyn) & 1023u)) & 1023u);
  const int NS = g.ns;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + (size_t)NS * STAGE);
  int* fin = reinterpret_cast<int*>(full + NS);  // per stage: warps done with it
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      fin[s] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t G = gridDim.x;
  const int64_t nmine = g.nitems > (int64_t)blockIdx.x ? (g.nitems - blockIdx.x + G - 1) / G : 0;
  auto decode = [&](int64_t i, int& slice, int& x0, int& y0, int& z0, int& z1) {
    int64_t r = blockIdx.x + i * G;
    slice = (int)(r % NSL);
    r /= NSL;
    x0 = (int)(r % g.tx) * kGridBX;
    r /= g.tx;
    y0 = (int)(r % g.ty) * kGridBY;
    z0 = g.zbeg + (int)(r / g.ty) * g.zstride;
    z1 = min(z0 + g.zchunk, g.zend);
  };
  // the plane copies in issue order: planes z0-1 .. z1 of item 0, 1, ...
  struct Cursor {
    int64_t i;
    int slice, x0, y0, z1, t;  // z1: last plane copied for the item
  };
  auto cur_start = [&](Cursor& c, int64_t i) {
    c.i = i;
    if (i < nmine) {
      int z0, z1;
      decode(i, c.slice, c.x0, c.y0, z0, z1);
      c.t = max(z0 - 1, g.tmin);
      c.z1 = min(z1, g.tmax);
    }
  };
  auto cur_next = [&](Cursor& c) {
    if (++c.t > c.z1) cur_start(c, c.i + 1);
  };
  auto issue = [&](const Cursor& c, int s) {  // one elected lane
    unsigned char* st = smraw + (size_t)s * STAGE;
    mbar_expect_tx(full + s, kGridBoxBytes + (VAR ? kGridValBytes : 0));
    tma_load_4d(st, &tm.p, c.slice * kGridW, c.x0 - 1, c.y0 - 1, c.t + g.zoff, full + s);
    if constexpr (VAR) {  // coefficients of rows t (in-plane), t-1 (dz+1), t+1 (dz-1)
      unsigned char* sv = st + kGridStageBytes;
      tma_load_4d(sv, &tm.v5, c.x0, c.y0, c.t, 1, full + s);
      tma_load_4d(sv + 5 * kGridTile * 8, &tm.v1, c.x0, c.y0, c.t - 1, 6, full + s);
      tma_load_4d(sv + 6 * kGridTile * 8, &tm.v1, c.x0, c.y0, c.t + 1, 0, full + s);
    }
  };
  // lockstep pacing (GridArgs::sync_every): called by the issuing lane before
  // the copy of step jn; counts this CTA into segment jn / sync_every and waits
  // for the grid.  A CTA that has issued its last copy adds a large constant so
  // nobody waits for it again.
  unsigned long long* gsync = &a.ctrl->grid_sync;
  auto pace = [&](uint32_t jn) {
    if constexpr (!PACE) return;
    if (g.sync_every <= 0 || jn % (uint32_t)g.sync_every != 0) return;
    const long long seg = jn / (uint32_t)g.sync_every;
    atomicAdd(gsync, 1ull);
    // the ring's first NS copies are issued unpaced: segments 0 .. seg0 - 1
    const long long seg0 = (NS - 1) / g.sync_every + 1;
    const long long want = (seg - g.sync_lead - seg0 + 1) * (long long)G;
    if (want <= 0) return;
    const long long t0 = clock64();
    while ((long long)*reinterpret_cast<volatile unsigned long long*>(gsync) < want)
      if (clock64() - t0 > (1ll << 21)) break;  // ~1 ms: never a correctness dependency
  };
  auto issued_last = [&](const Cursor& c) {  // c was this CTA's final copy
    if (PACE && g.sync_every > 0 && c.i + 1 >= nmine && c.t >= c.z1) atomicAdd(gsync, 1ull << 40);
  };
  Cursor ahead;  // the copy NS steps ahead of the plane being consumed
  cur_start(ahead, 0);
  for (int s = 0; s < NS; ++s) {
    if (threadIdx.x == 0 && ahead.i < nmine) {
      issue(ahead, s);
      issued_last(ahead);
    }
    if (ahead.i < nmine) cur_next(ahead);
  }

  double gram[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) gram[e] = 0.0;

  {
    // ---- consumers ----
    const int r = lane & 3, m = lane >> 2;
    // box row of group q's point: (yw + (q>>1) + 1) * pitch + 1 + xw + (q&1) + 2 r
    const int xw = BKG_GRID_ARR ? 8 * (warp & 1) : 0, yw = BKG_GRID_ARR ? 2 * (warp >> 1) : warp;
    const int ri0 = (yw + 1) * kGridPitch + 1 + xw + 2 * r;
    const int pidx0 = yw * kGridBX + xw + 2 * r;  // tile point of group 0 (coefficient tiles)
    uint32_t j = 0;
#pragma unroll 1
    for (int64_t i = 0; i < nmine; ++i) {
      int slice, x0, y0, z0, z1;
      decode(i, slice, x0, y0, z0, z1);
      double acc_a[4][2], acc_b[4][2], pown[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        acc_a[q][0] = acc_a[q][1] = acc_b[q][0] = acc_b[q][1] = pown[q][0] = pown[q][1] = 0.0;
      double* qbase = a.Q + slice * kGridW + 2 * m;
      const int tlo = max(z0 - 1, g.tmin), thi = min(z1, g.tmax);
      // rows t-1 are complete: store, Gram with their own P (the previous step's centre)
      auto emit_rows = [&](int t, const double (&qa)[4][2]) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int gx = x0 + xw + grid_gx(q) + 2 * r, gy = y0 + yw + grid_gy(q);
          if (gx < g.nx && gy < g.ny) {
            const int64_t row = ((int64_t)(t - 1) * g.ny + gy) * g.nx + gx;
            *reinterpret_cast<double2*>(qbase + row * K) = make_double2(qa[q][0], qa[q][1]);
          }
#pragma unroll
          for (int ii = 0; ii < 2; ++ii)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              double d[2] = {gram[(ii * 2 + jj) * 2], gram[(ii * 2 + jj) * 2 + 1]};
              dmma(d, pown[q][ii], qa[q][jj]);
              gram[(ii * 2 + jj) * 2] = d[0];
              gram[(ii * 2 + jj) * 2 + 1] = d[1];
            }
        }
      };
#pragma unroll 1
      for (int t = tlo; t <= thi; ++t, ++j) {
        const int s = (int)(j % NS);
        mbar_wait(full + s, (j / NS) & 1);
        const unsigned char* st = smraw + (size_t)s * STAGE;
        const double* sv = reinterpret_cast<const double*>(st + kGridStageBytes) + pidx0;  // VAR
        const bool emit = t > z0;  // row t-1 belongs to this item
        // Window of this lane's four points: box rows ri0 + (py-1) pitch + (px-1),
        // px, py = 0..3.  Each operand point is read once and feeds every group
        // q (point (1 + (q&1), 1 + (q>>1)) of the window) that has it as a
        // neighbour: rows t-1 (qa, finished here), t (na) and t+1 (nb).
        double qa[4][2], na[4][2], nb[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          qa[q][0] = acc_a[q][0];
          qa[q][1] = acc_a[q][1];
          na[q][0] = acc_b[q][0];
          na[q][1] = acc_b[q][1];
          nb[q][0] = nb[q][1] = 0.0;
        }
        if constexpr (ISO) {
          // Isotropic 27-point stencil: a coefficient depends only on how many
          // of dx, dy, dz are nonzero (centre c0, faces cf, edges ce, corners cc).
          // Per point and plane three sums -- the centre value, its 4 in-plane
          // face neighbours, its 4 in-plane diagonal neighbours -- feed row t
          // (c0, cf, ce) and rows t-1 / t+1 (cf, ce, cc, the same number w):
          // 15 FP64 operations per point and column instead of 27 FMAs.  The
          // two groups of a window row pair are done together (12 reads each).
          const double c0 = g.c[1][4], cf = g.c[1][1], ce = g.c[1][0], cc = g.c[0][0];
#pragma unroll
          for (int yo = 0; yo < 2; ++yo) {
            double s0[2][2], s1[2][2], s2[2][2];
#pragma unroll
            for (int xo = 0; xo < 2; ++xo)
              s0[xo][0] = s0[xo][1] = s1[xo][0] = s1[xo][1] = s2[xo][0] = s2[xo][1] = 0.0;
#pragma unroll
            for (int wy = 0; wy < 3; ++wy)
#pragma unroll
              for (int px = 0; px < 4; ++px) {
                const int row = ri0 + (yo + wy - 1) * kGridPitch + (px - 1);
                const double2 v =
                    *reinterpret_cast<const double2*>(st + row * 128 + ((m ^ (row & 7)) << 4));
#pragma unroll
                for (int xo = 0; xo < 2; ++xo) {
                  const int dx = px - 1 - xo;
                  if (dx < -1 || dx > 1) continue;
                  const int cls = (dx != 0) + (wy != 1);
                  if (cls == 0) {
                    s0[xo][0] = v.x;
                    s0[xo][1] = v.y;
                  } else if (cls == 1) {
                    s1[xo][0] += v.x;
                    s1[xo][1] += v.y;
                  } else {
                    s2[xo][0] += v.x;
                    s2[xo][1] += v.y;
                  }
                }
              }
#pragma unroll
            for (int xo = 0; xo < 2; ++xo) {
              const int q = yo * 2 + xo;
#pragma unroll
              for (int cidx = 0; cidx < 2; ++cidx) {
                const double w = fma(cc, s2[xo][cidx], fma(ce, s1[xo][cidx], cf * s0[xo][cidx]));
                na[q][cidx] =
                    fma(ce, s2[xo][cidx], fma(cf, s1[xo][cidx], fma(c0, s0[xo][cidx], na[q][cidx])));
                qa[q][cidx] += w;
                nb[q][cidx] = w;
                acc_b[q][cidx] = s0[xo][cidx];  // parked: next step's Gram operand
              }
            }
          }
        } else {
  #pragma unroll
          for (int py = 0; py < kGridWinY; ++py)
  #pragma unroll
            for (int px = 0; px < kGridWinX; ++px) {
              bool any = false;
  #pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int dx = px - 1 - grid_gx(q), dy = py - 1 - grid_gy(q);
                if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && (FULL27 || dx == 0 || dy == 0))
                  any = true;
              }
              if (!any) continue;
              const int row = ri0 + (py - 1) * kGridPitch + (px - 1);
              const double2 v =
                  *reinterpret_cast<const double2*>(st + row * 128 + ((m ^ (row & 7)) << 4));
  #pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int dx = px - 1 - grid_gx(q), dy = py - 1 - grid_gy(q);
                if (dx < -1 || dx > 1 || dy < -1 || dy > 1) continue;
                if (!(FULL27 || dx == 0 || dy == 0)) continue;
                const int o = (dy + 1) * 3 + dx + 1;
                double c0 = g.c[1][o], cp = g.c[2][o], cm = g.c[0][o];
                if constexpr (VAR) {  // row q's own coefficients from the DIA tiles
                  const int pq = grid_gy(q) * kGridBX + grid_gx(q);
                  const int sl = o == 1 ? 0 : o == 3 ? 1 : o == 4 ? 2 : o == 5 ? 3 : 4;
                  c0 = sv[sl * kGridTile + pq];
                  if (o == 4) {
                    cp = sv[5 * kGridTile + pq];
                    cm = sv[6 * kGridTile + pq];
                  }
                }
                na[q][0] = fma(c0, v.x, na[q][0]);
                na[q][1] = fma(c0, v.y, na[q][1]);
                if (FULL27 || o == 4) {
                  qa[q][0] = fma(cp, v.x, qa[q][0]);
                  qa[q][1] = fma(cp, v.y, qa[q][1]);
                  nb[q][0] = fma(cm, v.x, nb[q][0]);
                  nb[q][1] = fma(cm, v.y, nb[q][1]);
                }
                if (o == 4) {  // the group's own point: next step's Gram operand
                  acc_b[q][0] = v.x;  // parked in acc_b (dead: copied into na above)
                  acc_b[q][1] = v.y;
                }
              }
            }
        }
        if (emit) emit_rows(t, qa);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          pown[q][0] = acc_b[q][0];
          pown[q][1] = acc_b[q][1];
          acc_a[q][0] = na[q][0];
          acc_a[q][1] = na[q][1];
          acc_b[q][0] = nb[q][0];
          acc_b[q][1] = nb[q][1];
        }
        // the last warp done with stage s refills it with the plane NS steps ahead
        __threadfence_block();
        __syncwarp();
        if (lane == 0 && atomicAdd(fin + s, 1) == kGridWarps - 1) {
          fin[s] = 0;
          if (ahead.i < nmine) {
            pace(j + NS);
            issue(ahead, s);
            issued_last(ahead);
          }
        }
        if (ahead.i < nmine) cur_next(ahead);
      }
      if (thi < z1 && thi >= z0) emit_rows(thi + 1, acc_a);  // plane z1 does not exist: row z1-1 is done
    }
  }

  // ---- deterministic grid reduction of the slice Grams, lambda solve ----
  __syncthreads();  // the ring is reused as the reduction buffer
  const int myslice = (int)(blockIdx.x % NSL);  // grid is a multiple of NSL: one slice per CTA
  double acc[NACC];
#pragma unroll
  for (int sl = 0; sl < NSL; ++sl)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[sl * 8 + e] = sl == myslice ? gram[e] : 0.0;
  double* red = reinterpret_cast<double*>(smraw);
  if (!grid_reduce<32, NACC, kGridThreads>(acc, red, a.partials, a.gpart, a.ctrl->tickets,
                                           a.group))
    return;
  double* alpha = red + 32 * NACC;
  double* ws = alpha + 3 * S::CS;
  gather_gram_grid<K, P, GLOBAL>(red, alpha);
  __syncthreads();
  if (PACE && threadIdx.x == 0) *gsync = 0;  // every CTA is past its loop: ready for the next launch
  if (a.dist) {  // row-partitioned solver: publish this part's alpha (psolver.cu)
    for (int i = threadIdx.x; i < S::CS; i += kGridThreads)
      a.red1[i] = (a.dist_acc ? a.red1[i] : 0.0) + alpha[i];
    return;
  }
  const int bad = fast_bsolve<P>(S::NB, P, alpha, a.coef + S::CS, a.coef, ws);  // lambda
  if (bad >= 0) record_breakdown(a.ctrl, bad, 1);
}

// Dynamic shared memory of k1_grid with a ring of ns stages.
template <int K, int P, bool GLOBAL>
int k1_grid_smem(int ns, bool var) {
  using S = FastSmem<K, P, 1, GLOBAL>;
  const int main = ns * (var ? kGridStageBytesVar : kGridStageBytes) + ns * 8 + ns * 4;
  const int epi = (int)sizeof(double) *
                  (32 * 8 * (K / kGridW) + 3 * S::CS + bsolve_ws_doubles(P, kGridThreads) + K);
  return (main > epi ? main : epi) + 1024;  // + alignment slack
}

}  // namespace bkg
