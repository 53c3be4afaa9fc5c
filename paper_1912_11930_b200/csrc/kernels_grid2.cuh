// kernels_grid2.cuh — k1_grid for 2-D grids: the z-march of kernels_grid.cuh one
// dimension down.  Q = A P (kernels.hpp:129-157), alpha = <<P, Q>> (:59-88),
// last CTA: lambda = alpha^-1 rho_prev (:231-240) for a matrix that is exactly
// a 5- or 9-point stencil on a lexicographic nx x ny grid (grid.cu), constant
// coefficients or (VAR, 5-point) one coefficient per entry from the DIA copy.
//
// A 2-D grid has one plane, so the 3-D kernel's item is a single step and its
// 16 x 16 tiles re-read a 27% halo, the y part of it from DRAM (tiles adjacent
// in y run far apart).  Here a tile is 128 grid points of one grid line plus
// its two x neighbours, 16 columns wide -- ONE cp.async.bulk.tensor.3d copy
// (box 16 x 130 x 1, SWIZZLE_128B, zero fill outside the grid), a 1.6% halo --
// and the CTA marches in y: the 3 in-line values of line t feed rows t-1
// (their dy = +1 term: finished, stored, added to the Gram), t and t+1, exactly
// the scatter form of the z-march.  Work item = (y-chunk, x tile, 16-column
// slice); 8 warps per CTA, warp w owns points 16w .. 16w+15 of the tile as four
// row groups (x = 8 (g >> 1) + (g & 1) + 2 r), lane (r = lane & 3, m = lane >> 2)
// holding columns {2m, 2m+1}: conflict-free LDS.128 under the swizzle and the
// DMMA operand layout of the Gram at once (kernels_grid.cuh).  Lines stream
// through a ring of NS stages; the last warp done with a stage refills it.
#pragma once

#include "kernels_grid.cuh"

namespace bkg {

constexpr int kG2BX = 128;                  // grid points per tile (one line)
constexpr int kG2Warps = kG2BX / 16;        // 8
constexpr int kG2Threads = kG2Warps * 32;   // 256
constexpr int kG2BoxBytes = (kG2BX + 2) * 128;
constexpr int kG2StageBytes = (kG2BoxBytes + 1023) / 1024 * 1024;
constexpr int kG2ValBytes = 5 * kG2BX * 8;  // VAR: dx-1, 0, dx+1 of line t; dy+1 of t-1; dy-1 of t+1
constexpr int kG2StageBytesVar = kG2StageBytes + kG2ValBytes;
static_assert(kG2Threads == kThreads && kG2ValBytes % 1024 == 0, "grid_reduce, stage alignment");

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// GridArgs (kernels_grid.cuh) as used here: nx, ny; tx = x tiles; items cover
// lines [z0, min(z0 + zchunk, zend)), z0 = zbeg + c zstride; tmin / tmax = first
// / last grid line; c[1][(dy+1)*3 + dx+1] = the stencil.
template <int K, int P, bool GLOBAL, bool NINE, bool VAR>
__global__ void __launch_bounds__(kG2Threads, 2)
    k1_grid2(IterArgs a, GridArgs g, const __grid_constant__ GridMaps tm) {
  static_assert(!(VAR && NINE), "variable coefficients: 5-point stencils");
  using S = FastSmem<K, P, 1, GLOBAL>;
  constexpr int NSL = K / kGridW;
  constexpr int NACC = 8 * NSL;
  constexpr int STAGE = VAR ? kG2StageBytesVar : kG2StageBytes;
  if (stopped(a.ctrl)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  extern __shared__ unsigned char smdyn[];
  unsigned char* smraw = smdyn + ((1024u - (smem_u32(smdyn) & 1023u)) & 1023u);
  const int NS = g.ns;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + (size_t)NS * STAGE);
  int* fin = reinterpret_cast<int*>(full + NS);
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
  auto decode = [&](int64_t i, int& slice, int& x0, int& z0, int& z1) {
    int64_t r = blockIdx.x + i * G;
    slice = (int)(r % NSL);
    r /= NSL;
    x0 = (int)(r % g.tx) * kG2BX;
    z0 = g.zbeg + (int)(r / g.tx) * g.zstride;
    z1 = min(z0 + g.zchunk, g.zend);
  };
  struct Cursor {
    int64_t i;
    int slice, x0, z1, t;
  };
  auto cur_start = [&](Cursor& c, int64_t i) {
    c.i = i;
    if (i < nmine) {
      int z0, z1;
      decode(i, c.slice, c.x0, z0, z1);
      c.t = max(z0 - 1, g.tmin);
      c.z1 = min(z1, g.tmax);
    }
  };
  auto cur_next = [&](Cursor& c) {
    if (++c.t > c.z1) cur_start(c, c.i + 1);
  };
  auto issue = [&](const Cursor& c, int s) {  // one elected lane
    unsigned char* st = smraw + (size_t)s * STAGE;
    mbar_expect_tx(full + s, kG2BoxBytes + (VAR ? kG2ValBytes : 0));
    tma_load_3d(st, &tm.p, c.slice * kGridW, c.x0 - 1, c.t, full + s);
    if constexpr (VAR) {  // DIA slots 2..4 of line t, slot 5 of line t-1, slot 1 of line t+1
      unsigned char* sv = st + kG2StageBytes;
      tma_load_3d(sv, &tm.v5, c.x0, c.t, 2, full + s);
      tma_load_3d(sv + 3 * kG2BX * 8, &tm.v1, c.x0, c.t - 1, 5, full + s);
      tma_load_3d(sv + 4 * kG2BX * 8, &tm.v1, c.x0, c.t + 1, 1, full + s);
    }
  };
  Cursor ahead;
  cur_start(ahead, 0);
  for (int s = 0; s < NS; ++s) {
    if (threadIdx.x == 0 && ahead.i < nmine) issue(ahead, s);
    if (ahead.i < nmine) cur_next(ahead);
  }

  double gram[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) gram[e] = 0.0;
  {
    const int r = lane & 3, m = lane >> 2;
    const int xw = 16 * warp;
    const int ri0 = 1 + xw + 2 * r;    // box row of group 0's point
    const int pidx0 = xw + 2 * r;      // its tile point (coefficient tiles)
    uint32_t j = 0;
#pragma unroll 1
    for (int64_t i = 0; i < nmine; ++i) {
      int slice, x0, z0, z1;
      decode(i, slice, x0, z0, z1);
      double acc_a[4][2], acc_b[4][2], pown[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        acc_a[q][0] = acc_a[q][1] = acc_b[q][0] = acc_b[q][1] = pown[q][0] = pown[q][1] = 0.0;
      double* qbase = a.Q + slice * kGridW + 2 * m;
      const int tlo = max(z0 - 1, g.tmin), thi = min(z1, g.tmax);
      auto emit_rows = [&](int t, const double (&qa)[4][2]) {  // rows of line t-1 are complete
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int gx = x0 + xw + 8 * (q >> 1) + (q & 1) + 2 * r;
          if (gx < g.nx) {
            const int64_t row = (int64_t)(t - 1) * g.nx + gx;
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
        const double* sv = reinterpret_cast<const double*>(st + kG2StageBytes) + pidx0;  // VAR
        const bool emit = t > z0;
        double qa[4][2], na[4][2], nb[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          qa[q][0] = acc_a[q][0];
          qa[q][1] = acc_a[q][1];
          na[q][0] = acc_b[q][0];
          na[q][1] = acc_b[q][1];
          nb[q][0] = nb[q][1] = 0.0;
        }
        // window of the lane's four points: box rows ri0 + px - 1, px = 0..11
#pragma unroll
        for (int px = 0; px < 12; ++px) {
          bool any = false;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int dx = px - 1 - (8 * (q >> 1) + (q & 1));
            if (dx >= -1 && dx <= 1) any = true;
          }
          if (!any) continue;
          const int row = ri0 + px - 1;
          const double2 v =
              *reinterpret_cast<const double2*>(st + row * 128 + ((m ^ (row & 7)) << 4));
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int gxq = 8 * (q >> 1) + (q & 1);
            const int dx = px - 1 - gxq;
            if (dx < -1 || dx > 1) continue;
            double c0 = g.c[1][3 + dx + 1], cp = g.c[1][6 + dx + 1], cm = g.c[1][dx + 1];
            if constexpr (VAR) {
              c0 = sv[(dx + 1) * kG2BX + gxq];
              if (dx == 0) {
                cp = sv[3 * kG2BX + gxq];
                cm = sv[4 * kG2BX + gxq];
              }
            }
            na[q][0] = fma(c0, v.x, na[q][0]);
            na[q][1] = fma(c0, v.y, na[q][1]);
            if (NINE || dx == 0) {
              qa[q][0] = fma(cp, v.x, qa[q][0]);
              qa[q][1] = fma(cp, v.y, qa[q][1]);
              nb[q][0] = fma(cm, v.x, nb[q][0]);
              nb[q][1] = fma(cm, v.y, nb[q][1]);
            }
            if (dx == 0) {  // the group's own point: next step's Gram operand
              acc_b[q][0] = v.x;
              acc_b[q][1] = v.y;
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
        __threadfence_block();
        __syncwarp();
        if (lane == 0 && atomicAdd(fin + s, 1) == kG2Warps - 1) {
          fin[s] = 0;
          if (ahead.i < nmine) issue(ahead, s);
        }
        if (ahead.i < nmine) cur_next(ahead);
      }
      if (thi < z1 && thi >= z0) emit_rows(thi + 1, acc_a);  // line z1 does not exist
    }
  }

  __syncthreads();  // the ring is reused as the reduction buffer
  const int myslice = (int)(blockIdx.x % NSL);  // grid is a multiple of NSL
  double acc[NACC];
#pragma unroll
  for (int sl = 0; sl < NSL; ++sl)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[sl * 8 + e] = sl == myslice ? gram[e] : 0.0;
  double* red = reinterpret_cast<double*>(smraw);
  if (!grid_reduce<32, NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group)) return;
  double* alpha = red + 32 * NACC;
  double* ws = alpha + 3 * S::CS;
  gather_gram_grid<K, P, GLOBAL>(red, alpha);
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kG2Threads)
      a.red1[i] = (a.dist_acc ? a.red1[i] : 0.0) + alpha[i];
    return;
  }
  const int bad = fast_bsolve<P>(S::NB, P, alpha, a.coef + S::CS, a.coef, ws);  // lambda
  if (bad >= 0) record_breakdown(a.ctrl, bad, 1);
}

template <int K, int P, bool GLOBAL>
int k1_grid2_smem(int ns, bool var) {
  using S = FastSmem<K, P, 1, GLOBAL>;
  const int main = ns * (var ? kG2StageBytesVar : kG2StageBytes) + ns * 8 + ns * 4;
  const int epi = (int)sizeof(double) *
                  (32 * 8 * (K / kGridW) + 3 * S::CS + bsolve_ws_doubles(P, kG2Threads) + K);
  return (main > epi ? main : epi) + 1024;
}

}  // namespace bkg
