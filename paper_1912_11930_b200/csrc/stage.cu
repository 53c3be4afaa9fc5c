// stage.cu — the staged-block copy of a CSR matrix for k1_stage
// (kernels_stage.cuh), built on device once per matrix and block shape.
//
// Blocks: R row slots each (rowid, -1 = empty).  When the matrix pattern is a
// lexicographic grid stencil (grid_detect: the column offsets c - r of a
// sample of rows form the clusters {1}, {nx - 1 .. nx + 1}, {nx ny ..}), a
// block is a bx x by x bz box of grid points, so a block's operand rows -- the
// box plus its halo shell -- are ~2-3 rows per own row instead of ~5 (7-point)
// or ~10 (27-point) for R consecutive rows: that ratio is K1's L2 -> SM
// traffic.  Boxes are visited strip by strip (`strip` box rows in y), z-layer
// by z-layer inside a strip, so the z-neighbour planes of a layer-strip stay in
// L2 until the next layer reads them (P is read from DRAM ~once).  Any other
// matrix gets blocks of R consecutive rows.  The block shape never affects the
// result beyond the summation order of the Gram (fast-mode parity bars).
//
// For each block the staged set is the sorted union of its rows' column
// indices and its own rows (the Gram's P rows).  Runs of consecutive columns
// become segments {first row, rows}; entry (slot u of row slot i, CSR order)
// stores the index of its column inside the staged set (uint16) and its value,
// slot-major, padded with (the row's own staged index, 0.0) up to the block's
// longest row rounded up to 4 slots; one more index slot holds the staged
// position of the row itself (empty row slots: index 0, values 0).
//
// One warp per block merges the R sorted rows (CSR columns ascend,
// sparse_matrix.hpp:99-105) and the own rows: each step takes the warp-wide
// minimum head -- the next distinct column -- and every row whose head equals
// it records the staged index and advances.  Pass 0 counts (segments, staged
// rows, longest row); the host lays the blocks out; pass 1 writes.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <set>
#include <vector>

#include "bkg.h"
#include "common.cuh"
#include "host.cuh"

namespace bkg {

namespace {

constexpr int kStageSlotPad = 4;  // slots per block padded to the kernel's chunk

// rowid[b R + i]: consecutive rows (bx == 0) or grid boxes in strip order.
__global__ void k_stage_rowid(int64_t n, int R, int64_t nblk, int64_t nx, int64_t ny, int64_t nz,
                              int bx, int by, int bz, int strip, int32_t* __restrict__ rowid) {
  const int64_t tot = nblk * R;
  const int64_t nbx = bx ? (nx + bx - 1) / bx : 0, nby = bx ? (ny + by - 1) / by : 0;
  const int64_t nbz = bx ? (nz + bz - 1) / bz : 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / R;
    const int i = (int)(e % R);
    int64_t row = -1;
    if (bx == 0) {
      row = e < n ? e : -1;
    } else {
      const int64_t per_strip = (int64_t)strip * nbx * nbz;
      const int64_t t = b / per_strip, rem = b % per_strip;
      const int64_t h = min((int64_t)strip, nby - t * strip);  // box rows of this strip
      const int64_t bzi = rem / (h * nbx), rem2 = rem % (h * nbx);
      const int64_t byi = t * strip + rem2 / nbx, bxi = rem2 % nbx;
      const int64_t x = bxi * bx + i % bx, y = byi * by + (i / bx) % by,
                    z = bzi * bz + i / (bx * by);
      if (x < nx && y < ny && z < nz) row = (z * ny + y) * nx + x;
    }
    rowid[e] = (int32_t)row;
  }
}

template <int RL>  // row slots per lane: R <= 32 * RL
__global__ void k_stage_merge(int pass, int R, int64_t nblk, int smax,
                              const int32_t* __restrict__ rowid,
                              const int64_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                              const double* __restrict__ vals, int* __restrict__ cnt_seg,
                              int* __restrict__ cnt_rows, int* __restrict__ cnt_w,
                              const StageHdr* __restrict__ hdr, int2* __restrict__ segs,
                              uint16_t* __restrict__ lidx, double* __restrict__ svals) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = wid; b < nblk; b += nw) {
    int64_t e[RL], es[RL], ee[RL];
    int head[RL], ohead[RL];
    int w = 0;
#pragma unroll
    for (int t = 0; t < RL; ++t) {
      const int rl = lane + 32 * t;
      const int row = rl < R ? rowid[b * R + rl] : -1;
      e[t] = es[t] = ee[t] = 0;
      head[t] = INT_MAX;
      ohead[t] = row >= 0 ? row : INT_MAX;  // the row itself (the Gram's P row)
      if (row >= 0) {
        e[t] = es[t] = rowptr[row];
        ee[t] = rowptr[row + 1];
        if (e[t] < ee[t]) head[t] = cols[e[t]];
        w = max(w, (int)(ee[t] - es[t]));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
    w = (w + kStageSlotPad - 1) / kStageSlotPad * kStageSlotPad;
    int oidx[RL];  // staged index of the row itself (0 for an empty slot)
#pragma unroll
    for (int t = 0; t < RL; ++t) oidx[t] = 0;
    int cnt = 0, nseg = 0, last = 0, seg_first = 0, seg_len = 0;
    const int64_t ebase = pass ? hdr[b].ebeg : 0;
    const int64_t lbase = ebase + b * R;
    int2* sg = pass ? segs + b * smax : nullptr;
    while (true) {
      int h = INT_MAX;
#pragma unroll
      for (int t = 0; t < RL; ++t) h = min(h, min(head[t], ohead[t]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) h = min(h, __shfl_xor_sync(0xffffffffu, h, o));
      if (h == INT_MAX) break;
      if (cnt > 0 && h == last + 1) {
        ++seg_len;
      } else {
        if (pass && lane == 0 && cnt > 0) sg[nseg - 1] = make_int2(seg_first, seg_len);
        ++nseg;
        seg_first = h;
        seg_len = 1;
      }
#pragma unroll
      for (int t = 0; t < RL; ++t) {
        if (head[t] == h) {
          if (pass) {
            const int64_t off = (e[t] - es[t]) * R + lane + 32 * t;
            lidx[lbase + off] = (uint16_t)min(cnt, 0xFFFE);
            svals[ebase + off] = vals[e[t]];
          }
          ++e[t];
          head[t] = e[t] < ee[t] ? cols[e[t]] : INT_MAX;
        }
        if (ohead[t] == h) {
          oidx[t] = min(cnt, 0xFFFE);
          ohead[t] = INT_MAX;
        }
      }
      last = h;
      ++cnt;
    }
    if (pass) {
      if (lane == 0 && cnt > 0) sg[nseg - 1] = make_int2(seg_first, seg_len);
      for (int j = nseg + lane; j < smax; j += 32) sg[j] = make_int2(0, 0);
      // the row's own staged index (slot w), and the padding slots (rows
      // shorter than w, empty row slots): value 0 times the row's own operand
      // row -- a valid staged row, so the kernel's slot loop has no predicates
#pragma unroll
      for (int t = 0; t < RL; ++t) {
        const int rl = lane + 32 * t;
        if (rl >= R) continue;
        lidx[lbase + (int64_t)w * R + rl] = (uint16_t)oidx[t];
        for (int64_t u = ee[t] - es[t]; u < w; ++u) {
          lidx[lbase + u * R + rl] = (uint16_t)oidx[t];
          svals[ebase + u * R + rl] = 0.0;
        }
      }
    } else if (lane == 0) {
      cnt_seg[b] = nseg;
      cnt_rows[b] = cnt;
      cnt_w[b] = w;
    }
  }
}

template <int RL>
void merge_launch(bkg_ctx* c, int pass, int R, int64_t nblk, int smax, const int32_t* rowid,
                  const int64_t* rowptr, const int32_t* cols, const double* vals, int* cs, int* cr,
                  int* cw, const StageHdr* hdr, int2* segs, uint16_t* lidx, double* svals) {
  const int blocks = (int)std::min<int64_t>((nblk * 32 + 255) / 256, (int64_t)c->sm_count * 32);
  void* args[] = {&pass, &R, &nblk, &smax, &rowid, &rowptr, &cols, &vals,
                  &cs,   &cr, &cw,  &hdr,  &segs,  &lidx,   &svals};
  launch(c, (const void*)&k_stage_merge<RL>, std::max(1, blocks), 256, 0, args);
}

}  // namespace

// Grid shape of a lexicographically numbered stencil matrix from the column
// offsets c - r of a sample of rows from the middle of the matrix: the positive
// offsets cluster around 1, nx and nx ny (27-point: also nx ny +- nx).
// grid = {nx, ny, nz} and true when the clusters are consistent with n;
// otherwise false (blocks of consecutive rows are used).  A heuristic for the
// block shape only: no result depends on it.
bool grid_detect(bkg_ctx* c, int64_t n, const int64_t* rowptr, const int32_t* cols,
                 int64_t grid[3], std::vector<int64_t>* offsets) {
  grid[0] = grid[1] = grid[2] = 0;
  if (n < 64) return false;
  const int64_t ns = std::min<int64_t>(n, 4096), s0 = (n - ns) / 2;
  std::vector<int64_t> rp(ns + 1);
  d2h(c, rp.data(), rowptr + s0, ns + 1);
  sync(c);
  const int64_t e0 = rp[0], e1 = rp[ns];
  if (e1 - e0 <= 0 || e1 - e0 > ns * 64) return false;
  std::vector<int32_t> cl(e1 - e0);
  d2h(c, cl.data(), cols + e0, cl.size());
  sync(c);
  std::set<int64_t> offs, all;
  for (int64_t r = 0; r < ns; ++r)
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
      const int64_t d = (int64_t)cl[e - e0] - (s0 + r);
      if (d > 0) offs.insert(d);
      if (d != 0) all.insert(d);
      if (all.size() > 128) return false;
    }
  if (offsets) offsets->assign(all.begin(), all.end());
  // cluster centres of the positive offsets (a cluster = consecutive integers)
  std::vector<int64_t> centre;
  int64_t first = -1, prev = -1;
  for (int64_t d : offs) {
    if (first < 0) {
      first = prev = d;
    } else if (d == prev + 1) {
      prev = d;
    } else {
      centre.push_back((first + prev) / 2);
      first = prev = d;
    }
  }
  if (first >= 0) centre.push_back((first + prev) / 2);
  size_t i = 0;
  if (i < centre.size() && centre[i] == 1) ++i;  // the x neighbours
  if (i == centre.size()) return false;          // a 1-D chain: nothing to block
  const int64_t sy = centre[i++];
  int64_t sz = 0;
  const size_t left = centre.size() - i;
  if (left == 0) {
    sz = n;  // 2-D
  } else if (left == 1) {
    sz = centre[i];
  } else if (left == 3 && centre[i + 1] - centre[i] == sy && centre[i + 2] - centre[i + 1] == sy) {
    sz = centre[i + 1];
  } else {
    return false;
  }
  if (sy < 2 || sz % sy != 0 || n % sz != 0) return false;
  grid[0] = sy;
  grid[1] = sz / sy;
  grid[2] = n / sz;
  return true;
}

// Build (or rebuild) `out` with R row slots per block: boxes bx x by x bz of
// the grid {nx, ny, nz} when box[0] > 0 (R = bx by bz), consecutive rows
// otherwise.  Returns false -- and leaves out.R = 0 -- when a block needs more
// than `max_segs` segments or 0xFFFE staged rows (the kernel's limits).
bool stage_build(bkg_ctx* c, int64_t n, const int64_t* rowptr, const int32_t* cols,
                 const double* vals, int R, const int box[3], const int64_t grid[3], int strip,
                 int max_segs, StageCsr& out) {
  out.R = 0;
  BKG_REQUIRE(R >= 8 && R <= 256 && R % 8 == 0, BKG_INTERNAL, "stage_build: bad block height");
  const bool boxed = box && box[0] > 0;
  int64_t nblk;
  if (boxed) {
    BKG_REQUIRE(box[0] * box[1] * box[2] == R, BKG_INTERNAL, "stage_build: box != R");
    nblk = ((grid[0] + box[0] - 1) / box[0]) * ((grid[1] + box[1] - 1) / box[1]) *
           ((grid[2] + box[2] - 1) / box[2]);
  } else {
    nblk = (n + R - 1) / R;
  }
  out.rowid.ensure((size_t)nblk * R);
  {
    int64_t nn = n, nb = nblk, nx = boxed ? grid[0] : 0, ny = boxed ? grid[1] : 0,
            nz = boxed ? grid[2] : 0;
    int rr = R, bx = boxed ? box[0] : 0, by = boxed ? box[1] : 0, bz = boxed ? box[2] : 0;
    int st = std::max(1, strip);
    int32_t* rid = out.rowid.ptr;
    void* args[] = {&nn, &rr, &nb, &nx, &ny, &nz, &bx, &by, &bz, &st, &rid};
    launch(c, (const void*)&k_stage_rowid, elem_grid(c, nblk * R), 256, 0, args);
  }
  DevBuf<int> cnt((size_t)3 * nblk);
  int* cs = cnt.ptr;
  int* cr = cnt.ptr + nblk;
  int* cw = cnt.ptr + 2 * nblk;
  auto run = [&](int pass, int smax, const StageHdr* hdr, int2* segs, uint16_t* lidx, double* sv) {
    const int rl = (R + 31) / 32;
    const int32_t* rid = out.rowid.ptr;
    if (rl <= 1)
      merge_launch<1>(c, pass, R, nblk, smax, rid, rowptr, cols, vals, cs, cr, cw, hdr, segs, lidx, sv);
    else if (rl <= 2)
      merge_launch<2>(c, pass, R, nblk, smax, rid, rowptr, cols, vals, cs, cr, cw, hdr, segs, lidx, sv);
    else if (rl <= 4)
      merge_launch<4>(c, pass, R, nblk, smax, rid, rowptr, cols, vals, cs, cr, cw, hdr, segs, lidx, sv);
    else
      merge_launch<8>(c, pass, R, nblk, smax, rid, rowptr, cols, vals, cs, cr, cw, hdr, segs, lidx, sv);
  };
  run(0, 0, nullptr, nullptr, nullptr, nullptr);
  std::vector<int> h((size_t)3 * nblk);
  d2h(c, h.data(), cnt.ptr, h.size());
  sync(c);
  std::vector<StageHdr> hdr(nblk);
  int cap = 0, smax = 0, wmax = 0;
  int64_t ent = 0;
  for (int64_t b = 0; b < nblk; ++b) {
    const int ns = h[b], nr = h[nblk + b], w = h[2 * nblk + b];
    cap = std::max(cap, nr);
    smax = std::max(smax, ns);
    wmax = std::max(wmax, w);
    hdr[b] = StageHdr{ent, ns, w, nr, {0, 0, 0}};
    ent += (int64_t)w * R;
  }
  if (smax > max_segs || cap >= 0xFFFE) return false;
  smax = std::max(smax, 1);
  out.hdr.ensure(std::max<int64_t>(nblk, 1));
  out.segs.ensure(std::max<int64_t>(nblk * smax, 1));
  out.lidx.ensure(std::max<int64_t>(ent + nblk * R, 8));
  out.vals.ensure(std::max<int64_t>(ent, 1));
  h2d(c, out.hdr.ptr, hdr.data(), nblk);
  run(1, smax, out.hdr.ptr, out.segs.ptr, out.lidx.ptr, out.vals.ptr);
  sync(c);
  out.R = R;
  out.n = n;
  out.nblk = nblk;
  out.cap = cap;
  out.smax = smax;
  out.wmax = wmax;
  for (int d = 0; d < 3; ++d) {
    out.box[d] = boxed ? box[d] : 0;
    out.grid[d] = boxed ? grid[d] : 0;
  }
  return true;
}

}  // namespace bkg
