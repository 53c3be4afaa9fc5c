// stage.cu — the staged-block copy of a CSR matrix for k1_stage
// (kernels_stage.cuh), built on device once per matrix and block height R.
//
// For block b = rows [b R, b R + R) the staged set is the sorted union of the
// block's column indices and its own rows (the Gram's P rows).  Runs of
// consecutive columns become segments {first row, rows}; each entry (slot u
// of row i, CSR order) stores the index of its column inside the staged set
// (uint16) and its value, slot-major: entry (u, i) at bent[b] + u R + i,
// padding kNoSlot / 0.0 up to the block's longest row.
//
// One warp per block merges the R sorted rows (CSR columns ascend,
// sparse_matrix.hpp:99-105) and the own-row range: each step takes the
// warp-wide minimum head -- the next distinct column -- and every row whose
// head equals it records the staged index and advances.  Pass 0 counts
// (segments, staged rows, longest row); the host scans the counts; pass 1
// writes.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "bkg.h"
#include "common.cuh"
#include "host.cuh"

namespace bkg {

namespace {

constexpr uint16_t kNoSlotB = 0xFFFF;

template <int RL>  // rows per lane: R <= 32 * RL
__global__ void k_stage_merge(int pass, int64_t n, int R, int64_t nblk,
                              const int64_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                              const double* __restrict__ vals, int* __restrict__ cnt_seg,
                              int* __restrict__ cnt_rows, int* __restrict__ cnt_w,
                              const int64_t* __restrict__ bseg, const int64_t* __restrict__ bent,
                              int2* __restrict__ segs, uint16_t* __restrict__ lidx,
                              double* __restrict__ svals, int32_t* __restrict__ own) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = wid; b < nblk; b += nw) {
    const int64_t r0 = b * R, r1 = min(r0 + R, n);
    int64_t e[RL], es[RL], ee[RL];
    int head[RL];
    int w = 0;
#pragma unroll
    for (int t = 0; t < RL; ++t) {
      const int rl = lane + 32 * t;
      const int64_t row = r0 + rl;
      e[t] = es[t] = ee[t] = 0;
      head[t] = INT_MAX;
      if (rl < R && row < r1) {
        e[t] = es[t] = rowptr[row];
        ee[t] = rowptr[row + 1];
        if (e[t] < ee[t]) head[t] = cols[e[t]];
        w = max(w, (int)(ee[t] - es[t]));
      }
    }
    // own rows [r0, r1) as one more sorted list (lane 0)
    int ohead = lane == 0 ? (int)r0 : INT_MAX;
    const int oend = (int)r1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
    int cnt = 0, nseg = 0, last = 0, seg_first = 0, seg_len = 0;
    const int64_t sbase = pass ? bseg[b] : 0;
    const int64_t ebase = pass ? bent[b] : 0;
    while (true) {
      int h = ohead;
#pragma unroll
      for (int t = 0; t < RL; ++t) h = min(h, head[t]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) h = min(h, __shfl_xor_sync(0xffffffffu, h, o));
      if (h == INT_MAX) break;
      if (cnt > 0 && h == last + 1) {
        ++seg_len;
      } else {
        if (pass && lane == 0 && cnt > 0) segs[sbase + nseg - 1] = make_int2(seg_first, seg_len);
        ++nseg;
        seg_first = h;
        seg_len = 1;
      }
#pragma unroll
      for (int t = 0; t < RL; ++t) {
        if (head[t] == h) {
          if (pass) {
            const int64_t idx = ebase + (e[t] - es[t]) * R + lane + 32 * t;
            lidx[idx] = (uint16_t)min(cnt, 0xFFFE);
            svals[idx] = vals[e[t]];
          }
          ++e[t];
          head[t] = e[t] < ee[t] ? cols[e[t]] : INT_MAX;
        }
      }
      if (ohead == h) {
        if (pass && h == (int)r0) own[b] = cnt;
        ++ohead;
        if (ohead >= oend) ohead = INT_MAX;
      }
      last = h;
      ++cnt;
    }
    if (pass) {
      if (lane == 0 && cnt > 0) segs[sbase + nseg - 1] = make_int2(seg_first, seg_len);
      // padding slots: rows shorter than w and rows past n
#pragma unroll
      for (int t = 0; t < RL; ++t) {
        const int rl = lane + 32 * t;
        if (rl >= R) continue;
        for (int64_t u = ee[t] - es[t]; u < w; ++u) {
          const int64_t idx = ebase + u * R + rl;
          lidx[idx] = kNoSlotB;
          svals[idx] = 0.0;
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
void merge_launch(bkg_ctx* c, int pass, int64_t n, int R, int64_t nblk, const int64_t* rowptr,
                  const int32_t* cols, const double* vals, int* cs, int* cr, int* cw,
                  const int64_t* bseg, const int64_t* bent, int2* segs, uint16_t* lidx,
                  double* svals, int32_t* own) {
  const int blocks = (int)std::min<int64_t>((nblk * 32 + 255) / 256, (int64_t)c->sm_count * 32);
  void* args[] = {&pass, &n, &R, &nblk, &rowptr, &cols, &vals, &cs, &cr, &cw,
                  &bseg, &bent, &segs, &lidx, &svals, &own};
  launch(c, (const void*)&k_stage_merge<RL>, std::max(1, blocks), 256, 0, args);
}

}  // namespace

// Build (or rebuild) `out` for block height R.  Returns false -- and leaves
// out.R = 0 -- when a block needs more than `max_segs` segments or 0xFFFE
// staged rows (the kernel's limits); the caller then keeps the register-gather
// K1.
bool stage_build(bkg_ctx* c, int64_t n, const int64_t* rowptr, const int32_t* cols,
                 const double* vals, int R, int max_segs, StageCsr& out) {
  out.R = 0;
  const int64_t nblk = (n + R - 1) / R;
  DevBuf<int> cnt((size_t)3 * nblk);
  int* cs = cnt.ptr;
  int* cr = cnt.ptr + nblk;
  int* cw = cnt.ptr + 2 * nblk;
  auto run = [&](int pass, const int64_t* bseg, const int64_t* bent, int2* segs, uint16_t* lidx,
                 double* sv, int32_t* own) {
    const int rl = (R + 31) / 32;
    if (rl <= 1)
      merge_launch<1>(c, pass, n, R, nblk, rowptr, cols, vals, cs, cr, cw, bseg, bent, segs, lidx,
                      sv, own);
    else if (rl <= 2)
      merge_launch<2>(c, pass, n, R, nblk, rowptr, cols, vals, cs, cr, cw, bseg, bent, segs, lidx,
                      sv, own);
    else if (rl <= 4)
      merge_launch<4>(c, pass, n, R, nblk, rowptr, cols, vals, cs, cr, cw, bseg, bent, segs, lidx,
                      sv, own);
    else
      merge_launch<8>(c, pass, n, R, nblk, rowptr, cols, vals, cs, cr, cw, bseg, bent, segs, lidx,
                      sv, own);
  };
  BKG_REQUIRE(R <= 256 && R % 8 == 0, BKG_INTERNAL, "stage_build: bad block height");
  run(0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  std::vector<int> h((size_t)3 * nblk);
  d2h(c, h.data(), cnt.ptr, h.size());
  sync(c);
  std::vector<int64_t> bseg(nblk + 1), bent(nblk + 1);
  int cap = 0, smax = 0, wmax = 0;
  bseg[0] = bent[0] = 0;
  for (int64_t b = 0; b < nblk; ++b) {
    const int ns = h[b], nr = h[nblk + b], w = h[2 * nblk + b];
    cap = std::max(cap, nr);
    smax = std::max(smax, ns);
    wmax = std::max(wmax, w);
    bseg[b + 1] = bseg[b] + ns;
    bent[b + 1] = bent[b] + (int64_t)w * R;
  }
  if (smax > max_segs || cap >= 0xFFFE) return false;
  out.bseg.ensure(nblk + 1);
  out.bent.ensure(nblk + 1);
  out.segs.ensure(std::max<int64_t>(bseg[nblk], 1));
  out.lidx.ensure(std::max<int64_t>(bent[nblk], 8));
  out.vals.ensure(std::max<int64_t>(bent[nblk], 1));
  out.own.ensure(nblk);
  h2d(c, out.bseg.ptr, bseg.data(), nblk + 1);
  h2d(c, out.bent.ptr, bent.data(), nblk + 1);
  run(1, out.bseg.ptr, out.bent.ptr, out.segs.ptr, out.lidx.ptr, out.vals.ptr, out.own.ptr);
  sync(c);
  out.R = R;
  out.n = n;
  out.nblk = nblk;
  out.cap = cap;
  out.smax = smax;
  out.wmax = wmax;
  return true;
}

}  // namespace bkg
