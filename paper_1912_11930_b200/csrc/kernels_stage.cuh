// kernels_stage.cuh — K1 with the operand rows and the CSR stream staged in
// shared memory by the TMA engine (cp.async.bulk + mbarrier): Q = A P
// (kernels.hpp:129-157), alpha = <<P, Q>> (kernels.hpp:59-88), last CTA:
// lambda = alpha^-1 rho_prev (kernels.hpp:231-240).
//
// Why: the register-gather K1s (kernels_k1.cuh) are bound by per-warp
// memory-level parallelism -- a warp has about one row step of gathers in
// flight, and ncu shows long-scoreboard stalls at ~70% with DRAM and L1 both
// half idle (profiles/ncu_c5_r01.md) -- and every nonzero pulls a whole
// operand row segment through L2 -> L1 (5 of 7 per row on a 7-point stencil).
// Here the rows are cut into blocks (StageCsr, common.cuh / stage.cu: boxes of
// grid points on stencil matrices, R consecutive rows otherwise); a block's
// operand needs -- the distinct columns of its rows plus its own rows, merged
// into contiguous row runs ("segments") -- are copied global -> shared by one
// bulk copy per segment, plus one copy each for the block's slot-major values,
// staged-row indices and row ids.  The bytes in flight per SM are bounded by
// the shared-memory ring (NS stages), not by registers, and an operand row is
// fetched once per block that needs it (a 4x4x4 box: 2.5 rows per own row).
//
// CTA = 8 warps, persistent over the blocks (block j of the launch goes to
// CTA j % grid).  The last warp to finish block i (a shared-memory counter
// per stage) lane-parallel issues the copies of block i + NS into the stage
// it freed, so there is no CTA-wide barrier per block and the warps drift up
// to NS - 1 blocks apart.  Every warp prefetches the header and segment list
// of block i + NS at the top of block i (fixed-stride arrays: no dependent
// address), so the refill is issue-only -- fetched inside the refill, its two
// dependent global loads put ~2 us on the slowest warp of every block and
// paced the whole ring (ncu: half of all samples in the mbarrier wait).
// Every warp computes RPW x W tiles of the staged block, BKG_STAGE_NT tiles
// interleaved: lane (rr, cl) owns row rr and the columns {2cl, 2cl + 1, W/2 +
// 2cl, W/2 + 2cl + 1} of its warp's column slice, so each operand row read is
// two conflict-free LDS.128 per lane (8 lanes = one 128-byte row segment).
// Epilogue per tile as k1_wide: Q store, Gram P^T Q by FP64 DMMA (P fragments
// straight from the staged own rows, Q through a per-warp scratch),
// deterministic grid reduction, lambda solve in the last CTA.
#pragma once

#include <type_traits>

#include "kernels_k1.cuh"

namespace bkg {

// ------------------------------------------------------------ PTX ------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing `bytes` on `bar` (TMA, UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kStageSegLanes = 2;   // segments per lane of the issuing warp (<= 64 / block)
constexpr int kStageThreads = 512;  // 16 warps share one ring: 4 per scheduler hide the
                                    // shared-memory latency of the slot loop (ncu at 8
                                    // warps: 0.34 eligible warps per scheduler)

// Tiles interleaved per warp in the row loop (registers: 128 at 512 threads).
#ifndef BKG_STAGE_NT
#define BKG_STAGE_NT 1
#endif

// Row slots of a block are a multiple of R0: the 16 warps cover (16 / QW) row
// tiles of RPW rows x QW column slices per pass.
template <int K, int P, int W>
struct StageLayout {
  using L = WideLayout<K, P, W, 4>;
  static constexpr int NW = kStageThreads / 32;
  static constexpr int R0 = (NW / L::QW) * L::RPW;
  static_assert(R0 % 8 == 0, "staged index copies need 16-byte sizes");
};

// Bytes of one stage: cap staged rows of K doubles, wmax x R values,
// (wmax + 1) x R uint16 indices and R int32 row ids, 128-byte aligned.
__host__ __device__ __forceinline__ int stage_bytes(int K, int R, int cap, int wmax) {
  const int b = cap * K * 8 + wmax * R * 8 + (wmax + 1) * R * 2 + R * 4;
  return (b + 127) / 128 * 128;
}

__device__ __forceinline__ int4 ldg_nc_int4(const void* p) {
  int4 v;
  asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ int2 ldg_nc_int2(const void* p) {
  int2 v;
  asm volatile("ld.global.nc.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

template <int K, int P, int W, bool GLOBAL>
__global__ void __launch_bounds__(kStageThreads, 1) k1_stage(IterArgs a) {
  using L = WideLayout<K, P, W, 4>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  constexpr int LPR = L::LPR, RPW = L::RPW, SS = L::SS, QW = L::QW;
  constexpr int R0 = StageLayout<K, P, W>::R0;
  constexpr int NW = kStageThreads / 32;
  if (stopped(a.ctrl)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rr = lane / LPR, cl = lane % LPR;
  const int cs = warp % QW, wt = warp / QW;
  const int c0 = cs * W + 2 * cl, c1 = c0 + W / 2;
  const int NS = a.stg_nstage, cap = a.stg_cap, wmax = a.stg_wmax, R = a.stg_R;
  const int smax = a.stg_smax;
  const int tpw = R / R0;  // row tiles per warp per block
  const int sbytes = stage_bytes(K, R, cap, wmax);
  extern __shared__ __align__(128) unsigned char smraw[];
  double* scr = reinterpret_cast<double*>(smraw + (size_t)NS * sbytes) + warp * RPW * SS;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + (size_t)NS * sbytes + NW * RPW * SS * 8);
  int* fin = reinterpret_cast<int*>(bar + NS);  // per stage: warps done with it
  int* sw = fin + NS;                           // per stage: slots of the staged block
  const size_t off_vals = (size_t)cap * K * 8;
  const size_t off_lidx = off_vals + (size_t)wmax * R * 8;
  const size_t off_rid = off_lidx + (size_t)(wmax + 1) * R * 2;

  // blocks of this launch: all stg_cnt in order, or stg_map[0 .. stg_cnt)
  const int64_t ntot = a.stg_cnt;
  const int64_t nmine =
      ntot > (int64_t)blockIdx.x ? (ntot - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto block_of = [&](int64_t i) {  // block of this CTA's i-th step
    const int64_t j = blockIdx.x + i * gridDim.x;
    return a.stg_map ? __ldg(a.stg_map + j) : j;
  };

  // ---- header + segment list of the next block to issue (every warp) ----
  int64_t m_b = 0;
  int4 m_h = make_int4(0, 0, 0, 0);  // ebeg (lo, hi), nseg, w
  int m_staged = 0;
  int2 m_seg[kStageSegLanes];
  auto fetch_meta = [&](int64_t b) {
    m_b = b;
    const StageHdr* h = a.stg_hdr + b;
    m_h = ldg_nc_int4(h);
    m_staged = ldg_nc_int2(reinterpret_cast<const int*>(h) + 4).x;
#pragma unroll
    for (int t = 0; t < kStageSegLanes; ++t) {
      const int si = lane + 32 * t;
      m_seg[t] = si < smax ? ldg_nc_int2(a.stg_segs + b * smax + si) : make_int2(0, 0);
    }
  };
  auto issue = [&](int s) {
    // staged-row offsets of the segments: exclusive prefix of their lengths
    int base = 0;
    int off[kStageSegLanes];
#pragma unroll
    for (int t = 0; t < kStageSegLanes; ++t) {
      int v = m_seg[t].y;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += u;
      }
      off[t] = base + v - m_seg[t].y;
      base += __shfl_sync(kFull, v, 31);
    }
    const int w = m_h.w;
    const int64_t ebeg = ((int64_t)m_h.y << 32) | (uint32_t)m_h.x;
    const bool rows_on = !(a.stg_debug & 2);
    const uint32_t bytes = (rows_on ? (uint32_t)m_staged * K * 8 : 0u) + (uint32_t)w * R * 8 +
                           (uint32_t)(w + 1) * R * 2 + (uint32_t)R * 4;
    uint64_t* b = bar + s;
    unsigned char* st = smraw + (size_t)s * sbytes;
    if (lane == 0) {
      sw[s] = w;
      mbar_expect_tx(b, bytes);
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < kStageSegLanes; ++t)
      if (m_seg[t].y > 0 && rows_on)
        bulk_g2s(st + (size_t)off[t] * K * 8, a.P + (int64_t)m_seg[t].x * K,
                 (uint32_t)m_seg[t].y * K * 8, b);
    if (lane == 0 && w > 0) bulk_g2s(st + off_vals, a.stg_vals + ebeg, (uint32_t)w * R * 8, b);
    if (lane == 1)
      bulk_g2s(st + off_lidx, a.stg_lidx + ebeg + m_b * R, (uint32_t)(w + 1) * R * 2, b);
    if (lane == 2) bulk_g2s(st + off_rid, a.stg_rowid + m_b * R, (uint32_t)R * 4, b);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bar + s, 1);
      fin[s] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 0) {
    for (int64_t i = 0; i < NS && i < nmine; ++i) {
      fetch_meta(block_of(i));
      issue((int)i);
    }
  }
  int64_t bnext = NS < nmine ? block_of(NS) : 0;  // block of step i + NS
  __syncthreads();

  double acc[L::NACC];
#pragma unroll
  for (int e = 0; e < L::NACC; ++e) acc[e] = 0.0;

#pragma unroll 1
  for (int64_t i = 0; i < nmine; ++i) {
    const int s = (int)(i % NS);
    const bool refill = i + NS < nmine;
    if (refill) fetch_meta(bnext);
    if (i + NS + 1 < nmine) bnext = block_of(i + NS + 1);
    mbar_wait(bar + s, (uint32_t)((i / NS) & 1));
    const int w = sw[s];
    const unsigned char* st = smraw + (size_t)s * sbytes;
    const double* rows = reinterpret_cast<const double*>(st);
    const double* vals = reinterpret_cast<const double*>(st + off_vals);
    const uint16_t* lidx = reinterpret_cast<const uint16_t*>(st + off_lidx);
    const int32_t* rid = reinterpret_cast<const int32_t*>(st + off_rid);

    // NT row tiles of this warp at a time: slot loop, Q store, Gram
    auto tiles = [&](auto ntc, int tt0) {
      constexpr int NT = decltype(ntc)::value;
      constexpr int U = 4;  // the builder pads every block's slots to a multiple of 4
      int rl[NT];
      double q[NT][4];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        rl[t] = (wt * tpw + tt0 + t) * RPW + rr;
        q[t][0] = q[t][1] = q[t][2] = q[t][3] = 0.0;
      }
#pragma unroll 1
      for (int u0 = 0; u0 < w; u0 += U) {
        int li[NT][U];
        double v[NT][U];
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            li[t][u] = lidx[(u0 + u) * R + rl[t]];
            v[t][u] = vals[(u0 + u) * R + rl[t]];
          }
        double2 x[NT][U][2];
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const double* xr = rows + li[t][u] * K;
            x[t][u][0] = *reinterpret_cast<const double2*>(xr + c0);
            x[t][u][1] = *reinterpret_cast<const double2*>(xr + c1);
          }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            q[t][0] = fma(v[t][u], x[t][u][0].x, q[t][0]);
            q[t][1] = fma(v[t][u], x[t][u][0].y, q[t][1]);
            q[t][2] = fma(v[t][u], x[t][u][1].x, q[t][2]);
            q[t][3] = fma(v[t][u], x[t][u][1].y, q[t][3]);
          }
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int row = rid[rl[t]];
        if (row >= 0) {
          double* qd = a.Q + (int64_t)row * K;
          *reinterpret_cast<double2*>(qd + c0) = make_double2(q[t][0], q[t][1]);
          *reinterpret_cast<double2*>(qd + c1) = make_double2(q[t][2], q[t][3]);
        }
        // Gram P^T Q over the tile: Q via the scratch (logical column c at
        // c < W/2 ? c : c + 2), P straight from the staged own rows
        *reinterpret_cast<double2*>(scr + rr * SS + 2 * cl) = make_double2(q[t][0], q[t][1]);
        *reinterpret_cast<double2*>(scr + rr * SS + W / 2 + 2 + 2 * cl) =
            make_double2(q[t][2], q[t][3]);
        __syncwarp();
        const int tile0 = rl[t] - rr;  // first row slot of the tile
#pragma unroll
        for (int cc = 0; cc < RPW / 4; ++cc) {
          const int tr = 4 * cc + (lane & 3);
          const int oi = lidx[w * R + tile0 + tr];  // staged index of the row itself
          const double* pr = rows + oi * K + cs * W + (lane >> 2);
          const double* qr = scr + tr * SS;
#pragma unroll
          for (int pi = 0; pi < L::NPAIR; ++pi) {
            int at, bt;
            wide_pair<K, P, W, 4>(pi, at, bt);
            const double av = pr[at * 8];  // an empty row slot has Q = 0
            const int qc = bt * 8 + (lane >> 2);  // logical column -> scratch column
            const double bv = qr[qc < W / 2 ? qc : qc + 2];
            double d[2] = {acc[2 * pi], acc[2 * pi + 1]};
            dmma(d, av, bv);
            acc[2 * pi] = d[0];
            acc[2 * pi + 1] = d[1];
          }
        }
        __syncwarp();
      }
    };
    int tt = (a.stg_debug & 1) ? tpw : 0;
    if constexpr (BKG_STAGE_NT > 1) {
#pragma unroll 1
      for (; tt + BKG_STAGE_NT <= tpw; tt += BKG_STAGE_NT)
        tiles(std::integral_constant<int, BKG_STAGE_NT>{}, tt);
    }
#pragma unroll 1
    for (; tt < tpw; ++tt) tiles(std::integral_constant<int, 1>{}, tt);

    // The last warp done with stage s refills it with block i + NS: no
    // CTA-wide barrier per block, warps drift up to NS - 1 blocks apart.
    __threadfence_block();
    int last = 0;
    if (lane == 0) last = atomicAdd(fin + s, 1) == NW - 1;
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      if (lane == 0) fin[s] = 0;
      if (refill) issue(s);
    }
  }
  __syncthreads();  // the stages are reused as the reduction buffer
  double* red = reinterpret_cast<double*>(smraw);
  if (!grid_reduce<L::TPR, L::NACC, kStageThreads>(acc, red, a.partials, a.gpart,
                                                   a.ctrl->tickets, a.group))
    return;
  double* alpha = red + L::RED;
  double* ws = alpha + 3 * S::CS;
  gather_gram_wide<K, P, W, 4, GLOBAL>(red, alpha);
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kStageThreads)
      a.red1[i] = (a.dist_acc ? a.red1[i] : 0.0) + alpha[i];
    return;
  }
  const int bad = fast_bsolve<P>(S::NB, P, alpha, a.coef + S::CS, a.coef, ws);  // lambda
  if (bad >= 0) record_breakdown(a.ctrl, bad, 1);
}

// Dynamic shared memory of k1_stage with NS stages of R row slots.
template <int K, int P, int W, bool GLOBAL>
int k1_stage_smem(int R, int cap, int wmax, int ns) {
  using L = WideLayout<K, P, W, 4>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  const int main = ns * stage_bytes(K, R, cap, wmax) + (kStageThreads / 32) * L::RPW * L::SS * 8 +
                   ns * 8 + ns * 8;
  const int epi =
      (int)sizeof(double) * (L::RED + 3 * S::CS + bsolve_ws_doubles(P, kStageThreads) + K);
  return main > epi ? main : epi;
}

}  // namespace bkg
