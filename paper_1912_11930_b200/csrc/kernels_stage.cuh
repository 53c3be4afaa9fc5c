// kernels_stage.cuh — K1 with the operand rows and the CSR stream staged in
// shared memory by the TMA engine (cp.async.bulk + mbarrier): Q = A P
// (kernels.hpp:129-157), alpha = <<P, Q>> (kernels.hpp:59-88), last CTA:
// lambda = alpha^-1 rho_prev (kernels.hpp:231-240).
//
// Why: the register-gather K1s (kernels_k1.cuh) are bound by per-warp
// memory-level parallelism -- a warp has about one row step of gathers in
// flight, and ncu shows long-scoreboard stalls at ~70% with DRAM and L1 both
// half idle (profiles/ncu_c5_r01.md).  Here the rows are cut into blocks of R
// consecutive rows; a block's operand needs -- the distinct columns of its
// rows plus its own rows, merged into contiguous row runs ("segments", built
// once per matrix, StageCsr in common.cuh) -- are copied global -> shared by
// one bulk copy per segment, plus one copy each for the block's slot-major
// values and staged-row indices.  A stencil block of R rows needs a handful
// of segments (7-point: own rows +- 1, y +- 1, z +- 1 = 5; 27-point: 9), so
// an R-row block costs ~5-9 bulk copies and the bytes in flight per SM are
// bounded by the shared-memory ring (NS stages), not by registers.  General
// CSR works the same way (worst case one segment per distinct column).
//
// CTA = 8 warps, persistent over the blocks (block j of the launch goes to
// CTA j % grid).  The last warp to finish block i (a shared-memory counter
// per stage) lane-parallel issues the copies of block i + NS into the stage
// it freed, so there is no CTA-wide barrier per block and the warps drift up
// to NS - 1 blocks apart.  Every warp
// computes RPW x W tiles of the staged block: lane (rr, cl) owns row rr and
// the columns {2cl, 2cl + 1, W/2 + 2cl, W/2 + 2cl + 1} of its warp's column
// slice, so each operand row read is two conflict-free LDS.128 per lane
// (8 lanes = one 128-byte row segment).  Epilogue per tile as k1_wide: Q
// store, Gram P^T Q by FP64 DMMA (P fragments straight from the staged own
// rows, Q through a per-warp scratch), deterministic grid reduction, lambda
// solve in the last CTA.
#pragma once

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

constexpr uint16_t kNoSlot = 0xFFFF;  // padding slot of a staged block
constexpr int kStageSegLanes = 2;     // segments per lane of the issuing warp (<= 64 / block)

// Block rows of k1_stage for (K, W, TPW): the 8 warps cover (8 / QW) x TPW
// tiles of RPW rows.
template <int K, int P, int W, int TPW>
struct StageLayout {
  using L = WideLayout<K, P, W, 4>;
  static constexpr int R = (kThreads / 32 / L::QW) * L::RPW * TPW;
  static_assert(R % 8 == 0, "staged-row index copies need 16-byte sizes");
};

// Bytes of one stage: cap staged rows of K doubles, wmax x R values and
// wmax x R uint16 indices, 128-byte aligned.
__host__ __device__ __forceinline__ int stage_bytes(int K, int R, int cap, int wmax) {
  const int b = cap * K * 8 + wmax * R * 8 + ((wmax * R * 2 + 15) / 16) * 16;
  return (b + 127) / 128 * 128;
}

template <int K, int P, int W, int TPW, bool GLOBAL>
__global__ void __launch_bounds__(kThreads, 1) k1_stage(IterArgs a) {
  using L = WideLayout<K, P, W, 4>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  constexpr int LPR = L::LPR, RPW = L::RPW, SS = L::SS, QW = L::QW;
  constexpr int R = StageLayout<K, P, W, TPW>::R;
  if (stopped(a.ctrl)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rr = lane / LPR, cl = lane % LPR;
  const int cs = warp % QW, wt = warp / QW;
  const int c0 = cs * W + 2 * cl, c1 = c0 + W / 2;
  const int NS = a.stg_nstage, cap = a.stg_cap, wmax = a.stg_wmax;
  const int sbytes = stage_bytes(K, R, cap, wmax);
  extern __shared__ __align__(128) unsigned char smraw[];
  double* scr = reinterpret_cast<double*>(smraw + (size_t)NS * sbytes) + warp * RPW * SS;
  uint64_t* bar =
      reinterpret_cast<uint64_t*>(smraw + (size_t)NS * sbytes + (kThreads / 32) * RPW * SS * 8);
  int* hdr = reinterpret_cast<int*>(bar + NS);  // per stage: own, w
  int* fin = hdr + 2 * NS;                      // per stage: warps done with it
  auto rows_of = [&](int s) { return reinterpret_cast<const double*>(smraw + (size_t)s * sbytes); };
  auto vals_of = [&](int s) {
    return reinterpret_cast<const double*>(smraw + (size_t)s * sbytes + (size_t)cap * K * 8);
  };
  auto lidx_of = [&](int s) {
    return reinterpret_cast<const uint16_t*>(smraw + (size_t)s * sbytes + (size_t)cap * K * 8 +
                                             (size_t)wmax * R * 8);
  };

  // blocks of this launch: [first1, first1 + cnt1) then [first2, first2 + cnt2),
  // or stg_map[0 .. cnt1 + cnt2) (the partitioned solver's interior / boundary)
  const int64_t ntot = a.stg_cnt1 + a.stg_cnt2;
  auto block_of = [&](int64_t j) {
    if (a.stg_map) return __ldg(a.stg_map + j);
    return j < a.stg_cnt1 ? a.stg_first1 + j : a.stg_first2 + (j - a.stg_cnt1);
  };
  const int64_t nmine =
      ntot > (int64_t)blockIdx.x ? (ntot - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  // ---- issuing warp state: segment list of the next block to issue ----
  int64_t m_sbeg = 0, m_ebeg = 0;
  int m_nseg = -1, m_own = 0, m_w = 0;
  int2 m_seg[kStageSegLanes];
  auto load_meta = [&](int64_t i) {
    m_nseg = -1;
    if (i >= nmine) return;
    const int64_t b = block_of(blockIdx.x + i * gridDim.x);
    m_sbeg = __ldg(a.stg_bseg + b);
    m_nseg = (int)(__ldg(a.stg_bseg + b + 1) - m_sbeg);
    m_ebeg = __ldg(a.stg_bent + b);
    m_w = (int)((__ldg(a.stg_bent + b + 1) - m_ebeg) / R);
    m_own = __ldg(a.stg_own + b);
#pragma unroll
    for (int t = 0; t < kStageSegLanes; ++t) {
      const int si = lane + 32 * t;
      m_seg[t] = si < m_nseg ? a.stg_segs[m_sbeg + si] : make_int2(0, 0);
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
    const uint32_t bytes = (uint32_t)base * K * 8 + (uint32_t)m_w * R * 10;
    uint64_t* b = bar + s;
    unsigned char* st = smraw + (size_t)s * sbytes;
    if (lane == 0) {
      mbar_expect_tx(b, bytes);
      hdr[2 * s] = m_own;
      hdr[2 * s + 1] = m_w;
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < kStageSegLanes; ++t)
      if (m_seg[t].y > 0)
        bulk_g2s(st + (size_t)off[t] * K * 8, a.P + (int64_t)m_seg[t].x * K,
                 (uint32_t)m_seg[t].y * K * 8, b);
    if (m_w > 0) {
      if (lane == 0)
        bulk_g2s(st + (size_t)cap * K * 8, a.stg_vals + m_ebeg, (uint32_t)m_w * R * 8, b);
      if (lane == 1)
        bulk_g2s(st + (size_t)cap * K * 8 + (size_t)wmax * R * 8, a.stg_lidx + m_ebeg,
                 (uint32_t)m_w * R * 2, b);
    }
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
      load_meta(i);
      issue((int)i);
    }
  }
  __syncthreads();

  double acc[L::NACC];
#pragma unroll
  for (int e = 0; e < L::NACC; ++e) acc[e] = 0.0;

#pragma unroll 1
  for (int64_t i = 0; i < nmine; ++i) {
    const int s = (int)(i % NS);
    mbar_wait(bar + s, (uint32_t)((i / NS) & 1));
    const int own = hdr[2 * s], w = hdr[2 * s + 1];
    const double* rows = rows_of(s);
    const double* vals = vals_of(s);
    const uint16_t* lidx = lidx_of(s);
    const int64_t r0 = block_of(blockIdx.x + i * gridDim.x) * R;
#pragma unroll 1
    for (int tt = 0; tt < TPW; ++tt) {
      const int tile = wt * TPW + tt;
      const int rl = tile * RPW + rr;
      const int64_t row = r0 + rl;
      double q[4] = {0.0, 0.0, 0.0, 0.0};
      constexpr int U = 4;
#pragma unroll 1
      for (int u0 = 0; u0 < w; u0 += U) {
        int li[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool in = u0 + u < w;
          li[u] = in ? lidx[(u0 + u) * R + rl] : kNoSlot;
          v[u] = in ? vals[(u0 + u) * R + rl] : 0.0;
        }
        double2 x[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (li[u] != kNoSlot) {
            const double* xr = rows + li[u] * K;
            x[u][0] = *reinterpret_cast<const double2*>(xr + c0);
            x[u][1] = *reinterpret_cast<const double2*>(xr + c1);
          } else {
            x[u][0] = x[u][1] = make_double2(0.0, 0.0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          q[0] = fma(v[u], x[u][0].x, q[0]);
          q[1] = fma(v[u], x[u][0].y, q[1]);
          q[2] = fma(v[u], x[u][1].x, q[2]);
          q[3] = fma(v[u], x[u][1].y, q[3]);
        }
      }
      if (row < a.n) {
        *reinterpret_cast<double2*>(a.Q + row * K + c0) = make_double2(q[0], q[1]);
        *reinterpret_cast<double2*>(a.Q + row * K + c1) = make_double2(q[2], q[3]);
      }
      // Gram P^T Q over the tile: Q via the scratch (logical column c at
      // c < W/2 ? c : c + 2), P straight from the staged own rows
      *reinterpret_cast<double2*>(scr + rr * SS + 2 * cl) = make_double2(q[0], q[1]);
      *reinterpret_cast<double2*>(scr + rr * SS + W / 2 + 2 + 2 * cl) = make_double2(q[2], q[3]);
      __syncwarp();
#pragma unroll
      for (int cc = 0; cc < RPW / 4; ++cc) {
        const int tr = 4 * cc + (lane & 3);
        const int64_t prow = r0 + tile * RPW + tr;
        const double* pr = rows + (own + tile * RPW + tr) * K + cs * W + (lane >> 2);
        const double* qr = scr + tr * SS;
#pragma unroll
        for (int pi = 0; pi < L::NPAIR; ++pi) {
          int at, bt;
          wide_pair<K, P, W, 4>(pi, at, bt);
          const double av = prow < a.n ? pr[at * 8] : 0.0;
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
    // The last warp done with stage s refills it with block i + NS: no
    // CTA-wide barrier per block, warps drift up to NS - 1 blocks apart.
    __threadfence_block();
    int last = 0;
    if (lane == 0) last = atomicAdd(fin + s, 1) == kThreads / 32 - 1;
    last = __shfl_sync(kFull, last, 0);
    if (last) {
      if (lane == 0) fin[s] = 0;
      if (i + NS < nmine) {
        load_meta(i + NS);
        issue(s);
      }
    }
  }
  __syncthreads();  // the stages are reused as the reduction buffer
  double* red = reinterpret_cast<double*>(smraw);
  if (!grid_reduce<L::TPR, L::NACC>(acc, red, a.partials, a.gpart, a.ctrl->tickets, a.group))
    return;
  double* alpha = red + L::RED;
  double* ws = alpha + 3 * S::CS;
  gather_gram_wide<K, P, W, 4, GLOBAL>(red, alpha);
  __syncthreads();
  if (a.dist) {
    for (int i = threadIdx.x; i < S::CS; i += kThreads)
      a.red1[i] = (a.dist_acc ? a.red1[i] : 0.0) + alpha[i];
    return;
  }
  const int bad = cta_bsolve<P>(S::NB, P, alpha, a.coef + S::CS, a.coef, ws);  // lambda
  if (bad >= 0) record_breakdown(a.ctrl, bad, 1);
}

// Dynamic shared memory of k1_stage with NS stages.
template <int K, int P, int W, int TPW, bool GLOBAL>
int k1_stage_smem(int cap, int wmax, int ns) {
  using L = WideLayout<K, P, W, 4>;
  using S = FastSmem<K, P, 1, GLOBAL>;
  constexpr int R = StageLayout<K, P, W, TPW>::R;
  const int main = ns * stage_bytes(K, R, cap, wmax) + (kThreads / 32) * L::RPW * L::SS * 8 +
                   ns * 8 + ns * 12;
  const int epi = (int)sizeof(double) * (L::RED + 3 * S::CS + bsolve_ws_doubles(P, kThreads) + K);
  return main > epi ? main : epi;
}

}  // namespace bkg
