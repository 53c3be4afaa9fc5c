// kernels_resident.cuh — latency path for small systems: the whole Block-CG
// loop (solver.hpp:157-201, M = I) as ONE persistent cooperative kernel.
//
// For systems like BASELINE config C1 (2D Poisson 128^2, k = 8: one block
// vector = 1 MB) the three-kernel iteration is pure latency: 3 launches, 3
// last-CTA reduction tails and 5 passes over L2-resident vectors cost ~42 us
// per iteration for ~2 MB of work.  Here every CTA owns RPT x RPC consecutive
// rows and keeps their X, R, P in registers for the whole solve; only P goes
// through global memory (the SpMM gathers neighbours' rows from L2).  One
// iteration is
//   A  Q = A P (kernels.hpp:129-157), per-CTA partials of alpha = <<P, Q>>
//      (kernels.hpp:59-88) and of rho_prev = <<P, R>> (from the previous C)
//      | grid barrier | every CTA sums the partials of all CTAs in the same
//      fixed order and solves lambda = alpha^-1 rho_prev itself
//      (kernels.hpp:231-240): no broadcast, identical bits everywhere
//   B  R -= Q lambda (kernels.hpp:94-125), partials of rho = <<R, R>> and
//      ||R_s||^2 | grid barrier | totals, beta = rho_prev^-1 rho, history and
//      stop test (solver.hpp:193-200), X += P lambda
//   C  P = R + P beta, P to global, partials of rho_prev' | grid barrier
// i.e. three grid barriers and no kernel boundary per iteration.  The grid
// barrier is a monotonic counter in global memory (release add, acquire
// poll); the launch is cooperative so all CTAs are co-resident.  Reductions
// are deterministic (fixed CTA order), so runs are bit-reproducible and the
// result differs from the three-kernel fast path only by summation order
// (same parity bars).
#pragma once

#include "kernels_fast.cuh"

namespace bkg {

struct ResidentArgs {
  IterArgs it;               // n, CSR, X, R, P, coef, limits, hist, ctrl
  double* pbuf1;             // G x EB1 partials [alpha | rho_prev']
  double* pbuf2;             // G x EB2 partials [rho | ||R_s||^2]
  unsigned long long* bar;   // grid barrier counter, zero at launch
  int max_steps;             // iterations per launch (history ring bound)
  long long* prof;           // tuning only (BKG_RESIDENT_PROF): CTA 0's cycles per phase
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// All CTAs of the (co-resident) grid: arrive and wait.  epoch: arrivals
// expected so far (per-thread copy, uniform).
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long& epoch) {
  epoch += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1ULL);
    while (ld_acquire_u64(bar) < epoch) {
    }
    __threadfence();
  }
  __syncthreads();
}

// Per-CTA sum of per-thread accumulators over the threads sharing
// pos = tid % TPR, fixed order: red[pos * NACC + e].  Every warp deposits its
// (shuffle-reduced) partials side by side and E threads then add the 8 warps'
// values in warp order -- the same sum as eight serial rounds of one warp
// each, in two barriers instead of nine (the serial form was 13% of a C1
// iteration).  part: (kThreads / 32) * TPR * NACC doubles of shared memory.
template <int TPR, int NACC>
__device__ __forceinline__ void cta_reduce(double (&acc)[NACC], double* red, double* part) {
  constexpr int E = TPR * NACC;
  constexpr int NW = kThreads / 32;
  static_assert(TPR <= 32, "every warp holds every position");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pos = tid % TPR;
  if constexpr (TPR < 32) {
#pragma unroll
    for (int off = TPR; off < 32; off <<= 1)
#pragma unroll
      for (int e = 0; e < NACC; ++e) acc[e] += __shfl_xor_sync(kFull, acc[e], off);
  }
  const bool rep = (TPR >= 32) || (lane < TPR);
  if (rep) {
#pragma unroll
    for (int e = 0; e < NACC; ++e) part[(size_t)warp * E + pos * NACC + e] = acc[e];
  }
  __syncthreads();
  for (int i = tid; i < E; i += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += part[(size_t)w * E + i];
    red[i] = s;
  }
  __syncthreads();
}

// tot[e] = sum over all CTAs c (ascending) of pbuf[c * EB + e], computed by
// every CTA identically: kThreads / EB partial ranges of CTAs per entry, then
// a fixed-order sum of the ranges.  tmp: max(EB, kThreads) doubles.
template <int EB>
__device__ __forceinline__ void grid_sum(const double* pbuf, double* tot, double* tmp) {
  constexpr int PARTS = EB >= kThreads ? 1 : kThreads / EB;
  const int G = gridDim.x;
  for (int i = threadIdx.x; i < EB * PARTS; i += kThreads) {
    const int e = i % EB, part = i / EB;
    const int c0 = (int)((long long)part * G / PARTS), c1 = (int)((long long)(part + 1) * G / PARTS);
    double s = 0.0;
    for (int c = c0; c < c1; c += 16) {  // 16 loads in flight, summed in CTA order
      double v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = c + j < c1 ? __ldcg(pbuf + (size_t)(c + j) * EB + e) : 0.0;
#pragma unroll
      for (int j = 0; j < 16; ++j) s += v[j];
    }
    tmp[i] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < EB; e += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int part = 0; part < PARTS; ++part) s += tmp[part * EB + e];
    tot[e] = s;
  }
  __syncthreads();
}

template <int CPT>
__device__ __forceinline__ void ld_cg(double (&d)[CPT], const double* p) {
  if constexpr (CPT == 2) {
    const double2 t = __ldcg(reinterpret_cast<const double2*>(p));
    d[0] = t.x;
    d[1] = t.y;
  } else {
    d[0] = __ldcg(p);
  }
}
template <int CPT>
__device__ __forceinline__ void st_cg(double* p, const double (&d)[CPT]) {
  if constexpr (CPT == 2) {
    __stcg(reinterpret_cast<double2*>(p), make_double2(d[0], d[1]));
  } else {
    __stcg(p, d[0]);
  }
}

template <int K, int P, int CPT, bool GLOBAL>
struct ResidentSmem {
  using L = Layout<K, P, CPT>;
  static constexpr int NB = GLOBAL ? 1 : K / P;
  static constexpr int CS = NB * P * P;
  static constexpr int E = L::TPR * P * CPT;  // one Gram's partial entries
  static constexpr int EB1 = 2 * E;           // [alpha | rho_prev']
  static constexpr int EB2 = E + K;           // [rho | ||R_s||^2]
  static constexpr int RED = EB1 > kThreads ? EB1 : kThreads;
  static int bytes() {
    // + the per-warp partials of cta_reduce and warp_bsolve's flag
    return (int)sizeof(double) * (2 * RED + 5 * CS + K + (kThreads / 32) * EB1 + 2);
  }
};

template <int K, int P, int CPT, bool GLOBAL, int RPT>
__global__ void __launch_bounds__(kThreads, 1) k_resident(ResidentArgs ra) {
  using L = Layout<K, P, CPT>;
  using S = ResidentSmem<K, P, CPT, GLOBAL>;
  constexpr int NG = P * CPT;
  constexpr int E = S::E, CS = S::CS;
  const IterArgs& a = ra.it;
  Ctrl* ctrl = a.ctrl;
  if (stopped(ctrl)) return;
  extern __shared__ double sm[];
  double* red = sm;            // RED
  double* tot = red + S::RED;  // RED
  double* alpha = tot + S::RED;
  double* rhop = alpha + CS;
  double* rho = rhop + CS;
  double* lam = rho + CS;
  double* beta = lam + CS;
  double* norms = beta + CS;  // K
  double* part = norms + K;  // (kThreads / 32) * EB1
  int* bad_s = reinterpret_cast<int*>(part + (kThreads / 32) * S::EB1);

  const int tid = threadIdx.x, pos = tid % L::TPR, slot = tid / L::TPR, lane = tid & 31;
  const int col0 = pos * CPT;
  const int gbase = (lane / L::GT) * L::GT;
  const int goff = (GLOBAL ? 0 : col0 / P) * P * P;
  const bool cta0 = blockIdx.x == 0;
  // phase clocks (thread 0 of CTA 0 only, when ra.prof is set)
  long long pc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long t_last = clock64();
  auto tick = [&](int i) {
    if (ra.prof && cta0 && tid == 0) {
      const long long t = clock64();
      pc[i] += t - t_last;
      t_last = t;
    }
  };

  int64_t row[RPT], beg[RPT], end[RPT];
  double x[RPT][CPT], r[RPT][CPT], p[RPT][CPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    row[u] = ((int64_t)blockIdx.x * RPT + u) * L::RPC + slot;
    beg[u] = end[u] = 0;
#pragma unroll
    for (int j = 0; j < CPT; ++j) x[u][j] = r[u][j] = p[u][j] = 0.0;
    if (row[u] < a.n) {
      beg[u] = __ldg(a.rowptr + row[u]);
      end[u] = __ldg(a.rowptr + row[u] + 1);
      ld_cg<CPT>(x[u], a.X + row[u] * K + col0);
      ld_cg<CPT>(r[u], a.R + row[u] * K + col0);
      ld_cg<CPT>(p[u], a.P + row[u] * K + col0);
    }
  }
  for (int i = tid; i < CS; i += kThreads) rhop[i] = __ldcg(a.coef + CS + i);
  uint64_t it = ctrl->iterations;
  const uint64_t max_iter = ctrl->max_iter;
  unsigned long long epoch = 0;
  bool have_rp = false;  // accp holds this CTA's partial of rho_prev' = <<P', R>>
  bool ended = false;    // converged / max_iter / breakdown inside this launch
  double accp[NG];
#pragma unroll
  for (int e = 0; e < NG; ++e) accp[e] = 0.0;
  __syncthreads();

#pragma unroll 1
  for (int step = 0; step < ra.max_steps; ++step) {
    // ---- A: Q = A P, alpha partials --------------------------------------
    double q[RPT][CPT];
    double acc[2 * NG];
#pragma unroll
    for (int e = 0; e < NG; ++e) {
      acc[e] = 0.0;
      acc[NG + e] = accp[e];
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
#pragma unroll
      for (int j = 0; j < CPT; ++j) q[u][j] = 0.0;
      constexpr int CH = 8;
#pragma unroll 1
      for (int64_t i = beg[u]; i < end[u]; i += CH) {
        double v[CH], xv[CH][CPT];
        int c[CH];
#pragma unroll
        for (int t = 0; t < CH; ++t) {
          const bool on = i + t < end[u];
          v[t] = on ? __ldg(a.vals + i + t) : 0.0;
          c[t] = on ? __ldg(a.cols + i + t) : kNoCol;
        }
#pragma unroll
        for (int t = 0; t < CH; ++t) {
          if (c[t] != kNoCol) {
            ld_cg<CPT>(xv[t], a.P + (int64_t)c[t] * K + col0);
          } else {
#pragma unroll
            for (int j = 0; j < CPT; ++j) xv[t][j] = 0.0;
          }
        }
#pragma unroll
        for (int t = 0; t < CH; ++t)
          if (c[t] != kNoCol) {
#pragma unroll
            for (int j = 0; j < CPT; ++j) q[u][j] = fma(v[t], xv[t][j], q[u][j]);
          }
      }
#pragma unroll
      for (int s = 0; s < L::GT; ++s)
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj) {
          const double ps = __shfl_sync(kFull, p[u][jj], gbase + s);
          const int aa = s * CPT + jj;
#pragma unroll
          for (int j = 0; j < CPT; ++j) acc[aa * CPT + j] = fma(ps, q[u][j], acc[aa * CPT + j]);
        }
    }
    tick(0);  // SpMM + alpha
    // acc layout per pos: [alpha NG | rho_prev' NG] -> pbuf1 as two E-blocks
    cta_reduce<L::TPR, 2 * NG>(acc, red, part);
    {
      double* mine = ra.pbuf1 + (size_t)blockIdx.x * S::EB1;
      for (int i = tid; i < S::EB1; i += kThreads) {
        const int half = i / E, e = i % E;  // red[pos * 2NG + half * NG + g]
        __stcg(mine + i, red[(e / NG) * 2 * NG + half * NG + e % NG]);
      }
    }
    tick(1);  // CTA reduce + partial store
    grid_barrier(ra.bar, epoch);
    tick(2);  // barrier
    grid_sum<S::EB1>(ra.pbuf1, tot, red);
    tick(3);  // grid sum
    gather_gram<K, P, CPT, GLOBAL, NG>(tot, 0, alpha);
    if (have_rp) gather_gram<K, P, CPT, GLOBAL, NG>(tot + E, 0, rhop);
    __syncthreads();
    int bad = warp_bsolve<P>(S::NB, alpha, rhop, lam, bad_s);  // lambda (kernels.hpp:231-240)
    tick(4);  // lambda solve
    if (bad >= 0) {  // singular alpha: X, R untouched (solver.hpp:192-195)
      if (cta0) record_breakdown(ctrl, bad, 1);
      ended = true;
      break;
    }
    __syncthreads();
    // ---- B: R -= Q lambda, rho and norm partials -----------------------
    double acc2[NG + CPT];
#pragma unroll
    for (int e = 0; e < NG + CPT; ++e) acc2[e] = 0.0;
    const double* lg = lam + goff;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
#pragma unroll
      for (int s = 0; s < L::GT; ++s)
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj) {
          const double qs = __shfl_sync(kFull, q[u][jj], gbase + s);
          const int b = s * CPT + jj;
#pragma unroll
          for (int j = 0; j < CPT; ++j) r[u][j] = fma(-qs, lg[b * P + (col0 + j) % P], r[u][j]);
        }
#pragma unroll
      for (int s = 0; s < L::GT; ++s)
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj) {
          const double zs = __shfl_sync(kFull, r[u][jj], gbase + s);
          const int aa = s * CPT + jj;
#pragma unroll
          for (int j = 0; j < CPT; ++j) acc2[aa * CPT + j] = fma(zs, r[u][j], acc2[aa * CPT + j]);
        }
#pragma unroll
      for (int j = 0; j < CPT; ++j) acc2[NG + j] = fma(r[u][j], r[u][j], acc2[NG + j]);
    }
    tick(5);  // R update + rho
    cta_reduce<L::TPR, NG + CPT>(acc2, red, part);
    {
      double* mine = ra.pbuf2 + (size_t)blockIdx.x * S::EB2;
      for (int i = tid; i < E; i += kThreads)
        __stcg(mine + i, red[(i / NG) * (NG + CPT) + i % NG]);
      for (int c = tid; c < K; c += kThreads)
        __stcg(mine + E + c, red[(c / CPT) * (NG + CPT) + NG + c % CPT]);
    }
    tick(6);
    grid_barrier(ra.bar, epoch);
    tick(7);
    grid_sum<S::EB2>(ra.pbuf2, tot, red);
    tick(8);
    gather_gram<K, P, CPT, GLOBAL, NG>(tot, 0, rho);
    for (int c = tid; c < K; c += kThreads) norms[c] = sqrt(tot[E + c]);
    __syncthreads();
    bad = warp_bsolve<P>(S::NB, rhop, rho, beta, bad_s);  // beta = rho_prev^-1 rho
    tick(9);  // beta solve
    // X += P lambda precedes the beta solve in the reference (solver.hpp:171-175)
#pragma unroll
    for (int u = 0; u < RPT; ++u)
#pragma unroll
      for (int s = 0; s < L::GT; ++s)
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj) {
          const double ps = __shfl_sync(kFull, p[u][jj], gbase + s);
          const int b = s * CPT + jj;
#pragma unroll
          for (int j = 0; j < CPT; ++j) x[u][j] = fma(ps, lg[b * P + (col0 + j) % P], x[u][j]);
        }
    if (bad >= 0) {
      if (cta0) record_breakdown(ctrl, bad, 2);
      ended = true;
      break;
    }
    // history, stop test (solver.hpp:193-200): identical in every CTA
    ++it;
    bool ok = true;
    for (int c = tid; c < K; c += kThreads) {
      const double v = norms[c];
      if (!(v <= a.limits[c])) ok = false;
      if (cta0 && a.hist) a.hist[(size_t)(it % a.hist_ring) * K + c] = v;
    }
    const int all_ok = __syncthreads_and(ok);
    const bool done = all_ok || it >= max_iter;
    if (cta0 && tid == 0) {
      ctrl->iterations = it;
      if (all_ok) ctrl->converged = 1;
      if (done) ctrl->done = 1;
    }
    if (done) {
      ended = true;
      break;
    }
    // ---- C: P = R + P beta, rho_prev' partials -------------------------
    const double* bg = beta + goff;
#pragma unroll
    for (int e = 0; e < NG; ++e) accp[e] = 0.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      double pn[CPT];
#pragma unroll
      for (int j = 0; j < CPT; ++j) pn[j] = r[u][j];
#pragma unroll
      for (int s = 0; s < L::GT; ++s)
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj) {
          const double ps = __shfl_sync(kFull, p[u][jj], gbase + s);
          const int b = s * CPT + jj;
#pragma unroll
          for (int j = 0; j < CPT; ++j) pn[j] = fma(ps, bg[b * P + (col0 + j) % P], pn[j]);
        }
#pragma unroll
      for (int j = 0; j < CPT; ++j) p[u][j] = pn[j];
      if (row[u] < a.n) st_cg<CPT>(a.P + row[u] * K + col0, pn);
#pragma unroll
      for (int s = 0; s < L::GT; ++s)
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj) {
          const double ps = __shfl_sync(kFull, pn[jj], gbase + s);
          const int aa = s * CPT + jj;
#pragma unroll
          for (int j = 0; j < CPT; ++j) accp[aa * CPT + j] = fma(ps, r[u][j], accp[aa * CPT + j]);
        }
    }
    have_rp = true;
    tick(10);  // X, stop test, P update
    grid_barrier(ra.bar, epoch);  // every P row is in L2 before the next gathers
    tick(11);
  }

  // ---- exit: state back to global for the host / the next launch --------
#pragma unroll
  for (int u = 0; u < RPT; ++u)
    if (row[u] < a.n) {
      st_cg<CPT>(a.X + row[u] * K + col0, x[u]);
      st_cg<CPT>(a.R + row[u] * K + col0, r[u]);
    }
  if (!ended && have_rp) {  // step limit: rho_prev' for the next launch's first A
    double acc[2 * NG];
#pragma unroll
    for (int e = 0; e < NG; ++e) {
      acc[e] = 0.0;
      acc[NG + e] = accp[e];
    }
    cta_reduce<L::TPR, 2 * NG>(acc, red, part);
    double* mine = ra.pbuf1 + (size_t)blockIdx.x * S::EB1;
    for (int i = tid; i < S::EB1; i += kThreads) {
      const int half = i / E, e = i % E;
      __stcg(mine + i, red[(e / NG) * 2 * NG + half * NG + e % NG]);
    }
    grid_barrier(ra.bar, epoch);
    grid_sum<S::EB1>(ra.pbuf1, tot, red);
    if (cta0) gather_gram<K, P, CPT, GLOBAL, NG>(tot + E, 0, a.coef + CS);
  }
  if (cta0 && tid == 0) {
    ctrl->xpending = 0;
    ctrl->xold = 0;
    if (ra.prof)
      for (int i = 0; i < 12; ++i) ra.prof[i] += pc[i];
  }
}

}  // namespace bkg
