// kernels_exact.cuh — exact-order sm_100a kernels (BKG_NUMERICS_EXACT).
//
// Each kernel reproduces the reference's per-element operation sequence with
// unfused IEEE double operations (__dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn), so
// results are bit-identical to the reference CPU build compiled with
// -ffp-contract=off.  Row-local kernels (BOP, BAXPY) are fully parallel; the
// row-ordered sums (BDOT entries, column norms) run as one serial chain per
// output entry fed by a cp.async multi-stage shared-memory pipeline.
// These kernels also serve every shape the tuned fast kernels do not cover.
#pragma once

#include <cuda_pipeline.h>

#include "common.cuh"

namespace bkg {

// Y = A X, one thread per (row, lane): kernels.hpp:146-155.
__global__ void k_spmm_exact(const Ctrl* ctrl, int64_t n, int k, const int64_t* __restrict__ rowptr,
                             const int32_t* __restrict__ cols, const double* __restrict__ vals,
                             const double* __restrict__ x, double* __restrict__ y) {
  if (stopped(ctrl)) return;
  const int64_t total = n * (int64_t)k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / k;
    const int c = (int)(idx - r * k);
    double acc = 0.0;
    const int64_t end = rowptr[r + 1];
    for (int64_t i = rowptr[r]; i < end; ++i)
      acc = __dadd_rn(acc, __dmul_rn(vals[i], x[(int64_t)cols[i] * k + c]));
    y[idx] = acc;
  }
}

// X <- X + Y * embed(gamma), one thread per element: kernels.hpp:109-123.
__global__ void k_baxpy_exact(const Ctrl* ctrl, int64_t n, int k, int p, int global,
                              double* __restrict__ x, const double* __restrict__ y,
                              const double* __restrict__ gamma) {
  if (stopped(ctrl)) return;
  const int64_t total = n * (int64_t)k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / k;
    const int c = (int)(idx - r * k);
    const int g = c / p, a = c - g * p;
    const double* blk = gamma + (size_t)(global ? 0 : g) * p * p;
    const double* yg = y + r * k + (int64_t)g * p;
    double acc = x[idx];
    for (int b = 0; b < p; ++b) acc = __dadd_rn(acc, __dmul_rn(yg[b], __ldg(blk + b * p + a)));
    x[idx] = acc;
  }
}

// out = b - out (solver.hpp:205-206), element-wise.
__global__ void k_residual_exact(int64_t total, const double* __restrict__ b,
                                 double* __restrict__ ax) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    ax[idx] = __dsub_rn(b[idx], ax[idx]);
}

// Row-ordered reduction chains.  Entry e of the output is
//   GRAM  hybrid: sum_r x[r, g p + a] * y[r, g p + b]        (kernels.hpp:74-85)
//         global: sum_r sum_g x[r, g p + a] * y[r, g p + b]   (same loop, block 0)
//   NORMS:        sqrt(sum_r x[r, c]^2)                         (block_vector.hpp:64-68)
// each accumulated by one thread in exactly the reference's order.  Row chunks
// (contiguous rows x all k lanes) are staged through shared memory with an
// S-stage cp.async pipeline so the serial chains never wait on DRAM.
constexpr int kChainThreads = 256;
constexpr int kChainStages = 4;

__host__ __device__ inline int chain_rows(int k) {
  int r = 1024 / k;
  return r < 1 ? 1 : r;
}

template <bool NORMS>
__global__ void __launch_bounds__(kChainThreads)
    k_chain_exact(const Ctrl* ctrl, int64_t n, int k, int p, int global, int entries, const double* __restrict__ x,
                  const double* __restrict__ y, double* __restrict__ out) {
  if (stopped(ctrl)) return;
  extern __shared__ double smem[];
  const int R = chain_rows(k);
  const int stage_elems = R * k;
  double* xs = smem;
  double* ys = smem + (size_t)kChainStages * stage_elems;
  const int tid = threadIdx.x;
  const int e = blockIdx.x * kChainThreads + tid;
  const bool active = e < entries;
  const int q = k / p;
  int ga = 0, gb = 0;  // column offsets of this entry's operands
  if (active) {
    if (NORMS) {
      ga = gb = e;
    } else {
      const int blk = e / (p * p);
      const int a = (e / p) % p, b = e % p;
      ga = blk * p + a;
      gb = blk * p + b;
    }
  }
  const int64_t nchunks = (n + R - 1) / R;
  auto issue = [&](int64_t chunk) {
    if (chunk < nchunks) {
      const int st = (int)(chunk % kChainStages);
      const int64_t r0 = chunk * R;
      const int rows = (int)(n - r0 < R ? n - r0 : R);
      const int cnt = rows * k;
      const double* xsrc = x + r0 * k;
      const double* ysrc = y + r0 * k;
      for (int i = tid; i < cnt; i += kChainThreads) {
        __pipeline_memcpy_async(xs + st * stage_elems + i, xsrc + i, sizeof(double));
        if (!NORMS) __pipeline_memcpy_async(ys + st * stage_elems + i, ysrc + i, sizeof(double));
      }
    }
    __pipeline_commit();
  };
  for (int s = 0; s < kChainStages - 1; ++s) issue(s);
  double acc = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) {
    issue(c + kChainStages - 1);
    __pipeline_wait_prior(kChainStages - 1);
    __syncthreads();
    if (active) {
      const int st = (int)(c % kChainStages);
      const double* xc = xs + st * stage_elems;
      const double* yc = NORMS ? xc : ys + st * stage_elems;
      const int rows = (int)(n - c * R < R ? n - c * R : R);
      if (NORMS || !global) {
        for (int rr = 0; rr < rows; ++rr)
          acc = __dadd_rn(acc, __dmul_rn(xc[rr * k + ga], yc[rr * k + gb]));
      } else {
        for (int rr = 0; rr < rows; ++rr)
          for (int g = 0; g < q; ++g)
            acc = __dadd_rn(acc, __dmul_rn(xc[rr * k + g * p + ga], yc[rr * k + g * p + gb]));
      }
    }
    __syncthreads();
  }
  if (active) out[e] = NORMS ? __dsqrt_rn(acc) : acc;
}

// Z = R (identity Preconditioner::apply, preconditioners.hpp:81-84).
__global__ void k_copy(const Ctrl* ctrl, int64_t total, const double* __restrict__ src,
                       double* __restrict__ dst) {
  if (stopped(ctrl)) return;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    dst[idx] = src[idx];
}

inline size_t chain_smem_bytes(int k, bool norms) {
  return (size_t)(norms ? 1 : 2) * kChainStages * chain_rows(k) * k * sizeof(double);
}

}  // namespace bkg
