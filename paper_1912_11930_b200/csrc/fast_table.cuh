// fast_table.cuh — instantiation table for the tuned fast kernels.
//
// The fused kernels are templated on (K lanes, P block width, CPT lanes per
// thread, GLOBAL).  Each K gets its own translation unit (fast_k*.cu) so the
// build parallelises; dispatch is a plain function-pointer table.
#pragma once

#include "kernels_fast.cuh"
#include "kernels_mma.cuh"

namespace bkg {

struct FastTable {
  const void* k1 = nullptr;
  const void* k2 = nullptr;
  const void* k3 = nullptr;
  const void* k2_jac = nullptr;  // K2 / K3 with Jacobi folded in (Z = D^-1 R)
  const void* k3_jac = nullptr;
  const void* spmm = nullptr;
  const void* gram = nullptr;
  const void* norms = nullptr;
  const void* baxpy = nullptr;
  int smem_iter = 0;   // dynamic smem of k1 / k2
  int smem_gram = 0;   // dynamic smem of gram
  int smem_norms = 0;  // dynamic smem of norms
  int cpt = 1;
  int rpc = 1;         // rows per CTA pass
  int e_iter = 0;      // partial entries per CTA (max of k1, k2)
  int e_gram = 0;
  int e_norms = 0;
  bool mma = false;  // K2/K3 are the DMMA kernels
  int rpc_mma = 1;    // their rows per CTA pass (8 rows per warp, Q warps per row block)
  int rpc_k1 = 1;     // rows per CTA pass of K1
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
  if constexpr (K % 8 == 0 && P <= 16) {  // warp-tile SpMM + DMMA Gram
    constexpr int W = K >= 16 ? 16 : 8;
    t->k1 = (const void*)&k1_tile<K, P, W, G>;
    t->rpc_k1 = (64 / W) * (8 * W / K);  // (rows per warp tile) x (row tiles per CTA)
  } else {
    t->k1 = (const void*)&k1_spmm_gram<K, P, CPT, G>;
    t->rpc_k1 = Layout<K, P, CPT>::RPC;
  }
  if constexpr (P == 8 || P == 16) {  // dense p x p contraction: FP64 DMMA
    t->k2 = (const void*)&k2_mma<K, P, G>;
    t->k3 = (const void*)&k3_mma<K, P, G>;
    t->k2_jac = (const void*)&k2_mma<K, P, G, true>;
    t->k3_jac = (const void*)&k3_mma<K, P, G, true>;
    t->mma = true;
    t->rpc_mma = 64 * P / K;
  } else {
    t->k2 = (const void*)&k2_update_gram<K, P, CPT, G>;
    t->k3 = (const void*)&k3_update_xp<K, P, CPT, G>;
    t->k2_jac = (const void*)&k2_update_gram<K, P, CPT, G, true>;
    t->k3_jac = (const void*)&k3_update_xp<K, P, CPT, G, true>;
  }
  t->spmm = (const void*)&k_spmm_fast<K, CPT>;
  t->gram = (const void*)&k_gram_fast<K, P, CPT, G>;
  t->norms = (const void*)&k_norms_fast<K, CPT>;
  t->baxpy = (const void*)&k_baxpy_fast<K, P, CPT, G>;
  t->smem_iter = S::bytes();
  t->smem_gram = (int)sizeof(double) * K * P;
  t->smem_norms = (int)sizeof(double) * K;
  t->cpt = CPT;
  t->rpc = Layout<K, P, CPT>::RPC;
  t->e_iter = S::RED;
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
