// skv_select.cuh -- per-sequence importance update + next-step selection.
//
// One CTA per sequence:
//   1. apply: fold the attend kernel's per-head-group weight sums into the fp64
//      head-summed importance, in fixed group order (deterministic):
//      acc_h[idx] += w (attention.hpp:219-227) reduced over heads
//      (head_summed_accum, attention.hpp:77-85); the step's new token and the
//      prefill seed (engine.hpp:508-512) assign instead of add.
//   2. select: swa_select (attention.hpp:142-171) for the next step's length:
//      exact fp64 top-k (skv_topk.cuh) over importance[0, n-k) plus the local
//      window, written ascending (SparseSelection::all, attention.hpp:31-38).
// Launched right after the attend kernel with programmatic dependent launch:
// it is resident early and waits (griddepcontrol.wait) for the attend grid.
#pragma once

#include "skv_topk.cuh"

namespace skvd {

constexpr int kSelectThreads = 256;

struct SelectParams {
    double* imp;  // [B][imp_ld]
    long long imp_ld;
    const float* wpart;  // [B][G][m_prev]
    int G, m_prev;
    const int* tok_prev;  // [B][tok_prev_ld]; nullptr = dense 0..m_prev-1
    long long tok_prev_ld;
    int apply;    // 0 none, 1 add (cur_tok assigned), 2 assign all
    int cur_tok;  // -1: none
    int select;   // compute a selection for (n, k, m, dense)
    int n, k, m, dense;
    int variant;  // 1 swa (dense when `dense`), 2 local, 3 strided (engine.hpp:531-569)
    int stride;   // strided only
    int sp_n;           // > 0: attention_sparsity of the folded row (length sp_n) into sparsity[b]
    double* sparsity;   // [B]
    int* idx;  // [B][idx_ld]
    long long idx_ld;
    int pdl_wait;
};

__host__ __device__ inline size_t select_smem(int nc) {
    return align_up(sizeof(TopkSmem<kSelectThreads>), 16) + static_cast<size_t>(nc > 0 ? nc : 0) * 8;
}

// The kernel itself is defined in skv_kernels.cu.

}  // namespace skvd
