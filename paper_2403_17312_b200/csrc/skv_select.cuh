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

#ifndef SKV_SELECT_THREADS
#define SKV_SELECT_THREADS 128
#endif
// standalone / batched select width: 128 measured best for the batched per-step launch
// (sequences x layers CTAs: more resident per SM; 64 / 256 / 512 were slower overall)
constexpr int kSelectThreads = SKV_SELECT_THREADS;

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
    // 1: tok_prev is an SWA top-k selection made at n0 = cur_tok + 1 (its k0
    // global picks, then the local window) over the importance as it stands
    // before this fold (the host tracks it per layer). The next selection may
    // then be derived from it (incremental_select) instead of a full top-k.
    int incr;
    // head sharding (the cache holds some of the model's heads): the step row
    // v[pos] = sum over ALL heads of w is summed across the shards between a
    // partial pass (wsum_out: this shard's head sum, nothing else) and the
    // fold (wsum: the all-reduced row, used instead of the local partials).
    double* wsum_out;    // [B][m_prev]
    const double* wsum;  // [B][m_prev]
    // several layers in one launch (blockIdx.y = layer offset): element
    // strides of imp, wpart, idx/tok_prev and sparsity per layer (0: one layer)
    long long ls_imp, ls_wpart, ls_idx, ls_sp;
    long long ls_wsum;  // per-layer stride of wsum / wsum_out (head-shard rows of a whole step)
    // long contexts: the candidates' keys live in global scratch laid out like
    // imp ([layers][B][imp_ld], same strides) instead of shared memory
    uint64_t* gkeys;
};

__host__ __device__ inline size_t select_smem(int nc) {
    return align_up(sizeof(TopkSmem<kSelectThreads>), 16) + static_cast<size_t>(nc > 0 ? nc : 0) * 8;
}

template <int NT>
struct SelectScratch {
    double red_max[NT / 32];
    int red_cnt[NT / 32];  // (unused since the count went to `below`)
    int below;             // the sparsity count, summed with shared atomics
};

// The body shared by swa_select_kernel and the attend kernel's tail: NT
// threads synchronised on named barrier BAR, sequence b. keys: shared memory
// for n-k order keys. Weight partials are read through L2 (__ldcg): in the
// attend tail they come from sibling CTAs of the same grid.
// Stage importance[0, nc) into shared memory as fp64, several loads in
// flight per thread.
template <int NT>
__device__ __forceinline__ void stage_candidates(double* kd, const double* imp, int nc, int tid) {
    int i = tid;
    for (; i + 3 * NT < nc; i += 4 * NT) {
        const double a = imp[i], b = imp[i + NT], c = imp[i + 2 * NT], d = imp[i + 3 * NT];
        kd[i] = a;
        kd[i + NT] = b;
        kd[i + 2 * NT] = c;
        kd[i + 3 * NT] = d;
    }
    for (; i < nc; i += NT) kd[i] = imp[i];
}

#ifdef SKV_SELECT_TRACE
#define SEL_TRACE(i) \
    if (tid == 0 && b == 0) g_sel_trace[i] = clock64();
#else
#define SEL_TRACE(i)
#endif

// Incremental swa_select (attention.hpp:142-171) for step n0 + 1 from the
// selection of step n0, exact under the reference's order (value desc, index
// asc). G0, the k0 global picks of step n0, are the top k0 of [0, n0 - k0)
// before the fold; the fold only raises their importance (w >= 0) and leaves
// every other candidate unchanged, so they are still the top k0 of that range.
// Step n0 + 1 selects k1 in {k0, k0 + 1} (k is non-decreasing, by <= 1 per
// step):
//  - k1 = k0: the range gains x = n0 - k0 (leaving the local window), and the
//    top k0 of G0 + {x} is G0 with its weakest member replaced by x if x ranks
//    above it;
//  - k1 = k0 + 1: same range, top k0 + 1 = G0 + the best candidate outside G0
//    (one pass over the candidates).
// Either way there are no radix passes, and for k1 = k0 (most steps) no
// candidate is read. G0 sits ascending in positions [0, k0) of the token
// list, x at k0; o may alias the token list (every read is in registers).
template <int NT, int BAR, int R>
__device__ __forceinline__ void incremental_select(const SelectParams& p, int tid, int k0, int n0, int nc,
                                                   const int (&ti)[R], const double (&nvi)[R], const double* imp,
                                                   uint32_t* bm, TopkSmem<NT>& s, int* o) {
    const int lane = tid & 31, warp = tid >> 5, k1 = p.k;
    const bool weak = k1 == k0;  // find G0's weakest member (else: the best candidate outside G0)
    // a ranks before b (the reference's comparator, matrix.hpp:168-173)
    auto beats = [](uint64_t ka, int ia, uint64_t kb, int ib) { return ka > kb || (ka == kb && ia < ib); };
    auto better = [&](uint64_t ka, int ia, uint64_t kb, int ib) {
        return weak ? beats(kb, ib, ka, ia) : beats(ka, ia, kb, ib);
    };
    uint64_t bk = weak ? ~0ull : 0ull;  // sentinels: every real element ranks below / above them
    int bi = weak ? -1 : 0x7fffffff;
    if (weak) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int pos = tid + r * NT;
            if (pos < k0) {
                const uint64_t kk = order_key(nvi[r]);
                if (better(kk, ti[r], bk, bi)) {
                    bk = kk;
                    bi = ti[r];
                }
            } else if (pos == k0) {
                s.mask = order_key(nvi[r]);  // x = n0 - k0, the first local token
            }
        }
    } else {
        const int words = (nc + 31) >> 5;
        for (int i = tid; i < words; i += NT) bm[i] = 0u;
        named_sync(BAR, NT);
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (tid + r * NT < k0) atomicOr(&bm[ti[r] >> 5], 1u << (ti[r] & 31));
        named_sync(BAR, NT);
        for (int i = tid; i < nc; i += NT) {
            if ((bm[i >> 5] >> (i & 31)) & 1u) continue;
            const uint64_t kk = order_key(imp[i]);
            if (better(kk, i, bk, bi)) {
                bk = kk;
                bi = i;
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (better(ok, oi, bk, bi)) {
            bk = ok;
            bi = oi;
        }
    }
    if (lane == 0) {
        s.warp_tot[warp] = bk;
        s.warp_and[warp] = static_cast<uint64_t>(static_cast<uint32_t>(bi));
    }
    named_sync(BAR, NT);
    if (tid == 0) {
        for (int w = 1; w < NT / 32; ++w) {
            const uint64_t ok = s.warp_tot[w];
            const int oi = static_cast<int>(static_cast<uint32_t>(s.warp_and[w]));
            if (better(ok, oi, bk, bi)) {
                bk = ok;
                bi = oi;
            }
        }
        // weak: the member of G0 that x replaces (-1: none); else the added candidate
        s.remaining = weak ? (beats(s.mask, n0 - k0, bk, bi) ? bi : -1) : bi;
    }
    named_sync(BAR, NT);
    const int e = s.remaining;
    if (weak) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int pos = tid + r * NT;
            if (pos >= k0 || ti[r] == e) continue;
            o[(e >= 0 && ti[r] > e) ? pos - 1 : pos] = ti[r];
        }
        if (e >= 0 && tid == 0) o[k0 - 1] = n0 - k0;
    } else {
        int below = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int pos = tid + r * NT;
            if (pos >= k0) continue;
            o[ti[r] > e ? pos + 1 : pos] = ti[r];
            below += ti[r] < e;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) below += __shfl_xor_sync(0xffffffffu, below, off);
        if (lane == 0) s.warp_tot[warp] = static_cast<uint64_t>(below);  // tid 0's reads precede the last barrier
        named_sync(BAR, NT);
        if (tid == 0) {
            int cnt = 0;
            for (int w = 0; w < NT / 32; ++w) cnt += static_cast<int>(s.warp_tot[w]);
            o[cnt] = e;
        }
    }
    for (int i = tid; i < k1; i += NT) o[k1 + i] = p.n - k1 + i;  // local window
}

template <int NT, int BAR, bool WIDE = false>
__device__ void fold_and_select(const SelectParams p, int b, int tid, TopkSmem<NT>& s, uint64_t* keys,
                                SelectScratch<NT>& sc) {
    double* imp = p.imp + static_cast<size_t>(b) * p.imp_ld;
    // top-k candidates [0, nc): staged as fp64 in the key buffer, keyed in place
    const bool topk = p.select && !p.dense && p.variant != 2 && p.variant != 3;
    const int nc = topk ? p.n - p.k : 0;
    double* kd = reinterpret_cast<double*>(keys);
    SEL_TRACE(0);
    // sparsity helpers: each warp's max of the step row goes to sc.red_max
    // before a barrier the fold already has (tid 0 zeroes the count there too)
    auto publish_max = [&](double vm) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double o = __shfl_xor_sync(0xffffffffu, vm, off);
            vm = o > vm ? o : vm;
        }
        if ((tid & 31) == 0) sc.red_max[tid >> 5] = vm;
        if (tid == 0) sc.below = 0;
    };
    auto row_max = [&]() {
        double mx = 0.0;
        for (int w = 0; w < NT / 32; ++w) mx = sc.red_max[w] > mx ? sc.red_max[w] : mx;
        return mx;
    };
    auto finish_sparsity = [&]() {
        if (tid == 0) {
            const double mx = row_max();
            const int sparse = mx == 0.0 ? p.sp_n : sc.below + (p.sp_n - p.m_prev);
            p.sparsity[b] = static_cast<double>(sparse) / static_cast<double>(p.sp_n);
        }
    };
    constexpr int R = 4;  // folded positions per thread held in registers (fast path)
    // Incremental selection (incremental_select): decided from the parameters
    // alone, before anything is staged.
    const int k0 = p.m_prev / 2, n0 = p.cur_tok + 1;
    const bool incr = p.incr && topk && p.apply == 1 && p.tok_prev != nullptr && !p.wsum && !p.wsum_out &&
                      k0 < R * NT && p.m_prev == 2 * k0 && 2 * k0 < n0 && p.n == n0 + 1 &&
                      (p.k == k0 || p.k == k0 + 1) && p.variant == 1;
    int ti[R];      // fast path: folded token per position (-1: none)
    double nvi[R];  // and its new importance
    if (p.apply) {
        const float* wp = p.wpart + static_cast<size_t>(b) * p.G * p.m_prev;
        const int* tp = p.tok_prev ? p.tok_prev + static_cast<size_t>(b) * p.tok_prev_ld : nullptr;
        const double* ws = p.wsum ? p.wsum + static_cast<size_t>(b) * p.m_prev : nullptr;
        // the head-summed weight of selected position pos, in fixed group order
        auto row = [&](int pos) {
            if (ws) return ws[pos];
            double v = 0.0;
            if constexpr (WIDE) {
                // fp32 attend tails (config 1's 32 one-head CTAs; the 16-bit
                // kernels' 56-register budget would spill): every load of a
                // 32-group block is issued before the first add -- one L2 round
                // trip instead of two batches of 16; the adds keep the group order
                int g = 0;
                for (; g + 32 <= p.G; g += 32) {
                    float x[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = __ldcg(wp + static_cast<size_t>(g + j) * p.m_prev + pos);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v += static_cast<double>(x[j]);
                }
                for (; g < p.G; ++g) v += static_cast<double>(__ldcg(wp + static_cast<size_t>(g) * p.m_prev + pos));
            } else {
                for (int g = 0; g < p.G; ++g) v += static_cast<double>(__ldcg(wp + static_cast<size_t>(g) * p.m_prev + pos));
            }
            return v;
        };
        if (p.wsum_out) {  // head-shard partial pass: this shard's sum only
            double* wo = p.wsum_out + static_cast<size_t>(b) * p.m_prev;
            for (int pos = tid; pos < p.m_prev; pos += NT) wo[pos] = row(pos);
            return;
        }
        const bool assign_all = p.apply == 2;
        double vmax = 0.0;
        double v[R];
        if (p.m_prev <= R * NT) {
            // Fast path: every global load of the fold (weight partials, old
            // importance of the folded tokens) and the candidate staging is
            // issued before the first barrier -- one memory round trip.
            int t[R];
            double old[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int pos = tid + r * NT;
                v[r] = 0.0;
                t[r] = -1;
                old[r] = 0.0;
                if (pos < p.m_prev) {
                    t[r] = tp ? tp[pos] : pos;
                    v[r] = row(pos);
                    if (!assign_all && t[r] != p.cur_tok) old[r] = imp[t[r]];
                }
            }
            if (!incr) stage_candidates<NT>(kd, imp, nc, tid);
#pragma unroll
            for (int r = 0; r < R; ++r) vmax = t[r] >= 0 && v[r] > vmax ? v[r] : vmax;
            if (p.sp_n > 0) publish_max(vmax);
            named_sync(BAR, NT);  // staged candidates complete; every old value read (+ the warps' maxima)
            DTR_T(9, tid);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                ti[r] = t[r];
                nvi[r] = 0.0;
                if (t[r] < 0) continue;
                const double nv = (assign_all || t[r] == p.cur_tok) ? v[r] : old[r] + v[r];
                imp[t[r]] = nv;
                nvi[r] = nv;
                if (!incr && t[r] < nc) kd[t[r]] = nv;
            }
        } else {
            // Long selections (config 4: m = 820 at 128 threads): rounds of R
            // positions per thread, every load of a round issued before its
            // adds (the serial per-position chain was latency-bound, profiles/r2)
            for (int base = tid; base < p.m_prev; base += R * NT) {
                int t[R];
                double w[R], old[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int pos = base + r * NT;
                    t[r] = -1;
                    w[r] = 0.0;
                    old[r] = 0.0;
                    if (pos < p.m_prev) {
                        t[r] = tp ? tp[pos] : pos;
                        w[r] = row(pos);
                        if (!assign_all && t[r] != p.cur_tok) old[r] = imp[t[r]];
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (t[r] < 0) continue;
                    imp[t[r]] = (assign_all || t[r] == p.cur_tok) ? w[r] : old[r] + w[r];
                    vmax = w[r] > vmax ? w[r] : vmax;
                }
            }
            if (p.sp_n > 0) publish_max(vmax);
            named_sync(BAR, NT);  // the folded importance is visible to the staging (+ the warps' maxima)
            if (incr) {
                // G0 and x (positions 0..k0 of the list) with their folded values, as the fast path
                // holds them; every read precedes incremental_select's first barrier (o may alias tp)
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int pos = tid + r * NT;
                    ti[r] = pos <= k0 ? tp[pos] : -1;
                }
#pragma unroll
                for (int r = 0; r < R; ++r) nvi[r] = ti[r] >= 0 ? imp[ti[r]] : 0.0;
            } else {
                stage_candidates<NT>(kd, imp, nc, tid);
            }
        }
        DTR_T(10, tid);
        if (p.sp_n > 0) {
            // attention_sparsity (attention.hpp:275-310) of the head-summed step
            // row new_aw_row (length sp_n, zeros off-selection), threshold 0.01.
            // The row max was published before the fold's barrier; the count is
            // summed into sc.below and read after the next barrier (finish_sparsity)
            const double mx = row_max();
            const double thr = 0.01 * mx;
            int below = 0;
            if (p.m_prev <= R * NT) {
#pragma unroll
                for (int r = 0; r < R; ++r) below += (tid + r * NT < p.m_prev) && v[r] < thr;
            } else {
                for (int base = tid; base < p.m_prev; base += R * NT) {
                    double w[R];
#pragma unroll
                    for (int r = 0; r < R; ++r) w[r] = base + r * NT < p.m_prev ? row(base + r * NT) : thr;
#pragma unroll
                    for (int r = 0; r < R; ++r) below += w[r] < thr;
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) below += __shfl_xor_sync(0xffffffffu, below, off);
            if ((tid & 31) == 0 && below) atomicAdd(&sc.below, below);
        }
    } else {
        stage_candidates<NT>(kd, imp, nc, tid);
    }
    if (!p.select) {
        if (p.sp_n > 0) {
            named_sync(BAR, NT);  // every warp's count is in
            finish_sparsity();
        }
        return;
    }
    named_sync(BAR, NT);  // the fold and the staged candidates are complete (and the sparsity count)
    if (p.sp_n > 0) finish_sparsity();
    DTR_T(7, tid);
    int* o = p.idx + static_cast<size_t>(b) * p.idx_ld;
    if (p.variant == 2) {  // local_attention_mask (attention.hpp:247-256): the last m tokens
        for (int i = tid; i < p.m; i += NT) o[i] = p.n - p.m + i;
        return;
    }
    if (p.variant == 3) {  // strided_attention_mask (attention.hpp:258-269), phased onto n-1
        const int phase = (p.n - 1) % p.stride;
        for (int i = tid; i < p.m; i += NT) o[i] = phase + i * p.stride;
        return;
    }
    if (p.dense) {
        for (int i = tid; i < p.m; i += NT) o[i] = i;
        return;
    }
    if (incr) {
        incremental_select<NT, BAR, R>(p, tid, k0, n0, nc, ti, nvi, imp, reinterpret_cast<uint32_t*>(keys), s, o);
        return;
    }
    SEL_TRACE(1);
    for (int i = tid; i < nc; i += NT) keys[i] = order_key(kd[i]);  // in place, same thread
    named_sync(BAR, NT);
    DTR_T(8, tid);
    SEL_TRACE(2);
    block_topk<NT, BAR>(keys, nc, p.k, o, s, tid);                  // global picks, ascending
    SEL_TRACE(3);
    for (int i = tid; i < p.k; i += NT) o[p.k + i] = p.n - p.k + i;  // local window
}

}  // namespace skvd
