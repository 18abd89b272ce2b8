// skv_topk.cuh -- block-wide exact top-k over fp64 importance.
//
// Replaces top_k_indices (matrix.hpp:162-176) as used by swa_select
// (attention.hpp:142-171): the k largest values under the total order
// (value desc, index asc), written ascending. Radix select on 64-bit order
// keys, MSB-first 8-bit digits with early exit, then one order-preserving
// compaction, so ties at the k-th value resolve to the lowest indices exactly
// as the reference's comparator does.
#pragma once

#include "skv_device.cuh"

namespace skvd {

#ifdef SKV_SELECT_TRACE  // phase timestamps of sequence 0 (debug builds only)
__device__ long long g_sel_trace[16];
#endif

template <int NT>
struct TopkSmem {
    uint32_t hist[256];
    uint64_t warp_tot[NT / 32];
    uint64_t warp_and[NT / 32], warp_or[NT / 32];
    uint64_t prefix;
    uint64_t mask;
    int remaining;
    int done;
};

// Inclusive warp scan of a u64.
__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += o;
    }
    return v;
}

// All NT threads of barrier `bar` call this (tid in [0, NT)). keys[0, nc) are
// order keys in shared memory; writes k ascending indices to out[0, k).
// Requires 1 <= k <= nc.
template <int NT, int BAR>
__device__ void block_topk(const uint64_t* keys, int nc, int k, int* out, TopkSmem<NT>& s,
                           int tid) {
    const int lane = tid & 31, warp = tid >> 5;
    // Bytes every candidate shares need no histogram pass: start the radix at
    // the first byte where the keys differ (importance values of one order of
    // magnitude share their sign/exponent byte).
    uint64_t kand = ~0ull, kor = 0;
    for (int i = tid; i < nc; i += NT) {
        kand &= keys[i];
        kor |= keys[i];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        kand &= __shfl_xor_sync(0xffffffffu, kand, off);
        kor |= __shfl_xor_sync(0xffffffffu, kor, off);
    }
    if (lane == 0) {
        s.warp_and[warp] = kand;
        s.warp_or[warp] = kor;
    }
    named_sync(BAR, NT);
    kand = ~0ull;
    kor = 0;
    for (int w = 0; w < NT / 32; ++w) {
        kand &= s.warp_and[w];
        kor |= s.warp_or[w];
    }
    const uint64_t diff = kand ^ kor;  // bits that vary among the candidates
    int top = 56;
    uint64_t prefix = 0, mask = 0;
    while (top > 0 && ((diff >> top) & 0xFFull) == 0) {
        mask |= 0xFFull << top;
        top -= 8;
    }
    prefix = kand & mask;
    int remaining = k;
#ifdef SKV_SELECT_TRACE
    int npass = 0;
#endif
    for (int shift = top; shift >= 0; shift -= 8) {
#ifdef SKV_SELECT_TRACE
        ++npass;
#endif
        for (int i = tid; i < 256; i += NT) s.hist[i] = 0;
        named_sync(BAR, NT);
#ifdef SKV_TOPK_MATCH
        // warp-aggregated histogram: lanes with the same digit add once
        for (int i0 = tid - lane; i0 < nc; i0 += NT) {
            const int i = i0 + lane;
            const uint64_t key = i < nc ? keys[i] : 0;
            const bool take = i < nc && (key & mask) == prefix;
            const unsigned bin = take ? static_cast<unsigned>((key >> shift) & 255u) : 256u + lane;
            const unsigned peers = __match_any_sync(0xffffffffu, bin);
            if (take && lane == __ffs(peers) - 1) atomicAdd(&s.hist[bin], static_cast<unsigned>(__popc(peers)));
        }
#else
        // Plain shared atomics, four keys in flight per thread. (Below the
        // common prefix the digits are spread, so same-bin conflicts are rare;
        // __match_any_sync aggregation measured ~2x slower per pass.)
        {
            int i = tid;
            for (; i + 3 * NT < nc; i += 4 * NT) {
                const uint64_t k0 = keys[i], k1 = keys[i + NT], k2 = keys[i + 2 * NT], k3 = keys[i + 3 * NT];
                if ((k0 & mask) == prefix) atomicAdd(&s.hist[(k0 >> shift) & 255u], 1u);
                if ((k1 & mask) == prefix) atomicAdd(&s.hist[(k1 >> shift) & 255u], 1u);
                if ((k2 & mask) == prefix) atomicAdd(&s.hist[(k2 >> shift) & 255u], 1u);
                if ((k3 & mask) == prefix) atomicAdd(&s.hist[(k3 >> shift) & 255u], 1u);
            }
            for (; i < nc; i += NT) {
                const uint64_t key = keys[i];
                if ((key & mask) == prefix) atomicAdd(&s.hist[(key >> shift) & 255u], 1u);
            }
        }
#endif
        named_sync(BAR, NT);
        if (warp == 0) {
            // lane l owns bins 255-8l .. 255-8l-7 (descending).
            uint32_t c[8];
            uint32_t tot = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = s.hist[255 - 8 * lane - j];
                tot += c[j];
            }
            uint32_t inc = tot;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, off);
                if (lane >= off) inc += o;
            }
            const uint32_t exc = inc - tot;
            const bool hit = exc < static_cast<uint32_t>(remaining) &&
                             static_cast<uint32_t>(remaining) <= inc;
            const unsigned ball = __ballot_sync(0xffffffffu, hit);
            if (lane == __ffs(ball) - 1) {
                uint32_t above = exc;
                int d = 0;
                uint32_t cnt = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (cnt == 0 && above + c[j] >= static_cast<uint32_t>(remaining)) {
                        d = 255 - 8 * lane - j;
                        cnt = c[j];
                    } else if (cnt == 0) {
                        above += c[j];
                    }
                }
                s.prefix = prefix | (static_cast<uint64_t>(d) << shift);
                s.mask = mask | (0xFFull << shift);
                s.remaining = remaining - static_cast<int>(above);
                s.done = (cnt == static_cast<uint32_t>(remaining) - above) ? 1 : 0;
            }
        }
        named_sync(BAR, NT);
        prefix = s.prefix;
        mask = s.mask;
        remaining = s.remaining;
        if (s.done) break;
    }
#ifdef SKV_SELECT_TRACE
    if (tid == 0 && blockIdx.x == 0) { g_sel_trace[8] = npass; g_sel_trace[9] = top; g_sel_trace[10] = clock64(); }
#endif
    // Order-preserving compaction. Element i is selected iff its masked key
    // is above the threshold prefix, or equal to it and among the first
    // `remaining` such elements by index.
    const int per = (nc + NT - 1) / NT;
    const int beg = min(tid * per, nc), end = min(beg + per, nc);
    uint32_t gt = 0, eq = 0;
    for (int i = beg; i < end; ++i) {
        const uint64_t km = keys[i] & mask;
        gt += km > prefix;
        eq += km == prefix;
    }
    const uint64_t v = (static_cast<uint64_t>(gt) << 32) | eq;
    const uint64_t inc = warp_incl_scan_u64(v, lane);
    if (lane == 31) s.warp_tot[warp] = inc;
    named_sync(BAR, NT);
    uint64_t wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s.warp_tot[w];
    const uint64_t exc = wbase + inc - v;
    uint32_t gt_before = static_cast<uint32_t>(exc >> 32);
    uint32_t eq_before = static_cast<uint32_t>(exc & 0xffffffffu);
    const uint32_t rem = static_cast<uint32_t>(remaining);
    for (int i = beg; i < end; ++i) {
        const uint64_t km = keys[i] & mask;
        if (km > prefix) {
            out[gt_before + min(eq_before, rem)] = i;
            ++gt_before;
        } else if (km == prefix) {
            if (eq_before < rem) out[gt_before + eq_before] = i;
            ++eq_before;
        }
    }
    named_sync(BAR, NT);
}

}  // namespace skvd
