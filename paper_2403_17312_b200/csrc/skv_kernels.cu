// skv_kernels.cu -- sm_100a kernels behind the C ABI other than the fused
// decode kernel: batched swa_select / top_k, fp64 quantize / dequantize,
// cache writes (append with fake-quant) and reads.
#include <algorithm>
#include <mutex>

#include "skv_internal.h"
#include "skv_select.cuh"
#include "skv_ledger.cuh"

namespace skvd {

// ---------------------------------------------------------------- selection
constexpr int kSelThreads = 512;


// ------------------------------------------------------------------- ledger
// Block-wide exclusive sum-scan of a u64; *total gets the block total.
template <int NT>
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t* warp_tot, uint64_t* total, int tid) {
    const int lane = tid & 31, warp = tid >> 5;
    const uint64_t inc = warp_incl_scan_u64(v, lane);
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    uint64_t base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        base += w < warp ? warp_tot[w] : 0;
        tot += warp_tot[w];
    }
    __syncthreads();
    *total = tot;
    return base + inc - v;
}

// Block-wide sum of an int (all threads get it).
template <int NT>
__device__ __forceinline__ long long block_sum(long long v, long long* red, int tid) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    long long t = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) t += red[w];
    __syncthreads();
    return t;
}

// KvLedger byte accounting of one (layer, sequence) step (thread 0): the
// device / host token deltas go into the cache's totals; the last sequence
// of the layer checks the device capacity after the layer's allocations --
// the reference checks before every store_new / reload / restore
// (memsim.hpp:99-109, 126-135, 158-165, 193-200), and since a layer's frees
// precede its allocations (engine.hpp:686-716) the running total peaks at
// the end, so the two agree. The failing request is reported with the
// reference's numbers: entries are tok_bytes each, so the first allocation
// that does not fit needs tok_bytes * (max(T0, floor(cap / tok_bytes)) + 1)
// bytes, T0 the tokens on device after the frees.
__device__ void ledger_account(const LedgerParams& p, int b, long long d_dev, long long d_host, long long allocs) {
    if (p.tot == nullptr) return;
    atomicAdd(&p.tot->dev_tokens, static_cast<unsigned long long>(d_dev));
    atomicAdd(&p.tot->host_tokens, static_cast<unsigned long long>(d_host));
    atomicAdd(p.layer_allocs, static_cast<unsigned long long>(allocs));
    __threadfence();
    const unsigned prev = atomicAdd(p.arrive, 1u);
    if (prev != gridDim.x - 1) return;
    __threadfence();
    const unsigned long long dev = atomicAdd(&p.tot->dev_tokens, 0ull);
    const unsigned long long al = atomicExch(p.layer_allocs, 0ull);
    atomicMax(&p.tot->peak_dev_tokens, dev);
    const unsigned long long e = p.tok_bytes;
    const unsigned long long ex = atomicExch(&p.tot->exhausted, 0ull);
    if (dev > p.cap_tokens) {  // dev * e > capacity: the reference's check comes first
        const unsigned long long t0 = dev - al;
        const unsigned long long fit = p.cap_tokens;
        report_status_inl(p.status, 2, p.layer, -1, -1, p.step, e * ((t0 > fit ? t0 : fit) + 1), p.cap_bytes);
    } else if (ex) {  // within the capacity, but one (layer, sequence) pool ran dry
        report_status_inl(p.status, 2, p.layer, -1, -1, p.step, 0ull, p.cap_bytes);
    }
    *p.arrive = 0;
}

// step_actions (scheduler.hpp:320-381) + apply_actions (engine.hpp:686-716)
// for one layer, one CTA per sequence. See skv_ledger.cuh. With a paged store
// the applied moves also free / allocate token slots: offloaded rows free
// theirs (tail of the FIFO, in token order), reloads, recomputes and the
// step's new token (store_new) take slots from the head, in that order.
__global__ void __launch_bounds__(kLedgerThreads) ledger_step_kernel(const LedgerParams p) {
    constexpr int NT = kLedgerThreads;
    constexpr uint64_t M21 = (1ull << 21) - 1;
    __shared__ uint64_t wt[NT / 32];
    __shared__ long long red[NT / 32];
    __shared__ int s_split;
    extern __shared__ __align__(128) uint8_t smem[];
    const int b = blockIdx.x, tid = threadIdx.x;
    // Phase I only stores the step's new token: nothing of the preceding
    // attend / select is read, so the next layer's attend may start at once.
    // Every other phase reads the selection the preceding kernel made.
    if (p.phase != 1) pdl_wait();
    pdl_launch_dependents();
    const int ntok = p.existing;
    const bool paged = p.slots.slot != nullptr;
    uint8_t* tg = p.tiers + static_cast<size_t>(b) * p.tier_ld;
    int* lists = p.lists + static_cast<size_t>(b) * 4 * p.list_ld;
    int* cnt = p.counts + static_cast<size_t>(b) * 4;
    int* aslots = p.act_slots ? p.act_slots + static_cast<size_t>(b) * 4 * p.list_ld : nullptr;
    int* slot = paged ? p.slots.slot + static_cast<size_t>(b) * p.slots.slot_ld : nullptr;
    int* fq = paged ? p.slots.fq + static_cast<size_t>(b) * p.slots.pcap : nullptr;
    unsigned* ht = paged ? p.slots.fq_ht + static_cast<size_t>(b) * 2 : nullptr;
    // store_new of the step's token (the current token is never on a list);
    // ht = (head, free count) of the FIFO ring
    auto store_current = [&](unsigned head, unsigned count) {
        if (paged) {
            if (count > 0) {
                slot[ntok] = fq[head];
                ht[0] = (head + 1) % static_cast<unsigned>(p.slots.pcap);
                ht[1] = count - 1;
            } else {
                slot[ntok] = -1;
                if (p.tot) atomicAdd(&p.tot->exhausted, 1ull);  // reported by ledger_account
            }
        }
        tg[ntok] = kTierDevice;
    };
    if (p.phase == 1) {
        if (tid < 4) cnt[tid] = 0;
        if (tid == 0 && p.aux) p.aux[b * 4] = 0;
        if (tid == 0 && p.store_current) {
            store_current(paged ? ht[0] : 0u, paged ? ht[1] : 0u);
            if (p.apply) ledger_account(p, b, 1, 0, 1);
        }
        return;
    }
    uint8_t* t8 = smem;          // pre-action tiers [ntok]
    uint8_t* act = smem + ntok;  // bit0 offload, bit1 delete, bit2 reload/recompute
    for (int i = tid; i < ntok; i += NT) {
        t8[i] = tg[i];
        act[i] = 0;
    }
    __syncthreads();
    const int n_tot = ntok + 1;
    const int nonlocal = n_tot > p.k ? n_tot - p.k : 0;
    const int per = (ntok + NT - 1) / NT;
    const int beg = min(tid * per, ntok), end = min(beg + per, ntok);

    // device / host counts and device-before-window count, packed 3 x 21 bits
    uint64_t dv = 0, hs = 0, dnl = 0;
    for (int i = beg; i < end; ++i) {
        dv += t8[i] == kTierDevice;
        hs += t8[i] == kTierHost;
        dnl += (t8[i] == kTierDevice) && i < nonlocal;
    }
    uint64_t tot;
    const uint64_t ex = block_excl_scan<NT>((dv << 42) | (hs << 21) | dnl, wt, &tot, tid);
    const long long ndev = static_cast<long long>(tot >> 42);
    const long long nh = static_cast<long long>((tot >> 21) & M21);
    const long long ndnl = static_cast<long long>(tot & M21);
    const long long to_off = p.target > nh ? p.target - nh : 0;
    const long long n_off = to_off < ndnl ? to_off : ndnl;
    // offload: the oldest to_off device tokens, stopping at the local window
    long long drank = static_cast<long long>(ex >> 42);
    for (int i = beg; i < end; ++i) {
        if (t8[i] != kTierDevice) continue;
        if (i < nonlocal && drank < to_off) {
            lists[drank] = i;
            act[i] |= 1;
        }
        ++drank;
    }
    __syncthreads();
    // Phase III: delete the oldest ceil(beta * host_after) of host U offloaded
    long long n_del = 0;
    const long long host_after = nh + n_off;
    if (p.phase == 3 && host_after > 0) {
        const long long to_del = static_cast<long long>(ceil(p.beta * static_cast<double>(host_after)));
        uint64_t hc = 0;
        for (int i = beg; i < end; ++i) hc += (t8[i] == kTierHost) || (act[i] & 1);
        uint64_t htot;
        long long hrank = static_cast<long long>(block_excl_scan<NT>(hc, wt, &htot, tid));
        for (int i = beg; i < end; ++i) {
            if (!((t8[i] == kTierHost) || (act[i] & 1))) continue;
            if (hrank < to_del) {
                lists[p.list_ld + hrank] = i;
                act[i] |= 2;
            }
            ++hrank;
        }
        n_del = to_del < host_after ? to_del : host_after;
        __syncthreads();
    }
    // selected tokens: reload (host or just offloaded) / recompute (deleted)
    const int* sel = p.sel + static_cast<size_t>(b) * p.sel_ld;
    const int sper = (p.m + NT - 1) / NT;
    const int sbeg = min(tid * sper, p.m), send = min(sbeg + sper, p.m);
    uint64_t rl = 0, rc = 0;
    for (int q = sbeg; q < send; ++q) {
        const int t = sel[q];
        if (t < 0 || t >= ntok || t8[t] == kTierAbsent) continue;  // the current token
        const bool rec = (act[t] & 2) || t8[t] == kTierDeleted;
        rc += rec;
        rl += !rec && (t8[t] == kTierHost || (act[t] & 1));
    }
    uint64_t stot;
    const uint64_t sex = block_excl_scan<NT>((rl << 32) | rc, wt, &stot, tid);
    long long rlr = static_cast<long long>(sex >> 32), rcr = static_cast<long long>(sex & 0xffffffffu);
    for (int q = sbeg; q < send; ++q) {
        const int t = sel[q];
        if (t < 0 || t >= ntok || t8[t] == kTierAbsent) continue;
        const bool rec = (act[t] & 2) || t8[t] == kTierDeleted;
        if (rec) {
            lists[3 * p.list_ld + rcr++] = t;
            act[t] |= 4;
        } else if (t8[t] == kTierHost || (act[t] & 1)) {
            lists[2 * p.list_ld + rlr++] = t;
            act[t] |= 4;
        }
    }
    __syncthreads();
    const int n_rl = static_cast<int>(stot >> 32), n_rc = static_cast<int>(stot & 0xffffffffu);
    if (tid == 0) {
        cnt[0] = static_cast<int>(n_off);
        cnt[1] = static_cast<int>(n_del);
        cnt[2] = n_rl;
        cnt[3] = n_rc;
        if (p.apply && p.tot) {
            atomicAdd(&p.tot->moved[0], static_cast<unsigned long long>(n_off));
            atomicAdd(&p.tot->moved[1], static_cast<unsigned long long>(n_del));
            atomicAdd(&p.tot->moved[2], static_cast<unsigned long long>(n_rl));
            atomicAdd(&p.tot->moved[3], static_cast<unsigned long long>(n_rc));
        }
    }
    if (!p.apply) return;
    // a token offloaded and re-selected in the same step keeps its device row
    // (the state the sequential offload-then-reload leaves): no slot moves
    auto kept = [&](int t) { return (act[t] & 1) && (act[t] & 4) && !(act[t] & 2); };
    if (paged) {
        const unsigned head0 = ht[0], cnt0 = ht[1], pcap = static_cast<unsigned>(p.slots.pcap);
        // frees: offloaded rows that are not kept, in offload-list (token) order
        int nf_mine = 0;
        const int oper = (static_cast<int>(n_off) + NT - 1) / NT;
        const int obeg = min(tid * oper, static_cast<int>(n_off)), oend = min(obeg + oper, static_cast<int>(n_off));
        for (int i = obeg; i < oend; ++i) nf_mine += !kept(lists[i]);
        uint64_t ftot;
        unsigned fr = static_cast<unsigned>(block_excl_scan<NT>(static_cast<uint64_t>(nf_mine), wt, &ftot, tid));
        for (int i = obeg; i < oend; ++i) {
            const int t = lists[i];
            const int sl = slot[t];
            aslots[i] = sl;  // the offload copies out of this slot
            if (!kept(t)) {
                fq[(head0 + cnt0 + fr++) % pcap] = sl;
                slot[t] = -1;
            }
        }
        const unsigned cnt1 = cnt0 + static_cast<unsigned>(ftot);
        // allocations: reload-list entries (not kept), then recompute entries
        const int n_al_lists = n_rl + n_rc;
        const int aper = (n_al_lists + NT - 1) / NT;
        const int abeg = min(tid * aper, n_al_lists), aend = min(abeg + aper, n_al_lists);
        int na_mine = 0;
        for (int i = abeg; i < aend; ++i) {
            const int t = i < n_rl ? lists[2 * p.list_ld + i] : lists[3 * p.list_ld + (i - n_rl)];
            na_mine += !(i < n_rl && kept(t));
        }
        if (tid == 0) s_split = n_rl;
        uint64_t atot;
        unsigned ar = static_cast<unsigned>(block_excl_scan<NT>(static_cast<uint64_t>(na_mine), wt, &atot, tid));
        for (int i = abeg; i < aend; ++i) {
            const bool rel = i < n_rl;
            const int t = rel ? lists[2 * p.list_ld + i] : lists[3 * p.list_ld + (i - n_rl)];
            int* as = rel ? aslots + 2 * p.list_ld + i : aslots + 3 * p.list_ld + (i - n_rl);
            if (rel && kept(t)) {  // keeps its row: nothing to copy in
                *as = -1;
                continue;
            }
            const unsigned a = ar++;
            if (a < cnt1) {
                const int sl = fq[(head0 + a) % pcap];
                slot[t] = sl;
                *as = sl;
                if (rel && a >= cnt0) atomicMin(&s_split, i);  // a slot this step's offload frees
            } else {
                slot[t] = -1;
                *as = -1;
                if (p.tot) atomicAdd(&p.tot->exhausted, 1ull);  // reported by ledger_account
            }
        }
        __syncthreads();
        if (tid == 0) {
            const unsigned used = static_cast<unsigned>(atot) < cnt1 ? static_cast<unsigned>(atot) : cnt1;
            const unsigned head1 = (head0 + used) % pcap, cnt2 = cnt1 - used;
            ht[0] = head1;
            ht[1] = cnt2;
            p.aux[b * 4] = s_split;
            if (p.store_current) store_current(head1, cnt2);
        }
    }
    // tiers after the step + the ledger's byte deltas
    long long post_dev = 0, post_host = 0, allocs = 0;
    for (int i = tid; i < ntok; i += NT) {
        const uint8_t a = act[i];
        uint8_t t = t8[i];
        if (a) {
            if (a & 1) t = kTierHost;
            if (a & 2) t = kTierDeleted;
            if (a & 4) t = kTierDevice;
            tg[i] = t;
            allocs += (a & 4) && !kept(i);
        }
        post_dev += t == kTierDevice;
        post_host += t == kTierHost;
    }
    if (p.tot) {  // reloads that keep their device row: listed, but no host -> device copy
        long long nk = 0;
        for (int i = tid; i < n_rl; i += NT) nk += kept(lists[2 * p.list_ld + i]);
        nk = block_sum<NT>(nk, red, tid);
        if (tid == 0) atomicAdd(&p.tot->kept, static_cast<unsigned long long>(nk));
    }
    post_dev = block_sum<NT>(post_dev, red, tid);
    post_host = block_sum<NT>(post_host, red, tid);
    allocs = block_sum<NT>(allocs, red, tid);
    if (tid == 0) {
        if (p.store_current && !paged) tg[ntok] = kTierDevice;
        const long long sc = p.store_current ? 1 : 0;
        ledger_account(p, b, post_dev + sc - ndev, post_host - nh, allocs + sc);
    }
}

// Bt [2h x h] = [Wk | Wv]^T for the recompute GEMM (16-bit elements);
// W* are [h x h] row-major (out = x . W). 32 x 32 tiles through smem.
__global__ void transpose_kv_weights_kernel(const uint16_t* __restrict__ wk, const uint16_t* __restrict__ wv,
                                            uint16_t* __restrict__ bt, int h) {
    __shared__ uint16_t tile[32][33];
    const int which = blockIdx.z;
    const uint16_t* w = which ? wv : wk;
    const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;  // rows i (input), cols j (output) of W
    for (int r = threadIdx.y; r < 32; r += blockDim.y) tile[r][threadIdx.x] = w[static_cast<size_t>(i0 + r) * h + j0 + threadIdx.x];
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y)
        bt[static_cast<size_t>(which * h + j0 + r) * h + i0 + threadIdx.x] = tile[threadIdx.x][r];
}

// Ascending list membership (the ledger's lists are in token order).
__device__ __forceinline__ bool in_sorted(const int* list, int cnt, int t) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(list + mid) < t) lo = mid + 1; else hi = mid;
    }
    return lo < cnt && __ldg(list + lo) == t;
}

// Offload / reload the rows of one action list: grid (token chunk, sequence[,
// direction]). 16-byte vectors; the host side is mapped pinned memory (PCIe
// zero-copy). With which = -1 one launch runs both lists at once, offload on
// blockIdx.z 0 and reload on 1, so device->host writes and host->device reads
// share the PCIe link in both directions. A token on both lists (offloaded
// and selected in the same step, scheduler.hpp:360-375) keeps its device row:
// the offload copies it out without poisoning it and the reload skips it --
// the state the sequential offload-then-reload leaves behind.
// Paged store: the device side is addressed by the ledger's slot lists. A
// reload into a slot that this step's offload frees must wait for that copy:
// those reloads (from aux[b*4] on) run in a second launch (second = 1).
__global__ void __launch_bounds__(256) kv_move_kernel(const MoveParams p) {
    pdl_wait();  // the lists come from the preceding ledger kernel
    pdl_launch_dependents();
    const int b = blockIdx.y;
    const bool both = p.which < 0;
    const int which = both ? (blockIdx.z == 0 ? 0 : 2) : p.which;
    int lo = 0, hi = p.counts[b * 4 + which];
    if (which == 2 && p.aux) {
        const int split = p.aux[b * 4];
        if (p.second) lo = split;
        else hi = split < hi ? split : hi;
    }
    const int* list = p.lists + (static_cast<size_t>(b) * 4 + which) * p.list_ld;
    const int* slots = p.act_slots ? p.act_slots + (static_cast<size_t>(b) * 4 + which) * p.list_ld : nullptr;
    const int ocnt = both ? p.counts[b * 4 + (2 - which)] : 0;
    const int* other = p.lists + (static_cast<size_t>(b) * 4 + (2 - which)) * p.list_ld;
    const long long vec_per_tok = p.tok_bytes / 16;
    const long long total = static_cast<long long>(hi - lo) * vec_per_tok;
    for (long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; v < total;
         v += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = lo + static_cast<int>(v / vec_per_tok);
        const int t = list[i];
        const int sl = slots ? slots[i] : t;
        if (sl < 0) continue;  // a kept row, or no slot (the ledger reported the OOM)
        const bool shared = both && in_sorted(other, ocnt, t);
        const size_t vo = static_cast<size_t>(v % vec_per_tok) * 16;
        const size_t hoff = static_cast<size_t>(b) * p.seq_bytes + static_cast<size_t>(t) * p.tok_bytes + vo;
        const size_t doff = static_cast<size_t>(b) * p.dev_seq_bytes + static_cast<size_t>(sl) * p.tok_bytes + vo;
        if (which == 0) {
            uint4* d = reinterpret_cast<uint4*>(p.dev + doff);
            *reinterpret_cast<uint4*>(p.host + hoff) = *d;
            if (p.poison && !shared) *d = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        } else if (!shared) {
            *reinterpret_cast<uint4*>(p.dev + doff) = *reinterpret_cast<const uint4*>(p.host + hoff);
        }
    }
}

// Importance fold + next selection, one CTA per sequence (skv_select.cuh).
__global__ void __launch_bounds__(kSelectThreads) swa_select_kernel(const SelectParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    TopkSmem<kSelectThreads>& s = *reinterpret_cast<TopkSmem<kSelectThreads>*>(smem);
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + align_up(sizeof(TopkSmem<kSelectThreads>), 16));
    __shared__ SelectScratch<kSelectThreads> scratch;
    pdl_launch_dependents();
    if (p.pdl_wait) pdl_wait();
    const long long y = blockIdx.y;
    if (p.gkeys) keys = p.gkeys + (y * p.ls_imp + static_cast<long long>(blockIdx.x) * p.imp_ld);
    if (y == 0) {
        fold_and_select<kSelectThreads, 1>(p, blockIdx.x, threadIdx.x, s, keys, scratch);
        return;
    }
    SelectParams q = p;  // layer blockIdx.y of a batched launch
    q.imp += y * p.ls_imp;
    q.wpart += y * p.ls_wpart;
    q.idx += y * p.ls_idx;
    if (q.tok_prev) q.tok_prev += y * p.ls_idx;
    q.sparsity += y * p.ls_sp;
    if (q.wsum) q.wsum += y * p.ls_wsum;
    if (q.wsum_out) q.wsum_out += y * p.ls_wsum;
    fold_and_select<kSelectThreads, 1>(q, blockIdx.x, threadIdx.x, s, keys, scratch);
}

// attend_over_indices' accumulator update for an arbitrary index list (any
// order, repeats; attention.hpp:219-227): every occurrence adds its weight.
// One CTA per sequence: the head-summed step row new_aw_row (length n, zeros
// off-selection) is scattered into a scratch row with fp64 atomics, then
// added to the importance, and attention_sparsity (attention.hpp:275-310) of
// that row is recorded.
__global__ void __launch_bounds__(256) scatter_fold_kernel(double* imp, long long imp_ld, const float* wpart, int G,
                                                           int m, const int* tok, long long tok_ld,
                                                           const double* wsum, int n, double* sparsity,
                                                           double* rows) {
    constexpr int NT = 256;
    __shared__ double red_max[NT / 32];
    __shared__ int red_cnt[NT / 32];
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* row = rows + static_cast<size_t>(b) * imp_ld;
    double* im = imp + static_cast<size_t>(b) * imp_ld;
    for (int t = tid; t < n; t += NT) row[t] = 0.0;
    __syncthreads();
    for (int pos = tid; pos < m; pos += NT) {
        double v = 0.0;
        if (wsum) {
            v = wsum[static_cast<size_t>(b) * m + pos];
        } else {
            for (int g = 0; g < G; ++g) v += static_cast<double>(wpart[(static_cast<size_t>(b) * G + g) * m + pos]);
        }
        atomicAdd(row + tok[static_cast<size_t>(b) * tok_ld + pos], v);
    }
    __syncthreads();
    double mx = 0.0;
    for (int t = tid; t < n; t += NT) {
        const double v = row[t];
        im[t] += v;
        mx = v > mx ? v : mx;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, mx, off);
        mx = o > mx ? o : mx;
    }
    if (lane == 0) red_max[warp] = mx;
    __syncthreads();
    mx = 0.0;
    for (int w = 0; w < NT / 32; ++w) mx = red_max[w] > mx ? red_max[w] : mx;
    const double thr = 0.01 * mx;
    int below = 0;
    for (int t = tid; t < n; t += NT) below += row[t] < thr;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) below += __shfl_xor_sync(0xffffffffu, below, off);
    if (lane == 0) red_cnt[warp] = below;
    __syncthreads();
    if (tid == 0) {
        int cnt = 0;
        for (int w = 0; w < NT / 32; ++w) cnt += red_cnt[w];
        sparsity[b] = static_cast<double>(mx == 0.0 ? n : cnt) / static_cast<double>(n);
    }
}

// top_k_indices (matrix.hpp:162-176) per row.
__global__ void __launch_bounds__(kSelThreads)
    top_k_kernel(const double* __restrict__ v, long long ld, int len, int k, int* __restrict__ out,
                 uint64_t* gkeys) {
    extern __shared__ __align__(128) uint8_t smem[];
    TopkSmem<kSelThreads>& s = *reinterpret_cast<TopkSmem<kSelThreads>*>(smem);
    const int b = blockIdx.x, tid = threadIdx.x;
    // keys in shared memory, or in the caller-row-shaped global scratch for long rows
    uint64_t* keys = gkeys ? gkeys + static_cast<size_t>(b) * ld
                           : reinterpret_cast<uint64_t*>(smem + align_up(sizeof(TopkSmem<kSelThreads>), 16));
    const double* row = v + static_cast<size_t>(b) * ld;
    for (int i = tid; i < len; i += kSelThreads) keys[i] = order_key(row[i]);
    named_sync(1, kSelThreads);
    block_topk<kSelThreads, 1>(keys, len, k, out + static_cast<size_t>(b) * k, s, tid);
}

// ------------------------------------------------------------------- quant
// quantize (quant.hpp:43-81): one warp per channel group, fp64 throughout.
__global__ void quantize_kernel(const double* __restrict__ x, long long groups, long long cs,
                                uint32_t bits, uint16_t* __restrict__ codes,
                                double* __restrict__ scales, long long* __restrict__ zps) {
    const long long grp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (grp >= groups) return;
    const double* c = x + grp * cs;
    double lo = c[0], hi = c[0];
    for (long long i = lane; i < cs; i += 32) {
        lo = c[i] < lo ? c[i] : lo;
        hi = hi < c[i] ? c[i] : hi;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double olo = __shfl_xor_sync(0xffffffffu, lo, off);
        const double ohi = __shfl_xor_sync(0xffffffffu, hi, off);
        lo = olo < lo ? olo : lo;
        hi = hi < ohi ? ohi : hi;
    }
    double scale;
    if (hi == lo) {
        const double a = fabs(lo);
        scale = a < 1e-12 ? 1e-12 : a;
    } else {
        const double levels = static_cast<double>((1ull << bits) - 1);
        const double s = (hi - lo) / levels;
        scale = s < 1e-12 ? 1e-12 : s;
    }
    const long long zp = rne_ref(-lo / scale);
    const long long max_code = static_cast<long long>((1ull << bits) - 1);
    for (long long i = lane; i < cs; i += 32) {
        long long code = rne_ref(c[i] / scale + static_cast<double>(zp));
        code = code < 0 ? 0 : (code > max_code ? max_code : code);
        codes[grp * cs + i] = static_cast<uint16_t>(code);
    }
    if (lane == 0) {
        scales[grp] = scale;
        zps[grp] = zp;
    }
}

// dequantize (quant.hpp:84-95)
__global__ void dequantize_kernel(const uint16_t* __restrict__ codes, long long len, long long cs,
                                  const double* __restrict__ scales,
                                  const long long* __restrict__ zps, double* __restrict__ out) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= len) return;
    const long long g = i / cs;
    out[i] = scales[g] * (static_cast<double>(codes[i]) - static_cast<double>(zps[g]));
}

// ------------------------------------------------------------- cache write
// One (token, K|V, head) row of D values from the compute dtype into the
// storage dtype, one warp; INT8 rows are engine.hpp:469-483's fake-quant
// (quant.hpp:43-81 per head_dim group, in fp64: bit-exact codes).
__device__ __forceinline__ void quant_row_u8(uint8_t* dst, float2* meta, const double (&x)[kHeadDim / 32], int lane) {
    constexpr int D = kHeadDim;
    double lo = x[0], hi = x[0];
#pragma unroll
    for (int i = 1; i < D / 32; ++i) {
        lo = x[i] < lo ? x[i] : lo;
        hi = hi < x[i] ? x[i] : hi;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double olo = __shfl_xor_sync(0xffffffffu, lo, off);
        const double ohi = __shfl_xor_sync(0xffffffffu, hi, off);
        lo = olo < lo ? olo : lo;
        hi = hi < ohi ? ohi : hi;
    }
    double scale;
    if (hi == lo) {
        const double a = fabs(lo);
        scale = a < 1e-12 ? 1e-12 : a;
    } else {
        const double s = (hi - lo) / 255.0;
        scale = s < 1e-12 ? 1e-12 : s;
    }
    const long long zp = rne_ref(-lo / scale);
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < D / 32; ++i) {
        long long c = rne_ref(x[i] / scale + static_cast<double>(zp));
        c = c < 0 ? 0 : (c > 255 ? 255 : c);
        packed |= static_cast<uint32_t>(c) << (8 * i);
    }
    reinterpret_cast<uint32_t*>(dst)[lane] = packed;
    if (lane == 0) *meta = make_float2(static_cast<float>(scale), static_cast<float>(-scale * static_cast<double>(zp)));
}

// One (token, K|V, head) row of D values from the compute dtype into the
// storage dtype, one warp; INT8 rows are engine.hpp:469-483's fake-quant
// (quant.hpp:43-81 per head_dim group, in fp64: bit-exact codes).
// tok: the token's storage; row (which, h) of H heads.
template <class QT, class KV>
__device__ __forceinline__ void store_row(uint8_t* tok, int which, int h, int H, const QT* src, int lane) {
    constexpr int D = kHeadDim;
    if constexpr (!KV::QUANT) {
        using T = typename KV::T;
        T* d = reinterpret_cast<T*>(tok + static_cast<size_t>(which * H + h) * kv_row_bytes<KV>());
        for (int i = lane; i < D; i += 32) d[i] = from_f<T>(to_f(src[i]));
    } else {
        double x[D / 32];
#pragma unroll
        for (int i = 0; i < D / 32; ++i) x[i] = static_cast<double>(to_f(src[lane * (D / 32) + i]));
        quant_row_u8(tok + u8_code_off(which, h, H), reinterpret_cast<float2*>(tok + u8_meta_off(which, h, H)), x,
                     lane);
    }
}

// AttentionState::append_token for a block of tokens (+ engine head_rows
// fake-quant). One warp per (b, t, kv, head) row of D elements. Paged store:
// prompt tokens take slot t (the FIFO hands slots out in order until the
// first decode allocation), and the sequence's FIFO head moves past them.
template <class QT, class KV>
__global__ void cache_write_kernel(const CacheView cv, double* __restrict__ imp, uint8_t* __restrict__ tiers,
                                   const QT* __restrict__ k, const QT* __restrict__ v, int H, int b0, int nb,
                                   int t0, int nt) {
    const long long row = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long rows = static_cast<long long>(nb) * nt * 2 * H;
    if (row >= rows) return;
    const int h = static_cast<int>(row % H);
    const int which = static_cast<int>((row / H) % 2);
    const int t = static_cast<int>((row / (2 * H)) % nt);
    const int bb = static_cast<int>(row / (2LL * H * nt));
    const QT* src = (which ? v : k) + ((static_cast<size_t>(bb) * nt + t) * H + h) * kHeadDim;
    const size_t tok = static_cast<size_t>(b0 + bb) * cv.Ncap + (t0 + t);
    const size_t srow = static_cast<size_t>(b0 + bb) * cv.kv_ncap + (t0 + t);  // slot t when paged
    uint8_t* tokp = cv.kv + srow * 2 * H * static_cast<size_t>(kv_row_bytes<KV>());
    store_row<QT, KV>(tokp, which, h, H, src, lane);
    if (lane == 0 && h == 0 && which == 0) {
        imp[tok] = 0.0;
        if (tiers) {
            if (cv.tot && tiers[tok] == kTierAbsent) atomicAdd(&cv.tot->dev_tokens, 1ull);
            tiers[tok] = kTierDevice;  // KvLedger::store_new: new KV lands on device
        }
        if (cv.slot) {
            cv.slot[tok] = t0 + t;
            if (t == nt - 1) {  // one thread per sequence: the FIFO moves past the prompt
                unsigned* ht = cv.fq_ht + static_cast<size_t>(b0 + bb) * 2;
                const unsigned pcap = static_cast<unsigned>(cv.kv_ncap);
                const unsigned used = pcap - ht[1];
                const unsigned ni = used > static_cast<unsigned>(t0 + nt) ? used : static_cast<unsigned>(t0 + nt);
                ht[0] = ni % pcap;
                ht[1] = pcap - ni;
            }
        }
    }
}

// INT8 recompute write-back (engine.hpp:718-737: recompute_kv re-applies
// head_rows' fake-quant): the recompute GEMM's fp32 rows [M][2h] are rounded
// to the compute dtype, as the appended rows were, and quantised into their
// slots. One warp per (row, K|V, head).
template <class QT>
__global__ void quant_scatter_kernel(const float* __restrict__ C, const int* __restrict__ m_dev, const int2* rowmap,
                                     uint8_t* kv, int H, int kv_ncap) {
    const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long M = *m_dev;
    if (w >= M * 2 * H) return;
    const int h = static_cast<int>(w % H), which = static_cast<int>((w / H) % 2);
    const long long r = w / (2LL * H);
    const int2 bt = rowmap[r];
    if (bt.y < 0) return;
    const float* src = C + (r * 2 * H + static_cast<long long>(which) * H + h) * kHeadDim;
    double x[kHeadDim / 32];
#pragma unroll
    for (int i = 0; i < kHeadDim / 32; ++i) x[i] = static_cast<double>(to_f(from_f<QT>(src[lane * (kHeadDim / 32) + i])));
    uint8_t* tokp = kv + (static_cast<size_t>(bt.x) * kv_ncap + bt.y) * 2 * H * kv_row_bytes<KvU8>();
    quant_row_u8(tokp + u8_code_off(which, h, H), reinterpret_cast<float2*>(tokp + u8_meta_off(which, h, H)), x, lane);
}

// Cache read-back to fp32 [nb][nt][2][H][D]; rows not on device (paged,
// slot -1) read as NaN.
template <class KV>
__global__ void cache_read_kernel(const CacheView cv, float* __restrict__ out, int H, int b0, int nb, int t0,
                                  int nt) {
    constexpr int D = kHeadDim;
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long total = static_cast<long long>(nb) * nt * 2 * H * D;
    if (i >= total) return;
    const int d = static_cast<int>(i % D);
    const long long r = i / D;  // row over [nb][nt][2][H]
    const int h = static_cast<int>(r % H);
    const int which = static_cast<int>((r / H) % 2);
    const int t = static_cast<int>((r / (2 * H)) % nt);
    const int bb = static_cast<int>(r / (2LL * H * nt));
    int st = t0 + t;
    if (cv.slot) {
        st = cv.slot[static_cast<size_t>(b0 + bb) * cv.Ncap + (t0 + t)];
        if (st < 0) {
            out[i] = __int_as_float(0x7fffffff);
            return;
        }
    }
    const size_t tok = static_cast<size_t>(b0 + bb) * cv.kv_ncap + st;
    if constexpr (KV::QUANT) {
        const uint8_t* tokp = cv.kv + tok * 2 * H * kv_row_bytes<KV>();
        const float2 ms = *reinterpret_cast<const float2*>(tokp + u8_meta_off(which, h, H));
        out[i] = fmaf(ms.x, static_cast<float>(tokp[u8_code_off(which, h, H) + d]), ms.y);
    } else {
        const uint8_t* row = cv.kv + ((tok * 2 + which) * H + h) * static_cast<size_t>(kv_row_bytes<KV>());
        using T = typename KV::T;
        out[i] = to_f(reinterpret_cast<const T*>(row)[d]);
    }
}

// INT8 layer -> fp16 [B][s][2][H][D] (the token-major layout the tensor-core
// prefill's TMA maps read), x = scale * code + bias per (token, K|V, head).
__global__ void dequant_layer_f16_kernel(const uint8_t* __restrict__ kv, __half* __restrict__ out, int H, int Ncap,
                                         int B, int s) {
    constexpr int D = kHeadDim;
    const long long rows = static_cast<long long>(B) * s * 2 * H;
    const long long r = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / (D / 8);
    const int c = static_cast<int>(threadIdx.x % (D / 8)) * 8;  // 8 codes per thread
    if (r >= rows) return;
    const int h = static_cast<int>(r % H);
    const int which = static_cast<int>((r / H) % 2);
    const int t = static_cast<int>((r / (2 * H)) % s);
    const int b = static_cast<int>(r / (2LL * H * s));
    const size_t tok = static_cast<size_t>(b) * Ncap + t;
    const uint8_t* tokp = kv + tok * 2 * H * static_cast<size_t>(kv_row_bytes<KvU8>());
    const float2 ms = *reinterpret_cast<const float2*>(tokp + u8_meta_off(which, h, H));
    const uint2 codes = *reinterpret_cast<const uint2*>(tokp + u8_code_off(which, h, H) + c);
    const uint8_t* cb = reinterpret_cast<const uint8_t*>(&codes);
    __half2 o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        o[i] = __floats2half2_rn(fmaf(ms.x, static_cast<float>(cb[2 * i]), ms.y),
                                 fmaf(ms.x, static_cast<float>(cb[2 * i + 1]), ms.y));
    *reinterpret_cast<uint4*>(out + r * D + c) = *reinterpret_cast<const uint4*>(o);
}

}  // namespace skvd

// ============================================================ launchers
namespace skv_impl {
using namespace skvd;

cudaError_t launch_select(const SelectParams& p, int batch, bool pdl, cudaStream_t st, int layers) {
    const int nc = (p.select && !p.dense && !p.gkeys) ? p.n - p.k : 0;
    const size_t smem = select_smem(nc);
    static std::mutex mu;  // the attribute only grows: concurrent callers stay safe
    static size_t set_smem = 0;
    cudaError_t e = cudaSuccess;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (smem > set_smem) {
            e = cudaFuncSetAttribute(swa_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem));
            if (e != cudaSuccess) return e;
            set_smem = smem;
        }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(batch, layers);
    cfg.blockDim = dim3(kSelectThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, swa_select_kernel, p);
    count_launch();
    return e;
}

cudaError_t launch_scatter_fold(double* imp, long long imp_ld, const float* wpart, int G, int m, const int* tok,
                                long long tok_ld, const double* wsum, int n, double* sparsity, double* rows, int batch,
                                cudaStream_t st) {
    scatter_fold_kernel<<<batch, 256, 0, st>>>(imp, imp_ld, wpart, G, m, tok, tok_ld, wsum, n, sparsity, rows);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_ledger(const LedgerParams& p, int batch, bool pdl, cudaStream_t st) {
    const size_t smem = static_cast<size_t>(p.existing > 0 ? p.existing : 0) * 2 + 16;
    cudaError_t e = cudaFuncSetAttribute(ledger_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(batch);
    cfg.blockDim = dim3(kLedgerThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, ledger_step_kernel, p);
    count_launch();
    return e;
}

cudaError_t launch_move(const MoveParams& p, int batch, int max_tokens, bool pdl, cudaStream_t st) {
    const long long vecs = static_cast<long long>(max_tokens) * (p.tok_bytes / 16);
    const int blocks = static_cast<int>(std::min<long long>((vecs + 255) / 256, 64));
    if (blocks <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks, batch, p.which < 0 ? 2 : 1);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kv_move_kernel, p);
    count_launch();
    return e;
}

cudaError_t launch_transpose_kv_weights(const void* wk, const void* wv, void* bt, int h, cudaStream_t st) {
    if (h % 32) return cudaErrorInvalidValue;
    transpose_kv_weights_kernel<<<dim3(h / 32, h / 32, 2), dim3(32, 8), 0, st>>>(
        static_cast<const uint16_t*>(wk), static_cast<const uint16_t*>(wv), static_cast<uint16_t*>(bt), h);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_top_k(const double* v, int batch, long long ld, int len, int k, int* out,
                         cudaStream_t st) {
    int dev = 0, max_smem = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    const bool long_row = static_cast<size_t>(len) * 8 + 8192 > static_cast<size_t>(max_smem);
    const size_t smem = align_up(sizeof(TopkSmem<kSelThreads>), 16) + (long_row ? 0 : static_cast<size_t>(len) * 8);
    uint64_t* gkeys = nullptr;
    if (long_row) {
        e = cudaMallocAsync(reinterpret_cast<void**>(&gkeys), static_cast<size_t>(batch) * ld * 8, st);
        if (e != cudaSuccess) return e;
    }
    e = cudaFuncSetAttribute(top_k_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    top_k_kernel<<<batch, kSelThreads, smem, st>>>(v, ld, len, k, out, gkeys);
    count_launch();
    e = cudaGetLastError();
    if (gkeys) cudaFreeAsync(gkeys, st);
    return e;
}

cudaError_t launch_quantize(const double* x, long long len, long long cs, uint32_t bits,
                            uint16_t* codes, double* scales, long long* zps, cudaStream_t st) {
    const long long groups = len / cs;
    const int threads = 256;
    const long long blocks = (groups * 32 + threads - 1) / threads;
    quantize_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(x, groups, cs, bits, codes, scales, zps);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_dequantize(const uint16_t* codes, long long len, long long cs, const double* scales,
                              const long long* zps, double* out, cudaStream_t st) {
    const int threads = 256;
    const long long blocks = (len + threads - 1) / threads;
    dequantize_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(codes, len, cs, scales, zps, out);
    count_launch();
    return cudaGetLastError();
}

template <class QT, class KV>
static cudaError_t write_t(const CacheView& cv, double* imp, uint8_t* tiers, const void* k, const void* v, int H,
                           int b0, int nb, int t0, int nt, cudaStream_t st) {
    const long long rows = static_cast<long long>(nb) * nt * 2 * H;
    const int threads = 256;
    const long long blocks = (rows * 32 + threads - 1) / threads;
    cache_write_kernel<QT, KV><<<static_cast<unsigned>(blocks), threads, 0, st>>>(
        cv, imp, tiers, static_cast<const QT*>(k), static_cast<const QT*>(v), H, b0, nb, t0, nt);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_cache_write(int kv_dtype, int q_dtype, const CacheView& cv, double* imp, uint8_t* tiers,
                               const void* k, const void* v, int H, int b0, int nb, int t0, int nt, cudaStream_t st) {
    switch (kv_dtype) {
    case SKV_F32:
        return write_t<float, KvF32>(cv, imp, tiers, k, v, H, b0, nb, t0, nt, st);
    case SKV_F16:
        return write_t<__half, KvF16>(cv, imp, tiers, k, v, H, b0, nb, t0, nt, st);
    case SKV_BF16:
        return write_t<__nv_bfloat16, KvBF16>(cv, imp, tiers, k, v, H, b0, nb, t0, nt, st);
    case SKV_U8:
        if (q_dtype == SKV_F32) return write_t<float, KvU8>(cv, imp, tiers, k, v, H, b0, nb, t0, nt, st);
        if (q_dtype == SKV_F16) return write_t<__half, KvU8>(cv, imp, tiers, k, v, H, b0, nb, t0, nt, st);
        return write_t<__nv_bfloat16, KvU8>(cv, imp, tiers, k, v, H, b0, nb, t0, nt, st);
    }
    return cudaErrorInvalidValue;
}

template <class KV>
static cudaError_t read_t(const CacheView& cv, float* out, int H, int b0, int nb, int t0, int nt, cudaStream_t st) {
    const long long total = static_cast<long long>(nb) * nt * 2 * H * kHeadDim;
    const int threads = 256;
    cache_read_kernel<KV><<<static_cast<unsigned>((total + threads - 1) / threads), threads, 0, st>>>(
        cv, out, H, b0, nb, t0, nt);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_cache_read(int kv_dtype, const CacheView& cv, float* out, int H, int b0, int nb, int t0, int nt,
                              cudaStream_t st) {
    switch (kv_dtype) {
    case SKV_F32: return read_t<KvF32>(cv, out, H, b0, nb, t0, nt, st);
    case SKV_F16: return read_t<KvF16>(cv, out, H, b0, nb, t0, nt, st);
    case SKV_BF16: return read_t<KvBF16>(cv, out, H, b0, nb, t0, nt, st);
    case SKV_U8: return read_t<KvU8>(cv, out, H, b0, nb, t0, nt, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_quant_scatter(int q_dtype, const float* C, const int* m_dev, int m_cap, const int2* rowmap,
                                 uint8_t* kv, int H, int kv_ncap, cudaStream_t st) {
    const long long warps = static_cast<long long>(m_cap) * 2 * H;
    const unsigned blocks = static_cast<unsigned>((warps * 32 + 255) / 256);
    if (q_dtype == SKV_F16)
        quant_scatter_kernel<__half><<<blocks, 256, 0, st>>>(C, m_dev, rowmap, kv, H, kv_ncap);
    else if (q_dtype == SKV_BF16)
        quant_scatter_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(C, m_dev, rowmap, kv, H, kv_ncap);
    else
        quant_scatter_kernel<float><<<blocks, 256, 0, st>>>(C, m_dev, rowmap, kv, H, kv_ncap);
    count_launch();
    return cudaGetLastError();
}

}  // namespace skv_impl

#ifdef SKV_SELECT_TRACE
extern "C" int skv_debug_select_trace(long long* out) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, skvd::g_sel_trace, sizeof(long long) * 16));
}
#endif

namespace skv_impl {
cudaError_t launch_dequant_layer_f16(const uint8_t* kv, void* out, int H, int Ncap, int B, int s, cudaStream_t st) {
    const long long threads = static_cast<long long>(B) * s * 2 * H * (skvd::kHeadDim / 8);
    skvd::dequant_layer_f16_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(
        kv, static_cast<__half*>(out), H, Ncap, B, s);
    count_launch();
    return cudaGetLastError();
}
}  // namespace skv_impl
