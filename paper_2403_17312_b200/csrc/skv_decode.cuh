// skv_decode.cuh -- the SWA decode attend kernel (one launch per layer-step).
//
// One CTA per (head group g, sequence b) gathers the selected tokens' K/V rows
// for its HG heads and computes, for each head:
//   logits = (q . K[t]) / sqrt(D); w = softmax(logits); attn = sum_t w_t V[t]
// -- attend_over_indices (attention.hpp:183-231) -- plus, in decode mode, the
// step's append of the new K/V row (AttentionState::append_token with the
// engine's fake-quant, attention.hpp:65-74, engine.hpp:469-483). The head-group
// sum of the weights per selected token goes to a small scratch buffer; the
// per-sequence select kernel (skv_select.cuh) folds it into the fp64
// importance and selects the next step's tokens.
//
// Data movement: a dedicated producer warp gathers token rows (HG*D contiguous
// elements of one token, token-major cache) with cp.async.bulk into an
// S-stage shared-memory ring guarded by mbarriers. 8 consumer warps read
// 128-bit vectors from shared memory; each lane owns RS rows of a stage, dots
// them with packed FFMA2 and reduces RS rows at once with a transposed
// butterfly (log2(LR)+RS-1 shuffles instead of RS*log2(LR)). K rows of every
// selected token stream first (pass 1), V rows second (pass 2): the exact
// softmax normaliser of the reference is known before any V is weighted, and
// the ring keeps HBM busy across the softmax in between.
#pragma once

#include <type_traits>

#include "skv_device.cuh"
#include "skv_ledger.cuh"
#include "skv_select.cuh"

#ifndef SKV_STAGE_BYTES
#define SKV_STAGE_BYTES 16384
#endif
#ifndef SKV_STAGES
#define SKV_STAGES 4
#endif

namespace skvd {

constexpr int kHeadDim = 128;
constexpr int kConsumerWarps = 8;
constexpr int kConsumerThreads = kConsumerWarps * 32;
// Bulk-copy issue is serial per warp (ELECT + R2UR + UBLKCP per copy), so the
// gather is issued by one producer warp per SM sub-partition.
constexpr int kProducerWarps = 4;
constexpr int kDecodeThreads = kConsumerThreads + kProducerWarps * 32;
constexpr int kBarConsumers = 1;  // named barrier: consumer warps only
constexpr int kBarAppend = 2;     // named barrier: consumers arrive, producer syncs

// Bytes of one stored head row: D elements, plus the inline (scale, bias)
// pair for INT8 rows.
template <class KV>
__host__ __device__ constexpr int kv_row_bytes() {
    return kHeadDim * KV::E + (KV::QUANT ? 8 : 0);
}

struct AttendParams {
    const uint8_t* kv;   // layer base [B][Ncap][2][H] rows of ROWE bytes (D elements [+ meta])
    uint8_t* kv_w;       // same storage (the append)
    const void* q;       // [B][H][D] compute dtype
    const void* k_new;   // [B][H][D] (append mode)
    const void* v_new;   // [B][H][D]
    void* out;           // [B][H][D] compute dtype or fp32
    const int* tok;      // [B][tok_ld] ascending token ids; nullptr = dense 0..m-1
    long long tok_ld;
    int* idx_out;        // optional [B][m]
    float* w_out;        // optional [B][H][m]
    float* wpart;        // [B][G][m]: sum over the CTA's heads of w, per position
    int B, H, Ncap, n, m;
    int append, out_f32, pdl_wait;  // pdl_wait: 1 before q / new rows, 2 at entry
    float scale;
    // Tail (fold != 0): the last CTA of each sequence folds the head-group
    // weight partials into the fp64 importance and selects the next step
    // (fold_and_select, skv_select.cuh) -- no separate select launch.
    int fold;
    unsigned* counters;  // [B], zero between launches
    // Long selections: the token list and the logits / weights live in global
    // scratch instead of shared memory ([B][G][Ncap] ids, [B][G][HG][Ncap] f32)
    int* gtok;
    float* gwts;
    // Paged store: token -> slot map of this layer ([B][Ncap], -1: not on
    // device) and the slot stride of kv; nullptr: kv is token-indexed.
    const int* slots;
    int kv_ncap;
    // Residency check (engine.hpp:625-628): with a plan attached, every
    // gathered token must be device-resident (tiers [B][Ncap] of this layer);
    // a violation is reported through status.
    const uint8_t* tiers;
    DevStatus* status;
    int layer;
    SelectParams sel;    // imp / wpart / apply / cur_tok / sparsity / next selection; tok_prev = this CTA's list
};

template <class KV, int HG>
struct DecodeCfg {
    static constexpr int D = kHeadDim;
    static constexpr int E = KV::E;
    static constexpr bool QUANT = KV::QUANT;
    static constexpr int VE = 16 / E;    // elements per 16-byte vector
    static constexpr int V2 = VE / 2;    // float2 pairs per vector
    static constexpr int LR = D / VE;    // lanes per head row
    static constexpr int RPW = 32 / LR;  // row groups per warp
    static constexpr int SLOTS = kConsumerWarps * RPW;
    static constexpr int META = QUANT ? 8 : 0;  // INT8 rows carry (scale, bias) inline
    static constexpr int ROWE = D * E + META;   // bytes per head row
    static constexpr int ROWB = HG * ROWE;
    static constexpr int TMIN = SLOTS / HG > 0 ? SLOTS / HG : 1;  // tokens per stage for RS = 1
    static constexpr int T0 = SKV_STAGE_BYTES / ROWB > 32 ? 32 : SKV_STAGE_BYTES / ROWB;
    static constexpr int T = ((T0 < TMIN ? TMIN : T0) + TMIN - 1) / TMIN * TMIN;
    static constexpr int RS = T * HG / SLOTS;  // rows per slot per stage
    // fp32 rows at 1-2 heads per CTA are the small-grid latency case (config
    // 1: b = 1, 32 CTAs on 148 SMs): a ring twice as deep keeps a whole K pass
    // (and the first V chunks) in flight instead of two round trips.
    static constexpr int S = (E == 4 && !QUANT && HG <= 2) ? 2 * SKV_STAGES : SKV_STAGES;
    // Ring stride of one token's rows. A whole INT8 block (HG = 8) is padded
    // by 96 bytes to a stride = 32 mod 128: the (scale, bias) pairs of four
    // consecutive tokens x four heads, read once per row by a warp, then fall
    // in 16 distinct bank pairs (with 1088 they met in the same banks).
    static constexpr int TS = (QUANT && HG == kU8Group) ? ROWB + 96 : ROWB;
    // INT8 8-head groups give each lane slot RS CONSECUTIVE tokens (others:
    // tokens SLOTS / HG apart), so those metadata reads spread over the banks
    static constexpr bool TOK_ROWS = QUANT && HG == kU8Group;
    static constexpr int STAGEB = T * TS;
    static_assert(SLOTS % HG == 0, "head group must tile the consumer slots");
    static_assert(T * HG % SLOTS == 0 && RS >= 1 && RS <= LR, "stage rows must tile the slots");
    static_assert(T <= 32, "one producer lane per token row");
    static_assert(!QUANT || (HG % 2 == 0 && kU8Group % HG == 0),
                  "INT8 head groups split the 8-head storage blocks into 16-byte sized copies");
    // reduction scratch: per slot, each lane's VE partial sums padded to VE + 1
    // floats, so a warp's stores hit 32 distinct banks
    static constexpr int RED_SP = LR * (VE + 1);
    static_assert(SLOTS * RED_SP * 4 <= S * STAGEB, "reduction scratch aliases the ring");
};

struct DecodeSmem {
    size_t ring, bars, tok, slot, wts, topk, scratch, flag, total;
};

// Shared-memory carve-up; identical on host (launch size) and device. gmem:
// the token list and the weights are in global scratch (long selections).
template <class KV, int HG>
__host__ __device__ inline DecodeSmem decode_smem(int m, bool gmem = false, bool paged = false) {
    if (gmem) m = 0;
    using C = DecodeCfg<KV, HG>;
    DecodeSmem s;
    size_t o = 0;
    s.ring = o;
    o = align_up(o + static_cast<size_t>(C::S) * C::STAGEB, 16);
    s.bars = o;
    o += 2 * C::S * 8;
    s.tok = o;
    o = align_up(o + static_cast<size_t>(m) * 4, 16);
    s.slot = o;  // paged: the selected tokens' slots
    o = align_up(o + (paged ? static_cast<size_t>(m) * 4 : 0), 16);
    s.wts = o;  // logits, then weights [HG][m] f32
    o = align_up(o + static_cast<size_t>(HG) * m * 4, 16);
    s.topk = o;
    o = align_up(o + sizeof(TopkSmem<kConsumerThreads>), 16);
    s.scratch = o;
    o = align_up(o + sizeof(SelectScratch<kConsumerThreads>), 16);
    s.flag = o;
    o += 16;
    s.total = o;
    return s;
}

// Reduce RS per-row partial sums across the LR lanes of a row group. Returns
// the full sum of row `row` (same value in every lane sharing the high bits);
// the first RS levels are transposed so each shuffle moves half the rows.
template <int RS, int LR>
__device__ __forceinline__ float reduce_rows(float (&v)[RS], int c, int& row) {
    row = 0;
    int cnt = RS;
#pragma unroll
    for (int o = LR / 2; o >= 1; o >>= 1) {
        if (cnt > 1) {
            const int half = cnt / 2;
            const bool up = (c & o) != 0;
#pragma unroll
            for (int i = 0; i < RS / 2; ++i) {
                if (i < half) {
                    const float send = up ? v[i] : v[i + half];
                    const float keep = up ? v[i + half] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            if (up) row += half;
            cnt = half;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
    return v[0];
}

// CTAs per SM the register budget must allow (ptxas otherwise picked
// budgets that spilled): 3 for 16-bit rows, 2 for fp32 and INT8 rows.
template <class KV>
constexpr int attend_min_blocks() {
    // fp32 rows (config 1, the latency-bound parity case) need no third CTA per SM
    return (KV::QUANT || KV::E == 4) ? 2 : 3;
}

template <class KV, class QT, int HG>
__global__ void __launch_bounds__(kDecodeThreads, attend_min_blocks<KV>())
    swa_attend_kernel(const AttendParams p) {
    using C = DecodeCfg<KV, HG>;
    constexpr int D = C::D, VE = C::VE, V2 = C::V2, LR = C::LR, RPW = C::RPW, SLOTS = C::SLOTS;
    constexpr int ROWE = C::ROWE, ROWB = C::ROWB, T = C::T, S = C::S, RS = C::RS;
    constexpr int STAGEB = C::STAGEB;
    constexpr bool QUANT = C::QUANT;

    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = blockIdx.x, b = blockIdx.y, G = gridDim.x;
    const int H = p.H, n = p.n, m = p.m;
    const bool gmem = p.gtok != nullptr;
    const bool paged = p.slots != nullptr;
    const DecodeSmem L = decode_smem<KV, HG>(m, gmem, paged);

    uint8_t* ring = smem + L.ring;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + S;
    int* tok = gmem ? p.gtok + (static_cast<size_t>(b) * gridDim.x + g) * p.Ncap
                    : reinterpret_cast<int*>(smem + L.tok);
    float* wts = gmem ? p.gwts + (static_cast<size_t>(b) * gridDim.x + g) * HG * p.Ncap
                      : reinterpret_cast<float*>(smem + L.wts);  // [HG][m]

    // pdl_wait == 2: a PDL launch that reads its predecessor's outputs from
    // the start (per-layer steps, skv_capi.cu launch_attend_c): wait first,
    // so a kernel launched behind this one never overtakes that predecessor.
    if (p.pdl_wait == 2) pdl_wait();
    // Let the next kernel in the stream (the select kernel) get scheduled now;
    // it waits for this grid's completion before touching our outputs.
    pdl_launch_dependents();
#ifdef SKV_DECODE_TRACE
    if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) dtr[0] = gtimer();
#endif

    const size_t TOKB = static_cast<size_t>(2) * H * ROWE;  // bytes per token (K and V planes)
    // this sequence's token rows; a token holds K then V, H heads each
    // (INT8: blocks of 8 heads, codes then (scale, bias), see u8_code_off)
    const uint8_t* kvb = p.kv + static_cast<size_t>(b) * p.kv_ncap * TOKB;
    const int* slot_row = paged ? p.slots + static_cast<size_t>(b) * p.Ncap : nullptr;
    // smem slot list (paged, shared-memory token list); long selections look slots up in the producer
    int* tslot = (paged && !gmem) ? reinterpret_cast<int*>(smem + L.slot) : nullptr;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], kProducerWarps);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_barrier_init();
    }
    {
        const int* src = p.tok ? p.tok + static_cast<size_t>(b) * p.tok_ld : nullptr;
        const uint8_t* trow = p.tiers ? p.tiers + static_cast<size_t>(b) * p.Ncap : nullptr;
        for (int i = tid; i < m; i += kDecodeThreads) {
            const int t = src ? src[i] : i;
            tok[i] = t;
            const bool cur = p.append && i == m - 1;  // the appended token: stored by this kernel
            if (trow && !cur && trow[t] != kTierDevice && g == 0)
                report_status(p.status, 1, p.layer, b, t, -1, 0ull, 0ull);  // engine.hpp:625-628
            if (tslot) {
                int sl = slot_row[t];
                if (sl < 0) {
                    if (g == 0) report_status(p.status, 1, p.layer, b, t, -1, 0ull, 0ull);
                    sl = 0;
                }
                tslot[i] = sl;
            }
        }
    }
    __syncthreads();

    const int nchunks = (m + T - 1) / T;

    if (warp >= kConsumerWarps) {
        // ================================================= producer warps
        // Producer warp pw issues the rows i = pw, pw + P, ... of every stage
        // and posts its own byte count on the stage's full barrier.
        const int pw = warp - kConsumerWarps;
        const uint64_t pol = policy_evict_first();
        // The appended token (position m-1) is copied from the step's input row
        // (non-quantized storage) or, once the consumers have stored its codes,
        // from the cache (quantized storage).
        const uint8_t* knew = static_cast<const uint8_t*>(p.k_new) +
                              (static_cast<size_t>(b) * H + g * HG) * ROWE;
        const uint8_t* vnew = static_cast<const uint8_t*>(p.v_new) +
                              (static_cast<size_t>(b) * H + g * HG) * ROWE;
        // per-token offsets of this head group's K and V rows (INT8: codes, then (scale, bias))
        const uint32_t off_k = QUANT ? static_cast<uint32_t>(u8_code_off(0, g * HG, H))
                                     : static_cast<uint32_t>(g * HG * ROWE);
        const uint32_t off_v = QUANT ? static_cast<uint32_t>(u8_code_off(1, g * HG, H))
                                     : static_cast<uint32_t>((H + g * HG) * ROWE);
        const uint32_t moff_k = QUANT ? static_cast<uint32_t>(u8_meta_off(0, g * HG, H)) : 0u;
        const uint32_t moff_v = QUANT ? static_cast<uint32_t>(u8_meta_off(1, g * HG, H)) : 0u;
        bool synced = !p.append;
        for (int u = 0; u < 2 * nchunks; ++u) {
            const int vsel = u >= nchunks;
            const int base = (vsel ? u - nchunks : u) * T;
            const int cnt = min(T, m - base);
            const int stage = u % S;
            if (u >= S) mbar_wait(&empty[stage], ((u / S) - 1) & 1);
            const bool has_cur = p.append && base + cnt == m;
            if (has_cur && !synced) {
                if (QUANT) named_sync(kBarAppend, kDecodeThreads);
                else if (p.pdl_wait) pdl_wait();
                synced = true;
            }
            const int mine = cnt > pw ? (cnt - pw + kProducerWarps - 1) / kProducerWarps : 0;
            if (lane == 0) mbar_arrive_expect_tx(&full[stage], mine * ROWB);
            __syncwarp();
            if (lane < mine) {
                const int i = pw + lane * kProducerWarps;
                int t = tslot ? tslot[base + i] : tok[base + i];
                if (paged && !tslot) t = max(slot_row[t], 0);
                const uint8_t* tb = kvb + static_cast<size_t>(t) * TOKB;
                uint8_t* dst = ring + stage * STAGEB + i * C::TS;
                const uint8_t* src = tb + (vsel ? off_v : off_k);
                if constexpr (QUANT) {
                    if constexpr (HG == kU8Group) {  // codes + (scale, bias) of the block: one copy
                        bulk_g2s(dst, src, ROWB, &full[stage], pol);
                    } else {  // part of a block: codes, then their (scale, bias) pairs
                        bulk_g2s(dst, src, HG * D, &full[stage], pol);
                        bulk_g2s(dst + HG * D, tb + (vsel ? moff_v : moff_k), HG * 8, &full[stage], pol);
                    }
                } else {
                    if (has_cur && i == cnt - 1) src = vsel ? vnew : knew;
                    bulk_g2s(dst, src, ROWB, &full[stage], pol);
                }
            }
        }
        return;
    }

    // ====================================================== consumer warps
    const int ctid = tid;
    if (p.pdl_wait) pdl_wait();  // q / new rows may come from the previous kernel

    // ---- append the step's new K/V rows for this head group (token n-1)
    if (p.append) {
        const int cur_slot = paged ? max(slot_row[n - 1], 0) : n - 1;
        const size_t tok_base = (static_cast<size_t>(b) * p.kv_ncap + cur_slot) * TOKB;
        const size_t tok_off = tok_base + static_cast<size_t>(g) * ROWB;  // non-quantized rows of the group
        if constexpr (!QUANT) {
            constexpr int VPR = ROWB / 16;  // compute dtype == storage dtype
            for (int i = ctid; i < 2 * VPR; i += kConsumerThreads) {
                const int kv = i / VPR, j = i % VPR;
                const uint8_t* srcb = static_cast<const uint8_t*>(kv ? p.v_new : p.k_new) +
                                      (static_cast<size_t>(b) * H + g * HG) * ROWE;
                reinterpret_cast<uint4*>(p.kv_w + tok_off + kv * H * ROWE)[j] =
                    reinterpret_cast<const uint4*>(srcb)[j];
            }
        } else {
            // quant.hpp:43-81 per (token, head) group of D values, in fp64.
            for (int grp = warp; grp < 2 * HG; grp += kConsumerWarps) {
                const int kv = grp / HG, h = grp % HG;
                const QT* src = static_cast<const QT*>(kv ? p.v_new : p.k_new) +
                                (static_cast<size_t>(b) * H + g * HG + h) * D;
                double x[D / 32];
#pragma unroll
                for (int i = 0; i < D / 32; ++i) x[i] = static_cast<double>(to_f(src[lane * (D / 32) + i]));
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
                uint8_t* row = p.kv_w + tok_base + u8_code_off(kv, g * HG + h, H);
                reinterpret_cast<uint32_t*>(row)[lane] = packed;
                if (lane == 0)
                    *reinterpret_cast<float2*>(p.kv_w + tok_base + u8_meta_off(kv, g * HG + h, H)) =
                        make_float2(static_cast<float>(scale), static_cast<float>(-scale * static_cast<double>(zp)));
            }
            fence_global_to_async();
            named_arrive(kBarAppend, kDecodeThreads);
        }
    }

    // ---- per-lane query slice (row group `slot` always sees head h)
    const int slot = warp * RPW + lane / LR;
    const int h = slot % HG;
    const int c = lane % LR;
    float2 q2[V2];
    // INT8 codes against an fp16 query: the logit dot runs on FHFMA over the
    // packed query halves (dot_u8_f16)
    constexpr bool kFh = QUANT && std::is_same<QT, __half>::value;
    uint32_t qh[kFh ? 8 : 1];
    {
        const QT* qrow = static_cast<const QT*>(p.q) + (static_cast<size_t>(b) * H + g * HG + h) * D + c * VE;
#pragma unroll
        for (int i = 0; i < V2; ++i) q2[i] = make_float2(to_f(qrow[2 * i]), to_f(qrow[2 * i + 1]));
        if constexpr (kFh) {
            const uint4 a = reinterpret_cast<const uint4*>(qrow)[0], bq = reinterpret_cast<const uint4*>(qrow)[1];
            qh[0] = a.x, qh[1] = a.y, qh[2] = a.z, qh[3] = a.w;
            qh[4] = bq.x, qh[5] = bq.y, qh[6] = bq.z, qh[7] = bq.w;
        }
    }
    float qsum = 0.f;
    if constexpr (QUANT) {
#pragma unroll
        for (int i = 0; i < V2; ++i) qsum += q2[i].x + q2[i].y;
#pragma unroll
        for (int off = LR / 2; off > 0; off >>= 1) qsum += __shfl_xor_sync(0xffffffffu, qsum, off);
    }
    // A lane's row i of a stage is (token row_tok(i), head h): rows SLOTS
    // apart (token (slot + i SLOTS) / HG), or for INT8 8-head groups RS
    // consecutive tokens. INT8 rows sit at 128-byte strides inside their
    // token's block, the (scale, bias) pairs after them.
    constexpr int TS = C::TS;
    const int tok0 = C::TOK_ROWS ? (slot / HG) * RS : 0;
    auto row_tok = [&](int i) { return C::TOK_ROWS ? tok0 + i : (slot + i * SLOTS) / HG; };
    const uint32_t lane_off =
        QUANT ? static_cast<uint32_t>((C::TOK_ROWS ? tok0 : slot / HG) * TS + (slot % HG) * D + c * 16)
              : static_cast<uint32_t>(slot * ROWE + c * 16);
    constexpr int RSTRIDE = C::TOK_ROWS ? TS : (QUANT ? (SLOTS / HG) * TS : SLOTS * ROWE);
    auto meta_of = [&](const uint8_t* stage_base, int t) {  // (scale, bias) of token t, head h
        return *reinterpret_cast<const float2*>(stage_base + t * TS + HG * D + h * 8);
    };
    const float scale = p.scale;
    // 16-byte vector at q (16-byte aligned for every storage type)
    auto ld16 = [](const uint8_t* q) -> uint4 { return *reinterpret_cast<const uint4*>(q); };

    DTR(1);  // consumers: token list, append and q done
    // ---- pass 1: logits = (q . k) * scale  (attention.hpp:204-212)
    for (int u = 0; u < nchunks; ++u) {
        const int stage = u % S;
        mbar_wait(&full[stage], (u / S) & 1);
        const int base = u * T;
        const int cnt = min(T, m - base);  // tokens copied this round
        const uint8_t* st = ring + stage * STAGEB + lane_off;
        uint4 raw[RS];
        if (cnt == T) {
#pragma unroll
            for (int i = 0; i < RS; ++i) raw[i] = ld16(st + i * RSTRIDE);
        } else {  // last chunk: rows past it were not copied this round
#pragma unroll
            for (int i = 0; i < RS; ++i)
                raw[i] = row_tok(i) < cnt ? ld16(st + i * RSTRIDE) : make_uint4(0u, 0u, 0u, 0u);
        }
        float part[RS];
#pragma unroll
        for (int i = 0; i < RS; ++i) {
            if constexpr (kFh) {
                part[i] = dot_u8_f16(raw[i], qh);  // biased codes, like cvt16x2 (KvU8)
            } else {
                float2 kf[V2];
                cvt16x2(raw[i], kf, KV{});
                float2 a = __fmul2_rn(q2[0], kf[0]);
#pragma unroll
                for (int j = 1; j < V2; ++j) a = __ffma2_rn(q2[j], kf[j], a);
                part[i] = a.x + a.y;
            }
        }
        int rsel;
        const float dot = reduce_rows<RS, LR>(part, c, rsel);
        const int t = row_tok(rsel);
        if ((c & (LR / RS - 1)) == 0 && t < cnt) {
            float logit;
            if constexpr (QUANT) {
                const float2 ms = meta_of(ring + stage * STAGEB, t);
                // codes arrive as 1024 + c (cvt16x2, KvU8): dot = q.c + 1024 * sum(q)
                logit = fmaf(ms.x, dot, fmaf(-kBiasU8, ms.x, ms.y) * qsum) * scale;
            } else {
                logit = dot * scale;
            }
            wts[h * m + base + t] = logit;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
    }
    named_sync(kBarConsumers, kConsumerThreads);

    DTR(2);
    // ---- softmax with the reference's normaliser (attention.hpp:213-218)
    if constexpr (HG < kConsumerWarps) {
        // fewer heads than warps (fp32 / bf16 groups): WPH warps share a head's
        // row, max and sum combined through shared memory (the select scratch,
        // idle until the tail) -- config 1 ran this on one warp of eight
        constexpr int WPH = kConsumerWarps / HG;
        float* sred = reinterpret_cast<float*>(smem + L.scratch);  // [2][kConsumerWarps]
        const int hh = warp / WPH, part = warp % WPH;
        float* wl = wts + hh * m;
        const int i0 = part * 32 + lane;
        float mx = -INFINITY;
        for (int i = i0; i < m; i += WPH * 32) mx = fmaxf(mx, wl[i]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (lane == 0) sred[warp] = mx;
        named_sync(kBarConsumers, kConsumerThreads);
        mx = sred[hh * WPH];
#pragma unroll
        for (int j = 1; j < WPH; ++j) mx = fmaxf(mx, sred[hh * WPH + j]);
        float sum = 0.f;
        for (int i = i0; i < m; i += WPH * 32) {
            const float e = expf(wl[i] - mx);
            wl[i] = e;
            sum += e;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        if (lane == 0) sred[kConsumerWarps + warp] = sum;
        named_sync(kBarConsumers, kConsumerThreads);
        sum = 0.f;
#pragma unroll
        for (int j = 0; j < WPH; ++j) sum += sred[kConsumerWarps + hh * WPH + j];
        const float inv = 1.0f / sum;
        for (int i = i0; i < m; i += WPH * 32) wl[i] *= inv;
    }
    for (int hh = warp; hh < HG && HG >= kConsumerWarps; hh += kConsumerWarps) {
        float* wl = wts + hh * m;
        float mx = -INFINITY;
        for (int i = lane; i < m; i += 32) mx = fmaxf(mx, wl[i]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        float sum = 0.f;
        for (int i = lane; i < m; i += 32) {
            const float e = expf(wl[i] - mx);
            wl[i] = e;
            sum += e;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        const float inv = 1.0f / sum;
        for (int i = lane; i < m; i += 32) wl[i] *= inv;
    }
    named_sync(kBarConsumers, kConsumerThreads);

    DTR(3);
    // ---- head-group partial of the importance update (+ optional outputs)
    {
        float* wp = p.wpart + (static_cast<size_t>(b) * G + g) * m;
        for (int pos = ctid; pos < m; pos += kConsumerThreads) {
            float s = 0.f;
#pragma unroll
            for (int hh = 0; hh < HG; ++hh) s += wts[hh * m + pos];
            wp[pos] = s;
        }
        if (p.idx_out != nullptr && g == 0)
            for (int pos = ctid; pos < m; pos += kConsumerThreads) p.idx_out[static_cast<size_t>(b) * m + pos] = tok[pos];
        if (p.w_out != nullptr)
            for (int i = ctid; i < HG * m; i += kConsumerThreads)
                p.w_out[(static_cast<size_t>(b) * H + g * HG) * m + i] = wts[i];
    }

    DTR(4);
    // ---- pass 2: attn = sum_t w_t * V[t]  (attention.hpp:219-225)
    float2 acc[V2];
#pragma unroll
    for (int i = 0; i < V2; ++i) acc[i] = make_float2(0.f, 0.f);
    float bsum = 0.f;
    const float* wh = wts + h * m;
    for (int u = nchunks; u < 2 * nchunks; ++u) {
        const int stage = u % S;
        mbar_wait(&full[stage], (u / S) & 1);
        const int base = (u - nchunks) * T;
        const int cnt = min(T, m - base);
        const uint8_t* st = ring + stage * STAGEB + lane_off;
        if (cnt == T) {
            uint4 raw[RS];
#pragma unroll
            for (int i = 0; i < RS; ++i) raw[i] = ld16(st + i * RSTRIDE);
#pragma unroll
            for (int i = 0; i < RS; ++i) {
                const int t = row_tok(i);
                const float w = wh[base + t];
                float2 vf[V2];
                cvt16x2(raw[i], vf, KV{});
                if constexpr (QUANT) {
                    const float2 ms = meta_of(ring + stage * STAGEB, t);
                    const float a = w * ms.x;
                    const float2 a2 = make_float2(a, a);
#pragma unroll
                    for (int j = 0; j < V2; ++j) acc[j] = __ffma2_rn(a2, vf[j], acc[j]);
                    bsum = fmaf(w, fmaf(-kBiasU8, ms.x, ms.y), bsum);  // biased codes
                } else {
                    const float2 w2 = make_float2(w, w);
#pragma unroll
                    for (int j = 0; j < V2; ++j) acc[j] = __ffma2_rn(w2, vf[j], acc[j]);
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < RS; ++i) {
                const int t = row_tok(i);
                if (t < cnt) {
                    const float w = wh[base + t];
                    float2 vf[V2];
                    cvt16x2(ld16(st + i * RSTRIDE), vf, KV{});
                    if constexpr (QUANT) {
                        const float2 ms = meta_of(ring + stage * STAGEB, t);
                        const float a = w * ms.x;
                        const float2 a2 = make_float2(a, a);
#pragma unroll
                        for (int j = 0; j < V2; ++j) acc[j] = __ffma2_rn(a2, vf[j], acc[j]);
                        bsum = fmaf(w, fmaf(-kBiasU8, ms.x, ms.y), bsum);  // biased codes
                    } else {
                        const float2 w2 = make_float2(w, w);
#pragma unroll
                        for (int j = 0; j < V2; ++j) acc[j] = __ffma2_rn(w2, vf[j], acc[j]);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
    }
    // all stages consumed, no copy in flight: the ring is free scratch now
    named_sync(kBarConsumers, kConsumerThreads);
    float* red = reinterpret_cast<float*>(ring);  // [SLOTS][LR][VE + 1]
    constexpr int SP = C::RED_SP;
#pragma unroll
    for (int i = 0; i < V2; ++i) {
        red[slot * SP + c * (VE + 1) + 2 * i] = acc[i].x + bsum;
        red[slot * SP + c * (VE + 1) + 2 * i + 1] = acc[i].y + bsum;
    }
    named_sync(kBarConsumers, kConsumerThreads);
    for (int o = ctid; o < HG * D; o += kConsumerThreads) {
        const int hh = o / D, d = o % D;
        const int cell = (d / VE) * (VE + 1) + d % VE;
        float s = 0.f;
#pragma unroll
        for (int sl = 0; sl < SLOTS / HG; ++sl) s += red[(sl * HG + hh) * SP + cell];
        const size_t at = (static_cast<size_t>(b) * H + g * HG + hh) * D + d;
        if (p.out_f32)
            static_cast<float*>(p.out)[at] = s;
        else
            static_cast<QT*>(p.out)[at] = from_f<QT>(s);
    }

    DTR(5);
    // ---- tail: the last CTA of the sequence folds the G partials (fixed
    // group order, deterministic) into the importance and selects the next
    // step's tokens, while the other sequences' CTAs keep streaming.
    if (p.fold) {
        int* s_last = reinterpret_cast<int*>(smem + L.flag);
        named_sync(kBarConsumers, kConsumerThreads);  // ring free: it becomes the key buffer
        if (ctid == 0) {
            __threadfence();
            const unsigned prev = atomicAdd(&p.counters[b], 1u);
            *s_last = (prev == static_cast<unsigned>(G - 1)) ? 1 : 0;
        }
        named_sync(kBarConsumers, kConsumerThreads);
        if (*s_last) {
            __threadfence();
            SelectParams sp = p.sel;
            sp.tok_prev = tok;  // this CTA's (shared) token list, same for every group
            sp.tok_prev_ld = 0;
            DTR_TAIL(6);
            fold_and_select<kConsumerThreads, kBarConsumers, (KV::E == 4 && !KV::QUANT)>(
                sp, b, ctid, *reinterpret_cast<TopkSmem<kConsumerThreads>*>(smem + L.topk),
                reinterpret_cast<uint64_t*>(ring), *reinterpret_cast<SelectScratch<kConsumerThreads>*>(smem + L.scratch));
            if (ctid == 0) p.counters[b] = 0;
#ifdef SKV_DECODE_TRACE
            if (ctid == 0 && p.n % 50 == 0) {
                const unsigned long long t = gtimer();
                printf("DTR n=%d: cta0 start->q %llu, pass1 %llu, softmax %llu, wpart %llu, pass2+out %llu | "
                       "tail wait %llu, fold %llu (loads %llu, adds %llu, sparsity %llu), keys %llu, topk %llu ns; "
                       "total %llu\n", p.n, dtr[1] - dtr[0],
                       dtr[2] - dtr[1], dtr[3] - dtr[2], dtr[4] - dtr[3], dtr[5] - dtr[4], dtr[6] - dtr[5],
                       dtr[7] - dtr[6], dtr[9] - dtr[6], dtr[10] - dtr[9], dtr[7] - dtr[10], dtr[8] - dtr[7],
                       t - dtr[8], t - dtr[0]);
            }
#endif
        }
    }
}

}  // namespace skvd
