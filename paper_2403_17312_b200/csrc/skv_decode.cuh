// skv_decode.cuh -- the fused SWA decode kernel (one launch per layer-step).
//
// One CTA per (head group g, sequence b). It replaces, for its HG heads:
//   * AttentionState::append_token + head_rows fake-quant (attention.hpp:65-74,
//     engine.hpp:469-483): the step's new K/V row is (quantized and) stored;
//   * swa_select / top_k_indices (attention.hpp:142-171, matrix.hpp:162-176):
//     every CTA of a sequence runs the same exact fp64 top-k on the
//     head-summed importance while the local window is already streaming in;
//   * attend_over_indices (attention.hpp:183-231): gathered QK^T, exact
//     softmax with the reference's normaliser, PV;
//   * the accumulator update acc[idx] += w (attention.hpp:219-227), reduced
//     over heads in a fixed order by the last CTA of the sequence.
//
// Data movement: a dedicated producer warp gathers selected token rows
// (HG*D contiguous elements of one token, token-major cache) with
// cp.async.bulk into an S-stage shared-memory ring guarded by mbarriers; 8
// consumer warps read 128-bit vectors from shared memory and reduce with warp
// shuffles. K rows of every selected token stream first (pass 1), V rows
// second (pass 2); the ring keeps HBM busy across the softmax in between.
#pragma once

#include "skv_device.cuh"
#include "skv_topk.cuh"

namespace skvd {

constexpr int kHeadDim = 128;
constexpr int kConsumerWarps = 8;
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kDecodeThreads = kConsumerThreads + 32;
constexpr int kBarConsumers = 1;  // named barrier: consumer warps only
constexpr int kBarSelect = 2;     // named barrier: consumers arrive, producer syncs

enum DecodeMode : int {
    kModeSwaStep = 0,   // append + in-kernel selection (dense when 2k >= n)
    kModeExplicit = 1,  // caller-provided ascending indices, importance +=
    kModeSeed = 2,      // dense over [0, n), importance = (prefill seeding)
};

struct DecodeParams {
    const uint8_t* kv;   // layer base [B][Ncap][2][H][D] elements of KV::T
    uint8_t* kv_w;       // same storage, for the append
    const float2* meta;  // layer base [B][Ncap][2][H] (scale, bias) when quantized
    float2* meta_w;
    double* imp;         // layer base [B][Ncap] head-summed importance
    const void* q;       // [B][H][D] compute dtype
    const void* k_new;   // [B][H][D]
    const void* v_new;   // [B][H][D]
    void* out;           // [B][H][D]
    const int* idx_in;   // kModeExplicit: [B][m] ascending
    int* idx_out;        // optional [B][m], ascending
    float* w_out;        // optional [B][H][m], softmax weights in ascending order
    float* wpart;        // scratch [B][G][m]
    unsigned* counters;  // [B], zero between launches
    int B, H, Ncap, n, k, m;
    int mode, append, dense;
    float scale;
};

template <class KV, int HG>
struct DecodeCfg {
    static constexpr int D = kHeadDim;
    static constexpr int E = KV::E;
    static constexpr bool QUANT = KV::QUANT;
    static constexpr int VE = 16 / E;    // elements per 16-byte vector
    static constexpr int LR = D / VE;    // lanes per head row
    static constexpr int RPW = 32 / LR;  // head rows per warp instruction
    static constexpr int SLOTS = kConsumerWarps * RPW;
    static constexpr int ROWE = D * E;   // bytes per head row
    static constexpr int ROWB = HG * ROWE;
    static constexpr int T = (8192 / ROWB) < 1 ? 1 : ((8192 / ROWB) > 32 ? 32 : 8192 / ROWB);
    static constexpr int S = 6;
    static constexpr int STAGEB = T * ROWB;
    static constexpr int METAB = QUANT ? T * HG * 8 : 0;
    static_assert(SLOTS % HG == 0, "head group must tile the consumer slots");
    static_assert(!QUANT || HG >= 2, "quantized rows need >= 16-byte meta copies");
    static_assert(SLOTS * D * 4 <= S * STAGEB, "reduction scratch aliases the ring");
};

struct DecodeSmem {
    size_t ring, meta, cur, bars, tok, uni, topk, flag, total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Shared-memory carve-up; identical on host (launch size) and device.
template <class KV, int HG>
__host__ __device__ inline DecodeSmem decode_smem(int m, int nc) {
    using C = DecodeCfg<KV, HG>;
    DecodeSmem s;
    size_t o = 0;
    s.ring = o;
    o += static_cast<size_t>(C::S) * C::STAGEB;
    s.meta = o;
    o = align_up(o + static_cast<size_t>(C::S) * C::METAB, 128);
    s.cur = o;  // cur K row, cur V row, cur meta (2*HG float2)
    o = align_up(o + 2 * C::ROWB + 2 * HG * 8, 16);
    s.bars = o;
    o += 2 * C::S * 8;
    s.tok = o;
    o = align_up(o + static_cast<size_t>(m) * 4, 16);
    s.uni = o;  // logits/weights [HG][m] f32  U  order keys [nc] u64
    const size_t lg = static_cast<size_t>(HG) * m * 4, ks = static_cast<size_t>(nc) * 8;
    o = align_up(o + (lg > ks ? lg : ks), 16);
    s.topk = o;
    o = align_up(o + sizeof(TopkSmem<kConsumerThreads>), 16);
    s.flag = o;
    o += 16;
    s.total = o;
    return s;
}

template <class KV, class QT, int HG>
__global__ void __launch_bounds__(kDecodeThreads)
    swa_decode_kernel(const DecodeParams p) {
    using C = DecodeCfg<KV, HG>;
    constexpr int D = C::D, VE = C::VE, LR = C::LR, RPW = C::RPW, SLOTS = C::SLOTS;
    constexpr int ROWE = C::ROWE, ROWB = C::ROWB, T = C::T, S = C::S;
    constexpr int STAGEB = C::STAGEB, METAB = C::METAB;
    constexpr bool QUANT = C::QUANT;

    extern __shared__ __align__(128) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = blockIdx.x, b = blockIdx.y, G = gridDim.x;
    const int H = p.H, n = p.n, k = p.k, m = p.m;
    const int nc = (p.mode == kModeSwaStep && !p.dense) ? n - k : 0;
    const DecodeSmem L = decode_smem<KV, HG>(m, nc);

    uint8_t* ring = smem + L.ring;
    float2* metaR = reinterpret_cast<float2*>(smem + L.meta);
    uint8_t* curK = smem + L.cur;
    uint8_t* curV = curK + ROWB;
    float2* curM = reinterpret_cast<float2*>(curV + ROWB);  // [2][HG]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + S;
    int* tok = reinterpret_cast<int*>(smem + L.tok);
    float* wts = reinterpret_cast<float*>(smem + L.uni);  // [HG][m]
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem + L.uni);
    TopkSmem<kConsumerThreads>& tks = *reinterpret_cast<TopkSmem<kConsumerThreads>*>(smem + L.topk);
    int* s_last = reinterpret_cast<int*>(smem + L.flag);

    const size_t TOKB = static_cast<size_t>(2) * H * ROWE;  // bytes per token (K and V planes)
    const uint8_t* kvb = p.kv + static_cast<size_t>(b) * p.Ncap * TOKB + static_cast<size_t>(g) * ROWB;
    const float2* metab = QUANT ? p.meta + static_cast<size_t>(b) * p.Ncap * 2 * H + g * HG : nullptr;

    // ---- prologue: barriers and the index positions known before selection
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_barrier_init();
    }
    const bool sel_in_kernel = (p.mode == kModeSwaStep) && !p.dense;
    if (p.mode == kModeExplicit) {
        for (int i = tid; i < m; i += kDecodeThreads) tok[i] = p.idx_in[static_cast<size_t>(b) * m + i];
    } else if (!sel_in_kernel) {
        for (int i = tid; i < m; i += kDecodeThreads) tok[i] = i;
    } else {
        // local window without the current token, then (after select) the
        // k global picks, then the current token n-1 last.
        for (int i = tid; i < k - 1; i += kDecodeThreads) tok[i] = n - k + i;
        if (tid == 0) tok[m - 1] = n - 1;
    }
    __syncthreads();

    const int nchunks = (m + T - 1) / T;

    if (warp == kConsumerWarps) {
        // ================================================== producer warp
        const uint64_t pol = policy_evict_first();
        const int known = sel_in_kernel ? k - 1 : m;
        bool have_all = !sel_in_kernel;
        for (int u = 0; u < 2 * nchunks; ++u) {
            const int vsel = u >= nchunks;
            const int base = (vsel ? u - nchunks : u) * T;
            const int cnt = min(T, m - base);
            const int stage = u % S;
            if (u >= S) mbar_wait(&empty[stage], ((u / S) - 1) & 1);
            if (!have_all && base + cnt > known) {
                named_sync(kBarSelect, kConsumerThreads + 32);
                have_all = true;
            }
            const int ncopy = cnt - ((p.append && base + cnt == m) ? 1 : 0);
            if (lane == 0)
                mbar_arrive_expect_tx(&full[stage], ncopy * (ROWB + (QUANT ? HG * 8 : 0)));
            __syncwarp();
            if (lane < ncopy) {
                const int t = tok[base + lane];
                const uint8_t* src = kvb + static_cast<size_t>(t) * TOKB + vsel * H * ROWE;
                bulk_g2s(ring + stage * STAGEB + lane * ROWB, src, ROWB, &full[stage], pol);
                if constexpr (QUANT) {
                    const float2* msrc = metab + static_cast<size_t>(t) * 2 * H + vsel * H;
                    bulk_g2s(reinterpret_cast<uint8_t*>(metaR) + stage * METAB + lane * HG * 8, msrc,
                             HG * 8, &full[stage], pol);
                }
            }
        }
        return;
    }

    // ====================================================== consumer warps
    const int ctid = tid;  // 0 .. kConsumerThreads-1

    // ---- append the step's new K/V rows for this head group
    if (p.append) {
        const size_t tok_off = (static_cast<size_t>(b) * p.Ncap + (n - 1)) * TOKB +
                               static_cast<size_t>(g) * ROWB;
        if constexpr (!QUANT) {
            // compute dtype == storage dtype: straight 16-byte copies
            constexpr int VPR = ROWB / 16;
            for (int i = ctid; i < 2 * VPR; i += kConsumerThreads) {
                const int kv = i / VPR, j = i % VPR;
                const uint8_t* srcb = static_cast<const uint8_t*>(kv ? p.v_new : p.k_new) +
                                      (static_cast<size_t>(b) * H + g * HG) * ROWE;
                const uint4 val = reinterpret_cast<const uint4*>(srcb)[j];
                reinterpret_cast<uint4*>(p.kv_w + tok_off + kv * H * ROWE)[j] = val;
                reinterpret_cast<uint4*>(kv ? curV : curK)[j] = val;
            }
        } else {
            // quant.hpp:43-81 per (token, head) group of D values, in fp64.
            for (int grp = warp; grp < 2 * HG; grp += kConsumerWarps) {
                const int kv = grp / HG, h = grp % HG;
                const QT* src = static_cast<const QT*>(kv ? p.v_new : p.k_new) +
                                (static_cast<size_t>(b) * H + g * HG + h) * D;
                double x[D / 32];
                double lo, hi;
#pragma unroll
                for (int i = 0; i < D / 32; ++i) x[i] = static_cast<double>(to_f(src[lane * (D / 32) + i]));
                lo = x[0];
                hi = x[0];
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
                uint8_t* dst = p.kv_w + tok_off + kv * H * ROWE + h * ROWE;
                reinterpret_cast<uint32_t*>(dst)[lane] = packed;
                reinterpret_cast<uint32_t*>((kv ? curV : curK) + h * ROWE)[lane] = packed;
                if (lane == 0) {
                    const float2 ms = make_float2(static_cast<float>(scale),
                                                  static_cast<float>(-scale * static_cast<double>(zp)));
                    p.meta_w[(static_cast<size_t>(b) * p.Ncap + (n - 1)) * 2 * H + kv * H + g * HG + h] = ms;
                    curM[kv * HG + h] = ms;
                }
            }
        }
    }

    // ---- selection (attention.hpp:142-171) over importance[0, n-k)
    if (sel_in_kernel) {
        const double* imp = p.imp + static_cast<size_t>(b) * p.Ncap;
        for (int i = ctid; i < nc; i += kConsumerThreads) keys[i] = order_key(imp[i]);
        named_sync(kBarConsumers, kConsumerThreads);
        block_topk<kConsumerThreads, kBarConsumers>(keys, nc, k, tok + (k - 1), tks, ctid);
        named_arrive(kBarSelect, kConsumerThreads + 32);
    } else {
        named_sync(kBarConsumers, kConsumerThreads);
    }

    // ---- per-lane query slice
    const int slot = warp * RPW + lane / LR;
    const int h = slot % HG;
    const int c = lane % LR;
    float qf[VE];
    {
        const QT* qrow = static_cast<const QT*>(p.q) + (static_cast<size_t>(b) * H + g * HG + h) * D + c * VE;
#pragma unroll
        for (int i = 0; i < VE; ++i) qf[i] = to_f(qrow[i]);
    }
    float qsum = 0.f;
    if constexpr (QUANT) {
#pragma unroll
        for (int i = 0; i < VE; ++i) qsum += qf[i];
#pragma unroll
        for (int off = LR / 2; off > 0; off >>= 1) qsum += __shfl_xor_sync(0xffffffffu, qsum, off);
    }
    const int warp_row0 = warp * RPW;

    // ---- pass 1: logits = (q . k) * scale  (attention.hpp:204-212)
    for (int u = 0; u < nchunks; ++u) {
        const int stage = u % S;
        mbar_wait(&full[stage], (u / S) & 1);
        const int base = u * T;
        const int rows = min(T, m - base) * HG;
        const uint8_t* st = ring + stage * STAGEB;
        for (int r0 = warp_row0; r0 < rows; r0 += SLOTS) {
            const int r = r0 + (slot - warp_row0);
            const bool valid = r < rows;
            const int t = r / HG;
            const int pos = base + t;
            const bool cur = p.append && pos == m - 1;
            const uint8_t* rowp = cur ? curK + h * ROWE : st + r * ROWE;
            float kf[VE];
            cvt16(*reinterpret_cast<const uint4*>(rowp + c * 16), kf, KV{});
            float dot = 0.f;
#pragma unroll
            for (int i = 0; i < VE; ++i) dot = fmaf(qf[i], kf[i], dot);
#pragma unroll
            for (int off = LR / 2; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
            if (valid && c == 0) {
                float logit;
                if constexpr (QUANT) {
                    const float2 ms = cur ? curM[h] : metaR[stage * (METAB / 8) + t * HG + h];
                    logit = fmaf(ms.x, dot, ms.y * qsum) * p.scale;
                } else {
                    logit = dot * p.scale;
                }
                wts[h * m + pos] = logit;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
    }
    named_sync(kBarConsumers, kConsumerThreads);

    // ---- softmax with the reference's normaliser (attention.hpp:213-218)
    for (int hh = warp; hh < HG; hh += kConsumerWarps) {
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
        for (int i = lane; i < m; i += 32) wl[i] = wl[i] * inv;
    }
    named_sync(kBarConsumers, kConsumerThreads);

    // ---- head-group partial of the importance update + optional outputs
    auto sorted_pos = [&](int pos) -> int {
        if (!sel_in_kernel) return pos;
        if (pos < k - 1) return pos + k;    // local window n-k .. n-2
        if (pos < 2 * k - 1) return pos - (k - 1);  // global picks (ascending)
        return pos;                         // current token n-1
    };
    {
        float* wp = p.wpart + (static_cast<size_t>(b) * G + g) * m;
        for (int pos = ctid; pos < m; pos += kConsumerThreads) {
            float s = 0.f;
#pragma unroll
            for (int hh = 0; hh < HG; ++hh) s += wts[hh * m + pos];
            wp[pos] = s;
            if (p.idx_out != nullptr && g == 0) p.idx_out[static_cast<size_t>(b) * m + sorted_pos(pos)] = tok[pos];
        }
        if (p.w_out != nullptr) {
            for (int i = ctid; i < HG * m; i += kConsumerThreads) {
                const int hh = i / m, pos = i % m;
                p.w_out[(static_cast<size_t>(b) * H + g * HG + hh) * m + sorted_pos(pos)] = wts[i];
            }
        }
    }

    // ---- pass 2: attn = sum_t w_t * V[t]  (attention.hpp:219-225)
    float acc[VE];
#pragma unroll
    for (int i = 0; i < VE; ++i) acc[i] = 0.f;
    float bsum = 0.f;
    for (int u = nchunks; u < 2 * nchunks; ++u) {
        const int stage = u % S;
        mbar_wait(&full[stage], (u / S) & 1);
        const int base = (u - nchunks) * T;
        const int rows = min(T, m - base) * HG;
        const uint8_t* st = ring + stage * STAGEB;
        for (int r0 = warp_row0; r0 < rows; r0 += SLOTS) {
            const int r = r0 + (slot - warp_row0);
            if (r < rows) {
                const int t = r / HG;
                const int pos = base + t;
                const bool cur = p.append && pos == m - 1;
                const uint8_t* rowp = cur ? curV + h * ROWE : st + r * ROWE;
                float vf[VE];
                cvt16(*reinterpret_cast<const uint4*>(rowp + c * 16), vf, KV{});
                const float w = wts[h * m + pos];
                if constexpr (QUANT) {
                    const float2 ms = cur ? curM[HG + h] : metaR[stage * (METAB / 8) + t * HG + h];
                    const float a = w * ms.x;
#pragma unroll
                    for (int i = 0; i < VE; ++i) acc[i] = fmaf(a, vf[i], acc[i]);
                    bsum = fmaf(w, ms.y, bsum);
                } else {
#pragma unroll
                    for (int i = 0; i < VE; ++i) acc[i] = fmaf(w, vf[i], acc[i]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
    }
    // all stages consumed and no copy in flight: the ring is free scratch now
    named_sync(kBarConsumers, kConsumerThreads);
    float* red = reinterpret_cast<float*>(ring);  // [SLOTS][D]
#pragma unroll
    for (int i = 0; i < VE; ++i) red[slot * D + c * VE + i] = acc[i] + bsum;
    named_sync(kBarConsumers, kConsumerThreads);
    for (int o = ctid; o < HG * D; o += kConsumerThreads) {
        const int hh = o / D, d = o % D;
        float s = 0.f;
        for (int sl = hh; sl < SLOTS; sl += HG) s += red[sl * D + d];
        static_cast<QT*>(p.out)[(static_cast<size_t>(b) * H + g * HG + hh) * D + d] = from_f<QT>(s);
    }

    // ---- importance: last CTA of the sequence folds the G head-group
    // partials in fixed order (deterministic) into the fp64 accumulator.
    named_sync(kBarConsumers, kConsumerThreads);
    if (ctid == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(&p.counters[b], 1u);
        *s_last = (prev == static_cast<unsigned>(G - 1)) ? 1 : 0;
    }
    named_sync(kBarConsumers, kConsumerThreads);
    if (*s_last) {
        __threadfence();
        double* imp = p.imp + static_cast<size_t>(b) * p.Ncap;
        const float* wp = p.wpart + static_cast<size_t>(b) * G * m;
        for (int pos = ctid; pos < m; pos += kConsumerThreads) {
            double s = 0.0;
            for (int gg = 0; gg < G; ++gg) s += static_cast<double>(__ldcg(wp + static_cast<size_t>(gg) * m + pos));
            const int t = tok[pos];
            if (p.mode == kModeSeed || (p.append && pos == m - 1))
                imp[t] = s;
            else
                imp[t] += s;
        }
        if (ctid == 0) p.counters[b] = 0;
    }
}

}  // namespace skvd
