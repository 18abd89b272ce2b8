// skv_prefill.cu -- dense causal prefill attention on tcgen05 tensor cores and
// the accumulator seeding that starts the SWA decode.
//
// Engine::prefill (engine.hpp:485-529) runs dense_attention (attention.hpp:
// 91-117) with the causal mask over the prompt, seeds each head's accumulator
// with the LAST attention row (engine.hpp:508-512) and records
// attention_sparsity(aw, 0.01, causal) per layer (engine.hpp:513-518).
//
// Flash-style, two passes over the causal key tiles of each 128-query tile;
// nothing of size s x s ever reaches HBM:
//   pass 1 (stats): S = Q K^T (tcgen05, TMEM accumulator), per-row running
//                   max and sum -> (m, l) per query row;
//   pass 2 (exact): S again (same MMAs, bit-identical), w = exp(S/sqrt(D) - m)
//                   / l is final, so there is no rescaling: w is counted
//                   against the 0.01 x row-max threshold (e < 0.01: the row
//                   max of e is exactly 1), written out for the last query
//                   row (the seed), stored 16-bit into TMEM over the S
//                   columns it came from and multiplied into O += P V on the
//                   tensor cores (A from TMEM, V read MN-major straight from
//                   the cache tile).
// Q, K, V come from the caller's q and the cache through 3D tensor maps whose
// token extent is the prompt length s, so keys / queries >= s are zero-filled
// by TMA and never carry uninitialised cache bytes into the MMAs.
// Roles per CTA (192 threads): warp 0 TMA producer, warp 1 MMA issuer (+ TMEM
// allocation), warps 2..5 one query row per thread (softmax, P, epilogue).
// bf16 keeps 8 mantissa bits, too few for the 1e-3 output bound: P is split
// into hi + lo bf16 halves and both are multiplied against V (fp16 P, 11
// bits, is stored once). (kind::f16 needs A and B of one type, so an fp16 P
// against bf16 V is not an option: it faults.)
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "skv_internal.h"

namespace skvd {

constexpr int kFTile = 128;    // query rows and keys per tile
constexpr int kFHalf = 16384;  // one 64-column SW128 box of a 128-row tile
constexpr int kFTileBytes = 2 * kFHalf;
constexpr int kFThreads = 192;

struct FlashParams {
    int s, H, HD;
    float c1;         // log2(e) / sqrt(D): exp(x / sqrt(D)) = exp2(x * c1)
    float2* ml;       // [Z][s] row max (log2 units) and sum, from pass 1
    void* out;        // [B][s][H][D], 16-bit or fp32 (out_f32)
    int out_f32;
    float* wlast;     // [Z][s] the last query row's weights
    unsigned* below;  // [Z] cells with w < 0.01 x row max
};

__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// K-major operand, canonical SWIZZLE_128B (8-row groups of 1024 B).
__device__ __forceinline__ uint64_t desc_k(const void* p) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | (1ull << 16) | ((1024ull >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// MN-major operand, SWIZZLE_128B: 64-element MN atoms kFHalf bytes apart
// (LBO), 8-row K groups 1024 B apart (SBO).
__device__ __forceinline__ uint64_t desc_mn(const void* p) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | (uint64_t(kFHalf >> 4) << 16) | ((1024ull >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}

__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t addr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
          "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
          "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <bool BF16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    if constexpr (BF16)
        return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(a))) |
               (static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(b))) << 16);
    else
        return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(a))) |
               (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(b))) << 16);
}

__device__ __forceinline__ float bf16_rest(float a) { return a - __bfloat162float(__float2bfloat16_rn(a)); }

// instruction descriptor, kind::f16, fp32 accumulate, M = N = 128, A K-major
template <bool BF16, bool B_MN>
__host__ __device__ constexpr uint32_t flash_idesc() {
    return (1u << 4) | ((BF16 ? 1u : 0u) << 7) | ((BF16 ? 1u : 0u) << 10) | ((B_MN ? 1u : 0u) << 16) |
           (uint32_t(kFTile >> 3) << 17) | (uint32_t(kFTile >> 4) << 24);
}

template <bool BF16, bool STATS>
struct FlashSmem {
    static constexpr int kQ = 0;
    static constexpr int kK = kQ + kFTileBytes;                    // pass 1: 2 stages, pass 2: 1
    static constexpr int kV = kK + (STATS ? 2 : 1) * kFTileBytes;  // pass 2: 1 stage
    static constexpr int kBar = kV + (STATS ? 0 : kFTileBytes);
    static constexpr int kBytes = kBar + 256 + 1024;  // barriers + alignment slack
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// A operand from TMEM (P), B from shared memory (V)
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

// Two CTAs per SM (96 KB shared memory, 256 TMEM columns, <= 168 registers
// each) so one CTA's softmax overlaps the other's MMAs. TMEM per CTA:
//   pass 1: S double buffer, columns [0, 256);
//   pass 2: S / P in [0, 128) -- P is written over the S columns it came
//           from, 32 keys per 32-column chunk: hi in the chunk's first 16
//           columns, bf16 lo in the next 16 -- and O in [128, 256).
template <bool BF16, bool STATS>
__global__ void __launch_bounds__(kFThreads, 2)
    flash_prefill_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                         const FlashParams p) {
    using L = FlashSmem<BF16, STATS>;
    constexpr uint32_t kCols = 256;
    constexpr int KS = STATS ? 2 : 1;  // K stages
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm + L::kQ;
    uint8_t* sK = sm + L::kK;
    uint8_t* sV = sm + L::kV;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::kBar);
    uint64_t* q_full = bar;
    uint64_t* k_full = bar + 1;    // [KS]
    uint64_t* k_empty = bar + 3;   // [KS]
    uint64_t* v_full = bar + 5;
    uint64_t* v_empty = bar + 6;
    uint64_t* s_full = bar + 7;    // [2]
    uint64_t* s_empty = bar + 9;   // [2] (pass 1)
    uint64_t* p_full = bar + 11;
    uint64_t* p_empty = bar + 12;
    uint64_t* o_full = bar + 13;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 14);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int z = blockIdx.x, qt = gridDim.y - 1 - blockIdx.y;  // heaviest query tiles first
    const int b = z / p.H, h = z % p.H;
    const int m0 = qt * kFTile;
    const int T = qt + 1;  // causal key tiles

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], 128);
        }
        mbar_init(v_full, 1);
        mbar_init(v_empty, 1);
        mbar_init(p_full, 128);
        mbar_init(p_empty, 1);
        mbar_init(o_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA
        if (lane == 0) {
            const int xq = h * 128;
            mbar_arrive_expect_tx(q_full, kFTileBytes);
            tma3d(sQ, &map_q, xq, m0, b, q_full);
            tma3d(sQ + kFHalf, &map_q, xq + 64, m0, b, q_full);
            for (int j = 0; j < T; ++j) {
                const int st = j % KS;
                if (j >= KS) mbar_wait(&k_empty[st], ((j / KS) - 1) & 1);
                uint8_t* dk = sK + st * kFTileBytes;
                mbar_arrive_expect_tx(&k_full[st], kFTileBytes);
                tma3d(dk, &map_kv, xq, j * kFTile, b, &k_full[st]);
                tma3d(dk + kFHalf, &map_kv, xq + 64, j * kFTile, b, &k_full[st]);
                if constexpr (!STATS) {
                    if (j >= 1) mbar_wait(v_empty, (j - 1) & 1);
                    mbar_arrive_expect_tx(v_full, kFTileBytes);
                    tma3d(sV, &map_kv, p.HD + xq, j * kFTile, b, v_full);
                    tma3d(sV + kFHalf, &map_kv, p.HD + xq + 64, j * kFTile, b, v_full);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA
        if (lane == 0) {
            constexpr uint32_t id_s = flash_idesc<BF16, false>();
            constexpr uint32_t id_o = flash_idesc<BF16, true>();
            mbar_wait(q_full, 0);
            auto issue_s = [&](int j, uint32_t dst) {
                const int st = j % KS;
                mbar_wait(&k_full[st], (j / KS) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint8_t* k = sK + st * kFTileBytes;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int off = (kk >> 2) * kFHalf + (kk & 3) * 32;
                    umma(dst, desc_k(sQ + off), desc_k(k + off), id_s, kk > 0);
                }
                umma_commit(&k_empty[st]);
            };
            if constexpr (STATS) {
                for (int j = 0; j < T; ++j) {
                    const int sb = j & 1;
                    if (j >= 2) {
                        mbar_wait(&s_empty[sb], ((j >> 1) - 1) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    }
                    issue_s(j, tmem + sb * 128);
                    umma_commit(&s_full[sb]);
                }
            } else {
                for (int j = 0; j < T; ++j) {
                    // S_j overwrites P_{j-1}: PV_{j-1} must have consumed it
                    if (j >= 1) {
                        mbar_wait(p_empty, (j - 1) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    }
                    issue_s(j, tmem);
                    umma_commit(&s_full[0]);
                    mbar_wait(v_full, j & 1);
                    mbar_wait(p_full, j & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {  // 16 keys: chunk kk/2, half kk%2
                        const uint32_t pa = tmem + (kk >> 1) * 32 + (kk & 1) * 8;
                        umma_ts(tmem + 128, pa, desc_mn(sV + kk * 2048), id_o, (j | kk) != 0);
                        if constexpr (BF16) umma_ts(tmem + 128, pa + 16, desc_mn(sV + kk * 2048), id_o, 1);
                    }
                    umma_commit(p_empty);
                    umma_commit(v_empty);
                }
                umma_commit(o_full);
            }
        }
    } else {
        // ------------------------------------------------ rows: softmax / P / O
        const int q4 = warp & 3;  // TMEM lane quarter this warp may access
        const int rl = q4 * 32 + lane;
        const int r = m0 + rl;
        const bool valid = r < p.s;
        const uint32_t tl = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
        const size_t zrow = static_cast<size_t>(z) * p.s;
        float m = -INFINITY, l = 0.f, inv_l = 0.f;
        if constexpr (!STATS) {
            if (valid) {
                const float2 v = p.ml[zrow + r];
                m = v.x;
                inv_l = 1.0f / v.y;
            }
        }
        unsigned cnt = 0;
        const bool last_row = r == p.s - 1;
        for (int j = 0; j < T; ++j) {
            const int sb = STATS ? (j & 1) : 0;
            mbar_wait(&s_full[sb], STATS ? ((j >> 1) & 1) : (j & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int lim = valid ? min(r - j * kFTile, kFTile - 1) : -1;  // keys 0..lim of this tile count
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                float sv[32];
                const uint32_t ca = tl + sb * 128 + c * 32;
                tmem_ld32(ca, sv);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int cl = lim - c * 32;  // keys 0..cl of this chunk count
                if constexpr (STATS) {
                    if (cl >= 0) {
                        float mx = m;
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (k <= cl) mx = fmaxf(mx, sv[k] * p.c1);
                        float acc = 0.f;
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (k <= cl) acc += ex2(sv[k] * p.c1 - mx);
                        l = l * ex2(m - mx) + acc;
                        m = mx;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        float e = 0.f;
                        if (k <= cl) {
                            e = ex2(sv[k] * p.c1 - m);
                            cnt += e < 0.01f;
                        }
                        sv[k] = e * inv_l;
                    }
                    if (last_row) {
                        float* wl = p.wlast + zrow + j * kFTile + c * 32;
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (k <= cl) wl[k] = sv[k];
                    }
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) pk[i] = pack2<BF16>(sv[2 * i], sv[2 * i + 1]);
                    tmem_st16(ca, pk);
                    if constexpr (BF16) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) pk[i] = pack2<true>(bf16_rest(sv[2 * i]), bf16_rest(sv[2 * i + 1]));
                        tmem_st16(ca + 16, pk);
                    }
                }
            }
            if constexpr (STATS) {
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&s_empty[sb]);
            } else {
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(p_full);
            }
        }
        if constexpr (STATS) {
            if (valid) p.ml[zrow + r] = make_float2(m, l);
        } else {
            mbar_wait(o_full, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const size_t row0 = (static_cast<size_t>(b) * p.s + r) * p.HD + static_cast<size_t>(h) * 128;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                float o[32];
                tmem_ld32(tl + 128 + c * 32, o);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (!valid) continue;
                if (p.out_f32) {
                    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.out) + row0 + c * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
                } else {
                    uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(p.out) + row0 + c * 32);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        uint4 v;
                        v.x = pack2<BF16>(o[8 * i + 0], o[8 * i + 1]);
                        v.y = pack2<BF16>(o[8 * i + 2], o[8 * i + 3]);
                        v.z = pack2<BF16>(o[8 * i + 4], o[8 * i + 5]);
                        v.w = pack2<BF16>(o[8 * i + 6], o[8 * i + 7]);
                        dst[i] = v;
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            if (lane == 0 && cnt) atomicAdd(&p.below[z], cnt);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
    }
}

// importance[b][j] = sum_h w_last (head order, fp64): engine.hpp:508-512
// seeds each head's accumulator, attention.hpp:77-85 sums them. Block x = 0
// also folds the per-head sparsity counts (engine.hpp:513-518).
__global__ void prefill_seed_kernel(const float* __restrict__ wlast, const unsigned* __restrict__ below,
                                    double* __restrict__ imp, double* __restrict__ psp, int H, int s,
                                    long long imp_ld) {
    const int b = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (psp != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
        const double cells = 0.5 * static_cast<double>(s) * static_cast<double>(s + 1);
        double sp = 0.0;
        for (int h = 0; h < H; ++h) sp += static_cast<double>(below[b * H + h]) / cells;
        psp[b] = sp / static_cast<double>(H);
    }
    if (j >= s) return;
    double acc = 0.0;
    for (int h = 0; h < H; ++h) acc += static_cast<double>(wlast[(static_cast<size_t>(b) * H + h) * s + j]);
    imp[static_cast<size_t>(b) * imp_ld + j] = acc;
}

}  // namespace skvd

namespace skv_impl {
using namespace skvd;

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// [seqs][tokens][cols] 16-bit, tokens bounded to `tokens` (TMA zero-fills
// beyond), box {64 cols, 128 tokens, 1}.
bool map3d(CUtensorMap* m, const void* base, bool bf16, uint64_t cols, uint64_t tokens, uint64_t seqs,
           uint64_t row_bytes, uint64_t seq_bytes) {
    EncodeFn fn = encoder();
    if (!fn) return false;
    const cuuint64_t dims[3] = {cols, tokens, seqs};
    const cuuint64_t strides[2] = {row_bytes, seq_bytes};
    const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(kFTile), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base),
              dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool BF16, bool STATS>
cudaError_t run_flash(const CUtensorMap& mq, const CUtensorMap& mkv, const FlashParams& p, int Z, int nqt,
                      cudaStream_t st) {
    constexpr int smem = FlashSmem<BF16, STATS>::kBytes;
    const void* fn = reinterpret_cast<const void*>(&flash_prefill_kernel<BF16, STATS>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<CUtensorMap*>(&mq), const_cast<CUtensorMap*>(&mkv), const_cast<FlashParams*>(&p)};
    e = cudaLaunchKernel(fn, dim3(Z, nqt), dim3(kFThreads), args, smem, st);
    count_launch();
    return e;
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

// ml float2 [Z][s], wlast fp32 [Z][s], below u32 [Z]
size_t prefill_scratch_bytes(int B, int H, int s) {
    const size_t Z = static_cast<size_t>(B) * H;
    return align256(Z * s * 8) + align256(Z * s * 4) + align256(Z * 4);
}

// Causal prefill of one cache layer (see the file comment). kv: layer base
// of a 16-bit cache [B][Ncap][2][H][D]; q/out: [B][s][H][D] (out fp32 when
// out_f32); imp: layer importance [B][imp_ld]; psp (nullable): [B].
cudaError_t launch_prefill(bool bf16, bool out_f32, const void* kv, const void* q, void* out, double* imp,
                           long long imp_ld, double* psp, int B, int H, int D, int Ncap, int s, uint8_t* scratch,
                           cudaStream_t st) {
    if (D != 128) return cudaErrorInvalidValue;
    const int Z = B * H, nqt = (s + kFTile - 1) / kFTile;
    const uint64_t HD = static_cast<uint64_t>(H) * D;
    float2* ml = reinterpret_cast<float2*>(scratch);
    float* wlast = reinterpret_cast<float*>(scratch + align256(static_cast<size_t>(Z) * s * 8));
    unsigned* below = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(wlast) +
                                                  align256(static_cast<size_t>(Z) * s * 4));
    cudaError_t e = cudaMemsetAsync(below, 0, static_cast<size_t>(Z) * 4, st);
    if (e != cudaSuccess) return e;
    CUtensorMap mq, mkv;
    if (!map3d(&mq, q, bf16, HD, s, B, HD * 2, HD * 2 * s) ||
        !map3d(&mkv, kv, bf16, 2 * HD, s, B, 2 * HD * 2, 2 * HD * 2 * Ncap))
        return cudaErrorInvalidValue;
    FlashParams p{};
    p.s = s;
    p.H = H;
    p.HD = static_cast<int>(HD);
    p.c1 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(D)));
    p.ml = ml;
    p.out = out;
    p.out_f32 = out_f32 ? 1 : 0;
    p.wlast = wlast;
    p.below = below;
    e = bf16 ? run_flash<true, true>(mq, mkv, p, Z, nqt, st) : run_flash<false, true>(mq, mkv, p, Z, nqt, st);
    if (e != cudaSuccess) return e;
    e = bf16 ? run_flash<true, false>(mq, mkv, p, Z, nqt, st) : run_flash<false, false>(mq, mkv, p, Z, nqt, st);
    if (e != cudaSuccess) return e;
    prefill_seed_kernel<<<dim3((s + 255) / 256, B), 256, 0, st>>>(wlast, below, imp, psp, H, s, imp_ld);
    count_launch();
    return cudaGetLastError();
}

}  // namespace skv_impl
