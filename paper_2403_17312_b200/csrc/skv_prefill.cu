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
//   pass 1 (max):  S = Q K^T (tcgen05, TMEM accumulator) and the row max M
//                  over the causal keys (one FMNMX per score);
//   pass 2:        S again (same MMAs, bit-identical), e = exp(S/sqrt(D) - M)
//                  with the final max, so there is no rescaling: e is
//                  counted against the 0.01 x row-max threshold (e < 0.01:
//                  the row max of e is 1), summed into l, kept for the last
//                  query row (the seed, w = e / l), stored 16-bit into TMEM
//                  over the S columns it came from and multiplied into
//                  O += P V on the tensor cores (A from TMEM, V read MN-major
//                  straight from the cache tile); O / l at the end.
// Q, K, V come from the caller's q and the cache through 3D tensor maps whose
// token extent is the prompt length s, so keys / queries >= s are zero-filled
// by TMA and never carry uninitialised cache bytes into the MMAs.
// bf16 keeps 8 mantissa bits, too few for the 1e-3 output bound: P is split
// into hi + lo bf16 halves and both are multiplied against V (fp16 P, 11
// bits, is stored once). (kind::f16 needs A and B of one type, so an fp16 P
// against bf16 V is not an option: it faults.)
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <mutex>

#include "skv_internal.h"

namespace skvd {

constexpr int kFTile = 128;    // query rows per tile
constexpr int kFKeys = 128;    // keys per tile (N = 128 S MMAs: an M = 128 MMA costs about the same for N <= 256)
constexpr int kFHalf = 16384;  // one 64-column SW128 box of the 128-row Q tile
constexpr int kFTileBytes = 2 * kFHalf;
constexpr int kFKHalf = kFKeys * 128;  // one 64-column SW128 box of a 64-key K / V tile
constexpr int kFKBytes = 2 * kFKHalf;
constexpr int kFBufs = 2;    // S / P buffers in TMEM, K / V stages in shared memory
constexpr int kFHK = kFKeys / 2;  // keys per row thread per tile
constexpr int kFThreads = 448;  // warps 0..3 control / epilogue, 4..11 rows, 12..13 epilogue

struct FlashParams {
    int s, H, HD;
    int Z, nqt;       // work items: Z x nqt query tiles
    int s_pad;        // nqt * 128: row stride of mrow
    float c1;         // log2(e) / sqrt(D): exp(x / sqrt(D)) = exp2(x * c1)
    float* mrow;      // [Z][s_pad] row max of S = Q K^T over the causal keys (pass 1)
    void* out;        // [B][s][H][D], 16-bit or fp32 (out_f32)
    int out_f32;
    float* wlast;     // [Z][s] the last query row's e = exp(S/sqrt(D) - max)
    float* llast;     // [Z] its sum (w = e / l)
    unsigned* below;  // [Z] cells with w < 0.01 x row max, i.e. e < 0.01
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

// MN-major operand, SWIZZLE_128B: 64-element MN atoms kFKHalf bytes apart
// (LBO), 8-row K groups 1024 B apart (SBO).
__device__ __forceinline__ uint64_t desc_mn(const void* p) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | (uint64_t(kFKHalf >> 4) << 16) | ((1024ull >> 4) << 32) | (1ull << 46) |
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

// a -> low half, b -> high half; one F2FP.PACK_AB (separate F2F conversions
// would run on the XU pipe next to the exp2s)
template <bool BF16>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    uint32_t r;
    if constexpr (BF16) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        r = *reinterpret_cast<const uint32_t*>(&h);
    } else {
        const __half2 h = __floats2half2_rn(a, b);
        r = *reinterpret_cast<const uint32_t*>(&h);
    }
    return r;
}

__device__ __forceinline__ float bf16_rest(float a) {
    // a - bf16(a): bf16 rounding is exact on the fp32 bit pattern (RNE on the low 16 bits)
    const uint32_t u = __float_as_uint(a);
    const uint32_t hi = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    return a - __uint_as_float(hi);
}

// instruction descriptor, kind::f16, fp32 accumulate, M = 128, A K-major
template <bool BF16, bool B_MN, int N>
__host__ __device__ constexpr uint32_t flash_idesc() {
    return (1u << 4) | ((BF16 ? 1u : 0u) << 7) | ((BF16 ? 1u : 0u) << 10) | ((B_MN ? 1u : 0u) << 16) |
           (uint32_t(N >> 3) << 17) | (uint32_t(kFTile >> 4) << 24);
}

template <bool BF16, bool STATS>
struct FlashSmem {
    static constexpr int kQ = 0;                                // [2] query tiles (double buffered across items)
    static constexpr int kK = kQ + 2 * kFTileBytes;             // [kFBufs] key tiles (pass 1: 256 keys)
    static constexpr int kV = kK + kFBufs * kFKBytes * (STATS ? 2 : 1);  // [kFBufs] value tiles (pass 2)
    static constexpr int kM = kV + (STATS ? 0 : kFBufs * kFKBytes);  // [2][128] row max (pass 2)
    static constexpr int kR = kM + 2 * 128 * 4;                 // [2][2][128] per-half row partials
    static constexpr int kL = kR + 2 * 2 * 128 * 4;             // [2][128] 1 / l per O buffer (pass 2)
    static constexpr int kBar = kL + 2 * 128 * 4;
    static constexpr int kNBar = 40;
    static constexpr int kBytes = kBar + kNBar * 8 + 16 + 1024;  // barriers, TMEM slot, alignment
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// The same, but issued unconditionally: in the causal (diagonal) tiles the
// masked cells select 0 afterwards (FSEL). Left to the compiler, the mask
// became a predicate over each cell's constant reload, FFMA and MUFU, a
// serial chain that made a diagonal tile cost ~2.5 k cycles against ~1.3 k
// for a full one (PF_TRACE).
__device__ __forceinline__ float ex2_all(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
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

// Persistent, one CTA per SM over a contiguous run of work items (query
// tiles). Keys go in tiles of 128 through a double-buffered pipeline: K / V
// stages in shared memory, S / P buffers in TMEM, so the MMA for key tile
// g + 1 runs while the row threads work on tile g. Q (and the pass-1 row
// max) is double buffered across items so the next item's loads overlap the
// current item's tail. (An M = 128 tcgen05.mma costs about the same for any
// N <= 256 -- measured ~130 cycles per K = 16 step at N = 64 -- so the S
// MMAs use N = 128 key tiles rather than 64.)
// TMEM: S / P buffer b at columns [128 b, 128 b + 128) -- P is written over
// the S columns it came from, 32 keys per 32-column chunk: hi in the first
// 16 columns, bf16 lo in the next 16 -- and O buffers in [256, 512).
// Warps: 0 TMA, 1 MMA (+ TMEM allocation), 4..7 and 8..11 the row threads:
// warp w owns rows 32 (w % 4) .. (its TMEM lane quarter) and key columns
// 64 hf .. 64 hf + 63 of every tile (hf = 0 for warps 4..7, 1 for 8..11);
// 2, 3, 12, 13 (lane quarters 2, 3, 0, 1) drain O (double buffered: columns
// [256, 384) and [384, 512)) while the row threads move on to the next item.
#ifdef PF_TRACE
__device__ long long g_pft[2][8][32];
__device__ __forceinline__ int pft_tag(const char* t) {
    return t[0] == 't' ? 0 : t[4] == 's' && t[0] == 'm' ? 1 : t[4] == 's' ? 2 : t[4] == 'l' ? 3 : t[4] == 'm' ? 4 : t[4] == 'p' && t[0] == 'r' ? 5 : 6;
}
#define PFT(tag, gg)                                                                  \
    do {                                                                              \
        if (blockIdx.x == 0 && (gg) < 32) g_pft[STATS ? 0 : 1][pft_tag(tag)][gg] = clock64(); \
    } while (0)
#else
#define PFT(tag, gg) \
    do {             \
    } while (0)
#endif

template <bool BF16, bool STATS>
__global__ void __launch_bounds__(kFThreads, 1)
    flash_prefill_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kv,
                         const FlashParams p) {
    using L = FlashSmem<BF16, STATS>;
    // Key tile of this pass: the max pass has no P.V, so its S tiles are 256
    // keys wide (two 256-column TMEM buffers) -- a tcgen05.mma costs the same
    // ~163 cycles for any N <= 256 (scripts/mma_probe.cu), so N = 256 halves
    // the pass's tensor time; the P.V pass keeps 128-key tiles (its TMEM
    // holds S / P and two O buffers).
    constexpr int NK = STATS ? 2 * kFKeys : kFKeys;
    constexpr int NKH = NK * 128;  // one 64-column SW128 box of a key tile
    constexpr int NKB = 2 * NKH;
    constexpr int HK = NK / 2;     // keys per row thread per tile
    auto key_tiles = [](int qt) { return (qt * kFTile + kFTile + NK - 1) / NK; };
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* sQ = sm + L::kQ;
    uint8_t* sK = sm + L::kK;
    uint8_t* sV = sm + L::kV;
    float* sM = reinterpret_cast<float*>(sm + L::kM);  // [2][128]
    float* sR = reinterpret_cast<float*>(sm + L::kR);  // [2][2][128]
    float* sL = reinterpret_cast<float*>(sm + L::kL);  // [2][128]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::kBar);
    uint64_t* q_full = bar;        // [2]
    uint64_t* q_empty = bar + 2;   // [2]
    uint64_t* k_full = bar + 4;    // [4]
    uint64_t* k_empty = bar + 8;   // [4]
    uint64_t* v_full = bar + 12;   // [4]
    uint64_t* v_empty = bar + 16;  // [4]
    uint64_t* s_full = bar + 20;   // [4] MMA -> rows
    uint64_t* s_free = bar + 24;   // [4] pass 1: rows read S; pass 2: PV consumed P
    uint64_t* p_full = bar + 28;   // [4] pass 2: rows wrote P
    uint64_t* o_full = bar + 32;   // [2] MMA -> epilogue
    uint64_t* o_empty = bar + 34;  // [2] epilogue read O
    uint64_t* l_full = bar + 36;   // [2] rows wrote 1 / l
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + L::kNBar);

    if (threadIdx.x == 0) {
        for (int i = 0; i < 38; ++i) mbar_init(&bar[i], 1);
        if (!STATS) {
            // Q + row-max buffer: MMA commit after the item's last S + every row
            // thread after reading its row max
            mbar_init(&q_empty[0], 257);
            mbar_init(&q_empty[1], 257);
        }
        for (int i = 0; i < 4; ++i) {
            if (STATS) mbar_init(&s_free[i], 256);
            mbar_init(&p_full[i], 256);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&o_empty[i], 128);
            mbar_init(&l_full[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    // Contiguous runs of items, (sequence, head)-major with the heaviest query
    // tile first: consecutive items re-read the same K / V from L2 and the
    // concurrent working set (one (sequence, head) per SM) stays in L2.
    const int items = p.Z * p.nqt;
    const int first = static_cast<int>(static_cast<long long>(items) * blockIdx.x / gridDim.x);
    const int last = static_cast<int>(static_cast<long long>(items) * (blockIdx.x + 1) / gridDim.x);

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int g = 0, n = 0;
            for (int it = first; it < last; ++it, ++n) {
                const int qt = p.nqt - 1 - it % p.nqt, z = it / p.nqt;
                const int b = z / p.H, xq = (z % p.H) * 128;
                const int T = key_tiles(qt);
                const int qb = n & 1;
                if (n >= 2) mbar_wait(&q_empty[qb], ((n >> 1) - 1) & 1);
                mbar_arrive_expect_tx(&q_full[qb], kFTileBytes + (STATS ? 0 : 512));
                uint8_t* dq = sQ + qb * kFTileBytes;
                tma3d(dq, &map_q, xq, qt * kFTile, b, &q_full[qb]);
                tma3d(dq + kFHalf, &map_q, xq + 64, qt * kFTile, b, &q_full[qb]);
                if constexpr (!STATS)
                    bulk_g2s(sM + qb * 128, p.mrow + static_cast<size_t>(z) * p.s_pad + qt * kFTile, 512,
                             &q_full[qb], pol);
                for (int j = 0; j < T; ++j, ++g) {
                    const int st = g & 1;
                    if (g >= 2) mbar_wait(&k_empty[st], ((g >> 1) - 1) & 1);
                    PFT("tma_k", g);
                    uint8_t* dk = sK + st * NKB;
                    mbar_arrive_expect_tx(&k_full[st], NKB);
                    tma3d(dk, &map_kv, xq, j * NK, b, &k_full[st]);
                    tma3d(dk + NKH, &map_kv, xq + 64, j * NK, b, &k_full[st]);
                    if constexpr (!STATS) {
                        if (g >= 2) mbar_wait(&v_empty[st], ((g >> 1) - 1) & 1);
                        uint8_t* dv = sV + st * kFKBytes;
                        mbar_arrive_expect_tx(&v_full[st], kFKBytes);
                        tma3d(dv, &map_kv, p.HD + xq, j * kFKeys, b, &v_full[st]);
                        tma3d(dv + kFKHalf, &map_kv, p.HD + xq + 64, j * kFKeys, b, &v_full[st]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA
        if (lane == 0) {
            constexpr uint32_t id_s = flash_idesc<BF16, false, NK>();
            constexpr uint32_t id_o = flash_idesc<BF16, true, 128>();
            int g = 0, n = 0;
            auto issue_s = [&](int gg, const uint8_t* q) {
                const int sb = gg & 1;
                if (gg >= 2) mbar_wait(&s_free[sb], ((gg >> 1) - 1) & 1);  // buffer's S / P consumed
                mbar_wait(&k_full[sb], (gg >> 1) & 1);
                PFT("mma_s", gg);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint8_t* k = sK + sb * NKB;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma(tmem + sb * NK, desc_k(q + (kk >> 2) * kFHalf + (kk & 3) * 32),
                         desc_k(k + (kk >> 2) * NKH + (kk & 3) * 32), id_s, kk > 0);
                umma_commit(&k_empty[sb]);
                umma_commit(&s_full[sb]);
            };
            // The S stream runs one tile ahead of the PV stream, across item
            // boundaries: the next item's first S is on the tensor pipe while
            // the row threads finish the current item (O is double buffered and
            // drained by the epilogue warps).
            int itS = first, jS = 0, nS = 0, gS = 0;
            auto issue_next_s = [&]() {
                if (itS >= last) return;
                const int TS = key_tiles(p.nqt - 1 - itS % p.nqt);
                const int qb = nS & 1;
                if (jS == 0) mbar_wait(&q_full[qb], (nS >> 1) & 1);
                issue_s(gS++, sQ + qb * kFTileBytes);
                if (++jS == TS) {
                    umma_commit(&q_empty[qb]);  // the item's last S: Q is free
                    jS = 0;
                    ++itS;
                    ++nS;
                }
            };
            issue_next_s();
            for (int it = first; it < last; ++it, ++n) {
                const int T = key_tiles(p.nqt - 1 - it % p.nqt);
                const int ob = n & 1;
                for (int j = 0; j < T; ++j, ++g) {
                    issue_next_s();  // S_{g+1}
                    if constexpr (!STATS) {
                        const int sb = g & 1;
                        mbar_wait(&v_full[sb], (g >> 1) & 1);
                        mbar_wait(&p_full[sb], (g >> 1) & 1);
                        if (j == 0 && n >= 2) mbar_wait(&o_empty[ob], ((n >> 1) - 1) & 1);  // O buffer drained
                        PFT("mma_pv", g);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint8_t* v = sV + sb * kFKBytes;
                        const uint32_t od = tmem + 256 + ob * 128;
#pragma unroll
                        for (int kk = 0; kk < kFKeys / 16; ++kk) {  // 16 keys: 32-key chunk kk/2, 8-column group kk%2
                            const uint32_t pa = tmem + sb * kFKeys + (kk >> 1) * 32 + (kk & 1) * 8;
                            umma_ts(od, pa, desc_mn(v + kk * 2048), id_o, (j | kk) != 0);
                            if constexpr (BF16) umma_ts(od, pa + 16, desc_mn(v + kk * 2048), id_o, 1);
                        }
                        umma_commit(&v_empty[sb]);
                        umma_commit(&s_free[sb]);
                        if (j + 1 == T) umma_commit(&o_full[ob]);
                    }
                }
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ------------------------------------------------ rows: softmax / P / O
        const int q4 = warp & 3;      // TMEM lane quarter this warp may access
        const int hf = (warp - 4) >> 2;  // key half of each tile / O half
        const int rl = q4 * 32 + lane;
        const uint32_t tl = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
        int g = 0, n = 0;
        for (int it = first; it < last; ++it, ++n) {
            const int qt = p.nqt - 1 - it % p.nqt, z = it / p.nqt;
            const int T = key_tiles(qt);
            const int r = qt * kFTile + rl;
            const int qb = n & 1;
            const bool valid = r < p.s;
            const size_t zrow = static_cast<size_t>(z) * p.s;
            float mx = -INFINITY;  // pass 1: raw row max (this half's keys)
            float mc = 0.f;        // pass 2: row max x c1
            float l = 0.f;         // pass 2: sum of e (this half's keys)
            if constexpr (!STATS) {
                mbar_wait(&q_full[qb], (n >> 1) & 1);
                mc = valid ? sM[qb * 128 + rl] * p.c1 : 0.f;
                mbar_arrive(&q_empty[qb]);
            }
            unsigned cnt = 0;
            const bool last_row = r == p.s - 1;
            for (int j = 0; j < T; ++j, ++g) {
                const int sb = g & 1;
                // key tiles past the query tile's first row need the causal mask
                const bool diag = (j + 1) * NK - 1 > qt * kFTile;
                const uint32_t ca = tl + sb * NK + hf * HK;
                mbar_wait(&s_full[sb], (g >> 1) & 1);
                if (warp == 4 && lane == 0) PFT("row_s", g);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const int lim = valid ? min(r - j * NK - hf * HK, HK - 1) : -1;  // keys 0..lim of this half count
                if constexpr (STATS) {
                    // 128 keys per thread: two 64-key rounds of loads (register budget)
                    float m4[4] = {mx, mx, mx, mx};
#pragma unroll
                    for (int c0 = 0; c0 < HK; c0 += 64) {
                        float sv[64];
                        tmem_ld32(ca + c0, sv);
                        tmem_ld32(ca + c0 + 32, sv + 32);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (c0 + 64 == HK) {
                            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                            mbar_arrive(&s_free[sb]);
                        }
                        if (diag) {
#pragma unroll
                            for (int k = 0; k < 64; ++k)
                                if (c0 + k <= lim) m4[k & 3] = fmaxf(m4[k & 3], sv[k]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 64; ++k) m4[k & 3] = fmaxf(m4[k & 3], sv[k]);
                        }
                    }
                    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                } else {
                    if constexpr (BF16) {
                        // bf16: scalar row math and count (the packed path costs its hi + lo P a spill)
                        float sv[kFHK];
    #pragma unroll
                        for (int c = 0; c < kFHK / 32; ++c) tmem_ld32(ca + c * 32, sv + c * 32);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (warp == 4 && lane == 0) PFT("row_ld", g);
                        float l4[4] = {0.f, 0.f, 0.f, 0.f};
                        unsigned c4[4] = {0u, 0u, 0u, 0u};
                        if (diag) {
                            const float c1 = p.c1;
    #pragma unroll
                            for (int k = 0; k < kFHK; ++k) {
                                const float ex = ex2_all(fmaf(sv[k], c1, -mc));
                                const bool in = k <= lim;
                                const float e = in ? ex : 0.f;
                                c4[k & 3] += in & (e < 0.01f);
                                l4[k & 3] += e;
                                sv[k] = e;
                            }
                        } else {
    #pragma unroll
                            for (int k = 0; k < kFHK; ++k) {
                                const float e = ex2(fmaf(sv[k], p.c1, -mc));
                                c4[k & 3] += e < 0.01f;
                                l4[k & 3] += e;
                                sv[k] = e;
                            }
                        }
                        l += (l4[0] + l4[1]) + (l4[2] + l4[3]);
                        const unsigned ct = (c4[0] + c4[1]) + (c4[2] + c4[3]);
                        cnt += valid ? ct : 0u;
                        if (last_row) {
                            float* wl = p.wlast + zrow + j * kFKeys + hf * kFHK;
    #pragma unroll
                            for (int k = 0; k < kFHK; ++k)
                                if (k <= lim) wl[k] = sv[k];
                        }
    #pragma unroll
                        for (int c = 0; c < kFHK / 32; ++c) {  // 32-key chunks: hi in 16 columns, bf16 lo in the next 16
                            uint32_t pk[16];
    #pragma unroll
                            for (int i = 0; i < 16; ++i) pk[i] = pack2<BF16>(sv[c * 32 + 2 * i], sv[c * 32 + 2 * i + 1]);
                            tmem_st16(ca + c * 32, pk);
                            if constexpr (BF16) {
    #pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    pk[i] = pack2<true>(bf16_rest(sv[c * 32 + 2 * i]), bf16_rest(sv[c * 32 + 2 * i + 1]));
                                tmem_st16(ca + c * 32 + 16, pk);
                            }
                        }
                    } else {
                        float sv[kFHK];
    #pragma unroll
                        for (int c = 0; c < kFHK / 32; ++c) tmem_ld32(ca + c * 32, sv + c * 32);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (warp == 4 && lane == 0) PFT("row_ld", g);
                        // packed pairs: FFMA2 for S * c1 - max, FADD2 for l. fp16: the sparsity count
                        // runs on the packed P (HSET2 + HADD2 per pair, e < 0.01 in fp16), masked
                        // cells (P = 0) taken off after; bf16 counts the fp32 e.
                        constexpr bool kHCount = !BF16;
                        float2 l2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                        unsigned c4[4] = {0u, 0u, 0u, 0u};
                        const float2 c1v = make_float2(p.c1, p.c1), nmc = make_float2(-mc, -mc);
                        if (diag) {
    #pragma unroll
                            for (int k = 0; k < kFHK; k += 2) {
                                const float2 x = __ffma2_rn(make_float2(sv[k], sv[k + 1]), c1v, nmc);
                                const float x0 = ex2_all(x.x), x1 = ex2_all(x.y);
                                const bool in0 = k <= lim, in1 = k + 1 <= lim;
                                const float e0 = in0 ? x0 : 0.f, e1 = in1 ? x1 : 0.f;
                                if (!kHCount) {
                                    c4[k & 3] += in0 & (e0 < 0.01f);
                                    c4[(k + 1) & 3] += in1 & (e1 < 0.01f);
                                }
                                l2[(k >> 1) & 1] = __fadd2_rn(l2[(k >> 1) & 1], make_float2(e0, e1));
                                sv[k] = e0;
                                sv[k + 1] = e1;
                            }
                        } else {
    #pragma unroll
                            for (int k = 0; k < kFHK; k += 2) {
                                const float2 x = __ffma2_rn(make_float2(sv[k], sv[k + 1]), c1v, nmc);
                                const float e0 = ex2(x.x), e1 = ex2(x.y);
                                if (!kHCount) {
                                    c4[k & 3] += e0 < 0.01f;
                                    c4[(k + 1) & 3] += e1 < 0.01f;
                                }
                                l2[(k >> 1) & 1] = __fadd2_rn(l2[(k >> 1) & 1], make_float2(e0, e1));
                                sv[k] = e0;
                                sv[k + 1] = e1;
                            }
                        }
                        l += (l2[0].x + l2[0].y) + (l2[1].x + l2[1].y);
                        if (last_row) {
                            float* wl = p.wlast + zrow + j * kFKeys + hf * kFHK;
    #pragma unroll
                            for (int k = 0; k < kFHK; ++k)
                                if (k <= lim) wl[k] = sv[k];
                        }
                        __half2 hc = __floats2half2_rn(0.f, 0.f);
                        const __half2 thr = __floats2half2_rn(0.01f, 0.01f);
    #pragma unroll
                        for (int c = 0; c < kFHK / 32; ++c) {  // 32-key chunks: hi in 16 columns, bf16 lo in the next 16
                            uint32_t pk[16];
    #pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                pk[i] = pack2<BF16>(sv[c * 32 + 2 * i], sv[c * 32 + 2 * i + 1]);
                                if constexpr (kHCount) {
                                    __half2 ph;
                                    memcpy(&ph, &pk[i], 4);
                                    hc = __hadd2(hc, __hlt2(ph, thr));
                                }
                            }
                            tmem_st16(ca + c * 32, pk);
                            if constexpr (BF16) {
    #pragma unroll
                                for (int i = 0; i < 16; ++i)
                                    pk[i] = pack2<true>(bf16_rest(sv[c * 32 + 2 * i]), bf16_rest(sv[c * 32 + 2 * i + 1]));
                                tmem_st16(ca + c * 32 + 16, pk);
                            }
                        }
                        unsigned ct;
                        if constexpr (kHCount) {  // masked cells (k > lim) hold P = 0: not part of the count
                            const int kept = lim < 0 ? 0 : min(lim + 1, kFHK);
                            ct = static_cast<unsigned>(__half2float(__low2half(hc)) + __half2float(__high2half(hc))) -
                                 static_cast<unsigned>(kFHK - kept);
                        } else {
                            ct = (c4[0] + c4[1]) + (c4[2] + c4[3]);
                        }
                        cnt += valid ? ct : 0u;
                    }
                    if (warp == 4 && lane == 0) PFT("row_math", g);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    mbar_arrive(&p_full[sb]);
                    if (warp == 4 && lane == 0) PFT("row_p", g);
                }
            }
            // combine the two key halves of each row
            float* red = sR + (n & 1) * 256;
            red[hf * 128 + rl] = STATS ? mx : l;
            named_sync(1, 256);
            const float other = red[(hf ^ 1) * 128 + rl];
            if constexpr (STATS) {
                if (hf == 0 && valid) p.mrow[static_cast<size_t>(z) * p.s_pad + r] = fmaxf(mx, other);
            } else {
                l += other;
                if (hf == 0) {
                    if (last_row) p.llast[z] = l;
                    const int ob = n & 1;
                    if (n >= 2) mbar_wait(&o_empty[ob], ((n >> 1) - 1) & 1);  // sL[ob] of item n - 2 read
                    sL[ob * 128 + rl] = 1.0f / l;
                    mbar_arrive(&l_full[ob]);
                }
#pragma unroll
                for (int o2 = 16; o2 > 0; o2 >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o2);
                if (lane == 0 && cnt) atomicAdd(&p.below[z], cnt);
            }
        }
    } else if (!STATS && (warp >= 12 || warp == 2 || warp == 3)) {
        // ------------------------------------------- O epilogue (lane quarters 2, 3, 0, 1)
        const int q4 = warp & 3;
        const int rl = q4 * 32 + lane;
        const uint32_t tl = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
        int n = 0;
        for (int it = first; it < last; ++it, ++n) {
            const int qt = p.nqt - 1 - it % p.nqt, z = it / p.nqt;
            const int r = qt * kFTile + rl;
            const bool valid = r < p.s;
            const int ob = n & 1;
            mbar_wait(&l_full[ob], (n >> 1) & 1);
            const float inv_l = sL[ob * 128 + rl];
            mbar_wait(&o_full[ob], (n >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const size_t row0 =
                (static_cast<size_t>(z / p.H) * p.s + r) * p.HD + static_cast<size_t>(z % p.H) * 128;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                float o[32];
                tmem_ld32(tl + 256 + ob * 128 + c * 32, o);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (!valid) continue;
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] *= inv_l;
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
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&o_empty[ob]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
#ifdef PF_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const char* names[7] = {"tma_k", "mma_s", "row_s", "row_ld", "row_math", "row_p", "mma_pv"};
        const long long t0 = g_pft[STATS ? 0 : 1][0][0];
        for (int gg = 0; gg < 32; ++gg) {
            printf("P%d g=%2d", STATS ? 1 : 2, gg);
            for (int t = 0; t < 7; ++t) printf(" %s=%8lld", names[t], g_pft[STATS ? 0 : 1][t][gg] - t0);
            printf("\n");
        }
    }
#endif
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    }
}

// ============================================================================
// 2-CTA version (cta_group::2): a cluster of two CTAs on one TPC processes a
// 256-query super-tile; the leader's single thread issues M = 256 MMAs whose
// A / D halves live in each CTA (its 128 query rows) and whose B operand is
// split by N (each CTA stages half of the key tile, or half of V's head
// dims). scripts/mma2_probe.cu: an M = 256, N = 128 2-CTA MMA costs ~86
// (SS) / ~94 (TS) cycles against ~163 for the 1-CTA M = 128 one -- four times
// the work per SM-cycle at N = 128. Barrier protocol:
//  - TMA: each CTA loads its Q tile and its B half into its own shared memory
//    with .cta_group::2, completing bytes on the LEADER's full barrier (the
//    leader posts expect_tx for both halves); each CTA recycles a stage on
//    its own empty barrier, which the leader's commit multicasts to both.
//  - rows / epilogue of both CTAs arrive (one lane per warp) on the leader's
//    p_full / s_free / o_pair barriers through shared::cluster addresses; the
//    leader's commits multicast s_full / o_full / q_empty to both CTAs.
// Rows and epilogue run per CTA exactly as in the 1-CTA kernel, on the CTA's
// own TMEM lanes.
// K / V shared-memory stages. V runs six tiles deep: one TMA thread issues
// K(g) then V(g), and V(g) waits for P.V(g - stages) -- with three stages
// the P.V stream waited ~6 k cycles per tile for V (PF_TRACE: the V load
// latency every three tiles), and K behind it.
template <bool STATS>
struct F2Stages {
    static constexpr int K = STATS ? 4 : 3;
    static constexpr int V = 6;
};
// Warps as the 1-CTA kernel: 0 TMA, 1 MMA, 4..11 rows (two per TMEM lane
// quarter, each half of a tile's keys), 2, 3, 12, 13 the O epilogue. TMEM:
// two S / P buffers, two O buffers.
constexpr int kF2RowQ = 2;
constexpr int kF2Threads = 448;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same offset in the leader CTA (rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
    return r;
}
// (default .release.cta semantics, as CUTLASS's ClusterBarrier::arrive: the
// TMEM data it publishes is ordered by the tcgen05 fences, and a cluster-scope
// release measured as the pass's top stall)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA 3D load into this CTA's shared memory, bytes completed on the leader's
// barrier at the same offset (peer bit cleared, as CUTLASS's 2SM loads)
__device__ __forceinline__ void tma3d_2sm(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar) & 0xFEFFFFFFu)
        : "memory");
}
__device__ __forceinline__ void umma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// completion of the leader's MMAs so far -> the barrier at this offset in the CTAs of `mask`
__device__ __forceinline__ void umma2_commit(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// MN-major B of one CTA's half of V: a single 64-dim SW128 atom column, 8-key groups 1024 B apart
__device__ __forceinline__ uint64_t desc_mn64(const void* p) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | (uint64_t(kFKHalf >> 4) << 16) | ((1024ull >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}

template <bool BF16, bool STATS>
struct Flash2Smem {
    static constexpr int NK = STATS ? 2 * kFKeys : kFKeys;  // keys per S tile
    static constexpr int KHB = (NK / 2) * 128;  // one 64-column SW128 box of this CTA's key half
    static constexpr int KB = 2 * KHB;          // this CTA's key half, both 64-column boxes
    static constexpr int VB = kFKeys * 128;     // this CTA's 64 head dims of a 128-key V tile
    static constexpr int kQ = 0;                                     // [2] query tiles
    static constexpr int kK = kQ + 2 * kFTileBytes;                  // [K stages] key halves
    static constexpr int kV = kK + F2Stages<STATS>::K * KB;          // [V stages] value halves (pass 2)
    static constexpr int kM = kV + (STATS ? 0 : F2Stages<STATS>::V * VB);  // [2][128] row max (pass 2)
    static constexpr int kR = kM + 2 * 128 * 4;                      // [2][kF2RowQ][128] per-quarter row partials
    static constexpr int kL = kR + 2 * kF2RowQ * 128 * 4;            // [2][128] 1 / l per O buffer
    static constexpr int kBar = kL + 2 * 128 * 4;
    static constexpr int kNBar = 48;
    static constexpr int kBytes = kBar + kNBar * 8 + 16 + 1024;
    static_assert(kBytes <= 227 * 1024, "shared memory");
};

#ifdef PF_TRACE
__device__ long long g_pft2[2][8][32];
#define PFT2(slot, gg)                                                                     \
    do {                                                                                   \
        if (blockIdx.x < 2 && (gg) < 32) g_pft2[blockIdx.x][slot][gg] = clock64();           \
    } while (0)
#else
#define PFT2(slot, gg) \
    do {               \
    } while (0)
#endif
template <bool BF16, bool STATS>
__global__ void __launch_bounds__(kF2Threads, 1)
    flash2_prefill_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                          const __grid_constant__ CUtensorMap map_v, const FlashParams p) {
    using L = Flash2Smem<BF16, STATS>;
    constexpr int NK = L::NK, KHB = L::KHB, KB = L::KB, VB = L::VB;
    constexpr int HK = NK / kF2RowQ;  // keys per row thread per tile
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    uint8_t* sQ = sm + L::kQ;
    uint8_t* sK = sm + L::kK;
    uint8_t* sV = sm + L::kV;
    float* sM = reinterpret_cast<float*>(sm + L::kM);
    float* sR = reinterpret_cast<float*>(sm + L::kR);
    float* sL = reinterpret_cast<float*>(sm + L::kL);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::kBar);
    uint64_t* q_full = bar;         // [2] leader: both Q tiles landed
    uint64_t* q_empty = bar + 2;    // [2] each: leader's commit (+ own rows read sM)
    constexpr int KS = F2Stages<STATS>::K, VS = F2Stages<STATS>::V;
    uint64_t* k_full = bar + 4;     // [4] leader: both key halves landed
    uint64_t* k_empty = bar + 8;    // [4] each: leader's commit
    uint64_t* v_full = bar + 12;    // [6] leader
    uint64_t* v_empty = bar + 18;   // [6] each
    uint64_t* s_full = bar + 24;    // [kSB] each: S in this CTA's TMEM
    uint64_t* s_free = bar + 27;    // [kSB] leader: pass 1 rows of both read S (16 warps); pass 2 P.V consumed P
    uint64_t* p_full = bar + 30;    // [kSB] leader: rows of both wrote P (16 warps)
    uint64_t* o_full = bar + 33;    // [2] each: the item's O complete
    uint64_t* o_pair = bar + 35;    // [2] leader: both epilogues read O (8 warps)
    uint64_t* o_empty = bar + 37;   // [2] each: own epilogue read O and 1 / l (128)
    uint64_t* l_full = bar + 39;    // [2] each: rows wrote 1 / l (128)
    uint64_t* m_full = bar + 41;    // [2] each: own row max landed (pass 2)
    constexpr int kSB = 2;  // S / P buffers
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + L::kNBar);

    if (threadIdx.x == 0) {
        for (int i = 0; i < 43; ++i) mbar_init(&bar[i], 1);
        if (!STATS) {
            mbar_init(&q_empty[0], 257);  // the leader's commit + this CTA's 256 row threads (sM read)
            mbar_init(&q_empty[1], 257);
        }
        for (int i = 0; i < kSB; ++i) {
            if (STATS) mbar_init(&s_free[i], 16);  // 8 row warps x 2 CTAs
            mbar_init(&p_full[i], 16);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&o_pair[i], 8);  // 4 epilogue warps x 2 CTAs
            mbar_init(&o_empty[i], 128);
            mbar_init(&l_full[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    // Work items: (sequence-head z, 256-query super-tile qs), heaviest first,
    // contiguous runs per CTA pair; rank r owns query tile 2 qs + r.
    const int nqs = (p.nqt + 1) / 2;
    const int items = p.Z * nqs;
    const int npairs = gridDim.x / 2, pair = blockIdx.x / 2;
    const int first = static_cast<int>(static_cast<long long>(items) * pair / npairs);
    const int last = static_cast<int>(static_cast<long long>(items) * (pair + 1) / npairs);
    const int nkt = (p.s + NK - 1) / NK;
    auto key_tiles = [&](int qs) { return min(nkt, (qs * 2 * kFTile + 2 * kFTile + NK - 1) / NK); };

    if (warp == 0) {
        // ------------------------------------------------------------ TMA (both CTAs)
        if (lane == 0) {
            int g = 0, n = 0;
            for (int it = first; it < last; ++it, ++n) {
                const int qs = nqs - 1 - it % nqs, z = it / nqs;
                const int qt = 2 * qs + static_cast<int>(rank);
                const int b = z / p.H, xq = (z % p.H) * 128;
                const int T = key_tiles(qs);
                const int qb = n & 1;
                if (n >= 2) mbar_wait(&q_empty[qb], ((n >> 1) - 1) & 1);
                if (leader) mbar_arrive_expect_tx(&q_full[qb], 2 * kFTileBytes);
                uint8_t* dq = sQ + qb * kFTileBytes;
                tma3d_2sm(dq, &map_q, xq, qt * kFTile, b, &q_full[qb]);
                tma3d_2sm(dq + kFHalf, &map_q, xq + 64, qt * kFTile, b, &q_full[qb]);
                if constexpr (!STATS) {
                    mbar_arrive_expect_tx(&m_full[qb], 512);
                    bulk_g2s(sM + qb * 128, p.mrow + static_cast<size_t>(z) * p.s_pad + qt * kFTile, 512, &m_full[qb],
                             policy_evict_first());
                }
                for (int j = 0; j < T; ++j, ++g) {
                    const int st = g % KS;
                    if (g >= KS) mbar_wait(&k_empty[st], ((g / KS) - 1) & 1);
                    if (leader) mbar_arrive_expect_tx(&k_full[st], 2 * KB);
                    PFT2(0, g);
                    uint8_t* dk = sK + st * KB;
                    const int key0 = j * NK + static_cast<int>(rank) * (NK / 2);
                    tma3d_2sm(dk, &map_k, xq, key0, b, &k_full[st]);
                    tma3d_2sm(dk + KHB, &map_k, xq + 64, key0, b, &k_full[st]);
                    if constexpr (!STATS) {
                        const int vt = g % VS;
                        if (g >= VS) mbar_wait(&v_empty[vt], ((g / VS) - 1) & 1);
                        if (leader) mbar_arrive_expect_tx(&v_full[vt], 2 * VB);
                        PFT2(3, g);
                        tma3d_2sm(sV + vt * VB, &map_v, p.HD + xq + static_cast<int>(rank) * 64, j * kFKeys, b,
                                  &v_full[vt]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------- MMA (the leader's one thread)
        if (leader && lane == 0) {
            constexpr uint32_t id_s = (1u << 4) | ((BF16 ? 1u : 0u) << 7) | ((BF16 ? 1u : 0u) << 10) |
                                      (uint32_t(NK >> 3) << 17) | (uint32_t(256 >> 4) << 24);
            constexpr uint32_t id_o = (1u << 4) | ((BF16 ? 1u : 0u) << 7) | ((BF16 ? 1u : 0u) << 10) | (1u << 16) |
                                      (uint32_t(128 >> 3) << 17) | (uint32_t(256 >> 4) << 24);
            int g = 0, n = 0;
            auto issue_s = [&](int gg, const uint8_t* q) {
                const int sb = gg % kSB, ks = gg % KS;
                if (gg >= kSB) mbar_wait(&s_free[sb], ((gg / kSB) - 1) & 1);
                mbar_wait(&k_full[ks], (gg / KS) & 1);
                PFT2(1, gg);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint8_t* k = sK + ks * KB;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma2(tmem + sb * NK, desc_k(q + (kk >> 2) * kFHalf + (kk & 3) * 32),
                          desc_k(k + (kk >> 2) * KHB + (kk & 3) * 32), id_s, kk > 0);
                umma2_commit(&k_empty[ks], 3);
                umma2_commit(&s_full[sb], 3);
            };
            int itS = first, jS = 0, nS = 0, gS = 0;
            auto issue_next_s = [&]() {
                if (itS >= last) return;
                const int TS = key_tiles(nqs - 1 - itS % nqs);
                const int qb = nS & 1;
                if (jS == 0) mbar_wait(&q_full[qb], (nS >> 1) & 1);
                issue_s(gS++, sQ + qb * kFTileBytes);
                if (++jS == TS) {
                    umma2_commit(&q_empty[qb], 3);  // the item's last S: both Q tiles are free
                    jS = 0;
                    ++itS;
                    ++nS;
                }
            };
            issue_next_s();
            for (int it = first; it < last; ++it, ++n) {
                const int T = key_tiles(nqs - 1 - it % nqs);
                const int ob = n & 1;
                for (int j = 0; j < T; ++j, ++g) {
                    issue_next_s();  // S_{g+1}
                    if constexpr (!STATS) {
                        const int sb = g % kSB, vs = g % VS;
                        mbar_wait(&v_full[vs], (g / VS) & 1);
                        mbar_wait(&p_full[sb], (g / kSB) & 1);
                        if (j == 0 && n >= 2) mbar_wait(&o_pair[ob], ((n >> 1) - 1) & 1);  // both drained this O buffer
                        PFT2(6, g);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint8_t* v = sV + vs * VB;
                        const uint32_t od = tmem + 256 + ob * 128;
#pragma unroll
                        for (int kk = 0; kk < kFKeys / 16; ++kk) {
                            const uint32_t pa = tmem + sb * kFKeys + (kk >> 1) * 32 + (kk & 1) * 8;
                            umma2_ts(od, pa, desc_mn64(v + kk * 2048), id_o, (j | kk) != 0);
                            if constexpr (BF16) umma2_ts(od, pa + 16, desc_mn64(v + kk * 2048), id_o, 1);
                        }
                        umma2_commit(&v_empty[vs], 3);
                        umma2_commit(&s_free[sb], 1);
                        if (j + 1 == T) umma2_commit(&o_full[ob], 3);
                    }
                }
            }
        }
    } else if (warp >= 4 && warp < 4 + 4 * kF2RowQ) {
        // ------------------------------------------ rows: softmax / P (this CTA's 128 rows)
        const int q4 = warp & 3;
        const int hf = (warp - 4) >> 2;  // key quarter
        const int rl = q4 * 32 + lane;
        const uint32_t tl = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
        const uint32_t s_free_l = leader_addr(&s_free[0]), p_full_l = leader_addr(&p_full[0]);
        int g = 0, n = 0;
        for (int it = first; it < last; ++it, ++n) {
            const int qs = nqs - 1 - it % nqs, z = it / nqs;
            const int qt = 2 * qs + static_cast<int>(rank);
            const int T = key_tiles(qs);
            const int r = qt * kFTile + rl;
            const int qb = n & 1;
            const bool valid = r < p.s;
            const size_t zrow = static_cast<size_t>(z) * p.s;
            float mx = -INFINITY;
            float mc = 0.f;
            float l = 0.f;
            if constexpr (!STATS) {
                mbar_wait(&m_full[qb], (n >> 1) & 1);
                mc = valid ? sM[qb * 128 + rl] * p.c1 : 0.f;
                mbar_arrive(&q_empty[qb]);
            }
            unsigned cnt = 0;
            const bool last_row = r == p.s - 1;
            for (int j = 0; j < T; ++j, ++g) {
                const int sb = g % kSB;
                const bool diag = (j + 1) * NK - 1 > qt * kFTile;
                const uint32_t ca = tl + sb * NK + hf * HK;
                mbar_wait(&s_full[sb], (g / kSB) & 1);
                if (warp == 4 && lane == 0) PFT2(2, g);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const int lim = valid ? min(r - j * NK - hf * HK, HK - 1) : -1;
                if constexpr (STATS) {
                    float m4[4] = {mx, mx, mx, mx};
#pragma unroll
                    for (int c0 = 0; c0 < HK; c0 += 32) {
                        float sv[32];
                        tmem_ld32(ca + c0, sv);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (c0 + 32 == HK) {
                            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster(s_free_l + sb * 8);
                        }
                        if (diag) {
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                if (c0 + k <= lim) m4[k & 3] = fmaxf(m4[k & 3], sv[k]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 32; ++k) m4[k & 3] = fmaxf(m4[k & 3], sv[k]);
                        }
                    }
                    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                } else {
                    // 32-key chunks (register budget of 576 threads); packed pairs: FFMA2 for
                    // S * c1 - max, FADD2 for l
                    float2 l2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                    unsigned c4[4] = {0u, 0u, 0u, 0u};
                    const float2 c1v = make_float2(p.c1, p.c1), nmc = make_float2(-mc, -mc);
#pragma unroll
                    for (int c0 = 0; c0 < HK; c0 += 32) {
                        float sv[32];
                        tmem_ld32(ca + c0, sv);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (diag && __all_sync(0xffffffffu, lim < c0)) {
                            // keys past every row of the warp (the causal triangle, or the pair's
                            // last tile for rank 0's rows): P = 0, no exps
#pragma unroll
                            for (int k = 0; k < 32; ++k) sv[k] = 0.f;
                        } else if (diag) {
#pragma unroll
                            for (int k = 0; k < 32; k += 2) {
                                const float2 x = __ffma2_rn(make_float2(sv[k], sv[k + 1]), c1v, nmc);
                                const bool in0 = c0 + k <= lim, in1 = c0 + k + 1 <= lim;
                                const float x0 = ex2_all(x.x), x1 = ex2_all(x.y);
                                const float e0 = in0 ? x0 : 0.f, e1 = in1 ? x1 : 0.f;
                                c4[k & 3] += in0 & (e0 < 0.01f);
                                c4[(k + 1) & 3] += in1 & (e1 < 0.01f);
                                l2[(k >> 1) & 1] = __fadd2_rn(l2[(k >> 1) & 1], make_float2(e0, e1));
                                sv[k] = e0;
                                sv[k + 1] = e1;
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < 32; k += 2) {
                                const float2 x = __ffma2_rn(make_float2(sv[k], sv[k + 1]), c1v, nmc);
                                const float e0 = ex2(x.x), e1 = ex2(x.y);
                                c4[k & 3] += e0 < 0.01f;
                                c4[(k + 1) & 3] += e1 < 0.01f;
                                l2[(k >> 1) & 1] = __fadd2_rn(l2[(k >> 1) & 1], make_float2(e0, e1));
                                sv[k] = e0;
                                sv[k + 1] = e1;
                            }
                        }
                        if (last_row) {
                            float* wl = p.wlast + zrow + j * kFKeys + hf * HK + c0;
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                if (c0 + k <= lim) wl[k] = sv[k];
                        }
                        uint32_t pk[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) pk[i] = pack2<BF16>(sv[2 * i], sv[2 * i + 1]);
                        tmem_st16(ca + c0, pk);
                        if constexpr (BF16) {
#pragma unroll
                            for (int i = 0; i < 16; ++i) pk[i] = pack2<true>(bf16_rest(sv[2 * i]), bf16_rest(sv[2 * i + 1]));
                            tmem_st16(ca + c0 + 16, pk);
                        }
                    }
                    l += (l2[0].x + l2[0].y) + (l2[1].x + l2[1].y);
                    const unsigned ct = (c4[0] + c4[1]) + (c4[2] + c4[3]);
                    cnt += valid ? ct : 0u;
                    if (warp == 4 && lane == 0) PFT2(4, g);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(p_full_l + sb * 8);
                    if (warp == 4 && lane == 0) PFT2(5, g);
                }
            }
            // combine the key quarters of each row (fixed order)
            float* red = sR + (n & 1) * (kF2RowQ * 128);
            red[hf * 128 + rl] = STATS ? mx : l;
            named_sync(1, kF2RowQ * 128);
            if constexpr (STATS) {
                if (hf == 0 && valid) {
                    float m = red[rl];
#pragma unroll
                    for (int q = 1; q < kF2RowQ; ++q) m = fmaxf(m, red[q * 128 + rl]);
                    p.mrow[static_cast<size_t>(z) * p.s_pad + r] = m;
                }
            } else {
                l = red[rl];
#pragma unroll
                for (int q = 1; q < kF2RowQ; ++q) l += red[q * 128 + rl];
                if (hf == 0) {
                    if (last_row) p.llast[z] = l;
                    const int ob = n & 1;
                    if (n >= 2) mbar_wait(&o_empty[ob], ((n >> 1) - 1) & 1);  // sL[ob] of item n - 2 read
                    sL[ob * 128 + rl] = 1.0f / l;
                    mbar_arrive(&l_full[ob]);
                }
#pragma unroll
                for (int o2 = 16; o2 > 0; o2 >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o2);
                if (lane == 0 && cnt) atomicAdd(&p.below[z], cnt);
            }
        }
    } else if (!STATS && (warp >= 4 + 4 * kF2RowQ || warp == 2 || warp == 3)) {
        // ------------------------------------------- O epilogue (this CTA's 128 rows)
        const int q4 = warp & 3;
        const int rl = q4 * 32 + lane;
        const uint32_t tl = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
        const uint32_t o_pair_l = leader_addr(&o_pair[0]);
        int n = 0;
        for (int it = first; it < last; ++it, ++n) {
            const int qs = nqs - 1 - it % nqs, z = it / nqs;
            const int qt = 2 * qs + static_cast<int>(rank);
            const int r = qt * kFTile + rl;
            const bool valid = r < p.s;
            const int ob = n & 1;
            mbar_wait(&l_full[ob], (n >> 1) & 1);
            const float inv_l = sL[ob * 128 + rl];
            mbar_wait(&o_full[ob], (n >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const size_t row0 =
                (static_cast<size_t>(z / p.H) * p.s + r) * p.HD + static_cast<size_t>(z % p.H) * 128;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                float o[32];
                tmem_ld32(tl + 256 + ob * 128 + c * 32, o);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (!valid) continue;
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] *= inv_l;
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
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&o_empty[ob]);
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(o_pair_l + ob * 8);
            if (warp == 2 && lane == 0) PFT2(7, n);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
#ifdef PF_TRACE
    cluster_sync_all();
    if (blockIdx.x == 0 && threadIdx.x == 0 && !STATS) {
        const char* names[8] = {"tma_k", "mma_s", "row_s", "tma_v", "row_math", "row_p", "mma_pv", "epi_rel(n)"};
        const long long t0 = g_pft2[0][0][0];
        for (int rk = 0; rk < 2; ++rk)
            for (int gg = 0; gg < 24; ++gg) {
                printf("Q2 r%d g=%2d", rk, gg);
                for (int t = 0; t < 8; ++t) printf(" %s=%7lld", names[t], g_pft2[rk][t][gg] - t0);
                printf("\n");
            }
    }
#endif
    cluster_sync_all();  // the peer's last MMAs and arrives are done before the TMEM goes
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    }
}

// importance[b][j] = sum_h e_h[j] / l_h (head order, fp64): engine.hpp:
// 508-512 seeds each head's accumulator with the last attention row,
// attention.hpp:77-85 sums them. Block x = 0 also folds the per-head
// sparsity counts (engine.hpp:513-518).
__global__ void prefill_seed_kernel(const float* __restrict__ wlast, const float* __restrict__ llast,
                                    const unsigned* __restrict__ below, double* __restrict__ imp,
                                    double* __restrict__ psp, int H, int s, long long imp_ld, int h_div) {
    extern __shared__ double inv_l[];  // [H] 1 / l per head, once per block (not one fp64 divide per cell)
    const int b = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    for (int h = threadIdx.x; h < H; h += blockDim.x) inv_l[h] = 1.0 / static_cast<double>(llast[b * H + h]);
    if (psp != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
        const double cells = 0.5 * static_cast<double>(s) * static_cast<double>(s + 1);
        double sp = 0.0;
        for (int h = 0; h < H; ++h) sp += static_cast<double>(below[b * H + h]) / cells;
        psp[b] = sp / static_cast<double>(h_div);  // h_div = all heads of the model (H unless head-sharded)
    }
    __syncthreads();
    if (j >= s) return;
    const float* w = wlast + static_cast<size_t>(b) * H * s + j;
    double acc = 0.0;
#pragma unroll 8
    for (int h = 0; h < H; ++h) acc = fma(static_cast<double>(w[static_cast<size_t>(h) * s]), inv_l[h], acc);
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
// beyond), box {64 cols, box_tokens, 1}.
bool map3d(CUtensorMap* m, const void* base, bool bf16, uint64_t cols, uint64_t tokens, uint64_t seqs,
           uint64_t row_bytes, uint64_t seq_bytes, uint32_t box_tokens) {
    EncodeFn fn = encoder();
    if (!fn) return false;
    const cuuint64_t dims[3] = {cols, tokens, seqs};
    const cuuint64_t strides[2] = {row_bytes, seq_bytes};
    const cuuint32_t box[3] = {64, box_tokens, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base),
              dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool BF16, bool STATS>
cudaError_t run_flash(const CUtensorMap& mq, const CUtensorMap& mkv, const FlashParams& p, cudaStream_t st) {
    constexpr int smem = FlashSmem<BF16, STATS>::kBytes;
    const void* fn = reinterpret_cast<const void*>(&flash_prefill_kernel<BF16, STATS>);
    static std::once_flag once;  // a constant size: set the attribute once per instantiation
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [&] { attr = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
    cudaError_t e = attr;
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<CUtensorMap*>(&mq), const_cast<CUtensorMap*>(&mkv), const_cast<FlashParams*>(&p)};
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::max(1, std::min(sms, p.Z * p.nqt));
    e = cudaLaunchKernel(fn, dim3(grid), dim3(kFThreads), args, smem, st);
    count_launch();
    return e;
}

// The 2-CTA kernel: clusters of two CTAs (one TPC), one pair per two SMs.
template <bool BF16, bool STATS>
cudaError_t run_flash2(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const FlashParams& p,
                       cudaStream_t st) {
    constexpr int smem = Flash2Smem<BF16, STATS>::kBytes;
    const void* fn = reinterpret_cast<const void*>(&flash2_prefill_kernel<BF16, STATS>);
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [&] { attr = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
    if (attr != cudaSuccess) return attr;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int items = p.Z * ((p.nqt + 1) / 2);
    const int pairs = std::max(1, std::min(sms / 2, items));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kF2Threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    void* args[] = {const_cast<CUtensorMap*>(&mq), const_cast<CUtensorMap*>(&mk), const_cast<CUtensorMap*>(&mv),
                    const_cast<FlashParams*>(&p)};
    const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    count_launch();
    return e;
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }


}  // namespace

// mrow fp32 [Z][s_pad], wlast fp32 [Z][s], llast fp32 [Z], below u32 [Z]
size_t prefill_scratch_bytes(int B, int H, int s) {
    const size_t Z = static_cast<size_t>(B) * H, s_pad = (static_cast<size_t>(s) + kFTile - 1) / kFTile * kFTile;
    return align256(Z * s_pad * 4) + align256(Z * s * 4) + align256(Z * 4) + align256(Z * 4);
}

// Causal prefill of one cache layer (see the file comment). kv: layer base
// of a 16-bit cache [B][Ncap][2][H][D]; q/out: [B][s][H][D] (out fp32 when
// out_f32); imp: layer importance [B][imp_ld]; psp (nullable): [B].
cudaError_t launch_prefill(bool bf16, bool out_f32, const void* kv, const void* q, void* out, double* imp,
                           long long imp_ld, double* psp, int B, int H, int D, int Ncap, int s, uint8_t* scratch,
                           cudaStream_t st, int h_div) {
    if (D != 128) return cudaErrorInvalidValue;
    const int Z = B * H, nqt = (s + kFTile - 1) / kFTile;
    const uint64_t HD = static_cast<uint64_t>(H) * D;
    const int s_pad = nqt * kFTile;
    float* mrow = reinterpret_cast<float*>(scratch);
    float* wlast = reinterpret_cast<float*>(scratch + align256(static_cast<size_t>(Z) * s_pad * 4));
    float* llast = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(wlast) + align256(static_cast<size_t>(Z) * s * 4));
    unsigned* below = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(llast) + align256(static_cast<size_t>(Z) * 4));
    cudaError_t e = cudaMemsetAsync(below, 0, static_cast<size_t>(Z) * 4, st);
    if (e != cudaSuccess) return e;
    CUtensorMap mq, mkv, mk256;  // mk256: the max pass's 256-key tiles
    if (!map3d(&mq, q, bf16, HD, s, B, HD * 2, HD * 2 * s, kFTile) ||
        !map3d(&mkv, kv, bf16, 2 * HD, s, B, 2 * HD * 2, 2 * HD * 2 * Ncap, kFKeys) ||
        !map3d(&mk256, kv, bf16, 2 * HD, s, B, 2 * HD * 2, 2 * HD * 2 * Ncap, 2 * kFKeys))
        return cudaErrorInvalidValue;
    FlashParams p{};
    p.s = s;
    p.H = H;
    p.HD = static_cast<int>(HD);
    p.Z = Z;
    p.nqt = nqt;
    p.s_pad = s_pad;
    p.c1 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(D)));
    p.mrow = mrow;
    p.llast = llast;
    p.out = out;
    p.out_f32 = out_f32 ? 1 : 0;
    p.wlast = wlast;
    p.below = below;
    // CTA pairs from s = 1536 on: measured faster at s = 2048 (1.96 vs 2.17 ms, config 5's prompt), slower
    // at s = 512 / 1024 (0.43 vs 0.39 ms, 3.63 vs 3.48 ms): with the MMAs four times cheaper, both kernels
    // are bound by the row softmax, and the pair's lock-step costs more on short items.
    // SKV_PREFILL_1CTA=1 / SKV_PREFILL_2CTA=1 force one kernel (A/B, tests).
    static const bool force1 = std::getenv("SKV_PREFILL_1CTA") != nullptr;
    static const bool force2 = std::getenv("SKV_PREFILL_2CTA") != nullptr;
    const bool one_cta = force1 || (!force2 && s < 1536);
    if (one_cta) {
        e = bf16 ? run_flash<true, true>(mq, mk256, p, st) : run_flash<false, true>(mq, mk256, p, st);
        if (e != cudaSuccess) return e;
        e = bf16 ? run_flash<true, false>(mq, mkv, p, st) : run_flash<false, false>(mq, mkv, p, st);
        if (e != cudaSuccess) return e;
    } else {
        // each CTA of a pair stages half a key tile: 128 keys of the max pass's 256, 64 of the P.V
        // pass's 128; and 64 of V's 128 head dims
        CUtensorMap mk64, mv64;
        if (!map3d(&mk64, kv, bf16, 2 * HD, s, B, 2 * HD * 2, 2 * HD * 2 * Ncap, kFKeys / 2) ||
            !map3d(&mv64, kv, bf16, 2 * HD, s, B, 2 * HD * 2, 2 * HD * 2 * Ncap, kFKeys))
            return cudaErrorInvalidValue;
        e = bf16 ? run_flash2<true, true>(mq, mkv, mkv, p, st) : run_flash2<false, true>(mq, mkv, mkv, p, st);
        if (e != cudaSuccess) return e;
        e = bf16 ? run_flash2<true, false>(mq, mk64, mv64, p, st) : run_flash2<false, false>(mq, mk64, mv64, p, st);
        if (e != cudaSuccess) return e;
    }
    prefill_seed_kernel<<<dim3((s + 127) / 128, B), 128, static_cast<size_t>(H) * 8, st>>>(
        wlast, llast, below, imp, psp, H, s, imp_ld, h_div > 0 ? h_div : H);
    count_launch();
    return cudaGetLastError();
}

}  // namespace skv_impl
