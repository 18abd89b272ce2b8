// skv_prefill.cu -- dense causal prefill attention on tcgen05 tensor cores and
// the accumulator seeding that starts the SWA decode.
//
// Engine::prefill (engine.hpp:485-529) runs dense_attention (attention.hpp:
// 91-117) with the causal mask for every prompt position, seeds each head's
// accumulator with the LAST attention row (engine.hpp:508-512) and records
// attention_sparsity(aw, 0.01, causal) per layer (engine.hpp:513-518). Per
// (sequence, head) z:
//   1. S = Q K^T          batched tcgen05 GEMM, K read in place from the cache
//                         (2D tensor maps with per-(b, h) coordinates), tiles
//                         strictly above the diagonal skipped;
//   2. P = softmax(S/sqrt(D)) causal, fp32 math, P stored 16-bit; the last
//                         row's weights (fp32) and the sparsity counts kept;
//   3. O = P V            batched tcgen05 GEMM against V^T (one transpose),
//                         K-range clipped to the causal bound, O written as
//                         [B][s][H][D].
//   4. importance[b][j] = sum_h w_last[b][h][j] in fixed head order (fp64).
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "skv_internal.h"

namespace skvd {

constexpr int kPBM = 128, kPBK = 64, kPStages = 4, kPThreads = 192;

struct BGemm {
    int M, N, K;                 // per batch item z: C is M x N, reduction K
    int Hz;                      // z = zb * Hz + zh
    int a_row_b, a_row_h, a_col_h, a_col0;  // A tile y = zb*a_row_b + zh*a_row_h + m0; x = zh*a_col_h + a_col0 + k
    int b_row_b, b_row_h, b_col_h, b_col0;  // Bt tile likewise with n0
    long long c_b, c_h, ldc;     // C element offset = zb*c_b + zh*c_h + row*ldc + col
    int causal_skip;             // QK: skip tiles whose first key is past the tile's last query
    int causal_k;                // PV: reduce only over keys < m0 + BM
    int split;                   // > 0: A = [hi | lo] halves `split` columns apart, both against the same B
    void* C;
};

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | (1ull << 16) | ((1024ull >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

template <bool BF16, int BN, bool OUT16>
__global__ void __launch_bounds__(kPThreads, 1)
    bgemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, const BGemm g) {
    constexpr int ABYTES = kPBM * kPBK * 2, BBYTES = BN * kPBK * 2, STAGE = ABYTES + BBYTES;
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kPStages * STAGE);
    uint64_t* empty = full + kPStages;
    uint64_t* done = empty + kPStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * BN, m0 = blockIdx.y * kPBM, z = blockIdx.z;
    const int zb = z / g.Hz, zh = z % g.Hz;
    if (m0 >= g.M || n0 >= g.N) return;
    if (g.causal_skip && n0 > m0 + kPBM - 1) return;
    int kend = g.K;
    if (g.causal_k) kend = min(g.K, (m0 + kPBM + kPBK - 1) / kPBK * kPBK);
    const int kb1 = kend / kPBK, kblocks = g.split ? 2 * kb1 : kb1;
    const int ay = zb * g.a_row_b + zh * g.a_row_h + m0, ax = zh * g.a_col_h + g.a_col0;
    const int by = zb * g.b_row_b + zh * g.b_row_h + n0, bx = zh * g.b_col_h + g.b_col0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "n"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0)
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % kPStages;
                if (kb >= kPStages) mbar_wait(&empty[s], ((kb / kPStages) - 1) & 1);
                uint8_t* st = sm + s * STAGE;
                mbar_arrive_expect_tx(&full[s], STAGE);
                const int hi = kb < kb1 ? kb : kb - kb1;
                tma2d(st, &map_a, ax + (kb < kb1 ? 0 : g.split) + hi * kPBK, ay, &full[s]);
                tma2d(st + ABYTES, &map_b, bx + hi * kPBK, by, &full[s]);
            }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | ((BF16 ? 1u : 0u) << 7) | ((BF16 ? 1u : 0u) << 10) |
                                   (uint32_t(BN >> 3) << 17) | (uint32_t(kPBM >> 4) << 24);
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % kPStages;
                mbar_wait(&full[s], (kb / kPStages) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint8_t* st = sm + s * STAGE;
                const uint64_t da = sw128_desc(st), db = sw128_desc(st + ABYTES);
#pragma unroll
                for (int k = 0; k < kPBK / 16; ++k) {
                    const uint32_t acc = (kb | k) != 0;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                        "l"(da + uint64_t(2 * k)), "l"(db + uint64_t(2 * k)), "r"(idesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&empty[s]))
                             : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(done))
                         : "memory");
        }
    } else {
        const int quarter = warp & 3;
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int row = m0 + quarter * 32 + lane;
        const long long cbase = static_cast<long long>(zb) * g.c_b + static_cast<long long>(zh) * g.c_h +
                                static_cast<long long>(row) * g.ldc + n0;
        for (int c = 0; c < BN / 32; ++c) {
            uint32_t v[32];
            const uint32_t ta = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(c * 32);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (row >= g.M) continue;
            const int col0 = n0 + c * 32;
            if constexpr (!OUT16) {
                float* C = static_cast<float*>(g.C) + cbase + c * 32;
                if (col0 + 32 <= g.N) {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        reinterpret_cast<float4*>(C)[i] =
                            make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                        __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (col0 + i < g.N) C[i] = __uint_as_float(v[i]);
                }
            } else {
                uint16_t* C = static_cast<uint16_t*>(g.C) + cbase + c * 32;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float a = __uint_as_float(v[2 * i]), b = __uint_as_float(v[2 * i + 1]);
                    uint32_t pk;
                    if constexpr (BF16) {
                        const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
                        memcpy(&pk, &h, 4);
                    } else {
                        const __half2 h = __floats2half2_rn(a, b);
                        memcpy(&pk, &h, 4);
                    }
                    if (col0 + 2 * i + 1 < g.N) {
                        reinterpret_cast<uint32_t*>(C)[i] = pk;
                    } else if (col0 + 2 * i < g.N) {
                        C[2 * i] = static_cast<uint16_t>(pk & 0xFFFF);
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
    }
}

// 2. causal softmax rows of S (fp32 [Z][s][ld]) -> P 16-bit (zeros past the
// diagonal up to ld), the last row's weights (fp32) and per-z counts of cells
// below 0.01 x row max (attention_sparsity, attention.hpp:275-310). One warp
// per row; same arithmetic as softmax_rows (matrix.hpp:137-158) in fp32.
// bf16 keeps 8 mantissa bits, too few for the 1e-3 output bound: its P rows
// are [hi | lo] (2 x ld, lo = bf16(w - hi)) and the PV GEMM reduces over both
// halves, so the weights carry ~16 bits. fp16 P (11 bits) is stored once.
template <bool BF16>
__global__ void __launch_bounds__(256)
    prefill_softmax_kernel(const float* __restrict__ S, uint16_t* __restrict__ P, float* __restrict__ wlast,
                           unsigned* __restrict__ below, int s, int ld, float scale) {
    constexpr int kHalves = BF16 ? 2 : 1;
    const int z = blockIdx.y;
    const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= s) return;
    const float* row = S + (static_cast<size_t>(z) * s + i) * ld;
    uint16_t* prow = P + (static_cast<size_t>(z) * s + i) * ld * kHalves;
    float mx = -INFINITY;
    for (int j = lane; j <= i; j += 32) mx = fmaxf(mx, row[j] * scale);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int j = lane; j <= i; j += 32) sum += expf(row[j] * scale - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float inv = 1.0f / sum;
    const float thr = 0.01f * inv;  // the row max of the weights is exp(0)/sum
    unsigned cnt = 0;
    for (int j = lane; j < ld; j += 32) {
        float w = 0.f;
        if (j <= i) {
            w = expf(row[j] * scale - mx) * inv;
            cnt += w < thr;
            if (i == s - 1) wlast[static_cast<size_t>(z) * s + j] = w;
        }
        if constexpr (BF16) {
            const __nv_bfloat16 hi = __float2bfloat16_rn(w);
            prow[j] = __bfloat16_as_ushort(hi);
            prow[ld + j] = __bfloat16_as_ushort(__float2bfloat16_rn(w - __bfloat162float(hi)));
        } else {
            prow[j] = __half_as_ushort(__float2half_rn(w));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt) atomicAdd(&below[z], cnt);
}

// V^T per z: Vt[z][d][j] = V[b][j][h][d] (cache rows), zero for s <= j < ld.
__global__ void prefill_vt_kernel(const uint16_t* __restrict__ kv, uint16_t* __restrict__ vt, int H, int D, int Ncap,
                                  int s, int ld, long long row_elems) {
    __shared__ uint16_t tile[32][33];
    const int z = blockIdx.z, b = z / H, h = z % H;
    const int j0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int j = j0 + r;
        // token row: [K plane: H*D][V plane: H*D]
        tile[r][threadIdx.x] = j < s ? kv[(static_cast<size_t>(b) * Ncap + j) * row_elems + static_cast<size_t>(H) * D +
                                          static_cast<size_t>(h) * D + d0 + threadIdx.x]
                                     : uint16_t(0);
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y)
        vt[(static_cast<size_t>(z) * D + d0 + r) * ld + j0 + threadIdx.x] = tile[threadIdx.x][r];
}

// 4. importance[b][j] = sum_h w_last (head order, fp64): engine.hpp:508-512
// seeds each head's accumulator, attention.hpp:77-85 sums them.
__global__ void prefill_seed_kernel(const float* __restrict__ wlast, const unsigned* __restrict__ below,
                                    double* __restrict__ imp, double* __restrict__ psp, int H, int s,
                                    long long imp_ld) {
    const int b = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (psp != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
        // engine.hpp:513-518: mean over heads of each head's causal sparsity
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

// rows x cols 16-bit matrix with a row stride (elements), box {64, box_rows}.
bool map2d(CUtensorMap* m, const void* base, bool bf16, uint64_t rows, uint64_t cols, uint64_t stride_elems,
           uint32_t box_rows) {
    EncodeFn fn = encoder();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {stride_elems * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kPBK), box_rows};
    const cuuint32_t es[2] = {1, 1};
    return fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base),
              dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool BF16, int BN, bool OUT16>
cudaError_t run_bgemm(const CUtensorMap& ma, const CUtensorMap& mb, const BGemm& g, int Z, cudaStream_t st) {
    constexpr int smem = kPStages * (kPBM * kPBK * 2 + BN * kPBK * 2) + 1024 + 256;
    const void* fn = reinterpret_cast<const void*>(&bgemm_kernel<BF16, BN, OUT16>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((g.N + BN - 1) / BN, (g.M + kPBM - 1) / kPBM, Z);
    void* args[] = {const_cast<CUtensorMap*>(&ma), const_cast<CUtensorMap*>(&mb), const_cast<BGemm*>(&g)};
    e = cudaLaunchKernel(fn, grid, dim3(kPThreads), args, smem, st);
    count_launch();
    return e;
}

}  // namespace

// One chunk of B sequences. kv: their base in a 16-bit cache layer
// [B][Ncap][2][H][D]; q/out: [B][s][H][D] (out fp32 when out_f32); scratch:
// S fp32 [Z][s][ld], P 16-bit [Z][s][ld], Vt 16-bit [Z][D][ld], wlast fp32
// [Z][s], below u32 [Z] (zeroed here), ld = s rounded up to 256; psp
// (nullable): [B] prefill sparsity.
static cudaError_t prefill_chunk(bool bf16, bool out_f32, const void* kv, const void* q, void* out, double* imp,
                           long long imp_ld, double* psp, int B, int H, int D, int Ncap, int s, float* S, void* P,
                           void* Vt, float* wlast, unsigned* below, cudaStream_t st) {
    const int Z = B * H, ld = (s + 255) / 256 * 256;
    const long long row_elems = 2LL * H * D;
    cudaError_t e = cudaMemsetAsync(below, 0, static_cast<size_t>(Z) * 4, st);
    if (e != cudaSuccess) return e;
    // 1. S = Q K^T
    CUtensorMap mq, mk;
    if (!map2d(&mq, q, bf16, static_cast<uint64_t>(B) * s, static_cast<uint64_t>(H) * D, static_cast<uint64_t>(H) * D,
               kPBM) ||
        !map2d(&mk, kv, bf16, static_cast<uint64_t>(B) * Ncap, static_cast<uint64_t>(row_elems),
               static_cast<uint64_t>(row_elems), 256))
        return cudaErrorInvalidValue;
    BGemm g1{};
    g1.M = s;
    g1.N = s;
    g1.K = D;
    g1.Hz = H;
    g1.a_row_b = s;
    g1.a_col_h = D;
    g1.b_row_b = Ncap;
    g1.b_col_h = D;
    g1.c_b = static_cast<long long>(H) * s * ld;
    g1.c_h = static_cast<long long>(s) * ld;
    g1.ldc = ld;
    g1.causal_skip = 1;
    g1.C = S;
    e = bf16 ? run_bgemm<true, 256, false>(mq, mk, g1, Z, st) : run_bgemm<false, 256, false>(mq, mk, g1, Z, st);
    if (e != cudaSuccess) return e;
    // 2. softmax -> P (+ seed row, sparsity counts)
    const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(D)));
    dim3 sg((s + 7) / 8, Z);
    if (bf16)
        prefill_softmax_kernel<true><<<sg, 256, 0, st>>>(S, static_cast<uint16_t*>(P), wlast, below, s, ld, scale);
    else
        prefill_softmax_kernel<false><<<sg, 256, 0, st>>>(S, static_cast<uint16_t*>(P), wlast, below, s, ld, scale);
    count_launch();
    // V^T
    prefill_vt_kernel<<<dim3(ld / 32, D / 32, Z), dim3(32, 8), 0, st>>>(
        static_cast<const uint16_t*>(kv), static_cast<uint16_t*>(Vt), H, D, Ncap, s, ld, row_elems);
    count_launch();
    // 3. O = P V
    CUtensorMap mp, mv;
    const int halves = bf16 ? 2 : 1;
    if (!map2d(&mp, P, bf16, static_cast<uint64_t>(Z) * s, static_cast<uint64_t>(ld) * halves,
               static_cast<uint64_t>(ld) * halves, kPBM) ||
        !map2d(&mv, Vt, bf16, static_cast<uint64_t>(Z) * D, static_cast<uint64_t>(ld), static_cast<uint64_t>(ld), 128))
        return cudaErrorInvalidValue;
    BGemm g2{};
    g2.M = s;
    g2.N = D;
    g2.K = ld;
    g2.Hz = H;
    g2.a_row_b = H * s;
    g2.a_row_h = s;
    g2.b_row_b = H * D;
    g2.b_row_h = D;
    g2.c_b = static_cast<long long>(s) * H * D;
    g2.c_h = D;
    g2.ldc = static_cast<long long>(H) * D;
    g2.causal_k = 1;
    g2.split = bf16 ? ld : 0;
    g2.C = out;
    if (out_f32)
        e = bf16 ? run_bgemm<true, 128, false>(mp, mv, g2, Z, st) : run_bgemm<false, 128, false>(mp, mv, g2, Z, st);
    else
        e = bf16 ? run_bgemm<true, 128, true>(mp, mv, g2, Z, st) : run_bgemm<false, 128, true>(mp, mv, g2, Z, st);
    if (e != cudaSuccess) return e;
    // 4. seed
    prefill_seed_kernel<<<dim3((s + 255) / 256, B), 256, 0, st>>>(wlast, below, imp, psp, H, s, imp_ld);
    count_launch();
    return cudaGetLastError();
}


static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

size_t prefill_scratch_bytes(bool bf16, int nseq, int H, int D, int s) {
    const size_t Z = static_cast<size_t>(nseq) * H, ld = (static_cast<size_t>(s) + 255) / 256 * 256;
    const size_t halves = bf16 ? 2 : 1;
    return align256(Z * s * ld * 4) + align256(Z * s * ld * 2 * halves) + align256(Z * D * ld * 2) +
           align256(Z * s * 4) + align256(Z * 4);
}

// Causal prefill of one cache layer (see the file comment), in chunks of
// whole sequences sized to the scratch buffer.
cudaError_t launch_prefill(bool bf16, bool out_f32, const void* kv, const void* q, void* out, double* imp,
                           long long imp_ld, double* psp, int B, int H, int D, int Ncap, int s, uint8_t* scratch,
                           size_t scratch_bytes, cudaStream_t st) {
    const size_t per_seq = prefill_scratch_bytes(bf16, 1, H, D, s);
    const int chunk = static_cast<int>(std::min<size_t>(B, scratch_bytes / per_seq));
    if (chunk < 1) return cudaErrorInvalidValue;
    const size_t Z = static_cast<size_t>(chunk) * H, ld = (static_cast<size_t>(s) + 255) / 256 * 256;
    float* S = reinterpret_cast<float*>(scratch);
    uint8_t* P = scratch + align256(Z * s * ld * 4);
    uint8_t* Vt = P + align256(Z * s * ld * 2 * (bf16 ? 2 : 1));
    float* wlast = reinterpret_cast<float*>(Vt + align256(Z * D * ld * 2));
    unsigned* below = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(wlast) + align256(Z * s * 4));
    const size_t row_bytes = 2ull * H * D * 2, qrow = static_cast<size_t>(H) * D;
    const size_t obytes = out_f32 ? 4 : 2;
    for (int b0 = 0; b0 < B; b0 += chunk) {
        const int nb = std::min(chunk, B - b0);
        cudaError_t e = prefill_chunk(
            bf16, out_f32, static_cast<const uint8_t*>(kv) + static_cast<size_t>(b0) * Ncap * row_bytes,
            static_cast<const uint8_t*>(q) + static_cast<size_t>(b0) * s * qrow * 2,
            static_cast<uint8_t*>(out) + static_cast<size_t>(b0) * s * qrow * obytes, imp + b0 * imp_ld, imp_ld,
            psp ? psp + b0 : nullptr, nb, H, D, Ncap, s, S, P, Vt, wlast, below, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace skv_impl
