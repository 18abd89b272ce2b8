// skv_gemm.cu -- tcgen05 (5th-gen tensor core) GEMM for KV recomputation.
//
// recompute_kv (engine.hpp:718-737) re-derives a deleted token's K and V from
// its retained post-LN1 row: k = x Wk, v = x Wv. For all tokens a layer must
// recompute in one step that is one dense GEMM
//     C[M x 2h] = A[M x h] . Bt[2h x h]^T,   Bt = [Wk | Wv]^T (K-major)
// with M = the gathered rows. Blackwell-native: TMA (SWIZZLE_128B) tiles into
// a 4-stage shared-memory ring, one elected thread issues
// tcgen05.mma.cta_group::1.kind::f16 (128 x 256 x 16) into a TMEM fp32
// accumulator, four epilogue warps drain TMEM with tcgen05.ld. One CTA per
// 128 x 256 output tile.
#include <cuda.h>

#include <mutex>

#include "skv_internal.h"

namespace skvd {

constexpr int kGemmBM = 128, kGemmBN = 256, kGemmBK = 64, kGemmStages = 4;
constexpr int kGemmThreads = 192;  // warp 0 TMA, warp 1 MMA (+TMEM alloc), warps 2..5 epilogue
constexpr int kGemmABytes = kGemmBM * kGemmBK * 2;  // 16 KB
constexpr int kGemmBBytes = kGemmBN * kGemmBK * 2;  // 32 KB
constexpr int kGemmStageBytes = kGemmABytes + kGemmBBytes;
constexpr int kGemmSmem = kGemmStages * kGemmStageBytes + 1024 /* align */ + 256 /* barriers */;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor, K-major operand in the canonical
// SWIZZLE_128B layout (8-row groups of 1024 bytes).
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem_ptr) {
    const uint64_t addr = smem_u32(smem_ptr);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;          // start address  [0,14)
    d |= (uint64_t(1) & 0x3FFFull) << 16;  // leading byte offset (unused for swizzled K-major) [16,30)
    d |= (uint64_t(1024 >> 4) & 0x3FFFull) << 32;  // stride byte offset: 8 rows x 128 B [32,46)
    d |= uint64_t(1) << 46;                // descriptor version (sm_100)
    d |= uint64_t(2) << 61;                // layout: SWIZZLE_128B
    return d;
}

// Instruction descriptor for kind::f16: fp32 accumulate, K-major A and B.
__host__ __device__ constexpr uint32_t umma_idesc(bool bf16, int M, int N) {
    return (1u << 4)                          // c_format F32
           | ((bf16 ? 1u : 0u) << 7)          // a_format
           | ((bf16 ? 1u : 0u) << 10)         // b_format
           | (uint32_t(N >> 3) << 17)         // n_dim
           | (uint32_t(M >> 4) << 24);        // m_dim
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_c, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_c),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

template <bool BF16, bool SCATTER>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   float* __restrict__ C, const int* __restrict__ m_dev, int M_cap, int N, int K,
                   const KvScatter sc) {
    extern __shared__ __align__(1024) uint8_t gsm_raw[];
    uint8_t* gsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(gsm + kGemmStages * kGemmStageBytes);
    uint64_t* empty = full + kGemmStages;
    uint64_t* tmem_full = empty + kGemmStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * kGemmBN, m0 = blockIdx.y * kGemmBM;
    const int M = m_dev ? *m_dev : M_cap;
    if (m0 >= M) return;  // rows beyond this launch's real count
    const int kblocks = K / kGemmBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kGemmStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) {  // TMEM: 256 fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % kGemmStages;
                if (kb >= kGemmStages) mbar_wait(&empty[s], ((kb / kGemmStages) - 1) & 1);
                uint8_t* sa = gsm + s * kGemmStageBytes;
                mbar_arrive_expect_tx(&full[s], kGemmStageBytes);
                tma_load_2d(sa, &map_a, kb * kGemmBK, m0, &full[s]);
                tma_load_2d(sa + kGemmABytes, &map_b, kb * kGemmBK, n0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer (one thread)
            constexpr uint32_t idesc = umma_idesc(BF16, kGemmBM, kGemmBN);
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % kGemmStages;
                mbar_wait(&full[s], (kb / kGemmStages) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint8_t* sa = gsm + s * kGemmStageBytes;
                const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + kGemmABytes);
#pragma unroll
                for (int k = 0; k < kGemmBK / 16; ++k)  // UMMA_K = 16 elements = 32 bytes
                    umma_f16(tmem, da + uint64_t(k * 2), db + uint64_t(k * 2), idesc, (kb | k) != 0);
                umma_commit(&empty[s]);  // frees the smem stage once these MMAs finish
            }
            umma_commit(tmem_full);  // accumulator complete
        }
    } else {
        // ===== epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 (rows of the tile)
        const int quarter = warp & 3;
        mbar_wait(tmem_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int row = m0 + quarter * 32 + lane;
        for (int c = 0; c < kGemmBN / 32; ++c) {
            uint32_t v[32];
            const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(c * 32);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (row < M) {
                if constexpr (!SCATTER) {
                    float4* dst = reinterpret_cast<float4*>(C + static_cast<size_t>(row) * N + n0 + c * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                             __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                } else {
                    const int2 bt = sc.rowmap[row];
                    if (bt.y < 0) continue;  // no slot (paged OOM, reported by the ledger)
                    const int hidden = sc.H * sc.D;
                    const int j = n0 + c * 32;
                    const int kvsel = j / hidden, hh = (j % hidden) / sc.D, d = j % sc.D;
                    uint8_t* dst = sc.kv + ((static_cast<size_t>(bt.x) * sc.Ncap + bt.y) * 2 + kvsel) *
                                               static_cast<size_t>(sc.H) * sc.row_bytes +
                                   static_cast<size_t>(hh) * sc.row_bytes + static_cast<size_t>(d) * 2;
                    uint32_t packed[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float a = __uint_as_float(v[2 * i]), b = __uint_as_float(v[2 * i + 1]);
                        if constexpr (BF16) {
                            const __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
                            memcpy(&packed[i], &h2, 4);
                        } else {
                            const __half2 h2 = __floats2half2_rn(a, b);
                            memcpy(&packed[i], &h2, 4);
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        reinterpret_cast<uint4*>(dst)[i] =
                            make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

// recompute_kv gather: the post-LN1 rows of this step's recompute tokens of
// every sequence (lists from the ledger) into a dense A [M x h], with the row
// map (b, t). One CTA per sequence; offsets by a prefix over sequences.
__global__ void __launch_bounds__(256)
    recompute_gather_kernel(const uint8_t* __restrict__ x, long long x_seq, long long x_row, const int* lists,
                            const int* counts, long long list_ld, uint8_t* __restrict__ A, int2* rowmap, int* m_out,
                            int B, const int* dst_slots) {
    const int b = blockIdx.x;
    int off = 0;
    for (int i = 0; i < b; ++i) off += counts[i * 4 + 3];
    const int cnt = counts[b * 4 + 3];
    const int* list = lists + (static_cast<size_t>(b) * 4 + 3) * list_ld;
    const int* dslot = dst_slots ? dst_slots + (static_cast<size_t>(b) * 4 + 3) * list_ld : nullptr;
    const int vecs = static_cast<int>(x_row / 16);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (int i = warp; i < cnt; i += nwarps) {  // one warp per row: no 64-bit index division
        const int t = list[i];
        const uint4* src = reinterpret_cast<const uint4*>(x + b * x_seq + static_cast<long long>(t) * x_row);
        uint4* dst = reinterpret_cast<uint4*>(A + static_cast<size_t>(off + i) * x_row);
        for (int v = lane; v < vecs; v += 32) dst[v] = src[v];
        if (lane == 0)  // paged: the destination is the slot the ledger allocated
            rowmap[off + i] = make_int2(b, dslot ? dslot[i] : t);
    }
    if (b == B - 1 && threadIdx.x == 0) *m_out = off + cnt;
}

}  // namespace skvd

namespace skv_impl {

cudaError_t launch_recompute_gather(const uint8_t* x, long long x_seq, long long x_row, const int* lists,
                                    const int* counts, long long list_ld, uint8_t* A, int2* rowmap, int* m_out,
                                    int B, cudaStream_t st, const int* dst_slots) {
    skvd::recompute_gather_kernel<<<B, 256, 0, st>>>(x, x_seq, x_row, lists, counts, list_ld, A, rowmap, m_out, B,
                                                     dst_slots);
    count_launch();
    return cudaGetLastError();
}
using namespace skvd;

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
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

// Row-major [rows x cols] 16-bit matrix, box {64 cols, box_rows}, 128B swizzle.
bool make_map(CUtensorMap* m, const void* base, bool bf16, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kGemmBK), box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
              const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// C[M_cap x N] (fp32, row-major) = A[M_cap x K] . Bt[N x K]^T for 16-bit A, Bt.
// Rows >= *m_dev (when given) are skipped. N % 256 == 0, K % 64 == 0,
// M_cap % 128 == 0.
cudaError_t launch_gemm_tn(const void* A, const void* Bt, float* C, const int* m_dev, int M_cap, int N, int K,
                           bool bf16, cudaStream_t st, const KvScatter* sc) {
    if (N % kGemmBN || K % kGemmBK || M_cap % kGemmBM || M_cap <= 0) return cudaErrorInvalidValue;
    CUtensorMap ma, mb;
    if (!make_map(&ma, A, bf16, static_cast<uint64_t>(M_cap), static_cast<uint64_t>(K), kGemmBM) ||
        !make_map(&mb, Bt, bf16, static_cast<uint64_t>(N), static_cast<uint64_t>(K), kGemmBN))
        return cudaErrorInvalidValue;
    const void* fns[4] = {reinterpret_cast<const void*>(&gemm_tn_kernel<false, false>),
                          reinterpret_cast<const void*>(&gemm_tn_kernel<true, false>),
                          reinterpret_cast<const void*>(&gemm_tn_kernel<false, true>),
                          reinterpret_cast<const void*>(&gemm_tn_kernel<true, true>)};
    const void* fn = fns[(bf16 ? 1 : 0) + (sc ? 2 : 0)];
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmem);
    if (e != cudaSuccess) return e;
    KvScatter none{};
    const KvScatter& s = sc ? *sc : none;
    dim3 grid(N / kGemmBN, M_cap / kGemmBM);
    void* args[] = {&ma, &mb, &C, const_cast<int**>(&m_dev), &M_cap, &N, &K, const_cast<KvScatter*>(&s)};
    e = cudaLaunchKernel(fn, grid, dim3(kGemmThreads), args, kGemmSmem, st);
    count_launch();
    return e;
}

}  // namespace skv_impl
