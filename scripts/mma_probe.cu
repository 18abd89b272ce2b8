// mma_probe.cu -- issue-to-completion cost of tcgen05.mma variants on one SM
// (sm_100a). Operands are whatever is in shared memory / TMEM (timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build_var/mma_probe scripts/mma_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t desc(const void* p, uint32_t lbo, uint32_t sbo) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | (uint64_t(lbo >> 4) << 16) | (uint64_t(sbo >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

__host__ __device__ constexpr uint32_t idesc(int n, bool b_mn) {
    return (1u << 4) | ((b_mn ? 1u : 0u) << 16) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

__global__ void probe(long long* out, int variant, int n, int iters) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        long long t0 = 0;
        for (int rep = 0; rep < 2; ++rep) {
            t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const int kk = i & 7;
                switch (variant) {
                    case 0:  // SS, A K-major, B K-major
                        mma_ss(tmem + 256, desc(sm + kk * 32, 16, 1024), desc(sm + 65536 + kk * 32, 16, 1024),
                               idesc(n, false), 1);
                        break;
                    case 1:  // SS, A K-major, B MN-major
                        mma_ss(tmem + 256, desc(sm + kk * 32, 16, 1024), desc(sm + 65536 + kk * 2048, 16384, 1024),
                               idesc(n, true), 1);
                        break;
                    case 2:  // TS (A from TMEM), B MN-major
                        mma_ts(tmem + 256, tmem + kk * 8, desc(sm + 65536 + kk * 2048, 16384, 1024), idesc(n, true), 1);
                        break;
                    case 3:  // TS (A from TMEM), B K-major
                        mma_ts(tmem + 256, tmem + kk * 8, desc(sm + 65536 + kk * 32, 16, 1024), idesc(n, false), 1);
                        break;
                    case 4:  // SS A-K B-K, two independent accumulators alternating
                        mma_ss(tmem + 256 + (i & 1) * 128, desc(sm + kk * 32, 16, 1024),
                               desc(sm + 65536 + kk * 32, 16, 1024), idesc(n, false), 1);
                        break;
                    case 5:  // alternating an S-like SS MMA and a P.V-like TS MMA into separate accumulators
                        if (i & 1)
                            mma_ts(tmem + 384, tmem + kk * 8, desc(sm + 65536 + kk * 2048, 16384, 1024), idesc(128, true), 1);
                        else
                            mma_ss(tmem + 256, desc(sm + kk * 32, 16, 1024), desc(sm + 65536 + kk * 32, 16, 1024),
                                   idesc(n > 128 ? 128 : n, false), 1);
                        break;
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&bar))
                         : "memory");
            uint32_t ok = 0;
            while (!ok)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, "
                    "p;\n\t}"
                    : "=r"(ok)
                    : "r"(smem_u32(&bar)), "r"(rep & 1));
        }
        out[0] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[6] = {"SS  A-K B-K ", "SS  A-K B-MN", "TS  A-T B-MN", "TS  A-T B-K ", "SS x2 accum ",
                            "SS|TS alt   "};
    for (int v = 0; v < 6; ++v)
        for (int n : {64, 128, 256}) {
            if (v >= 4 && n > 128) continue;  // two 128-column accumulators at 256 and 384
            const int iters = 512;
            probe<<<1, 128, 200 * 1024>>>(d, v, n, iters);
            long long t = 0;
            cudaError_t e = cudaMemcpy(&t, d, 8, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                printf("%s N=%3d error %s\n", names[v], n, cudaGetErrorString(e));
                return 1;
            }
            printf("%s N=%3d: %.1f cycles per M128xN%dxK16 MMA (%.0f MAC/clk)\n", names[v], n, double(t) / iters, n,
                   128.0 * n * 16 / (double(t) / iters));
        }
    return 0;
}
