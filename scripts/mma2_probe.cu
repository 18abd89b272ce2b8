// mma2_probe.cu -- cost per instruction of a 2-CTA (cta_group::2, M = 256)
// tcgen05.mma against the 1-CTA M = 128 one (mma_probe.cu): does a CTA pair
// get twice the work per instruction? Timing only (operands are garbage).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build_var/mma2_probe scripts/mma2_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(const void* p, uint32_t lbo, uint32_t sbo) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | (uint64_t(lbo >> 4) << 16) | (uint64_t(sbo >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n, bool b_mn) {
    return (1u << 4) | ((b_mn ? 1u : 0u) << 16) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) probe2(long long* out, int n, int iters, int ts) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t rank = cta_rank();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (rank == 0 && threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        long long t0 = 0;
        for (int rep = 0; rep < 2; ++rep) {
            t0 = clock64();
            for (int i = 0; i < iters; ++i) {
                const int kk = i & 7;
                const uint32_t d = tmem + 256;
                const uint32_t acc = 1;
                if (ts) {  // A from TMEM (P.V-like), B MN-major
                    const uint32_t a = tmem + kk * 8;
                    const uint64_t b = desc(sm + 65536 + kk * 2048, 16384, 1024);
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                        "r"(a), "l"(b), "r"(idesc(256, n, true)), "r"(acc));
                } else {
                    const uint64_t a = desc(sm + kk * 32, 16, 1024), b = desc(sm + 65536 + kk * 32, 16, 1024);
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(a), "l"(b), "r"(idesc(256, n, false)), "r"(acc));
                }
            }
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&bar)),
                "h"(static_cast<unsigned short>(1))
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
    cluster_sync();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int ts = 0; ts < 2; ++ts)
        for (int n : {64, 128, 256}) {
            const int iters = 512;
            probe2<<<2, 128, 200 * 1024>>>(d, n, iters, ts);
            long long t = 0;
            cudaError_t e = cudaMemcpy(&t, d, 8, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                printf("%s N=%3d error %s\n", ts ? "TS" : "SS", n, cudaGetErrorString(e));
                return 1;
            }
            printf("2-CTA %s M256 N=%3d: %.1f cycles per MMA (%.0f MAC/clk per SM)\n", ts ? "TS A-T B-MN" : "SS A-K B-K ",
                   n, double(t) / iters, 256.0 * n * 16 / (double(t) / iters) / 2);
        }
    return 0;
}
