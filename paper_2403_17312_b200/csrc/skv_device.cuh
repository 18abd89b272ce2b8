// skv_device.cuh -- sm_100a device primitives shared by the SWA kernels:
// mbarrier + cp.async.bulk (TMA bulk engine, SASS UBLKCP) staging, named
// barriers, 16-byte vector conversions, fp64 order keys and round-half-even.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace skvd {

// ---------------------------------------------------------------- smem / sync
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

// Make barrier inits visible to the async (TMA) proxy before first use.
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// L2 policy for streamed-once KV rows.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Bulk async copy global -> this CTA's shared memory; completion is counted in
// bytes on `bar`. bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// Named barriers (id 0 is __syncthreads). `count` is a multiple of 32.
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ----------------------------------------------------------- number helpers
// Reference round_half_even (common.hpp:43-54), floor-based, fp64.
__device__ __forceinline__ long long rne_ref(double x) {
    const double f = floor(x);
    const double frac = x - f;
    const long long lo = static_cast<long long>(f);
    if (frac > 0.5) return lo + 1;
    if (frac < 0.5) return lo;
    return (lo % 2 == 0) ? lo : lo + 1;
}

// Monotone map fp64 -> u64 (larger double => larger key). -0.0 is folded onto
// +0.0 because the reference compares with `!=` / `>` (matrix.hpp:168-173).
__device__ __forceinline__ uint64_t order_key(double x) {
    if (x == 0.0) x = 0.0;
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// --------------------------------------------------------- element types
// Storage type tags for the KV cache.
struct KvF32 {
    using T = float;
    static constexpr int E = 4;
    static constexpr bool QUANT = false;
};
struct KvF16 {
    using T = __half;
    static constexpr int E = 2;
    static constexpr bool QUANT = false;
};
struct KvBF16 {
    using T = __nv_bfloat16;
    static constexpr int E = 2;
    static constexpr bool QUANT = false;
};
struct KvU8 {  // affine 8-bit codes + per (token, head) fp32 (scale, bias)
    using T = uint8_t;
    static constexpr int E = 1;
    static constexpr bool QUANT = true;
};

// 16 bytes -> 16/E floats.
__device__ __forceinline__ void cvt16(const uint4& r, float (&f)[4], KvF32) {
    f[0] = __uint_as_float(r.x);
    f[1] = __uint_as_float(r.y);
    f[2] = __uint_as_float(r.z);
    f[3] = __uint_as_float(r.w);
}
__device__ __forceinline__ void cvt16(const uint4& r, float (&f)[8], KvF16) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        __half2 h;
        memcpy(&h, &w[i], 4);
        const float2 v = __half22float2(h);
        f[2 * i] = v.x;
        f[2 * i + 1] = v.y;
    }
}
__device__ __forceinline__ void cvt16(const uint4& r, float (&f)[8], KvBF16) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        // bf16 -> f32 is a 16-bit shift.
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}
__device__ __forceinline__ void cvt16(const uint4& r, float (&f)[16], KvU8) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            // 0x4B0000bb is 2^23 + bb exactly; one PRMT + one FADD per code.
            const uint32_t bits = __byte_perm(w[i], 0x4B000000u, 0x7540u | j);
            f[4 * i + j] = __uint_as_float(bits) - 8388608.0f;
        }
    }
}

// 16 bytes -> float2 pairs (feed the packed FFMA2 pipe).
__device__ __forceinline__ void cvt16x2(const uint4& r, float2 (&f)[2], KvF32) {
    f[0] = make_float2(__uint_as_float(r.x), __uint_as_float(r.y));
    f[1] = make_float2(__uint_as_float(r.z), __uint_as_float(r.w));
}
__device__ __forceinline__ void cvt16x2(const uint4& r, float2 (&f)[4], KvF16) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        __half2 h;
        memcpy(&h, &w[i], 4);
        f[i] = __half22float2(h);
    }
}
__device__ __forceinline__ void cvt16x2(const uint4& r, float2 (&f)[4], KvBF16) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u));
}
__device__ __forceinline__ void cvt16x2(const uint4& r, float2 (&f)[8], KvU8) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    const float2 off = make_float2(-8388608.0f, -8388608.0f);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        // 0x4B0000bb == 2^23 + bb exactly: one PRMT per code, one FADD2 per pair.
        const float2 a = make_float2(__uint_as_float(__byte_perm(w[i], 0x4B000000u, 0x7540u)),
                                     __uint_as_float(__byte_perm(w[i], 0x4B000000u, 0x7541u)));
        const float2 b = make_float2(__uint_as_float(__byte_perm(w[i], 0x4B000000u, 0x7542u)),
                                     __uint_as_float(__byte_perm(w[i], 0x4B000000u, 0x7543u)));
        f[2 * i] = __fadd2_rn(a, off);
        f[2 * i + 1] = __fadd2_rn(b, off);
    }
}

// Programmatic dependent launch (PDL).
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Make this thread's generic-proxy global writes visible to later async-proxy
// (bulk copy) reads issued by other threads after a barrier.
__device__ __forceinline__ void fence_global_to_async() {
    __threadfence();
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Scalar loads of a compute-side (q / new k,v) element as float.
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) {
    return x;
}
template <>
__device__ __forceinline__ __half from_f<__half>(float x) {
    return __float2half_rn(x);
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}

}  // namespace skvd
