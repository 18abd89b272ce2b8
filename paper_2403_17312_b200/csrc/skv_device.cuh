// skv_device.cuh -- sm_100a device primitives shared by the SWA kernels:
// mbarrier + cp.async.bulk (TMA bulk engine, SASS UBLKCP) staging, named
// barriers, 16-byte vector conversions, fp64 order keys and round-half-even.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#ifdef SKV_DECODE_TRACE
#include <cstdio>
#endif

namespace skvd {

// Debug build only (-DSKV_DECODE_TRACE): globaltimer stamps of CTA (0, 0)'s
// phases and the tail's, printed every 50th n (latency anatomy of config 1).
#ifdef SKV_DECODE_TRACE
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DTR(slot) do { if (ctid == 0 && (blockIdx.x == 0 && blockIdx.y == 0)) dtr[slot] = gtimer(); } while (0)
#define DTR_TAIL(slot) do { if (ctid == 0) dtr[slot] = gtimer(); } while (0)
#define DTR_T(slot, id) do { if ((id) == 0) dtr[slot] = gtimer(); } while (0)
__device__ unsigned long long dtr[16];
#else
#define DTR(slot) do { } while (0)
#define DTR_TAIL(slot) do { } while (0)
#define DTR_T(slot, id) do { } while (0)
#endif

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

// INT8 storage of one token: for K then V, the heads in blocks of 8, each
// block [8 x 128 codes][8 x (scale, bias) fp32] = 1088 bytes, so every code
// row is 16-byte aligned (one 128-bit shared-memory load per vector, no bank
// conflicts) and a head group of 8 is still one contiguous bulk copy.
constexpr int kU8Group = 8;
constexpr int kU8Block = kU8Group * (128 + 8);
__host__ __device__ inline size_t u8_code_off(int which, int h, int H) {
    return static_cast<size_t>(which * (H / kU8Group) + h / kU8Group) * kU8Block +
           static_cast<size_t>(h % kU8Group) * 128;
}
__host__ __device__ inline size_t u8_meta_off(int which, int h, int H) {
    return static_cast<size_t>(which * (H / kU8Group) + h / kU8Group) * kU8Block + kU8Group * 128 +
           static_cast<size_t>(h % kU8Group) * 8;
}

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
// INT8 codes come out BIASED: 1024 + c. One PRMT packs two codes under the
// f16 exponent of 1024 (0x64bb == 1024 + bb exactly), one HADD2.F32 widens the
// pair: 1.5 instructions per code with the FFMA2, against 2 for a per-code
// PRMT into 2^23 + c and an FADD2 to remove it. The attend kernel folds the
// bias into the per-token affine term: bias' = bias - 1024 * scale (kBiasU8).
constexpr float kBiasU8 = 1024.0f;
__device__ __forceinline__ void cvt16x2(const uint4& r, float2 (&f)[8], KvU8) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t lo = __byte_perm(w[i], 0x64646464u, 0x4140u);  // {1024 + b0, 1024 + b1}
        const uint32_t hi = __byte_perm(w[i], 0x64646464u, 0x4342u);  // {1024 + b2, 1024 + b3}
        __half2 a, b;
        memcpy(&a, &lo, 4);
        memcpy(&b, &hi, 4);
        f[2 * i] = __half22float2(a);
        f[2 * i + 1] = __half22float2(b);
    }
}

// Mixed-precision FMA (SASS FHFMA): f16 x f16 products are exact in f32, so
// this is as precise as FFMA on these inputs. *hi selects the upper half.
__device__ __forceinline__ float fhfma(uint32_t a, bool ahi, uint32_t b, bool bhi, float c) {
    float d;
    const uint16_t x = static_cast<uint16_t>(ahi ? (a >> 16) : a);
    const uint16_t y = static_cast<uint16_t>(bhi ? (b >> 16) : b);
    asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(x), "h"(y), "f"(c));
    return d;
}

// q . (1024 + c) over 16 INT8 codes against 16 fp16 query values (8 packed
// words): one PRMT per code pair and one FHFMA per code -- 1.5 instructions
// per code against 2 for the f32 route. Two chains for ILP.
__device__ __forceinline__ float dot_u8_f16(const uint4& r, const uint32_t (&qh)[8]) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t lo = __byte_perm(w[j], 0x64646464u, 0x4140u);  // {1024 + b0, 1024 + b1}
        const uint32_t hi = __byte_perm(w[j], 0x64646464u, 0x4342u);  // {1024 + b2, 1024 + b3}
        a0 = fhfma(lo, false, qh[2 * j], false, a0);
        a1 = fhfma(lo, true, qh[2 * j], true, a1);
        a0 = fhfma(hi, false, qh[2 * j + 1], false, a0);
        a1 = fhfma(hi, true, qh[2 * j + 1], true, a1);
    }
    return a0 + a1;
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
