// skv_decode.cu -- instantiations of the fused SWA decode kernel and their
// dispatch table (kv dtype x compute dtype x heads-per-CTA).
#include "skv_internal.h"

namespace skv_impl {
using namespace skvd;

namespace {

template <class KV, class QT, int HG>
size_t smem_of(int m, bool gmem, bool paged) {
    return decode_smem<KV, HG>(m, gmem, paged).total;
}

template <class KV, class QT, int HG>
DecodeLaunch make() {
    return DecodeLaunch{reinterpret_cast<const void*>(&swa_attend_kernel<KV, QT, HG>),
                        &smem_of<KV, QT, HG>, HG,
                        static_cast<size_t>(DecodeCfg<KV, HG>::S) * DecodeCfg<KV, HG>::STAGEB};
}

struct Entry {
    int kv, q, hg;
    DecodeLaunch dl;
};

const Entry* table(int* count) {
    static const Entry t[] = {
        {SKV_F32, SKV_F32, 1, make<KvF32, float, 1>()},
        {SKV_F32, SKV_F32, 2, make<KvF32, float, 2>()},
        {SKV_F32, SKV_F32, 4, make<KvF32, float, 4>()},
        {SKV_F32, SKV_F32, 8, make<KvF32, float, 8>()},
        {SKV_F16, SKV_F16, 1, make<KvF16, __half, 1>()},
        {SKV_F16, SKV_F16, 2, make<KvF16, __half, 2>()},
        {SKV_F16, SKV_F16, 4, make<KvF16, __half, 4>()},
        {SKV_F16, SKV_F16, 8, make<KvF16, __half, 8>()},
        {SKV_BF16, SKV_BF16, 1, make<KvBF16, __nv_bfloat16, 1>()},
        {SKV_BF16, SKV_BF16, 2, make<KvBF16, __nv_bfloat16, 2>()},
        {SKV_BF16, SKV_BF16, 4, make<KvBF16, __nv_bfloat16, 4>()},
        {SKV_BF16, SKV_BF16, 8, make<KvBF16, __nv_bfloat16, 8>()},
        {SKV_U8, SKV_F32, 2, make<KvU8, float, 2>()},
        {SKV_U8, SKV_F32, 4, make<KvU8, float, 4>()},
        {SKV_U8, SKV_F32, 8, make<KvU8, float, 8>()},
        {SKV_U8, SKV_F16, 2, make<KvU8, __half, 2>()},
        {SKV_U8, SKV_F16, 4, make<KvU8, __half, 4>()},
        {SKV_U8, SKV_F16, 8, make<KvU8, __half, 8>()},
        {SKV_U8, SKV_BF16, 2, make<KvU8, __nv_bfloat16, 2>()},
        {SKV_U8, SKV_BF16, 4, make<KvU8, __nv_bfloat16, 4>()},
        {SKV_U8, SKV_BF16, 8, make<KvU8, __nv_bfloat16, 8>()},
    };
    *count = static_cast<int>(sizeof(t) / sizeof(t[0]));
    return t;
}

}  // namespace

const DecodeLaunch* find_decode(int kv_dtype, int q_dtype, int hg) {
    int cnt = 0;
    const Entry* t = table(&cnt);
    for (int i = 0; i < cnt; ++i)
        if (t[i].kv == kv_dtype && t[i].q == q_dtype && t[i].hg == hg) return &t[i].dl;
    return nullptr;
}

cudaError_t launch_attend(const DecodeLaunch& dl, const AttendParams& p, int grid_g, size_t smem, bool pdl,
                          cudaStream_t st) {
    // the dynamic-smem attribute was raised by pick_attend (skv_capi.cu)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid_g, p.B);
    cfg.blockDim = dim3(kDecodeThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    void* args[] = {const_cast<AttendParams*>(&p)};
    const cudaError_t e = cudaLaunchKernelExC(&cfg, dl.func, args);
    count_launch();
    return e;
}

}  // namespace skv_impl
