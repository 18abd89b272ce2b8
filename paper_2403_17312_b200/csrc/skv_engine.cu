// skv_engine.cu -- the dense (non-attention) operators of the reference's toy
// transformer step on the GPU (engine.hpp:250-303, 384-468, 571-684): token
// embedding + positional term, LayerNorm, the projections / FFN / logits
// GEMMs, GELU, and the dense causal attention of the prompt (prefill,
// attention.hpp:91-117) with its weight matrices for the importance seed and
// the prefill sparsity. fp64 like the reference; the SWA decode attention
// itself runs on the cache kernels (skv_decode.cuh). These are small,
// latency-bound operators at the toy shapes: plain CUDA, one thread per
// output element or one CTA per row.
#include <cmath>

#include "skv_internal.h"

namespace skvd {

// engine.hpp:360-381 (embed / embed_one) + positional_term (:131-144)
__global__ void eng_embed_kernel(const double* __restrict__ emb, int h, const long long* __restrict__ ids, int n,
                                 int pos0, double* __restrict__ out) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(n) * h) return;
    const int t = static_cast<int>(i / h), d = static_cast<int>(i % h);
    const int e = d & ~1;  // the even index of the (sin, cos) pair
    const double freq = pow(10000.0, -static_cast<double>(e) / static_cast<double>(h));
    const double ang = static_cast<double>(pos0 + t) * freq;
    const double pe = (d & 1) ? cos(ang) : sin(ang);
    out[i] = emb[static_cast<size_t>(ids[t]) * h + d] + pe;
}

// engine.hpp:111-129 layer_norm, one CTA per row, the reference's sum order
// replaced by a tree (fp64)
__global__ void eng_layernorm_kernel(const double* __restrict__ x, int h, const double* __restrict__ gain,
                                     const double* __restrict__ bias, double* __restrict__ out) {
    __shared__ double red[32];
    const double* row = x + static_cast<size_t>(blockIdx.x) * h;
    double* o = out + static_cast<size_t>(blockIdx.x) * h;
    auto block_sum = [&](double v) {
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        __syncthreads();
        return t;
    };
    double s = 0.0;
    for (int i = threadIdx.x; i < h; i += blockDim.x) s += row[i];
    const double mean = block_sum(s) / h;
    double v = 0.0;
    for (int i = threadIdx.x; i < h; i += blockDim.x) v += (row[i] - mean) * (row[i] - mean);
    const double inv = 1.0 / sqrt(block_sum(v) / h + 1e-5);
    for (int i = threadIdx.x; i < h; i += blockDim.x) o[i] = (row[i] - mean) * inv * gain[i] + bias[i];
}

// C[M x N] (+)= A[M x K] . B[K x N], fp64, 16 x 16 tiles through shared memory
__global__ void eng_gemm_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                                int M, int N, int K, int accumulate) {
    __shared__ double ta[16][17], tb[16][17];
    const int r = blockIdx.y * 16 + threadIdx.y, c = blockIdx.x * 16 + threadIdx.x;
    double acc = 0.0;
    for (int k0 = 0; k0 < K; k0 += 16) {
        ta[threadIdx.y][threadIdx.x] = (r < M && k0 + threadIdx.x < K) ? A[static_cast<size_t>(r) * K + k0 + threadIdx.x] : 0.0;
        tb[threadIdx.y][threadIdx.x] = (k0 + threadIdx.y < K && c < N) ? B[static_cast<size_t>(k0 + threadIdx.y) * N + c] : 0.0;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) acc = fma(ta[threadIdx.y][k], tb[k][threadIdx.x], acc);
        __syncthreads();
    }
    if (r < M && c < N) {
        double* o = C + static_cast<size_t>(r) * N + c;
        *o = accumulate ? *o + acc : acc;
    }
}

// engine.hpp:127-129 gelu (tanh form)
__global__ void eng_gelu_kernel(double* x, long long n) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = x[i];
    x[i] = 0.5 * v * (1.0 + tanh(0.7978845608028654 * (v + 0.044715 * v * v * v)));
}

__global__ void eng_convert_kernel(const double* __restrict__ in, float* __restrict__ out, long long n) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = static_cast<float>(in[i]);
}

__global__ void eng_widen_kernel(const float* __restrict__ in, double* __restrict__ out, long long n) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = static_cast<double>(in[i]);
}

// dense_attention (attention.hpp:91-117) with the causal mask bottom-right
// aligned, per head of row-major [s][H*D] q/k/v (the layer's head slices,
// engine.hpp:398-410): one CTA per (query row, head); aw [H][sq][sk].
__global__ void eng_causal_attention_kernel(const double* __restrict__ q, const double* __restrict__ k,
                                            const double* __restrict__ v, int sq, int sk, int H, int D,
                                            double* __restrict__ out, double* __restrict__ aw) {
    extern __shared__ double sh[];  // [sk] logits / weights, then [32] reduction
    double* red = sh + sk;
    const int i = blockIdx.x, hd = blockIdx.y, hD = H * D;
    const int lim = i + (sk - sq);  // keys j <= lim are visible
    const double scale = 1.0 / sqrt(static_cast<double>(D));
    const double* qi = q + static_cast<size_t>(i) * hD + hd * D;
    for (int j = threadIdx.x; j < sk; j += blockDim.x) {
        if (j > lim) {
            sh[j] = -INFINITY;
            continue;
        }
        const double* kj = k + static_cast<size_t>(j) * hD + hd * D;
        double dot = 0.0;
        for (int d = 0; d < D; ++d) dot += qi[d] * kj[d];
        sh[j] = dot * scale;
    }
    __syncthreads();
    auto reduce = [&](double x, bool is_max) {
        for (int off = 16; off > 0; off >>= 1) {
            const double o = __shfl_xor_sync(0xffffffffu, x, off);
            x = is_max ? fmax(x, o) : x + o;
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
        __syncthreads();
        double t = is_max ? -INFINITY : 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t = is_max ? fmax(t, red[w]) : t + red[w];
        __syncthreads();
        return t;
    };
    double mx = -INFINITY;
    for (int j = threadIdx.x; j < sk; j += blockDim.x) mx = fmax(mx, sh[j]);
    mx = reduce(mx, true);
    double sum = 0.0;
    for (int j = threadIdx.x; j < sk; j += blockDim.x) {
        const double e = j > lim ? 0.0 : exp(sh[j] - mx);
        sh[j] = e;
        sum += e;
    }
    sum = reduce(sum, false);
    double* awr = aw + (static_cast<size_t>(hd) * sq + i) * sk;
    for (int j = threadIdx.x; j < sk; j += blockDim.x) {
        sh[j] /= sum;
        awr[j] = sh[j];
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        double a = 0.0;
        for (int j = 0; j <= lim && j < sk; ++j) a += sh[j] * v[static_cast<size_t>(j) * hD + hd * D + d];
        out[static_cast<size_t>(i) * hD + hd * D + d] = a;
    }
}

}  // namespace skvd

namespace {
inline cudaStream_t as_st(void* s) { return static_cast<cudaStream_t>(s); }
inline unsigned blocks_for(long long n, int t) { return static_cast<unsigned>((n + t - 1) / t); }
skv_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return SKV_OK;
    skv_impl::fail_msg(SKV_ERR_CUDA, cudaGetErrorString(e));
    return SKV_ERR_CUDA;
}
}  // namespace

extern "C" {

skv_status skv_engine_embed(const double* emb, int h, const int64_t* ids, int n, int pos0, double* out,
                            void* stream) {
    if (!emb || !ids || !out || h <= 0 || n <= 0 || h % 2) return skv_impl::fail_msg(SKV_ERR_CONTRACT, "embed: bad argument");
    skvd::eng_embed_kernel<<<blocks_for(static_cast<long long>(n) * h, 256), 256, 0, as_st(stream)>>>(
        emb, h, reinterpret_cast<const long long*>(ids), n, pos0, out);
    skv_impl::count_launch();
    return cuda_status(cudaGetLastError());
}

skv_status skv_engine_layernorm(const double* x, int rows, int h, const double* gain, const double* bias,
                                double* out, void* stream) {
    if (!x || !gain || !bias || !out || rows <= 0 || h <= 0)
        return skv_impl::fail_msg(SKV_ERR_CONTRACT, "layer_norm: bad argument");
    skvd::eng_layernorm_kernel<<<rows, 256, 0, as_st(stream)>>>(x, h, gain, bias, out);
    skv_impl::count_launch();
    return cuda_status(cudaGetLastError());
}

skv_status skv_engine_gemm(const double* A, const double* B, double* C, int M, int N, int K, int accumulate,
                           void* stream) {
    if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0)
        return skv_impl::fail_msg(SKV_ERR_CONTRACT, "matmul: inner dimensions differ");
    dim3 grid((N + 15) / 16, (M + 15) / 16);
    skvd::eng_gemm_kernel<<<grid, dim3(16, 16), 0, as_st(stream)>>>(A, B, C, M, N, K, accumulate);
    skv_impl::count_launch();
    return cuda_status(cudaGetLastError());
}

skv_status skv_engine_gelu(double* x, size_t n, void* stream) {
    if (!x) return skv_impl::fail_msg(SKV_ERR_CONTRACT, "gelu: null argument");
    if (n == 0) return SKV_OK;
    skvd::eng_gelu_kernel<<<blocks_for(static_cast<long long>(n), 256), 256, 0, as_st(stream)>>>(x, static_cast<long long>(n));
    skv_impl::count_launch();
    return cuda_status(cudaGetLastError());
}

skv_status skv_engine_convert(const double* in, float* out, size_t n, void* stream) {
    if (!in || !out) return skv_impl::fail_msg(SKV_ERR_CONTRACT, "convert: null argument");
    if (n == 0) return SKV_OK;
    skvd::eng_convert_kernel<<<blocks_for(static_cast<long long>(n), 256), 256, 0, as_st(stream)>>>(in, out, static_cast<long long>(n));
    skv_impl::count_launch();
    return cuda_status(cudaGetLastError());
}

skv_status skv_engine_widen(const float* in, double* out, size_t n, void* stream) {
    if (!in || !out) return skv_impl::fail_msg(SKV_ERR_CONTRACT, "widen: null argument");
    if (n == 0) return SKV_OK;
    skvd::eng_widen_kernel<<<blocks_for(static_cast<long long>(n), 256), 256, 0, as_st(stream)>>>(in, out, static_cast<long long>(n));
    skv_impl::count_launch();
    return cuda_status(cudaGetLastError());
}

skv_status skv_engine_causal_attention(const double* q, const double* k, const double* v, int sq, int sk, int heads,
                                       int head_dim, double* out, double* aw, void* stream) {
    if (!q || !k || !v || !out || !aw || heads <= 0 || head_dim <= 0)
        return skv_impl::fail_msg(SKV_ERR_CONTRACT, "dense_attention: null argument");
    if (sq <= 0 || sk <= 0) return skv_impl::fail_msg(SKV_ERR_CONTRACT, "dense_attention: empty input");
    if (sq > sk) return skv_impl::fail_msg(SKV_ERR_CONTRACT, "softmax_rows: row has no finite entry");
    const size_t smem = (static_cast<size_t>(sk) + 32) * 8;
    if (smem > 200 * 1024) return skv_impl::fail_msg(SKV_ERR_UNSUPPORTED, "dense_attention: key length too long for the toy kernel");
    cudaFuncSetAttribute(skvd::eng_causal_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    skvd::eng_causal_attention_kernel<<<dim3(sq, heads), 128, smem, as_st(stream)>>>(q, k, v, sq, sk, heads, head_dim,
                                                                                     out, aw);
    skv_impl::count_launch();
    return cuda_status(cudaGetLastError());
}

}  // extern "C"
