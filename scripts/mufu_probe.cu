// mufu_probe.cu -- per-SM throughput of MUFU.EX2, FFMA, FFMA2 on sm_100a
// (the prefill's row softmax is bound by one of them).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build_var/mufu_probe scripts/mufu_probe.cu
#include <cstdio>

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int KIND>
__global__ void k(float* out, int iters, long long* cyc) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
    float2 b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = make_float2(a[i], -a[i]);
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0) a[i] = ex2(a[i]) - 1.0001f;
            if (KIND == 1) a[i] = fmaf(a[i], 0.999f, 0.0001f);
            if (KIND == 2) b[i] = __ffma2_rn(b[i], make_float2(0.999f, 0.999f), make_float2(1e-4f, 1e-4f));
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i] + b[i].x + b[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float* o;
    long long* c;
    cudaMalloc(&o, 1 << 20);
    cudaMalloc(&c, 8);
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        for (int kind = 0; kind < 3; ++kind) {
            void (*f)(float*, int, long long*) = kind == 0 ? k<0> : (kind == 1 ? k<1> : k<2>);
            f<<<1, warps * 32>>>(o, iters, c);
            long long cy = 0;
            cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
            const double ops = double(iters) * 8 * warps * 32 * (kind == 2 ? 2 : 1);
            printf("%-6s warps=%2d: %.2f lane-ops/clk/SM (%.2f cycles per warp-instruction per SMSP)\n",
                   kind == 0 ? "EX2" : (kind == 1 ? "FFMA" : "FFMA2"), warps, ops / cy,
                   double(cy) / (double(iters) * 8 * warps / 4));
        }
    }
    return 0;
}
