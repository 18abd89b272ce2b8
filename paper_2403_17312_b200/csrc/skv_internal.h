// skv_internal.h -- declarations shared by the translation units of
// libskv_b200.so (not part of the public ABI; see include/skv_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "skv_b200.h"
#include "skv_decode.cuh"
#include "skv_select.cuh"
#include "skv_ledger.cuh"

namespace skv_impl {

void count_launch();
skv_status fail_msg(skv_status s, const char* msg);  // sets skv_last_error()

cudaError_t launch_select(const skvd::SelectParams& p, int batch, bool pdl, cudaStream_t st, int layers = 1);
cudaError_t launch_scatter_fold(double* imp, long long imp_ld, const float* wpart, int G, int m, const int* tok,
                                long long tok_ld, const double* wsum, int n, double* sparsity, double* rows, int batch,
                                cudaStream_t st);
cudaError_t launch_ledger(const skvd::LedgerParams& p, int batch, bool pdl, cudaStream_t st);
cudaError_t launch_transpose_kv_weights(const void* wk, const void* wv, void* bt, int h, cudaStream_t st);
cudaError_t launch_move(const skvd::MoveParams& p, int batch, int max_tokens, bool pdl, cudaStream_t st);
cudaError_t launch_top_k(const double* v, int batch, long long ld, int len, int k, int* out,
                         cudaStream_t st);
cudaError_t launch_quantize(const double* x, long long len, long long cs, uint32_t bits,
                            uint16_t* codes, double* scales, long long* zps, cudaStream_t st);
cudaError_t launch_dequantize(const uint16_t* codes, long long len, long long cs,
                              const double* scales, const long long* zps, double* out,
                              cudaStream_t st);
cudaError_t launch_cache_write(int kv_dtype, int q_dtype, const skvd::CacheView& cv, double* imp, uint8_t* tiers,
                               const void* k, const void* v, int H, int b0, int nb, int t0, int nt, cudaStream_t st);
cudaError_t launch_cache_read(int kv_dtype, const skvd::CacheView& cv, float* out, int H, int b0, int nb, int t0,
                              int nt, cudaStream_t st);
// INT8 recompute write-back: fp32 GEMM rows [M][2h] -> quantised rows at rowmap's (b, slot)
cudaError_t launch_quant_scatter(int q_dtype, const float* C, const int* m_dev, int m_cap, const int2* rowmap,
                                 uint8_t* kv, int H, int kv_ncap, cudaStream_t st);

}  // namespace skv_impl
namespace skvd {
// Epilogue target of the recompute GEMM (skv_gemm.cu): output row r is token
// rowmap[r] = (b, t); column j < h is K, else V, of head (j mod h) / D.
struct KvScatter {
    uint8_t* kv;          // layer base of the cache, rows of `row_bytes`
    const int2* rowmap;   // [M] (b, t)
    int H, D, Ncap, row_bytes;
};
}
namespace skv_impl {
cudaError_t launch_gemm_tn(const void* A, const void* Bt, float* C, const int* m_dev, int M_cap, int N, int K,
                           bool bf16, cudaStream_t st, const skvd::KvScatter* sc = nullptr);
cudaError_t launch_prefill(bool bf16, bool out_f32, const void* kv, const void* q, void* out, double* imp,
                           long long imp_ld, double* psp, int B, int H, int D, int Ncap, int s, uint8_t* scratch,
                           cudaStream_t st, int h_div = 0);
size_t prefill_scratch_bytes(int B, int H, int s);
// INT8 cache layer -> fp16 [B][s][2][H][D] for the tensor-core prefill
cudaError_t launch_dequant_layer_f16(const uint8_t* kv, void* out, int H, int Ncap, int B, int s, cudaStream_t st);
cudaError_t launch_recompute_gather(const uint8_t* x, long long x_seq, long long x_row, const int* lists,
                                    const int* counts, long long list_ld, uint8_t* A, int2* rowmap, int* m_out,
                                    int B, cudaStream_t st, const int* dst_slots = nullptr);

// Fused decode kernel: one instantiation per (kv dtype, q dtype, HG).
struct DecodeLaunch {
    const void* func;
    size_t (*smem)(int m, bool gmem, bool paged);  // gmem: token list + weights in global scratch
    int hg;
    size_t ring_bytes;  // shared-memory ring (reused for the tail's selection keys)
};
// Returns nullptr when no kernel is compiled for the combination.
const DecodeLaunch* find_decode(int kv_dtype, int q_dtype, int hg);
cudaError_t launch_attend(const DecodeLaunch& dl, const skvd::AttendParams& p, int grid_g,
                          size_t smem, bool pdl, cudaStream_t st);

}  // namespace skv_impl
