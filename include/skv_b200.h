/*
 * skv_b200.h -- C ABI of the B200 (sm_100a) SWA decode hot path.
 *
 * Drop-in boundary for the reference's header-only C++ library `skv`
 * (/root/reference/proj/include/skv, consumed through the CMake INTERFACE
 * target at proj/CMakeLists.txt:10-14). Each entry point names the reference
 * function it replaces. Plain pointers and sizes only; `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Errors: every call returns skv_status; the codes map 1:1 onto the
 * reference exception classes (common.hpp:12-34) and skv_last_error()
 * returns the message of the calling thread's last failure.
 *
 * Threading: like AttentionState a cache handle has one
 * owner; calls on distinct handles are independent. One handle lives on one
 * device.
 */
#ifndef SKV_B200_H
#define SKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum skv_status {
    SKV_OK = 0,
    SKV_ERR_CONTRACT = 1,    /* skv::ContractViolation   (common.hpp:12) */
    SKV_ERR_OOM = 2,         /* skv::OutOfDeviceMemory   (common.hpp:17) */
    SKV_ERR_INFEASIBLE = 3,  /* skv::InfeasiblePlan      (common.hpp:22) */
    SKV_ERR_CUDA = 4,        /* CUDA runtime failure                      */
    SKV_ERR_UNSUPPORTED = 5  /* shape/dtype outside the compiled kernels  */
} skv_status;

typedef enum skv_dtype {
    SKV_F32 = 0,
    SKV_F16 = 1,
    SKV_BF16 = 2,
    /* 8-bit affine codes, one (scale, bias) fp32 pair per (token, K|V, head):
     * quant.hpp:43-95 applied per head_dim group as engine.hpp:469-483 does. */
    SKV_U8 = 3
} skv_dtype;

typedef struct skv_cache skv_cache;

typedef struct skv_cache_desc {
    int32_t layers;    /* L */
    int32_t batch;     /* B sequences (the reference has one; engine.hpp:289) */
    int32_t heads;     /* H */
    int32_t head_dim;  /* D (128) */
    int32_t capacity;  /* tokens per sequence (Ncap) */
    int32_t kv_dtype;  /* skv_dtype of stored K/V */
    int32_t q_dtype;   /* compute dtype of q / new k,v / out: F32, F16, BF16 */
    int32_t device;    /* CUDA ordinal */
    int32_t out_f32;   /* nonzero: attention outputs are fp32 instead of q_dtype */
} skv_cache_desc;

const char* skv_last_error(void);
const char* skv_version(void);
/* Kernels launched by this library since load (all entry points). */
uint64_t skv_launch_count(void);

/* attention.hpp:122-138. Return 0 (and set SKV_ERR_CONTRACT's message) for r
 * outside (0, 1]. */
size_t skv_swa_window_k(size_t n, double r);
size_t skv_swa_keep_count(size_t n, double r);

/* ---- cache: AttentionState (attention.hpp:45-86) for L layers x B sequences.
 * Device layout: K/V [L][B][Ncap][2][H][D] (token-major), fp64 head-summed
 * importance [L][B][Ncap] (attention.hpp:77-85 kept pre-reduced). */
skv_status skv_cache_create(const skv_cache_desc* desc, skv_cache** out);
skv_status skv_cache_destroy(skv_cache* cache);
skv_status skv_cache_get_desc(const skv_cache* cache, skv_cache_desc* desc, uint64_t* device_bytes);

/* A cache whose device K/V is a PAGED POOL bounded by a KvLedger device
 * capacity (memsim.hpp:77-215, CostParams::device_capacity): every
 * (layer, sequence) owns floor(capacity / (L * B * token bytes)) token slots
 * (at most `capacity` tokens), token bytes = 2 * H * row. With a plan and a
 * host tier attached (skv_cache_set_plan, skv_cache_enable_host_tier), each
 * decode step's offloads and deletions free slots and its reloads,
 * recomputations and the new token (store_new) take them, so a KV larger
 * than the budget decodes within it. The prompt must be written in order
 * (skv_cache_write, token t takes slot t) before the first decode step; a
 * plan is required to decode. The KvLedger capacity check raises
 * SKV_ERR_OOM with the reference's message. */
skv_status skv_cache_create_paged(const skv_cache_desc* desc, uint64_t device_capacity, skv_cache** out);
/* The KvLedger device capacity in bytes for a non-paged cache (default:
 * unbounded): store_new / reload / restore beyond it fail with SKV_ERR_OOM
 * (memsim.hpp:193-200). Decode-time accounting runs with a plan attached. */
skv_status skv_cache_set_capacity(skv_cache* cache, uint64_t device_capacity);
/* KvLedger::device_bytes / host_bytes (memsim.hpp:86-87) summed over layers
 * and sequences, the peak device bytes so far and the capacity; synchronises
 * `stream`. Returns the first failure a kernel reported (SKV_ERR_OOM:
 * "simulated OOM: device tier needs X bytes, capacity C"; SKV_ERR_CONTRACT:
 * a gathered token not device-resident, engine.hpp:625-628). Every decode
 * entry point also returns such a failure on its next call. */
skv_status skv_ledger_totals(const skv_cache* cache, uint64_t* device_bytes, uint64_t* host_bytes,
                             uint64_t* peak_device_bytes, uint64_t* capacity, void* stream);
/* Cumulative rows the applied step_actions listed since creation, summed
 * over layers and sequences: rows[0] offloaded, [1] deleted, [2] reloaded,
 * [3] recomputed, [4] reloads of rows offloaded by the same step (they keep
 * their device row: no host -> device copy). rows holds 5 values.
 * Synchronises `stream`. */
skv_status skv_ledger_counters(const skv_cache* cache, uint64_t* rows, void* stream);
/* Calibration hook for CostParams::bandwidth (bench.hpp's fit is for
 * mac_rate; the reference takes bandwidth as given): times the real duplex
 * movement kernel moving `rows` token rows per sequence device->host and
 * `rows` others host->device on `layer`, `reps` times; *ms per launch. Needs a
 * non-paged cache with a host tier; overwrites that layer's rows and lists. */
skv_status skv_profile_move(skv_cache* cache, int layer, int rows, int reps, double* ms, void* stream);
/* Storage shape: token slots per (layer, sequence), bytes of the device K/V
 * pool, and bytes of the full [L][B][capacity] K/V it stands for. */
skv_status skv_cache_storage(const skv_cache* cache, int32_t* slots_per_sequence, uint64_t* kv_pool_bytes,
                             uint64_t* full_kv_bytes);

/* AttentionState::append_token for tokens [t0, t0+nt) of sequences
 * [b0, b0+nb) (attention.hpp:65-74; fake-quant as engine.hpp:469-483 when
 * kv_dtype is SKV_U8). k, v: device [nb][nt][H][D] in q_dtype. Zeroes the
 * importance of the written tokens (acc.resize(n, 0.0), attention.hpp:219). */
skv_status skv_cache_write(skv_cache* cache, int layer, int b0, int nb, int t0, int nt,
                           const void* k, const void* v, void* stream);
/* Read back (dequantized) K/V as fp32 into device out [nb][nt][2][H][D]. */
skv_status skv_cache_read(const skv_cache* cache, int layer, int b0, int nb, int t0, int nt,
                          float* out, void* stream);
/* Importance accumulator rows: device src/dst [nb][len] fp64. */
skv_status skv_importance_set(skv_cache* cache, int layer, int b0, int nb, int len,
                              const double* src, void* stream);
skv_status skv_importance_get(const skv_cache* cache, int layer, int b0, int nb, int len,
                              double* dst, void* stream);

/* Prefill seeding (engine.hpp:508-512): attend the prompt's last query over
 * all n cached tokens of every sequence and set importance[0, n) to the
 * head-summed attention row. q_last, out: device [B][H][D] q_dtype. */
skv_status skv_prefill_seed(skv_cache* cache, int layer, int n, const void* q_last, void* out,
                            void* stream);

/* Engine::prefill's attention for one layer (engine.hpp:485-529) on tcgen05
 * tensor cores: causal dense_attention (attention.hpp:91-117) of the s prompt
 * queries over cached tokens [0, s) (written first with skv_cache_write),
 * importance[0, s) set to the head-summed last attention row
 * (engine.hpp:508-512) and the per-sequence prefill sparsity recorded
 * (engine.hpp:513-518). fp16/bf16 caches only. q: device [B][s][H][D]
 * q_dtype; out: device [B][s][H][D] (fp32 when out_f32). */
skv_status skv_prefill_layer(skv_cache* cache, int layer, int s, const void* q, void* out, void* stream);
/* Mean over heads of attention_sparsity(aw, 0.01, causal) of the last
 * skv_prefill_layer on `layer`, per sequence: dst [B] (host or device). */
skv_status skv_prefill_sparsity_get(const skv_cache* cache, int layer, double* dst, void* stream);

/* ---- the hot path ---------------------------------------------------------
 * One SWA decode step of one layer for all B sequences, in the engine's
 * order (engine.hpp:592-629): append the new K/V as token n-1, select from
 * the pre-step importance (swa_select, attention.hpp:142-171; dense when
 * 2k >= n), attend over the selection (attend_over_indices,
 * attention.hpp:183-231) and fold the weights into the importance.
 * n counts the current token. q, k_new, v_new: device [B][H][D] q_dtype; out
 * [B][H][D] in q_dtype (fp32 when the cache was created with out_f32).
 * idx_out (nullable): device int32 [B][m] ascending (SparseSelection::all);
 * w_out (nullable): device fp32 [B][H][m] softmax weights in idx order.
 * m = skv_swa_keep_count(n, r). One kernel launch. */
skv_status skv_swa_decode_layer(skv_cache* cache, int layer, int n, double r, const void* q,
                                const void* k_new, const void* v_new, void* out,
                                int32_t* idx_out, float* w_out, void* stream);
/* The part of a decode step of `layer` at length n before its attend
 * (engine.hpp:601-606): variant_selection for (n, r) when none is pending
 * (the previous step normally made it) and, with a plan attached, that
 * step's step_actions + apply_actions on the device ledger. A following
 * skv_swa_decode_layer at (n, r) then only attends. Lets a host read the
 * step's actions (skv_ledger_counters) before the attend runs. */
skv_status skv_decode_prepare(skv_cache* cache, int layer, int n, double r, void* stream);
/* All L layers of one decode step (q/k/v/out device [L][B][H][D]); L launches. */
skv_status skv_swa_decode_step(skv_cache* cache, int n, double r, const void* q,
                               const void* k_new, const void* v_new, void* out, void* stream);
/* Same with HOST buffers (pinned for overlap; pageable works but serialises):
 * the layers are cut into chunks whose q/k/v uploads, attention and output
 * downloads overlap on two internal copy streams ordered against `stream`.
 * Returns after enqueueing: the host buffers must stay untouched until
 * `stream` is synchronised, which also covers every copy of the call. */
skv_status skv_swa_decode_step_host(skv_cache* cache, int n, double r, const void* q_host,
                                    const void* k_host, const void* v_host, void* out_host,
                                    void* stream);

/* attend_over_indices (attention.hpp:183-231) with caller-chosen indices
 * (device int32 [B][m], each < n, any order, repeats allowed: each occurrence
 * is one softmax term and adds its own weight, importance[idx] += w, as the
 * reference loops over them). w_out holds the weights per occurrence. */
skv_status skv_attend_over_indices(skv_cache* cache, int layer, int n, const int32_t* idx,
                                   int m, const void* q, void* out, float* w_out, void* stream);

/* ---- standalone primitives on device buffers ----------------------------- */
/* swa_select (attention.hpp:142-171) for `batch` rows of importance
 * (row stride ld): writes SparseSelection::all() ascending to idx_out
 * [batch][m]; *m_out = m (host). Rows of more than ~27 k candidates keep
 * their keys in a stream-ordered device scratch (cudaMallocAsync) instead of
 * shared memory; the same holds for skv_top_k_indices. Lengths are not
 * capped by the decode path either: long selections move the attend's token
 * list and weights to global scratch. */
skv_status skv_swa_select(const double* importance, int batch, int64_t ld, int n, double r,
                          int32_t* idx_out, int32_t* m_out, void* stream);
/* top_k_indices (matrix.hpp:162-176) per row: out [batch][k] ascending. */
skv_status skv_top_k_indices(const double* v, int batch, int64_t ld, int len, int k,
                             int32_t* out, void* stream);
/* quantize / dequantize (quant.hpp:43-95), bit-exact fp64. */
skv_status skv_quantize(const double* x, size_t len, uint32_t bits, size_t channel_size,
                        uint16_t* codes, double* scales, int64_t* zero_points, void* stream);
skv_status skv_dequantize(const uint16_t* codes, size_t len, size_t channel_size,
                          const double* scales, const int64_t* zero_points, double* out,
                          void* stream);

/* ---- attention variants (AttentionVariant, attention.hpp:15-21) -----------
 * Engine::variant_selection (engine.hpp:531-569) for the decode entry points:
 * DENSE = swa_select at r = 1; SWA (default); LOCAL = the last
 * swa_keep_count(n, r) tokens; STRIDED = every stride-th token phased onto
 * n-1 (stride 0: ceil(n / swa_keep_count(n, r))). */
typedef enum skv_variant {
    SKV_VARIANT_DENSE = 0,
    SKV_VARIANT_SWA = 1,
    SKV_VARIANT_LOCAL = 2,
    SKV_VARIANT_STRIDED = 3
} skv_variant;
skv_status skv_cache_set_variant(skv_cache* cache, int variant, int stride);
/* Selection size m (and its window k) of a step at length n for the cache's
 * variant: what idx_out / w_out of skv_swa_decode_layer hold. */
skv_status skv_selection_size(const skv_cache* cache, int n, double r, int32_t* m, int32_t* k);
/* The selection the next decode step of `layer` will attend at length n
 * with ratio r (SparseSelection::all(), attention.hpp:31-38), made by the
 * previous step's select kernel: idx_out [B][m] int32 ascending (any memory),
 * *m_out = m. SKV_ERR_CONTRACT when no selection for (n, r) is pending. */
skv_status skv_pending_selection(const skv_cache* cache, int layer, int n, double r, int32_t* idx_out,
                                 int32_t* m_out, void* stream);
/* attention_sparsity(new_aw_row, 0.01) (attention.hpp:275-310) of each
 * sequence's last decode step of `layer`; dst [nb] fp64 (host or device). */
skv_status skv_sparsity_get(const skv_cache* cache, int layer, int b0, int nb, double* dst, void* stream);

/* ---- head sharding (SURVEY §8 e: when B < #GPU, e.g. config 1) -----------
 * The selection ranks tokens by the attention weight summed over ALL heads
 * (head_summed_accum, attention.hpp:77-85), so a cache that holds only heads
 * [head_offset, head_offset + H) of total_heads needs, once per layer-step,
 * the head-summed row of the step summed across the shards. The library
 * calls `reduce(buf, count, stream, user)` at that point with `count` fp64
 * values in device memory: it must sum `buf` element-wise across the shards
 * in place, ordered on `stream` (ncclAllReduce(buf, buf, count, ncclDouble,
 * ncclSum, comm, stream) is the intended body). Every shard
 * then folds the same row and makes the same selection. q / k / v / out
 * carry the shard's H heads. The tensor-core prefill's seed row and its
 * sparsity are exchanged the same way. reduce = NULL restores the unsharded
 * cache (head_offset 0, total_heads H or 0). Returning nonzero from reduce
 * fails the calling entry point with that status. */
typedef skv_status (*skv_reduce_fn)(double* buf, size_t count, void* stream, void* user);
skv_status skv_cache_set_head_shard(skv_cache* cache, int head_offset, int total_heads, skv_reduce_fn reduce,
                                    void* user);

/* ---- KV residency bookkeeping for the three-phase schedule ----------------
 * SchedulePlan (scheduler.hpp:28-39) + the workload lengths step_actions reads
 * from CostParams (input_len s, output_len n). */
typedef struct skv_plan {
    double alpha, beta;
    int64_t p1, p2;
    int32_t recompute_enabled;
    int64_t input_len, output_len;
} skv_plan;
/* CostParams (memsim.hpp:15-38): h, l, b, s, n, r, B (bytes/s), element
 * bytes, device capacity (bytes), simulated MAC rate, recompute overhead. */
typedef struct skv_cost_params {
    int64_t hidden, layers, batch, input_len, output_len;
    double ratio, bandwidth;
    int32_t bytes_per_element;
    uint64_t device_capacity;
    double mac_rate, recompute_overhead;
} skv_cost_params;
/* PlanPrediction (scheduler.hpp:75-81) + per-phase PhasePrediction. */
typedef struct skv_plan_prediction {
    double total_seconds, prefill_compute_seconds;
    double phase_compute[3], phase_transfer[3], phase_recompute[3];
    int64_t phase_steps[3];
    uint64_t peak_device_bytes;
    int32_t feasible;
} skv_plan_prediction;
/* solve_plan (scheduler.hpp:207-303), host-side, offline: p1 from capacity,
 * then greedy coordinate descent over (alpha, beta, p2). SKV_ERR_INFEASIBLE
 * as InfeasiblePlan. input_len/output_len of the plan are NOT filled. */
skv_status skv_solve_plan(const skv_cost_params* cost, skv_plan* plan, skv_plan_prediction* prediction);
/* predict_plan (scheduler.hpp:174-186): the simulated objective of a plan. */
skv_status skv_predict_plan(const skv_cost_params* cost, const skv_plan* plan, skv_plan_prediction* prediction);
/* Attach (or with NULL detach) a plan. While attached, every decode step also
 * runs step_actions + apply_actions for the NEXT step on the device ledger
 * right after selecting it (so the lists are ready before that step runs). */
skv_status skv_cache_set_plan(skv_cache* cache, const skv_plan* plan);
/* Host tier for Phase II/III: a pinned, device-mapped mirror of the KV
 * layout. With it (and a plan) every decode step also MOVES the rows the
 * ledger lists: offloads copy device -> host (and with `poison` overwrite the
 * device row with NaN, so any read of a non-resident row shows up), reloads
 * copy host -> device -- apply_actions (engine.hpp:686-716). */
skv_status skv_cache_enable_host_tier(skv_cache* cache, int poison);
/* recompute_kv (engine.hpp:718-737) sources for `layer`: the caller's retained
 * post-LN1 rows x_ln1 [B][capacity][H*D] (stay owned by the caller, must live
 * as long as the attachment) and the projections Wk, Wv [H*D][H*D] row-major
 * (k = x . Wk), copied transposed. With the host tier and a plan, every step
 * then re-derives the ledger's recompute list with one tcgen05 GEMM and writes
 * the K/V rows back. fp16/bf16 caches; x_ln1 = NULL detaches. */
skv_status skv_cache_attach_recompute(skv_cache* cache, int layer, const void* x_ln1, const void* wk,
                                      const void* wv, void* stream);
/* KvLedger tiers per token (memsim.hpp:72): 0 Device, 1 Host, 2 Deleted,
 * 255 not stored. src/dst: [nb][len] bytes (host or device). skv_cache_write
 * marks written tokens Device (store_new). */
skv_status skv_ledger_set(skv_cache* cache, int layer, int b0, int nb, int len, const uint8_t* src, void* stream);
skv_status skv_ledger_get(const skv_cache* cache, int layer, int b0, int nb, int len, uint8_t* dst, void* stream);
/* step_actions (scheduler.hpp:320-381) for step j of `layer`, every
 * sequence, with selection `selected` (device [B][m], ascending; k its
 * window). apply != 0 also applies them (engine.hpp:686-716). lists_out
 * (nullable): [B][4][capacity] offload, delete, reload, recompute;
 * counts_out (nullable): [B][4]. Both any memory; enqueued on `stream`. */
skv_status skv_step_actions(skv_cache* cache, int layer, int j, const int32_t* selected, int m, int k, int apply,
                            int32_t* lists_out, int32_t* counts_out, void* stream);
/* The action lists of the last step_actions run on `layer` (same layout). */
skv_status skv_last_actions(const skv_cache* cache, int layer, int32_t* lists_out, int32_t* counts_out,
                            void* stream);

/* The tcgen05 GEMM recompute_kv uses (C = A . Bt^T; A [M x K], Bt [N x K]
 * row-major fp16 (bf16 != 0: bf16), C [M x N] fp32; M % 128, N % 256,
 * K % 64 == 0). Exposed for tests. */
skv_status skv_gemm_tn(const void* A, const void* Bt, float* C, int M, int N, int K, int bf16, void* stream);

/* ---- the reference toy transformer's dense operators on the GPU (fp64) ---
 * For an engine step around the SWA attention (engine.hpp:571-684, the
 * include/skv/b200_engine.hpp mirror of skv::Engine). All buffers device
 * fp64 row-major, enqueued on `stream`.
 * embed: out[t] = emb[ids[t]] + positional_term(pos0 + t) (engine.hpp:131-144,
 *   360-381); ids device int64 [n].
 * layernorm: layer_norm per row (engine.hpp:111-125), eps 1e-5.
 * gemm: C (+)= A[M x K] . B[K x N] (matmul, matrix.hpp).
 * gelu: tanh GELU in place (engine.hpp:127-129).
 * convert / widen: fp64 -> fp32 and back (the attention cache dtype).
 * causal_attention: dense_attention(q_h, k_h, v_h, true) for every head of
 *   [s][heads*head_dim] q/k/v (attention.hpp:91-117, bottom-right aligned):
 *   out [sq][heads*head_dim], aw [heads][sq][sk]. */
skv_status skv_engine_embed(const double* emb, int h, const int64_t* ids, int n, int pos0, double* out,
                            void* stream);
skv_status skv_engine_layernorm(const double* x, int rows, int h, const double* gain, const double* bias,
                                double* out, void* stream);
skv_status skv_engine_gemm(const double* A, const double* B, double* C, int M, int N, int K, int accumulate,
                           void* stream);
skv_status skv_engine_gelu(double* x, size_t n, void* stream);
skv_status skv_engine_convert(const double* in, float* out, size_t n, void* stream);
skv_status skv_engine_widen(const float* in, double* out, size_t n, void* stream);
skv_status skv_engine_causal_attention(const double* q, const double* k, const double* v, int sq, int sk, int heads,
                                       int head_dim, double* out, double* aw, void* stream);

/* ---- device memory helpers for hosts without the CUDA headers (the C++
 * mirror include/skv/b200.hpp uses these). skv_copy is cudaMemcpyDefault
 * (any direction, UVA) on `stream`, then synchronizes that stream. */
skv_status skv_device_alloc(int device, size_t bytes, void** out);
skv_status skv_device_free(void* ptr);
skv_status skv_copy(void* dst, const void* src, size_t bytes, void* stream);
/* Pinned (page-locked, device-mapped) host memory for the *_host entry
 * points, whose copies overlap compute only from pinned buffers; and a
 * stream synchronisation for hosts without the CUDA runtime. */
skv_status skv_host_alloc(size_t bytes, void** out);
skv_status skv_host_free(void* ptr);
skv_status skv_stream_synchronize(void* stream);

/* ---- measurement hooks (bench.py) ----------------------------------------
 * While enabled, every decode-kernel launch on a cache is bracketed by CUDA
 * events on its own stream; skv_profile_read sums the measured durations. */
skv_status skv_profile_enable(skv_cache* cache, int enable);
skv_status skv_profile_read(skv_cache* cache, double* total_ms, int64_t* launches,
                            uint64_t* algo_bytes);
/* Steady-state attend timing: `reps` x L attend launches back to back
 * (chained with programmatic dependent launch, as inside a decode step, no
 * select kernels) at length n, which must be the pending step of every layer.
 * Re-appends token n-1 with the given rows; importance is not touched.
 * *total_ms = event time around the whole chain. */
skv_status skv_profile_attend_chain(skv_cache* cache, int n, double r, const void* q, const void* k_new,
                                    const void* v_new, void* out, int reps, double* total_ms, void* stream);
/* Launch shape of the last attend launch: heads per CTA, CTAs, dynamic shared
 * memory bytes, resident CTAs per SM. */
skv_status skv_attend_config(const skv_cache* cache, int32_t* heads_per_cta, int32_t* grid,
                             int32_t* smem_bytes, int32_t* ctas_per_sm);

#ifdef __cplusplus
}
#endif

#endif /* SKV_B200_H */
