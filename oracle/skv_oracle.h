/*
 * skv_oracle.h -- CPU restatement of the reference SWA decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the CUDA path in
 * paper_2403_17312_b200/csrc. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it. The product
 * library never links or calls it.
 *
 * Every function restates one reference function from
 * /root/reference/proj/include/skv/ (cited per function). All arithmetic
 * is fp64 in the same operation order as the reference, so results are
 * bit-identical to the reference compiled with the same compiler flags
 * (verified by tests/test_oracle.py against oracle/_ref and tests/golden).
 *
 * Status codes mirror the reference exception classes (common.hpp:12-34):
 *   0 ok, 1 ContractViolation, 2 OutOfDeviceMemory, 3 InfeasiblePlan.
 */
#ifndef SKV_ORACLE_H
#define SKV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OC_OK = 0, OC_CONTRACT = 1, OC_OOM = 2, OC_INFEASIBLE = 3 };

const char* oc_last_error(void);

/* common.hpp:43-54 */
int64_t oc_round_half_even(double x);

/* matrix.hpp:57-105 (std::mt19937_64 + explicit transforms) */
typedef struct {
    uint64_t mt[312];
    int mti;
    double spare;
    int has_spare;
} oc_rng;
void oc_rng_init(oc_rng* r, uint64_t seed);
uint64_t oc_rng_next_u64(oc_rng* r);
double oc_rng_uniform(oc_rng* r);
double oc_rng_normal(oc_rng* r);
uint64_t oc_rng_integer(oc_rng* r, uint64_t bound);
/* Convenience for tests: n successive normal() draws scaled by `gain`. */
void oc_fill_normal(uint64_t seed, double gain, double* out, size_t n);

/* attention.hpp:122-138. Returns 0 and sets OC_CONTRACT when r is outside (0,1]. */
size_t oc_swa_window_k(size_t n, double r);
size_t oc_swa_keep_count(size_t n, double r);

/* matrix.hpp:162-176: k largest, ties -> lower index, result ascending. */
int oc_top_k_indices(const double* v, size_t len, size_t k, int64_t* out);

/* attention.hpp:142-171 + SparseSelection::all (:31-38).
 * Writes the merged selection ascending into out_all (capacity >= n),
 * local/global parts into out_local/out_global when non-NULL. */
int oc_swa_select(const double* importance, size_t importance_len, size_t n, double r,
                  int64_t* out_all, size_t* m_out, size_t* k_out,
                  int64_t* out_local, size_t* n_local, int64_t* out_global,
                  size_t* n_global);

/* attention.hpp:77-85. acc is [H][acc_ld]; sums the first len entries. */
void oc_head_summed_accum(size_t H, const double* acc, size_t acc_ld, size_t len, double* out);

/* attention.hpp:183-231. keys/values are [H][ncap][D] (rows 0..n-1 valid),
 * acc is [H][acc_ld] with entries >= the previous length zero (the
 * reference's acc.resize(n, 0.0)); q is [H][D]; attn [H][D]; new_aw_row [n]. */
int oc_attend_over_indices(size_t H, size_t D, size_t n, size_t ncap, const double* keys,
                           const double* values, double* acc, size_t acc_ld,
                           const double* q, const int64_t* idx, size_t m, double* attn,
                           double* new_aw_row);

/* attention.hpp:235-244: head-sum -> swa_select -> attend. idx_out capacity n. */
int oc_swa_attention(size_t H, size_t D, size_t n, size_t ncap, const double* keys,
                     const double* values, double* acc, size_t acc_ld, const double* q,
                     double r, double* attn, double* new_aw_row, int64_t* idx_out,
                     size_t* m_out);

/* attention.hpp:247-256 / 258-269: index lists of the baseline variants. */
size_t oc_local_attention_mask(size_t n, size_t window, int64_t* out);
size_t oc_strided_attention_mask(size_t n, size_t stride, int64_t* out);
/* engine.hpp:531-569 for Local / Strided (stride 0 = derive from ratio). */
size_t oc_variant_selection(int variant, size_t n_tot, double r, size_t stride, int64_t* out, size_t* k_out);
/* attention.hpp:275-310 */
double oc_attention_sparsity(size_t rows, size_t cols, const double* aw, double rel, int causal);

/* matrix.hpp:137-158 */
int oc_softmax_rows(size_t rows, size_t cols, const double* in, double* out);

/* attention.hpp:91-117 (+ matmul, matrix.hpp:107-122). q [sq][D], k/v [sk][D],
 * attn [sq][D], aw [sq][sk]. */
int oc_dense_attention(size_t sq, size_t sk, size_t D, const double* q, const double* k,
                       const double* v, int causal, double* attn, double* aw);

/* quant.hpp:28-37, 43-81, 84-95 */
int oc_quantize(const double* x, size_t len, uint32_t bits, size_t channel_size,
                uint16_t* codes, double* scales, int64_t* zero_points);
int oc_dequantize(const uint16_t* codes, size_t len, size_t channel_size,
                  const double* scales, const int64_t* zero_points, double* out);

/* memsim.hpp:15-70 (the subset of CostParams the per-step path reads). */
typedef struct {
    size_t hidden, layers, batch, input_len, output_len;
    double ratio, bandwidth;
    size_t bytes_per_element;
    uint64_t device_capacity;
    double mac_rate, recompute_overhead;
} oc_cost;
uint64_t oc_token_kv_bytes(const oc_cost* p);
uint64_t oc_layer_kv_bytes(const oc_cost* p);

/* memsim.hpp:72 Tier */
enum { OC_TIER_DEVICE = 0, OC_TIER_HOST = 1, OC_TIER_DELETED = 2 };

/* memsim.hpp:77-215 KvLedger, with a fixed per-layer token capacity. */
typedef struct {
    size_t layers, ntok_cap;
    uint64_t capacity, device_bytes, host_bytes;
    size_t* row_len;   /* [layers]: the reference's entries_[layer].size() */
    uint8_t* present;  /* [layers][ntok_cap] */
    uint8_t* tier;     /* [layers][ntok_cap] */
    uint64_t* bytes;   /* [layers][ntok_cap] */
} oc_ledger;
int oc_ledger_init(oc_ledger* L, size_t layers, uint64_t capacity, size_t ntok_cap);
void oc_ledger_free(oc_ledger* L);
int oc_ledger_store_new(oc_ledger* L, size_t layer, size_t token, uint64_t bytes);
int oc_ledger_offload(oc_ledger* L, size_t layer, const int64_t* toks, size_t nt, uint64_t* moved);
int oc_ledger_reload(oc_ledger* L, size_t layer, const int64_t* toks, size_t nt, uint64_t* moved);
int oc_ledger_erase(oc_ledger* L, size_t layer, const int64_t* toks, size_t nt, uint64_t* freed);
int oc_ledger_restore(oc_ledger* L, size_t layer, size_t token, uint64_t bytes);
size_t oc_ledger_tokens_in_tier(const oc_ledger* L, size_t layer, int tier, int64_t* out);
int oc_ledger_exists(const oc_ledger* L, size_t layer, size_t token);
/* -1 when not stored */
int oc_ledger_tier(const oc_ledger* L, size_t layer, size_t token);

/* scheduler.hpp:28-39 SchedulePlan (fields the per-step path reads). */
typedef struct {
    double alpha, beta;
    size_t p1, p2;
    int recompute_enabled;
} oc_plan;

/* scheduler.hpp:52-60 */
int oc_phase_of_step(const oc_plan* plan, size_t j);

/* scheduler.hpp:320-381. selection = ascending merged list (SparseSelection::all)
 * plus its k. Output lists have capacity >= ntok_cap. */
int oc_step_actions(const oc_plan* plan, size_t j, const int64_t* selected, size_t m,
                    size_t k, const oc_ledger* L, size_t layer, const oc_cost* p,
                    int* phase, int64_t* offload, size_t* n_off, int64_t* del,
                    size_t* n_del, int64_t* reload, size_t* n_rel, int64_t* recompute,
                    size_t* n_rec);

/* CPU timing leg for bench.py (port kind): `threads` share-nothing workers run
 * oc_swa_attention over (sequence, layer) work items of random N(0,1) data,
 * one decode step per item at length n. Returns wall seconds. */
double oc_bench_swa(size_t H, size_t D, size_t n, double r, size_t items, size_t threads,
                    uint64_t seed);

#ifdef __cplusplus
}
#endif

#endif
