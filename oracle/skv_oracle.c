/*
 * skv_oracle.c -- CPU restatement of the reference SWA decode hot path.
 * TEST INFRASTRUCTURE ONLY (see skv_oracle.h). Each function cites the
 * reference function it restates; operation order follows the reference so
 * fp64 results are bit-identical to it.
 */
#define _GNU_SOURCE
#include "skv_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[256];

const char* oc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ---- common.hpp:43-54: floor-based round-half-even ---------------------- */
int64_t oc_round_half_even(double x) {
    const double f = floor(x);
    const double frac = x - f;
    int64_t lo = (int64_t)f;
    if (frac > 0.5) return lo + 1;
    if (frac < 0.5) return lo;
    return (lo % 2 == 0) ? lo : lo + 1;
}

/* ---- matrix.hpp:57-105: SeededRng = mt19937_64 + explicit transforms ---- */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void oc_rng_init(oc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    r->mti = MT_N;
    r->spare = 0.0;
    r->has_spare = 0;
}

uint64_t oc_rng_next_u64(oc_rng* r) {
    if (r->mti >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            const uint64_t y = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
            uint64_t v = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = v;
        }
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

double oc_rng_uniform(oc_rng* r) { return (double)(oc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

double oc_rng_normal(oc_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = oc_rng_uniform(r);
    double u2 = oc_rng_uniform(r);
    while (u1 <= 0.0) u1 = oc_rng_uniform(r);
    const double mag = sqrt(-2.0 * log(u1));
    const double ang = 6.283185307179586476925286766559 * u2;
    r->spare = mag * sin(ang);
    r->has_spare = 1;
    return mag * cos(ang);
}

uint64_t oc_rng_integer(oc_rng* r, uint64_t bound) {
    if (bound == 0) return 0;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x = oc_rng_next_u64(r);
    while (x >= limit) x = oc_rng_next_u64(r);
    return x % bound;
}

void oc_fill_normal(uint64_t seed, double gain, double* out, size_t n) {
    oc_rng r;
    oc_rng_init(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = oc_rng_normal(&r) * gain;
}

/* ---- attention.hpp:122-138 ---------------------------------------------- */
size_t oc_swa_window_k(size_t n, double r) {
    if (!(r > 0.0 && r <= 1.0)) {
        fail(OC_CONTRACT, "swa_window_k: ratio out of (0,1]");
        return 0;
    }
    if (n < 2) return 1;
    if (r >= 1.0) return (n + 1) / 2;
    const int64_t rounded = oc_round_half_even((double)n * r / 2.0);
    return rounded < 1 ? 1 : (size_t)rounded;
}

size_t oc_swa_keep_count(size_t n, double r) {
    const size_t k2 = 2 * oc_swa_window_k(n, r);
    return k2 < n ? k2 : n;
}

/* ---- matrix.hpp:162-176: top_k_indices ----------------------------------- */
static __thread const double* t_sort_v;

static int cmp_value_desc_index_asc(const void* a, const void* b) {
    const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
    const double va = t_sort_v[ia], vb = t_sort_v[ib];
    if (va != vb) return va > vb ? -1 : 1;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int oc_top_k_indices(const double* v, size_t len, size_t k, int64_t* out) {
    if (k > len) return fail(OC_CONTRACT, "top_k_indices: k exceeds length");
    int64_t* idx = (int64_t*)malloc((len ? len : 1) * sizeof(int64_t));
    for (size_t i = 0; i < len; ++i) idx[i] = (int64_t)i;
    /* The (value desc, index asc) order is total, so a full sort selects
     * exactly the set partial_sort selects. */
    t_sort_v = v;
    qsort(idx, len, sizeof(int64_t), cmp_value_desc_index_asc);
    qsort(idx, k, sizeof(int64_t), cmp_i64);
    memcpy(out, idx, k * sizeof(int64_t));
    free(idx);
    return OC_OK;
}

/* ---- attention.hpp:142-171 + SparseSelection::all (:31-38) --------------- */
int oc_swa_select(const double* importance, size_t importance_len, size_t n, double r,
                  int64_t* out_all, size_t* m_out, size_t* k_out, int64_t* out_local,
                  size_t* n_local, int64_t* out_global, size_t* n_global) {
    g_err[0] = 0;
    const size_t k = oc_swa_window_k(n, r);
    if (k == 0) return OC_CONTRACT;
    size_t nl = 0, ng = 0;
    int64_t* loc = (int64_t*)malloc((n + 1) * sizeof(int64_t));
    int64_t* glo = (int64_t*)malloc((n + 1) * sizeof(int64_t));
    if (n < 2) {
        for (size_t i = 0; i < n; ++i) loc[nl++] = (int64_t)i;
    } else if (2 * k >= n) {
        const size_t window = k < n ? k : n;
        for (size_t i = n - window; i < n; ++i) loc[nl++] = (int64_t)i;
        for (size_t i = 0; i < n - window; ++i) glo[ng++] = (int64_t)i;
    } else {
        if (importance_len != n - 1) {
            free(loc);
            free(glo);
            return fail(OC_CONTRACT, "swa_select: importance length must be n-1");
        }
        for (size_t i = n - k; i < n; ++i) loc[nl++] = (int64_t)i;
        const int rc = oc_top_k_indices(importance, n - k, k, glo);
        if (rc) {
            free(loc);
            free(glo);
            return rc;
        }
        ng = k;
    }
    /* all(): global then local, sorted ascending */
    size_t m = 0;
    for (size_t i = 0; i < ng; ++i) out_all[m++] = glo[i];
    for (size_t i = 0; i < nl; ++i) out_all[m++] = loc[i];
    qsort(out_all, m, sizeof(int64_t), cmp_i64);
    if (m_out) *m_out = m;
    if (k_out) *k_out = k;
    if (out_local) memcpy(out_local, loc, nl * sizeof(int64_t));
    if (n_local) *n_local = nl;
    if (out_global) memcpy(out_global, glo, ng * sizeof(int64_t));
    if (n_global) *n_global = ng;
    free(loc);
    free(glo);
    return OC_OK;
}

/* ---- attention.hpp:77-85 ------------------------------------------------- */
void oc_head_summed_accum(size_t H, const double* acc, size_t acc_ld, size_t len, double* out) {
    for (size_t i = 0; i < len; ++i) out[i] = 0.0;
    for (size_t h = 0; h < H; ++h)
        for (size_t i = 0; i < len; ++i) out[i] += acc[h * acc_ld + i];
}

/* ---- attention.hpp:183-231 ----------------------------------------------- */
int oc_attend_over_indices(size_t H, size_t D, size_t n, size_t ncap, const double* keys,
                           const double* values, double* acc, size_t acc_ld,
                           const double* q, const int64_t* idx, size_t m, double* attn,
                           double* new_aw_row) {
    if (n < 1) return fail(OC_CONTRACT, "attend_over_indices: empty cache");
    if (m == 0) return fail(OC_CONTRACT, "attend_over_indices: empty selection");
    for (size_t t = 0; t < m; ++t)
        if (idx[t] < 0 || (size_t)idx[t] >= n)
            return fail(OC_CONTRACT, "attend_over_indices: index out of range");
    for (size_t i = 0; i < H * D; ++i) attn[i] = 0.0;
    for (size_t i = 0; i < n; ++i) new_aw_row[i] = 0.0;
    const double scale = 1.0 / sqrt((double)D);
    double* logits = (double*)malloc(m * sizeof(double));
    for (size_t h = 0; h < H; ++h) {
        const double* kh = keys + h * ncap * D;
        const double* vh = values + h * ncap * D;
        const double* qh = q + h * D;
        double mx = -INFINITY;
        for (size_t t = 0; t < m; ++t) {
            double dot = 0.0;
            const double* krow = kh + (size_t)idx[t] * D;
            for (size_t d = 0; d < D; ++d) dot += qh[d] * krow[d];
            logits[t] = dot * scale;
            if (mx < logits[t]) mx = logits[t];
        }
        double sum = 0.0;
        for (size_t t = 0; t < m; ++t) {
            logits[t] = exp(logits[t] - mx);
            sum += logits[t];
        }
        double* ah = acc + h * acc_ld;
        for (size_t t = 0; t < m; ++t) {
            const double w = logits[t] / sum;
            const double* vrow = vh + (size_t)idx[t] * D;
            for (size_t d = 0; d < D; ++d) attn[h * D + d] += w * vrow[d];
            ah[idx[t]] += w;
            new_aw_row[idx[t]] += w;
        }
    }
    free(logits);
    return OC_OK;
}

/* ---- attention.hpp:235-244 ----------------------------------------------- */
int oc_swa_attention(size_t H, size_t D, size_t n, size_t ncap, const double* keys,
                     const double* values, double* acc, size_t acc_ld, const double* q,
                     double r, double* attn, double* new_aw_row, int64_t* idx_out,
                     size_t* m_out) {
    if (n < 1) return fail(OC_CONTRACT, "swa_attention: empty cache");
    const size_t len = n - 1; /* accumulators cover every attended token */
    double* imp = (double*)malloc((len ? len : 1) * sizeof(double));
    oc_head_summed_accum(H, acc, acc_ld, len, imp);
    size_t m = 0;
    int rc = oc_swa_select(imp, len, n, r, idx_out, &m, NULL, NULL, NULL, NULL, NULL);
    free(imp);
    if (rc) return rc;
    if (m_out) *m_out = m;
    return oc_attend_over_indices(H, D, n, ncap, keys, values, acc, acc_ld, q, idx_out, m,
                                  attn, new_aw_row);
}

/* ---- attention.hpp:247-256 ----------------------------------------------- */
size_t oc_local_attention_mask(size_t n, size_t window, int64_t* out) {
    if (window < 1) {
        fail(OC_CONTRACT, "local_attention_mask: window must be >= 1");
        return 0;
    }
    const size_t w = window < n ? window : n;
    size_t c = 0;
    for (size_t i = n - w; i < n; ++i) out[c++] = (int64_t)i;
    return c;
}

/* ---- attention.hpp:258-269 ----------------------------------------------- */
size_t oc_strided_attention_mask(size_t n, size_t stride, int64_t* out) {
    if (stride < 1) {
        fail(OC_CONTRACT, "strided_attention_mask: stride must be >= 1");
        return 0;
    }
    if (n == 0) return 0;
    const size_t phase = (n - 1) % stride;
    size_t c = 0;
    for (size_t i = phase; i < n; i += stride) out[c++] = (int64_t)i;
    return c;
}

/* ---- engine.hpp:545-566 (Local = 2, Strided = 3); result = sel.all() ------ */
size_t oc_variant_selection(int variant, size_t n_tot, double r, size_t stride, int64_t* out, size_t* k_out) {
    if (variant == 2) {
        const size_t w = oc_swa_keep_count(n_tot, r);
        const size_t c = oc_local_attention_mask(n_tot, w, out);
        if (k_out) *k_out = c;
        return c;
    }
    if (stride == 0) {
        const size_t budget = oc_swa_keep_count(n_tot, r);
        stride = (n_tot + budget - 1) / budget;
        if (stride < 1) stride = 1;
    }
    /* local = {n_tot-1}, global = mask minus n_tot-1; all() sorts them back */
    const size_t c = oc_strided_attention_mask(n_tot, stride, out);
    if (k_out) *k_out = 1;
    return c;
}

/* ---- attention.hpp:275-310 ----------------------------------------------- */
double oc_attention_sparsity(size_t rows, size_t cols, const double* aw, double rel, int causal) {
    const long long offset = (long long)cols - (long long)rows;
    size_t counted = 0, sparse = 0;
    for (size_t i = 0; i < rows; ++i) {
        double mx = 0.0;
        size_t cells = 0;
        for (size_t j = 0; j < cols; ++j) {
            if (causal && (long long)j > (long long)i + offset) continue;
            if (mx < aw[i * cols + j]) mx = aw[i * cols + j];
            ++cells;
        }
        counted += cells;
        if (mx == 0.0) {
            sparse += cells;
            continue;
        }
        const double thr = rel * mx;
        for (size_t j = 0; j < cols; ++j) {
            if (causal && (long long)j > (long long)i + offset) continue;
            if (aw[i * cols + j] < thr) ++sparse;
        }
    }
    return counted == 0 ? 0.0 : (double)sparse / (double)counted;
}

/* ---- matrix.hpp:137-158 -------------------------------------------------- */
int oc_softmax_rows(size_t rows, size_t cols, const double* in, double* out) {
    if (rows == 0 || cols == 0) return fail(OC_CONTRACT, "softmax_rows: empty matrix");
    for (size_t i = 0; i < rows; ++i) {
        const double* x = in + i * cols;
        double* y = out + i * cols;
        double mx = -INFINITY;
        for (size_t j = 0; j < cols; ++j)
            if (mx < x[j]) mx = x[j];
        if (!isfinite(mx)) return fail(OC_CONTRACT, "softmax_rows: row has no finite entry");
        double sum = 0.0;
        for (size_t j = 0; j < cols; ++j) {
            const double e = isinf(x[j]) ? 0.0 : exp(x[j] - mx);
            y[j] = e;
            sum += e;
        }
        for (size_t j = 0; j < cols; ++j) y[j] /= sum;
    }
    return OC_OK;
}

/* ---- attention.hpp:91-117 with matmul (matrix.hpp:107-122) --------------- */
int oc_dense_attention(size_t sq, size_t sk, size_t D, const double* q, const double* k,
                       const double* v, int causal, double* attn, double* aw) {
    if (sq == 0 || sk == 0) return fail(OC_CONTRACT, "dense_attention: empty input");
    const double scale = 1.0 / sqrt((double)D);
    double* logits = (double*)malloc(sq * sk * sizeof(double));
    const long long offset = (long long)sk - (long long)sq;
    for (size_t i = 0; i < sq; ++i) {
        for (size_t j = 0; j < sk; ++j) {
            if (causal && (long long)j > (long long)i + offset) {
                logits[i * sk + j] = -INFINITY;
                continue;
            }
            double dot = 0.0;
            for (size_t d = 0; d < D; ++d) dot += q[i * D + d] * k[j * D + d];
            logits[i * sk + j] = dot * scale;
        }
    }
    int rc = oc_softmax_rows(sq, sk, logits, aw);
    free(logits);
    if (rc) return rc;
    for (size_t i = 0; i < sq * D; ++i) attn[i] = 0.0;
    for (size_t i = 0; i < sq; ++i) {
        for (size_t kk = 0; kk < sk; ++kk) {
            const double aik = aw[i * sk + kk];
            if (aik == 0.0) continue;
            for (size_t j = 0; j < D; ++j) attn[i * D + j] += aik * v[kk * D + j];
        }
    }
    return OC_OK;
}

/* ---- quant.hpp:28-37, 43-81 ---------------------------------------------- */
static double quant_scale(double lo, double hi, uint32_t bits) {
    const double floor_ = 1e-12;
    if (hi == lo) {
        const double a = fabs(lo);
        return a > floor_ ? a : floor_;
    }
    const double levels = (double)((1ULL << bits) - 1);
    const double s = (hi - lo) / levels;
    return s > floor_ ? s : floor_;
}

int oc_quantize(const double* x, size_t len, uint32_t bits, size_t channel_size,
                uint16_t* codes, double* scales, int64_t* zero_points) {
    if (len == 0) return fail(OC_CONTRACT, "quantize: empty input");
    if (bits != 4 && bits != 8) return fail(OC_CONTRACT, "quantize: bits must be 4 or 8");
    if (channel_size == 0) channel_size = len;
    if (len % channel_size != 0)
        return fail(OC_CONTRACT, "quantize: channel_size must divide length");
    const size_t groups = len / channel_size;
    const int64_t max_code = (int64_t)((1ULL << bits) - 1);
    for (size_t g = 0; g < groups; ++g) {
        const double* c = x + g * channel_size;
        double lo = c[0], hi = c[0];
        for (size_t i = 0; i < channel_size; ++i) {
            if (c[i] < lo) lo = c[i];
            if (hi < c[i]) hi = c[i];
        }
        const double scale = quant_scale(lo, hi, bits);
        const int64_t zp = oc_round_half_even(-lo / scale);
        scales[g] = scale;
        zero_points[g] = zp;
        for (size_t i = 0; i < channel_size; ++i) {
            int64_t code = oc_round_half_even(c[i] / scale + (double)zp);
            if (code < 0) code = 0;
            if (code > max_code) code = max_code;
            codes[g * channel_size + i] = (uint16_t)code;
        }
    }
    return OC_OK;
}

/* ---- quant.hpp:84-95 ----------------------------------------------------- */
int oc_dequantize(const uint16_t* codes, size_t len, size_t channel_size,
                  const double* scales, const int64_t* zero_points, double* out) {
    if (channel_size == 0 || len % channel_size != 0)
        return fail(OC_CONTRACT, "dequantize: bad channel size");
    for (size_t g = 0; g < len / channel_size; ++g) {
        const double scale = scales[g];
        const double zp = (double)zero_points[g];
        for (size_t i = 0; i < channel_size; ++i) {
            const size_t at = g * channel_size + i;
            out[at] = scale * ((double)codes[at] - zp);
        }
    }
    return OC_OK;
}

/* ---- memsim.hpp:42-48 ---------------------------------------------------- */
uint64_t oc_token_kv_bytes(const oc_cost* p) {
    return 2ULL * p->bytes_per_element * p->batch * p->layers * p->hidden;
}
uint64_t oc_layer_kv_bytes(const oc_cost* p) {
    return 2ULL * p->bytes_per_element * p->batch * p->hidden;
}

/* ---- memsim.hpp:77-215 KvLedger ------------------------------------------ */
int oc_ledger_init(oc_ledger* L, size_t layers, uint64_t capacity, size_t ntok_cap) {
    memset(L, 0, sizeof *L);
    if (layers == 0) return fail(OC_CONTRACT, "KvLedger: zero layers");
    L->layers = layers;
    L->ntok_cap = ntok_cap;
    L->capacity = capacity;
    L->row_len = (size_t*)calloc(layers, sizeof(size_t));
    L->present = (uint8_t*)calloc(layers * ntok_cap, 1);
    L->tier = (uint8_t*)calloc(layers * ntok_cap, 1);
    L->bytes = (uint64_t*)calloc(layers * ntok_cap, sizeof(uint64_t));
    return OC_OK;
}

void oc_ledger_free(oc_ledger* L) {
    free(L->row_len);
    free(L->present);
    free(L->tier);
    free(L->bytes);
    memset(L, 0, sizeof *L);
}

int oc_ledger_exists(const oc_ledger* L, size_t layer, size_t token) {
    return token < L->row_len[layer] && L->present[layer * L->ntok_cap + token];
}

int oc_ledger_tier(const oc_ledger* L, size_t layer, size_t token) {
    if (!oc_ledger_exists(L, layer, token)) return -1;
    return L->tier[layer * L->ntok_cap + token];
}

static int check_fit(const oc_ledger* L, uint64_t incoming) {
    if (L->device_bytes + incoming > L->capacity) {
        snprintf(g_err, sizeof g_err,
                 "simulated OOM: device tier needs %llu bytes, capacity %llu",
                 (unsigned long long)(L->device_bytes + incoming),
                 (unsigned long long)L->capacity);
        return OC_OOM;
    }
    return OC_OK;
}

int oc_ledger_store_new(oc_ledger* L, size_t layer, size_t token, uint64_t bytes) {
    if (layer >= L->layers) return fail(OC_CONTRACT, "KvLedger: layer out of range");
    if (token >= L->ntok_cap) return fail(OC_CONTRACT, "KvLedger: token beyond capacity");
    if (token >= L->row_len[layer]) L->row_len[layer] = token + 1;
    const size_t at = layer * L->ntok_cap + token;
    if (L->present[at]) return fail(OC_CONTRACT, "KvLedger: token already stored");
    int rc = check_fit(L, bytes);
    if (rc) return rc;
    L->present[at] = 1;
    L->tier[at] = OC_TIER_DEVICE;
    L->bytes[at] = bytes;
    L->device_bytes += bytes;
    return OC_OK;
}

static int entry_for_move(const oc_ledger* L, size_t layer, int64_t t, size_t* at) {
    if (layer >= L->layers) return fail(OC_CONTRACT, "KvLedger: layer out of range");
    if (t < 0 || !oc_ledger_exists(L, layer, (size_t)t))
        return fail(OC_CONTRACT, "KvLedger: entry not stored");
    *at = layer * L->ntok_cap + (size_t)t;
    if (L->tier[*at] == OC_TIER_DELETED) return fail(OC_CONTRACT, "KvLedger: entry is deleted");
    return OC_OK;
}

int oc_ledger_offload(oc_ledger* L, size_t layer, const int64_t* toks, size_t nt, uint64_t* moved) {
    uint64_t mv = 0;
    for (size_t i = 0; i < nt; ++i) {
        size_t at;
        int rc = entry_for_move(L, layer, toks[i], &at);
        if (rc) return rc;
        if (L->tier[at] != OC_TIER_DEVICE)
            return fail(OC_CONTRACT, "offload: entry not device-resident");
        L->tier[at] = OC_TIER_HOST;
        L->device_bytes -= L->bytes[at];
        L->host_bytes += L->bytes[at];
        mv += L->bytes[at];
    }
    if (moved) *moved = mv;
    return OC_OK;
}

int oc_ledger_reload(oc_ledger* L, size_t layer, const int64_t* toks, size_t nt, uint64_t* moved) {
    uint64_t mv = 0;
    for (size_t i = 0; i < nt; ++i) {
        size_t at;
        int rc = entry_for_move(L, layer, toks[i], &at);
        if (rc) return rc;
        if (L->tier[at] != OC_TIER_HOST) return fail(OC_CONTRACT, "reload: entry not host-resident");
        rc = check_fit(L, L->bytes[at]);
        if (rc) return rc;
        L->tier[at] = OC_TIER_DEVICE;
        L->host_bytes -= L->bytes[at];
        L->device_bytes += L->bytes[at];
        mv += L->bytes[at];
    }
    if (moved) *moved = mv;
    return OC_OK;
}

int oc_ledger_erase(oc_ledger* L, size_t layer, const int64_t* toks, size_t nt, uint64_t* freed) {
    uint64_t fr = 0;
    for (size_t i = 0; i < nt; ++i) {
        size_t at;
        int rc = entry_for_move(L, layer, toks[i], &at);
        if (rc) return rc;
        if (L->tier[at] == OC_TIER_DEVICE)
            L->device_bytes -= L->bytes[at];
        else
            L->host_bytes -= L->bytes[at];
        fr += L->bytes[at];
        L->tier[at] = OC_TIER_DELETED;
        L->bytes[at] = 0;
    }
    if (freed) *freed = fr;
    return OC_OK;
}

int oc_ledger_restore(oc_ledger* L, size_t layer, size_t token, uint64_t bytes) {
    if (layer >= L->layers) return fail(OC_CONTRACT, "KvLedger: layer out of range");
    if (!oc_ledger_exists(L, layer, token)) return fail(OC_CONTRACT, "restore: entry never stored");
    const size_t at = layer * L->ntok_cap + token;
    if (L->tier[at] != OC_TIER_DELETED) return fail(OC_CONTRACT, "restore: entry not deleted");
    int rc = check_fit(L, bytes);
    if (rc) return rc;
    L->tier[at] = OC_TIER_DEVICE;
    L->bytes[at] = bytes;
    L->device_bytes += bytes;
    return OC_OK;
}

size_t oc_ledger_tokens_in_tier(const oc_ledger* L, size_t layer, int tier, int64_t* out) {
    size_t c = 0;
    for (size_t t = 0; t < L->row_len[layer]; ++t) {
        const size_t at = layer * L->ntok_cap + t;
        if (L->present[at] && L->tier[at] == tier) out[c++] = (int64_t)t;
    }
    return c;
}

/* ---- scheduler.hpp:52-60 ------------------------------------------------- */
int oc_phase_of_step(const oc_plan* plan, size_t j) {
    if (j < plan->p1) return 1;
    if (j < plan->p2 || !plan->recompute_enabled) return 2;
    return 3;
}

static int in_sorted(const int64_t* a, size_t n, int64_t t) {
    size_t lo = 0, hi = n;
    while (lo < hi) {
        const size_t mid = (lo + hi) / 2;
        if (a[mid] < t)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo < n && a[lo] == t;
}

/* ---- scheduler.hpp:320-381 ----------------------------------------------- */
int oc_step_actions(const oc_plan* plan, size_t j, const int64_t* selected, size_t m,
                    size_t k, const oc_ledger* L, size_t layer, const oc_cost* p,
                    int* phase, int64_t* offload, size_t* n_off, int64_t* del,
                    size_t* n_del, int64_t* reload, size_t* n_rel, int64_t* recompute,
                    size_t* n_rec) {
    *n_off = *n_del = *n_rel = *n_rec = 0;
    if (!(j < p->output_len)) return fail(OC_CONTRACT, "step_actions: step beyond output length");
    if (layer >= L->layers) return fail(OC_CONTRACT, "KvLedger: layer out of range");
    *phase = oc_phase_of_step(plan, j);
    if (*phase == 1) return OC_OK;
    const size_t existing = p->input_len + j;
    const size_t n_tot = existing + 1;
    const size_t nonlocal = n_tot > k ? n_tot - k : 0;

    int64_t* device = (int64_t*)malloc((L->ntok_cap + 1) * sizeof(int64_t));
    int64_t* host = (int64_t*)malloc((L->ntok_cap + 1) * sizeof(int64_t));
    const size_t nd = oc_ledger_tokens_in_tier(L, layer, OC_TIER_DEVICE, device);
    const size_t nh = oc_ledger_tokens_in_tier(L, layer, OC_TIER_HOST, host);

    const size_t target = (size_t)ceil(plan->alpha * (double)existing);
    size_t to_offload = target > nh ? target - nh : 0;
    for (size_t i = 0; i < nd; ++i) {
        const int64_t t = device[i];
        if (to_offload == 0 || (size_t)t >= nonlocal) break;
        offload[(*n_off)++] = t;
        --to_offload;
    }
    const size_t host_after = nh + *n_off;
    if (*phase == 3 && host_after > 0) {
        size_t to_delete = (size_t)ceil(plan->beta * (double)host_after);
        int64_t* host_then = (int64_t*)malloc((host_after + 1) * sizeof(int64_t));
        memcpy(host_then, host, nh * sizeof(int64_t));
        memcpy(host_then + nh, offload, *n_off * sizeof(int64_t));
        qsort(host_then, host_after, sizeof(int64_t), cmp_i64);
        for (size_t i = 0; i < host_after; ++i) {
            if (to_delete == 0) break;
            del[(*n_del)++] = host_then[i];
            --to_delete;
        }
        free(host_then);
    }
    for (size_t i = 0; i < m; ++i) {
        const int64_t t = selected[i];
        if (!oc_ledger_exists(L, layer, (size_t)t)) continue;
        const int tier = oc_ledger_tier(L, layer, (size_t)t);
        if (in_sorted(del, *n_del, t) || tier == OC_TIER_DELETED)
            recompute[(*n_rec)++] = t;
        else if (tier == OC_TIER_HOST || in_sorted(offload, *n_off, t))
            reload[(*n_rel)++] = t;
    }
    free(device);
    free(host);
    return OC_OK;
}

/* ---- CPU timing leg ------------------------------------------------------ */
typedef struct {
    size_t H, D, n0, items;
    double r;
    uint64_t seed;
    pthread_barrier_t* bar;
    double t_start, t_end;
} bench_arg;

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* Rounds of up to 16 decode items (append + swa_attention) at n = n0 .. n0+15,
 * then the state is truncated back to n0-1 tokens, so every timed item runs at
 * the requested length. Only the item loops are timed (busy time). */
static void* bench_worker(void* vp) {
    bench_arg* a = (bench_arg*)vp;
    const size_t H = a->H, D = a->D, round = 16, ncap = a->n0 + round;
    double* keys = (double*)malloc(H * ncap * D * sizeof(double));
    double* vals = (double*)malloc(H * ncap * D * sizeof(double));
    double* acc = (double*)calloc(H * ncap, sizeof(double));
    double* acc0 = (double*)calloc(H * ncap, sizeof(double));
    double* qin = (double*)malloc(round * H * D * sizeof(double));
    double* kin = (double*)malloc(round * H * D * sizeof(double));
    double* vin = (double*)malloc(round * H * D * sizeof(double));
    double* attn = (double*)malloc(H * D * sizeof(double));
    double* aw = (double*)malloc(ncap * sizeof(double));
    int64_t* idx = (int64_t*)malloc(ncap * sizeof(int64_t));
    oc_rng rng;
    oc_rng_init(&rng, a->seed);
    for (size_t h = 0; h < H; ++h)
        for (size_t t = 0; t + 1 < a->n0; ++t) {
            for (size_t d = 0; d < D; ++d) {
                keys[(h * ncap + t) * D + d] = oc_rng_normal(&rng);
                vals[(h * ncap + t) * D + d] = oc_rng_normal(&rng);
            }
            acc0[h * ncap + t] = oc_rng_uniform(&rng);
        }
    pthread_barrier_wait(a->bar);
    double busy = 0.0;
    for (size_t done = 0; done < a->items;) {
        memcpy(acc, acc0, H * ncap * sizeof(double));
        const size_t cnt = a->items - done < round ? a->items - done : round;
        for (size_t i = 0; i < cnt * H * D; ++i) { /* the round's inputs (untimed) */
            kin[i] = oc_rng_normal(&rng);
            vin[i] = oc_rng_normal(&rng);
            qin[i] = oc_rng_normal(&rng);
        }
        const double t0 = now_s();
        for (size_t it = 0; it < cnt; ++it) {
            const size_t n = a->n0 + it; /* append token n-1, then attend */
            for (size_t h = 0; h < H; ++h) {
                memcpy(keys + (h * ncap + n - 1) * D, kin + (it * H + h) * D, D * sizeof(double));
                memcpy(vals + (h * ncap + n - 1) * D, vin + (it * H + h) * D, D * sizeof(double));
            }
            size_t m;
            oc_swa_attention(H, D, n, ncap, keys, vals, acc, ncap, qin + it * H * D, a->r, attn, aw, idx, &m);
        }
        busy += now_s() - t0;
        done += cnt;
    }
    a->t_start = 0.0;
    a->t_end = busy;
    free(keys);
    free(vals);
    free(acc);
    free(acc0);
    free(qin);
    free(kin);
    free(vin);
    free(attn);
    free(aw);
    free(idx);
    return NULL;
}

double oc_bench_swa(size_t H, size_t D, size_t n, double r, size_t items, size_t threads,
                    uint64_t seed) {
    if (threads == 0) threads = 1;
    pthread_t* th = (pthread_t*)malloc(threads * sizeof(pthread_t));
    bench_arg* args = (bench_arg*)malloc(threads * sizeof(bench_arg));
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)threads);
    for (size_t i = 0; i < threads; ++i) {
        const size_t share = items / threads + (i < items % threads ? 1 : 0);
        args[i] = (bench_arg){H, D, n, share, r, seed + 7919u * i, &bar, 0.0, 0.0};
        pthread_create(&th[i], NULL, bench_worker, &args[i]);
    }
    for (size_t i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    double busy = 0.0; /* the slowest worker's timed item time */
    for (size_t i = 0; i < threads; ++i)
        if (args[i].t_end > busy) busy = args[i].t_end;
    pthread_barrier_destroy(&bar);
    free(th);
    free(args);
    return busy;
}
