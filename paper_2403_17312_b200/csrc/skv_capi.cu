// skv_capi.cu -- the C ABI (include/skv_b200.h): argument checking with the
// reference's error semantics, the device cache object, kernel selection and
// launch, host-buffer step, and the measurement hooks used by bench.py.
#include <algorithm>
#include <mutex>
#include <map>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "skv_internal.h"

namespace skv_impl {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace skv_impl

using namespace skv_impl;

namespace {

thread_local std::string g_err;
}  // namespace

namespace skv_impl {
skv_status fail_msg(skv_status s, const char* msg) {
    g_err = msg;
    return s;
}
}  // namespace skv_impl

namespace {

skv_status fail(skv_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define SKV_CUDA(expr)                                                                   \
    do {                                                                                 \
        const cudaError_t e_ = (expr);                                                   \
        if (e_ != cudaSuccess) return fail(SKV_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

#define SKV_REQUIRE(cond, msg)                                \
    do {                                                      \
        if (!(cond)) return fail(SKV_ERR_CONTRACT, "%s", msg); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

size_t dtype_size(int dt) {
    switch (dt) {
    case SKV_F32: return 4;
    case SKV_F16: return 2;
    case SKV_BF16: return 2;
    case SKV_U8: return 1;
    }
    return 0;
}

// common.hpp:43-54 semantics: floor-based half-to-even, FP-env independent.
long long round_half_even_host(double x) {
    const double f = std::floor(x);
    const double frac = x - f;
    const long long lo = static_cast<long long>(f);
    if (frac > 0.5) return lo + 1;
    if (frac < 0.5) return lo;
    return (lo % 2 == 0) ? lo : lo + 1;
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

struct skv_cache;
static size_t out_size(const skv_cache* c);

struct skv_cache {
    skv_cache_desc d{};
    size_t row_bytes = 0;    // one head row of D elements (storage dtype)
    size_t tok_bytes = 0;    // K+V of one token, all heads
    size_t layer_bytes = 0;  // device K/V of one layer: [B][pcap] token slots
    size_t host_layer_bytes = 0;  // host tier of one layer: [B][Ncap] tokens
    uint8_t* kv = nullptr;
    float2* meta = nullptr;
    double* imp = nullptr;
    float* wpart = nullptr;  // [L][B][H][Ncap] per-head-group weight sums of the last attend
    int* idx = nullptr;      // [L][B][Ncap] selection (ascending) for the pending step
    uint8_t* tiers = nullptr;  // [L][B][Ncap] KvLedger tiers: 0 device, 1 host, 2 deleted, 255 absent
    int* act_lists = nullptr;  // [L][B][4][Ncap] last step_actions lists
    int* act_counts = nullptr; // [L][B][4]
    double* sparsity = nullptr;  // [L][B] attention_sparsity of the last step's row
    uint8_t* host_kv = nullptr;  // host tier: mapped pinned mirror of the device layout (or null)
    // recompute_kv sources (engine.hpp:718-737): per layer the caller's retained
    // post-LN1 rows [B][Ncap][h] and our transposed [Wk | Wv]^T [2h][h]
    std::vector<const uint8_t*> rec_x;
    std::vector<uint8_t*> rec_wt;
    uint8_t* rec_a = nullptr;  // gathered rows [B*Ncap][h]
    float* rec_c = nullptr;    // INT8 caches: the GEMM's fp32 K|V rows [B*Ncap][2h] before quantisation
    int2* rec_map = nullptr;   // [B*Ncap] (b, t)
    unsigned* counters = nullptr;  // [L][B] attend-tail arrival counters (zero between launches)
    int* rec_m = nullptr;      // gathered row count
    bool poison = false;         // offload overwrites device rows (checks residency)
    int variant = SKV_VARIANT_SWA, stride = 0;  // SparsityConfig (attention.hpp:15-21)
    bool has_plan = false;
    skv_plan plan{};
    std::vector<long long> ledger_j;  // per layer: last step whose actions were applied (-1: none)
    std::vector<int> pend_n;     // per layer: n the index buffer was selected for (-1: none)
    std::vector<double> pend_r;  // per layer: its ratio
    std::vector<uint8_t> pend_topk;  // per layer: the pending selection is an SWA top-k (incremental_select)
    uint64_t device_bytes = 0;
    int num_sms = 0;
    int max_smem = 0;
    // tensor-core prefill: scratch (grown on demand) and per-(layer, b)
    // prefill sparsity (engine.hpp:513-518)
    uint8_t* pf_scratch = nullptr;
    size_t pf_bytes = 0;
    double* pf_sparsity = nullptr;
    // host-buffer step staging: layer chunks pipelined over two copy streams
    uint8_t* stage = nullptr;
    size_t stage_bytes = 0;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    // whole-step decode: the batched select of the first layers runs on this
    // side stream while the remaining layers' attends stream on the caller's
    cudaStream_t sel_st = nullptr;
    cudaEvent_t ev_sel_in = nullptr, ev_sel_out = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_comp, ev_out;  // per chunk
    // head sharding: this cache holds heads [head_offset, head_offset + H) of
    // total_heads; the head-summed rows are summed across shards by `reduce`
    skv_reduce_fn reduce = nullptr;
    void* reduce_user = nullptr;
    int head_offset = 0, total_heads = 0;
    double* xbuf = nullptr;  // head shards: [L][B][Ncap] step rows of a whole step / prefill seed rows + [B] sparsity
    uint64_t* gkeys = nullptr;  // [L][B][Ncap] top-k keys of long contexts (lazily)
    int* gtok = nullptr;        // [B][H][Ncap] attend token lists of long selections (lazily)
    float* gwts = nullptr;      // [B][H][Ncap] their logits / weights
    double* frow = nullptr;     // [B][Ncap] step-row scratch of attend_over_indices with unsorted / repeated indices
    // whole-step decode with separate select kernels: the layers' fold+select
    // launches are collected and issued as one batched launch after the
    // step's attends (they only feed the next step), instead of one select
    // CTA set interleaved with every attend
    bool in_step = false;  // inside skv_swa_decode_step(_host): a whole step's layers
    bool defer_select = false;
    std::vector<std::pair<int, skvd::SelectParams>> deferred;  // (layer, params)
    // paged store (skv_cache_create_paged): every (layer, sequence) owns pcap
    // token slots of the device pool; offload / erase free them, reload /
    // restore / store_new allocate them (ledger_step_kernel)
    bool paged = false;
    int pcap = 0;                  // slots per (layer, sequence); the capacity when not paged
    int* slot = nullptr;           // [L][B][Ncap] token -> slot, -1 not on device
    int* fq = nullptr;             // [L][B][pcap] free-slot FIFO rings
    unsigned* fq_ht = nullptr;     // [L][B][2] (head, free count)
    int* act_slots = nullptr;      // [L][B][4][Ncap] slots of the last action lists
    int* aux = nullptr;            // [L][B][4] reload split (recycled destinations)
    // KvLedger byte accounting (memsim.hpp:77-215) and the device status
    skvd::LedgerTotals* tot = nullptr;
    unsigned* arrive = nullptr;                // [L]
    unsigned long long* layer_allocs = nullptr;  // [L]
    uint64_t cap_bytes = ~0ull;                // KvLedger device_capacity
    skvd::DevStatus* status = nullptr;         // mapped pinned host memory
    skvd::DevStatus* status_dev = nullptr;     // its device alias
    std::vector<int> ident;        // [L][B] prompt high-water mark (tokens written in order from 0)
    std::vector<char> decoded;     // [L] a decode step ran on this layer
    // measurement
    bool prof = false;
    std::vector<cudaEvent_t> ev;  // start/stop pairs
    std::vector<cudaEvent_t> ev_pool;
    int64_t attend_launches = 0;
    uint64_t algo_bytes = 0;
    int last_hg = 0, last_grid = 0, last_occ = 0;
    const void* attr_func = nullptr;  // attend kernel whose smem attribute was last set
    size_t attr_smem = 0;
    size_t last_smem = 0;
};

constexpr int kHostChunks = 2;  // layer chunks of the host-buffer step pipeline (2 measured best: 1.08 ms vs 0.97 ms copy bound at config 2)

static size_t out_size(const skv_cache* c) { return c->d.out_f32 ? 4 : dtype_size(c->d.q_dtype); }

// The device status (mapped pinned memory) as an error: the first KvLedger
// OOM (memsim.hpp:193-200, the reference's message) or residency violation
// (engine.hpp:625-628) a kernel reported. Sticky, like the reference's throw.
static skv_status check_status(const skv_cache* c) {
    if (c == nullptr || c->status == nullptr) return SKV_OK;
    const volatile skvd::DevStatus* st = c->status;
    const int code = st->code;
    if (code <= 0) return SKV_OK;
    if (code == 2) {
        if (st->needed > 0)
            return fail(SKV_ERR_OOM, "simulated OOM: device tier needs %llu bytes, capacity %llu",
                        static_cast<unsigned long long>(st->needed), static_cast<unsigned long long>(st->capacity));
        return fail(SKV_ERR_OOM, "device KV pool exhausted: a (layer, sequence) slot pool of layer %d is full at "
                    "step %lld", st->layer, static_cast<long long>(st->step));
    }
    return fail(SKV_ERR_CONTRACT, "decode_step: gathered token not device-resident (layer %d sequence %d token %d)",
                st->layer, st->seq, st->token);
}

static skvd::CacheView cache_view(skv_cache* c, int layer) {
    skvd::CacheView v{};
    const size_t lt = static_cast<size_t>(layer) * c->d.batch * c->d.capacity;
    v.kv = c->kv + layer * c->layer_bytes;
    v.Ncap = c->d.capacity;
    v.kv_ncap = c->pcap;
    v.slot = c->paged ? c->slot + lt : nullptr;
    v.fq_ht = c->paged ? c->fq_ht + static_cast<size_t>(layer) * c->d.batch * 2 : nullptr;
    v.tot = c->tot;
    return v;
}

extern "C" {

const char* skv_last_error(void) { return g_err.c_str(); }

const char* skv_version(void) { return "skv_b200 0.1 sm_100a"; }

uint64_t skv_launch_count(void) { return g_launches.load(); }

// attention.hpp:122-132
size_t skv_swa_window_k(size_t n, double r) {
    if (!(r > 0.0 && r <= 1.0)) {
        fail(SKV_ERR_CONTRACT, "swa_window_k: ratio out of (0,1]");
        return 0;
    }
    if (n < 2) return 1;
    if (r >= 1.0) return (n + 1) / 2;
    const long long rounded = round_half_even_host(static_cast<double>(n) * r / 2.0);
    return rounded < 1 ? 1 : static_cast<size_t>(rounded);
}

// attention.hpp:136-138
size_t skv_swa_keep_count(size_t n, double r) {
    const size_t k = skv_swa_window_k(n, r);
    if (k == 0) return 0;
    return 2 * k < n ? 2 * k : n;
}

static skv_status cache_create_impl(const skv_cache_desc* desc, uint64_t paged_capacity, skv_cache** out) {
    SKV_REQUIRE(desc != nullptr && out != nullptr, "skv_cache_create: null argument");
    const skv_cache_desc& d = *desc;
    SKV_REQUIRE(d.layers > 0 && d.batch > 0 && d.heads > 0 && d.capacity > 0,
                "skv_cache_create: zero dimension");
    if (d.head_dim != skvd::kHeadDim)
        return fail(SKV_ERR_UNSUPPORTED, "skv_cache_create: head_dim %d (compiled for %d)", d.head_dim,
                    skvd::kHeadDim);
    const bool ok_pair = (d.kv_dtype == d.q_dtype && d.kv_dtype != SKV_U8) ||
                         (d.kv_dtype == SKV_U8 && d.q_dtype != SKV_U8 && dtype_size(d.q_dtype) > 0);
    if (!ok_pair || dtype_size(d.kv_dtype) == 0)
        return fail(SKV_ERR_UNSUPPORTED, "skv_cache_create: kv_dtype %d with q_dtype %d", d.kv_dtype,
                    d.q_dtype);
    if (d.kv_dtype == SKV_U8 && d.heads % skvd::kU8Group != 0)
        return fail(SKV_ERR_UNSUPPORTED, "skv_cache_create: INT8 storage groups heads by %d (heads %d)",
                    skvd::kU8Group, d.heads);
    DeviceGuard guard(d.device);
    skv_cache* c = new skv_cache();
    c->d = d;
    // one stored head row; INT8 rows carry their (scale, bias) pair inline
    c->row_bytes = static_cast<size_t>(d.head_dim) * dtype_size(d.kv_dtype) + (d.kv_dtype == SKV_U8 ? 8 : 0);
    c->tok_bytes = 2 * static_cast<size_t>(d.heads) * c->row_bytes;
    c->paged = paged_capacity > 0;
    if (c->paged) {
        // the KvLedger capacity split evenly over (layer, sequence) slot pools
        const uint64_t per = paged_capacity / (static_cast<uint64_t>(d.layers) * d.batch * c->tok_bytes);
        if (per < 1) {
            delete c;
            return fail(SKV_ERR_OOM, "simulated OOM: device tier needs %llu bytes, capacity %llu",
                        static_cast<unsigned long long>(static_cast<uint64_t>(d.layers) * d.batch * c->tok_bytes),
                        static_cast<unsigned long long>(paged_capacity));
        }
        c->pcap = static_cast<int>(std::min<uint64_t>(per, static_cast<uint64_t>(d.capacity)));
        c->cap_bytes = paged_capacity;
    } else {
        c->pcap = d.capacity;
    }
    c->layer_bytes = static_cast<size_t>(d.batch) * c->pcap * c->tok_bytes;
    c->host_layer_bytes = static_cast<size_t>(d.batch) * d.capacity * c->tok_bytes;
    const size_t kv_bytes = c->layer_bytes * d.layers;
    const size_t meta_bytes = 0;  // inline in the INT8 rows
    const size_t cells = static_cast<size_t>(d.layers) * d.batch * d.capacity;
    const size_t imp_bytes = cells * 8;
    const size_t wpart_bytes = cells * d.heads * 4;
    const size_t cnt_bytes = cells * 4;  // selections
    const size_t tier_bytes = cells;
    const size_t list_bytes = cells * 4 * 4;
    const size_t acnt_bytes = static_cast<size_t>(d.layers) * d.batch * 4 * 4;
    const size_t sp_bytes = static_cast<size_t>(d.layers) * d.batch * 8;
    const size_t ctr_bytes = static_cast<size_t>(d.layers) * d.batch * 4;
    auto alloc = [&](void** p, size_t bytes) -> bool {
        if (bytes == 0) return true;
        if (cudaMalloc(p, bytes) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        c->device_bytes += bytes;
        return true;
    };
    bool ok = alloc(reinterpret_cast<void**>(&c->kv), kv_bytes) &&
              alloc(reinterpret_cast<void**>(&c->meta), meta_bytes) &&
              alloc(reinterpret_cast<void**>(&c->imp), imp_bytes) &&
              alloc(reinterpret_cast<void**>(&c->wpart), wpart_bytes) &&
              alloc(reinterpret_cast<void**>(&c->idx), cnt_bytes) &&
              alloc(reinterpret_cast<void**>(&c->tiers), tier_bytes) &&
              alloc(reinterpret_cast<void**>(&c->act_lists), list_bytes) &&
              alloc(reinterpret_cast<void**>(&c->act_counts), acnt_bytes) &&
              alloc(reinterpret_cast<void**>(&c->sparsity), sp_bytes) &&
              alloc(reinterpret_cast<void**>(&c->counters), ctr_bytes) &&
              alloc(reinterpret_cast<void**>(&c->tot), sizeof(skvd::LedgerTotals)) &&
              alloc(reinterpret_cast<void**>(&c->arrive), static_cast<size_t>(d.layers) * 4) &&
              alloc(reinterpret_cast<void**>(&c->layer_allocs), static_cast<size_t>(d.layers) * 8);
    if (ok && c->paged)
        ok = alloc(reinterpret_cast<void**>(&c->slot), cells * 4) &&
             alloc(reinterpret_cast<void**>(&c->fq), static_cast<size_t>(d.layers) * d.batch * c->pcap * 4) &&
             alloc(reinterpret_cast<void**>(&c->fq_ht), static_cast<size_t>(d.layers) * d.batch * 8) &&
             alloc(reinterpret_cast<void**>(&c->act_slots), list_bytes) &&
             alloc(reinterpret_cast<void**>(&c->aux), acnt_bytes);
    if (ok) {
        void* h = nullptr;
        ok = cudaHostAlloc(&h, sizeof(skvd::DevStatus), cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess;
        if (ok) {
            c->status = static_cast<skvd::DevStatus*>(h);
            std::memset(c->status, 0, sizeof(skvd::DevStatus));
            void* dp = nullptr;
            ok = cudaHostGetDevicePointer(&dp, h, 0) == cudaSuccess;
            c->status_dev = static_cast<skvd::DevStatus*>(dp);
        }
        if (!ok) cudaGetLastError();
    }
    if (!ok) {
        const uint64_t want = kv_bytes + imp_bytes + wpart_bytes + cnt_bytes + tier_bytes + list_bytes + acnt_bytes;
        skv_cache_destroy(c);
        return fail(SKV_ERR_OOM, "skv_cache_create: cannot allocate %llu device bytes",
                    static_cast<unsigned long long>(want));
    }
    SKV_CUDA(cudaMemset(c->imp, 0, imp_bytes));
    SKV_CUDA(cudaMemset(c->tiers, 0xFF, tier_bytes));
    SKV_CUDA(cudaMemset(c->act_counts, 0, acnt_bytes));
    SKV_CUDA(cudaMemset(c->sparsity, 0, sp_bytes));
    SKV_CUDA(cudaMemset(c->counters, 0, ctr_bytes));
    SKV_CUDA(cudaMemset(c->tot, 0, sizeof(skvd::LedgerTotals)));
    SKV_CUDA(cudaMemset(c->arrive, 0, static_cast<size_t>(d.layers) * 4));
    SKV_CUDA(cudaMemset(c->layer_allocs, 0, static_cast<size_t>(d.layers) * 8));
    if (c->paged) {
        SKV_CUDA(cudaMemset(c->slot, 0xFF, cells * 4));
        SKV_CUDA(cudaMemset(c->aux, 0, acnt_bytes));
        // every ring starts full, slots in order: the prompt takes slot t for token t
        std::vector<int> ring(c->pcap);
        for (int i = 0; i < c->pcap; ++i) ring[i] = i;
        std::vector<unsigned> ht(static_cast<size_t>(d.layers) * d.batch * 2);
        for (size_t i = 0; i < ht.size(); i += 2) {
            ht[i] = 0;
            ht[i + 1] = static_cast<unsigned>(c->pcap);
        }
        for (size_t r = 0; r < static_cast<size_t>(d.layers) * d.batch; ++r)
            SKV_CUDA(cudaMemcpy(c->fq + r * c->pcap, ring.data(), ring.size() * 4, cudaMemcpyHostToDevice));
        SKV_CUDA(cudaMemcpy(c->fq_ht, ht.data(), ht.size() * 4, cudaMemcpyHostToDevice));
    }
    c->pend_n.assign(d.layers, -1);
    c->pend_r.assign(d.layers, 0.0);
    c->pend_topk.assign(d.layers, 0);
    c->ledger_j.assign(d.layers, -1);
    c->rec_x.assign(d.layers, nullptr);
    c->rec_wt.assign(d.layers, nullptr);
    c->ident.assign(static_cast<size_t>(d.layers) * d.batch, 0);
    c->decoded.assign(d.layers, 0);
    SKV_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, d.device));
    SKV_CUDA(cudaDeviceGetAttribute(&c->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, d.device));
    *out = c;
    return SKV_OK;
}

skv_status skv_cache_create(const skv_cache_desc* desc, skv_cache** out) { return cache_create_impl(desc, 0, out); }

skv_status skv_cache_create_paged(const skv_cache_desc* desc, uint64_t device_capacity, skv_cache** out) {
    SKV_REQUIRE(device_capacity > 0, "KvLedger: zero device capacity");
    return cache_create_impl(desc, device_capacity, out);
}

skv_status skv_cache_destroy(skv_cache* c) {
    if (c == nullptr) return SKV_OK;
    DeviceGuard guard(c->d.device);
    cudaFree(c->kv);
    cudaFree(c->meta);
    cudaFree(c->imp);
    cudaFree(c->wpart);
    cudaFree(c->idx);
    cudaFree(c->tiers);
    cudaFree(c->act_lists);
    cudaFree(c->act_counts);
    cudaFree(c->sparsity);
    cudaFree(c->counters);
    cudaFree(c->tot);
    cudaFree(c->arrive);
    cudaFree(c->layer_allocs);
    cudaFree(c->slot);
    cudaFree(c->fq);
    cudaFree(c->fq_ht);
    cudaFree(c->act_slots);
    cudaFree(c->aux);
    cudaFree(c->rec_c);
    if (c->status) cudaFreeHost(c->status);
    if (c->host_kv) cudaFreeHost(c->host_kv);
    for (uint8_t* w : c->rec_wt) cudaFree(w);
    cudaFree(c->rec_a);
    cudaFree(c->rec_map);
    cudaFree(c->rec_m);
    cudaFree(c->stage);
    cudaFree(c->xbuf);
    cudaFree(c->gkeys);
    cudaFree(c->gtok);
    cudaFree(c->gwts);
    cudaFree(c->frow);
    for (auto* v : {&c->ev_in, &c->ev_comp, &c->ev_out})
        for (cudaEvent_t e : *v) cudaEventDestroy(e);
    if (c->h2d) cudaStreamDestroy(c->h2d);
    if (c->sel_st) cudaStreamDestroy(c->sel_st);
    if (c->ev_sel_in) cudaEventDestroy(c->ev_sel_in);
    if (c->ev_sel_out) cudaEventDestroy(c->ev_sel_out);
    if (c->d2h) cudaStreamDestroy(c->d2h);
    cudaFree(c->pf_scratch);
    cudaFree(c->pf_sparsity);
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    delete c;
    return SKV_OK;
}

skv_status skv_cache_get_desc(const skv_cache* c, skv_cache_desc* desc, uint64_t* device_bytes) {
    SKV_REQUIRE(c != nullptr, "skv_cache_get_desc: null cache");
    if (desc) *desc = c->d;
    if (device_bytes) *device_bytes = c->device_bytes;
    return SKV_OK;
}

static skv_status check_block(const skv_cache* c, int layer, int b0, int nb, int t0, int nt) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    SKV_REQUIRE(b0 >= 0 && nb > 0 && b0 + nb <= c->d.batch, "batch range out of bounds");
    SKV_REQUIRE(t0 >= 0 && nt > 0 && t0 + nt <= c->d.capacity, "token range exceeds cache capacity");
    return SKV_OK;
}

skv_status skv_cache_write(skv_cache* c, int layer, int b0, int nb, int t0, int nt, const void* k,
                           const void* v, void* stream) {
    if (skv_status s = check_block(c, layer, b0, nb, t0, nt)) return s;
    SKV_REQUIRE(k != nullptr && v != nullptr, "append_token: null rows");
    if (skv_status s = check_status(c)) return s;
    DeviceGuard guard(c->d.device);
    const cudaStream_t st = as_stream(stream);
    const size_t lt = static_cast<size_t>(layer) * c->d.batch * c->d.capacity;
    // tokens this write stores for the first time (KvLedger::store_new)
    uint64_t fresh = 0;
    for (int b = b0; b < b0 + nb; ++b) {
        const int hw = c->ident[static_cast<size_t>(layer) * c->d.batch + b];
        fresh += static_cast<uint64_t>(std::max(0, t0 + nt - std::max(hw, t0)));
        if (c->paged)
            SKV_REQUIRE(!c->decoded[layer] && t0 <= hw,
                        "paged cache: skv_cache_write fills the prompt in order before the first decode step");
    }
    if (c->cap_bytes != ~0ull && fresh > 0) {
        // memsim.hpp:99-109: store_new checks the device capacity per token
        skvd::LedgerTotals tot{};
        SKV_CUDA(cudaMemcpyAsync(&tot, c->tot, sizeof tot, cudaMemcpyDeviceToHost, st));
        SKV_CUDA(cudaStreamSynchronize(st));
        const uint64_t e = c->tok_bytes;
        if ((tot.dev_tokens + fresh) * e > c->cap_bytes || (c->paged && t0 + nt > c->pcap)) {
            const uint64_t fit = c->cap_bytes / e;
            return fail(SKV_ERR_OOM, "simulated OOM: device tier needs %llu bytes, capacity %llu",
                        static_cast<unsigned long long>(e * (std::max<uint64_t>(tot.dev_tokens, fit) + 1)),
                        static_cast<unsigned long long>(c->cap_bytes));
        }
    }
    c->pend_n[layer] = -1;
    const skvd::CacheView cv = cache_view(c, layer);
    SKV_CUDA(launch_cache_write(c->d.kv_dtype, c->d.q_dtype, cv, c->imp + lt, c->tiers + lt, k, v, c->d.heads, b0, nb,
                                t0, nt, st));
    for (int b = b0; b < b0 + nb; ++b) {
        int& hw = c->ident[static_cast<size_t>(layer) * c->d.batch + b];
        hw = std::max(hw, t0 + nt);
    }
    return SKV_OK;
}

skv_status skv_cache_read(const skv_cache* c, int layer, int b0, int nb, int t0, int nt, float* out,
                          void* stream) {
    if (skv_status s = check_block(c, layer, b0, nb, t0, nt)) return s;
    SKV_REQUIRE(out != nullptr, "skv_cache_read: null output");
    DeviceGuard guard(c->d.device);
    const skvd::CacheView cv = cache_view(const_cast<skv_cache*>(c), layer);
    SKV_CUDA(launch_cache_read(c->d.kv_dtype, cv, out, c->d.heads, b0, nb, t0, nt, as_stream(stream)));
    return SKV_OK;
}

skv_status skv_importance_set(skv_cache* c, int layer, int b0, int nb, int len, const double* src,
                              void* stream) {
    if (skv_status s = check_block(c, layer, b0, nb, 0, len)) return s;
    DeviceGuard guard(c->d.device);
    double* dst = c->imp + (static_cast<size_t>(layer) * c->d.batch + b0) * c->d.capacity;
    c->pend_n[layer] = -1;
    SKV_CUDA(cudaMemcpy2DAsync(dst, c->d.capacity * 8, src, static_cast<size_t>(len) * 8,
                               static_cast<size_t>(len) * 8, nb, cudaMemcpyDefault, as_stream(stream)));
    return SKV_OK;
}

skv_status skv_importance_get(const skv_cache* c, int layer, int b0, int nb, int len, double* dst,
                              void* stream) {
    if (skv_status s = check_block(c, layer, b0, nb, 0, len)) return s;
    DeviceGuard guard(c->d.device);
    const double* src = c->imp + (static_cast<size_t>(layer) * c->d.batch + b0) * c->d.capacity;
    SKV_CUDA(cudaMemcpy2DAsync(dst, static_cast<size_t>(len) * 8, src, c->d.capacity * 8,
                               static_cast<size_t>(len) * 8, nb, cudaMemcpyDefault, as_stream(stream)));
    return SKV_OK;
}

}  // extern "C"

namespace {

// Pick heads-per-CTA. Bigger head groups mean bigger bulk copies (the
// producer's per-copy issue cost is the limiter, profiles/r1_v3_*) and fewer
// per-CTA select/softmax phases; layer-to-layer PDL overlap covers a grid
// smaller than one wave. So: the largest group that still gives at least one
// CTA per SM (config 3: HG 4, 160 CTAs -- isolated 0.44 -> 0.50 of the copy
// peak at an equal step, profiles/r2); for tiny batches the smallest group
// (most parallelism). SKV_HG overrides (tuning).
//
// Selections too long for any head group's shared-memory token list and
// weights (m beyond ~24 k) run with both in global scratch (gmem).
skv_status pick_attend(skv_cache* c, int m, const DecodeLaunch** dl_out, size_t* smem_out, bool* gmem_out) {
    static const int env_hg = [] {
        const char* s = std::getenv("SKV_HG");
        return s ? std::atoi(s) : 0;
    }();
    const int cands[4] = {8, 4, 2, 1};
    const DecodeLaunch* chosen = nullptr;
    size_t chosen_smem = 0;
    bool gmem = false;
    for (int pass = 0; pass < 2 && !chosen; ++pass) {
        gmem = pass == 1;
        const DecodeLaunch* smallest = nullptr;
        size_t smallest_smem = 0;
        for (int hg : cands) {
            if (c->d.heads % hg != 0) continue;
            if (env_hg && hg != env_hg) continue;
            const DecodeLaunch* dl = find_decode(c->d.kv_dtype, c->d.q_dtype, hg);
            if (!dl) continue;
            const size_t smem = dl->smem(m, gmem, c->paged);
            if (smem > static_cast<size_t>(c->max_smem)) continue;
            smallest = dl;
            smallest_smem = smem;
            const long long ctas = static_cast<long long>(c->d.batch) * (c->d.heads / hg);
            if (!chosen && ctas >= c->num_sms) {
                chosen = dl;
                chosen_smem = smem;
            }
        }
        if (!chosen) {
            chosen = smallest;
            chosen_smem = smallest_smem;
        }
    }
    *gmem_out = gmem;
    if (!chosen)
        return fail(SKV_ERR_UNSUPPORTED, "no attend kernel fits (heads %d, m %d, shared memory %d)", c->d.heads, m,
                    c->max_smem);
    // The attribute costs host time on every launch: it is set per function
    // (all caches share it) and only ever grows, which keeps concurrent
    // callers safe; the occupancy (reported, not used) is recomputed when this
    // cache's launch size changes.
    {
        static std::mutex mu;
        static std::map<const void*, size_t> set_smem;
        std::lock_guard<std::mutex> lock(mu);
        size_t& cur = set_smem[chosen->func];
        if (chosen_smem > cur) {
            SKV_CUDA(cudaFuncSetAttribute(chosen->func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(chosen_smem)));
            cur = chosen_smem;
        }
    }
    if (c->attr_func != chosen->func || c->attr_smem != chosen_smem) {
        cudaFuncAttributes fa{};
        SKV_CUDA(cudaFuncGetAttributes(&fa, chosen->func));
        int smem_sm = 0, reserved = 0;
        SKV_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->d.device));
        SKV_CUDA(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, c->d.device));
        const size_t per = chosen_smem + fa.sharedSizeBytes + static_cast<size_t>(reserved);
        int occ = static_cast<int>(static_cast<size_t>(smem_sm) / per);
        occ = std::min(occ, 2048 / skvd::kDecodeThreads);
        if (fa.numRegs > 0) occ = std::min(occ, 65536 / (fa.numRegs * skvd::kDecodeThreads));
        c->last_occ = occ;
        c->attr_func = chosen->func;
        c->attr_smem = chosen_smem;
    }
    *dl_out = chosen;
    *smem_out = chosen_smem;
    return SKV_OK;
}

// Algorithmic HBM bytes of one attend launch (the roofline numerator): q in,
// out out, new K/V rows in and stored, every other selected row of K and V
// gathered once.
uint64_t attend_algo_bytes(const skv_cache* c, int m, bool append) {
    const uint64_t H = c->d.heads, D = c->d.head_dim;
    const uint64_t eq = dtype_size(c->d.q_dtype), eo = out_size(c), ekv = dtype_size(c->d.kv_dtype);
    const uint64_t meta = c->d.kv_dtype == SKV_U8 ? 8 : 0;
    const uint64_t row = D * ekv + meta;  // one head row as stored
    uint64_t per = H * D * (eq + eo);
    uint64_t gathered = static_cast<uint64_t>(m);
    if (append) {
        per += 2 * H * D * eq + 2 * H * row;
        gathered -= 1;
    }
    per += 2 * gathered * H * row;
    return per * static_cast<uint64_t>(c->d.batch);
}

struct StepShape {
    int k, m, stride;
    bool dense;
};

// The selection shape of one step for the cache's variant
// (Engine::variant_selection, engine.hpp:531-569).
skv_status step_shape(const skv_cache* c, int n, double r, StepShape* s) {
    SKV_REQUIRE(n >= 1, "swa_attention: empty cache");
    SKV_REQUIRE(n <= c->d.capacity, "decode_step: context overflow");
    s->stride = 0;
    if (c->variant == SKV_VARIANT_DENSE) r = 1.0;  // swa_select(imp, n, 1.0)
    const size_t k = skv_swa_window_k(static_cast<size_t>(n), r);
    if (k == 0) return SKV_ERR_CONTRACT;
    const int keep = static_cast<int>(std::min<size_t>(2 * k, static_cast<size_t>(n)));
    if (c->variant == SKV_VARIANT_LOCAL) {  // local_attention_mask(n, keep)
        s->m = keep;
        s->k = keep;
        s->dense = false;
        return SKV_OK;
    }
    if (c->variant == SKV_VARIANT_STRIDED) {  // strided_attention_mask(n, stride)
        const int stride = c->stride > 0 ? c->stride : std::max(1, (n + keep - 1) / keep);
        const int phase = (n - 1) % stride;
        s->stride = stride;
        s->m = (n - 1 - phase) / stride + 1;
        s->k = 1;
        s->dense = false;
        return SKV_OK;
    }
    s->k = static_cast<int>(k);
    s->dense = n < 2 || 2 * static_cast<int>(k) >= n;
    s->m = s->dense ? n : 2 * s->k;
    return SKV_OK;
}

int* layer_idx(const skv_cache* c, int layer) {
    return c->idx + static_cast<size_t>(layer) * c->d.batch * c->d.capacity;
}

// The per-sequence select kernel for one layer: optionally fold the attend
// kernel's weight partials into the importance, optionally select for
// (n_next, r_next) into the layer's index buffer (recorded as pending).
// SelectParams for one layer: fold the last attend's partials (apply != 0)
// and/or select for (n_next, r_next) (n_next <= 0: no selection).
skv_status make_select_params(skv_cache* c, int layer, int apply, const int* tok_prev, long long tok_prev_ld,
                              int m_prev, int G, int cur_tok, int n_next, double r_next, int sp_n,
                              skvd::SelectParams* out) {
    skvd::SelectParams p{};
    p.sp_n = apply ? sp_n : 0;
    p.sparsity = c->sparsity + static_cast<size_t>(layer) * c->d.batch;
    p.imp = c->imp + static_cast<size_t>(layer) * c->d.batch * c->d.capacity;
    p.imp_ld = c->d.capacity;
    p.wpart = c->wpart + static_cast<size_t>(layer) * c->d.batch * c->d.heads * c->d.capacity;
    p.G = G;
    p.m_prev = m_prev;
    p.tok_prev = tok_prev;
    p.tok_prev_ld = tok_prev_ld;
    p.apply = apply;
    p.cur_tok = cur_tok;
    p.idx = layer_idx(c, layer);
    p.idx_ld = c->d.capacity;
    p.pdl_wait = 1;
    if (n_next > 0 && n_next <= c->d.capacity) {
        StepShape s;
        if (skv_status e = step_shape(c, n_next, r_next, &s)) return e;
        if (!s.dense && c->variant != SKV_VARIANT_LOCAL && c->variant != SKV_VARIANT_STRIDED &&
            static_cast<size_t>(n_next - s.k) * 8 + 8192 > static_cast<size_t>(c->max_smem)) {
            // long context: the candidates' keys go to global scratch shaped like the importance
            if (!c->gkeys) {
                const size_t bytes = static_cast<size_t>(c->d.layers) * c->d.batch * c->d.capacity * 8;
                if (cudaMalloc(reinterpret_cast<void**>(&c->gkeys), bytes) != cudaSuccess) {
                    cudaGetLastError();
                    return fail(SKV_ERR_OOM, "swa_select: cannot allocate %zu bytes of key scratch", bytes);
                }
                c->device_bytes += bytes;
            }
            p.gkeys = c->gkeys + static_cast<size_t>(layer) * c->d.batch * c->d.capacity;
        }
        p.select = 1;
        p.n = n_next;
        p.k = s.k;
        p.m = s.m;
        p.dense = s.dense ? 1 : 0;
        p.variant = c->variant == SKV_VARIANT_DENSE ? SKV_VARIANT_SWA : c->variant;
        p.stride = s.stride;
    }
    *out = p;
    return SKV_OK;
}

// Key bytes the selection needs in shared memory (0 for index generators).
size_t select_key_bytes(const skvd::SelectParams& p) {
    if (!p.select || p.dense || p.variant == 2 || p.variant == 3) return 0;
    return static_cast<size_t>(p.n - p.k) * 8;
}

void note_pending(skv_cache* c, int layer, const skvd::SelectParams& p, double r_next) {
    if (p.select) {
        c->pend_n[layer] = p.n;
        c->pend_r[layer] = r_next;
        c->pend_topk[layer] = !p.dense && p.variant == 1;
    } else {
        c->pend_n[layer] = -1;
    }
}

// A fold of the pending selection of layer (tok = its index buffer, made by
// an SWA top-k at n = cur_tok + 1 with ratio r_next, nothing else written to
// the importance since: any other writer drops pend_n) lets the select kernel
// derive the next selection incrementally (incremental_select). Head shards
// sum the step rows across GPUs first and keep the full top-k.
bool incr_ok(const skv_cache* c, int layer, const int* tok, int cur_tok, double r_next) {
    static const bool off = std::getenv("SKV_SELECT_FULL") != nullptr;  // A/B: always the full top-k
    return !off && !c->reduce && tok == layer_idx(c, layer) && c->pend_topk[layer] &&
           c->pend_n[layer] == cur_tok + 1 && c->pend_r[layer] == r_next;
}

// The standalone per-sequence select kernel (skv_select.cuh).
skv_status launch_select_c(skv_cache* c, int layer, int apply, const int* tok_prev, long long tok_prev_ld,
                           int m_prev, int G, int cur_tok, int n_next, double r_next, bool pdl, cudaStream_t st,
                           int sp_n = 0, double* wsum_out = nullptr, const double* wsum = nullptr) {
    skvd::SelectParams p;
    const bool incr = apply == 1 && incr_ok(c, layer, tok_prev, cur_tok, r_next);
    c->pend_n[layer] = -1;
    if (skv_status e = make_select_params(c, layer, apply, tok_prev, tok_prev_ld, m_prev, G, cur_tok, n_next, r_next,
                                          sp_n, &p))
        return e;
    p.incr = incr ? 1 : 0;
    p.wsum_out = wsum_out;
    p.wsum = wsum;
    if (!p.apply && !p.select) return SKV_OK;
    SKV_CUDA(launch_select(p, c->d.batch, pdl, st));
    note_pending(c, layer, p, r_next);
    return SKV_OK;
}

// What an attend launch folds in its tail (apply 0: nothing).
struct FoldSpec {
    int apply = 0;    // 1 add (cur_tok assigned), 2 assign all
    int cur_tok = -1;
    int sp_n = 0;     // sparsity row length (0: skip)
    int n_next = 0;   // select for the next step (0: none)
    double r_next = 0.0;
};

skv_status launch_attend_c(skv_cache* c, int layer, int n, int m, const int* tok, long long tok_ld, bool append,
                           const void* q, const void* k_new, const void* v_new, void* out, int32_t* idx_out,
                           float* w_out, bool pdl, cudaStream_t st, int* G_out, const FoldSpec& fold = FoldSpec{}) {
    const DecodeLaunch* dl = nullptr;
    size_t smem = 0;
    bool gmem = false;
    if (skv_status s = pick_attend(c, m, &dl, &smem, &gmem)) return s;
    if (gmem && !c->gtok) {  // long selection: token list + weights in global scratch
        const size_t cells = static_cast<size_t>(c->d.batch) * c->d.heads * c->d.capacity;
        if (cudaMalloc(reinterpret_cast<void**>(&c->gtok), cells * 4) != cudaSuccess ||
            cudaMalloc(reinterpret_cast<void**>(&c->gwts), cells * 4) != cudaSuccess) {
            cudaGetLastError();
            return fail(SKV_ERR_OOM, "attend: cannot allocate %zu bytes of long-selection scratch", 2 * cells * 4);
        }
        c->device_bytes += 2 * cells * 4;
    }
    const int G = c->d.heads / dl->hg;
    skvd::SelectParams sel{};
    bool fused = fold.apply != 0;
    if (fused) {
        if (skv_status e = make_select_params(c, layer, fold.apply, nullptr, 0, m, G, fold.cur_tok, fold.n_next,
                                              fold.r_next, fold.sp_n, &sel))
            return e;
        sel.incr = fold.apply == 1 && incr_ok(c, layer, tok, fold.cur_tok, fold.r_next) ? 1 : 0;
        // The tail's selection runs on one CTA per sequence while it holds its
        // attend slot: worth it for short candidate lists (configs 2/3: step
        // 0.98->1.02, 0.88->1.01), not for n-k in the thousands (config 4:
        // 0.88->0.79), which keep the separate select kernel.
        if (select_key_bytes(sel) > std::min<size_t>(dl->ring_bytes, 2048 * 8)) fused = false;
        if (c->reduce) fused = false;  // the step row is summed across head shards first
        // Whole-step decode keeps the attend kernel free of the tail: the
        // layers' selects run as one batched launch after the attends (or, when
        // profiling, as separate launches). Per-layer calls keep the tail.
        // Measured at config 2 / 3: the step is equal within 1% (0.985 vs
        // 0.994, 1.005 vs 0.997), the attend launch alone 0.69 vs 0.52 and
        // 0.41 vs 0.31 of the copy peak. SKV_STEP_TAIL=1 restores the tail.
        static const bool step_tail = std::getenv("SKV_STEP_TAIL") != nullptr;
        if (c->in_step && !step_tail) fused = false;
    }
    const size_t lt = static_cast<size_t>(layer) * c->d.batch * c->d.capacity;
    skvd::AttendParams p{};
    p.kv = c->kv + layer * c->layer_bytes;
    p.kv_w = c->kv + layer * c->layer_bytes;
    p.kv_ncap = c->pcap;
    p.slots = c->paged ? c->slot + lt : nullptr;
    p.tiers = c->has_plan ? c->tiers + lt : nullptr;  // residency check (engine.hpp:625-628)
    p.status = c->status_dev;
    p.layer = layer;
    p.q = q;
    p.k_new = k_new;
    p.v_new = v_new;
    p.out = out;
    p.tok = tok;
    p.tok_ld = tok_ld;
    p.idx_out = idx_out;
    p.w_out = w_out;
    p.wpart = c->wpart + static_cast<size_t>(layer) * c->d.batch * c->d.heads * c->d.capacity;
    p.B = c->d.batch;
    p.H = c->d.heads;
    p.Ncap = c->d.capacity;
    p.n = n;
    p.m = m;
    p.append = append ? 1 : 0;
    p.out_f32 = c->d.out_f32 ? 1 : 0;
    p.pdl_wait = 0;  // inputs are complete before the first (non-PDL) launch of a call
    p.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c->d.head_dim)));
    if (gmem) {
        p.gtok = c->gtok;
        p.gwts = c->gwts;
    }
    if (fused) {
        p.fold = 1;
        p.sel = sel;
        p.counters = c->counters + static_cast<size_t>(layer) * c->d.batch;
    }
    const int grid_g = G;
    *G_out = grid_g;
    c->last_hg = dl->hg;
    c->last_grid = grid_g * c->d.batch;
    c->last_smem = smem;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->prof) {
        auto take = [&]() {
            cudaEvent_t e;
            if (!c->ev_pool.empty()) {
                e = c->ev_pool.back();
                c->ev_pool.pop_back();
            } else {
                cudaEventCreate(&e);
            }
            return e;
        };
        e0 = take();
        e1 = take();
        SKV_CUDA(cudaEventRecord(e0, st));
        pdl = false;
    }
    // Long selections share one [B][G][Ncap] token-list / weight scratch
    // across layers: a PDL-overlapped predecessor could still be using it,
    // so such launches wait for the previous grid to finish.
    if (gmem) pdl = false;
    // A per-layer step whose attend carries the fold + select tail (config 1:
    // the whole step is this one launch), and the first attend of a whole
    // step, launch with PDL and wait at entry: resident while the previous
    // step drains (its select triggers at entry), hiding the launch gap. The
    // chained attends behind it launch only once it has passed its wait.
    // Not with a plan: the ledger kernel of Phase I steps does not wait on
    // its predecessor, so waiting on it would not order after the attend.
    static const bool entry_pdl = std::getenv("SKV_NO_ENTRY_PDL") == nullptr;
    if (!pdl && (fused || c->in_step) && entry_pdl && !c->has_plan && !c->prof) {
        pdl = true;
        p.pdl_wait = 2;
    }
    SKV_CUDA(launch_attend(*dl, p, grid_g, smem, pdl, st));
    c->algo_bytes += attend_algo_bytes(c, m, append);
    c->attend_launches += 1;
    if (c->prof) {
        SKV_CUDA(cudaEventRecord(e1, st));
        c->ev.push_back(e0);
        c->ev.push_back(e1);
    }
    if (fold.apply) {
        if (fused) {
            note_pending(c, layer, sel, fold.r_next);
        } else if (c->reduce && !c->defer_select) {
            // head shards: this shard's head-summed row -> all-reduce across
            // the shards (the caller's collective, ordered on st) -> fold it
            // and select; every shard then holds the same importance and
            // makes the same selection.
            if (skv_status e = launch_select_c(c, layer, fold.apply, tok, tok_ld, m, G, fold.cur_tok, 0, 0.0,
                                               !c->prof, st, 0, c->xbuf, nullptr))
                return e;
            if (skv_status e = c->reduce(c->xbuf, static_cast<size_t>(c->d.batch) * m, st, c->reduce_user))
                return fail(e, "head-shard reduce failed (%d)", static_cast<int>(e));
            if (skv_status e = launch_select_c(c, layer, fold.apply, tok, tok_ld, m, G, fold.cur_tok, fold.n_next,
                                               fold.r_next, false, st, fold.sp_n, nullptr, c->xbuf))
                return e;
        } else if (c->defer_select) {
            skvd::SelectParams sp;
            if (skv_status e = make_select_params(c, layer, fold.apply, tok, tok_ld, m, G, fold.cur_tok, fold.n_next,
                                                  fold.r_next, fold.sp_n, &sp))
                return e;
            sp.incr = fold.apply == 1 && incr_ok(c, layer, tok, fold.cur_tok, fold.r_next) ? 1 : 0;
            c->pend_n[layer] = -1;
            c->deferred.emplace_back(layer, sp);
            note_pending(c, layer, sp, fold.r_next);
        } else {  // fold + select in the separate kernel instead
            const int* tp = tok;
            if (skv_status e = launch_select_c(c, layer, fold.apply, tp, tok_ld, m, G, fold.cur_tok, fold.n_next,
                                               fold.r_next, !c->prof, st, fold.sp_n))
                return e;
        }
    }
    return SKV_OK;
}

// phase_of_step (scheduler.hpp:52-60)
int phase_of(const skv_plan& pl, long long j) {
    if (j < pl.p1) return 1;
    if (j < pl.p2 || !pl.recompute_enabled) return 2;
    return 3;
}

// step_actions + apply_actions for step j of one layer on the device ledger,
// with the given (ascending) selection.
skv_status launch_ledger_c(skv_cache* c, int layer, long long j, const int* sel, long long sel_ld, int m, int k,
                           bool apply, bool store_current, bool pdl, cudaStream_t st) {
    const skv_plan& pl = c->plan;
    skvd::LedgerParams p{};
    const size_t lt = static_cast<size_t>(layer) * c->d.batch * c->d.capacity;
    p.tiers = c->tiers + lt;
    p.tier_ld = c->d.capacity;
    p.sel = sel;
    p.sel_ld = sel_ld;
    p.m = m;
    p.k = k;
    p.existing = static_cast<int>(pl.input_len + j);
    p.phase = phase_of(pl, j);
    p.target = static_cast<long long>(std::ceil(pl.alpha * static_cast<double>(p.existing)));
    p.beta = pl.beta;
    p.lists = c->act_lists + lt * 4;
    p.list_ld = c->d.capacity;
    p.counts = c->act_counts + static_cast<size_t>(layer) * c->d.batch * 4;
    p.apply = apply ? 1 : 0;
    p.store_current = store_current ? 1 : 0;
    if (c->paged) {
        p.slots.slot = c->slot + lt;
        p.slots.slot_ld = c->d.capacity;
        p.slots.fq = c->fq + static_cast<size_t>(layer) * c->d.batch * c->pcap;
        p.slots.fq_ht = c->fq_ht + static_cast<size_t>(layer) * c->d.batch * 2;
        p.slots.pcap = c->pcap;
        p.act_slots = c->act_slots + lt * 4;
        p.aux = c->aux + static_cast<size_t>(layer) * c->d.batch * 4;
    }
    if (apply) {  // KvLedger byte accounting + the capacity check (memsim.hpp:193-200)
        p.tot = c->tot;
        p.arrive = c->arrive + layer;
        p.layer_allocs = c->layer_allocs + layer;
    }
    p.cap_bytes = c->cap_bytes;
    p.tok_bytes = c->tok_bytes;
    p.cap_tokens = c->cap_bytes == ~0ull ? ~0ull : c->cap_bytes / c->tok_bytes;  // unbounded: never fails
    p.layer = layer;
    p.step = j;
    p.status = c->status_dev;
    SKV_REQUIRE(p.existing < c->d.capacity, "step_actions: step beyond the cache capacity");
    SKV_CUDA(launch_ledger(p, c->d.batch, pdl, st));
    if (apply) c->ledger_j[layer] = j;
    return SKV_OK;
}

// apply_actions data movement for one layer (engine.hpp:686-716): offload
// then reload over the host tier, after the ledger kernel made the lists.
// m_sel: the step's selection size, which bounds every list's length per
// sequence (the recompute GEMM's row count is at most B * m_sel).
skv_status launch_movement(skv_cache* c, int layer, bool pdl, cudaStream_t st, int m_sel = 0) {
    if (!c->host_kv) return SKV_OK;
    skvd::MoveParams mp{};
    const size_t lt = static_cast<size_t>(layer) * c->d.batch;
    mp.dev = c->kv + layer * c->layer_bytes;
    mp.host = c->host_kv + layer * c->host_layer_bytes;
    mp.lists = c->act_lists + lt * 4 * c->d.capacity;
    mp.counts = c->act_counts + lt * 4;
    mp.list_ld = c->d.capacity;
    mp.tok_bytes = static_cast<long long>(c->tok_bytes);
    mp.seq_bytes = static_cast<long long>(c->tok_bytes) * c->d.capacity;
    mp.dev_seq_bytes = static_cast<long long>(c->tok_bytes) * c->pcap;
    mp.poison = c->poison ? 1 : 0;
    mp.which = -1;  // offload and reload in one launch: both PCIe directions at once
    if (c->paged) {
        mp.act_slots = c->act_slots + lt * 4 * c->d.capacity;
        mp.aux = c->aux + lt * 4;
    }
    SKV_CUDA(launch_move(mp, c->d.batch, c->d.capacity, pdl, st));
    if (c->paged) {  // reloads into slots this step's offload frees: after those copies
        mp.which = 2;
        mp.second = 1;
        SKV_CUDA(launch_move(mp, c->d.batch, c->d.capacity, pdl, st));
    }
    if (c->rec_x[layer]) {
        // recompute_kv for this step's list: gather the retained rows, one
        // tcgen05 GEMM against [Wk | Wv]^T, K/V written straight into the rows
        // (INT8: through fp32 rows and the fake-quant, engine.hpp:729-730)
        const long long h = static_cast<long long>(c->d.heads) * c->d.head_dim;
        const long long xrow = h * static_cast<long long>(dtype_size(c->d.q_dtype));
        SKV_CUDA(launch_recompute_gather(c->rec_x[layer], xrow * c->d.capacity, xrow, mp.lists, mp.counts,
                                         c->d.capacity, c->rec_a, c->rec_map, c->rec_m, c->d.batch, st,
                                         c->paged ? mp.act_slots : nullptr));
        const long long per = m_sel > 0 ? std::min(m_sel, c->d.capacity) : c->d.capacity;
        const int m_cap = static_cast<int>((static_cast<long long>(c->d.batch) * per + 127) / 128 * 128);
        if (c->d.kv_dtype == SKV_U8) {
            SKV_CUDA(launch_gemm_tn(c->rec_a, c->rec_wt[layer], c->rec_c, c->rec_m, m_cap, static_cast<int>(2 * h),
                                    static_cast<int>(h), c->d.q_dtype == SKV_BF16, st, nullptr));
            SKV_CUDA(launch_quant_scatter(c->d.q_dtype, c->rec_c, c->rec_m, m_cap, c->rec_map, mp.dev, c->d.heads,
                                          c->pcap, st));
        } else {
            skvd::KvScatter sc{};
            sc.kv = mp.dev;
            sc.rowmap = c->rec_map;
            sc.H = c->d.heads;
            sc.D = c->d.head_dim;
            sc.Ncap = c->pcap;
            sc.row_bytes = static_cast<int>(c->row_bytes);
            SKV_CUDA(launch_gemm_tn(c->rec_a, c->rec_wt[layer], nullptr, c->rec_m, m_cap, static_cast<int>(2 * h),
                                    static_cast<int>(h), c->d.q_dtype == SKV_BF16, st, &sc));
        }
    }
    return SKV_OK;
}

// The part of a decode step before its attend (engine.hpp:601-606):
// variant_selection when no selection for (n, r) is pending, and with a plan
// that step's step_actions + apply_actions (normally done right after the
// previous step). *fresh: a selection was made here.
skv_status prepare_step(skv_cache* c, int layer, int n, double r, const StepShape& s, cudaStream_t st, bool* fresh) {
    *fresh = false;
    if (c->pend_n[layer] == n && c->pend_r[layer] == r) return SKV_OK;
    if (skv_status e = launch_select_c(c, layer, 0, nullptr, 0, 0, 0, -1, n, r, false, st)) return e;
    *fresh = true;
    if (c->has_plan) {
        const long long j = static_cast<long long>(n) - 1 - c->plan.input_len;
        if (j >= 0 && j < c->plan.output_len && c->ledger_j[layer] != j) {
            if (skv_status e = launch_ledger_c(c, layer, j, layer_idx(c, layer), c->d.capacity, s.m, s.k, true, true,
                                               false, st))
                return e;
            if (phase_of(c->plan, j) > 1)  // Phase I lists are empty: nothing to move
                if (skv_status e = launch_movement(c, layer, true, st, s.m)) return e;
        }
    }
    return SKV_OK;
}

// One layer of one decode step: [select if no matching pending selection] ->
// attend (append + gather + softmax + PV) -> select kernel (fold weights into
// the importance, select for n+1 with the same ratio).
skv_status decode_layer_impl(skv_cache* c, int layer, int n, double r, const void* q, const void* k_new,
                             const void* v_new, void* out, int32_t* idx_out, float* w_out, bool chained,
                             cudaStream_t st) {
    StepShape s;
    if (skv_status e = step_shape(c, n, r, &s)) return e;
    if (c->paged && !c->has_plan)
        return fail(SKV_ERR_CONTRACT, "paged cache: attach a plan (skv_cache_set_plan) before decoding");
    c->decoded[layer] = 1;
    bool fresh = false;
    if (skv_status e = prepare_step(c, layer, n, r, s, st, &fresh)) return e;
    int G = 0;
    FoldSpec fold;
    fold.apply = 1;
    fold.cur_tok = n - 1;
    fold.sp_n = n;
    fold.n_next = n + 1;
    fold.r_next = r;
    if (skv_status e = launch_attend_c(c, layer, n, s.m, layer_idx(c, layer), c->d.capacity, true, q, k_new, v_new,
                                       out, idx_out, w_out, chained && !fresh, st, &G, fold))
        return e;
    if (c->has_plan && c->pend_n[layer] == n + 1) {
        // the next step's KV residency actions (scheduler.hpp:320-381) on the
        // device ledger, from the selection just made, then its store_new
        const long long j_next = static_cast<long long>(n) - c->plan.input_len;
        if (j_next >= 0 && j_next < c->plan.output_len) {
            StepShape sn;
            if (skv_status e = step_shape(c, n + 1, r, &sn)) return e;
            if (skv_status e = launch_ledger_c(c, layer, j_next, layer_idx(c, layer), c->d.capacity, sn.m, sn.k,
                                               true, true, !c->prof, st))
                return e;
            if (phase_of(c->plan, j_next) == 1) return SKV_OK;  // Phase I lists are empty: nothing to move
            return launch_movement(c, layer, !c->prof, st, sn.m);
        }
    }
    return SKV_OK;
}

}  // namespace

extern "C" {

skv_status skv_prefill_seed(skv_cache* c, int layer, int n, const void* q_last, void* out, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    SKV_REQUIRE(n >= 1 && n <= c->d.capacity, "prefill: prompt length out of range");
    SKV_REQUIRE(q_last != nullptr && out != nullptr, "prefill: null argument");
    DeviceGuard guard(c->d.device);
    const cudaStream_t st = as_stream(stream);
    int G = 0;
    FoldSpec fold;
    fold.apply = 2;  // engine.hpp:508-512: the seed assigns
    return launch_attend_c(c, layer, n, n, nullptr, 0, false, q_last, nullptr, nullptr, out, nullptr, nullptr, false,
                           st, &G, fold);
}

// Engine::prefill's attention for one layer (engine.hpp:485-529) on tensor
// cores: dense causal attention of the s prompt queries over the s cached
// tokens, importance seeded with the head-summed last row, prefill sparsity
// recorded. See skv_prefill.cu.
skv_status skv_prefill_layer(skv_cache* c, int layer, int s, const void* q, void* out, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    SKV_REQUIRE(s >= 1 && s <= c->d.capacity, "prefill: prompt length out of range");
    SKV_REQUIRE(q != nullptr && out != nullptr, "prefill: null argument");
    // INT8 caches (fp16 queries): the layer is dequantised to fp16 for the
    // tensor cores; the seed row (and the last query's output) is then redone
    // by the decode kernel on the exact fp32 dequantisation.
    const bool int8 = c->d.kv_dtype == SKV_U8 && c->d.q_dtype == SKV_F16;
    if (!int8 && !(c->d.kv_dtype == c->d.q_dtype && (c->d.q_dtype == SKV_F16 || c->d.q_dtype == SKV_BF16)))
        return fail(SKV_ERR_UNSUPPORTED, "prefill: tensor-core prefill needs an fp16/bf16 cache or INT8 with fp16 q");
    DeviceGuard guard(c->d.device);
    const cudaStream_t st = as_stream(stream);
    const int B = c->d.batch, H = c->d.heads;
    const size_t base_scratch = (prefill_scratch_bytes(B, H, s) + 255) / 256 * 256;
    const size_t deq_bytes = int8 ? static_cast<size_t>(B) * s * 2 * H * c->d.head_dim * 2 : 0;
    const size_t want = base_scratch + deq_bytes;
    if (c->pf_bytes < want) {
        SKV_CUDA(cudaStreamSynchronize(st));
        cudaFree(c->pf_scratch);
        c->pf_scratch = nullptr;
        c->pf_bytes = 0;
        if (cudaMalloc(reinterpret_cast<void**>(&c->pf_scratch), want) != cudaSuccess) {
            cudaGetLastError();
            return fail(SKV_ERR_OOM, "prefill: cannot allocate %zu scratch bytes", want);
        }
        c->pf_bytes = want;
    }
    if (c->pf_sparsity == nullptr) {
        const size_t bytes = static_cast<size_t>(c->d.layers) * B * 8;
        if (cudaMalloc(reinterpret_cast<void**>(&c->pf_sparsity), bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(SKV_ERR_OOM, "prefill: cannot allocate sparsity");
        }
        SKV_CUDA(cudaMemset(c->pf_sparsity, 0, bytes));
    }
    const size_t lay = static_cast<size_t>(layer);
    double* imp = c->imp + lay * B * c->d.capacity;
    double* psp = c->pf_sparsity + lay * B;
    const void* kv = c->kv + lay * c->layer_bytes;
    int kv_ncap = c->pcap;
    if (c->paged)  // the TMA maps read the prompt rows in place: token t must sit in slot t
        for (int b = 0; b < B; ++b)
            SKV_REQUIRE(!c->decoded[layer] && c->ident[lay * B + b] >= s,
                        "paged cache: the tensor-core prefill needs the prompt written in order first");
    if (int8) {
        uint8_t* deq = c->pf_scratch + base_scratch;
        SKV_CUDA(launch_dequant_layer_f16(c->kv + lay * c->layer_bytes, deq, H, c->pcap, B, s, st));
        kv = deq;
        kv_ncap = s;
    }
    if (c->reduce) {
        // head shards: seed rows and the sparsity share (local sum / all heads)
        // into xbuf, summed across the shards, then into the importance
        double* xs = c->xbuf + static_cast<size_t>(B) * c->d.capacity;
        SKV_CUDA(launch_prefill(c->d.q_dtype == SKV_BF16, c->d.out_f32 != 0, kv, q, out, c->xbuf, c->d.capacity, xs,
                                B, H, c->d.head_dim, kv_ncap, s, c->pf_scratch, st, c->total_heads));
        if (skv_status e = c->reduce(c->xbuf, static_cast<size_t>(B) * (c->d.capacity + 1), st, c->reduce_user))
            return fail(e, "head-shard reduce failed (%d)", static_cast<int>(e));
        SKV_CUDA(cudaMemcpy2DAsync(imp, c->d.capacity * 8, c->xbuf, c->d.capacity * 8, static_cast<size_t>(s) * 8,
                                   B, cudaMemcpyDeviceToDevice, st));
        SKV_CUDA(cudaMemcpyAsync(psp, xs, static_cast<size_t>(B) * 8, cudaMemcpyDeviceToDevice, st));
    } else {
        SKV_CUDA(launch_prefill(c->d.q_dtype == SKV_BF16, c->d.out_f32 != 0, kv, q, out, imp, c->d.capacity, psp, B,
                                H, c->d.head_dim, kv_ncap, s, c->pf_scratch, st));
    }
    if (int8) {
        // exact seed (engine.hpp:508-512) and last-row output from the fp32
        // dequantisation: the decode kernel's dense attend of query s-1
        const size_t row = static_cast<size_t>(H) * c->d.head_dim * 2;  // fp16 q row [H][D]
        const size_t orow = static_cast<size_t>(H) * c->d.head_dim * out_size(c);
        uint8_t* qlast = c->pf_scratch + base_scratch;  // the fp16 copy is no longer needed
        uint8_t* olast = qlast + static_cast<size_t>(B) * row;
        SKV_CUDA(cudaMemcpy2DAsync(qlast, row, static_cast<const uint8_t*>(q) + (s - 1) * row, s * row, row, B,
                                   cudaMemcpyDeviceToDevice, st));
        int G = 0;
        FoldSpec fold;
        fold.apply = 2;
        if (skv_status e = launch_attend_c(c, layer, s, s, nullptr, 0, false, qlast, nullptr, nullptr, olast, nullptr,
                                           nullptr, false, st, &G, fold))
            return e;
        SKV_CUDA(cudaMemcpy2DAsync(static_cast<uint8_t*>(out) + (s - 1) * orow, s * orow, olast, orow, orow, B,
                                   cudaMemcpyDeviceToDevice, st));
    }
    c->pend_n[layer] = -1;  // importance changed: any pending selection is stale
    return SKV_OK;
}

skv_status skv_prefill_sparsity_get(const skv_cache* c, int layer, double* dst, void* stream) {
    SKV_REQUIRE(c != nullptr && dst != nullptr, "null argument");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    SKV_REQUIRE(c->pf_sparsity != nullptr, "prefill sparsity: no tensor-core prefill has run");
    DeviceGuard guard(c->d.device);
    const cudaStream_t st = as_stream(stream);
    SKV_CUDA(cudaMemcpyAsync(dst, c->pf_sparsity + static_cast<size_t>(layer) * c->d.batch,
                             static_cast<size_t>(c->d.batch) * 8, cudaMemcpyDefault, st));
    SKV_CUDA(cudaStreamSynchronize(st));
    return SKV_OK;
}

skv_status skv_decode_prepare(skv_cache* c, int layer, int n, double r, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    if (skv_status e = check_status(c)) return e;
    StepShape s;
    if (skv_status e = step_shape(c, n, r, &s)) return e;
    DeviceGuard guard(c->d.device);
    bool fresh = false;
    return prepare_step(c, layer, n, r, s, as_stream(stream), &fresh);
}

skv_status skv_swa_decode_layer(skv_cache* c, int layer, int n, double r, const void* q, const void* k_new,
                                const void* v_new, void* out, int32_t* idx_out, float* w_out, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    SKV_REQUIRE(q && k_new && v_new && out, "decode_step: null argument");
    if (skv_status e = check_status(c)) return e;
    DeviceGuard guard(c->d.device);
    return decode_layer_impl(c, layer, n, r, q, k_new, v_new, out, idx_out, w_out, false, as_stream(stream));
}

// Layers [l0, l1) of one decode step; layer l > l0 launches with programmatic
// dependent launch: its inputs were complete before the range's first launch,
// so it can stream while the previous layer's kernels drain.
// One batched select launch over the deferred layers (consecutive, same
// shape) on stream st; clears the deferred list.
static skv_status launch_deferred(skv_cache* c, cudaStream_t st) {
    if (c->deferred.empty()) return SKV_OK;
    skvd::SelectParams p = c->deferred.front().second;
    const int first = c->deferred.front().first;
    const int cnt = static_cast<int>(c->deferred.size());
    for (int i = 0; i < cnt; ++i) {
        SKV_REQUIRE(c->deferred[i].first == first + i && c->deferred[i].second.m_prev == p.m_prev &&
                        c->deferred[i].second.G == p.G,
                    "decode_step: deferred selects must be consecutive layers of one shape");
        p.incr &= c->deferred[i].second.incr;  // one flag for the whole batched launch
    }
    p.ls_imp = static_cast<long long>(c->d.batch) * c->d.capacity;
    p.ls_wpart = static_cast<long long>(c->d.batch) * c->d.heads * c->d.capacity;
    p.ls_idx = static_cast<long long>(c->d.batch) * c->d.capacity;
    p.ls_sp = c->d.batch;
    p.pdl_wait = 0;
    const std::vector<std::pair<int, skvd::SelectParams>> pending = std::move(c->deferred);
    c->deferred.clear();
    cudaError_t le = cudaSuccess;
    if (c->reduce) {
        // head shards: every layer's head-summed step row of this shard in one
        // pass, ONE all-reduce of the whole step's rows across the shards (the
        // caller's collective on st), then every layer's fold + selection
        // from the summed rows -- off the per-layer critical path
        skvd::SelectParams pp = p;
        pp.wsum_out = c->xbuf;
        pp.ls_wsum = static_cast<long long>(c->d.batch) * p.m_prev;
        pp.select = 0;
        le = launch_select(pp, c->d.batch, false, st, cnt);
        if (le == cudaSuccess) {
            const skv_status e =
                c->reduce(c->xbuf, static_cast<size_t>(cnt) * c->d.batch * p.m_prev, st, c->reduce_user);
            if (e != SKV_OK) {
                for (const auto& d : pending) c->pend_n[d.first] = -1;
                return fail(e, "head-shard reduce failed (%d)", static_cast<int>(e));
            }
            p.wsum = c->xbuf;
            p.ls_wsum = pp.ls_wsum;
            le = launch_select(p, c->d.batch, false, st, cnt);
        }
    } else {
        le = launch_select(p, c->d.batch, false, st, cnt);
    }
    if (le != cudaSuccess) {
        for (const auto& d : pending) c->pend_n[d.first] = -1;
        return fail(SKV_ERR_CUDA, "decode_step: batched select launch: %s", cudaGetErrorString(le));
    }
    return SKV_OK;
}

// Layers [l0, l1) of one decode step; layer l > l0 launches with programmatic
// dependent launch: its inputs were complete before the range's first launch,
// so it can stream while the previous layer's kernels drain. The selects of
// a step only feed the next step: the first `split` layers' batched select
// runs on a side stream behind an event, overlapping the remaining layers'
// attends (HBM-bound) with its fold + top-k (latency-bound), and the rest run
// batched after the last attend; the caller's stream then joins the side
// stream. SKV_SELECT_SPLIT=0 keeps one batched select after all attends.
static skv_status decode_layers(skv_cache* c, int l0, int l1, int n, double r, const void* q, const void* k_new,
                                const void* v_new, void* out, cudaStream_t st) {
    const size_t per_layer = static_cast<size_t>(c->d.batch) * c->d.heads * c->d.head_dim * dtype_size(c->d.q_dtype);
    const size_t per_layer_out = static_cast<size_t>(c->d.batch) * c->d.heads * c->d.head_dim * out_size(c);
    static const int env_split = [] {
        const char* e = std::getenv("SKV_SELECT_SPLIT");  // tuning override: layers per side-stream batch
        return e ? std::atoi(e) : -1;
    }();
    // Selects that cannot ride in the attend tail are batched after the
    // layers (plans and head shards need them per layer: ledger / exchange).
    c->in_step = l1 - l0 > 1;  // a single layer gains nothing from batching: keep its tail
    // With a plan, the next step's ledger needs this step's selections per
    // layer -- except when that step is a Phase I step (its lists are empty;
    // the ledger only stores the new token), so Phase I steps batch too.
    const long long j_next = static_cast<long long>(n) - (c->has_plan ? c->plan.input_len : 0);
    const bool next_phase1 = c->has_plan && (j_next >= c->plan.output_len || phase_of(c->plan, j_next) == 1);
    c->defer_select = (!c->has_plan || next_phase1) && !c->prof;  // head shards exchange the whole step's rows at once
    c->deferred.clear();
    const int nl = l1 - l0;
    // measured: config 2 +1%, config 3 +0%, config 4 -1.6% -> off unless asked for
    const int split = (!c->defer_select || c->reduce || env_split <= 0) ? 0 : std::min(env_split, nl - 1);
    bool side = false;
    skv_status status = SKV_OK;
    for (int l = l0; l < l1 && status == SKV_OK; ++l) {
        const size_t o = per_layer * l;
        status = decode_layer_impl(c, l, n, r, static_cast<const uint8_t*>(q) + o,
                                   static_cast<const uint8_t*>(k_new) + o, static_cast<const uint8_t*>(v_new) + o,
                                   static_cast<uint8_t*>(out) + per_layer_out * l, nullptr, nullptr, l > l0, st);
        if (status == SKV_OK && split > 0 && l == l0 + split - 1 && !c->deferred.empty()) {
            if (!c->sel_st) {
                SKV_CUDA(cudaStreamCreateWithFlags(&c->sel_st, cudaStreamNonBlocking));
                SKV_CUDA(cudaEventCreateWithFlags(&c->ev_sel_in, cudaEventDisableTiming));
                SKV_CUDA(cudaEventCreateWithFlags(&c->ev_sel_out, cudaEventDisableTiming));
            }
            SKV_CUDA(cudaEventRecord(c->ev_sel_in, st));
            SKV_CUDA(cudaStreamWaitEvent(c->sel_st, c->ev_sel_in, 0));
            status = launch_deferred(c, c->sel_st);
            SKV_CUDA(cudaEventRecord(c->ev_sel_out, c->sel_st));
            side = true;
        }
    }
    c->defer_select = false;
    c->in_step = false;
    if (status != SKV_OK) {
        // a failed step leaves its deferred selections uncomputed: drop them
        for (const auto& d : c->deferred) c->pend_n[d.first] = -1;
        c->deferred.clear();
        if (side) cudaStreamWaitEvent(st, c->ev_sel_out, 0);
        return status;
    }
    // in plain stream order: it needs every attend of the range complete (the
    // PDL-chained attends only order against their direct predecessor)
    status = launch_deferred(c, st);
    if (side) SKV_CUDA(cudaStreamWaitEvent(st, c->ev_sel_out, 0));
    return status;
}

skv_status skv_swa_decode_step(skv_cache* c, int n, double r, const void* q, const void* k_new,
                               const void* v_new, void* out, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(q && k_new && v_new && out, "decode_step: null argument");
    if (skv_status e = check_status(c)) return e;
    StepShape s;
    if (skv_status st = step_shape(c, n, r, &s)) return st;
    DeviceGuard guard(c->d.device);
    return decode_layers(c, 0, c->d.layers, n, r, q, k_new, v_new, out, as_stream(stream));
}

// Host buffers: the step's layers are cut into chunks; chunk i's q/k/v go up
// on the h2d copy stream, its layers run on `stream` once they have landed,
// and its outputs go down on the d2h copy stream, so PCIe traffic in both
// directions overlaps the attention of the other chunks (and, across calls,
// of the previous step). Staging hazards are per chunk: the upload of chunk i
// waits for the previous step's compute of chunk i (the last reader of its
// staging), the compute waits for the previous download of chunk i (the last
// reader of its output staging). `stream` finally waits for the last download,
// so synchronising it covers every copy of the call.
static skv_status host_pipe_init(skv_cache* c, int chunks) {
    if (!c->h2d) SKV_CUDA(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    if (!c->d2h) SKV_CUDA(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    for (auto* v : {&c->ev_in, &c->ev_comp, &c->ev_out})
        while (static_cast<int>(v->size()) < chunks) {
            cudaEvent_t e;
            SKV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            v->push_back(e);
        }
    return SKV_OK;
}

skv_status skv_swa_decode_step_host(skv_cache* c, int n, double r, const void* q_host, const void* k_host,
                                    const void* v_host, void* out_host, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(q_host && k_host && v_host && out_host, "decode_step: null argument");
    if (skv_status e = check_status(c)) return e;
    StepShape shape;
    if (skv_status st = step_shape(c, n, r, &shape)) return st;
    DeviceGuard guard(c->d.device);
    const int L = c->d.layers;
    const size_t per_layer = static_cast<size_t>(c->d.batch) * c->d.heads * c->d.head_dim * dtype_size(c->d.q_dtype);
    const size_t per_layer_out = static_cast<size_t>(c->d.batch) * c->d.heads * c->d.head_dim * out_size(c);
    const size_t bytes = per_layer * L, obytes = per_layer_out * L;
    if (c->stage_bytes < 3 * bytes + obytes) {
        cudaFree(c->stage);
        c->stage = nullptr;
        if (cudaMalloc(reinterpret_cast<void**>(&c->stage), 3 * bytes + obytes) != cudaSuccess) {
            cudaGetLastError();
            c->stage_bytes = 0;
            return fail(SKV_ERR_OOM, "decode_step_host: cannot allocate staging");
        }
        c->stage_bytes = 3 * bytes + obytes;
    }
    static const int env_chunks = [] {
        const char* e = std::getenv("SKV_HOST_CHUNKS");  // tuning override
        return e ? std::max(1, std::atoi(e)) : kHostChunks;
    }();
    const int chunks = std::min(L, env_chunks);
    if (skv_status s = host_pipe_init(c, chunks)) return s;
    const cudaStream_t st = as_stream(stream);
    uint8_t *dq = c->stage, *dk = dq + bytes, *dv = dk + bytes, *dout = dv + bytes;
    const uint8_t* src[3] = {static_cast<const uint8_t*>(q_host), static_cast<const uint8_t*>(k_host),
                             static_cast<const uint8_t*>(v_host)};
    uint8_t* dst[3] = {dq, dk, dv};
    for (int i = 0; i < chunks; ++i) {
        const int l0 = L * i / chunks, l1 = L * (i + 1) / chunks;
        const size_t o = per_layer * l0, len = per_layer * (l1 - l0);
        SKV_CUDA(cudaStreamWaitEvent(c->h2d, c->ev_comp[i], 0));
        for (int t = 0; t < 3; ++t)
            SKV_CUDA(cudaMemcpyAsync(dst[t] + o, src[t] + o, len, cudaMemcpyHostToDevice, c->h2d));
        SKV_CUDA(cudaEventRecord(c->ev_in[i], c->h2d));
        SKV_CUDA(cudaStreamWaitEvent(st, c->ev_in[i], 0));
        SKV_CUDA(cudaStreamWaitEvent(st, c->ev_out[i], 0));
        if (skv_status s = decode_layers(c, l0, l1, n, r, dq, dk, dv, dout, st)) return s;
        SKV_CUDA(cudaEventRecord(c->ev_comp[i], st));
        SKV_CUDA(cudaStreamWaitEvent(c->d2h, c->ev_comp[i], 0));
        SKV_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(out_host) + per_layer_out * l0, dout + per_layer_out * l0,
                                 per_layer_out * (l1 - l0), cudaMemcpyDeviceToHost, c->d2h));
        SKV_CUDA(cudaEventRecord(c->ev_out[i], c->d2h));
    }
    SKV_CUDA(cudaStreamWaitEvent(st, c->ev_out[chunks - 1], 0));
    return SKV_OK;
}

skv_status skv_attend_over_indices(skv_cache* c, int layer, int n, const int32_t* idx, int m, const void* q,
                                   void* out, float* w_out, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    SKV_REQUIRE(n >= 1 && n <= c->d.capacity, "attend_over_indices: empty cache");
    SKV_REQUIRE(m >= 1, "attend_over_indices: empty selection");
    SKV_REQUIRE(m <= n, "attend_over_indices: more indices than tokens");
    SKV_REQUIRE(idx && q && out, "attend_over_indices: null argument");
    if (skv_status e = check_status(c)) return e;
    DeviceGuard guard(c->d.device);
    const cudaStream_t st = as_stream(stream);
    // The reference validates every index (attention.hpp:186-192). Indices
    // may come in any order and repeat (the reference loops over them as
    // given): each occurrence is its own softmax term and adds its own weight.
    std::vector<int32_t> h(static_cast<size_t>(c->d.batch) * m);
    SKV_CUDA(cudaMemcpyAsync(h.data(), idx, h.size() * 4, cudaMemcpyDefault, st));
    SKV_CUDA(cudaStreamSynchronize(st));
    bool ascending = true;
    for (int b = 0; b < c->d.batch; ++b)
        for (int i = 0; i < m; ++i) {
            const int32_t t = h[static_cast<size_t>(b) * m + i];
            SKV_REQUIRE(t >= 0 && t < n, "attend_over_indices: index out of range");
            if (i > 0 && t <= h[static_cast<size_t>(b) * m + i - 1]) ascending = false;
        }
    int G = 0;
    FoldSpec fold;
    fold.apply = 1;  // acc[idx] += w (attention.hpp:219-227)
    fold.sp_n = n;
    if (ascending)  // unique positions: the attend tail / select kernel folds them in place
        return launch_attend_c(c, layer, n, m, idx, m, false, q, nullptr, nullptr, out, nullptr, w_out, false, st,
                               &G, fold);
    // any order / repeats: attend without the fold, then scatter the per-
    // position head sums into the step row with fp64 atomics and fold that
    if (skv_status e = launch_attend_c(c, layer, n, m, idx, m, false, q, nullptr, nullptr, out, nullptr, w_out, false,
                                       st, &G, FoldSpec{}))
        return e;
    if (!c->frow) {
        const size_t bytes = static_cast<size_t>(c->d.batch) * c->d.capacity * 8;
        if (cudaMalloc(reinterpret_cast<void**>(&c->frow), bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(SKV_ERR_OOM, "attend_over_indices: cannot allocate %zu bytes of step-row scratch", bytes);
        }
        c->device_bytes += bytes;
    }
    const size_t lt = static_cast<size_t>(layer) * c->d.batch;
    const double* ws = nullptr;
    if (c->reduce) {  // head shards: the per-position head sums are summed across the shards first
        if (skv_status e = launch_select_c(c, layer, 1, idx, m, m, G, -1, 0, 0.0, false, st, 0, c->xbuf, nullptr))
            return e;
        if (skv_status e = c->reduce(c->xbuf, static_cast<size_t>(c->d.batch) * m, st, c->reduce_user))
            return fail(e, "head-shard reduce failed (%d)", static_cast<int>(e));
        ws = c->xbuf;
    }
    SKV_CUDA(launch_scatter_fold(c->imp + lt * c->d.capacity, c->d.capacity,
                                 c->wpart + lt * c->d.heads * c->d.capacity, G, m, idx, m, ws, n, c->sparsity + lt,
                                 c->frow, c->d.batch, st));
    c->pend_n[layer] = -1;  // importance changed: any pending selection is stale
    return SKV_OK;
}

skv_status skv_swa_select(const double* importance, int batch, int64_t ld, int n, double r, int32_t* idx_out,
                          int32_t* m_out, void* stream) {
    SKV_REQUIRE(batch >= 1, "swa_select: empty batch");
    SKV_REQUIRE(idx_out != nullptr, "swa_select: null output");
    SKV_REQUIRE(n >= 0, "swa_select: negative length");
    const size_t k = skv_swa_window_k(static_cast<size_t>(n), r);
    if (k == 0) return SKV_ERR_CONTRACT;
    const bool dense = n < 2 || 2 * static_cast<int>(k) >= n;
    const int m = dense ? n : 2 * static_cast<int>(k);
    if (m_out) *m_out = m;
    if (m == 0) return SKV_OK;
    if (!dense) {
        SKV_REQUIRE(importance != nullptr, "swa_select: importance length must be n-1");
        SKV_REQUIRE(ld >= n - 1, "swa_select: row stride shorter than n-1");
    }
    // long rows: the candidates' keys go to a stream-ordered scratch
    // ([batch][ld], the importance layout) instead of shared memory
    int dev = 0, max_smem = 0;
    SKV_CUDA(cudaGetDevice(&dev));
    SKV_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const bool long_row = !dense && static_cast<size_t>(n - k) * 8 + 8192 > static_cast<size_t>(max_smem);
    uint64_t* gkeys = nullptr;
    if (long_row && cudaMallocAsync(reinterpret_cast<void**>(&gkeys), static_cast<size_t>(batch) * ld * 8,
                                    as_stream(stream)) != cudaSuccess) {
        cudaGetLastError();
        return fail(SKV_ERR_OOM, "swa_select: cannot allocate key scratch for %d candidates", n - static_cast<int>(k));
    }
    skvd::SelectParams p{};
    p.gkeys = gkeys;
    p.imp = const_cast<double*>(importance);
    p.imp_ld = ld;
    p.select = 1;
    p.n = n;
    p.k = static_cast<int>(k);
    p.m = m;
    p.dense = dense ? 1 : 0;
    p.idx = idx_out;
    p.idx_ld = m;
    p.variant = SKV_VARIANT_SWA;
    const cudaError_t le = launch_select(p, batch, false, as_stream(stream));
    if (gkeys) cudaFreeAsync(gkeys, as_stream(stream));  // freed on the failure path too
    if (le != cudaSuccess) return fail(SKV_ERR_CUDA, "swa_select: %s", cudaGetErrorString(le));
    return SKV_OK;
}

skv_status skv_top_k_indices(const double* v, int batch, int64_t ld, int len, int k, int32_t* out, void* stream) {
    SKV_REQUIRE(k >= 0 && len >= 0 && k <= len, "top_k_indices: k exceeds length");
    SKV_REQUIRE(batch >= 1 && ld >= len, "top_k_indices: bad batch layout");
    if (k == 0) return SKV_OK;
    SKV_REQUIRE(v != nullptr && out != nullptr, "top_k_indices: null argument");
    SKV_CUDA(launch_top_k(v, batch, ld, len, k, out, as_stream(stream)));
    return SKV_OK;
}

skv_status skv_quantize(const double* x, size_t len, uint32_t bits, size_t channel_size, uint16_t* codes,
                        double* scales, int64_t* zero_points, void* stream) {
    SKV_REQUIRE(len > 0, "quantize: empty input");
    SKV_REQUIRE(bits == 4 || bits == 8, "quantize: bits must be 4 or 8");
    if (channel_size == 0) channel_size = len;
    SKV_REQUIRE(len % channel_size == 0, "quantize: channel_size must divide length");
    SKV_REQUIRE(x && codes && scales && zero_points, "quantize: null argument");
    SKV_CUDA(launch_quantize(x, static_cast<long long>(len), static_cast<long long>(channel_size), bits, codes,
                             scales, reinterpret_cast<long long*>(zero_points), as_stream(stream)));
    return SKV_OK;
}

skv_status skv_dequantize(const uint16_t* codes, size_t len, size_t channel_size, const double* scales,
                          const int64_t* zero_points, double* out, void* stream) {
    SKV_REQUIRE(channel_size > 0 && len % channel_size == 0, "dequantize: bad channel size");
    if (len == 0) return SKV_OK;
    SKV_REQUIRE(codes && scales && zero_points && out, "dequantize: null argument");
    SKV_CUDA(launch_dequantize(codes, static_cast<long long>(len), static_cast<long long>(channel_size), scales,
                               reinterpret_cast<const long long*>(zero_points), out, as_stream(stream)));
    return SKV_OK;
}

skv_status skv_cache_enable_host_tier(skv_cache* c, int poison) {
    SKV_REQUIRE(c != nullptr, "null cache");
    DeviceGuard guard(c->d.device);
    if (!c->host_kv) {
        void* h = nullptr;
        const size_t bytes = c->host_layer_bytes * c->d.layers;
        if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return fail(SKV_ERR_OOM, "host tier: cannot pin %llu bytes", static_cast<unsigned long long>(bytes));
        }
        c->host_kv = static_cast<uint8_t*>(h);
    }
    c->poison = poison != 0;
    return SKV_OK;
}

skv_status skv_cache_attach_recompute(skv_cache* c, int layer, const void* x_ln1, const void* wk, const void* wv,
                                      void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    if (!((c->d.kv_dtype == c->d.q_dtype || c->d.kv_dtype == SKV_U8) &&
          (c->d.q_dtype == SKV_F16 || c->d.q_dtype == SKV_BF16)))
        return fail(SKV_ERR_UNSUPPORTED, "recompute: fp16/bf16 compute (fp16/bf16 or INT8 caches) only");
    const long long h = static_cast<long long>(c->d.heads) * c->d.head_dim;
    if (h % 256 != 0) return fail(SKV_ERR_UNSUPPORTED, "recompute: hidden %lld not a multiple of 256", h);
    DeviceGuard guard(c->d.device);
    if (x_ln1 == nullptr) {
        c->rec_x[layer] = nullptr;
        return SKV_OK;
    }
    SKV_REQUIRE(wk && wv, "recompute: null weights");
    const cudaStream_t st = as_stream(stream);
    auto grab = [&](void** p, size_t bytes) -> bool {
        if (*p) return true;
        if (cudaMalloc(p, bytes) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return true;
    };
    const size_t rows = static_cast<size_t>((static_cast<long long>(c->d.batch) * c->d.capacity + 127) / 128 * 128);
    if (!grab(reinterpret_cast<void**>(&c->rec_wt[layer]), static_cast<size_t>(2 * h * h) * 2) ||
        !grab(reinterpret_cast<void**>(&c->rec_a), rows * static_cast<size_t>(h) * 2) ||
        !grab(reinterpret_cast<void**>(&c->rec_map), rows * sizeof(int2)) ||
        !grab(reinterpret_cast<void**>(&c->rec_m), sizeof(int)) ||
        (c->d.kv_dtype == SKV_U8 &&
         !grab(reinterpret_cast<void**>(&c->rec_c), rows * static_cast<size_t>(2 * h) * 4)))
        return fail(SKV_ERR_OOM, "recompute: cannot allocate buffers");
    SKV_CUDA(launch_transpose_kv_weights(wk, wv, c->rec_wt[layer], static_cast<int>(h), st));
    c->rec_x[layer] = static_cast<const uint8_t*>(x_ln1);
    return SKV_OK;
}

skv_status skv_cache_set_head_shard(skv_cache* c, int head_offset, int total_heads, skv_reduce_fn reduce,
                                    void* user) {
    SKV_REQUIRE(c != nullptr, "null cache");
    if (reduce == nullptr) {
        SKV_REQUIRE(head_offset == 0 && (total_heads == 0 || total_heads == c->d.heads),
                    "head shard: a cache without a reduce holds every head");
        c->reduce = nullptr;
        c->reduce_user = nullptr;
        c->head_offset = 0;
        c->total_heads = c->d.heads;
        return SKV_OK;
    }
    SKV_REQUIRE(total_heads >= c->d.heads && head_offset >= 0 && head_offset + c->d.heads <= total_heads,
                "head shard: heads [offset, offset + H) must lie inside total_heads");
    DeviceGuard guard(c->d.device);
    if (c->xbuf == nullptr) {
        // the prefill's seed rows + sparsity ([B][Ncap + 1]) or a whole
        // step's step rows ([L][B][m], m <= Ncap)
        const size_t cells = std::max(static_cast<size_t>(c->d.batch) * (c->d.capacity + 1),
                                      static_cast<size_t>(c->d.layers) * c->d.batch * c->d.capacity);
        const size_t bytes = cells * 8;
        if (cudaMalloc(reinterpret_cast<void**>(&c->xbuf), bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(SKV_ERR_OOM, "head shard: cannot allocate the exchange row");
        }
        SKV_CUDA(cudaMemset(c->xbuf, 0, bytes));
        c->device_bytes += bytes;
    }
    c->reduce = reduce;
    c->reduce_user = user;
    c->head_offset = head_offset;
    c->total_heads = total_heads;
    return SKV_OK;
}

skv_status skv_cache_set_variant(skv_cache* c, int variant, int stride) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(variant >= SKV_VARIANT_DENSE && variant <= SKV_VARIANT_STRIDED, "unknown attention variant");
    SKV_REQUIRE(stride >= 0, "strided_attention_mask: stride must be >= 1");
    c->variant = variant;
    c->stride = stride;
    for (auto& p : c->pend_n) p = -1;
    return SKV_OK;
}

skv_status skv_selection_size(const skv_cache* c, int n, double r, int32_t* m, int32_t* k) {
    SKV_REQUIRE(c != nullptr, "null cache");
    StepShape s;
    if (skv_status e = step_shape(c, n, r, &s)) return e;
    if (m) *m = s.m;
    if (k) *k = s.k;
    return SKV_OK;
}

skv_status skv_pending_selection(const skv_cache* c, int layer, int n, double r, int32_t* idx_out, int32_t* m_out,
                                 void* stream) {
    SKV_REQUIRE(c != nullptr && idx_out != nullptr, "pending selection: null argument");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    SKV_REQUIRE(c->pend_n[layer] == n && c->pend_r[layer] == r,
                "pending selection: no selection was made for this (n, r) on this layer");
    StepShape s;
    if (skv_status e = step_shape(c, n, r, &s)) return e;
    DeviceGuard guard(c->d.device);
    SKV_CUDA(cudaMemcpy2DAsync(idx_out, static_cast<size_t>(s.m) * 4, layer_idx(c, layer), c->d.capacity * 4,
                               static_cast<size_t>(s.m) * 4, c->d.batch, cudaMemcpyDefault, as_stream(stream)));
    if (m_out) *m_out = s.m;
    return SKV_OK;
}

skv_status skv_sparsity_get(const skv_cache* c, int layer, int b0, int nb, double* dst, void* stream) {
    if (skv_status s = check_block(c, layer, b0, nb, 0, 1)) return s;
    SKV_REQUIRE(dst != nullptr, "sparsity: null output");
    DeviceGuard guard(c->d.device);
    SKV_CUDA(cudaMemcpyAsync(dst, c->sparsity + static_cast<size_t>(layer) * c->d.batch + b0,
                             static_cast<size_t>(nb) * 8, cudaMemcpyDefault, as_stream(stream)));
    return SKV_OK;
}

skv_status skv_cache_set_plan(skv_cache* c, const skv_plan* plan) {
    SKV_REQUIRE(c != nullptr, "null cache");
    if (plan == nullptr) {
        c->has_plan = false;
        return SKV_OK;
    }
    // validate_plan (scheduler.hpp:26-35)
    const skv_plan& p = *plan;
    SKV_REQUIRE(p.input_len >= 0 && p.output_len >= 0, "plan: negative workload");
    if (p.p1 == p.p2) {
        SKV_REQUIRE(p.p1 == p.output_len, "plan: degenerate plans must have p1 == p2 == n");
    } else {
        SKV_REQUIRE(p.p1 < p.p2 && p.p2 <= p.output_len, "plan: requires 0 <= p1 < p2 <= n");
        SKV_REQUIRE(p.alpha > 0.0 && p.alpha < 1.0, "plan: alpha out of (0,1)");
        SKV_REQUIRE(p.beta > 0.0 && p.beta < 1.0, "plan: beta out of (0,1)");
    }
    c->plan = p;
    c->has_plan = true;
    for (auto& j : c->ledger_j) j = -1;
    return SKV_OK;
}

skv_status skv_ledger_set(skv_cache* c, int layer, int b0, int nb, int len, const uint8_t* src, void* stream) {
    if (skv_status s = check_block(c, layer, b0, nb, 0, len)) return s;
    if (c->paged) return fail(SKV_ERR_UNSUPPORTED, "paged cache: tiers follow the slots; set them by decoding");
    DeviceGuard guard(c->d.device);
    uint8_t* dst = c->tiers + (static_cast<size_t>(layer) * c->d.batch + b0) * c->d.capacity;
    SKV_CUDA(cudaMemcpy2DAsync(dst, c->d.capacity, src, len, len, nb, cudaMemcpyDefault, as_stream(stream)));
    return SKV_OK;
}

skv_status skv_ledger_get(const skv_cache* c, int layer, int b0, int nb, int len, uint8_t* dst, void* stream) {
    if (skv_status s = check_block(c, layer, b0, nb, 0, len)) return s;
    DeviceGuard guard(c->d.device);
    const uint8_t* src = c->tiers + (static_cast<size_t>(layer) * c->d.batch + b0) * c->d.capacity;
    SKV_CUDA(cudaMemcpy2DAsync(dst, len, src, c->d.capacity, len, nb, cudaMemcpyDefault, as_stream(stream)));
    return SKV_OK;
}

skv_status skv_cache_set_capacity(skv_cache* c, uint64_t device_capacity) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(device_capacity > 0, "KvLedger: zero device capacity");
    c->cap_bytes = device_capacity;
    return SKV_OK;
}

skv_status skv_ledger_totals(const skv_cache* c, uint64_t* device_bytes, uint64_t* host_bytes,
                             uint64_t* peak_device_bytes, uint64_t* capacity, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    DeviceGuard guard(c->d.device);
    skvd::LedgerTotals t{};
    SKV_CUDA(cudaMemcpyAsync(&t, c->tot, sizeof t, cudaMemcpyDeviceToHost, as_stream(stream)));
    SKV_CUDA(cudaStreamSynchronize(as_stream(stream)));
    if (device_bytes) *device_bytes = t.dev_tokens * c->tok_bytes;
    if (host_bytes) *host_bytes = t.host_tokens * c->tok_bytes;
    if (peak_device_bytes) *peak_device_bytes = std::max(t.peak_dev_tokens, t.dev_tokens) * c->tok_bytes;
    if (capacity) *capacity = c->cap_bytes;
    return check_status(c);
}

skv_status skv_ledger_counters(const skv_cache* c, uint64_t* rows, void* stream) {
    SKV_REQUIRE(c != nullptr && rows != nullptr, "null argument");
    DeviceGuard guard(c->d.device);
    skvd::LedgerTotals t{};
    SKV_CUDA(cudaMemcpyAsync(&t, c->tot, sizeof t, cudaMemcpyDeviceToHost, as_stream(stream)));
    SKV_CUDA(cudaStreamSynchronize(as_stream(stream)));
    for (int i = 0; i < 4; ++i) rows[i] = t.moved[i];
    rows[4] = t.kept;
    return SKV_OK;
}

// Calibration of CostParams::bandwidth on the real movement kernel: `rows`
// token rows per sequence offloaded and `rows` others reloaded in one duplex
// launch (as a Phase II step does), `reps` times, on layer `layer` of a
// non-paged cache with a host tier. Overwrites that layer's action lists and
// moves real rows: calibrate on a scratch cache.
skv_status skv_profile_move(skv_cache* c, int layer, int rows, int reps, double* ms, void* stream) {
    SKV_REQUIRE(c != nullptr && ms != nullptr, "null argument");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    SKV_REQUIRE(c->host_kv != nullptr && !c->paged, "profile_move: a non-paged cache with a host tier");
    SKV_REQUIRE(rows >= 1 && 2 * rows <= c->d.capacity && reps >= 1, "profile_move: bad size");
    DeviceGuard guard(c->d.device);
    const cudaStream_t st = as_stream(stream);
    const size_t lt = static_cast<size_t>(layer) * c->d.batch;
    std::vector<int> lists(static_cast<size_t>(c->d.batch) * 4 * c->d.capacity, 0), counts(c->d.batch * 4, 0);
    for (int b = 0; b < c->d.batch; ++b) {
        for (int i = 0; i < rows; ++i) {
            lists[(static_cast<size_t>(b) * 4 + 0) * c->d.capacity + i] = i;
            lists[(static_cast<size_t>(b) * 4 + 2) * c->d.capacity + i] = rows + i;
        }
        counts[b * 4 + 0] = rows;
        counts[b * 4 + 2] = rows;
    }
    SKV_CUDA(cudaMemcpyAsync(c->act_lists + lt * 4 * c->d.capacity, lists.data(), lists.size() * 4,
                             cudaMemcpyHostToDevice, st));
    SKV_CUDA(cudaMemcpyAsync(c->act_counts + lt * 4, counts.data(), counts.size() * 4, cudaMemcpyHostToDevice, st));
    const bool poison = c->poison;
    c->poison = false;
    const uint8_t* rec = c->rec_x[layer];  // movement only: no recompute GEMM
    c->rec_x[layer] = nullptr;
    cudaEvent_t e0, e1;
    SKV_CUDA(cudaEventCreate(&e0));
    SKV_CUDA(cudaEventCreate(&e1));
    skv_status out = launch_movement(c, layer, false, st);  // warm-up
    SKV_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < reps && out == SKV_OK; ++i) out = launch_movement(c, layer, false, st);
    SKV_CUDA(cudaEventRecord(e1, st));
    SKV_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    SKV_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->poison = poison;
    c->rec_x[layer] = rec;
    *ms = t / reps;
    return out;
}

skv_status skv_cache_storage(const skv_cache* c, int32_t* slots_per_sequence, uint64_t* kv_pool_bytes,
                             uint64_t* full_kv_bytes) {
    SKV_REQUIRE(c != nullptr, "null cache");
    if (slots_per_sequence) *slots_per_sequence = c->pcap;
    if (kv_pool_bytes) *kv_pool_bytes = c->layer_bytes * c->d.layers;
    if (full_kv_bytes) *full_kv_bytes = c->host_layer_bytes * c->d.layers;
    return SKV_OK;
}

skv_status skv_step_actions(skv_cache* c, int layer, int j, const int32_t* selected, int m, int k, int apply,
                            int32_t* lists_out, int32_t* counts_out, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(c->has_plan, "step_actions: no plan attached (skv_cache_set_plan)");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    SKV_REQUIRE(j >= 0 && j < c->plan.output_len, "step_actions: step beyond output length");
    SKV_REQUIRE(selected != nullptr && m >= 0 && k >= 1, "step_actions: bad selection");
    if (c->paged && apply)
        return fail(SKV_ERR_UNSUPPORTED, "paged cache: actions are applied (with their data movement) by decoding");
    if (skv_status e = check_status(c)) return e;
    DeviceGuard guard(c->d.device);
    const cudaStream_t st = as_stream(stream);
    if (skv_status e = launch_ledger_c(c, layer, j, selected, m, m, k, apply != 0, false, false, st)) return e;
    const size_t lt = static_cast<size_t>(layer) * c->d.batch;
    if (lists_out)
        SKV_CUDA(cudaMemcpyAsync(lists_out, c->act_lists + lt * 4 * c->d.capacity,
                                 static_cast<size_t>(c->d.batch) * 4 * c->d.capacity * 4, cudaMemcpyDefault, st));
    if (counts_out)
        SKV_CUDA(cudaMemcpyAsync(counts_out, c->act_counts + lt * 4, static_cast<size_t>(c->d.batch) * 16,
                                 cudaMemcpyDefault, st));
    return SKV_OK;
}

skv_status skv_last_actions(const skv_cache* c, int layer, int32_t* lists_out, int32_t* counts_out, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(layer >= 0 && layer < c->d.layers, "KvLedger: layer out of range");
    DeviceGuard guard(c->d.device);
    const cudaStream_t st = as_stream(stream);
    const size_t lt = static_cast<size_t>(layer) * c->d.batch;
    if (lists_out)
        SKV_CUDA(cudaMemcpyAsync(lists_out, c->act_lists + lt * 4 * c->d.capacity,
                                 static_cast<size_t>(c->d.batch) * 4 * c->d.capacity * 4, cudaMemcpyDefault, st));
    if (counts_out)
        SKV_CUDA(cudaMemcpyAsync(counts_out, c->act_counts + lt * 4, static_cast<size_t>(c->d.batch) * 16,
                                 cudaMemcpyDefault, st));
    return SKV_OK;
}

skv_status skv_gemm_tn(const void* A, const void* Bt, float* C, int M, int N, int K, int bf16, void* stream) {
    SKV_REQUIRE(A && Bt && C, "gemm: null argument");
    SKV_REQUIRE(M > 0 && M % 128 == 0 && N > 0 && N % 256 == 0 && K > 0 && K % 64 == 0,
                "gemm: M % 128, N % 256, K % 64 must be 0");
    SKV_CUDA(launch_gemm_tn(A, Bt, C, nullptr, M, N, K, bf16 != 0, as_stream(stream)));
    return SKV_OK;
}

skv_status skv_device_alloc(int device, size_t bytes, void** out) {
    SKV_REQUIRE(out != nullptr, "skv_device_alloc: null output");
    DeviceGuard guard(device);
    *out = nullptr;
    if (bytes == 0) return SKV_OK;
    if (cudaMalloc(out, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(SKV_ERR_OOM, "skv_device_alloc: cannot allocate %llu bytes", static_cast<unsigned long long>(bytes));
    }
    return SKV_OK;
}

skv_status skv_device_free(void* ptr) {
    if (ptr) SKV_CUDA(cudaFree(ptr));
    return SKV_OK;
}

skv_status skv_copy(void* dst, const void* src, size_t bytes, void* stream) {
    if (bytes == 0) return SKV_OK;
    SKV_REQUIRE(dst && src, "skv_copy: null pointer");
    SKV_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
    SKV_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return SKV_OK;
}

skv_status skv_host_alloc(size_t bytes, void** out) {
    SKV_REQUIRE(out != nullptr, "skv_host_alloc: null output");
    *out = nullptr;
    if (bytes == 0) return SKV_OK;
    if (cudaHostAlloc(out, bytes, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return fail(SKV_ERR_OOM, "skv_host_alloc: cannot pin %zu bytes", bytes);
    }
    return SKV_OK;
}

skv_status skv_host_free(void* ptr) {
    if (ptr) SKV_CUDA(cudaFreeHost(ptr));
    return SKV_OK;
}

skv_status skv_stream_synchronize(void* stream) {
    SKV_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return SKV_OK;
}

skv_status skv_profile_enable(skv_cache* c, int enable) {
    SKV_REQUIRE(c != nullptr, "null cache");
    DeviceGuard guard(c->d.device);
    c->prof = enable != 0;
    for (cudaEvent_t e : c->ev) c->ev_pool.push_back(e);
    c->ev.clear();
    c->attend_launches = 0;
    c->algo_bytes = 0;
    return SKV_OK;
}

skv_status skv_attend_config(const skv_cache* c, int32_t* heads_per_cta, int32_t* grid, int32_t* smem_bytes,
                             int32_t* ctas_per_sm) {
    SKV_REQUIRE(c != nullptr, "null cache");
    if (heads_per_cta) *heads_per_cta = c->last_hg;
    if (grid) *grid = c->last_grid;
    if (smem_bytes) *smem_bytes = static_cast<int32_t>(c->last_smem);
    if (ctas_per_sm) *ctas_per_sm = c->last_occ;
    return SKV_OK;
}

skv_status skv_profile_attend_chain(skv_cache* c, int n, double r, const void* q, const void* k_new,
                                    const void* v_new, void* out, int reps, double* total_ms, void* stream) {
    SKV_REQUIRE(c != nullptr, "null cache");
    SKV_REQUIRE(reps >= 1 && q && k_new && v_new && out && total_ms, "profile_attend_chain: bad argument");
    StepShape s;
    if (skv_status e = step_shape(c, n, r, &s)) return e;
    for (int l = 0; l < c->d.layers; ++l)
        SKV_REQUIRE(c->pend_n[l] == n && c->pend_r[l] == r, "profile_attend_chain: no pending selection for n");
    DeviceGuard guard(c->d.device);
    const cudaStream_t st = as_stream(stream);
    const bool prof = c->prof;
    c->prof = false;
    const size_t per_layer = static_cast<size_t>(c->d.batch) * c->d.heads * c->d.head_dim * dtype_size(c->d.q_dtype);
    const size_t per_layer_out = static_cast<size_t>(c->d.batch) * c->d.heads * c->d.head_dim * out_size(c);
    cudaEvent_t e0, e1;
    SKV_CUDA(cudaEventCreate(&e0));
    SKV_CUDA(cudaEventCreate(&e1));
    SKV_CUDA(cudaEventRecord(e0, st));
    for (int rep = 0; rep < reps; ++rep)
        for (int l = 0; l < c->d.layers; ++l) {
            int G = 0;
            if (skv_status e = launch_attend_c(c, l, n, s.m, layer_idx(c, l), c->d.capacity, true,
                                               static_cast<const uint8_t*>(q) + per_layer * l,
                                               static_cast<const uint8_t*>(k_new) + per_layer * l,
                                               static_cast<const uint8_t*>(v_new) + per_layer * l,
                                               static_cast<uint8_t*>(out) + per_layer_out * l, nullptr, nullptr,
                                               rep + l > 0, st, &G)) {
                c->prof = prof;
                return e;
            }
        }
    SKV_CUDA(cudaEventRecord(e1, st));
    SKV_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    SKV_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->prof = prof;
    *total_ms = ms;
    return SKV_OK;
}

skv_status skv_profile_read(skv_cache* c, double* total_ms, int64_t* launches, uint64_t* algo) {
    SKV_REQUIRE(c != nullptr, "null cache");
    DeviceGuard guard(c->d.device);
    double tot = 0.0;
    for (size_t i = 0; i + 1 < c->ev.size(); i += 2) {
        SKV_CUDA(cudaEventSynchronize(c->ev[i + 1]));
        float ms = 0.f;
        SKV_CUDA(cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]));
        tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = c->attend_launches;
    if (algo) *algo = c->algo_bytes;
    return SKV_OK;
}

}  // extern "C"
