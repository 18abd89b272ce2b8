// skv/b200.hpp -- C++ mirror of the reference `skv` API for the SWA decode
// hot path, running on the B200 kernels behind include/skv_b200.h.
//
// Include it next to the reference headers (the reference's include dir stays
// on the path; its types are reused, nothing is redefined):
//
//   #include "skv/attention.hpp"   // reference: Matrix, AttentionState, ...
//   #include "skv/b200.hpp"        // this mirror
//
// Two layers:
//  * skv::b200::<same name as the reference>(<same signature>) -- compat
//    entry points taking the reference's host types. They move the state to
//    the device, run the sm_100a kernels, and write results back into the
//    reference types (per-head accumulators included), so existing callers
//    switch by namespace. Errors throw the reference exception classes
//    (common.hpp:12-34). Compute is fp32 on device: results match the fp64
//    reference within 1e-5 relative; selections are bit-exact.
//  * skv::b200::DeviceCache -- the device-resident, batched state
//    (L layers x B sequences) for throughput; inputs/outputs stay in HBM.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>
#include <utility>

#include "skv/attention.hpp"
#include "skv/common.hpp"
#include "skv/matrix.hpp"
#include "skv/quant.hpp"
#include "skv/memsim.hpp"
#include "skv/scheduler.hpp"
#include "skv_b200.h"

namespace skv::b200 {

inline void check(skv_status s) {
    if (s == SKV_OK) return;
    const std::string msg = skv_last_error();
    switch (s) {
    case SKV_ERR_CONTRACT: throw ContractViolation(msg);
    case SKV_ERR_OOM: throw OutOfDeviceMemory(msg);
    case SKV_ERR_INFEASIBLE: throw InfeasiblePlan(msg);
    default: throw std::runtime_error("skv_b200: " + msg);
    }
}

// RAII device buffer.
class DeviceBuffer {
  public:
    DeviceBuffer() = default;
    DeviceBuffer(std::size_t bytes, int device = 0) : bytes_(bytes) {
        check(skv_device_alloc(device, bytes, &ptr_));
    }
    ~DeviceBuffer() { skv_device_free(ptr_); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(o.ptr_), bytes_(o.bytes_) { o.ptr_ = nullptr; }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            skv_device_free(ptr_);
            ptr_ = o.ptr_;
            bytes_ = o.bytes_;
            o.ptr_ = nullptr;
        }
        return *this;
    }
    void* get() const { return ptr_; }
    template <class T>
    T* as() const {
        return static_cast<T*>(ptr_);
    }
    void upload(const void* src, std::size_t bytes) { check(skv_copy(ptr_, src, bytes, nullptr)); }
    void download(void* dst, std::size_t bytes) const { check(skv_copy(dst, ptr_, bytes, nullptr)); }

  private:
    void* ptr_ = nullptr;
    std::size_t bytes_ = 0;
};

// Device-resident decode state for `layers` x `batch` sequences.
class DeviceCache {
  public:
    DeviceCache(int layers, int batch, int heads, int head_dim, int capacity, skv_dtype kv = SKV_F16,
                skv_dtype q = SKV_F16, int device = 0, bool out_f32 = false) {
        skv_cache_desc d{layers, batch, heads, head_dim, capacity, kv, q, device, out_f32 ? 1 : 0};
        check(skv_cache_create(&d, &c_));
    }
    ~DeviceCache() { skv_cache_destroy(c_); }
    DeviceCache(const DeviceCache&) = delete;
    DeviceCache& operator=(const DeviceCache&) = delete;
    skv_cache* handle() const { return c_; }

    void append_tokens(int layer, int b0, int nb, int t0, int nt, const void* k, const void* v, void* st = nullptr) {
        check(skv_cache_write(c_, layer, b0, nb, t0, nt, k, v, st));
    }
    void prefill_seed(int layer, int n, const void* q_last, void* out, void* st = nullptr) {
        check(skv_prefill_seed(c_, layer, n, q_last, out, st));
    }
    void decode_layer(int layer, int n, double r, const void* q, const void* k, const void* v, void* out,
                      int32_t* idx_out = nullptr, float* w_out = nullptr, void* st = nullptr) {
        check(skv_swa_decode_layer(c_, layer, n, r, q, k, v, out, idx_out, w_out, st));
    }
    void decode_step(int n, double r, const void* q, const void* k, const void* v, void* out, void* st = nullptr) {
        check(skv_swa_decode_step(c_, n, r, q, k, v, out, st));
    }
    void attend_over_indices(int layer, int n, const int32_t* idx, int m, const void* q, void* out,
                             float* w_out = nullptr, void* st = nullptr) {
        check(skv_attend_over_indices(c_, layer, n, idx, m, q, out, w_out, st));
    }
    void set_importance(int layer, int b0, int nb, int len, const double* src, void* st = nullptr) {
        check(skv_importance_set(c_, layer, b0, nb, len, src, st));
    }
    void importance(int layer, int b0, int nb, int len, double* dst, void* st = nullptr) const {
        check(skv_importance_get(c_, layer, b0, nb, len, dst, st));
    }
    // Engine::prefill's attention on the tensor cores (engine.hpp:485-529)
    void prefill_layer(int layer, int s, const void* q, void* out, void* st = nullptr) {
        check(skv_prefill_layer(c_, layer, s, q, out, st));
    }
    void decode_step_host(int n, double r, const void* q, const void* k, const void* v, void* out,
                          void* st = nullptr) {
        check(skv_swa_decode_step_host(c_, n, r, q, k, v, out, st));
    }
    // Head sharding (B < #GPU): this cache holds heads [head_offset, +H) of
    // total_heads; `reduce` sums the fp64 step row across the shards on the
    // given stream, e.g. with ncclAllReduce.
    void set_head_shard(int head_offset, int total_heads, skv_reduce_fn reduce, void* user) {
        check(skv_cache_set_head_shard(c_, head_offset, total_heads, reduce, user));
    }
    // KvLedger / scheduler (memsim.hpp:72-215, scheduler.hpp:28-381) on the device
    void set_plan(const skv_plan& plan) { check(skv_cache_set_plan(c_, &plan)); }
    void ledger_set(int layer, int b0, int nb, int len, const std::uint8_t* tiers, void* st = nullptr) {
        check(skv_ledger_set(c_, layer, b0, nb, len, tiers, st));
    }
    void step_actions(int layer, int j, const int32_t* selected, int m, int k, bool apply, int32_t* lists,
                      int32_t* counts, void* st = nullptr) {
        check(skv_step_actions(c_, layer, j, selected, m, k, apply ? 1 : 0, lists, counts, st));
    }

  private:
    skv_cache* c_ = nullptr;
};

// ---- compat entry points (reference signatures) -----------------------------

// attention.hpp:122-138
inline std::size_t swa_window_k(std::size_t n, double r) {
    const std::size_t k = skv_swa_window_k(n, r);
    if (k == 0) throw ContractViolation(skv_last_error());
    return k;
}
inline std::size_t swa_keep_count(std::size_t n, double r) { return std::min(2 * swa_window_k(n, r), n); }

// matrix.hpp:162-176
inline IndexList top_k_indices(std::span<const double> v, std::size_t k) {
    if (k > v.size()) throw ContractViolation("top_k_indices: k exceeds length");
    IndexList out(k);
    if (k == 0) return out;
    DeviceBuffer dv(v.size() * 8), di(k * 4);
    dv.upload(v.data(), v.size() * 8);
    check(skv_top_k_indices(dv.as<double>(), 1, static_cast<int64_t>(v.size()), static_cast<int>(v.size()),
                            static_cast<int>(k), di.as<int32_t>(), nullptr));
    std::vector<int32_t> h(k);
    di.download(h.data(), k * 4);
    for (std::size_t i = 0; i < k; ++i) out[i] = static_cast<std::size_t>(h[i]);
    return out;
}

// attention.hpp:142-171
inline SparseSelection swa_select(std::span<const double> importance, std::size_t n, double r) {
    SparseSelection sel;
    sel.k = swa_window_k(n, r);
    const bool dense = n < 2 || 2 * sel.k >= n;
    if (!dense && importance.size() != n - 1)
        throw ContractViolation("swa_select: importance length must be n-1");
    const std::size_t m = dense ? n : 2 * sel.k;
    if (m == 0) return sel;
    DeviceBuffer dimp(std::max<std::size_t>(importance.size(), 1) * 8), didx(m * 4);
    if (!importance.empty()) dimp.upload(importance.data(), importance.size() * 8);
    int32_t mo = 0;
    check(skv_swa_select(dimp.as<double>(), 1, static_cast<int64_t>(std::max<std::size_t>(importance.size(), 1)),
                         static_cast<int>(n), r, didx.as<int32_t>(), &mo, nullptr));
    std::vector<int32_t> h(m);
    didx.download(h.data(), m * 4);
    // split back into the reference's local / global parts (attention.hpp:146-170)
    const std::size_t window = dense ? std::min(sel.k, n) : sel.k;
    for (std::size_t i = 0; i < m; ++i) {
        const auto t = static_cast<std::size_t>(h[i]);
        (t >= n - window ? sel.local_indices : sel.global_indices).push_back(t);
    }
    return sel;
}

// quant.hpp:43-81 (bit-exact)
inline QuantizedVector quantize(std::span<const double> x, std::uint32_t bits = 8, std::size_t channel_size = 0) {
    if (x.empty()) throw ContractViolation("quantize: empty input");
    const std::size_t cs = channel_size ? channel_size : x.size();
    const std::size_t groups = x.size() % cs == 0 ? x.size() / cs : 1;
    DeviceBuffer dx(x.size() * 8), dc(x.size() * 2), ds(groups * 8), dz(groups * 8);
    dx.upload(x.data(), x.size() * 8);
    check(skv_quantize(dx.as<double>(), x.size(), bits, channel_size, dc.as<uint16_t>(), ds.as<double>(),
                       dz.as<int64_t>(), nullptr));
    QuantizedVector q;
    q.bits = bits;
    q.channel_size = cs;
    q.codes.resize(x.size());
    q.scales.resize(groups);
    q.zero_points.resize(groups);
    dc.download(q.codes.data(), x.size() * 2);
    ds.download(q.scales.data(), groups * 8);
    dz.download(q.zero_points.data(), groups * 8);
    return q;
}

// quant.hpp:84-95
inline Vector dequantize(const QuantizedVector& q) {
    Vector out(q.codes.size());
    if (out.empty()) return out;
    DeviceBuffer dc(q.codes.size() * 2), ds(q.scales.size() * 8), dz(q.zero_points.size() * 8),
        dout(out.size() * 8);
    dc.upload(q.codes.data(), q.codes.size() * 2);
    ds.upload(q.scales.data(), q.scales.size() * 8);
    dz.upload(q.zero_points.data(), q.zero_points.size() * 8);
    check(skv_dequantize(dc.as<uint16_t>(), q.codes.size(), q.channel_size, ds.as<double>(),
                         dz.as<int64_t>(), dout.as<double>(), nullptr));
    dout.download(out.data(), out.size() * 8);
    return out;
}

inline Vector quantize_roundtrip(std::span<const double> x, std::uint32_t bits, std::size_t channel_size) {
    return b200::dequantize(b200::quantize(x, bits, channel_size));
}

namespace detail {

// Upload one reference AttentionState into a 1-layer, 1-sequence fp32 cache.
struct StagedState {
    std::size_t H, D, n;
    DeviceCache cache;
    StagedState(const AttentionState& st)
        : H(st.head_count), D(st.head_dim), n(st.tokens()),
          cache(1, 1, static_cast<int>(st.head_count), static_cast<int>(st.head_dim),
                static_cast<int>(std::max<std::size_t>(st.tokens(), 1)), SKV_F32, SKV_F32, 0, true) {
        std::vector<float> k(n * H * D), v(n * H * D);
        for (std::size_t t = 0; t < n; ++t)
            for (std::size_t h = 0; h < H; ++h)
                for (std::size_t d = 0; d < D; ++d) {
                    k[(t * H + h) * D + d] = static_cast<float>(st.keys[h].at(t, d));
                    v[(t * H + h) * D + d] = static_cast<float>(st.values[h].at(t, d));
                }
        DeviceBuffer dk(k.size() * 4), dv(v.size() * 4);
        dk.upload(k.data(), k.size() * 4);
        dv.upload(v.data(), v.size() * 4);
        cache.append_tokens(0, 0, 1, 0, static_cast<int>(n), dk.get(), dv.get());
    }
};

}  // namespace detail

// attention.hpp:183-231: same contract and state mutation as the reference
// (per-head accumulators grow to n and gain w at the selected positions).
// Indices may come in any order and repeat: every occurrence is one softmax
// term and adds its own weight, exactly as the reference loops over them.
inline StepAttentionResult attend_over_indices(AttentionState& state, const Matrix& q_step,
                                               const IndexList& indices) {
    const std::size_t n = state.tokens();
    require(n >= 1, "attend_over_indices: empty cache");
    require(q_step.rows == state.head_count && q_step.cols == state.head_dim,
            "attend_over_indices: query shape mismatch");
    require(!indices.empty(), "attend_over_indices: empty selection");
    for (const std::size_t idx : indices) require(idx < n, "attend_over_indices: index out of range");
    const std::size_t H = state.head_count, D = state.head_dim, m = indices.size();
    detail::StagedState s(state);
    std::vector<float> q(H * D);
    for (std::size_t i = 0; i < H * D; ++i) q[i] = static_cast<float>(q_step.data[i]);
    std::vector<int32_t> idx(m);
    for (std::size_t i = 0; i < m; ++i) idx[i] = static_cast<int32_t>(indices[i]);
    DeviceBuffer dq(H * D * 4), dout(H * D * 4), didx(m * 4), dw(H * m * 4);
    dq.upload(q.data(), q.size() * 4);
    didx.upload(idx.data(), m * 4);
    s.cache.attend_over_indices(0, static_cast<int>(n), didx.as<int32_t>(), static_cast<int>(m), dq.get(),
                                dout.get(), dw.as<float>());
    std::vector<float> out(H * D), w(H * m);
    dout.download(out.data(), out.size() * 4);
    dw.download(w.data(), w.size() * 4);
    StepAttentionResult res;
    res.attn = Matrix(H, D);
    for (std::size_t i = 0; i < H * D; ++i) res.attn.data[i] = out[i];
    res.new_aw_row = Vector(n, 0.0);
    for (std::size_t h = 0; h < H; ++h) {
        Vector& acc = state.attention_accum[h];
        acc.resize(n, 0.0);
        for (std::size_t t = 0; t < m; ++t) {
            acc[indices[t]] += w[h * m + t];
            res.new_aw_row[indices[t]] += w[h * m + t];
        }
    }
    return res;
}

// attention.hpp:235-244
inline StepAttentionResult swa_attention(AttentionState& state, const Matrix& q_step, const SparsityConfig& cfg) {
    const std::size_t n = state.tokens();
    require(n >= 1, "swa_attention: empty cache");
    const Vector importance = state.head_summed_accum();
    SparseSelection sel = b200::swa_select(importance, n, cfg.ratio);
    StepAttentionResult res = b200::attend_over_indices(state, q_step, sel.all());
    res.selection = std::move(sel);
    return res;
}

// attention.hpp:91-117: softmax(q k^T / sqrt(D)) v per query row; returns
// (attn, aw). The causal mask is aligned to the bottom-right corner as in the
// reference (:98-103): row i sees keys j <= i + (k.rows - q.rows). Same checks,
// messages and order as the reference; a causal row with no visible key fails
// like softmax_rows (matrix.hpp:145). Each row is one attend over its key
// range on a one-head fp32 cache: results match the fp64 reference within
// 1e-5 relative. head_dim 128 only (the compiled kernels).
inline std::pair<Matrix, Matrix> dense_attention(const Matrix& q, const Matrix& k, const Matrix& v, bool causal) {
    require(q.cols == k.cols && k.cols == v.cols, "dense_attention: head_dim mismatch");
    require(k.rows == v.rows, "dense_attention: key/value length mismatch");
    require(q.rows > 0 && k.rows > 0, "dense_attention: empty input");
    const std::size_t sq = q.rows, sk = k.rows, D = q.cols;
    const std::ptrdiff_t off = static_cast<std::ptrdiff_t>(sk) - static_cast<std::ptrdiff_t>(sq);
    require(!causal || off >= 0, "softmax_rows: row has no finite entry");
    std::pair<Matrix, Matrix> res{Matrix(sq, v.cols), Matrix(sq, sk)};
    DeviceCache cache(1, 1, 1, static_cast<int>(D), static_cast<int>(sk), SKV_F32, SKV_F32, 0, true);
    std::vector<float> kf(sk * D), vf(sk * D);
    for (std::size_t i = 0; i < sk * D; ++i) {
        kf[i] = static_cast<float>(k.data[i]);
        vf[i] = static_cast<float>(v.data[i]);
    }
    DeviceBuffer dk(kf.size() * 4), dv(vf.size() * 4), dq(D * 4), dout(D * 4), didx(sk * 4), dw(sk * 4);
    dk.upload(kf.data(), kf.size() * 4);
    dv.upload(vf.data(), vf.size() * 4);
    cache.append_tokens(0, 0, 1, 0, static_cast<int>(sk), dk.get(), dv.get());
    std::vector<int32_t> idx(sk);
    for (std::size_t i = 0; i < sk; ++i) idx[i] = static_cast<int32_t>(i);
    didx.upload(idx.data(), sk * 4);
    std::vector<float> qf(D), out(D), w(sk);
    for (std::size_t r = 0; r < sq; ++r) {
        const std::size_t n = causal ? r + 1 + static_cast<std::size_t>(off) : sk;
        for (std::size_t d = 0; d < D; ++d) qf[d] = static_cast<float>(q.at(r, d));
        dq.upload(qf.data(), D * 4);
        cache.attend_over_indices(0, static_cast<int>(n), didx.as<int32_t>(), static_cast<int>(n), dq.get(),
                                  dout.get(), dw.as<float>());
        dout.download(out.data(), D * 4);
        dw.download(w.data(), n * 4);
        for (std::size_t d = 0; d < v.cols; ++d) res.first.at(r, d) = out[d];
        for (std::size_t t = 0; t < n; ++t) res.second.at(r, t) = w[t];
    }
    return res;
}

// scheduler.hpp:320-381 on the reference's own types: the ledger row of
// `layer` and the selection go to a one-sequence device cache, the device
// kernel derives the four lists (the ones skv_swa_decode_step applies).
inline StepActions step_actions(const SchedulePlan& plan, std::size_t j, const SparseSelection& selection,
                                const KvLedger& ledger, std::size_t layer, const CostParams& p) {
    require(j < p.output_len, "step_actions: step beyond output length");
    require(layer < ledger.layers(), "KvLedger: layer out of range");
    const std::size_t cap = p.input_len + j + 1;
    DeviceCache cache(static_cast<int>(layer) + 1, 1, 1, 128, static_cast<int>(cap), SKV_F16, SKV_F16);
    skv_plan pl{plan.alpha, plan.beta, static_cast<int64_t>(plan.p1), static_cast<int64_t>(plan.p2),
                plan.recompute_enabled ? 1 : 0, static_cast<int64_t>(p.input_len),
                static_cast<int64_t>(p.output_len)};
    cache.set_plan(pl);
    std::vector<std::uint8_t> tiers(cap, 255);
    for (std::size_t t = 0; t < cap; ++t)
        if (ledger.exists(layer, t)) tiers[t] = static_cast<std::uint8_t>(ledger.tier(layer, t));
    cache.ledger_set(static_cast<int>(layer), 0, 1, static_cast<int>(cap), tiers.data());
    const IndexList all = selection.all();
    std::vector<int32_t> sel(all.begin(), all.end());
    DeviceBuffer dsel(std::max<std::size_t>(sel.size(), 1) * 4);
    if (!sel.empty()) dsel.upload(sel.data(), sel.size() * 4);
    std::vector<int32_t> lists(4 * cap), counts(4);
    cache.step_actions(static_cast<int>(layer), static_cast<int>(j), dsel.as<int32_t>(), static_cast<int>(sel.size()),
                       static_cast<int>(selection.k), false, lists.data(), counts.data());
    check(skv_stream_synchronize(nullptr));
    StepActions a;
    // phase_of_step (scheduler.hpp:52-60)
    a.phase = j < plan.p1 ? 1 : ((j < plan.p2 || !plan.recompute_enabled) ? 2 : 3);
    IndexList* out[4] = {&a.offload, &a.delete_tokens, &a.reload, &a.recompute};
    for (int l = 0; l < 4; ++l)
        for (int i = 0; i < counts[l]; ++i) out[l]->push_back(static_cast<std::size_t>(lists[l * cap + i]));
    return a;
}

}  // namespace skv::b200
