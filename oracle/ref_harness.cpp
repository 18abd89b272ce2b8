// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI over the UNMODIFIED reference library, compiled straight from the
// read-only headers in /root/reference/proj/include (see oracle/Makefile; the
// output goes to oracle/_ref/ only). It exists to (1) pin the C restatement in
// skv_oracle.c bit-for-bit against the reference itself, (2) generate the
// golden fixtures under tests/golden/, and (3) serve as bench.py's
// `--impl reference` CPU arm. No reference source is copied here: every
// function below only marshals arrays into the reference's own types and
// calls the reference function named in its comment.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "skv/attention.hpp"
#include "skv/common.hpp"
#include "skv/matrix.hpp"
#include "skv/memsim.hpp"
#include "skv/quant.hpp"
#include "skv/scheduler.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const skv::ContractViolation& e) {
        g_err = e.what();
        return 1;
    } catch (const skv::OutOfDeviceMemory& e) {
        g_err = e.what();
        return 2;
    } catch (const skv::InfeasiblePlan& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

skv::AttentionState make_state(size_t H, size_t D, size_t n, size_t ncap, const double* keys,
                               const double* values, const double* acc, size_t acc_ld,
                               size_t acc_len) {
    skv::AttentionState st(H, D);
    for (size_t h = 0; h < H; ++h) {
        for (size_t t = 0; t < n; ++t) {
            st.keys[h].append_row({keys + (h * ncap + t) * D, D});
            st.values[h].append_row({values + (h * ncap + t) * D, D});
        }
        st.attention_accum[h].assign(acc + h * acc_ld, acc + h * acc_ld + acc_len);
    }
    return st;
}

void copy_idx(const skv::IndexList& v, int64_t* out) {
    for (size_t i = 0; i < v.size(); ++i) out[i] = static_cast<int64_t>(v[i]);
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int64_t ref_round_half_even(double x) { return skv::round_half_even(x); }

// matrix.hpp SeededRng
void ref_fill_normal(uint64_t seed, double gain, double* out, size_t n) {
    skv::SeededRng rng(seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng.normal() * gain;
}
void ref_fill_u64(uint64_t seed, uint64_t* out, size_t n) {
    skv::SeededRng rng(seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}
void ref_fill_uniform(uint64_t seed, double* out, size_t n) {
    skv::SeededRng rng(seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng.uniform();
}

// attention.hpp:122-138
size_t ref_swa_window_k(size_t n, double r) {
    size_t k = 0;
    guarded([&] { k = skv::swa_window_k(n, r); });
    return k;
}
size_t ref_swa_keep_count(size_t n, double r) {
    size_t k = 0;
    guarded([&] { k = skv::swa_keep_count(n, r); });
    return k;
}

// matrix.hpp:162-176
int ref_top_k_indices(const double* v, size_t len, size_t k, int64_t* out) {
    return guarded([&] { copy_idx(skv::top_k_indices({v, len}, k), out); });
}

// attention.hpp:142-171 (+ SparseSelection::all)
int ref_swa_select(const double* importance, size_t importance_len, size_t n, double r,
                   int64_t* out_all, size_t* m_out, size_t* k_out, int64_t* out_local,
                   size_t* n_local, int64_t* out_global, size_t* n_global) {
    return guarded([&] {
        const skv::SparseSelection sel = skv::swa_select({importance, importance_len}, n, r);
        const skv::IndexList all = sel.all();
        copy_idx(all, out_all);
        if (m_out) *m_out = all.size();
        if (k_out) *k_out = sel.k;
        if (out_local) copy_idx(sel.local_indices, out_local);
        if (n_local) *n_local = sel.local_indices.size();
        if (out_global) copy_idx(sel.global_indices, out_global);
        if (n_global) *n_global = sel.global_indices.size();
    });
}

// attention.hpp:183-231. acc in/out [H][acc_ld]; acc_len = current length.
int ref_attend_over_indices(size_t H, size_t D, size_t n, size_t ncap, const double* keys,
                            const double* values, double* acc, size_t acc_ld, size_t acc_len,
                            const double* q, const int64_t* idx, size_t m, double* attn,
                            double* new_aw_row) {
    return guarded([&] {
        skv::AttentionState st = make_state(H, D, n, ncap, keys, values, acc, acc_ld, acc_len);
        skv::Matrix qm(H, D);
        std::memcpy(qm.data.data(), q, H * D * sizeof(double));
        skv::IndexList sel(idx, idx + m);
        for (size_t i = 0; i < m; ++i) sel[i] = static_cast<size_t>(idx[i]);
        const skv::StepAttentionResult res = skv::attend_over_indices(st, qm, sel);
        std::memcpy(attn, res.attn.data.data(), H * D * sizeof(double));
        std::memcpy(new_aw_row, res.new_aw_row.data(), res.new_aw_row.size() * sizeof(double));
        for (size_t h = 0; h < H; ++h)
            std::memcpy(acc + h * acc_ld, st.attention_accum[h].data(),
                        st.attention_accum[h].size() * sizeof(double));
    });
}

// attention.hpp:235-244
int ref_swa_attention(size_t H, size_t D, size_t n, size_t ncap, const double* keys,
                      const double* values, double* acc, size_t acc_ld, const double* q,
                      double r, double* attn, double* new_aw_row, int64_t* idx_out,
                      size_t* m_out) {
    return guarded([&] {
        skv::AttentionState st = make_state(H, D, n, ncap, keys, values, acc, acc_ld, n - 1);
        skv::Matrix qm(H, D);
        std::memcpy(qm.data.data(), q, H * D * sizeof(double));
        skv::SparsityConfig cfg;
        cfg.variant = skv::AttentionVariant::Swa;
        cfg.ratio = r;
        const skv::StepAttentionResult res = skv::swa_attention(st, qm, cfg);
        std::memcpy(attn, res.attn.data.data(), H * D * sizeof(double));
        std::memcpy(new_aw_row, res.new_aw_row.data(), res.new_aw_row.size() * sizeof(double));
        const skv::IndexList all = res.selection.all();
        copy_idx(all, idx_out);
        if (m_out) *m_out = all.size();
        for (size_t h = 0; h < H; ++h)
            std::memcpy(acc + h * acc_ld, st.attention_accum[h].data(),
                        st.attention_accum[h].size() * sizeof(double));
    });
}

// attention.hpp:247-269
size_t ref_local_attention_mask(size_t n, size_t window, int64_t* out) {
    size_t c = 0;
    guarded([&] {
        const skv::IndexList l = skv::local_attention_mask(n, window);
        copy_idx(l, out);
        c = l.size();
    });
    return c;
}
size_t ref_strided_attention_mask(size_t n, size_t stride, int64_t* out) {
    size_t c = 0;
    guarded([&] {
        const skv::IndexList l = skv::strided_attention_mask(n, stride);
        copy_idx(l, out);
        c = l.size();
    });
    return c;
}
// attention.hpp:275-310
double ref_attention_sparsity(size_t rows, size_t cols, const double* aw, double rel, int causal) {
    double r = -1.0;
    guarded([&] {
        skv::Matrix m(rows, cols);
        std::memcpy(m.data.data(), aw, rows * cols * sizeof(double));
        r = skv::attention_sparsity(m, rel, causal != 0);
    });
    return r;
}

// matrix.hpp:137-158
int ref_softmax_rows(size_t rows, size_t cols, const double* in, double* out) {
    return guarded([&] {
        skv::Matrix m(rows, cols);
        std::memcpy(m.data.data(), in, rows * cols * sizeof(double));
        const skv::Matrix s = skv::softmax_rows(m);
        std::memcpy(out, s.data.data(), rows * cols * sizeof(double));
    });
}

// attention.hpp:91-117
int ref_dense_attention(size_t sq, size_t sk, size_t D, const double* q, const double* k,
                        const double* v, int causal, double* attn, double* aw) {
    return guarded([&] {
        skv::Matrix qm(sq, D), km(sk, D), vm(sk, D);
        std::memcpy(qm.data.data(), q, sq * D * sizeof(double));
        std::memcpy(km.data.data(), k, sk * D * sizeof(double));
        std::memcpy(vm.data.data(), v, sk * D * sizeof(double));
        auto [a, w] = skv::dense_attention(qm, km, vm, causal != 0);
        std::memcpy(attn, a.data.data(), sq * D * sizeof(double));
        std::memcpy(aw, w.data.data(), sq * sk * sizeof(double));
    });
}

// quant.hpp:43-81
int ref_quantize(const double* x, size_t len, uint32_t bits, size_t channel_size,
                 uint16_t* codes, double* scales, int64_t* zero_points) {
    return guarded([&] {
        const skv::QuantizedVector qv = skv::quantize({x, len}, bits, channel_size);
        std::memcpy(codes, qv.codes.data(), qv.codes.size() * sizeof(uint16_t));
        std::memcpy(scales, qv.scales.data(), qv.scales.size() * sizeof(double));
        std::memcpy(zero_points, qv.zero_points.data(), qv.zero_points.size() * sizeof(int64_t));
    });
}

// quant.hpp:84-95
int ref_dequantize(const uint16_t* codes, size_t len, size_t channel_size, const double* scales,
                   const int64_t* zero_points, double* out) {
    return guarded([&] {
        skv::QuantizedVector qv;
        qv.codes.assign(codes, codes + len);
        qv.channel_size = channel_size;
        const size_t g = len / channel_size;
        qv.scales.assign(scales, scales + g);
        qv.zero_points.assign(zero_points, zero_points + g);
        const skv::Vector x = skv::dequantize(qv);
        std::memcpy(out, x.data(), len * sizeof(double));
    });
}

// scheduler.hpp:320-381 over a KvLedger rebuilt from per-token tiers
// (tier: -1 absent, 0 device, 1 host, 2 deleted) for one layer.
int ref_step_actions(double alpha, double beta, size_t p1, size_t p2, int recompute_enabled,
                     size_t j, const int64_t* selected, size_t m, size_t k,
                     const int8_t* tiers, size_t ntok, size_t layers, size_t layer,
                     size_t input_len, size_t output_len, int* phase, int64_t* offload,
                     size_t* n_off, int64_t* del, size_t* n_del, int64_t* reload,
                     size_t* n_rel, int64_t* recompute, size_t* n_rec) {
    return guarded([&] {
        skv::SchedulePlan plan;
        plan.alpha = alpha;
        plan.beta = beta;
        plan.p1 = p1;
        plan.p2 = p2;
        plan.recompute_enabled = recompute_enabled != 0;
        skv::CostParams p;
        p.hidden = 1;
        p.layers = layers;
        p.input_len = input_len;
        p.output_len = output_len;
        skv::KvLedger ledger(layers, std::numeric_limits<uint64_t>::max() / 4);
        for (size_t t = 0; t < ntok; ++t) {
            if (tiers[t] < 0) continue;
            ledger.store_new(layer, t, 1);
            const size_t one[1] = {t};
            if (tiers[t] == 1) ledger.offload(layer, one);
            if (tiers[t] == 2) ledger.erase(layer, one);
        }
        skv::SparseSelection sel;
        sel.k = k;
        for (size_t i = 0; i < m; ++i) sel.local_indices.push_back(static_cast<size_t>(selected[i]));
        const skv::StepActions a = skv::step_actions(plan, j, sel, ledger, layer, p);
        *phase = a.phase;
        copy_idx(a.offload, offload);
        *n_off = a.offload.size();
        copy_idx(a.delete_tokens, del);
        *n_del = a.delete_tokens.size();
        copy_idx(a.reload, reload);
        *n_rel = a.reload.size();
        copy_idx(a.recompute, recompute);
        *n_rec = a.recompute.size();
    });
}

// scheduler.hpp:207-303 solve_plan. plan_out = {alpha, beta, p1, p2};
// pred_out = {total, prefill, compute[3], transfer[3], recompute[3], steps[3]}.
int ref_solve_plan(size_t hidden, size_t layers, size_t batch, size_t input_len, size_t output_len,
                   double ratio, double bandwidth, size_t bpe, uint64_t capacity, double mac_rate,
                   double overhead, double* plan_out, double* pred_out) {
    return guarded([&] {
        skv::CostParams p;
        p.hidden = hidden;
        p.layers = layers;
        p.batch = batch;
        p.input_len = input_len;
        p.output_len = output_len;
        p.ratio = ratio;
        p.bandwidth = bandwidth;
        p.bytes_per_element = bpe;
        p.device_capacity = capacity;
        p.mac_rate = mac_rate;
        p.recompute_overhead = overhead;
        const skv::SchedulePlan plan = skv::solve_plan(p);
        plan_out[0] = plan.alpha;
        plan_out[1] = plan.beta;
        plan_out[2] = static_cast<double>(plan.p1);
        plan_out[3] = static_cast<double>(plan.p2);
        pred_out[0] = plan.predicted_total_seconds;
        pred_out[1] = plan.prefill_compute_seconds;
        for (int i = 0; i < 3; ++i) {
            pred_out[2 + i] = plan.phases[i].compute_seconds;
            pred_out[5 + i] = plan.phases[i].transfer_seconds;
            pred_out[8 + i] = plan.phases[i].recompute_seconds;
            pred_out[11 + i] = static_cast<double>(plan.phases[i].steps);
        }
    });
}

// CPU timing arm: share-nothing threads, one AttentionState per worker. Each
// work item = append one token then skv::swa_attention (one (sequence, layer)
// decode step). Items run in rounds of up to 16 at n = n0 .. n0+15; between
// rounds the state's tail is trimmed back to n0-1 tokens (untimed), so every
// timed item runs at the requested length. Returns the slowest worker's
// timed (busy) seconds.
double ref_bench_swa(size_t H, size_t D, size_t n0, double r, size_t items, size_t threads,
                     uint64_t seed) {
    if (threads == 0) threads = 1;
    std::atomic<size_t> ready{0};
    std::atomic<bool> go{false};
    std::vector<double> busy(threads, 0.0);
    std::vector<std::thread> pool;
    using clk = std::chrono::steady_clock;
    for (size_t w = 0; w < threads; ++w) {
        const size_t share = items / threads + (w < items % threads ? 1 : 0);
        pool.emplace_back([&, w, share] {
            skv::SeededRng rng(seed + 7919u * w);
            skv::AttentionState st(H, D);
            skv::Matrix kr(H, D), vr(H, D);
            std::vector<skv::Matrix> kin(16, skv::Matrix(H, D)), vin(16, skv::Matrix(H, D)),
                qin(16, skv::Matrix(H, D));
            for (size_t t = 0; t + 1 < n0; ++t) {
                for (double& x : kr.data) x = rng.normal();
                for (double& x : vr.data) x = rng.normal();
                st.append_token(kr, vr);
            }
            std::vector<skv::Vector> acc0(H, skv::Vector(n0 - 1));
            for (size_t h = 0; h < H; ++h)
                for (double& a : acc0[h]) a = rng.uniform();
            skv::SparsityConfig cfg;
            cfg.variant = skv::AttentionVariant::Swa;
            cfg.ratio = r;
            ready.fetch_add(1);
            while (!go.load()) std::this_thread::yield();
            for (size_t done = 0; done < share;) {
                for (size_t h = 0; h < H; ++h) {  // trim back to n0-1 tokens (untimed)
                    st.keys[h].rows = n0 - 1;
                    st.keys[h].data.resize((n0 - 1) * D);
                    st.values[h].rows = n0 - 1;
                    st.values[h].data.resize((n0 - 1) * D);
                    st.attention_accum[h] = acc0[h];
                }
                const size_t cnt = std::min<size_t>(16, share - done);
                for (size_t it = 0; it < cnt; ++it) {  // the round's inputs (untimed)
                    for (double& x : kin[it].data) x = rng.normal();
                    for (double& x : vin[it].data) x = rng.normal();
                    for (double& x : qin[it].data) x = rng.normal();
                }
                const auto t0 = clk::now();
                for (size_t it = 0; it < cnt; ++it) {
                    st.append_token(kin[it], vin[it]);
                    (void)skv::swa_attention(st, qin[it], cfg);
                }
                busy[w] += std::chrono::duration<double>(clk::now() - t0).count();
                done += cnt;
            }
        });
    }
    while (ready.load() < threads) std::this_thread::yield();
    go.store(true);
    for (auto& t : pool) t.join();
    double b = 0.0;
    for (double x : busy) b = std::max(b, x);
    return b;
}

// memsim.hpp:77-215: a live reference KvLedger behind an opaque handle, so
// the tests can drive it with the same action sequence as the device ledger
// and compare byte totals and the OutOfDeviceMemory point and message.
void* ref_ledger_new(size_t layers, uint64_t capacity) {
    skv::KvLedger* l = nullptr;
    guarded([&] { l = new skv::KvLedger(layers, capacity); });
    return l;
}
void ref_ledger_free(void* h) { delete static_cast<skv::KvLedger*>(h); }
// op: 0 store_new (each token), 1 offload, 2 reload, 3 erase, 4 restore (each token)
int ref_ledger_op(void* h, int op, size_t layer, const int64_t* toks, size_t nt, uint64_t bytes) {
    auto& L = *static_cast<skv::KvLedger*>(h);
    return guarded([&] {
        std::vector<std::size_t> t(toks, toks + nt);
        switch (op) {
        case 0:
            for (std::size_t x : t) L.store_new(layer, x, bytes);
            break;
        case 1: L.offload(layer, t); break;
        case 2: L.reload(layer, t); break;
        case 3: L.erase(layer, t); break;
        case 4:
            for (std::size_t x : t) L.restore(layer, x, bytes);
            break;
        default: throw std::runtime_error("ref_ledger_op: unknown op");
        }
    });
}
void ref_ledger_bytes(void* h, uint64_t* device_bytes, uint64_t* host_bytes) {
    auto& L = *static_cast<skv::KvLedger*>(h);
    *device_bytes = L.device_bytes();
    *host_bytes = L.host_bytes();
}
// tiers of tokens [0, ntok) of `layer`: -1 not stored, else Tier
void ref_ledger_tiers(void* h, size_t layer, size_t ntok, int8_t* out) {
    auto& L = *static_cast<skv::KvLedger*>(h);
    for (size_t t = 0; t < ntok; ++t)
        out[t] = L.exists(layer, t) ? static_cast<int8_t>(L.tier(layer, t)) : static_cast<int8_t>(-1);
}

} // extern "C"
