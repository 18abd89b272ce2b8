// C++ drop-in check: the reference `skv` functions vs their B200 mirrors in
// include/skv/b200.hpp, called with the reference's own types. Built against
// the unmodified reference headers (tests/cpp/Makefile); run by
// tests/test_cpp_shim.py on the GPU box. Exit 0 = parity.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "skv/attention.hpp"
#include "skv/b200.hpp"
#include "skv/quant.hpp"
#include "skv/scheduler.hpp"
#include "skv/memsim.hpp"

using namespace skv;

static int fails = 0;
#define CHECK(c, ...)                         \
    do {                                      \
        if (!(c)) {                           \
            std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);         \
            std::printf("\n");                \
            ++fails;                          \
        }                                     \
    } while (0)

static double rel_err(const Matrix& a, const Matrix& b) {
    double mx = 0, worst = 0;
    for (double x : b.data) mx = std::max(mx, std::abs(x));
    for (std::size_t i = 0; i < a.data.size(); ++i)
        worst = std::max(worst, std::abs(a.data[i] - b.data[i]) / (std::abs(b.data[i]) + mx));
    return worst;
}

int main() {
    SeededRng rng(2403);
    // top_k_indices / swa_select: bit-exact including ties
    for (int rep = 0; rep < 30; ++rep) {
        const std::size_t len = 1 + rng.integer(3000);
        Vector v(len);
        for (double& x : v) x = std::round(rng.uniform() * (rep % 2 ? 8.0 : 1e6)) / 8.0;
        const std::size_t k = rng.integer(len + 1);
        CHECK(top_k_indices(v, k) == b200::top_k_indices(v, k), "top_k len=%zu k=%zu", len, k);
        const std::size_t n = len + 1;
        for (double r : {0.05, 0.2, 0.7, 1.0}) {
            const SparseSelection a = swa_select(v, n, r), b = b200::swa_select(v, n, r);
            CHECK(a.k == b.k && a.local_indices == b.local_indices && a.global_indices == b.global_indices,
                  "swa_select n=%zu r=%g", n, r);
        }
    }
    // quantize / dequantize: bit-exact
    for (int rep = 0; rep < 10; ++rep) {
        Vector x(128 * 16);
        for (double& e : x) e = rng.normal() * (rep + 1);
        for (std::uint32_t bits : {4u, 8u}) {
            const QuantizedVector a = quantize(x, bits, 128), b = b200::quantize(x, bits, 128);
            CHECK(a.codes == b.codes && a.scales == b.scales && a.zero_points == b.zero_points, "quantize");
            CHECK(dequantize(a) == b200::dequantize(b), "dequantize");
        }
    }
    // swa_attention trajectory on the reference AttentionState type
    const std::size_t H = 4, D = 128, s = 200;
    AttentionState ref(H, D), dev(H, D);
    Matrix kr(H, D), vr(H, D), q(H, D);
    for (std::size_t t = 0; t < s; ++t) {
        for (double& x : kr.data) x = static_cast<float>(rng.normal());
        for (double& x : vr.data) x = static_cast<float>(rng.normal());
        ref.append_token(kr, vr);
        dev.append_token(kr, vr);
    }
    for (std::size_t h = 0; h < H; ++h) {
        ref.attention_accum[h].resize(s - 1);
        for (double& a : ref.attention_accum[h]) a = rng.uniform();
        dev.attention_accum[h] = ref.attention_accum[h];
    }
    SparsityConfig cfg;
    cfg.variant = AttentionVariant::Swa;
    cfg.ratio = 0.2;
    for (int step = 0; step < 10; ++step) {
        if (step > 0) {
            for (double& x : kr.data) x = static_cast<float>(rng.normal());
            for (double& x : vr.data) x = static_cast<float>(rng.normal());
            ref.append_token(kr, vr);
            dev.append_token(kr, vr);
        }
        for (double& x : q.data) x = static_cast<float>(rng.normal());
        const StepAttentionResult a = swa_attention(ref, q, cfg);
        const StepAttentionResult b = b200::swa_attention(dev, q, cfg);
        CHECK(a.selection.all() == b.selection.all(), "selection step %d", step);
        const double e = rel_err(b.attn, a.attn);
        CHECK(e <= 1e-5, "attn step %d rel err %g", step, e);
        double acc_err = 0;
        for (std::size_t h = 0; h < H; ++h)
            for (std::size_t i = 0; i < ref.attention_accum[h].size(); ++i)
                acc_err = std::max(acc_err, std::abs(ref.attention_accum[h][i] - dev.attention_accum[h][i]));
        CHECK(acc_err <= 1e-5, "accumulators step %d err %g", step, acc_err);
    }
    // dense_attention (attention.hpp:91-117): causal (bottom-right aligned,
    // :98-103) and full, square and non-square, fp32 device vs fp64
    for (bool causal : {true, false})
        for (std::size_t sq : {1, 17, 70})
            for (std::size_t sk : {70, 128}) {
                const std::size_t Dd = 128;
                Matrix qm(sq, Dd), km(sk, Dd), vm(sk, Dd);
                for (double& x : qm.data) x = static_cast<float>(rng.normal() * 0.5);
                for (double& x : km.data) x = static_cast<float>(rng.normal());
                for (double& x : vm.data) x = static_cast<float>(rng.normal());
                const auto a = dense_attention(qm, km, vm, causal);
                const auto b = b200::dense_attention(qm, km, vm, causal);
                const double e1 = rel_err(b.first, a.first);
                double e2 = 0;
                for (std::size_t i = 0; i < a.second.data.size(); ++i)
                    e2 = std::max(e2, std::abs(a.second.data[i] - b.second.data[i]));
                CHECK(e1 <= 1e-5 && e2 <= 1e-5, "dense_attention causal=%d sq=%zu sk=%zu attn %g aw %g", causal, sq,
                      sk, e1, e2);
            }
    // dense_attention contract: empty input and a causal row with no key throw
    // the reference's ContractViolation
    {
        const Matrix e0(0, 128), k1(5, 128), q9(9, 128);
        for (int which = 0; which < 3; ++which) {
            int ref_threw = 0, dev_threw = 0;
            const Matrix& qq = which == 2 ? q9 : (which == 0 ? e0 : k1);
            const Matrix& kk = which == 1 ? e0 : k1;
            const Matrix& vv = which == 1 ? e0 : k1;
            try {
                dense_attention(qq, kk, vv, true);
            } catch (const ContractViolation&) {
                ref_threw = 1;
            }
            try {
                b200::dense_attention(qq, kk, vv, true);
            } catch (const ContractViolation&) {
                dev_threw = 1;
            }
            CHECK(ref_threw == 1 && dev_threw == 1, "dense_attention contract case %d: ref %d dev %d", which,
                  ref_threw, dev_threw);
        }
    }
    // attend_over_indices (attention.hpp:183-231) with unsorted and repeated
    // indices: every occurrence is a softmax term and adds its own weight
    for (int rep = 0; rep < 6; ++rep) {
        AttentionState ra(H, D), da(H, D);
        const std::size_t nt = 90 + rng.integer(60);
        for (std::size_t t = 0; t < nt; ++t) {
            for (double& x : kr.data) x = static_cast<float>(rng.normal());
            for (double& x : vr.data) x = static_cast<float>(rng.normal());
            ra.append_token(kr, vr);
            da.append_token(kr, vr);
        }
        for (std::size_t h = 0; h < H; ++h) {
            ra.attention_accum[h].assign(nt - 1 - rep % 3, 0.0);
            for (double& a : ra.attention_accum[h]) a = rng.uniform();
            da.attention_accum[h] = ra.attention_accum[h];
        }
        IndexList idx;
        const std::size_t m = 5 + rng.integer(40);
        for (std::size_t i = 0; i < m; ++i) idx.push_back(rng.integer(nt));
        if (rep % 2 == 0) idx.push_back(idx.front());  // a guaranteed repeat
        for (double& x : q.data) x = static_cast<float>(rng.normal());
        const StepAttentionResult a = attend_over_indices(ra, q, idx);
        const StepAttentionResult b = b200::attend_over_indices(da, q, idx);
        const double e = rel_err(b.attn, a.attn);
        double acc_err = 0, row_err = 0;
        for (std::size_t h = 0; h < H; ++h) {
            CHECK(ra.attention_accum[h].size() == da.attention_accum[h].size(), "acc size rep %d", rep);
            for (std::size_t i = 0; i < ra.attention_accum[h].size(); ++i)
                acc_err = std::max(acc_err, std::abs(ra.attention_accum[h][i] - da.attention_accum[h][i]));
        }
        for (std::size_t i = 0; i < a.new_aw_row.size(); ++i)
            row_err = std::max(row_err, std::abs(a.new_aw_row[i] - b.new_aw_row[i]));
        CHECK(e <= 1e-5 && acc_err <= 1e-5 && row_err <= 1e-5 && a.new_aw_row.size() == b.new_aw_row.size(),
              "attend_over_indices unsorted/repeated rep %d: attn %g acc %g row %g", rep, e, acc_err, row_err);
    }
    // step_actions (scheduler.hpp:320-381) on the reference KvLedger / SchedulePlan
    for (int rep = 0; rep < 40; ++rep) {
        CostParams cp;
        cp.hidden = 64;
        cp.layers = 2;
        cp.batch = 1;
        cp.input_len = 60 + rng.integer(60);
        cp.output_len = 40;
        cp.ratio = 0.2;
        cp.device_capacity = 1ull << 40;
        const std::size_t j = rng.integer(cp.output_len);
        const std::size_t layer = rng.integer(2);
        const std::size_t existing = cp.input_len + j;
        KvLedger ledger(2, cp.device_capacity);
        for (std::size_t t = 0; t < existing; ++t) ledger.store_new(layer, t, 64);
        IndexList off, del;
        for (std::size_t t = 0; t < existing; ++t) {
            const double u = rng.uniform();
            if (u < 0.3) off.push_back(t);
        }
        ledger.offload(layer, off);
        for (const std::size_t t : off)
            if (rng.uniform() < 0.3) del.push_back(t);
        ledger.erase(layer, del);
        SchedulePlan plan;
        // valid plans only (validate_plan, scheduler.hpp:41-49): pure device, or 0 <= p1 < p2 <= n
        plan.alpha = 0.05 + rng.uniform() * 0.6;
        plan.beta = 0.05 + rng.uniform() * 0.5;
        if (rep % 8 == 0) {
            plan.p1 = plan.p2 = cp.output_len;
        } else {
            plan.p1 = rng.integer(cp.output_len);
            plan.p2 = plan.p1 + 1 + rng.integer(cp.output_len - plan.p1);
        }
        plan.recompute_enabled = rep % 3 != 0;
        Vector imp(existing);
        for (double& x : imp) x = rng.uniform();
        const SparseSelection sel = swa_select(imp, existing + 1, 0.2);
        const StepActions a = step_actions(plan, j, sel, ledger, layer, cp);
        const StepActions b = b200::step_actions(plan, j, sel, ledger, layer, cp);
        CHECK(a.phase == b.phase && a.offload == b.offload && a.delete_tokens == b.delete_tokens &&
                  a.reload == b.reload && a.recompute == b.recompute,
              "step_actions rep %d (phase %d/%d, offload %zu/%zu, delete %zu/%zu, reload %zu/%zu, recompute %zu/%zu)",
              rep, a.phase, b.phase, a.offload.size(), b.offload.size(), a.delete_tokens.size(),
              b.delete_tokens.size(), a.reload.size(), b.reload.size(), a.recompute.size(), b.recompute.size());
    }
    // error semantics: reference exception classes
    bool threw = false;
    try {
        b200::attend_over_indices(dev, q, IndexList{0, dev.tokens()});
    } catch (const ContractViolation&) {
        threw = true;
    }
    CHECK(threw, "index out of range must throw ContractViolation");
    threw = false;
    try {
        b200::swa_window_k(10, 1.5);
    } catch (const ContractViolation&) {
        threw = true;
    }
    CHECK(threw, "ratio out of range must throw ContractViolation");
    std::printf(fails ? "FAILED %d\n" : "ALL OK\n", fails);
    return fails ? 1 : 0;
}
