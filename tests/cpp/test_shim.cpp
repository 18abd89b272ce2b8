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
