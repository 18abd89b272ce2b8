// End-to-end parity of the GPU toy engine (include/skv/b200_engine.hpp,
// SURVEY §8 f4) with the unmodified reference skv::Engine (engine.hpp:214-742)
// on the same RunConfig, plus the cached-vs-no-cache oracle
// (tests/oracles.hpp:196-265 logits_from_scratch). The GPU run's metrics are
// written with the reference's own report.hpp as skvsim.metrics.v1 JSON and
// skvsim.steps.v1 CSV (argv[1] = output directory, optional). Exit 0 = parity.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>

#include "oracles.hpp"
#include "skv/b200_engine.hpp"
#include "skv/config.hpp"
#include "skv/engine.hpp"
#include "skv/report.hpp"

using namespace skv;

static int fails = 0;
#define CHECK(c, ...)                                       \
    do {                                                    \
        if (!(c)) {                                         \
            std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                       \
            std::printf("\n");                              \
            ++fails;                                        \
        }                                                   \
    } while (0)

static bool close(double a, double b, double rel, double abs_) {
    return std::abs(a - b) <= abs_ + rel * std::max(std::abs(a), std::abs(b));
}

static RunConfig base_config() {
    RunConfig c;
    c.shape.layers = 2;
    c.shape.heads = 8;
    c.shape.head_dim = 128;
    c.shape.vocab = 96;
    c.shape.ffn_mult = 2;
    c.skewed_init = true;
    c.batch = 4;
    c.prompt_len = 40;
    c.gen_len = 24;
    c.seed = 2403;
    c.bandwidth = 2e9;
    c.mac_rate = 5e11;
    return c;
}

// Engine::run on both sides with teacher forcing from the reference's own
// generated ids (so one near-tie argmax cannot fork the trajectories), then
// every StepMetrics field.
static void compare_runs(const char* name, const RunConfig& rc, const std::string& outdir) {
    const EngineConfig ec = rc.engine_config();
    Engine ref(ec);
    const RunMetrics a = ref.run();
    RunOptions forced;
    forced.forced_tokens = a.generated_ids;
    forced.record_mean_logits = true;
    Engine ref2(ec);
    const RunMetrics a2 = ref2.run(forced);
    b200::Engine dev(ec);
    const RunMetrics b = dev.run(forced);
    RunOptions free_run;
    b200::Engine dev_free(ec);
    const RunMetrics bf = dev_free.run(free_run);
    CHECK(bf.generated_ids == a.generated_ids, "%s: free-running GPU engine generated other tokens", name);
    CHECK(ref.plan().p1 == dev.plan().p1 && ref.plan().p2 == dev.plan().p2 && ref.plan().alpha == dev.plan().alpha &&
              ref.plan().beta == dev.plan().beta,
          "%s: plan differs", name);
    CHECK(a2.steps.size() == b.steps.size(), "%s: step count %zu vs %zu", name, a2.steps.size(), b.steps.size());
    int phases[4] = {0, 0, 0, 0};
    for (std::size_t j = 0; j < std::min(a2.steps.size(), b.steps.size()); ++j) {
        const StepMetrics &x = a2.steps[j], &y = b.steps[j];
        ++phases[x.phase];
        CHECK(x.phase == y.phase && x.token_id == y.token_id && x.kept_tokens == y.kept_tokens &&
                  x.device_bytes == y.device_bytes && x.host_bytes == y.host_bytes && x.recomputed == y.recomputed &&
                  x.deleted == y.deleted,
              "%s step %zu: phase %d/%d kept %zu/%zu dev %llu/%llu host %llu/%llu rec %zu/%zu del %zu/%zu", name, j,
              x.phase, y.phase, x.kept_tokens, y.kept_tokens, (unsigned long long)x.device_bytes,
              (unsigned long long)y.device_bytes, (unsigned long long)x.host_bytes, (unsigned long long)y.host_bytes,
              x.recomputed, y.recomputed, x.deleted, y.deleted);
        CHECK(close(x.compute_seconds, y.compute_seconds, 1e-12, 0) &&
                  close(x.transfer_seconds, y.transfer_seconds, 1e-12, 1e-300) &&
                  close(x.recompute_seconds, y.recompute_seconds, 1e-12, 1e-300) &&
                  close(x.d2h_tokens, y.d2h_tokens, 1e-12, 1e-300) && close(x.h2d_tokens, y.h2d_tokens, 1e-12, 1e-300),
              "%s step %zu: cost-model seconds / tokens differ", name, j);
        const double n = static_cast<double>(rc.prompt_len + j + 1);
        for (std::size_t l = 0; l < x.sparsity_per_layer.size(); ++l)
            CHECK(std::abs(x.sparsity_per_layer[l] - y.sparsity_per_layer[l]) <= 1.0 / n + 1e-12,
                  "%s step %zu layer %zu: sparsity %g vs %g", name, j, l, x.sparsity_per_layer[l],
                  y.sparsity_per_layer[l]);
    }
    for (std::size_t l = 0; l < a2.prefill_sparsity_per_layer.size(); ++l)
        CHECK(std::abs(a2.prefill_sparsity_per_layer[l] - b.prefill_sparsity_per_layer[l]) <= 1e-3,
              "%s prefill sparsity layer %zu: %g vs %g", name, l, a2.prefill_sparsity_per_layer[l],
              b.prefill_sparsity_per_layer[l]);
    double worst = 0.0, scale = 0.0;
    for (double v : a2.mean_logits) scale = std::max(scale, std::abs(v));
    for (std::size_t v = 0; v < a2.mean_logits.size(); ++v)
        worst = std::max(worst, std::abs(a2.mean_logits[v] - b.mean_logits[v]) / (scale + 1e-30));
    CHECK(worst <= 1e-4, "%s: mean logits rel err %g", name, worst);
    CHECK(a2.peak_device_bytes == b.peak_device_bytes && a2.peak_host_bytes == b.peak_host_bytes &&
              close(a2.total_seconds, b.total_seconds, 1e-12, 0) && a2.transferred_bytes == b.transferred_bytes,
          "%s: run totals differ", name);
    std::printf("%s: %zu steps (phases I/II/III: %d/%d/%d), mean-logit rel err %.2e, peak device %llu B\n", name,
                b.steps.size(), phases[1], phases[2], phases[3], worst, (unsigned long long)b.peak_device_bytes);
    if (!outdir.empty()) {
        std::ofstream(outdir + "/engine_" + name + "_steps.csv") << steps_csv(b);
        std::ofstream(outdir + "/engine_" + name + "_metrics.json") << metrics_to_json(b, rc).dump(1) << "\n";
    }
}

int main(int argc, char** argv) {
    const std::string outdir = argc > 1 ? argv[1] : "";
    {   // SWA r = 0.3, the dynamic plan under a device budget: Phases I-III
        // (a fast recompute rate makes solve_plan choose deletion + recomputation)
        RunConfig c = base_config();
        c.sparsity.variant = AttentionVariant::Swa;
        c.sparsity.ratio = 0.3;
        c.bandwidth = 1e9;
        c.mac_rate = 2e13;
        const CostParams p = c.cost_params();
        c.device_capacity = token_kv_bytes(p) * (c.prompt_len + 6);
        compare_runs("swa_3phase", c, outdir);
    }
    {   // SWA r = 0.3 with the dynamic plan: Phases I-II
        RunConfig c = base_config();
        c.sparsity.variant = AttentionVariant::Swa;
        c.sparsity.ratio = 0.3;
        const CostParams p = c.cost_params();
        c.device_capacity = token_kv_bytes(p) * (c.prompt_len + 4);
        compare_runs("swa_dynamic", c, outdir);
    }
    {   // Dense (r = 1): every token kept, all on device
        RunConfig c = base_config();
        c.sparsity.variant = AttentionVariant::Dense;
        c.mode = ScheduleMode::AllDevice;
        compare_runs("dense", c, outdir);
    }
    {   // INT8 KV (quant.enabled: head_rows fake-quant), static split
        RunConfig c = base_config();
        c.sparsity.variant = AttentionVariant::Swa;
        c.sparsity.ratio = 0.5;
        c.quant.enabled = true;
        c.mode = ScheduleMode::StaticSplit;
        c.static_fraction = 0.4;
        compare_runs("swa_int8_static", c, outdir);
    }
    {   // Local and Strided variants, all on device
        RunConfig c = base_config();
        c.mode = ScheduleMode::AllDevice;
        c.sparsity.variant = AttentionVariant::Local;
        c.sparsity.ratio = 0.25;
        compare_runs("local", c, outdir);
        c.sparsity.variant = AttentionVariant::Strided;
        c.sparsity.stride = 3;
        compare_runs("strided", c, outdir);
    }
    {   // cached vs no-cache (oracles.hpp:196-265): the dense-attention decode
        // through the GPU cache reproduces the from-scratch forward's logits
        RunConfig c = base_config();
        c.sparsity.variant = AttentionVariant::Dense;
        c.mode = ScheduleMode::AllDevice;
        c.gen_len = 8;
        const EngineConfig ec = c.engine_config();
        b200::Engine dev(ec);
        RunOptions o;
        o.record_mean_logits = true;
        const RunMetrics m = dev.run(o);
        std::vector<std::int64_t> tokens = m.prompt_ids;
        Vector mean(c.shape.vocab, 0.0);
        for (std::size_t j = 0; j < m.generated_ids.size(); ++j) {
            tokens.push_back(m.generated_ids[j]);
            const Vector lg = oracle::logits_from_scratch(dev.model(), tokens);
            for (std::size_t v = 0; v < mean.size(); ++v) mean[v] += lg[v] / static_cast<double>(m.generated_ids.size());
        }
        double worst = 0.0, scale = 0.0;
        for (double v : mean) scale = std::max(scale, std::abs(v));
        for (std::size_t v = 0; v < mean.size(); ++v)
            worst = std::max(worst, std::abs(mean[v] - m.mean_logits[v]) / (scale + 1e-30));
        CHECK(worst <= 1e-4, "cached vs from-scratch logits rel err %g", worst);
        std::printf("cached_vs_no_cache: %zu steps, mean-logit rel err %.2e\n", m.generated_ids.size(), worst);
    }
    {   // OutOfDeviceMemory: the engine throws the reference's error at the same point
        RunConfig c = base_config();
        c.mode = ScheduleMode::AllDevice;
        const CostParams p = c.cost_params();
        c.device_capacity = token_kv_bytes(p) * (c.prompt_len + 3);
        std::string ra, rb;
        try {
            Engine(c.engine_config()).run();
        } catch (const OutOfDeviceMemory& e) {
            ra = e.what();
        }
        try {
            b200::Engine(c.engine_config()).run();
        } catch (const OutOfDeviceMemory& e) {
            rb = e.what();
        }
        CHECK(!ra.empty() && ra == rb, "OOM: reference '%s' vs gpu '%s'", ra.c_str(), rb.c_str());
    }
    std::printf(fails ? "FAILED %d\n" : "ALL OK\n", fails);
    return fails ? 1 : 0;
}
