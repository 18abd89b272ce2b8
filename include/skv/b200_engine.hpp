// skv/b200_engine.hpp -- skv::b200::Engine: the reference's toy-transformer
// engine (engine.hpp:214-742, skv::Engine) with every step on the GPU.
//
// Same constructor, run() and metrics (skv::RunMetrics / StepMetrics, so the
// reference's report.hpp writes skvsim.steps.v1 / skvsim.metrics.v1 from
// them unchanged). Per decode step and layer, in the reference's order
// (engine.hpp:592-684):
//   embed_one -> LayerNorm -> q/k/v projections            (skv_engine_*, fp64)
//   variant_selection + step_actions + apply_actions        (skv_decode_prepare,
//                                                            device select + ledger)
//   append (fake-quant for INT8) + attend over the selection (skv_swa_decode_layer)
//   attention_sparsity of the step row                      (folded in the select)
//   Wo + residual, LayerNorm, FFN (GELU) + residual, logits (skv_engine_*, fp64)
// The prefill runs the dense causal attention of the prompt on the GPU, caches
// the prompt K/V, seeds the importance with the last attention row and
// records the prefill sparsity (engine.hpp:485-529).
//
// Like the reference (a simulator of the memory hierarchy: memsim.hpp), the
// engine keeps the ledger's tiers and byte totals on the device and leaves
// the K/V rows resident; the real PCIe movement, slot reclamation and
// recomputation are the cache's host tier / paged store (skv_b200.h).
// Precision: fp64 dense operators as in the reference; the attention cache is
// fp32 (INT8 codes when quant is enabled), so logits agree within ~1e-6.
// head_dim must be 128 (the compiled attention kernels).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "skv/b200.hpp"
#include "skv/engine.hpp"

namespace skv::b200 {

class Engine {
  public:
    explicit Engine(const EngineConfig& cfg) : cfg_(cfg) {
        cfg_.cost.validate();
        cfg_.validate();
        if (cfg_.shape.head_dim != 128)
            throw std::runtime_error("skv_b200: Engine needs head_dim 128 (the compiled attention kernels)");
        model_ = ToyModel::create(cfg_.shape, cfg_.seed, cfg_.skewed_init);
        plan_ = make_plan();
        const std::size_t h = cfg_.shape.hidden(), L = cfg_.shape.layers, f = cfg_.shape.ffn_mult;
        auto up = [](const std::vector<double>& v) {
            DeviceBuffer b(std::max<std::size_t>(v.size(), 1) * 8);
            if (!v.empty()) b.upload(v.data(), v.size() * 8);
            return b;
        };
        emb_ = up(model_.embedding.data);
        for (const LayerWeights& lw : model_.layers) {
            DevLayer d;
            d.wq = up(lw.wq.data);
            d.wk = up(lw.wk.data);
            d.wv = up(lw.wv.data);
            d.wo = up(lw.wo.data);
            d.fin = up(lw.ffn_in.data);
            d.fout = up(lw.ffn_out.data);
            d.g1 = up(lw.ln1_gain);
            d.b1 = up(lw.ln1_bias);
            d.g2 = up(lw.ln2_gain);
            d.b2 = up(lw.ln2_bias);
            layers_.push_back(std::move(d));
        }
        fg_ = up(model_.final_ln_gain);
        fb_ = up(model_.final_ln_bias);
        proj_ = up(model_.output_proj.data);
        const std::size_t ncap = cfg_.prompt_len + cfg_.gen_len + 1;
        const bool quant = cfg_.quant.enabled;
        if (quant && cfg_.quant.bits != 8)
            throw std::runtime_error("skv_b200: the INT8 cache stores 8-bit codes (quant.bits = 8)");
        cache_ = std::make_unique<DeviceCache>(static_cast<int>(L), 1, static_cast<int>(cfg_.shape.heads), 128,
                                               static_cast<int>(ncap), quant ? SKV_U8 : SKV_F32, SKV_F32, 0, true);
        int variant = SKV_VARIANT_SWA;
        switch (cfg_.sparsity.variant) {
        case AttentionVariant::Dense: variant = SKV_VARIANT_DENSE; break;
        case AttentionVariant::Swa: variant = SKV_VARIANT_SWA; break;
        case AttentionVariant::Local: variant = SKV_VARIANT_LOCAL; break;
        case AttentionVariant::Strided: variant = SKV_VARIANT_STRIDED; break;
        }
        check(skv_cache_set_variant(cache_->handle(), variant, static_cast<int>(cfg_.sparsity.stride)));
        skv_plan pl{plan_.alpha, plan_.beta, static_cast<int64_t>(plan_.p1), static_cast<int64_t>(plan_.p2),
                    plan_.recompute_enabled ? 1 : 0, static_cast<int64_t>(cfg_.prompt_len),
                    static_cast<int64_t>(cfg_.gen_len)};
        cache_->set_plan(pl);
        // The device ledger counts entries of the cache's own row size (tb_);
        // the reference's entries are layer_kv_bytes (memsim.hpp:46-48). The
        // capacity check is made here, per allocation in the reference's
        // order (fit()): the device ledger applies each step's actions one
        // step ahead, so its own check would fire a step early.
        lb_ = layer_kv_bytes(cfg_.cost);
        skv_cache_desc dd{};
        check(skv_cache_get_desc(cache_->handle(), &dd, nullptr));
        tb_ = 2ull * dd.heads * (quant ? 136 : 512);
        scratch_x_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * 8);
        scratch_n_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * 8);
        scratch_q_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * 8);
        scratch_k_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * 8);
        scratch_v_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * 8);
        scratch_a_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * 8);
        scratch_f_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * f * 8);
        f32_q_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * 4);
        f32_k_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * 4);
        f32_v_ = DeviceBuffer(std::max<std::size_t>(ncap, 1) * h * 4);
        f32_o_ = DeviceBuffer(h * 4);
        logits_ = DeviceBuffer(cfg_.shape.vocab * 8);
        ids_ = DeviceBuffer(std::max<std::size_t>(cfg_.prompt_len, 1) * 8);
    }

    const SchedulePlan& plan() const { return plan_; }
    const ToyModel& model() const { return model_; }

    // engine.hpp:250-303
    RunMetrics run(const RunOptions& opts = {}) {
        RunMetrics metrics;
        metrics.plan = plan_;
        metrics.prompt_tokens = cfg_.prompt_len;
        std::vector<std::int64_t> prompt = make_prompt();
        metrics.prompt_ids = prompt;
        Vector logits = prefill(prompt, metrics);
        Vector logit_sum(cfg_.shape.vocab, 0.0);
        std::int64_t next = argmax_token(logits);
        for (std::size_t j = 0; j < cfg_.gen_len; ++j) {
            std::int64_t input_token = next;
            if (j < opts.forced_tokens.size()) input_token = opts.forced_tokens[j];
            logits = decode_step(j, input_token, metrics);
            if (opts.record_mean_logits)
                for (std::size_t v = 0; v < logit_sum.size(); ++v) logit_sum[v] += logits[v];
            next = argmax_token(logits);
            metrics.generated_ids.push_back(input_token);
            metrics.sequence_tokens = j + 1;
            if (cfg_.eos_id >= 0 && next == cfg_.eos_id) {
                metrics.hit_eos = true;
                break;
            }
        }
        if (opts.record_mean_logits && metrics.sequence_tokens > 0) {
            metrics.mean_logits = logit_sum;
            for (double& v : metrics.mean_logits) v /= static_cast<double>(metrics.sequence_tokens);
        }
        metrics.generated_tokens = static_cast<std::uint64_t>(cfg_.cost.batch) * metrics.sequence_tokens;
        metrics.compute_seconds = clock_.compute_seconds();
        metrics.transfer_seconds = clock_.transfer_seconds();
        metrics.recompute_seconds = clock_.recompute_seconds();
        metrics.total_seconds = clock_.total_seconds();
        metrics.transferred_bytes = clock_.transferred_bytes();
        if (metrics.generated_tokens > 0 && metrics.total_seconds > 0.0) {
            metrics.throughput_tokens_per_second =
                static_cast<double>(metrics.generated_tokens) / metrics.total_seconds;
            metrics.seconds_per_token = metrics.total_seconds / static_cast<double>(metrics.generated_tokens);
        }
        // the device ledger (no further step to prepare) must agree with the accounting
        uint64_t dev = 0, host = 0;
        check(skv_ledger_totals(cache_->handle(), &dev, &host, nullptr, nullptr, nullptr));
        if (dev / tb_ * lb_ != dev_bytes_ || host / tb_ * lb_ != host_bytes_)
            throw std::runtime_error("skv_b200: device ledger totals disagree with the step accounting");
        return metrics;
    }

    // The tokens the ledger's device tier holds, in the reference's bytes.
    uint64_t device_bytes() const { return dev_bytes_; }
    uint64_t host_bytes() const { return host_bytes_; }

  private:
    struct DevLayer {
        DeviceBuffer wq, wk, wv, wo, fin, fout, g1, b1, g2, b2;
    };

    // engine.hpp:314-341, with solve_plan on the C ABI (skv_plan.cpp)
    SchedulePlan make_plan() const {
        const std::size_t n = cfg_.gen_len;
        SchedulePlan plan;
        switch (cfg_.mode) {
        case ScheduleMode::Dynamic: {
            const CostParams& p = cfg_.cost;
            skv_cost_params cp{static_cast<int64_t>(p.hidden), static_cast<int64_t>(p.layers),
                               static_cast<int64_t>(p.batch), static_cast<int64_t>(p.input_len),
                               static_cast<int64_t>(p.output_len), p.ratio, p.bandwidth,
                               static_cast<int32_t>(p.bytes_per_element), p.device_capacity, p.mac_rate,
                               p.recompute_overhead};
            skv_plan out{};
            skv_plan_prediction pred{};
            check(skv_solve_plan(&cp, &out, &pred));
            plan.alpha = out.alpha;
            plan.beta = out.beta;
            plan.p1 = static_cast<std::size_t>(out.p1);
            plan.p2 = static_cast<std::size_t>(out.p2);
            plan.predicted_total_seconds = pred.total_seconds;
            plan.prefill_compute_seconds = pred.prefill_compute_seconds;
            for (int i = 0; i < 3; ++i) {
                plan.phases[i].steps = static_cast<std::size_t>(pred.phase_steps[i]);
                plan.phases[i].compute_seconds = pred.phase_compute[i];
                plan.phases[i].transfer_seconds = pred.phase_transfer[i];
                plan.phases[i].recompute_seconds = pred.phase_recompute[i];
            }
            plan.recompute_enabled = cfg_.recompute_enabled;
            break;
        }
        case ScheduleMode::AllDevice:
            plan.p1 = plan.p2 = n;
            break;
        case ScheduleMode::StaticSplit:
            plan.alpha = cfg_.static_fraction;
            plan.beta = 0.05;
            plan.p1 = 0;
            plan.p2 = n;
            plan.recompute_enabled = false;
            if (n == 0) plan.p1 = plan.p2 = 0;
            break;
        }
        return plan;
    }

    std::vector<std::int64_t> make_prompt() const {  // engine.hpp:343-350
        SeededRng rng(cfg_.seed ^ 0x9e3779b97f4a7c15ull);
        std::vector<std::int64_t> prompt(cfg_.prompt_len);
        for (auto& t : prompt) t = static_cast<std::int64_t>(rng.integer(cfg_.shape.vocab));
        return prompt;
    }

    static std::int64_t argmax_token(const Vector& logits) {  // engine.hpp:444-452
        std::size_t best = 0;
        for (std::size_t i = 1; i < logits.size(); ++i)
            if (logits[i] > logits[best]) best = i;
        return static_cast<std::int64_t>(best);
    }

    // attention_sparsity (attention.hpp:275-310) of a causal [rows][cols] map
    static double causal_sparsity(const double* aw, std::size_t rows, std::size_t cols) {
        const auto off = static_cast<std::ptrdiff_t>(cols) - static_cast<std::ptrdiff_t>(rows);
        std::size_t counted = 0, sparse = 0;
        for (std::size_t i = 0; i < rows; ++i) {
            const auto lim = static_cast<std::ptrdiff_t>(i) + off;
            double mx = 0.0;
            std::size_t cells = 0;
            for (std::size_t j = 0; j < cols && static_cast<std::ptrdiff_t>(j) <= lim; ++j) {
                mx = std::max(mx, aw[i * cols + j]);
                ++cells;
            }
            counted += cells;
            if (mx == 0.0) {
                sparse += cells;
                continue;
            }
            for (std::size_t j = 0; j < cols && static_cast<std::ptrdiff_t>(j) <= lim; ++j)
                sparse += aw[i * cols + j] < 0.01 * mx;
        }
        return counted == 0 ? 0.0 : static_cast<double>(sparse) / static_cast<double>(counted);
    }

    Vector logits_of(const double* x_row) {
        const int h = static_cast<int>(cfg_.shape.hidden()), V = static_cast<int>(cfg_.shape.vocab);
        check(skv_engine_layernorm(x_row, 1, h, fg_.as<double>(), fb_.as<double>(), scratch_n_.as<double>(), nullptr));
        check(skv_engine_gemm(scratch_n_.as<double>(), proj_.as<double>(), logits_.as<double>(), 1, V, h, 0, nullptr));
        Vector out(V);
        logits_.download(out.data(), out.size() * 8);
        for (const double v : out) require(std::isfinite(v), "logits: non-finite value");
        return out;
    }

    // engine.hpp:485-529 on the GPU
    Vector prefill(const std::vector<std::int64_t>& prompt, RunMetrics& metrics) {
        require(!prompt.empty(), "prefill: empty prompt");
        const int s = static_cast<int>(prompt.size()), h = static_cast<int>(cfg_.shape.hidden());
        const int H = static_cast<int>(cfg_.shape.heads), hf = h * static_cast<int>(cfg_.shape.ffn_mult);
        clock_.begin_step(0);
        ids_.upload(prompt.data(), prompt.size() * 8);
        double* x = scratch_x_.as<double>();
        double *xn = scratch_n_.as<double>(), *q = scratch_q_.as<double>(), *k = scratch_k_.as<double>(),
               *v = scratch_v_.as<double>(), *a = scratch_a_.as<double>(), *f = scratch_f_.as<double>();
        check(skv_engine_embed(emb_.as<double>(), h, ids_.as<int64_t>(), s, 0, x, nullptr));
        DeviceBuffer aw(static_cast<std::size_t>(H) * s * s * 8);
        std::vector<double> awh(static_cast<std::size_t>(H) * s * s);
        for (std::size_t l = 0; l < cfg_.shape.layers; ++l) {
            const DevLayer& w = layers_[l];
            check(skv_engine_layernorm(x, s, h, w.g1.as<double>(), w.b1.as<double>(), xn, nullptr));
            check(skv_engine_gemm(xn, w.wq.as<double>(), q, s, h, h, 0, nullptr));
            check(skv_engine_gemm(xn, w.wk.as<double>(), k, s, h, h, 0, nullptr));
            check(skv_engine_gemm(xn, w.wv.as<double>(), v, s, h, h, 0, nullptr));
            check(skv_engine_causal_attention(q, k, v, s, s, H, 128, a, aw.as<double>(), nullptr));
            check(skv_engine_gemm(a, w.wo.as<double>(), x, s, h, h, 1, nullptr));  // x += attn . Wo
            check(skv_engine_layernorm(x, s, h, w.g2.as<double>(), w.b2.as<double>(), xn, nullptr));
            check(skv_engine_gemm(xn, w.fin.as<double>(), f, s, hf, h, 0, nullptr));
            check(skv_engine_gelu(f, static_cast<std::size_t>(s) * hf, nullptr));
            check(skv_engine_gemm(f, w.fout.as<double>(), x, s, h, hf, 1, nullptr));  // x += FFN
            // the prompt's K/V (head_rows, fake-quant by the INT8 cache) and store_new
            check(skv_engine_convert(k, f32_k_.as<float>(), static_cast<std::size_t>(s) * h, nullptr));
            check(skv_engine_convert(v, f32_v_.as<float>(), static_cast<std::size_t>(s) * h, nullptr));
            for (int t = 0; t < s; ++t) {  // KvLedger::store_new per prompt token (memsim.hpp:99-109)
                fit(lb_);
                dev_bytes_ += lb_;
            }
            cache_->append_tokens(static_cast<int>(l), 0, 1, 0, s, f32_k_.get(), f32_v_.get());
            // importance seed: the head-summed last attention row (attention.hpp:77-85 order)
            aw.download(awh.data(), awh.size() * 8);
            std::vector<double> seed(s, 0.0);
            double sp = 0.0;
            for (int hd = 0; hd < H; ++hd) {
                const double* m = awh.data() + static_cast<std::size_t>(hd) * s * s;
                for (int t = 0; t < s; ++t) seed[t] += m[static_cast<std::size_t>(s - 1) * s + t];
                sp += causal_sparsity(m, s, s);
            }
            DeviceBuffer ds(seed.size() * 8);
            ds.upload(seed.data(), seed.size() * 8);
            cache_->set_importance(static_cast<int>(l), 0, 1, s, ds.as<double>());
            metrics.prefill_sparsity_per_layer.push_back(sp / static_cast<double>(H));
        }
        clock_.charge_compute(compute_time(cfg_.cost, static_cast<std::size_t>(s) * (s + 1) / 2));
        metrics.prefill_seconds = clock_.compute_seconds();
        clock_.end_step(dev_bytes_, host_bytes_);
        metrics.peak_device_bytes = std::max(metrics.peak_device_bytes, dev_bytes_);
        return logits_of(x + static_cast<std::size_t>(s - 1) * h);
    }

    // KvLedger's capacity check before an allocation (memsim.hpp:193-200)
    void fit(uint64_t add) const {
        if (dev_bytes_ + add > cfg_.cost.device_capacity)
            throw OutOfDeviceMemory("simulated OOM: device tier needs " + std::to_string(dev_bytes_ + add) +
                                    " bytes, capacity " + std::to_string(cfg_.cost.device_capacity));
    }

    // apply_actions' accounting (engine.hpp:686-716) of one layer's lists,
    // with the KvLedger byte totals (memsim.hpp:77-215) in the reference's
    // entry size and its capacity check before each allocation
    void account(const int32_t* cnt, StepMetrics& sm) {
        const double layers_d = static_cast<double>(cfg_.shape.layers);
        const uint64_t off = cnt[0], del = cnt[1], rel = cnt[2], rec = cnt[3];
        if (off) {
            dev_bytes_ -= off * lb_;
            host_bytes_ += off * lb_;
            clock_.charge_transfer(off * lb_, static_cast<double>(off) / layers_d, 0.0, cfg_.cost.bandwidth);
            step_d2h_ += static_cast<double>(off) / layers_d;
        }
        if (del) {
            host_bytes_ -= del * lb_;  // deleted tokens come from the host tier (or were just offloaded)
            sm.deleted += del;
        }
        for (uint64_t i = 0; i < rel; ++i) {
            fit(lb_);
            dev_bytes_ += lb_;
            host_bytes_ -= lb_;
        }
        if (rel) {
            clock_.charge_transfer(rel * lb_, 0.0, static_cast<double>(rel) / layers_d, cfg_.cost.bandwidth);
            step_h2d_ += static_cast<double>(rel) / layers_d;
        }
        for (uint64_t i = 0; i < rec; ++i) {
            fit(lb_);
            dev_bytes_ += lb_;
        }
        if (rec) {
            clock_.charge_recompute(recompute_time(cfg_.cost, rec) / layers_d);
            sm.recomputed += rec;
        }
        fit(lb_);  // store_new of the step's token
        dev_bytes_ += lb_;
    }

    // engine.hpp:571-684 on the GPU
    Vector decode_step(std::size_t j, std::int64_t token, RunMetrics& metrics) {
        const std::size_t pos = cfg_.prompt_len + j;
        require(pos < cfg_.prompt_len + cfg_.gen_len, "decode_step: context overflow");
        const int h = static_cast<int>(cfg_.shape.hidden()), hf = h * static_cast<int>(cfg_.shape.ffn_mult);
        clock_.begin_step(j + 1);
        StepMetrics sm;
        sm.step = j;
        sm.token_id = token;
        sm.phase = phase_of_step(plan_, j);
        const double c0 = clock_.compute_seconds(), t0 = clock_.transfer_seconds(), r0 = clock_.recompute_seconds();
        const double d2h0 = step_d2h_, h2d0 = step_h2d_;
        require(token >= 0 && token < static_cast<std::int64_t>(cfg_.shape.vocab), "embed: token id out of range");
        ids_.upload(&token, 8);
        double* x = scratch_x_.as<double>();
        double *xn = scratch_n_.as<double>(), *q = scratch_q_.as<double>(), *k = scratch_k_.as<double>(),
               *v = scratch_v_.as<double>(), *a = scratch_a_.as<double>(), *f = scratch_f_.as<double>();
        check(skv_engine_embed(emb_.as<double>(), h, ids_.as<int64_t>(), 1, static_cast<int>(pos), x, nullptr));
        const int n_tot = static_cast<int>(pos) + 1;
        const double r = cfg_.sparsity.ratio;
        std::size_t kept = 0;
        std::vector<int32_t> lists(4 * (cfg_.prompt_len + cfg_.gen_len + 1)), cnt(4);
        for (std::size_t l = 0; l < cfg_.shape.layers; ++l) {
            const DevLayer& w = layers_[l];
            const int li = static_cast<int>(l);
            check(skv_engine_layernorm(x, 1, h, w.g1.as<double>(), w.b1.as<double>(), xn, nullptr));
            check(skv_engine_gemm(xn, w.wq.as<double>(), q, 1, h, h, 0, nullptr));
            check(skv_engine_gemm(xn, w.wk.as<double>(), k, 1, h, h, 0, nullptr));
            check(skv_engine_gemm(xn, w.wv.as<double>(), v, 1, h, h, 0, nullptr));
            // variant_selection + step_actions + apply_actions of this step
            check(skv_decode_prepare(cache_->handle(), li, n_tot, r, nullptr));
            check(skv_last_actions(cache_->handle(), li, lists.data(), cnt.data(), nullptr));
            check(skv_stream_synchronize(nullptr));
            account(cnt.data(), sm);
            int32_t m = 0;
            check(skv_selection_size(cache_->handle(), n_tot, r, &m, nullptr));
            kept = std::max<std::size_t>(kept, static_cast<std::size_t>(m));
            check(skv_engine_convert(q, f32_q_.as<float>(), h, nullptr));
            check(skv_engine_convert(k, f32_k_.as<float>(), h, nullptr));
            check(skv_engine_convert(v, f32_v_.as<float>(), h, nullptr));
            cache_->decode_layer(li, n_tot, r, f32_q_.get(), f32_k_.get(), f32_v_.get(), f32_o_.get());
            double sp = 0.0;
            check(skv_sparsity_get(cache_->handle(), li, 0, 1, &sp, nullptr));
            check(skv_stream_synchronize(nullptr));
            sm.sparsity_per_layer.push_back(sp);
            check(skv_engine_widen(f32_o_.as<float>(), a, h, nullptr));
            check(skv_engine_gemm(a, w.wo.as<double>(), x, 1, h, h, 1, nullptr));
            check(skv_engine_layernorm(x, 1, h, w.g2.as<double>(), w.b2.as<double>(), xn, nullptr));
            check(skv_engine_gemm(xn, w.fin.as<double>(), f, 1, hf, h, 0, nullptr));
            check(skv_engine_gelu(f, hf, nullptr));
            check(skv_engine_gemm(f, w.fout.as<double>(), x, 1, h, hf, 1, nullptr));
        }
        clock_.charge_compute(compute_time(cfg_.cost, kept));
        sm.kept_tokens = kept;
        sm.compute_seconds = clock_.compute_seconds() - c0;
        sm.transfer_seconds = clock_.transfer_seconds() - t0;
        sm.recompute_seconds = clock_.recompute_seconds() - r0;
        sm.d2h_tokens = step_d2h_ - d2h0;
        sm.h2d_tokens = step_h2d_ - h2d0;
        sm.device_bytes = dev_bytes_;
        sm.host_bytes = host_bytes_;
        if (!sm.sparsity_per_layer.empty()) {
            double total = 0.0;
            for (const double s : sm.sparsity_per_layer) total += s;
            sm.sparsity_mean = total / static_cast<double>(sm.sparsity_per_layer.size());
        }
        clock_.end_step(dev_bytes_, host_bytes_);
        metrics.peak_device_bytes = std::max(metrics.peak_device_bytes, dev_bytes_);
        metrics.peak_host_bytes = std::max(metrics.peak_host_bytes, host_bytes_);
        metrics.steps.push_back(std::move(sm));
        return logits_of(x);
    }

    EngineConfig cfg_;
    ToyModel model_;
    SchedulePlan plan_;
    std::unique_ptr<DeviceCache> cache_;
    DeviceBuffer emb_, fg_, fb_, proj_;
    std::vector<DevLayer> layers_;
    DeviceBuffer scratch_x_, scratch_n_, scratch_q_, scratch_k_, scratch_v_, scratch_a_, scratch_f_;
    DeviceBuffer f32_q_, f32_k_, f32_v_, f32_o_, logits_, ids_;
    TransferLedger clock_;
    uint64_t lb_ = 0, tb_ = 0, dev_bytes_ = 0, host_bytes_ = 0;
    double step_d2h_ = 0.0, step_h2d_ = 0.0;
};

}  // namespace skv::b200
