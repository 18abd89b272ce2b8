// skv_plan.cpp -- host-side offline planner for the three-phase schedule.
//
// The reference plans once per workload on the host (scheduler.hpp:64-303:
// phase1_limit, simulate_plan, solve_plan over the memsim.hpp:42-70 cost
// model); the per-step bookkeeping it drives runs on the device
// (skv_ledger.cuh). This is a restatement with the same arithmetic order, so
// plans and predictions match the reference exactly (tests/test_planner.py
// against fixtures produced by the reference itself).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "skv_b200.h"

namespace skv_impl {
skv_status fail_msg(skv_status s, const char* msg);  // skv_capi.cu: sets skv_last_error()
}
using skv_impl::fail_msg;

namespace {

uint64_t kv_bytes_per_token(const skv_cost_params& p) {  // memsim.hpp:42-44
    return 2ull * static_cast<uint64_t>(p.bytes_per_element) * static_cast<uint64_t>(p.batch) *
           static_cast<uint64_t>(p.layers) * static_cast<uint64_t>(p.hidden);
}

double seconds_transfer(const skv_cost_params& p, uint64_t d2h, uint64_t h2d) {  // memsim.hpp:50-54
    return static_cast<double>(kv_bytes_per_token(p)) * static_cast<double>(d2h + h2d) / p.bandwidth;
}

double seconds_compute(const skv_cost_params& p, uint64_t kept) {  // memsim.hpp:57-61
    return 2.0 * static_cast<double>(p.batch) * static_cast<double>(p.layers) * static_cast<double>(p.hidden) *
           static_cast<double>(kept) / p.mac_rate;
}

double seconds_recompute(const skv_cost_params& p, uint64_t tokens) {  // memsim.hpp:65-70
    return p.recompute_overhead * 2.0 * static_cast<double>(p.batch) * static_cast<double>(p.layers) *
           static_cast<double>(p.hidden) * static_cast<double>(p.hidden) * static_cast<double>(tokens) /
           p.mac_rate;
}

// attention.hpp:122-138 (host copies of the window rules)
uint64_t window_k(uint64_t n, double r) { return skv_swa_window_k(n, r); }
uint64_t keep_count(uint64_t n, double r) { return skv_swa_keep_count(n, r); }

bool valid_cost(const skv_cost_params& p) {  // CostParams::validate (memsim.hpp:28-37)
    return p.hidden > 0 && p.layers > 0 && p.batch > 0 && (p.output_len > 0 || p.input_len > 0) &&
           p.ratio > 0.0 && p.ratio <= 1.0 && p.bandwidth > 0.0 &&
           (p.bytes_per_element == 1 || p.bytes_per_element == 2) && p.mac_rate > 0.0 &&
           p.recompute_overhead >= 1.0;
}

enum Slot : uint8_t { kDevice, kHost, kDeleted };

// scheduler.hpp:90-186: deterministic position-level model; global picks are
// pessimistically the oldest non-window positions, eviction oldest-first.
skv_plan_prediction simulate(const skv_plan& plan, const skv_cost_params& p) {
    const uint64_t s = static_cast<uint64_t>(p.input_len), n = static_cast<uint64_t>(p.output_len);
    const uint64_t tb = kv_bytes_per_token(p);
    skv_plan_prediction out{};
    out.prefill_compute_seconds = seconds_compute(p, s * (s + 1) / 2);
    out.total_seconds = out.prefill_compute_seconds;
    std::vector<uint8_t> pos(s, kDevice);
    pos.reserve(s + n);
    uint64_t on_host = 0, deleted = 0;
    uint64_t peak = tb * s;
    out.feasible = (peak <= p.device_capacity && tb <= p.device_capacity) ? 1 : 0;
    for (uint64_t j = 0; j < n; ++j) {
        const uint64_t existing = s + j, n_tot = existing + 1;
        const uint64_t k = window_k(n_tot, p.ratio), kept = keep_count(n_tot, p.ratio);
        int phase = 3;
        if (static_cast<int64_t>(j) < plan.p1)
            phase = 1;
        else if (static_cast<int64_t>(j) < plan.p2 || !plan.recompute_enabled)
            phase = 2;
        out.phase_steps[phase - 1] += 1;
        if (phase >= 2) {
            const uint64_t nonlocal = n_tot - k;
            const auto target = static_cast<uint64_t>(std::ceil(plan.alpha * static_cast<double>(existing)));
            uint64_t want = target > on_host ? target - on_host : 0, moved = 0;
            for (uint64_t i = 0; i < nonlocal && want > 0 && i < pos.size(); ++i)
                if (pos[i] == kDevice) {
                    pos[i] = kHost;
                    --want;
                    ++moved;
                }
            on_host += moved;
            const double t_off = seconds_transfer(p, moved, 0);
            out.phase_transfer[phase - 1] += t_off;
            out.total_seconds += t_off;
            if (phase == 3 && on_host > 0) {
                auto del = static_cast<uint64_t>(std::ceil(plan.beta * static_cast<double>(on_host)));
                for (uint64_t i = 0; i < pos.size() && del > 0; ++i)
                    if (pos[i] == kHost) {
                        pos[i] = kDeleted;
                        --del;
                        --on_host;
                        ++deleted;
                    }
            }
            const uint64_t picks = kept - k;
            uint64_t back = 0, redo = 0;
            for (uint64_t i = 0; i < picks && i < pos.size(); ++i) {
                if (pos[i] == kHost) {
                    pos[i] = kDevice;
                    ++back;
                } else if (pos[i] == kDeleted) {
                    pos[i] = kDevice;
                    ++redo;
                }
            }
            on_host -= back;
            deleted -= redo;
            const double t_rel = seconds_transfer(p, 0, back);
            out.phase_transfer[phase - 1] += t_rel;
            out.total_seconds += t_rel;
            const double t_rec = seconds_recompute(p, redo);
            out.phase_recompute[phase - 1] += t_rec;
            out.total_seconds += t_rec;
        }
        const double t_cmp = seconds_compute(p, kept);
        out.phase_compute[phase - 1] += t_cmp;
        out.total_seconds += t_cmp;
        pos.push_back(kDevice);
        const uint64_t on_device = pos.size() - on_host - deleted;
        peak = std::max(peak, tb * on_device);
        if (peak > p.device_capacity) out.feasible = 0;
    }
    out.peak_device_bytes = peak;
    return out;
}

skv_status check_plan(const skv_plan& plan, int64_t n) {  // validate_plan (scheduler.hpp:26-35)
    if (plan.p1 == plan.p2) return plan.p1 == n ? SKV_OK : SKV_ERR_CONTRACT;
    if (!(plan.p1 >= 0 && plan.p1 < plan.p2 && plan.p2 <= n)) return SKV_ERR_CONTRACT;
    if (!(plan.alpha > 0.0 && plan.alpha < 1.0 && plan.beta > 0.0 && plan.beta < 1.0)) return SKV_ERR_CONTRACT;
    return SKV_OK;
}

}  // namespace

extern "C" {

skv_status skv_predict_plan(const skv_cost_params* p, const skv_plan* plan, skv_plan_prediction* out) {
    if (!p || !plan || !out || !valid_cost(*p)) return fail_msg(SKV_ERR_CONTRACT, "CostParams: invalid");
    if (skv_status s = check_plan(*plan, p->output_len)) return fail_msg(s, "plan: invalid (validate_plan)");
    *out = simulate(*plan, *p);
    return SKV_OK;
}

// scheduler.hpp:207-303: p1 from the capacity constraint, then greedy
// coordinate descent over (alpha, beta, p2) on the 0.05 grid, two sweeps,
// restricted to plans whose simulated peak fits the device.
skv_status skv_solve_plan(const skv_cost_params* p, skv_plan* plan_out, skv_plan_prediction* pred_out) {
    if (!p || !plan_out || !valid_cost(*p)) return fail_msg(SKV_ERR_CONTRACT, "CostParams: invalid");
    const uint64_t tb = kv_bytes_per_token(*p);
    if (tb > p->device_capacity)
        return fail_msg(SKV_ERR_INFEASIBLE, "single token's KV exceeds device capacity");
    if (tb * static_cast<uint64_t>(p->input_len) > p->device_capacity)
        return fail_msg(SKV_ERR_INFEASIBLE, "prompt KV alone exceeds device capacity");
    const int64_t n = p->output_len;
    int64_t p1 = n;  // phase1_limit (scheduler.hpp:64-73)
    for (int64_t j = 0; j < n; ++j)
        if (tb * static_cast<uint64_t>(p->input_len + j + 1) > p->device_capacity) {
            p1 = j;
            break;
        }
    skv_plan best{};
    best.recompute_enabled = 1;
    if (p1 == n) {
        best.p1 = best.p2 = n;
        const skv_plan_prediction pr = simulate(best, *p);
        *plan_out = best;
        if (pred_out) *pred_out = pr;
        return SKV_OK;
    }
    std::vector<double> grid;
    for (int i = 1; i <= 19; ++i) grid.push_back(0.05 * i);
    auto eval = [&](double a, double b, int64_t p2, skv_plan_prediction* pr) {
        skv_plan c{};
        c.alpha = a;
        c.beta = b;
        c.p1 = p1;
        c.p2 = p2;
        c.recompute_enabled = 1;
        *pr = simulate(c, *p);
        return pr->feasible != 0;
    };
    double ba = 0.0, bb = grid.front();
    int64_t bp2 = n;
    skv_plan_prediction bpred{}, pr{};
    bool found = false;
    for (double a : grid)
        if (eval(a, bb, bp2, &pr)) {
            ba = a;
            bpred = pr;
            found = true;
            break;
        }
    if (!found) return fail_msg(SKV_ERR_INFEASIBLE, "no feasible (alpha, beta, p2) under device capacity");
    for (int sweep = 0; sweep < 2; ++sweep) {
        for (double a : grid)
            if (eval(a, bb, bp2, &pr) && pr.total_seconds < bpred.total_seconds) {
                bpred = pr;
                ba = a;
            }
        for (double b : grid)
            if (eval(ba, b, bp2, &pr) && pr.total_seconds < bpred.total_seconds) {
                bpred = pr;
                bb = b;
            }
        for (int64_t p2 = p1 + 1; p2 <= n; ++p2)
            if (eval(ba, bb, p2, &pr) && pr.total_seconds < bpred.total_seconds) {
                bpred = pr;
                bp2 = p2;
            }
    }
    best.alpha = ba;
    best.beta = bb;
    best.p1 = p1;
    best.p2 = bp2;
    *plan_out = best;
    if (pred_out) *pred_out = bpred;
    return SKV_OK;
}

}  // extern "C"
