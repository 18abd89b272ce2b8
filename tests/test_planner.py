"""The host planner (csrc/skv_plan.cpp, scheduler.hpp:64-303) against plans the
unmodified reference computed (tests/golden, make_golden.py): identical
(alpha, beta, p1, p2), identical predictions, InfeasiblePlan where the
reference throws it. Host-only: no GPU needed."""
import numpy as np
import pytest

from paper_2403_17312_b200 import api


def test_solve_plan_matches_reference(golden):
    rows = golden["plan_rows"]
    solved = infeasible = phased = 0
    for row in rows:
        hidden, layers, batch, s_len, out_len, ratio, bw, bpe, cap, mac, ovh, rc = row[:12]
        cost = dict(hidden=int(hidden), layers=int(layers), batch=int(batch), input_len=int(s_len),
                    output_len=int(out_len), ratio=float(ratio), bandwidth=float(bw), bytes_per_element=int(bpe),
                    device_capacity=int(cap), mac_rate=float(mac), recompute_overhead=float(ovh))
        if int(rc) == 3:
            with pytest.raises(api.InfeasiblePlan):
                api.solve_plan(cost)
            infeasible += 1
            continue
        assert int(rc) == 0
        plan, pred = api.solve_plan(cost)
        want_plan, want_pred = row[12:16], row[16:]
        assert [plan["alpha"], plan["beta"], plan["p1"], plan["p2"]] == list(want_plan)
        got_pred = [pred["total_seconds"], pred["prefill_compute_seconds"], *pred["phase_compute"],
                    *pred["phase_transfer"], *pred["phase_recompute"], *pred["phase_steps"]]
        assert got_pred == list(want_pred)
        solved += 1
        phased += plan["p1"] < plan["p2"]
    assert solved >= 10 and infeasible >= 3 and phased >= 3


def test_predict_plan_rejects_invalid_plans():
    cost = dict(hidden=16, layers=2, batch=1, input_len=8, output_len=10, ratio=0.5, bandwidth=1e6,
                device_capacity=10 ** 9, mac_rate=1e9)
    with pytest.raises(api.ContractViolation):
        api.predict_plan(cost, {"alpha": 0.5, "beta": 0.5, "p1": 3, "p2": 3})  # degenerate must be p1 == n
    with pytest.raises(api.ContractViolation):
        api.predict_plan(cost, {"alpha": 1.5, "beta": 0.5, "p1": 2, "p2": 5})
    pred = api.predict_plan(cost, {"alpha": 0.5, "beta": 0.5, "p1": 2, "p2": 5})
    assert pred["phase_steps"] == [2, 3, 5]
