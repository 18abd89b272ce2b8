"""Latency of one standalone swa_select launch (one CTA per sequence) vs the
candidate count: the per-layer cost the attend tail adds to a launch. 50
launches back to back between events; an empty kernel for the launch floor."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api


def per_launch(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / reps


x = torch.zeros(1, device="cuda")
print(f"empty kernel: {per_launch(lambda: x.add_(1)):.2f} us per launch")
for n in (128, 520, 768, 1536, 4096):
    imp = torch.rand(16, n, device="cuda", dtype=torch.float64)
    idx = torch.empty(16, n, dtype=torch.int32, device="cuda")
    print(f"n={n}: swa_select {per_launch(lambda: api.swa_select(imp, n, 0.2)):.2f} us per launch")
