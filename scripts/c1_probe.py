"""Config 1 (fp32, b=1, H=32, one layer, n ~ 520) step anatomy: CUDA events
over 200 steps, and a CUPTI kernel timeline (torch.profiler) of 10 steps --
kernel durations vs the gaps between them (launch-bound or device-bound)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api  # noqa: E402

L, B, H, D, s = 1, 1, 32, 128, 511
c = api.SwaCache(L, B, H, D, s + 400, kv_dtype="f32", q_dtype="f32")
g = torch.Generator(device="cuda").manual_seed(0)
c.append_tokens(0, 0, 0, torch.randn(B, s, H, D, device="cuda", generator=g),
                torch.randn(B, s, H, D, device="cuda", generator=g))
c.prefill_seed(0, s, torch.randn(B, H, D, device="cuda", generator=g))
pool = [tuple(torch.randn(L, B, H, D, device="cuda", generator=g) for _ in range(3)) for _ in range(8)]
out = torch.empty_like(pool[0][0])
n = s
for i in range(20):
    n += 1
    c.swa_decode_step(n, 0.2, *pool[i % 8], out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(200):
    n += 1
    c.swa_decode_step(n, 0.2, *pool[i % 8], out)
e1.record()
torch.cuda.synchronize()
print(f"C1 step {e0.elapsed_time(e1) / 200 * 1000:.2f} us (events, 200 steps)")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(10):
        n += 1
        c.swa_decode_step(n, 0.2, *pool[i % 8], out)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
prev = None
for e in ev:
    gap = (e.time_range.start - prev) if prev is not None else 0.0
    print(f"C1TR {e.name[:45]:45s} dur {e.time_range.end - e.time_range.start:6.2f} gap {gap:6.2f}")
    prev = e.time_range.end
