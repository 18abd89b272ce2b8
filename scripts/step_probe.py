"""Probe the config-4 step: events around (a) whole decode steps, (b) the
attend chain alone, (c) the attends of a step with the deferred select
launch on a side path -- to locate the step-vs-chain gap."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api  # noqa: E402

L, B, H, D, s = int(os.environ.get("PL", 48)), 32, 56, 128, 4095
c = api.SwaCache(L, B, H, D, s + 64, kv_dtype="u8", q_dtype="f16")
g = torch.Generator(device="cuda").manual_seed(0)
for l in range(L):
    k = torch.randn(B, s, H, D, device="cuda", generator=g).half()
    c.append_tokens(l, 0, 0, k, k)
    c.prefill_seed(l, s, torch.randn(B, H, D, device="cuda", generator=g).half())
q, kn, vn = (torch.randn(L, B, H, D, device="cuda", generator=g).half() for _ in range(3))
out = torch.empty_like(q)
n = s
for _ in range(3):
    n += 1
    c.swa_decode_step(n, 0.2, q, kn, vn, out)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(12)]
reps = 10
e[0].record()
for _ in range(reps):
    n += 1
    c.swa_decode_step(n, 0.2, q, kn, vn, out)
e[1].record()
torch.cuda.synchronize()
step = e[0].elapsed_time(e[1]) / reps
chain = c.attend_chain_ms(n + 1, 0.2, q, kn, vn, out, 3) if hasattr(c, "attend_chain_ms") else None
print(f"L={L}: step {step:.3f} ms; chain per step {chain / 3 if chain else None}")
