"""Probe the config-4 step: events around (a) whole decode steps, (b) the
attend chain alone -- to locate the step-vs-chain gap. Env switches mirror
bench.py's setup: PF=1 tensor-core prefill (else the seed only), KV2=1
separate random K and V, ROT=1 eight rotating step inputs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api  # noqa: E402

L, B, H, D, s = int(os.environ.get("PL", 48)), 32, 56, 128, 4095
PF, KV2, ROT = (os.environ.get(k) == "1" for k in ("PF", "KV2", "ROT"))
c = api.SwaCache(L, B, H, D, s + 64, kv_dtype="u8", q_dtype="f16")
g = torch.Generator(device="cuda").manual_seed(0)
for l in range(L):
    k = torch.randn(B, s, H, D, device="cuda", generator=g).half()
    v = torch.randn(B, s, H, D, device="cuda", generator=g).half() if KV2 else k
    c.append_tokens(l, 0, 0, k, v)
    del k, v
    if PF:
        c.prefill_layer(l, torch.randn(B, s, H, D, device="cuda", generator=g).half() * 0.5)
    else:
        c.prefill_seed(l, s, torch.randn(B, H, D, device="cuda", generator=g).half())
pool = [tuple(torch.randn(L, B, H, D, device="cuda", generator=g).half() for _ in range(3))
        for _ in range(8 if ROT else 1)]
out = torch.empty_like(pool[0][0])
n = s
for i in range(3):
    n += 1
    c.swa_decode_step(n, 0.2, *pool[i % len(pool)], out)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
reps = 10
e[0].record()
for i in range(reps):
    n += 1
    c.swa_decode_step(n, 0.2, *pool[i % len(pool)], out)
e[1].record()
torch.cuda.synchronize()
step = e[0].elapsed_time(e[1]) / reps
q, kn, vn = pool[0]
chain3 = c.attend_chain_ms(n + 1, 0.2, q, kn, vn, out, 3) / 3
chain1 = min(c.attend_chain_ms(n + 1, 0.2, q, kn, vn, out, 1) for _ in range(3))
print(f"L={L} PF={PF} KV2={KV2} ROT={ROT}: step {step:.3f} ms; chain per step (3 steps chained) {chain3:.3f}; "
      f"one step's attends alone {chain1:.3f}")

if os.environ.get("TRACE") == "1":
    # kernel timeline of two steps (CUPTI via torch.profiler): gaps and overlaps
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(2):
            n += 1
            c.swa_decode_step(n, 0.2, *pool[i % len(pool)], out)
        torch.cuda.synchronize()
    ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    sels = [i for i, e in enumerate(ev) if "select" in e.name]
    print("TR kernels", len(ev), "selects at", sels)
    for i, e in enumerate(ev):
        st, en = e.time_range.start - t0, e.time_range.end - t0
        print(f"TR {i:3d} {e.name[13:30]:17s} start {st:9.1f} end {en:9.1f} dur {en - st:7.1f}")
