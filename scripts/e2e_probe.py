"""e2e (host-buffer) step timing at config-2 shape vs the layer-chunk count
(SKV_HOST_CHUNKS is read once per process, so one process per setting)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api

L, B, H, D, s = (int(os.environ.get("PL", 32)), int(os.environ.get("PB", 64)), int(os.environ.get("PH", 32)), 128,
              int(os.environ.get("PS", 512)))
c = api.SwaCache(L, B, H, D, s + 160, kv_dtype="f16")
g = torch.Generator(device="cuda").manual_seed(0)
for l in range(L):
    k = torch.randn(B, s, H, D, device="cuda", generator=g).half()
    c.append_tokens(l, 0, 0, k, k)
    c.prefill_seed(l, s, torch.randn(B, H, D, device="cuda", generator=g).half())
qh, kh, vh, oh = (torch.randn(L, B, H, D).half().pin_memory() for _ in range(4))
n = s
for _ in range(3):
    n += 1; c.swa_decode_step_host(n, 0.2, qh, kh, vh, oh)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30):
    n += 1; c.swa_decode_step_host(n, 0.2, qh, kh, vh, oh)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 30
# copies alone, same sizes, same two streams pattern (no compute)
d = torch.empty(3, L, B, H, D, dtype=torch.half, device="cuda"); do = torch.empty(L, B, H, D, dtype=torch.half, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def copies():
    with torch.cuda.stream(s1):
        for i, t in enumerate((qh, kh, vh)): d[i].copy_(t, non_blocking=True)
    with torch.cuda.stream(s2): oh.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
copies(); torch.cuda.synchronize()
e0.record(); [copies() for _ in range(30)]; e1.record(); torch.cuda.synchronize()
cms = e0.elapsed_time(e1) / 30
# device step alone
qd, kd, vd = qh.cuda(), kh.cuda(), vh.cuda(); od = torch.empty_like(qd)
e0.record()
for _ in range(30):
    n += 1; c.swa_decode_step(n, 0.2, qd, kd, vd, od)
e1.record(); torch.cuda.synchronize()
dms = e0.elapsed_time(e1) / 30
print(f"chunks={os.environ.get('SKV_HOST_CHUNKS', 'default')}: e2e {ms:.3f} ms/step ({B/ms*1e3:.0f} tok/s)  "
      f"copies-only {cms:.3f} ms  device-only {dms:.3f} ms")
# host enqueue cost per call (no synchronisation): if it approaches the
# step time the GPU waits on the host
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(30):
    n += 1; c.swa_decode_step(n, 0.2, qd, kd, vd, od)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
for _ in range(30):
    n += 1; c.swa_decode_step_host(n, 0.2, qh, kh, vh, oh)
t3 = time.perf_counter()
torch.cuda.synchronize()
print(f"host enqueue per call: device step {(t1 - t0) / 30 * 1e3:.3f} ms, host-buffer step {(t3 - t2) / 30 * 1e3:.3f} ms")
