"""HBM read-only bandwidth on the box (context for the attend roofline: the
decode gather is ~98% reads, MEASURED_PEAKS.json's hbm_gbs is a read+write
copy). Best of several torch reductions over 8 GiB, CUDA events."""
import torch

x = torch.empty(8 << 30, dtype=torch.uint8, device="cuda").view(torch.float32)
x.fill_(1.0)
best = {}
for name, fn in (("sum f32", lambda: x.sum()), ("amax f32", lambda: x.amax()),
                 ("sum bf16 view", lambda: x.view(torch.bfloat16).sum(dtype=torch.float32)),
                 ("copy (r+w)", lambda: y.copy_(x[: x.numel() // 2]))):
    if name.startswith("copy"):
        y = torch.empty(x.numel() // 2, dtype=torch.float32, device="cuda")
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    nbytes = x.numel() * 4 if not name.startswith("copy") else x.numel() * 4  # copy: half read + half written
    best[name] = nbytes / (min(ts) / 1e3) / 1e9
    print(f"{name}: {best[name]:.0f} GB/s")
