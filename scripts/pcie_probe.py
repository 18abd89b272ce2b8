"""PCIe copy bandwidths on the box (context for the e2e number): pinned
host->device, device->host, and both at once on two streams."""
import torch

def bw(nbytes, fn, iters=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(iters)]; e1.record(); torch.cuda.synchronize()
    return nbytes * iters / (e0.elapsed_time(e1) / 1e3) / 1e9

for mb in (2, 8, 50):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    print(f"{mb} MB: h2d {bw(n, lambda: d.copy_(h, non_blocking=True)):.1f} GB/s  "
          f"d2h {bw(n, lambda: h2.copy_(d2, non_blocking=True)):.1f} GB/s  both {bw(2*n, both):.1f} GB/s total")
