"""Does an HBM-saturating kernel slow host->device copies? H2D of 50 MB
alone vs while a device-to-device copy of 8 GB runs on another stream."""
import torch

n = 50 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
big_a = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
big_b = torch.empty_like(big_a)
s_copy, s_hbm = torch.cuda.Stream(), torch.cuda.Stream()


def h2d_ms(busy: bool) -> float:
    torch.cuda.synchronize()
    if busy:
        with torch.cuda.stream(s_hbm):
            for _ in range(4):
                big_b.copy_(big_a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s_copy):
        e0.record()
        for _ in range(5):
            d.copy_(h, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 5


for busy in (False, True, False, True):
    ms = h2d_ms(busy)
    print(f"H2D 50 MB {'while HBM busy' if busy else 'alone'}: {ms:.3f} ms = {n / ms / 1e6:.1f} GB/s")
