"""Host-side placement of the pinned buffers vs PCIe bandwidth: for each NUMA
node of the box, pin this process to that node's cores, allocate (first
touch) pinned buffers there and time 50 MB host<->device copies. Prints the
GPU's NVML CPU affinity beside it (the node bench.py binds to)."""
import glob
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cpulist(path):
    out = []
    for part in open(path).read().strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out += range(int(a), int(b) + 1)
        elif part:
            out.append(int(part))
    return out


def bw(nbytes, fn, iters=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(iters)]; e1.record(); torch.cuda.synchronize()
    return nbytes * iters / (e0.elapsed_time(e1) / 1e3) / 1e9


torch.cuda.init()
print("cpus", os.cpu_count(), "affinity at start", len(os.sched_getaffinity(0)))
try:
    from paper_2403_17312_b200 import hostaff
    print("GPU-local cpus (NVML):", hostaff.gpu_local_cpus(0))
except Exception as e:  # noqa: BLE001
    print("hostaff:", e)
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
print("numa nodes", [os.path.basename(n) for n in nodes])
n = 50 << 20
for nd in nodes + [None]:
    if nd is not None:
        cpus = [c for c in cpulist(os.path.join(nd, "cpulist")) if c < os.cpu_count()]
        if not cpus:
            continue
        os.sched_setaffinity(0, cpus)
        tag = os.path.basename(nd)
    else:
        os.sched_setaffinity(0, range(os.cpu_count()))
        tag = "all"
    h = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    h.fill_(1); h2.fill_(2)
    d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    print(f"{tag}: h2d {bw(n, lambda: d.copy_(h, non_blocking=True)):.1f} GB/s  "
          f"d2h {bw(n, lambda: h2.copy_(d2, non_blocking=True)):.1f} GB/s  both {bw(2 * n, both):.1f} GB/s", flush=True)
    del h, h2
