"""Host NUMA placement for the host-buffer (e2e) path.

Pinned host buffers are placed on the NUMA node of the thread that allocates
them. On a two-socket box, buffers that land on the socket away from the GPU's
PCIe root cross the inter-socket link on every copy. `pinned_near_gpu`
allocates them on the GPU's own node, which it reads from the device's sysfs
`local_cpulist`. The allocating thread is bound to those cores for the
allocation only, and its affinity is restored afterwards.
"""
import contextlib
import os

import torch


def _cpulist(text):
    out = []
    for part in text.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out += range(int(a), int(b) + 1)
        elif part:
            out.append(int(part))
    return out


def gpu_local_cpus(device=0):
    """The allowed CPUs on the GPU's NUMA node, or None when unknown or when it is every allowed CPU."""
    p = torch.cuda.get_device_properties(device)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    try:
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            local = set(_cpulist(f.read()))
    except (OSError, ValueError):
        return None
    allowed = os.sched_getaffinity(0)
    cpus = sorted(local & allowed)
    return cpus if cpus and len(cpus) < len(allowed) else None


@contextlib.contextmanager
def near_gpu(device=0):
    """Run the body bound to the GPU-local cores (no-op when unknown)."""
    cpus = gpu_local_cpus(device)
    if cpus is None:
        yield None
        return
    old = os.sched_getaffinity(0)
    os.sched_setaffinity(0, cpus)
    try:
        yield cpus
    finally:
        os.sched_setaffinity(0, old)


def pinned_near_gpu(shape, dtype, device=0):
    """A pinned host tensor whose pages sit on the GPU's NUMA node (first touch under near_gpu)."""
    with near_gpu(device):
        t = torch.empty(shape, dtype=dtype).pin_memory()
        t.view(-1).view(torch.uint8).zero_()
    return t
