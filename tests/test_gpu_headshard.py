"""GPU head sharding (SURVEY §8 e; skv_cache_set_head_shard): each rank's
cache holds a slice of the heads, and the head-summed step row (and the
prefill seed row + sparsity) is SUM-all-reduced across the ranks before the
fold, through the same torch.distributed reducer bench.py uses. Two ranks
share the box's one GPU over gloo (NCCL refuses two ranks on one device);
the one-rank NCCL case checks the NCCL call ordering on the library stream.
Reference: the unsharded cache on the same inputs, itself pinned to the
oracle by test_gpu_parity / test_gpu_prefill."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

L, B, H, D, S, STEPS, R = 2, 2, 8, 128, 96, 5, 0.2


def _inputs():
    g = torch.Generator().manual_seed(3)
    kv = torch.randn((L, B, S + STEPS, 2, H, D), generator=g).half()
    qp = (torch.randn((L, B, S, H, D), generator=g) * 0.5).half()
    qs = torch.randn((STEPS, L, B, H, D), generator=g).half()
    return kv, qp, qs


def _run(h0, nh, reducer=None, whole_step=False):
    """whole_step: skv_swa_decode_step over all layers (the head shards
    exchange every layer's step rows in ONE all-reduce per step); else one
    skv_swa_decode_layer per layer (one exchange per layer-step)."""
    from paper_2403_17312_b200 import api

    kv, qp, qs = _inputs()
    hs = slice(h0, h0 + nh)
    cache = api.SwaCache(L, B, nh, D, S + STEPS, kv_dtype="f16")
    if reducer is not None:
        cache.set_head_shard(h0, H, reducer)
    res = {"out": [], "idx": [], "pf": [], "sp": []}
    for l in range(L):
        cache.append_tokens(l, 0, 0, kv[l, :, :S, 0, hs].contiguous().cuda(), kv[l, :, :S, 1, hs].contiguous().cuda())
        res["pf"].append(cache.prefill_layer(l, qp[l, :, :, hs].contiguous().cuda()).cpu())
        res["sp"].append(cache.prefill_sparsity(l).cpu())
    for j in range(STEPS):
        n = S + j + 1
        if whole_step:
            for l in range(L):
                res["idx"].append(cache.pending_selection(l, n, R).cpu() if j > 0 else torch.zeros(0))
            out = torch.empty((L, B, nh, D), dtype=torch.float16, device="cuda")
            cache.swa_decode_step(n, R, qs[j, :, :, hs].contiguous().cuda(), kv[:, :, n - 1, 0, hs].contiguous().cuda(),
                                  kv[:, :, n - 1, 1, hs].contiguous().cuda(), out)
            res["out"].extend(out.cpu().unbind(0))
            continue
        for l in range(L):
            out, idx, _ = cache.swa_decode_layer(l, n, R, qs[j, l, :, hs].contiguous().cuda(),
                                                 kv[l, :, n - 1, 0, hs].contiguous().cuda(),
                                                 kv[l, :, n - 1, 1, hs].contiguous().cuda(), return_indices=True)
            res["out"].append(out.cpu())
            res["idx"].append(idx.cpu())
    res["imp"] = [cache.importance(l, S + STEPS).cpu() for l in range(L)]
    torch.cuda.synchronize()
    return res


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, path, whole_step=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world, device_id=torch.device("cuda", 0)
                            if backend == "nccl" else None)
    try:
        from paper_2403_17312_b200.shard import dist_reducer, head_shard_range

        h0, nh = head_shard_range(H, world, rank)
        torch.save((h0, nh, _run(h0, nh, dist_reducer(), whole_step)), os.path.join(path, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


def _check(want, parts):
    for h0, nh, got in parts:
        hs = slice(h0, h0 + nh)
        for a, b in zip(want["idx"], got["idx"]):
            assert torch.equal(a, b)  # every shard makes the unsharded selection
        for a, b in zip(want["out"], got["out"]):
            torch.testing.assert_close(b.float(), a[:, hs].float(), rtol=1e-3, atol=1e-3)
        for a, b in zip(want["pf"], got["pf"]):
            torch.testing.assert_close(b.float(), a[:, :, hs].float(), rtol=1e-3, atol=1e-3)
        for a, b in zip(want["imp"], got["imp"]):
            torch.testing.assert_close(b, a, rtol=1e-5, atol=1e-9)  # f32 per-group sums regroup
        for a, b in zip(want["sp"], got["sp"]):
            torch.testing.assert_close(b, a, rtol=0, atol=1e-12)


@pytest.mark.parametrize("whole_step", [False, True])
@pytest.mark.parametrize("world,backend", [(2, "gloo"), (1, "nccl")])
def test_head_sharded_equals_unsharded(tmp_path, world, backend, whole_step):
    want = _run(0, H, whole_step=whole_step)
    mp.start_processes(_worker, args=(world, _free_port(), backend, str(tmp_path), whole_step), nprocs=world,
                       start_method="spawn")
    _check(want, [torch.load(os.path.join(tmp_path, f"rank{r}.pt")) for r in range(world)])


def test_head_shard_argument_errors():
    from paper_2403_17312_b200 import api

    c = api.SwaCache(1, 1, 4, 128, 32, kv_dtype="f16")
    with pytest.raises(api.ContractViolation):  # heads [6, 10) do not fit in 8
        c.set_head_shard(6, 8, lambda buf, st: None)
    with pytest.raises(api.ContractViolation):  # fewer total heads than this shard holds
        c.set_head_shard(0, 2, lambda buf, st: None)
    c.set_head_shard(4, 8, lambda buf, st: None)
    c.set_head_shard(0, 0, None)  # back to unsharded


def test_head_shard_reduce_failure_surfaces():
    """A failing reduce fails the calling entry point (no silent fallback)."""
    from paper_2403_17312_b200 import api

    B, H, D, s = 1, 4, 128, 16
    c = api.SwaCache(1, B, H, D, s + 1, kv_dtype="f16")
    kv = torch.randn(B, s, H, D, device="cuda").half()
    c.append_tokens(0, 0, 0, kv, kv)

    def broken(buf, st):
        raise RuntimeError("link down")

    c.set_head_shard(0, 2 * H, broken)
    with pytest.raises(Exception):
        c.prefill_seed(0, s, torch.randn(B, H, D, device="cuda").half())
        torch.cuda.synchronize()
