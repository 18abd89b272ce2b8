"""Multi-rank host logic (gloo, world size 2, CPU): batch sharding of the SWA
decode path has no data-path collective -- every rank decodes its own
sequences -- so the union of the per-rank results must equal the whole-batch
result, and the timing reduction is a max over ranks. The per-rank compute in
this CPU test is the oracle (the GPU kernels are covered by the -m gpu tests).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_17312_b200.shard import gather_batch, max_over_ranks, shard_range


def test_shard_range_partitions():
    for B in (0, 1, 7, 64, 128, 129):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(B, world, r) for r in range(world)]
            assert sum(nb for _, nb in spans) == B
            pos = 0
            for b0, nb in spans:
                assert b0 == pos
                pos += nb
            assert max(nb for _, nb in spans) - min(nb for _, nb in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        from skv_testlib import OracleSeq

        port_ = Oracle("port")
        H, D, s, steps, r = 2, 128, 40, 4, 0.2
        rng = np.random.default_rng(5)  # same global data on every rank
        kv = rng.standard_normal((B, s + steps, 2, H, D))
        qs = rng.standard_normal((steps + 1, B, H, D))
        b0, nb = shard_range(B, world, rank)
        outs = np.zeros((steps, nb, H, D))
        idxs = []
        for i, b in enumerate(range(b0, b0 + nb)):
            seq = OracleSeq(port_, H, D, s + steps)
            for t in range(s):
                seq.append(t, kv[b, t, 0], kv[b, t, 1])
            seq.seed(s, qs[0, b])
            for j in range(steps):
                n = s + j + 1
                seq.append(n - 1, kv[b, n - 1, 0], kv[b, n - 1, 1])
                attn, _, idx = seq.step(n, r, qs[j + 1, b])
                outs[j, i] = attn
                idxs.append(idx)
        gathered = [gather_batch(torch.from_numpy(outs[j]), B).numpy() for j in range(steps)]
        slowest = max_over_ranks(1.0 + rank)
        if rank == 0:
            np.savez(result_path, out=np.stack(gathered), slowest=slowest)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [4, 5])
def test_batch_sharded_decode_equals_whole_batch(tmp_path, B, port):
    from skv_testlib import OracleSeq

    world = 2
    res = str(tmp_path / "r.npz")
    mp.start_processes(_worker, args=(world, _free_port(), B, res), nprocs=world, start_method="spawn")
    got = np.load(res)
    assert got["slowest"] == 2.0  # max over ranks
    H, D, s, steps, r = 2, 128, 40, 4, 0.2
    rng = np.random.default_rng(5)
    kv = rng.standard_normal((B, s + steps, 2, H, D))
    qs = rng.standard_normal((steps + 1, B, H, D))
    for b in range(B):
        seq = OracleSeq(port, H, D, s + steps)
        for t in range(s):
            seq.append(t, kv[b, t, 0], kv[b, t, 1])
        seq.seed(s, qs[0, b])
        for j in range(steps):
            n = s + j + 1
            seq.append(n - 1, kv[b, n - 1, 0], kv[b, n - 1, 1])
            attn, _, _ = seq.step(n, r, qs[j + 1, b])
            assert np.array_equal(got["out"][j, b], attn)


# ---- head sharding (SURVEY §8 e: B < #GPU, e.g. config 1) -------------------
def test_head_shard_range():
    from paper_2403_17312_b200.shard import head_shard_range

    assert [head_shard_range(32, 4, r) for r in range(4)] == [(0, 8), (8, 8), (16, 8), (24, 8)]
    assert [head_shard_range(40, 3, r) for r in range(3)] == [(0, 14), (14, 13), (27, 13)]
    with pytest.raises(ValueError):
        head_shard_range(2, 4, 0)


def _head_worker(rank, world, port, result_path):
    """One sequence, heads split over the ranks. Per step every rank selects
    from its (identical) importance copy, attends over its heads, and the
    head-summed step rows are SUM-all-reduced before the fold -- the exchange
    the library performs through skv_cache_set_head_shard."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle

        from paper_2403_17312_b200.shard import head_shard_range

        o = Oracle("port")
        H, D, s, steps, r = 6, 128, 50, 5, 0.2
        rng = np.random.default_rng(11)
        kv = rng.standard_normal((s + steps, 2, H, D))
        qs = rng.standard_normal((steps + 1, H, D))
        h0, nh = head_shard_range(H, world, rank)
        keys = np.ascontiguousarray(kv[:, 0, h0:h0 + nh].transpose(1, 0, 2))
        vals = np.ascontiguousarray(kv[:, 1, h0:h0 + nh].transpose(1, 0, 2))
        imp = np.zeros(s + steps)
        row = np.zeros(s)  # seed: the last row of the causal prefill, summed over this rank's heads
        for h in range(nh):
            row += o.dense_attention(qs[0, h0 + h][None], keys[h, :s], vals[h, :s], True)[1][0]
        t = torch.from_numpy(row)
        dist.all_reduce(t)
        imp[:s] = t.numpy()
        outs, sels = [], []
        for j in range(steps):
            n = s + j + 1
            sel = o.swa_select(imp[:n - 1], n, r)[0]
            acc = np.zeros((nh, n))
            attn, aw = o.attend_over_indices(keys, vals, acc, n, qs[j + 1, h0:h0 + nh], sel, n)
            t = torch.from_numpy(np.ascontiguousarray(aw))
            dist.all_reduce(t)
            imp[:n - 1] += t.numpy()[:n - 1]
            imp[n - 1] = t.numpy()[n - 1]
            outs.append(attn)
            sels.append(sel)
        parts = [None] * world
        dist.all_gather_object(parts, (h0, outs))
        if rank == 0:
            full = np.zeros((steps, H, D))
            for hh0, po in parts:
                for j in range(steps):
                    full[j, hh0:hh0 + len(po[j])] = po[j]
            np.savez(result_path, out=full, sel=np.stack([np.pad(x, (0, 64 - len(x)), constant_values=-1)
                                                          for x in sels]))
    finally:
        dist.destroy_process_group()


def test_head_sharded_decode_equals_unsharded(tmp_path, port):
    """Head-sharded SWA (world 2, gloo) == the unsharded oracle: identical
    selections, per-head outputs within fp64 rounding of the head-sum order."""
    from skv_testlib import OracleSeq

    world = 2
    res = str(tmp_path / "h.npz")
    mp.start_processes(_head_worker, args=(world, _free_port(), res), nprocs=world, start_method="spawn")
    got = np.load(res)
    H, D, s, steps, r = 6, 128, 50, 5, 0.2
    rng = np.random.default_rng(11)
    kv = rng.standard_normal((s + steps, 2, H, D))
    qs = rng.standard_normal((steps + 1, H, D))
    seq = OracleSeq(port, H, D, s + steps)
    for t in range(s):
        seq.append(t, kv[t, 0], kv[t, 1])
    seq.seed(s, qs[0])
    for j in range(steps):
        n = s + j + 1
        seq.append(n - 1, kv[n - 1, 0], kv[n - 1, 1])
        attn, _, idx = seq.step(n, r, qs[j + 1])
        sel = got["sel"][j]
        assert np.array_equal(sel[sel >= 0], idx), j
        np.testing.assert_allclose(got["out"][j], attn, rtol=1e-12, atol=1e-14)


def test_mesh_coords():
    from paper_2403_17312_b200.shard import mesh_coords

    assert [mesh_coords(8, r, 2) for r in range(8)] == [(r // 2, r % 2, 4) for r in range(8)]
    assert [mesh_coords(4, r, 4) for r in range(4)] == [(0, r, 1) for r in range(4)]
    assert mesh_coords(8, 5, 1) == (5, 0, 8)
    with pytest.raises(ValueError):
        mesh_coords(8, 0, 3)
