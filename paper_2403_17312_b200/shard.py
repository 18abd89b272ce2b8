"""Multi-GPU plumbing for the SWA decode path: batch sharding (the default)
and head sharding (when there are fewer sequences than GPUs).

Selection is per (sequence, layer) (attention.hpp:235-244), so sequences are
independent: each rank owns a contiguous slice of the batch and runs the
decode path on it with no collective. Collectives are used only for
measurement (max-over-ranks time) and, when a caller wants the whole batch's
outputs on every rank, one all-gather of the attention outputs.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [b0, b0 + nb) of `global_batch` sequences for `rank`;
    the first global_batch % world ranks take one extra sequence."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if global_batch < 0:
        raise ValueError("negative batch")
    base, rem = divmod(global_batch, world)
    b0 = rank * base + min(rank, rem)
    return b0, base + (1 if rank < rem else 0)


def max_over_ranks(value: float, device=None) -> float:
    """The slowest rank's time: what a multi-GPU step costs."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_batch(local: torch.Tensor, global_batch: int) -> torch.Tensor:
    """All-gather per-rank [nb, ...] slices (shard_range order) into the
    global [global_batch, ...] tensor on every rank. Pads uneven shards."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    width = -(-global_batch // world)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    out = [parts[r][: shard_range(global_batch, world, r)[1]] for r in range(world)]
    return torch.cat(out, 0)


def head_shard_range(heads: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous heads [h0, h0 + nh) of `heads` for `rank` (same split rule
    as shard_range). Head sharding is for B < #GPU (SURVEY §8 e): attention
    per head is independent, only the head-summed step row that ranks the
    tokens (head_summed_accum, attention.hpp:77-85) crosses ranks."""
    if heads < world:
        raise ValueError(f"{heads} heads cannot be split over {world} ranks")
    return shard_range(heads, world, rank)


def mesh_coords(world: int, rank: int, head_shards: int) -> tuple[int, int, int]:
    """batch x head mesh: world = batch_groups * head_shards; rank ->
    (batch group, head shard, batch groups). The head shards of one batch
    group are consecutive ranks (one NVSwitch hop either way on a B200 box)."""
    if head_shards < 1 or world % head_shards:
        raise ValueError(f"{head_shards} head shards do not divide {world} ranks")
    return rank // head_shards, rank % head_shards, world // head_shards


def head_groups(world: int, head_shards: int):
    """One process group per batch group over its head shards (every rank
    must call this, in the same order). Returns the list, index = batch group."""
    if head_shards == 1:
        return [None] * world
    return [dist.new_group(list(range(g * head_shards, (g + 1) * head_shards)))
            for g in range(world // head_shards)]


def dist_reducer(group=None):
    """The head-shard exchange (SwaCache.set_head_shard): one SUM all-reduce
    of the fp64 step row across the process group. NCCL (over NVLink on a
    GPU box) is enqueued on the library's stream, so the exchange stays
    asynchronous; host-transport backends (gloo: the -m gpu tests, where two
    ranks share one GPU) synchronise the stream and reduce a host copy."""

    def reduce(buf: torch.Tensor, stream) -> None:
        if dist.get_backend(group) == "nccl":
            with torch.cuda.stream(stream):
                dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
            return
        stream.synchronize()
        host = buf.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        buf.copy_(host)  # on the current stream: synchronise it before the library reads buf
        torch.cuda.current_stream(buf.device).synchronize()

    return reduce
