"""Multi-GPU sharding of the hot path.

Invocation batches (configs 2/5), pipeline instances (config 3) and scenario replicas (config 4)
are independent units: rank g owns the contiguous range ``[g*N/G, (g+1)*N/G)``, profile tables
are replicated, and there is no collective on the data path.  The helpers below are the only
exchange steps, used when a caller wants whole-job results:

* ``reduce_counters``   exact integer decision counters, all-reduce SUM (int64)
* ``gather_partials``   per-rank FP partial sums, all-gathered and summed on every rank in
                        rank order (deterministic for a fixed world size)
* ``gather_decisions``  the decision records of every shard, in global invocation order
* ``gather_observations``  online mode (config 5): the 16-byte observation records (table
                        entry, observed latency) of every shard of a batch, in global invocation
                        order, so every rank folds the identical ordered stream and the replicated
                        profile tables stay bit-identical without a broadcast

They take torch tensors and work with NCCL (CUDA tensors, B200 / NVLink) and gloo (CPU tensors,
the multi-process CPU tests).
"""
from __future__ import annotations

from typing import Mapping, Sequence


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard of ``n`` units owned by ``rank`` (sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def decision_counters(code):
    """[none, assign, delay, feasible] counts of a decision-code tensor (int64)."""
    import torch

    kind = code & 3
    return torch.stack([
        (kind == 0).sum(), (kind == 1).sum(), (kind == 2).sum(), ((code >> 2) & 1).sum(),
    ]).to(torch.int64)


def reduce_counters(counters, group=None):
    import torch.distributed as dist

    out = counters.clone()
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def gather_partials(partial, group=None):
    """All-gather one FP partial per rank; returns the rank-ordered sum (same on every rank)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return partial.clone()
    world = dist.get_world_size(group)
    parts = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(parts, partial, group=group)
    total = parts[0].clone()
    for p in parts[1:]:
        total = total + p
    return total


def gather_decisions(arrays: Mapping[str, "object"], n_total: int, group=None) -> dict:
    """All-gather per-shard decision arrays (shards from ``shard_range``) into full arrays."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return {k: v.clone() for k, v in arrays.items()}
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, g, world) for g in range(world)]
    longest = max(b - a for a, b in sizes)
    out = {}
    for name, v in arrays.items():
        pad = torch.zeros((longest,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)
        pad[: v.shape[0]] = v
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        out[name] = torch.cat([p[: b - a] for p, (a, b) in zip(parts, sizes)])
    return out


def gather_observations(idx, obs, n_total: int, group=None):
    """All-gather one batch's observation records from every shard (``shard_range`` layout).

    ``idx`` (int32, entry index or -1 for "no observation") and ``obs`` (float64) are this rank's
    shard; returns the whole batch ``(idx, obs)`` in global invocation order on every rank.  The
    records travel as one (n, 2) float64 tensor (16 B per observation, the index is exact in f64),
    i.e. one collective per batch.
    """
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return idx.clone(), obs.clone()
    rec = torch.stack([idx.to(torch.float64), obs.to(torch.float64)], dim=1)
    full = gather_decisions({"rec": rec}, n_total, group=group)["rec"]
    return full[:, 0].to(torch.int32), full[:, 1].contiguous()
