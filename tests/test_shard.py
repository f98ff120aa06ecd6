"""Multi-rank host logic (world_size 2, gloo on CPU): sharding, exact counter reduction,
deterministic FP aggregation and decision gathering reproduce the single-process result.
Per-shard decisions come from the CPU oracle here; on B200 the same helpers run over NCCL with
the K2 kernel producing the shards (bench.py --gpus N)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_01887_b200.shard import (
    decision_counters, gather_decisions, gather_partials, reduce_counters, shard_range,
)


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, g, world) for g in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload():
    from oracle import optable
    from paper_2102_01887_b200 import synth

    t = optable.from_spec(synth.synth_spec(False), synth.synth_scenario(), ["cpu", "gpu"])
    inv = synth.synth_invocations(600, t.lat, t.gkind, seed=77)
    return t, inv


def _rank_main(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import optable

    t, inv = _workload()
    a, b = shard_range(inv.N, rank, world)
    r = optable.select_many([t], inv.slack, 100.0, inv.avail, inv.supply, inv.min_batch, inv.flags,
                            None, a, b)
    code = torch.from_numpy(r["code"].astype(np.int64) | (r["feasible"].astype(np.int64) << 2))
    counters = reduce_counters(decision_counters(code))
    obj = torch.tensor([float(np.sum(r["obj"]))], dtype=torch.float64)
    total = gather_partials(obj)
    full = gather_decisions({"idx": torch.from_numpy(r["idx"].astype(np.int64)), "code": code}, inv.N)
    if rank == 0:
        torch.save({"counters": counters, "total": total, "idx": full["idx"], "code": full["code"]},
                   out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process(tmp_path):
    from oracle import optable

    out = tmp_path / "r0.pt"
    mp.start_processes(_rank_main, args=(2, _free_port(), str(out)), nprocs=2, join=True,
                       start_method="spawn")
    got = torch.load(out)
    t, inv = _workload()
    r = optable.select_many([t], inv.slack, 100.0, inv.avail, inv.supply, inv.min_batch, inv.flags)
    code = r["code"].astype(np.int64) | (r["feasible"].astype(np.int64) << 2)
    assert np.array_equal(got["idx"].numpy(), r["idx"])
    assert np.array_equal(got["code"].numpy(), code)
    want = decision_counters(torch.from_numpy(code))
    assert torch.equal(got["counters"], want)
    a, b = shard_range(inv.N, 0, 2)
    expect_total = float(np.sum(r["obj"][a:b])) + float(np.sum(r["obj"][b:]))
    assert got["total"].item() == expect_total
