"""Multi-rank host logic (world_size 2, gloo on CPU): sharding, exact counter reduction,
deterministic FP aggregation and decision gathering reproduce the single-process result.
Per-shard decisions come from the CPU oracle here; on B200 the same helpers run over NCCL with
the K2 kernel producing the shards (bench.py --gpus N)."""
from __future__ import annotations

import os
import socket
from pathlib import Path

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


# ---- online mode (config 5): per-batch all-gather of observation records ---------------------

def _online_batches():
    from oracle import optable
    from paper_2102_01887_b200 import synth

    t = optable.from_spec(synth.synth_spec(False), synth.synth_scenario(), ["cpu", "gpu"])
    inv = synth.synth_invocations(3 * 400, t.lat, t.gkind, seed=505)
    noise = np.exp(np.random.default_rng(9).normal(0.0, 0.3, size=inv.N))
    return t, inv, noise, 400


def _online_run(t, inv, noise, B, lo_hi, gather):
    """Decide each batch (this rank's shard) against the batch-start table, turn assigns into
    observations, gather the whole batch's records, fold them in global order."""
    from oracle import feedback, optable

    lat_init = t.lat.copy()
    st = feedback.FoldState(t.lat.copy(), lat_init, t.ref_index)
    for bt in range(inv.N // B):
        t.lat = st.lat.copy()  # batch-start snapshot
        a, b = lo_hi
        r = optable.select_many([t], inv.slack, 100.0, inv.avail, inv.supply, inv.min_batch, inv.flags,
                                None, bt * B + a, bt * B + b)
        idx = np.where(r["code"] == optable.ASSIGN, r["idx"], -1).astype(np.int32)
        obs = lat_init[np.maximum(idx, 0)] * noise[bt * B + a: bt * B + b]
        f_idx, f_obs = gather(idx, obs)
        keep = f_idx >= 0
        feedback.fold([st], None, f_idx[keep], f_obs[keep], beta=0.5, dfp_count=10)
    return st.lat


def _online_rank_main(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2102_01887_b200.shard import gather_observations

    t, inv, noise, B = _online_batches()

    def gather(idx, obs):
        gi, go = gather_observations(torch.from_numpy(idx), torch.from_numpy(obs), B)
        return gi.numpy(), go.numpy()

    lat = _online_run(t, inv, noise, B, shard_range(B, rank, world), gather)
    torch.save(torch.from_numpy(lat), f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_online_fold_keeps_replicas_identical(tmp_path):
    """Config 5 semantics at world_size 2: every rank folds the gathered, globally ordered
    observation stream, so the replicated tables end bit-identical to each other and to the
    single-process run."""
    out = tmp_path / "lat"
    mp.start_processes(_online_rank_main, args=(2, _free_port(), str(out)), nprocs=2, join=True,
                       start_method="spawn")
    l0 = torch.load(f"{out}.0").numpy()
    l1 = torch.load(f"{out}.1").numpy()
    t, inv, noise, B = _online_batches()
    single = _online_run(t, inv, noise, B, (0, B), lambda i, o: (i, o))
    assert np.array_equal(l0.view(np.uint64), l1.view(np.uint64))
    assert np.array_equal(l0.view(np.uint64), single.view(np.uint64))
    assert not np.array_equal(single, _online_batches()[0].lat)  # the fold did change the table


def test_bench_spawns_ranks_itself():
    """`bench.py --gpus 2` outside torchrun launches two ranks itself (torch.distributed.run on
    127.0.0.1); in --dist-selftest mode they rendezvous over gloo on the CPU and run the shard /
    counter / max-time / observation-gather plumbing of the GPU arms."""
    import json
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(Path(__file__).resolve().parent.parent / "bench.py"),
                        "--gpus", "2", "--dist-selftest"], capture_output=True, text=True,
                       timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["world"] == 2 and line["ranks_ok"] and line["t_max"] == 0.002
