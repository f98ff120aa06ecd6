"""The one-kernel cluster plan builder (sp_plan_cluster.cu) against the multi-kernel builder
(sp_plan.cu) and the CPU restatement (oracle/plan.py): every section of the plan image —
header counts, batch lookup table, per-kind thresholds, bucket tables and staircase rows, and
the candidate records — bit-identical, on the config-2 / config-5 tables at every alpha, the
AMBER tables, and heavily tied random tables (zero / negative latencies, 1..8 kinds, 1..16
batch sizes)."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import optable, plan
from test_gpu_select import _random_table, raw_table

pytestmark = pytest.mark.gpu


def _check(tab, K, alpha, arrays):
    cl = plan.parse_image(tab.plan_image(alpha, "cluster"))
    lg = plan.parse_image(tab.plan_image(alpha, "legacy"))
    assert cl["magic"] == lg["magic"] == 0x53504C4E
    assert plan.compare(cl, lg) == [], plan.compare(cl, lg)
    exp = plan.plan_image(*arrays, K, alpha)
    assert plan.compare(cl, exp) == [], plan.compare(cl, exp)
    assert cl["total_bytes"] == lg["total_bytes"]


@pytest.mark.parametrize("with_model", [False, True])
def test_cluster_plan_synthetic_tables(gpu_ctx, with_model):
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    spec = synth.synth_spec(with_model)
    tab = sp.OpTable(spec, synth.synth_scenario())
    t = optable.from_spec(spec, synth.synth_scenario(), ["cpu", "gpu"])
    arrays = (t.lat, t.res, t.batch_int, t.pool, t.price, t.gkind, t.id_rank)
    for alpha in ((0.0, 1.0, 100.0, 1000.0) if not with_model else (100.0, 0.0)):
        _check(tab, 2, alpha, arrays)
    tab.close()


def test_cluster_plan_amber_tables(gpu_ctx):
    import bench_workloads as bw
    import paper_2102_01887_b200 as sp
    from oracle import commit as oc

    with np.load(GOLDEN / "amber_trace.npz") as z:
        meta = json.loads(bytes(z["meta_json"]).decode())
    tabs = bw._amber_tables(sp, meta)
    otabs = oc.amber_tables(meta)
    K = len(meta["kinds"])
    for tab, t in zip(tabs, otabs):
        arrays = (t.lat, t.res, t.batch_int, t.pool, t.price, t.gkind, t.id_rank)
        for alpha in (100.0, 0.0):
            _check(tab, K, alpha, arrays)


@pytest.mark.parametrize("seed,M,nB,K,nonpos", [(1, 3000, 8, 2, False), (2, 2000, 16, 4, False),
                                                (3, 700, 13, 3, False), (4, 5000, 5, 8, False),
                                                (5, 1, 1, 1, False), (6, 64, 2, 2, False),
                                                (7, 900, 8, 2, True), (8, 300, 11, 3, True),
                                                (9, 12000, 16, 6, False)])
def test_cluster_plan_random_tables(gpu_ctx, seed, M, nB, K, nonpos):
    rng = np.random.default_rng(seed)
    t = _random_table(rng, M, nB, K, nonpos)
    tab = raw_table(t, K)
    arrays = (t.lat, t.res, t.batch_int, t.pool, t.price, t.gkind, t.id_rank)
    for alpha in (0.0, 7.5, 1000.0):
        _check(tab, K, alpha, arrays)
    tab.close()


@pytest.mark.parametrize("seed,M,nB,K,nonpos", [(11, 3000, 8, 2, False), (12, 900, 8, 2, True),
                                                (13, 4000, 16, 3, False)])
def test_cluster_plan_incremental_updates(gpu_ctx, seed, M, nB, K, nonpos):
    """The cluster builder keeps each segment's latency order between builds and merges only the
    entries whose latency changed (set_latency, the fold, the gate-lift rescale).  After every
    kind of update — a few entries, ties with unchanged entries, moves to the extremes, zero /
    negative values, more entries than the incremental cap — the image must equal the CPU
    restatement built from scratch and the multi-kernel builder."""
    import paper_2102_01887_b200 as sp

    rng = np.random.default_rng(seed)
    t = _random_table(rng, M, nB, K, nonpos)
    tab = raw_table(t, K)
    lat = t.lat.copy()
    arrays = lambda: (lat, t.res, t.batch_int, t.pool, t.price, t.gkind, t.id_rank)
    _check(tab, K, 7.5, arrays())
    for step in range(12):
        if step % 3 == 2:  # the fold writes the observed entries (dirty flags set on the device)
            n = int(rng.integers(1, 400))
            idx = rng.choice(rng.choice(M, size=int(rng.integers(1, 40)), replace=False), size=n).astype(np.int32)
            obs = rng.uniform(0.01, 5.0, size=n)
            sp.fold_observations([tab], None, idx, obs, beta=0.5, dfp_count=10**9, sync_host=False)
            lat = np.asarray(tab.get_latency()).copy()
        else:
            m = [3, 40, 700][step % 3] if step < 9 else int(rng.integers(1, 20))
            ix = rng.choice(M, size=min(m, M), replace=False).astype(np.int32)
            v = rng.uniform(0.01, 5.0, size=len(ix))
            tie = rng.random(len(ix)) < 0.4
            v[tie] = rng.choice(lat, size=int(tie.sum()))                 # exact ties with others
            v[rng.random(len(ix)) < 0.1] = lat.min() * 0.5                 # new minimum
            v[rng.random(len(ix)) < 0.1] = lat.max() * 2.0                 # new maximum
            if nonpos:
                v[rng.random(len(ix)) < 0.1] = 0.0
                v[rng.random(len(ix)) < 0.1] = -1.5
            tab.set_latency(ix, v)
            lat[ix] = v
        for alpha in (7.5,) if step % 2 else (0.0, 1000.0):
            _check(tab, K, alpha, arrays())
    tab.close()


@pytest.mark.parametrize("seed,M,nB,K,nonpos", [(21, 4096, 8, 2, False), (22, 1500, 16, 3, True),
                                                (23, 3000, 8, 4, False)])
def test_multi_plan_build(gpu_ctx, seed, M, nB, K, nonpos):
    """sp_table_prepare_many: the plans of several alphas built by ONE launch (one cluster per
    plan, the table's cached order replaced afterwards) — every image equal to the CPU
    restatement, after from-scratch invalidations and after incremental latency changes, and the
    decisions taken with them equal to the oracle's."""
    import paper_2102_01887_b200 as sp
    from oracle import cselect

    rng = np.random.default_rng(seed)
    t = _random_table(rng, M, nB, K, nonpos)
    tab = raw_table(t, K)
    lat = t.lat.copy()
    alphas = [0.0, 1.0, 100.0, 1000.0]
    for step in range(5):
        if step == 0:
            tab.invalidate_plans()
        else:
            ix = rng.choice(M, size=int(rng.integers(1, 300)), replace=False).astype(np.int32)
            v = rng.uniform(0.01, 5.0, size=len(ix))
            tie = rng.random(len(ix)) < 0.3
            v[tie] = rng.choice(lat, size=int(tie.sum()))  # exact ties with other entries
            tab.set_latency(ix, v)
            lat[ix] = v
        tab.prepare_many(alphas[: 2 + step % 3])
        for al in alphas[: 2 + step % 3]:
            img = plan.parse_image(tab.plan_image(al, "current"))
            exp = plan.plan_image(lat, t.res, t.batch_int, t.pool, t.price, t.gkind, t.id_rank, K, al)
            assert plan.compare(img, exp) == [], (step, al, plan.compare(img, exp))
    # decisions on the multi-built plans
    tab.invalidate_plans()
    tab.prepare_many(alphas)
    ot = optable.from_columns(lat=lat, res=t.res, batch=t.batch, pool=t.pool, price=t.price,
                              gkind=t.gkind, id_rank=t.id_rank, n_kinds=K)
    N = 2048
    slack = rng.uniform(-2, 10, size=(N, K))
    avail = rng.integers(1, 129, size=N).astype(np.int32)
    supply = rng.integers(0, 257, size=N).astype(np.int32)
    mb = np.ones(N, np.int32)
    flags = sp.make_flags(rng.random(N) < 0.5, 0)
    for al in alphas:
        got = sp.select_batch([tab], slack, al, avail, upstream_supply=supply, min_batch=mb,
                              flags=flags, mode="plan")
        exp = cselect.select_batch([ot], slack, al, avail, supply, mb, flags)
        assert np.array_equal(got["idx"], exp["idx"]), al
        assert np.array_equal(got["code"] & 3, exp["code"]), al
