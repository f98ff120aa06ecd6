"""K1 -> K2 fused kernel (sp_slack_select_batch) against the two-kernel path and the oracle.

Config-4 shaped snapshots on the AMBER pipeline (7 operations, 3 decomposed paths, 4 backend
kinds): per instance a target, a clock, per-kind queueing and drifted reference latencies; one
invocation of every operation is decided from that instance's slack.  The fused kernel must
reproduce, bit for bit, K1's slack (sp_slack_batch) fed to K2 (sp_select_batch), and the
oracle's compute_slack + OpTable.select on a sample."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import golden, golden_json
from test_gpu_amber import amber_tables

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _snapshots(meta, I, seed):
    rng = np.random.default_rng(seed)
    ops = meta["ops"]
    V, K = len(ops), len(meta["kinds"])
    ref0 = np.array([meta["tables"][o]["lat"][meta["tables"][o]["ref_index"]]
                     if meta["tables"][o]["ref_index"] >= 0 else 1.0 for o in ops])
    target = rng.uniform(0.5, 10.0, size=I) * 90.41885182994682
    now = rng.uniform(0.0, 1.0, size=I) * target
    Q = rng.exponential(1.0, size=(I, K)) * (0.02 * target)[:, None]
    Q[::7] *= 40.0  # some negative budgets
    ref = ref0[None, :] * np.exp(rng.normal(0.0, 0.2, size=(I, V)))
    N = I * V
    avail = rng.integers(1, 65, size=N).astype(np.int32)
    supply = rng.integers(0, 65, size=N).astype(np.int32)
    mb = np.where(rng.random(N) < 0.8, 1, rng.integers(1, 9, size=N)).astype(np.int32)
    flags = (rng.random(N) < 0.5).astype(np.uint32) | ((rng.random(N) < 0.1).astype(np.uint32) << 9)
    return ref, target, now, Q, avail, supply, mb, flags


@pytest.mark.parametrize("alpha", [0.0, 100.0])
def test_fused_matches_two_kernels(gpu_ctx, alpha):
    import paper_2102_01887_b200 as sp

    meta = golden_json(golden("amber_trace"), "meta_json")
    tabs = amber_tables(meta)
    g = sp.SlackGraph.from_paths([tuple(p) for p in meta["paths"]], meta["ops"])
    vpos = [meta["ops"].index(n) for n in g.value_names]
    ref, target, now, Q, avail, supply, mb, flags = _snapshots(meta, 20000, seed=4)
    refv = np.ascontiguousarray(ref[:, vpos])
    fused = g.slack_select_batch(tabs, alpha, refv, target, now, Q, avail, upstream_supply=supply,
                                 min_batch=mb, flags=flags, kslack=True)
    V, K = len(meta["ops"]), len(meta["kinds"])
    s = g.slack_batch(refv, target, now, Q)["slack"].reshape(-1, K)
    assert np.array_equal(bits(fused["kslack"]), bits(s))
    op = np.tile(np.arange(V, dtype=np.int32), len(target))
    two = sp.select_batch(tabs, np.ascontiguousarray(s), alpha, avail, upstream_supply=supply,
                          min_batch=mb, flags=flags, op=op)
    for k in ("idx", "code", "fill"):
        assert np.array_equal(fused[k], two[k]), k
    some = (two["code"] & 3) != 0
    for k in ("obj", "slack", "wait"):
        assert np.array_equal(bits(fused[k][some]), bits(two[k][some])), k
    # the generic-decision fused kernel and the two-kernel fallback inside the library agree
    for env in ("SP_K12_GENERIC", "SP_NO_K12"):
        os.environ[env] = "1"
        try:
            fb = g.slack_select_batch(tabs, alpha, refv, target, now, Q, avail, upstream_supply=supply,
                                      min_batch=mb, flags=flags)
        finally:
            del os.environ[env]
        assert np.array_equal(fb["idx"], fused["idx"]) and np.array_equal(fb["code"], fused["code"]), env
        assert np.array_equal(fb["fill"], fused["fill"]), env
        for k in ("obj", "slack", "wait"):
            assert np.array_equal(bits(fb[k][some]), bits(fused[k][some])), (env, k)


def test_fused_matches_oracle_sample(gpu_ctx):
    import paper_2102_01887_b200 as sp
    from oracle import commit as oc, optable, slack as osl

    meta = golden_json(golden("amber_trace"), "meta_json")
    tabs = amber_tables(meta)
    otabs = oc.amber_tables(meta)
    g = sp.SlackGraph.from_paths([tuple(p) for p in meta["paths"]], meta["ops"])
    vpos = [meta["ops"].index(n) for n in g.value_names]
    ref, target, now, Q, avail, supply, mb, flags = _snapshots(meta, 300, seed=9)
    refv = np.ascontiguousarray(ref[:, vpos])
    got = g.slack_select_batch(tabs, 100.0, refv, target, now, Q, avail, upstream_supply=supply,
                               min_batch=mb, flags=flags)
    ops, kinds = meta["ops"], meta["kinds"]
    paths = [tuple(p) for p in meta["paths"]]
    V = len(ops)
    for i in range(0, 300, 7):
        refd = {o: float(ref[i, j]) for j, o in enumerate(ops)}
        for s, op in enumerate(ops):
            sl = np.array([osl.compute_slack(op, target_s=float(target[i]), elapsed_s=float(now[i]),
                                             queueing_s=float(Q[i, kk]), paths=paths, ref=refd)
                           for kk in range(len(kinds))])
            d = i * V + s
            fl = int(flags[d])
            r = optable.select(otabs[s], sl, 100.0, int(avail[d]), allow_delay=bool(fl & 1),
                               upstream_supply=int(supply[d]), excluded_mask=fl >> 8,
                               min_batch=int(mb[d]))
            assert (got["code"][d] & 3) == r[0] and got["idx"][d] == r[1], (i, op)
            if r[0]:
                assert got["fill"][d] == r[2] and bits(got["obj"][d]) == bits(r[3])
