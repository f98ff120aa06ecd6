"""Workload generators and the full-size C checkers (CPU; no GPU needed)."""
from __future__ import annotations

import numpy as np

import bench_workloads as bw
from paper_2102_01887_b200 import synth


def test_sweep_seeds_are_per_replica_and_shard_invariant():
    """seeds r*5 + m depend on the global replica index, so a rank's
    shard [r0, r1) reproduces exactly that slice of the single-GPU workload."""
    meta, ops, ref0, cols = bw._c4_meta()
    K = len(meta["kinds"])
    whole = synth.amber_sweep(ref0, K, 0, 6)
    part = synth.amber_sweep(ref0, K, 2, 5)
    per_rep = 5 * 64
    for name in ("ref", "target", "now", "Q", "avail", "supply"):
        assert np.array_equal(getattr(whole, name)[2 * per_rep:5 * per_rep], getattr(part, name)), name
    rng = np.random.default_rng(3 * 5 + 4)  # replica 3, target 10x
    T = 10.0 * synth.SWEEP_CP_MIN
    assert np.array_equal(whole.Q[(3 * 5 + 4) * 64:(3 * 5 + 5) * 64], rng.exponential(0.02 * T, size=(64, K)))
    assert whole.avail.min() >= 1 and whole.avail.max() <= 64


def test_c4_c_oracle_matches_python_oracle():
    """The full-N config-4 checker (C: literal path-list Alg. 1 + OpTable.select scan) agrees
    with the numpy/Python restatement (oracle/slack.py slack_by_kind + oracle/optable.py select)
    decision by decision."""
    meta, ops, ref0, cols = bw._c4_meta()
    K, V = len(meta["kinds"]), len(ops)
    sw = synth.amber_sweep(ref0, K, 7, 9)
    g_names = ops  # value order = op order here
    work = (meta, [tuple(p) for p in meta["paths"]], g_names, 100.0)
    samp = np.arange(0, len(sw.target), 7)
    chk = bw._c4_cpu_worker((work, samp, sw.ref[samp], sw.target[samp], sw.now[samp], sw.Q[samp],
                             sw.avail[samp], sw.supply[samp]))
    from oracle import commit as oc
    from oracle import cselect

    sl = cselect.slack_paths(sw.ref, sw.target, sw.now, sw.Q, cols)
    I = len(sw.target)
    exp = cselect.select_batch(oc.amber_tables(meta), sl.reshape(I * V, K), 100.0, sw.avail.reshape(-1),
                               sw.supply.reshape(-1), np.ones(I * V, np.int32), np.ones(I * V, np.uint32),
                               op=np.tile(np.arange(V, dtype=np.int32), I))
    got = np.stack([exp["idx"].reshape(I, V)[samp], exp["code"].reshape(I, V)[samp]], -1)
    assert np.array_equal(chk, got)
    res = bw.c4_full_parity(meta, cols, ops, sw, 100.0, exp["idx"], exp["code"], exp["obj"])
    assert res["result"] == "bit-identical" and res["decisions"] == I * V
