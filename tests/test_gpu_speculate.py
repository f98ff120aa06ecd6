"""Speculation loop against the reference engine's own calls.

tests/golden/speculate_calls.npz holds 15,000 Configurator.speculate_from_buffer calls recorded
from the unmodified reference running the AMBER scenario (50 % and 25 % targets, dfp ablation),
interleaved with the set_latency calls that change the tables.  Calls between two latency
updates are independent, so they go to the device as one sp_speculate_batch call; every
invocation formed (entry, fill, slack, objective) and every stopping delay (entry, wait budget)
must match bit-for-bit.  A synthetic batch of 4,096 calls with multi-step loops checks the
device against the oracle restatement where the recorded runs are thin (long buffers, forced
warm-up, expired holds)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import golden, golden_json
from test_gpu_amber import amber_tables
from test_oracle_golden import speculate_call_inputs

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _pack(calls, K):
    """[(sq, cq)] -> w_ptr, w_tab, w_eidx, w_count in (call, queue, kind) order."""
    ptr, tab, eidx, cnt = [0], [], [], []
    for sq, cq in calls:
        for lists in (sq, cq):
            for k in range(K):
                for tb, e, c in lists[k]:
                    tab.append(tb)
                    eidx.append(e)
                    cnt.append(c)
                ptr.append(len(tab))
    return ptr, tab, eidx, cnt


def test_speculate_calls_replay(gpu_ctx):
    import paper_2102_01887_b200 as sp

    d = golden("speculate_calls")
    meta = golden_json(d, "meta_json")
    amb = golden_json(golden("amber_trace"), "meta_json")
    K = len(meta["kinds"])
    checked = formed = batches = 0
    for ri, rm in enumerate(meta["runs"]):
        tabs = amber_tables(amb)
        for t, name in zip(tabs, meta["ops"]):
            lat = np.asarray(rm["tables"][name]["lat"], dtype=np.float64)
            for e in range(len(lat)):
                if lat[e] != t.lat[e]:
                    t.set_latency(e, float(lat[e]))
        ev = [(int(s), 0, i) for i, s in enumerate(d["s_seq"]) if d["s_run"][i] == ri]
        ev += [(int(s), 1, i) for i, s in enumerate(d["c_seq"]) if d["c_run"][i] == ri]
        ev.sort()
        pending = []

        def flush():
            nonlocal checked, formed, batches
            if not pending:
                return
            ids = np.array(pending)
            w = _pack([speculate_call_inputs(d, i, K) for i in ids], K)
            r = sp.speculate_batch(tabs, rm["alpha"], rm["pool"], d["c_op"][ids], d["c_n"][ids],
                                   d["c_supply"][ids], d["c_now"][ids], d["c_target"][ids],
                                   d["c_rmin"][ids], d["c_rmax"][ids], d["c_slack0"][ids],
                                   d["c_flags"][ids], *w)
            for q, i in enumerate(ids):
                a, n = int(d["c_d_first"][i]), int(d["c_d_n"][i])
                assert r["n"][q] == n, i
                o = int(r["off"][q])
                assert np.array_equal(r["idx"][o:o + n], d["d_idx"][a:a + n]), i
                assert np.array_equal(r["fill"][o:o + n], d["d_fill"][a:a + n]), i
                assert np.array_equal(bits(r["slack"][o:o + n]), bits(d["d_slack"][a:a + n])), i
                exp_obj = d["d_obj"][a:a + n]
                got_obj = r["obj"][o:o + n]
                assert all((math.isnan(x) and math.isnan(y)) or x == y for x, y in zip(got_obj, exp_obj)), i
                assert r["delay_idx"][q] == d["c_delay_idx"][i], i
                assert bits(r["delay_wait"][q]) == bits(d["c_delay_wait"][i]), i
                formed += n
            checked += len(ids)
            batches += 1
            pending.clear()

        for _, typ, i in ev:
            if typ == 0:
                flush()
                tabs[d["s_op"][i]].set_latency(int(d["s_idx"][i]), float(d["s_val"][i]))
            else:
                pending.append(i)
        flush()
        for t in tabs:
            t.close()
    assert checked == 15000 and formed > 7000 and batches > 100


def test_speculate_synthetic_batch_vs_oracle(gpu_ctx):
    """4,096 synthetic calls on the AMBER tables with long buffers, random weights, forced
    warm-up and expired holds — device vs oracle/speculate.py."""
    import paper_2102_01887_b200 as sp
    from oracle import commit as oc
    from oracle import speculate as osp

    amb = golden_json(golden("amber_trace"), "meta_json")
    tabs = amber_tables(amb)
    otabs = oc.amber_tables(amb)
    K = len(amb["kinds"])
    rng = np.random.default_rng(17)
    R = 4096
    pk = {k: float(n * r) for k, n, r, _ in amb["backends"]}
    pool = [pk[k] for k in amb["kinds"]]
    alpha = 100.0
    ops = rng.integers(0, len(tabs), R)
    n_buf = rng.integers(1, 40, R)
    supply = rng.integers(0, 60, R)
    now = rng.uniform(0, 100, R)
    target = now + rng.uniform(-5, 80, R)
    rmin = rng.uniform(0.05, 0.5, R)
    rmax = rmin + rng.uniform(0, 0.5, R)
    flags = (rng.random(R) < 0.8).astype(np.uint32) | \
        np.where((rng.random(R) < 0.1) & np.array([otabs[o].ref_index >= 0 for o in ops]), 2, 0).astype(np.uint32) | \
        np.where(rng.random(R) < 0.1, 4, 0).astype(np.uint32)
    slack0 = rng.uniform(-2, 60, (R, K))
    calls = []
    for r in range(R):
        sq = [[] for _ in range(K)]
        cq = [[] for _ in range(K)]
        for _ in range(rng.integers(0, 8)):
            tb = int(rng.integers(0, len(tabs)))
            e = int(rng.integers(0, len(otabs[tb].lat)))
            k = int(otabs[tb].gkind[e])
            lst = sq if rng.random() < 0.6 else cq
            if not any(x[0] == tb and x[1] == e for x in lst[k]):
                lst[k].append([tb, e, int(rng.integers(1, 5))])
        calls.append((sq, cq))
    w = _pack(calls, K)
    res = sp.speculate_batch(tabs, alpha, pool, ops, n_buf, supply, now, target, rmin, rmax,
                             slack0, flags, *w)
    multi = 0
    for r in range(R):
        sq = [[list(x) for x in lst] for lst in calls[r][0]]
        cq = calls[r][1]
        dec, delay = osp.speculate(otabs, int(ops[r]), int(n_buf[r]), int(supply[r]), float(now[r]),
                                   float(target[r]), float(rmin[r]), float(rmax[r]), pool, alpha,
                                   int(flags[r]), sq, cq, slack0[r])
        assert res["n"][r] == len(dec), r
        o = int(res["off"][r])
        for j, (e, fill, s_k, obj) in enumerate(dec):
            assert res["idx"][o + j] == e and res["fill"][o + j] == fill, r
            assert bits(res["slack"][o + j]) == bits(s_k), r
            assert (math.isnan(obj) and math.isnan(res["obj"][o + j])) or res["obj"][o + j] == obj, r
        if delay is None:
            assert res["delay_idx"][r] == -1, r
        else:
            assert res["delay_idx"][r] == delay[0] and bits(res["delay_wait"][r]) == bits(delay[1]), r
        multi += len(dec) > 1
    assert multi > 500
    for t in tabs:
        t.close()
