"""Batched commit step against the reference engine's own rounds.

tests/golden/commit_rounds.npz holds 24,000 Configurator.pump_commits rounds recorded from the
unmodified reference running the AMBER scenario (50% target, fast target, pbc and eslc
ablations), interleaved with the set_latency calls that change the tables.  Rounds between two
latency updates are independent computations, so they go to the device as one batched
sp_commit_round call; every _commit_candidate result (entry, fill target, slack, objective) and
every round's committed op must match bit-for-bit."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, golden_json
from test_gpu_amber import amber_tables

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _rounds_input(d, idx, n_ops, K):
    R = len(idx)
    slack = np.zeros((R, n_ops, K))
    fill = np.zeros((R, n_ops), np.int32)
    buf = np.zeros((R, n_ops), np.int32)
    hid = np.zeros((R, n_ops), np.int64)
    hf = np.zeros((R, n_ops), np.uint32)
    sidx = np.zeros((R, n_ops), np.int32)
    ssl = np.zeros((R, n_ops))
    sob = np.zeros((R, n_ops))
    full = np.zeros(R, np.uint32)
    exp = {"idx": np.full((R, n_ops), -1, np.int32), "fill": np.zeros((R, n_ops), np.int32),
           "slack": np.zeros((R, n_ops)), "obj": np.zeros((R, n_ops)), "present": np.zeros((R, n_ops), bool)}
    for r, i in enumerate(idx):
        a, n = int(d["r_first_cand"][i]), int(d["r_n_cand"][i])
        for c in range(a, a + n):
            j = int(d["c_op"][c])
            slack[r, j] = np.nan_to_num(d["c_slack"][c], nan=0.0)
            fill[r, j] = d["c_fill"][c]
            buf[r, j] = d["c_buffered"][c]
            hid[r, j] = d["c_inv"][c]
            hf[r, j] = 1 | (2 if d["c_forced"][c] else 0)
            sidx[r, j] = max(int(d["c_spec_idx"][c]), 0)
            ssl[r, j] = d["c_spec_slack"][c]
            sob[r, j] = d["c_spec_obj"][c]
            full[r] = d["c_full_mask"][c]
            exp["idx"][r, j] = d["c_r_idx"][c]
            exp["fill"][r, j] = d["c_r_fill"][c]
            exp["slack"][r, j] = d["c_r_slack"][c]
            exp["obj"][r, j] = d["c_r_obj"][c]
            exp["present"][r, j] = True
    return (slack, fill, buf, hid, hf, sidx, ssl, sob, full), exp


def test_commit_rounds_replay(gpu_ctx):
    import paper_2102_01887_b200 as sp

    d = golden("commit_rounds")
    meta = golden_json(d, "meta_json")
    amb = golden_json(golden("amber_trace"), "meta_json")
    K = len(meta["kinds"])
    n_ops = len(meta["ops"])
    total = calls = 0
    for ri, rm in enumerate(meta["runs"]):
        tabs = amber_tables(amb)
        for t, name in zip(tabs, meta["ops"]):
            lat = np.asarray(rm["tables"][name]["lat"], dtype=np.float64)
            for e in range(len(lat)):
                if lat[e] != t.lat[e]:
                    t.set_latency(e, float(lat[e]))
        policy = sp.commit.policy_of(rm["ablations"])
        ev = [(int(s), 0, i) for i, s in enumerate(d["s_seq"]) if d["s_run"][i] == ri]
        ev += [(int(s), 1, i) for i, s in enumerate(d["r_seq"]) if d["r_run"][i] == ri]
        ev.sort()
        pending = []

        def flush():
            nonlocal total, calls
            if not pending:
                return
            args, exp = _rounds_input(d, pending, n_ops, K)
            slack, fill, buf, hid, hf, sidx, ssl, sob, full = args
            got = sp.commit_round(tabs, slack, fill, buf, hid, np.asarray(rm["depths"], np.int32), hf,
                                  alpha=rm["alpha"], full_mask=full, policy=policy, spec_idx=sidx,
                                  spec_slack=ssl, spec_obj=sob)
            p = exp["present"]
            assert np.array_equal(got["idx"][p], exp["idx"][p])
            some = p & (exp["idx"] >= 0)
            assert np.array_equal(got["fill"][some], exp["fill"][some])
            assert np.array_equal(bits(got["slack"][some]), bits(exp["slack"][some]))
            assert np.array_equal(bits(got["obj"][some]), bits(exp["obj"][some]))  # NaN: same bits
            assert np.array_equal(got["best"], np.asarray([d["r_winner_op"][i] for i in pending]))
            total += len(pending)
            calls += 1
            pending.clear()

        for _, typ, i in ev:
            if typ == 0:
                flush()
                tabs[d["s_op"][i]].set_latency(int(d["s_idx"][i]), float(d["s_val"][i]))
            else:
                pending.append(i)
        flush()
    assert total == len(d["r_run"])


def test_commit_candidates_single_round(gpu_ctx):
    """The per-round host form (what a GPU-backed pump_commits calls) on the first recorded
    rounds of the 50% run, with reference-shaped head objects."""
    import types

    import paper_2102_01887_b200 as sp

    d = golden("commit_rounds")
    meta = golden_json(d, "meta_json")
    amb = golden_json(golden("amber_trace"), "meta_json")
    tabs = amber_tables(amb)
    rm = meta["runs"][0]
    first_setl = int(d["s_seq"][0]) if len(d["s_seq"]) else 1 << 60
    checked = 0
    for i in range(len(d["r_run"])):
        if d["r_run"][i] != 0 or d["r_seq"][i] > first_setl or checked >= 50:
            break
        a, n = int(d["r_first_cand"][i]), int(d["r_n_cand"][i])
        heads, slacks, buf = [None] * len(tabs), [{}] * len(tabs), [0] * len(tabs)
        full = set()
        for c in range(a, a + n):
            j = int(d["c_op"][c])
            heads[j] = types.SimpleNamespace(fill=int(d["c_fill"][c]), forced=bool(d["c_forced"][c]),
                                             invocation_id=int(d["c_inv"][c]),
                                             spec_eidx=int(d["c_spec_idx"][c]),
                                             spec_slack_s=float(d["c_spec_slack"][c]),
                                             spec_objective=float(d["c_spec_obj"][c]))
            slacks[j] = {k: float(v) for k, v in zip(meta["kinds"], d["c_slack"][c]) if v == v}
            buf[j] = int(d["c_buffered"][c])
            full = {k for b, k in enumerate(meta["kinds"]) if (int(d["c_full_mask"][c]) >> b) & 1}
        w = sp.commit_candidates(tabs, slacks, heads, buf, rm["depths"], full, rm["alpha"])
        assert (w[0] if w else -1) == d["r_winner_op"][i]
        checked += 1
    assert checked > 10
