"""Pin the CPU oracle against the reference's golden vectors (CPU only, no GPU).

The oracle is the checker of every GPU parity test, so it is itself checked here against
fixtures produced by the unmodified reference (tests/golden/make_golden.py) and, in the build
container, against the live reference on fresh inputs.
"""
from __future__ import annotations

import math
import random

import numpy as np
import pytest

from conftest import KINDS3, golden, golden_json, select_case_specs
from oracle import cselect, feedback, optable, queueing, slack


def _same(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.array_equal(a.view(np.uint64), b.view(np.uint64)) or np.array_equal(a, b, equal_nan=True)


@pytest.fixture(scope="module")
def sel():
    return golden("select_cases")


def test_select_cases_oracle_matches_reference(sel):
    sc, specs = select_case_specs(sel)
    assert len(specs) == len(sel["x_code"]) >= 2900
    n_delay = n_none = 0
    for c, spec in enumerate(specs):
        t = optable.from_spec(spec, sc, KINDS3)
        r = optable.select(t, sel["slack"][c], float(sel["p_alpha"][c]), int(sel["p_avail"][c]),
                           allow_delay=bool(sel["p_allow_delay"][c]),
                           upstream_supply=int(sel["p_supply"][c]),
                           excluded_mask=int(sel["p_excl"][c]), min_batch=int(sel["p_min_batch"][c]))
        exp = tuple(sel[f"x_{k}"][c] for k in ("code", "idx", "fill", "obj", "slack", "wait", "feas"))
        assert r[0] == exp[0] and r[1] == exp[1] and r[2] == exp[2], f"case {c}"
        assert _same(r[3], exp[3]) and _same(r[4], exp[4]) and _same(r[5], exp[5]), f"case {c}"
        assert int(r[6]) == int(exp[6]), f"case {c}"
        n_delay += r[0] == 2
        n_none += r[0] == 0
        km = optable.kind_minima(t, sel["slack"][c], float(sel["p_alpha"][c]), 3)
        assert _same(km, sel["x_kind_min"][c]), f"case {c}"
        for k in range(3):
            a = optable.affinity(t, k, sel["slack"][c], float(sel["p_alpha"][c]))
            e = sel["x_affinity"][c, k]
            assert (a is None and math.isnan(e)) or _same(a, e), f"case {c} kind {k}"
    # the generator exercises every decision shape
    assert n_delay > 100 and n_none > 50


def test_select_cases_c_oracle_matches_reference(sel):
    sc, specs = select_case_specs(sel)
    tables = [optable.from_spec(s, sc, KINDS3) for s in specs]
    n = len(tables)
    flags = (sel["p_allow_delay"].astype(np.uint32) | (sel["p_excl"].astype(np.uint32) << 8))
    r = cselect.select_batch(tables, sel["slack"], 0.0, sel["p_avail"], sel["p_supply"],
                             sel["p_min_batch"], flags, op=np.arange(n))
    # alpha differs per case: run per alpha group
    for a in np.unique(sel["p_alpha"]):
        idx = np.flatnonzero(sel["p_alpha"] == a)
        r = cselect.select_batch([tables[i] for i in idx], sel["slack"][idx], float(a),
                                 sel["p_avail"][idx], sel["p_supply"][idx], sel["p_min_batch"][idx],
                                 flags[idx], op=np.arange(len(idx)))
        for k in ("code", "idx", "fill"):
            assert np.array_equal(r[k], sel[f"x_{k}"][idx]), k
        for k in ("obj", "slack", "wait"):
            assert _same(r[k], sel[f"x_{k}"][idx]), k
        assert np.array_equal(r["feasible"], sel["x_feas"][idx].astype(bool))


@pytest.fixture(scope="module")
def syn():
    return golden("synth_sample")


def test_synth_generator_matches_reference_profiler(syn):
    import hashlib

    from paper_2102_01887_b200 import synth

    for tag, with_model in (("c2", False), ("c5", True)):
        spec = synth.synth_spec(with_model)
        lat = np.array([e.latency_s for e in spec.entries])
        assert _same(lat, syn[f"{tag}_lat"])
        ids = hashlib.sha256("\n".join(e.config_id for e in spec.entries).encode()).digest()
        assert ids == bytes(syn[f"{tag}_ids_sha"])
        t = optable.from_spec(spec, synth.synth_scenario(), ["cpu", "gpu"])
        assert t.ref_index == int(syn[f"{tag}_ref_index"])
        inv = synth.synth_invocations(len(syn[f"{tag}_in_avail"]), t.lat, t.gkind,
                                      seed=20261017 if tag == "c2" else 5)
        for f in ("slack", "avail", "supply", "min_batch", "flags"):
            assert _same(getattr(inv, f), syn[f"{tag}_in_{f}"]) if f == "slack" else \
                np.array_equal(getattr(inv, f), syn[f"{tag}_in_{f}"]), f


@pytest.mark.parametrize("alpha", [0, 1, 100, 1000])
def test_synth_c_oracle_matches_reference(syn, alpha):
    from paper_2102_01887_b200 import synth

    t = optable.from_spec(synth.synth_spec(False), synth.synth_scenario(), ["cpu", "gpu"])
    r = cselect.select_batch([t], syn["c2_in_slack"], float(alpha), syn["c2_in_avail"],
                             syn["c2_in_supply"], syn["c2_in_min_batch"], syn["c2_in_flags"])
    for k in ("code", "idx", "fill"):
        assert np.array_equal(r[k], syn[f"c2_a{alpha}_{k}"]), k
    for k in ("obj", "slack", "wait"):
        assert _same(r[k], syn[f"c2_a{alpha}_{k}"]), k
    assert np.array_equal(r["feasible"], syn[f"c2_a{alpha}_feas"].astype(bool))


def test_synth_numpy_oracle_matches_reference_sample(syn):
    from paper_2102_01887_b200 import synth

    t = optable.from_spec(synth.synth_spec(False), synth.synth_scenario(), ["cpu", "gpu"])
    r = optable.select_many([t], syn["c2_in_slack"][:512], 100.0, syn["c2_in_avail"],
                            syn["c2_in_supply"], syn["c2_in_min_batch"], syn["c2_in_flags"])
    for k in ("code", "idx", "fill"):
        assert np.array_equal(r[k], syn[f"c2_a100_{k}"][:512]), k
    assert _same(r["obj"], syn["c2_a100_obj"][:512])


def test_c5_c_oracle_matches_reference(syn):
    from paper_2102_01887_b200 import synth

    t = optable.from_spec(synth.synth_spec(True), synth.synth_scenario(), ["cpu", "gpu"])
    r = cselect.select_batch([t], syn["c5_in_slack"], 100.0, syn["c5_in_avail"],
                             syn["c5_in_supply"], syn["c5_in_min_batch"], syn["c5_in_flags"])
    for k in ("code", "idx", "fill"):
        assert np.array_equal(r[k], syn[f"c5_a100_{k}"]), k
    assert _same(r["obj"], syn["c5_a100_obj"])


# ---- slack ---------------------------------------------------------------------------------

@pytest.fixture(scope="module")
def slk():
    return golden("slack_cases")


def _dag_case(d, c):
    names = [f"v{i:02d}" for i in range(d["v_off"][c + 1] - d["v_off"][c])]
    edges = [(names[s], names[t]) for s, t in zip(d["e_src"][d["e_off"][c]:d["e_off"][c + 1]],
                                                  d["e_dst"][d["e_off"][c]:d["e_off"][c + 1]])]
    ref = dict(zip(names, d["v_ref"][d["v_off"][c]:d["v_off"][c + 1]].tolist()))
    return names, edges, ref


def test_compute_slack_oracle_matches_reference(slk):
    cache = {}
    for q in range(len(slk["q_case"])):
        c = int(slk["q_case"][q])
        if c not in cache:
            names, edges, ref = _dag_case(slk, c)
            cache = {c: (names, ref, slack.decompose_paths(names, edges))}
        names, ref, paths = cache[c]
        got = slack.compute_slack(names[slk["q_op"][q]], target_s=float(slk["q_target"][q]),
                                  elapsed_s=float(slk["q_elapsed"][q]),
                                  queueing_s=float(slk["q_queue"][q]), paths=paths, ref=ref)
        assert _same(got, slk["q_expect"][q]), q


def test_forward_dp_restatement_is_exact(slk):
    """the forward left-to-right DP equals compute_slack bit-for-bit."""
    checked = 0
    for c in range(len(slk["v_off"]) - 1):
        names, edges, ref = _dag_case(slk, c)
        # topological numbering
        from paper_2102_01887_b200.pipeline import PipelineDag

        dag = PipelineDag(tuple(names), tuple(edges))
        order = dag.topological_order()
        pos = {v: i for i, v in enumerate(order)}
        preds = [[pos[p] for p in dag.predecessors(v)] for v in order]
        has_succ = {s for s, _ in edges}
        term = [v not in has_succ for v in order]
        refv = np.array([ref[v] for v in order])
        paths = slack.decompose_paths(names, edges)
        for v in order:
            lo, hi = slack.dp_ratios(order, preds, term, refv, pos[v])
            for budget in (17.5, -3.25, 0.0, math.inf, 1e-9, -1e9):
                want = slack.compute_slack(v, target_s=budget, elapsed_s=0.0, queueing_s=0.0,
                                           paths=paths, ref=ref)
                assert _same(slack.dp_slack(lo, hi, budget), want)
                checked += 1
    assert checked > 10000


def test_path_list_slack_oracle_matches_reference(slk):
    meta = golden_json(slk, "paths_json")
    for i, exp in enumerate(slk["paths_expect"]):
        got = slack.compute_slack(meta["op"][i], target_s=meta["budget"][i], elapsed_s=0.0,
                                  queueing_s=0.0, paths=[tuple(p) for p in meta["paths"][i]],
                                  ref=meta["ref"][i])
        assert _same(got, exp), i


# ---- feedback / queueing -------------------------------------------------------------------

def feedback_case_states(d):
    meta = golden_json(d, "meta_json")
    lo = oo = 0
    for m in meta:
        states = []
        for t in range(2):
            M = m["sizes"][t]
            states.append(feedback.FoldState(d["lat0"][lo:lo + M].copy(), d["latinit"][lo:lo + M].copy(),
                                             m["ref"][t]))
            lo += M
        n = m["n_obs"]
        yield m, states, d["obs_op"][oo:oo + n], d["obs_idx"][oo:oo + n], d["obs"][oo:oo + n]
        oo += n


def test_feedback_oracle_matches_reference():
    d = golden("feedback_cases")
    lo = 0
    lifted = 0
    for m, states, op, idx, obs in feedback_case_states(d):
        feedback.fold(states, op, idx, obs, beta=m["beta"], dfp_count=m["dfp"], dfp_on=m["dfp_on"],
                      fb_frozen=not m["fb"])
        for t, st in enumerate(states):
            M = m["sizes"][t]
            assert _same(st.lat, d["final_lat"][lo:lo + M])
            assert np.array_equal(st.obs_count, d["final_cnt"][lo:lo + M])
            assert st.completed_ref == m["completed_ref"][t]
            lifted += m["dfp_on"] and m["fb"] and st.completed_ref >= m["dfp"] > 0
            lo += M
    assert lifted > 20


def test_queueing_oracle_matches_reference():
    d = golden("queue_cases")
    for c in range(len(d["pool"])):
        a, b = d["off"][c], d["off"][c + 1]
        got = queueing.estimate_queueing(list(zip(d["lat"][a:b], d["res"][a:b])), float(d["pool"][c]))
        assert _same(got, d["expect"][c])


# ---- live reference (build container only) ---------------------------------------------------

def test_oracle_against_live_reference_random(ref):
    from slackpipe.configurator import OpTable as RefTable
    from slackpipe.pipeline import ConfigEntry as RCE, ConfigSpec as RCS
    from slackpipe.scenario import BackendSpec as RBS, GroundTruthModel, Scenario as RSc

    rng = random.Random(4242)
    sc = RSc("live", (RBS("cpu", 3, 8, 2e-5), RBS("gpu", 1, 16, 5e-4)), GroundTruthModel(per_op={}))
    for case in range(300):
        ents = [RCE("cpu-r1-b1", "cpu", {}, 1, 1, rng.uniform(0.1, 3), 1.0)]
        for i in range(rng.randint(1, 30)):
            k = rng.choice(["cpu", "gpu"])
            lat = rng.choice([0.5, 1.0, rng.uniform(0.01, 5)])
            ents.append(RCE(f"{k}-x{i}", k, {}, rng.choice([1, 2, 4, 8]), rng.choice([1, 2, 4, 8, 16]),
                            lat, lat))
        spec = RCS("op", ents, "cpu-r1-b1")
        rt = RefTable(spec, sc)
        t = optable.from_spec(spec, sc, ["cpu", "gpu"])
        s = {"cpu": rng.uniform(-1, 6), "gpu": rng.uniform(-1, 6)}
        avail, sup, mb = rng.randint(1, 10), rng.randint(0, 10), rng.choice([1, 2, 16])
        alpha = rng.choice([0.0, 100.0])
        d = rt.select(s, alpha, avail, allow_delay=True, upstream_supply=sup, min_batch=mb)
        r = optable.select(t, np.array([s["cpu"], s["gpu"]]), alpha, avail, allow_delay=True,
                           upstream_supply=sup, min_batch=mb)
        if d is None:
            assert r[0] == 0
        else:
            assert r[:3] == (2 if d.kind == "delay" else 1, d.entry_index, d.fill)
            assert _same(r[3], d.objective_value) and _same(r[5], d.wait_budget_s)


# ---- commit rounds (Configurator.pump_commits) --------------------------------------------------

def _commit_replay(max_rounds_per_run=None):
    """Yield (tables, round index, per-op inputs) in the recorded order, applying the recorded
    set_latency calls to the oracle tables in between."""
    from oracle import commit as oc

    d = golden("commit_rounds")
    meta = golden_json(d, "meta_json")
    amb = golden_json(golden("amber_trace"), "meta_json")
    runs = d["r_run"]
    for ri, rm in enumerate(meta["runs"]):
        tabs = oc.amber_tables(amb)
        for t, name in zip(tabs, meta["ops"]):
            t.lat[:] = rm["tables"][name]["lat"]
        ev = [(int(s), 0, i) for i, s in enumerate(d["s_seq"]) if d["s_run"][i] == ri]
        ev += [(int(s), 1, i) for i, s in enumerate(d["r_seq"]) if runs[i] == ri]
        ev.sort()
        seen = 0
        for _, typ, i in ev:
            if typ == 0:
                tabs[d["s_op"][i]].lat[d["s_idx"][i]] = d["s_val"][i]
                continue
            seen += 1
            if max_rounds_per_run and seen > max_rounds_per_run:
                break
            yield ri, rm, tabs, i


def test_commit_round_oracle_matches_reference_rounds():
    """oracle/commit.py reproduces every recorded round: each _commit_candidate result and the
    committed op (4 runs: 50% target, fast target, pbc and eslc ablations)."""
    from oracle import commit as oc

    d = golden("commit_rounds")
    n_rounds = n_cands = 0
    for ri, rm, tabs, i in _commit_replay(max_rounds_per_run=700):
        a, n = int(d["r_first_cand"][i]), int(d["r_n_cand"][i])
        heads, slacks, buffered = [None] * len(tabs), [None] * len(tabs), [0] * len(tabs)
        full = None
        for c in range(a, a + n):
            j = int(d["c_op"][c])
            heads[j] = oc.Head(int(d["c_fill"][c]), bool(d["c_forced"][c]), int(d["c_inv"][c]),
                               int(d["c_spec_idx"][c]), float(d["c_spec_slack"][c]),
                               float(d["c_spec_obj"][c]))
            slacks[j] = np.nan_to_num(d["c_slack"][c], nan=0.0)
            buffered[j] = int(d["c_buffered"][c])
            full = int(d["c_full_mask"][c])
            cand = oc.commit_candidate(tabs[j], slacks[j], heads[j], full, buffered[j], rm["alpha"],
                                       "eslc" in rm["ablations"])
            if d["c_r_idx"][c] < 0:
                assert cand is None
            else:
                assert cand[0] == d["c_r_idx"][c] and cand[1] == d["c_r_fill"][c]
                assert cand[2] == d["c_r_slack"][c]
                assert (math.isnan(cand[3]) and math.isnan(d["c_r_obj"][c])) or cand[3] == d["c_r_obj"][c]
            n_cands += 1
        w = oc.round_winner(tabs, slacks, heads, full, buffered, rm["depths"], rm["alpha"],
                            fifo="pbc" in rm["ablations"], eslc="eslc" in rm["ablations"])
        assert (w[0] if w else -1) == d["r_winner_op"][i]
        n_rounds += 1
    assert n_rounds == 4 * 700 and n_cands > 4000


def speculate_call_inputs(d, i, K):
    """(sq, cq) weight lists of recorded speculate call i, per global kind in dict order."""
    sq = [[] for _ in range(K)]
    cq = [[] for _ in range(K)]
    a, n = int(d["c_w_first"][i]), int(d["c_w_n"][i])
    for w in range(a, a + n):
        lst = sq if d["w_queue"][w] == 0 else cq
        lst[int(d["w_kind"][w])].append([int(d["w_tab"][w]), int(d["w_eidx"][w]), int(d["w_count"][w])])
    return sq, cq


def speculate_replay():
    """Yield (run meta, oracle tables, call index) in the recorded order, applying the recorded
    set_latency calls to the oracle tables in between."""
    from oracle import commit as oc

    d = golden("speculate_calls")
    meta = golden_json(d, "meta_json")
    amb = golden_json(golden("amber_trace"), "meta_json")
    for ri, rm in enumerate(meta["runs"]):
        tabs = oc.amber_tables(amb)
        for t, name in zip(tabs, meta["ops"]):
            t.lat[:] = rm["tables"][name]["lat"]
        ev = [(int(s), 0, i) for i, s in enumerate(d["s_seq"]) if d["s_run"][i] == ri]
        ev += [(int(s), 1, i) for i, s in enumerate(d["c_seq"]) if d["c_run"][i] == ri]
        ev.sort()
        for _, typ, i in ev:
            if typ == 0:
                tabs[d["s_op"][i]].lat[d["s_idx"][i]] = d["s_val"][i]
                continue
            yield rm, tabs, i


def test_speculate_oracle_matches_reference_calls():
    """oracle/speculate.py reproduces every recorded Configurator.speculate_from_buffer call of
    three AMBER runs (50 % and 25 % targets, dfp ablation): every invocation formed (entry,
    fill, slack, objective) and the delay the loop stopped on."""
    from oracle import speculate as osp

    d = golden("speculate_calls")
    meta = golden_json(d, "meta_json")
    K = len(meta["kinds"])
    calls = formed = 0
    for rm, tabs, i in speculate_replay():
        sq, cq = speculate_call_inputs(d, i, K)
        dec, delay = osp.speculate(tabs, int(d["c_op"][i]), int(d["c_n"][i]), int(d["c_supply"][i]),
                                   float(d["c_now"][i]), float(d["c_target"][i]), float(d["c_rmin"][i]),
                                   float(d["c_rmax"][i]), rm["pool"], rm["alpha"], int(d["c_flags"][i]),
                                   sq, cq, d["c_slack0"][i])
        a, n = int(d["c_d_first"][i]), int(d["c_d_n"][i])
        assert len(dec) == n, i
        for j, (e, fill, s_k, obj) in enumerate(dec):
            assert e == d["d_idx"][a + j] and fill == d["d_fill"][a + j], i
            assert s_k == d["d_slack"][a + j], i
            assert (math.isnan(obj) and math.isnan(d["d_obj"][a + j])) or obj == d["d_obj"][a + j], i
        if d["c_delay_idx"][i] >= 0:
            assert delay is not None and delay[0] == d["c_delay_idx"][i] and delay[1] == d["c_delay_wait"][i], i
        else:
            assert delay is None, i
        calls += 1
        formed += n
    assert calls == 15000 and formed > 7000


# ---- C restatements used for full-size checks (oracle/select_oracle.c) ----------------------

def test_c_dp_slack_matches_reference_compute_slack(slk):
    """oracle_slack_dp (forward DP in C, the config-3 full-size checker) reproduces the
    reference's compute_slack golden values on the 400 random DAGs."""
    from oracle import cselect
    from paper_2102_01887_b200.pipeline import PipelineDag

    checked = 0
    for c in range(len(slk["v_off"]) - 1):
        names, edges, ref = _dag_case(slk, c)
        dag = PipelineDag(tuple(names), tuple(edges))
        q = np.flatnonzero(slk["q_case"] == c)
        refm = np.repeat(np.array([ref[n] for n in names])[None, :], len(q), 0)
        out = cselect.slack_dp(dag, refm, slk["q_target"][q], slk["q_elapsed"][q],
                               slk["q_queue"][q].reshape(-1, 1))
        got = out[np.arange(len(q)), slk["q_op"][q], 0]
        assert _same(got, slk["q_expect"][q]), c
        checked += len(q)
    assert checked > 1000


def test_c_path_slack_matches_reference(slk):
    """oracle_slack_paths (literal _path_ratios / slack_by_kind in C, the config-4 checker)
    reproduces the reference's compute_slack on the 300 golden path lists."""
    from oracle import cselect

    meta = golden_json(slk, "paths_json")
    for i, exp in enumerate(slk["paths_expect"]):
        names = sorted({n for p in meta["paths"][i] for n in p})
        cols = [[names.index(n) for n in p] for p in meta["paths"][i]]
        refv = np.array([[meta["ref"][i][n] for n in names]])
        out = cselect.slack_paths(refv, [meta["budget"][i]], [0.0], [[0.0]], cols)
        assert _same(out[0, names.index(meta["op"][i]), 0], exp), i


def test_c_fold_matches_reference():
    """oracle_fold (sequential EWMA + gate lift in C, the config-5 full-run checker) against the
    reference's _apply_feedback golden streams (feedback on, gate on; tables are independent,
    so each table's sub-stream is folded on its own)."""
    from oracle import cselect

    d = golden("feedback_cases")
    lo = 0
    checked = 0
    for m, states, op, idx, obs in feedback_case_states(d):
        for t, st in enumerate(states):
            M = m["sizes"][t]
            if m["fb"] and m["dfp_on"]:
                cs = cselect.FoldState(st.lat, st.lat_init, st.ref_index)
                sel = np.asarray(op) == t
                cselect.fold(cs, np.asarray(idx)[sel], np.asarray(obs)[sel], beta=m["beta"],
                             dfp_count=m["dfp"])
                assert _same(cs.lat, d["final_lat"][lo:lo + M])
                assert np.array_equal(cs.obs_count, d["final_cnt"][lo:lo + M])
                assert int(cs.completed_ref[0]) == m["completed_ref"][t]
                checked += 1
            lo += M
    assert checked > 20
