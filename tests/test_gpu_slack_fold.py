"""K1 (Alg. 1 slack) and K3 (feedback fold) parity on the B200."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, golden_json
from oracle import feedback as ofb
from oracle import slack as osl

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def test_dag_slack_vs_reference_compute_slack(gpu_ctx):
    """400 random DAGs: SlackGraph.from_dag (per-source forward DP, no path enumeration)
    reproduces the reference's compute_slack over decompose_paths bit-for-bit."""
    from paper_2102_01887_b200 import PipelineDag, SlackGraph

    d = golden("slack_cases")
    for c in range(len(d["v_off"]) - 1):
        n = int(d["v_off"][c + 1] - d["v_off"][c])
        names = [f"v{i:02d}" for i in range(n)]
        es = range(d["e_off"][c], d["e_off"][c + 1])
        edges = tuple((names[d["e_src"][j]], names[d["e_dst"][j]]) for j in es)
        g = SlackGraph.from_dag(PipelineDag(tuple(names), edges))
        ref = d["v_ref"][d["v_off"][c]:d["v_off"][c + 1]]
        q = np.flatnonzero(d["q_case"] == c)
        # one instance per query row: target, now (= elapsed), one kind with Q = queueing
        r = g.slack_batch(ref, d["q_target"][q].copy(), d["q_elapsed"][q].copy(),
                          d["q_queue"][q].reshape(-1, 1).copy())
        got = r["slack"][np.arange(len(q)), d["q_op"][q], 0]
        assert np.array_equal(bits(got), bits(d["q_expect"][q])), c
        g.close()


def test_path_list_slack_vs_reference(gpu_ctx):
    from paper_2102_01887_b200 import compute_slack

    d = golden("slack_cases")
    meta = golden_json(d, "paths_json")
    for i, exp in enumerate(d["paths_expect"]):
        got = compute_slack(meta["op"][i], "cpu", target_s=meta["budget"][i], elapsed_s=0.0,
                            queueing_s=0.0, paths=[tuple(p) for p in meta["paths"][i]],
                            ref_latency=meta["ref"][i])
        assert bits(got.seconds) == bits(exp), i


def test_deep_dag_config3_vs_dp_oracle(gpu_ctx):
    """Config 3 (64 ops, 845 edges, ~3.3e9 paths) at full size: every slack and ratio of the
    100,000-instance launch (K1c, the default) against the C forward-DP restatement
    (oracle_slack_dp), plus a sample against the Python dp_ratios / dp_slack restatement."""
    from oracle import cselect
    from paper_2102_01887_b200 import SlackGraph
    from paper_2102_01887_b200 import synth

    dag = synth.deep_dag()
    assert len(dag.edges) == 845
    I = 100_000
    ref, T, now, Q = synth.deep_dag_instances(dag, I)
    g = SlackGraph.from_dag(dag)
    r = g.slack_batch(ref, T, now, Q, ratios=True)
    exp, rat = cselect.slack_dp(dag, ref, T, now, Q, ratios=True)
    assert np.array_equal(bits(r["slack"]), bits(exp))
    assert np.array_equal(bits(r["ratio"]), bits(rat))
    order = dag.topological_order()
    pos = {v: i for i, v in enumerate(order)}
    preds = [[pos[p] for p in dag.predecessors(v)] for v in order]
    term = [not dag.successors(v) for v in order]
    vcol = [dag.vertices.index(v) for v in order]
    rng = np.random.default_rng(0)
    for i in rng.choice(I, size=20, replace=False):
        refo = ref[i][vcol]
        for s, v in enumerate(dag.vertices):
            lo, hi = osl.dp_ratios(order, preds, term, refo, pos[v])
            assert bits(r["ratio"][i, s, 0]) == bits(lo) and bits(r["ratio"][i, s, 1]) == bits(hi)
            for k in range(4):
                b = (T[i] - now[i]) - Q[i, k]
                assert bits(r["slack"][i, s, k]) == bits(osl.dp_slack(lo, hi, b))
    assert np.isfinite(r["slack"]).all()


@pytest.fixture(params=[4, 2])
def k1c_lanes(request, gpu_ctx):
    """Both forms of the certified pass: four lanes per instance (default) and two."""
    gpu_ctx.set_option("SP_K1C_LANES", request.param)
    yield request.param
    gpu_ctx.set_option("SP_K1C_LANES", 4)


def test_deep_dag_certified_pass_equals_forward_dp(gpu_ctx, k1c_lanes):
    """K1c (certified backward pass, the default for config 3) against K1's forward DP on the
    full 100k-instance launch: every slack and ratio bit-identical.  A second batch with
    quantised refs (exact ties between paths), zeros, and a few negative / inf / NaN refs
    forces the per-source fallbacks."""
    from paper_2102_01887_b200 import SlackGraph
    from paper_2102_01887_b200 import synth

    dag = synth.deep_dag()
    ref, T, now, Q = synth.deep_dag_instances(dag, 100_000)
    rng = np.random.default_rng(11)
    tie = np.round(ref[:4000] * 4) / 4
    tie[rng.random(tie.shape) < 0.01] = 0.0
    tie[5, 3] = -1.0
    tie[17, 40] = np.inf
    tie[23, 12] = np.nan
    tie[29, :] = 0.0
    for refs, t, n, q in ((ref, T, now, Q), (tie, T[:4000], now[:4000], Q[:4000])):
        g = SlackGraph.from_dag(dag)
        got = g.slack_batch(refs, t, n, q, ratios=True)
        gpu_ctx.set_option("SP_K1_CERT", 1)  # off: K1's forward DP
        try:
            exp = g.slack_batch(refs, t, n, q, ratios=True)
        finally:
            gpu_ctx.set_option("SP_K1_CERT", 0)
        g.close()
        for key in ("slack", "ratio"):
            assert np.array_equal(bits(got[key]), bits(exp[key])), key


def test_dag_slack_certified_forced_vs_reference(gpu_ctx, k1c_lanes):
    """The 400 reference DAG cases with K1c forced on every graph (SP_K1_CERT=force), small
    integer-valued refs included: bit-identical to the reference's compute_slack."""
    gpu_ctx.set_option("SP_K1_CERT", 2)  # force
    try:
        test_dag_slack_vs_reference_compute_slack(gpu_ctx)
    finally:
        gpu_ctx.set_option("SP_K1_CERT", 0)


@pytest.fixture(params=["coop", "legacy"])
def fold_impl(request, gpu_ctx):
    """Both fold implementations: the one-kernel cooperative fold (default) and the multi-kernel
    radix-sort path (SP_FOLD_LEGACY)."""
    gpu_ctx.set_option("SP_FOLD_LEGACY", 1 if request.param == "legacy" else 0)
    yield request.param
    gpu_ctx.set_option("SP_FOLD_LEGACY", 0)



def _fold_tables(d, m, lo):
    import paper_2102_01887_b200 as sp

    tabs = []
    for t in range(2):
        M = m["sizes"][t]
        tabs.append(sp.RawTable(lat=d["lat0"][lo:lo + M], res=np.ones(M), batch=np.ones(M, np.int32),
                                pool=np.ones(M), price=np.ones(M), ref_index=m["ref"][t],
                                lat_init=d["latinit"][lo:lo + M]))
        lo += M
    return tabs


@pytest.mark.parametrize("chunked", [False, True])
def test_feedback_fold_vs_reference(gpu_ctx, fold_impl, chunked):
    """PipelineRun._apply_feedback streams (EWMA, counts, gate-lift rescale, fb/dfp ablations)
    folded on the device in one batch, or in random consecutive chunks."""
    import paper_2102_01887_b200 as sp

    d = golden("feedback_cases")
    meta = golden_json(d, "meta_json")
    lo = oo = 0
    rng = np.random.default_rng(1)
    for m in meta:
        tabs = _fold_tables(d, m, lo)
        n = m["n_obs"]
        op = d["obs_op"][oo:oo + n].astype(np.int32)
        idx = d["obs_idx"][oo:oo + n].astype(np.int32)
        obs = d["obs"][oo:oo + n].astype(np.float64)
        cuts = [0, n] if not chunked else sorted({0, n, *rng.integers(0, n + 1, size=3).tolist()})
        for a, b in zip(cuts[:-1], cuts[1:]):
            sp.fold_observations(tabs, op[a:b], idx[a:b], obs[a:b], beta=m["beta"],
                                 dfp_count=m["dfp"], dfp_on=m["dfp_on"], fb_frozen=not m["fb"],
                                 sync_host=False)
        for t in range(2):
            M = m["sizes"][t]
            got = tabs[t].get_latency()
            assert np.array_equal(bits(got), bits(d["final_lat"][lo:lo + M])), (m, t)
            cref, cnt = sp.table_counters(tabs[t]) if hasattr(tabs[t], "lat") else (None, None)
            assert cref == m["completed_ref"][t]
            assert np.array_equal(cnt, d["final_cnt"][lo:lo + M])
            lo += M
        oo += n
        for t in tabs:
            t.close()


def test_feedback_fold_skips_negative_indices(gpu_ctx, fold_impl):
    """idx < 0 marks 'no observation' (e.g. a None / delay decision passed straight through)."""
    import paper_2102_01887_b200 as sp

    rng = np.random.default_rng(12)
    M = 300
    lat0 = rng.uniform(0.1, 2.0, size=M)
    idx = rng.integers(-1, M, size=5000).astype(np.int32)
    idx[rng.random(5000) < 0.3] = -1
    idx[::40] = 0
    obs = rng.uniform(0.1, 3.0, size=5000)
    tab = sp.RawTable(lat=lat0, res=np.ones(M), batch=np.ones(M, np.int32), pool=np.ones(M),
                      price=np.ones(M), ref_index=0, lat_init=lat0)
    sp.fold_observations([tab], None, idx, obs, beta=0.5, dfp_count=7, sync_host=False)
    keep = idx >= 0
    st = ofb.FoldState(lat0.copy(), lat0.copy(), 0)
    ofb.fold([st], None, idx[keep], obs[keep], beta=0.5, dfp_count=7)
    assert np.array_equal(bits(tab.get_latency()), bits(st.lat))
    cref, cnt = sp.table_counters(tab)
    assert cref == st.completed_ref and np.array_equal(cnt, st.obs_count)


def test_feedback_fold_large_stream_vs_oracle(gpu_ctx, fold_impl):
    """A config-5-sized batch (65,536 observations over a 16,384-entry table, heavy skew)
    against the sequential oracle."""
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    spec = synth.synth_spec(True)
    lat0 = np.array([e.latency_s for e in spec.entries])
    M = len(lat0)
    rng = np.random.default_rng(5)
    n = 65536
    hot = rng.choice(M, size=64, replace=False)
    idx = np.where(rng.random(n) < 0.8, rng.choice(hot, size=n), rng.integers(0, M, size=n)).astype(np.int32)
    ref_index = 0
    idx[rng.random(n) < 0.01] = ref_index
    obs = lat0[idx] * np.exp(rng.normal(0, 0.3, size=n))
    tab = sp.RawTable(lat=lat0 * 0.7, res=np.ones(M), batch=np.ones(M, np.int32), pool=np.ones(M),
                      price=np.ones(M), ref_index=ref_index, lat_init=lat0 * 0.7)
    st = ofb.FoldState(lat0 * 0.7, lat0 * 0.7, ref_index)
    for a, b in ((0, 20000), (20000, n)):
        sp.fold_observations([tab], None, idx[a:b], obs[a:b], beta=0.5, dfp_count=10, sync_host=False)
        ofb.fold([st], None, idx[a:b], obs[a:b], beta=0.5, dfp_count=10)
    assert np.array_equal(bits(tab.get_latency()), bits(st.lat))
    cref, cnt = sp.table_counters(tab)
    assert cref == st.completed_ref and np.array_equal(cnt, st.obs_count)


@pytest.mark.parametrize("beta", [0.5, 0.3, 0.1, 0.9, 1.0, 0.01])
def test_feedback_fold_long_segments_vs_oracle(gpu_ctx, fold_impl, beta):
    """Hot entries with tens of thousands of observations in one batch take the coalescing
    window path (sp_fold.cu): the result must still equal the sequential fold bit for bit,
    including the gate inside a long reference segment, a segment whose range is too wide to
    coalesce (1e300 in its prefix: sequential fallback) and a non-finite observation."""
    import paper_2102_01887_b200 as sp

    rng = np.random.default_rng(int(beta * 1000) + 7)
    M, n = 4096, 60000
    lat0 = np.exp(rng.uniform(np.log(1e-3), np.log(1.0), size=M))
    ref_index = 0
    u = rng.random(n)
    idx = np.where(u < 0.55, 7, np.where(u < 0.75, ref_index, np.where(
        u < 0.8, 9, np.where(u < 0.85, 11, rng.integers(0, M, size=n))))).astype(np.int32)
    obs = lat0[idx] * np.exp(rng.normal(0, 0.5, size=n))
    nine = np.flatnonzero(idx == 9)
    obs[nine[50]] = 1e300          # range too wide for the window: sequential fallback
    if beta < 1.0:                 # (beta = 1 would turn inf into 0 * inf = nan)
        eleven = np.flatnonzero(idx == 11)
        obs[eleven[40]] = np.inf   # non-finite prefix: window disabled, result stays inf
    tab = sp.RawTable(lat=lat0 * 0.7, res=np.ones(M), batch=np.ones(M, np.int32), pool=np.ones(M),
                      price=np.ones(M), ref_index=ref_index, lat_init=lat0 * 0.7)
    st = ofb.FoldState(lat0 * 0.7, lat0 * 0.7, ref_index)
    for a, b in ((0, 1000), (1000, n)):   # the gate (5000th reference completion) lies in batch 2
        sp.fold_observations([tab], None, idx[a:b], obs[a:b], beta=beta, dfp_count=5000,
                             sync_host=False)
        ofb.fold([st], None, idx[a:b], obs[a:b], beta=beta, dfp_count=5000)
    got = tab.get_latency()
    assert np.array_equal(bits(got), bits(st.lat))
    cref, cnt = sp.table_counters(tab)
    assert cref == st.completed_ref and np.array_equal(cnt, st.obs_count)


@pytest.mark.parametrize("dfp_count", [10, 3000, 10**9])
def test_feedback_fold_multi_chunk_vs_oracle(gpu_ctx, fold_impl, dfp_count):
    """One call of 200,000 records over two tables: the one-kernel fold takes it in four chunks
    of 64 x 1024 records (the gate lifting inside a later chunk for dfp_count = 3000, never for
    1e9), skipped records and ragged last tile included."""
    import paper_2102_01887_b200 as sp

    rng = np.random.default_rng(dfp_count % 1000 + 3)
    sizes, n = (5000, 700), 200_003
    lat0 = [np.exp(rng.uniform(np.log(1e-3), 0.0, size=M)) for M in sizes]
    op = (rng.random(n) < 0.3).astype(np.int32)
    hot = [rng.choice(M, size=12, replace=False) for M in sizes]
    idx = np.empty(n, np.int32)
    for t, M in enumerate(sizes):
        sel = op == t
        k = int(sel.sum())
        idx[sel] = np.where(rng.random(k) < 0.7, rng.choice(hot[t], size=k), rng.integers(0, M, size=k))
    idx[(op == 0) & (rng.random(n) < 0.02)] = 1   # table 0's reference entry
    idx[rng.random(n) < 0.05] = -1
    obs = np.array([lat0[t][max(i, 0)] for t, i in zip(op, idx)]) * np.exp(rng.normal(0, 0.4, size=n))
    tabs = [sp.RawTable(lat=lat0[t] * 0.8, res=np.ones(M), batch=np.ones(M, np.int32), pool=np.ones(M),
                        price=np.ones(M), ref_index=(1 if t == 0 else 5), lat_init=lat0[t] * 0.8)
            for t, M in enumerate(sizes)]
    sts = [ofb.FoldState(lat0[t] * 0.8, lat0[t] * 0.8, 1 if t == 0 else 5) for t in range(2)]
    sp.fold_observations(tabs, op, idx, obs, beta=0.5, dfp_count=dfp_count, sync_host=False)
    keep = idx >= 0
    ofb.fold(sts, op[keep], idx[keep], obs[keep], beta=0.5, dfp_count=dfp_count)
    for t in range(2):
        assert np.array_equal(bits(tabs[t].get_latency()), bits(sts[t].lat)), t
        cref, cnt = sp.table_counters(tabs[t])
        assert cref == sts[t].completed_ref and np.array_equal(cnt, sts[t].obs_count), t
        tabs[t].close()


@pytest.mark.parametrize("beta", [0.5, 0.6, 0.75, 0.97, 0.999])
def test_feedback_fold_narrowed_window_vs_oracle(gpu_ctx, beta):
    """Segments just above and far above the narrowed-window length (64 + 24), observations
    spread over six orders of magnitude, exact repeats and start values far outside the
    observations' range: the interval-narrowed window must give the sequential fold's bits."""
    import paper_2102_01887_b200 as sp

    rng = np.random.default_rng(int(beta * 1000) + 99)
    M = 64
    lens = [88, 89, 90, 100, 150, 300, 1000, 4000] * 4
    idx = np.concatenate([np.full(n, e, np.int32) for e, n in enumerate(lens)])
    rng.shuffle(idx)
    n = len(idx)
    obs = np.exp(rng.normal(0.0, 2.0, size=n)) * 1e-2
    obs[rng.random(n) < 0.1] = 0.5                  # exact repeats
    lat0 = np.exp(rng.uniform(np.log(1e-6), np.log(1e4), size=M))
    tab = sp.RawTable(lat=lat0, res=np.ones(M), batch=np.ones(M, np.int32), pool=np.ones(M),
                      price=np.ones(M), ref_index=-1, lat_init=lat0)
    st = ofb.FoldState(lat0.copy(), lat0.copy(), -1)
    sp.fold_observations([tab], None, idx, obs, beta=beta, dfp_count=10, sync_host=False)
    ofb.fold([st], None, idx, obs, beta=beta, dfp_count=10)
    assert np.array_equal(bits(tab.get_latency()), bits(st.lat))
    tab.close()


@pytest.mark.parametrize("per_item", [False, True])
def test_simulate_and_fold_equals_two_kernels(gpu_ctx, per_item):
    """sp_simulate_and_fold (the simulated backend's observation law evaluated inside the
    cooperative fold's load phase) against sp_simulate_observations + sp_feedback_fold on the
    same decision batches: identical observation records and identical tables after every
    batch (gate lift included: the reference entry is forced into the first batches)."""
    import torch

    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    spec = synth.synth_spec(False)
    tabs = [sp.OpTable(spec, synth.synth_scenario()) for _ in range(2)]
    M = len(tabs[0].entries)
    rng = np.random.default_rng(7 + per_item)
    dev = torch.device("cuda", 0)
    base = torch.from_numpy(np.array([e.latency_initial_s for e in tabs[0].entries])).to(dev)
    pit = torch.from_numpy(rng.uniform(0.0, 0.01, size=M)).to(dev) if per_item else None
    ref = tabs[0].ref_index
    for bt in range(6):
        n = int(rng.integers(1000, 70000))
        code = rng.choice([0, 1, 2], size=n, p=[0.1, 0.8, 0.1]).astype(np.int32)
        hot = rng.choice(M, size=40, replace=False)
        idx = np.where(rng.random(n) < 0.7, rng.choice(hot, size=n), rng.integers(0, M, size=n)).astype(np.int32)
        if bt < 2:
            idx[rng.random(n) < 0.01] = ref
        dec = {"code": torch.from_numpy(code).to(dev), "idx": torch.from_numpy(idx).to(dev),
               "fill": torch.from_numpy(rng.integers(1, 129, size=n).astype(np.int32)).to(dev)}
        noise = torch.from_numpy(np.exp(rng.normal(0.0, 0.3, size=n))).to(dev)
        r1 = (torch.empty(n, dtype=torch.int32, device=dev), torch.empty(n, dtype=torch.float64, device=dev))
        r2 = (torch.empty(n, dtype=torch.int32, device=dev), torch.empty(n, dtype=torch.float64, device=dev))
        sp.simulate_observations(dec, base, noise, truth_per_item=pit, out=r1)
        sp.fold_observations([tabs[0]], None, r1[0], r1[1], beta=0.5, dfp_count=10, sync_host=False)
        sp.simulate_and_fold(tabs[1], dec, base, noise, truth_per_item=pit, out=r2, beta=0.5, dfp_count=10)
        torch.cuda.synchronize()
        assert torch.equal(r1[0], r2[0]), bt
        assert torch.equal(r1[1].view(torch.int64), r2[1].view(torch.int64)), bt
        for t in tabs:
            t.sync_from_device()
        a, b = np.asarray(tabs[0].lat).copy(), np.asarray(tabs[1].lat).copy()
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), bt
