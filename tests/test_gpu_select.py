"""K2 parity on the B200: batched OpTable.select / affinity / scores vs the reference's golden
vectors and the CPU oracle.  Selected indices, decision kinds and SLO flags are compared
bit-exactly; objective / slack / wait values too (SURVEY.md §8 P1-P3 make them exact)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import KINDS3, golden, select_case_specs
from oracle import cselect, optable

pytestmark = pytest.mark.gpu

FIELDS_I = ("code", "idx", "fill")
FIELDS_F = ("obj", "slack", "wait")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_same_decisions(got, exp, where=""):
    code = np.asarray(got["code"])
    assert np.array_equal(code & 3, np.asarray(exp["code"])), where + " code"
    assert np.array_equal(np.asarray(got["idx"]), np.asarray(exp["idx"])), where + " idx"
    some = (code & 3) != 0
    assert np.array_equal(np.asarray(got["fill"])[some], np.asarray(exp["fill"])[some]), where + " fill"
    for k in FIELDS_F:
        assert np.array_equal(bits(np.asarray(got[k])[some]), bits(np.asarray(exp[k])[some])), where + " " + k
    if "feasible" in exp:
        assert np.array_equal(((code >> 2) & 1).astype(bool)[some],
                              np.asarray(exp["feasible"]).astype(bool)[some]), where + " feasible"


def raw_table(t: optable.Arrays, K: int):
    import paper_2102_01887_b200 as sp

    return sp.RawTable(lat=t.lat, res=t.res, batch=t.batch_int, pool=t.pool, price=t.price,
                       kind=t.gkind, id_rank=t.id_rank, K=K, ref_index=t.ref_index,
                       lat_init=t.lat_init)


@pytest.fixture(scope="module")
def sel():
    return golden("select_cases")


def test_select_cases_object_api(gpu_ctx, sel):
    """OpTable.select / affinity / scores through the reference-shaped API, case by case."""
    import paper_2102_01887_b200 as sp

    sc, specs = select_case_specs(sel)
    for c, spec in enumerate(specs[:600]):
        t = sp.OpTable(spec, sc, kinds=KINDS3)
        s = {k: float(sel["slack"][c, i]) for i, k in enumerate(KINDS3)}
        ex = frozenset(k for i, k in enumerate(KINDS3) if (int(sel["p_excl"][c]) >> i) & 1)
        alpha = float(sel["p_alpha"][c])
        d = t.select(s, alpha, int(sel["p_avail"][c]), allow_delay=bool(sel["p_allow_delay"][c]),
                     upstream_supply=int(sel["p_supply"][c]), excluded_kinds=ex,
                     min_batch=int(sel["p_min_batch"][c]))
        if sel["x_code"][c] == 0:
            assert d is None, c
        else:
            assert d is not None, c
            assert d.kind == ("delay" if sel["x_code"][c] == 2 else "assign"), c
            assert d.entry_index == sel["x_idx"][c] and d.fill == sel["x_fill"][c], c
            assert d.entry is t.entries[d.entry_index]
            for f, k in (("objective_value", "obj"), ("slack_s", "slack"), ("wait_budget_s", "wait")):
                assert bits(getattr(d, f)) == bits(sel[f"x_{k}"][c]), (c, f)
        for i, k in enumerate(KINDS3):
            a = t.affinity(k, s, alpha)
            e = sel["x_affinity"][c, i]
            if math.isnan(e):
                assert a is None
            else:
                assert bits(a) == bits(e), (c, k)
        t.close()


@pytest.mark.parametrize("mode", ["plan", "scan"])
def test_select_cases_batched_multitable(gpu_ctx, sel, mode):
    """All ~3,000 golden cases as multi-table launches (op[] routes invocations to tables)."""
    import paper_2102_01887_b200 as sp

    sc, specs = select_case_specs(sel)
    arrays = [optable.from_spec(s, sc, KINDS3) for s in specs]
    flags = sp.make_flags(sel["p_allow_delay"], sel["p_excl"])
    group = 64 if mode == "plan" else 16
    for a in np.unique(sel["p_alpha"]):
        ids = np.flatnonzero(sel["p_alpha"] == a)
        for g0 in range(0, len(ids), group):
            g = ids[g0:g0 + group]
            tabs = [raw_table(arrays[i], 3) for i in g]
            r = sp.select_batch(tabs, np.ascontiguousarray(sel["slack"][g]), float(a),
                                np.ascontiguousarray(sel["p_avail"][g], np.int32),
                                upstream_supply=np.ascontiguousarray(sel["p_supply"][g], np.int32),
                                min_batch=np.ascontiguousarray(sel["p_min_batch"][g], np.int32),
                                flags=np.ascontiguousarray(flags[g]),
                                op=np.arange(len(g), dtype=np.int32), kind_min=True, mode=mode)
            exp = {k: sel[f"x_{k}"][g] for k in FIELDS_I + FIELDS_F}
            exp["feasible"] = sel["x_feas"][g]
            assert_same_decisions(r, exp, f"alpha={a} group={g0}")
            assert np.array_equal(bits(r["kind_min"]), bits(sel["x_kind_min"][g]))
            for t in tabs:
                t.close()


@pytest.fixture(scope="module")
def syn():
    return golden("synth_sample")


@pytest.fixture(scope="module")
def c2_table(gpu_ctx):
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    return sp.OpTable(synth.synth_spec(False), synth.synth_scenario())


@pytest.mark.parametrize("mode", ["plan", "scan"])
@pytest.mark.parametrize("alpha", [0, 1, 100, 1000])
def test_config2_sample_vs_reference(c2_table, syn, mode, alpha):
    r = c2_table.select_batch(syn["c2_in_slack"], float(alpha), syn["c2_in_avail"],
                              upstream_supply=syn["c2_in_supply"], min_batch=syn["c2_in_min_batch"],
                              flags=syn["c2_in_flags"], mode=mode)
    exp = {k: syn[f"c2_a{alpha}_{k}"] for k in FIELDS_I + FIELDS_F}
    exp["feasible"] = syn[f"c2_a{alpha}_feas"]
    assert_same_decisions(r, exp, f"{mode} alpha={alpha}")


def test_config2_affinity_vs_reference(c2_table, syn):
    for i in range(64):
        s = {"cpu": float(syn["c2_in_slack"][i, 0]), "gpu": float(syn["c2_in_slack"][i, 1])}
        for j, k in enumerate(("cpu", "gpu")):
            assert bits(c2_table.affinity(k, s, 100.0)) == bits(syn["c2_affinity"][i, j])


def test_config5_sample_vs_reference(gpu_ctx, syn):
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    t = sp.OpTable(synth.synth_spec(True), synth.synth_scenario())
    assert t.plan_supported()
    for mode in ("plan", "scan"):
        r = t.select_batch(syn["c5_in_slack"], 100.0, syn["c5_in_avail"],
                           upstream_supply=syn["c5_in_supply"], min_batch=syn["c5_in_min_batch"],
                           flags=syn["c5_in_flags"], mode=mode)
        exp = {k: syn[f"c5_a100_{k}"] for k in FIELDS_I + FIELDS_F}
        assert_same_decisions(r, exp, mode)
    t.close()


@pytest.mark.parametrize("alpha", [100.0, 0.0, 1.0, 1000.0])
def test_config2_full_size_vs_c_oracle(c2_table, alpha):
    """BASELINE config 2 at full size, every alpha of SURVEY.md §8(d): 2^20 invocations x
    4,096 configurations, plan and scan kernels against the C oracle."""
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    t = optable.from_spec(synth.synth_spec(False), synth.synth_scenario(), ["cpu", "gpu"])
    inv = synth.synth_invocations(1 << 20, t.lat, t.gkind)
    exp = cselect.select_batch([t], inv.slack, alpha, inv.avail, inv.supply, inv.min_batch, inv.flags)
    for mode in ("plan", "scan"):
        r = c2_table.select_batch(inv.slack, alpha, inv.avail, upstream_supply=inv.supply,
                                  min_batch=inv.min_batch, flags=inv.flags, mode=mode)
        assert_same_decisions(r, exp, mode)
    # every decision shape and both SLO outcomes occur at full size
    codes = np.bincount(exp["code"], minlength=3)
    assert codes.min() > 1000
    assert 0.05 < exp["feasible"][exp["code"] > 0].mean() < 0.95


def _random_table(rng, M, nB, K, nonpos=False):
    batch_vals = np.sort(rng.choice(np.arange(1, 300), size=nB, replace=False))
    lat_pool = rng.uniform(0.01, 5.0, size=max(3, M // 8))
    lat = np.where(rng.random(M) < 0.5, rng.choice(lat_pool, size=M), rng.uniform(0.01, 5.0, size=M))
    if nonpos:  # latencies set to <= 0 through set_latency (the reference does not forbid it)
        lat[rng.random(M) < 0.1] = 0.0
        lat[rng.random(M) < 0.1] = -rng.uniform(0.0, 2.0)
    res = rng.choice([1.0, 2.0, 4.0, 8.0], size=M)
    gk = rng.integers(0, K, size=M)
    gk[0] = 0
    pools = rng.choice([16.0, 64.0, 256.0], size=K)
    prices = rng.choice([1e-5, 3e-5, 2.5e-4], size=K)
    return optable.from_columns(lat=lat, res=res, batch=rng.choice(batch_vals, size=M),
                                pool=pools[gk], price=prices[gk], gkind=gk,
                                id_rank=rng.permutation(M), n_kinds=K)


@pytest.mark.parametrize("seed,M,nB,K,nonpos", [(1, 3000, 8, 2, False), (2, 2000, 16, 4, False),
                                                (3, 700, 13, 3, False), (4, 5000, 5, 8, False),
                                                (5, 1, 1, 1, False), (6, 64, 2, 2, False),
                                                (7, 900, 8, 2, True), (8, 300, 11, 3, True)])
def test_random_tables_plan_scan_oracle(gpu_ctx, seed, M, nB, K, nonpos):
    """Heavily tied random tables (repeated latencies, equal scores), every kind count and
    both plan widths (W = 8 / 16), also zero / negative latencies: plan == scan == C oracle."""
    import paper_2102_01887_b200 as sp

    rng = np.random.default_rng(seed)
    t = _random_table(rng, M, nB, K, nonpos)
    N = 20000
    slack = rng.uniform(-2, 6, size=(N, K))
    slack[rng.random((N, K)) < 0.05] = np.inf
    slack[rng.random((N, K)) < 0.02] = -np.inf
    pick = rng.random((N, K)) < 0.1
    slack[pick] = rng.choice(t.lat, size=int(pick.sum()))
    avail = rng.integers(0, 320, size=N).astype(np.int32)
    supply = rng.integers(0, 320, size=N).astype(np.int32)
    mb = np.where(rng.random(N) < 0.7, 1, rng.integers(-1, 300, size=N)).astype(np.int32)
    excl = rng.integers(0, 1 << K, size=N) * (rng.random(N) < 0.3)
    flags = sp.make_flags(rng.random(N) < 0.5, excl)
    tab = raw_table(t, K)
    for alpha in (0.0, 7.5, 1000.0):
        exp = cselect.select_batch([t], slack, alpha, avail, supply, mb, flags)
        for mode in ("plan", "scan"):
            r = sp.select_batch([tab], slack, alpha, avail, upstream_supply=supply, min_batch=mb,
                                flags=flags, mode=mode, kind_min=True)
            assert_same_decisions(r, exp, f"{mode} alpha={alpha}")
            km = np.stack([optable.kind_minima(t, slack[i], alpha, K) for i in range(64)])
            assert np.array_equal(bits(r["kind_min"][:64]), bits(km))
    tab.close()


@pytest.mark.parametrize("seed,M,nB,K,nonpos", [(11, 3000, 8, 2, False), (12, 2000, 16, 4, False),
                                                (13, 5000, 5, 8, False), (14, 900, 8, 2, True),
                                                (15, 64, 2, 2, False), (16, 700, 13, 3, False)])
def test_single_table_fast_kernel_vs_oracle(gpu_ctx, seed, M, nB, K, nonpos):
    """Once a plan's header has reached the host, single-table calls without kind minima run
    the specialised K2f kernel (K == 2, 4, 8 with positive thresholds; otherwise K2b): every
    such call must equal the C oracle, including repeated calls (plan pre-staged before the
    programmatic-dependent-launch wait) and a call right after a latency update."""
    import paper_2102_01887_b200 as sp

    rng = np.random.default_rng(seed)
    t = _random_table(rng, M, nB, K, nonpos)
    N = 30011
    slack = rng.uniform(-2, 6, size=(N, K))
    slack[rng.random((N, K)) < 0.05] = np.inf
    pick = rng.random((N, K)) < 0.1
    slack[pick] = rng.choice(t.lat, size=int(pick.sum()))
    avail = rng.integers(0, 320, size=N).astype(np.int32)
    supply = rng.integers(0, 320, size=N).astype(np.int32)
    mb = np.where(rng.random(N) < 0.7, 1, rng.integers(-1, 300, size=N)).astype(np.int32)
    flags = sp.make_flags(rng.random(N) < 0.5, rng.integers(0, 1 << K, size=N) * (rng.random(N) < 0.3))
    tab = raw_table(t, K)
    for alpha in (0.0, 7.5):
        exp = cselect.select_batch([t], slack, alpha, avail, supply, mb, flags)
        tab.prepare(alpha)
        gpu_ctx.synchronize()
        for rep in range(3):
            r = sp.select_batch([tab], slack, alpha, avail, upstream_supply=supply, min_batch=mb,
                                flags=flags, mode="plan")
            assert_same_decisions(r, exp, f"alpha={alpha} rep={rep}")
    # latency update -> rebuilt plan (captured into a CUDA graph, then replayed)
    for step in range(3):
        j = int(rng.integers(0, M))
        v = float(t.lat[j] * (0.5 + step))
        t.lat[j] = v
        tab.set_latency(np.array([j], np.int32), np.array([v]))
        exp = cselect.select_batch([t], slack, 7.5, avail, supply, mb, flags)
        for rep in range(2):
            r = sp.select_batch([tab], slack, 7.5, avail, upstream_supply=supply, min_batch=mb,
                                flags=flags, mode="plan")
            assert_same_decisions(r, exp, f"after update {step} rep={rep}")
    tab.close()


@pytest.mark.parametrize("N", [200_003, 151 * 1024, 1024 * 148 - 1])
def test_streamed_multitable_ragged_vs_oracle(gpu_ctx, N):
    """Sizes that exercise the TMA input ring (full tiles on every CTA), the ragged tail, and
    the below-threshold fallback, with an op[] array routing to two different tables."""
    import paper_2102_01887_b200 as sp

    rng = np.random.default_rng(N)
    tabs = [_random_table(rng, 1500, 8, 2), _random_table(rng, 700, 6, 2)]
    slack = rng.uniform(-1, 6, size=(N, 2))
    avail = rng.integers(1, 300, size=N).astype(np.int32)
    supply = rng.integers(0, 300, size=N).astype(np.int32)
    mb = np.where(rng.random(N) < 0.8, 1, rng.integers(1, 300, size=N)).astype(np.int32)
    flags = sp.make_flags(rng.random(N) < 0.5, rng.integers(0, 4, size=N) * (rng.random(N) < 0.2))
    op = (rng.random(N) < 0.3).astype(np.int32)
    exp = cselect.select_batch(tabs, slack, 50.0, avail, supply, mb, flags, op=op)
    raws = [raw_table(t, 2) for t in tabs]
    r = sp.select_batch(raws, slack, 50.0, avail, upstream_supply=supply, min_batch=mb, flags=flags,
                        op=op, mode="plan")
    assert_same_decisions(r, exp, f"N={N}")
    for t in raws:
        t.close()


def test_plan_rebuilds_after_latency_update(c2_table, syn):
    """set_latency invalidates the plan; decisions follow the live profile."""
    from paper_2102_01887_b200 import synth

    t = optable.from_spec(synth.synth_spec(False), synth.synth_scenario(), ["cpu", "gpu"])
    rng = np.random.default_rng(9)
    idx = rng.choice(len(t.lat), size=200, replace=False)
    for i in idx:
        v = float(t.lat[i] * rng.uniform(0.3, 3.0))
        t.lat[i] = v
        c2_table.set_latency(int(i), v)
    assert np.array_equal(bits(c2_table.lat), bits(t.lat))
    n = 4096
    exp = cselect.select_batch([t], syn["c2_in_slack"], 100.0, syn["c2_in_avail"], syn["c2_in_supply"],
                               syn["c2_in_min_batch"], syn["c2_in_flags"])
    r = c2_table.select_batch(syn["c2_in_slack"], 100.0, syn["c2_in_avail"],
                              upstream_supply=syn["c2_in_supply"], min_batch=syn["c2_in_min_batch"],
                              flags=syn["c2_in_flags"])
    assert_same_decisions(r, exp)
    # restore for other tests
    for i in idx:
        c2_table.set_latency(int(i), float(syn["c2_lat"][i]))


def test_device_resident_inputs_match_host(c2_table, syn):
    import torch

    dev = torch.device("cuda", 0)
    ins = {k: torch.from_numpy(np.ascontiguousarray(syn[f"c2_in_{k}"])).to(dev)
           for k in ("slack", "avail", "supply", "min_batch", "flags")}
    r = c2_table.select_batch(ins["slack"], 1000.0, ins["avail"], upstream_supply=ins["supply"],
                              min_batch=ins["min_batch"], flags=ins["flags"])
    c2_table._ctx.synchronize()
    got = {k: v.cpu().numpy() for k, v in r.items()}
    exp = {k: syn[f"c2_a1000_{k}"] for k in FIELDS_I + FIELDS_F}
    assert_same_decisions(got, exp)


def test_empty_batch_and_errors(c2_table):
    r = c2_table.select_batch(np.zeros((0, 2)), 1.0, np.zeros(0, np.int32),
                              upstream_supply=np.zeros(0, np.int32),
                              min_batch=np.zeros(0, np.int32), flags=np.zeros(0, np.uint32))
    assert len(r["idx"]) == 0
    with pytest.raises(ValueError):
        c2_table.select({"cpu": 1.0, "gpu": 1.0}, -1.0, 1, allow_delay=False)
    with pytest.raises(KeyError):
        c2_table.select({"cpu": 1.0}, 1.0, 1, allow_delay=False)


@pytest.mark.parametrize("N", [1 << 20, 200_003])
def test_pinned_host_buffers_zero_copy(gpu_ctx, N):
    """Pinned (mapped) host buffers take the zero-copy path (the kernel reads and writes host
    memory over PCIe in a single launch) and give the same decisions as the oracle; pageable
    buffers of the same call take the staged-copy path."""
    import torch

    import paper_2102_01887_b200 as sp

    rng = np.random.default_rng(N + 1)
    tabs = [_random_table(rng, 1500, 8, 2), _random_table(rng, 700, 6, 2)]
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    slack = rng.uniform(-1, 6, size=(N, 2))
    avail = rng.integers(1, 300, size=N).astype(np.int32)
    supply = rng.integers(0, 300, size=N).astype(np.int32)
    mb = np.where(rng.random(N) < 0.8, 1, rng.integers(1, 300, size=N)).astype(np.int32)
    flags = sp.make_flags(rng.random(N) < 0.5, rng.integers(0, 4, size=N) * (rng.random(N) < 0.2))
    op = (rng.random(N) < 0.3).astype(np.int32)
    exp = cselect.select_batch(tabs, slack, 50.0, avail, supply, mb, flags, op=op)
    raws = [raw_table(t, 2) for t in tabs]
    for t in raws:
        t.prepare(50.0)
    out = {"idx": pin(np.full(N, -7, np.int32)), "code": pin(np.full(N, -7, np.int32)),
           "fill": pin(np.zeros(N, np.int32)), "obj": pin(np.zeros(N)), "slack": pin(np.zeros(N)),
           "wait": pin(np.zeros(N))}
    ctx = sp.get_context(0)
    l0 = ctx.launch_count
    r = sp.select_batch(raws, pin(slack), 50.0, pin(avail), upstream_supply=pin(supply),
                        min_batch=pin(mb), flags=pin(flags), op=pin(op), mode="plan", out=out)
    assert ctx.launch_count - l0 == 1  # one decision launch, no chunked copies
    assert_same_decisions(r, exp, f"pinned N={N}")
    r2 = sp.select_batch(raws, slack, 50.0, avail, upstream_supply=supply, min_batch=mb,
                         flags=flags, op=op, mode="plan")
    assert_same_decisions(r2, exp, f"pageable N={N}")
    for t in raws:
        t.close()


@pytest.mark.parametrize("variant", ["SP_STAIR_SMEM", "SP_STAIR_GLOBAL", "SP_NO_PLAN_GRAPH",
                                     "SP_PLAN_LEGACY", "cluster"])
def test_staircase_builder_variants_vs_oracle(gpu_ctx, variant):
    """Every plan builder against the C oracle: the one-kernel cluster builder (default), the
    multi-kernel builder (SP_PLAN_LEGACY) with its fallback staircases (shared-memory run scans
    for kinds of 8,193-16,384 entries, the global-memory builder above that) and the un-graphed
    rebuild path — on ordinary tables plus a 20,000-entry kind (beyond the cluster builder's
    8,192, so it takes the multi-kernel global builder on its own)."""
    import paper_2102_01887_b200 as sp

    opts = {"SP_STAIR_SMEM": ["SP_PLAN_LEGACY", "SP_STAIR_SMEM"],
            "SP_STAIR_GLOBAL": ["SP_PLAN_LEGACY", "SP_STAIR_GLOBAL"],
            "SP_NO_PLAN_GRAPH": ["SP_NO_PLAN_GRAPH"], "SP_PLAN_LEGACY": ["SP_PLAN_LEGACY"],
            "cluster": []}[variant]
    for o in opts:
        gpu_ctx.set_option(o, 1)
    try:
        _builder_variant_cases(sp, variant)
    finally:
        for o in opts:
            gpu_ctx.set_option(o, 0)


def _builder_variant_cases(sp, variant):
    rng = np.random.default_rng(hash(variant) & 0xFFFF)
    for M, nB, K in ((3000, 8, 2), (1500, 16, 4), (20000, 8, 1)):
        t = _random_table(rng, M, nB, K)
        N = 20000
        slack = rng.uniform(-2, 6, size=(N, K))
        pick = rng.random((N, K)) < 0.1
        slack[pick] = rng.choice(t.lat, size=int(pick.sum()))
        avail = rng.integers(0, 320, size=N).astype(np.int32)
        supply = rng.integers(0, 320, size=N).astype(np.int32)
        mb = np.where(rng.random(N) < 0.7, 1, rng.integers(-1, 300, size=N)).astype(np.int32)
        flags = sp.make_flags(rng.random(N) < 0.5, rng.integers(0, 1 << K, size=N) * (rng.random(N) < 0.3))
        tab = raw_table(t, K)
        for step in range(3):  # first build, captured rebuild, replayed rebuild
            exp = cselect.select_batch([t], slack, 7.5, avail, supply, mb, flags)
            r = sp.select_batch([tab], slack, 7.5, avail, upstream_supply=supply, min_batch=mb,
                                flags=flags, mode="plan")
            assert_same_decisions(r, exp, f"{variant} M={M} step={step}")
            j = int(rng.integers(0, M))
            tab.set_latency(np.array([j], np.int32), np.array([float(t.lat[j] * 1.7)]))
        tab.close()


def test_device_group_fanout_matches_single_device(gpu_ctx):
    """sp_group_select_batch (single-process multi-GPU fan-out, SURVEY.md §8(b) Threading): the
    config-2 batch sharded over a group of member contexts (two independent contexts per
    visible GPU here; one per GPU on a full box) equals the single-context call and the C
    oracle bit for bit; set_latency and the feedback fold reach every replica."""
    import torch

    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    devs = [d for d in range(torch.cuda.device_count()) for _ in range(2)]
    g = sp.DeviceGroup(devs)
    spec = synth.synth_spec(False)
    gt = g.table(spec, synth.synth_scenario())
    t = optable.from_spec(spec, synth.synth_scenario(), ["cpu", "gpu"])
    inv = synth.synth_invocations((1 << 18) + 7, t.lat, t.gkind, seed=77)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    for host in (lambda a: np.ascontiguousarray(a), pin):  # pageable staging and zero-copy
        r = gt.select_batch(host(inv.slack), 100.0, host(inv.avail), upstream_supply=host(inv.supply),
                            min_batch=host(inv.min_batch), flags=host(inv.flags))
        exp = cselect.select_batch([t], inv.slack, 100.0, inv.avail, inv.supply, inv.min_batch, inv.flags)
        assert_same_decisions(r, exp, "group")
    # mutations go to every replica
    rng = np.random.default_rng(3)
    for i in rng.choice(len(gt.lat), size=20, replace=False):
        gt.set_latency(int(i), float(gt.lat[i]) * 1.5)
    idx = rng.integers(0, len(gt.lat), size=5000).astype(np.int32)
    obs = rng.uniform(0.01, 3.0, size=5000)
    gt.fold(idx, obs)
    for m in range(len(g)):
        assert np.array_equal(gt.replica_latency(m).view(np.uint64), np.asarray(gt.lat).view(np.uint64))
    t.lat[:] = gt.lat
    r = gt.select_batch(inv.slack, 1000.0, inv.avail, upstream_supply=inv.supply,
                        min_batch=inv.min_batch, flags=inv.flags)
    exp = cselect.select_batch([t], inv.slack, 1000.0, inv.avail, inv.supply, inv.min_batch, inv.flags)
    assert_same_decisions(r, exp, "group-after-fold")
    assert g.launch_count > 0
    gt.close()
    g.close()
