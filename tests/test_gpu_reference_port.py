"""The reference's own unit tests for the hot path (pkg/tests/test_configurator.py and the
feedback cases of test_manager.py), restated against the GPU-backed drop-in.  Expected values
are the reference tests' exact literals."""
from __future__ import annotations

import random
import time

import pytest

pytestmark = pytest.mark.gpu


def make_entry(config_id=None, *, kind="cpu", resource=1, batch=1, latency=1.0, schedulable=True,
               knob_values=None):
    from paper_2102_01887_b200 import ConfigEntry

    if config_id is None:
        config_id = f"{kind}-r{resource}-b{batch}"
        if knob_values:
            config_id += "-" + "-".join(f"{k}={v}" for k, v in sorted(knob_values.items()))
    return ConfigEntry(config_id, kind, dict(knob_values or {}), batch, resource, latency, latency,
                       schedulable=schedulable)


def make_spec(op, entries, reference_id=None):
    from paper_2102_01887_b200 import ConfigSpec

    return ConfigSpec(op, entries, reference_id or entries[0].config_id)


def make_scenario(rows):
    from paper_2102_01887_b200 import BackendSpec, Scenario

    return Scenario("test", tuple(BackendSpec(k, n, r, p) for k, n, r, p in rows))


def two_kind():
    return make_scenario([("cpu", 4, 4, 1e-5), ("gpu", 2, 8, 3e-4)])


# -- queueing / slack / objective (test_configurator.py:47-227) ------------------------------

QUEUEING_FIXTURES = [
    ([], 4.0, 0.0), ([(2.0, 1)], 4.0, 0.5), ([(2.0, 1), (3.0, 2)], 4.0, 2.0), ([(0.5, 4)], 8.0, 0.25),
    ([(0.25, 2), (0.25, 2)], 2.0, 0.5), ([(1.0, 1)] * 8, 16.0, 0.5), ([(4.0, 4)], 2.0, 8.0),
    ([(1.5, 2)], 4.0, 0.75), ([(0.125, 8)], 4.0, 0.25), ([(2.0, 2), (1.0, 4)], 8.0, 1.0),
    ([(3.0, 1), (1.0, 3)], 2.0, 3.0), ([(0.5, 1), (0.5, 1), (0.5, 2)], 4.0, 0.5),
    ([(10.0, 1)], 1.0, 10.0), ([(0.75, 4)], 16.0, 0.1875), ([(1.25, 2)], 4.0, 0.625),
    ([(6.0, 2), (2.0, 1)], 8.0, 1.75), ([(0.0625, 16)], 2.0, 0.5), ([(5.0, 1), (3.0, 1), (2.0, 1)], 4.0, 2.5),
    ([(1.0, 2), (2.0, 4), (0.5, 8)], 8.0, 1.75), ([(7.0, 2)], 2.0, 7.0),
]


@pytest.mark.parametrize("queued,pool,expected", QUEUEING_FIXTURES)
def test_queueing_matches_hand_computation(gpu_ctx, queued, pool, expected):
    from paper_2102_01887_b200 import estimate_queueing

    entries = [make_entry(f"q{i}", resource=r, latency=lat) for i, (lat, r) in enumerate(queued)]
    assert estimate_queueing(entries, pool) == expected


PATHS = (("a", "b", "d"), ("a", "c", "d"))
REF = {"a": 1.0, "b": 2.0, "c": 3.0, "d": 4.0}


def test_slack_fixtures(gpu_ctx):
    from paper_2102_01887_b200 import compute_slack, remaining_path_latency

    assert remaining_path_latency("b", ("a", "b", "d"), REF) == 6.0
    assert remaining_path_latency("a", ("a", "b", "d"), REF) == 7.0
    assert remaining_path_latency("d", ("a", "b", "d"), REF) == 4.0
    cs = lambda op, t, e, q: compute_slack(op, "cpu", target_s=t, elapsed_s=e, queueing_s=q,
                                           paths=PATHS, ref_latency=REF)
    got = cs("a", 20.0, 2.0, 1.0)
    assert got.seconds == 17.0 / 8.0 and got.backend_kind == "cpu"
    assert cs("d", 20.0, 2.0, 1.0).seconds == 17.0
    assert cs("c", 10.0, 0.0, 0.0).seconds == (3.0 / 7.0) * 10.0
    assert cs("b", 20.0, 0.0, 0.0).seconds == (2.0 / 6.0) * 20.0
    assert cs("b", 20.0, 6.0, 2.0).seconds == (2.0 / 6.0) * 12.0
    assert cs("a", 2.0, 2.0, 1.0).seconds == (1.0 / 7.0) * -1.0
    with pytest.raises(ValueError):
        cs("zz", 10.0, 0.0, 0.0)


def test_slack_min_over_paths_random(gpu_ctx):
    """test_configurator.py:164-185 with 150 random draws."""
    from paper_2102_01887_b200 import compute_slack

    for seed in range(150):
        rng = random.Random(seed)
        ops = [f"v{i}" for i in range(rng.randint(2, 6))]
        ref = {op: rng.choice([0.25, 0.5, 1.0, 2.0, 4.0]) for op in ops}
        paths = []
        for _ in range(rng.randint(1, 4)):
            k = rng.randint(1, len(ops))
            paths.append(tuple(sorted(rng.sample(ops, k), key=ops.index)))
        op = rng.choice([o for p in paths for o in p])
        budget = float(rng.randint(-8, 64))
        got = compute_slack(op, "cpu", target_s=budget, elapsed_s=0.0, queueing_s=0.0,
                            paths=tuple(paths), ref_latency=ref)
        per_path = []
        for p in paths:
            if op in p:
                tot = 0.0
                for o in p[p.index(op):]:
                    tot += ref[o]
                per_path.append(ref[op] / tot * budget)
        assert got.seconds == min(per_path)


def test_objective_fixtures(gpu_ctx):
    from paper_2102_01887_b200 import objective

    assert objective(make_entry(resource=1, batch=1, latency=0.5), 1.0, price_rate=1e-3,
                     pool_resources=8.0, alpha=100.0) == 0.0005
    assert objective(make_entry(resource=2, batch=4, latency=2.0), 3.0, price_rate=1e-3,
                     pool_resources=10.0, alpha=100.0) == 0.001
    assert objective(make_entry(resource=2, batch=4, latency=2.0), 1.0, price_rate=1e-3,
                     pool_resources=10.0, alpha=100.0) == 0.001 + 100.0 * (2.0 * 2 / (4 * 10.0))
    # boundary: latency == slack is penalized (strict <)
    assert objective(make_entry(resource=1, batch=1, latency=1.0), 1.0, price_rate=0.0,
                     pool_resources=100.0, alpha=100.0) == 1.0


# -- OpTable mechanics (test_configurator.py:240-390) -------------------------------------------

def test_table_filters_and_reference(gpu_ctx):
    from paper_2102_01887_b200 import OpTable

    spec = make_spec("op", [
        make_entry(kind="cpu", resource=1, batch=1, latency=1.0),
        make_entry(kind="cpu", resource=8, batch=1, latency=0.5),
        make_entry(kind="tpu", resource=1, batch=1, latency=0.1),
        make_entry(kind="cpu", resource=2, batch=1, latency=0.9, schedulable=False),
    ])
    assert [e.config_id for e in OpTable(spec, two_kind()).entries] == ["cpu-r1-b1"]
    with pytest.raises(ValueError):
        OpTable(make_spec("op", [make_entry(kind="cpu", resource=8, batch=1)]), two_kind())
    t = OpTable(make_spec("op", [make_entry(kind="cpu", resource=8, batch=1, latency=1.0),
                                 make_entry(kind="gpu", resource=4, batch=1, latency=0.2)]), two_kind())
    assert t.ref_index == -1 and t.ref_entry.config_id == "cpu-r8-b1"
    t = OpTable(make_spec("op", [make_entry(kind="cpu", resource=1, batch=1, latency=1.0)]), two_kind())
    t.set_latency(0, 2.5)
    assert t.lat[0] == 2.5 and t.entries[0].latency_s == 2.5
    score, cost = t.scores({"cpu": 10.0, "gpu": 10.0}, 100.0)
    assert score[0] == 2.5e-5 and cost[0] == 2.5e-5


def test_select_behaviours(gpu_ctx):
    from paper_2102_01887_b200 import OpTable

    sc = two_kind()
    t = OpTable(make_spec("op", [make_entry(kind="cpu", resource=1, batch=1, latency=1.0),
                                 make_entry(kind="gpu", resource=4, batch=1, latency=0.1)]), sc)
    assert t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 1, allow_delay=False).entry.config_id == "cpu-r1-b1"
    assert t.select({"cpu": 0.5, "gpu": 0.5}, 100.0, 1, allow_delay=False).entry.config_id == "gpu-r4-b1"
    t = OpTable(make_spec("op", [make_entry(kind="cpu", resource=2, batch=1, latency=1.0),
                                 make_entry(kind="cpu", resource=1, batch=1, latency=2.0)]), sc)
    assert t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 1, allow_delay=False).entry.config_id == "cpu-r1-b1"
    t = OpTable(make_spec("op", [make_entry(kind="cpu", resource=1, batch=1, latency=1.0, knob_values={"m": "b"}),
                                 make_entry(kind="cpu", resource=1, batch=1, latency=1.0, knob_values={"m": "a"})]), sc)
    assert t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 1, allow_delay=False).entry.config_id == "cpu-r1-b1-m=a"
    t = OpTable(make_spec("op", [make_entry(kind="cpu", resource=1, batch=1, latency=1.0),
                                 make_entry(kind="cpu", resource=1, batch=8, latency=2.0)]), sc)
    d = t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 2, allow_delay=True, upstream_supply=6)
    assert d.kind == "delay" and d.entry.batch_size == 8 and d.fill == 2 and d.wait_budget_s == 10.0 - 2.0
    d = t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 2, allow_delay=True, upstream_supply=1)
    assert d.kind == "assign" and d.entry.batch_size == 1 and d.fill == 1
    t = OpTable(make_spec("op", [make_entry(kind="cpu", resource=1, batch=1, latency=1.0),
                                 make_entry(kind="gpu", resource=4, batch=4, latency=0.2)]), sc)
    d = t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 3, allow_delay=False, excluded_kinds=frozenset({"cpu"}))
    assert d.kind == "assign" and d.fill == 3
    assert t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 4, allow_delay=False,
                    excluded_kinds=frozenset({"cpu"})).entry.backend_kind == "gpu"
    assert t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 4, allow_delay=False,
                    excluded_kinds=frozenset({"cpu", "gpu"})) is None
    assert t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 4, allow_delay=False, min_batch=2).entry.batch_size == 4
    assert t.select({"cpu": 10.0, "gpu": 10.0}, 100.0, 8, allow_delay=False, min_batch=8) is None


def test_affinity_ratio_and_edges(gpu_ctx):
    from paper_2102_01887_b200 import OpTable, TuningParams, affinity

    sc = two_kind()
    t = OpTable(make_spec("op", [make_entry(kind="cpu", resource=1, batch=1, latency=1.0),
                                 make_entry(kind="gpu", resource=4, batch=1, latency=0.1)]), sc)
    s = {"cpu": 10.0, "gpu": 10.0}
    assert t.affinity("gpu", s, 100.0) == pytest.approx(1e-5 / 1.2e-4, rel=1e-12)
    assert t.affinity("tpu", s, 100.0) is None
    solo = OpTable(make_spec("op", [make_entry(kind="cpu", resource=1, batch=1)]), sc)
    assert solo.affinity("cpu", s, 100.0) == float("inf")
    with pytest.raises(ValueError):
        affinity(make_spec("op", [make_entry(kind="cpu")]), sc, "gpu", s, TuningParams())


def _brute_force_pick(spec, scenario, slacks, alpha):
    best_key = best = None
    for e in spec.entries:
        if not e.schedulable:
            continue
        try:
            b = scenario.backend(e.backend_kind)
        except KeyError:
            continue
        if e.resource_request > b.resources_per_instance:
            continue
        pool = float(b.pool_resources)
        cost = (e.resource_request * e.latency_s) * b.price_rate / e.batch_size
        score = cost + 0.0 if e.latency_s < slacks[e.backend_kind] else \
            cost + alpha * ((e.latency_s * e.resource_request) / (e.batch_size * pool))
        key = (score, cost, e.resource_request, e.config_id)
        if best_key is None or key < best_key:
            best_key, best = key, e
    return best


@pytest.mark.parametrize("seed", [987654321, 24601])
def test_selection_matches_brute_force_on_randomized_instances(gpu_ctx, seed):
    """test_configurator.py:422-460 and test_acceptance.py:100-135 (1,000 instances each)."""
    from paper_2102_01887_b200 import TuningParams, select_config

    sc = make_scenario([("cpu", 4, 4, 1.32e-5), ("gpu", 2, 8, 3.0e-4), ("lite", 64, 2, 8.0e-6)])
    caps = {"cpu": 4, "gpu": 8, "lite": 2}
    rng = random.Random(seed)
    t0 = time.perf_counter()
    for case in range(1000):
        entries = [make_entry(kind="cpu", resource=rng.choice([1, 2]), batch=1,
                              latency=rng.uniform(0.05, 4.0), knob_values={"i": 0})]
        for i in range(rng.randint(0, 11)):
            kind = rng.choice(["cpu", "gpu", "lite"])
            res = rng.choice([1, 2, 4, 8])
            entries.append(make_entry(kind=kind, resource=res, batch=rng.choice([1, 2, 4, 8, 16]),
                                      latency=rng.uniform(0.01, 8.0), schedulable=res <= caps[kind],
                                      knob_values={"i": i + 1}))
        spec = make_spec("op", entries)
        slacks = {k: rng.uniform(-2.0, 5.0) for k in ("cpu", "gpu", "lite")}
        alpha = rng.choice([0.0, 1.0, 100.0, 1000.0])
        exp = _brute_force_pick(spec, sc, slacks, alpha)
        avail = max(e.batch_size for e in entries)
        got = select_config(spec, sc, slacks, available=avail, params=TuningParams(alpha=alpha),
                            allow_delay=False)
        assert got.entry.config_id == exp.config_id, case
        assert got.fill == min(got.entry.batch_size, avail)
    assert time.perf_counter() - t0 < 60.0


def test_select_config_exact_tie_prefers_cheaper_cost(gpu_ctx):
    from paper_2102_01887_b200 import TuningParams, select_config

    sc = make_scenario([("cpu", 192, 1, 0.5), ("gpu", 128, 1, 0.25)])
    spec = make_spec("op", [make_entry(kind="cpu", resource=1, batch=1, latency=1.0),
                            make_entry(kind="gpu", resource=1, batch=1, latency=1.0)])
    got = select_config(spec, sc, {"cpu": -1.0, "gpu": -1.0}, available=1,
                        params=TuningParams(alpha=96.0), allow_delay=False)
    assert got.objective_value == 1.0 and got.entry.config_id == "gpu-r1-b1"


# -- feedback (test_manager.py:28-41) -------------------------------------------------------------

def test_apply_feedback_fixtures(gpu_ctx):
    from paper_2102_01887_b200 import apply_feedback

    assert apply_feedback(2.0, 4.0, 0.5) == 3.0
    assert apply_feedback(2.0, 4.0, 1.0) == 4.0
    assert apply_feedback(2.0, 4.0, 0.25) == 2.5
    est = 0.5
    for _ in range(10):
        est = apply_feedback(est, 1.0, 0.5)
    assert 1.0 - est == 2.0 ** -11
