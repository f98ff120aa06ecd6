"""The run engine's source (csrc/sp_des.cuh) compiled for the host — a test harness, so the
CPU suite checks the engine logic without a GPU — against the reference's own runs: every
decision-log row, the report and the final latency tables of the 69 golden runs
(tests/golden/des/runs.json: the three bundled scenarios, 5 targets, every ablation, noise /
straggle / failure injection, profile scaling, and 40 config-4 replicas), and against the live
reference on fresh random cases in the build container.  The device kernel runs the same source
(tests/test_gpu_engine.py)."""
from __future__ import annotations

import numpy as np
import pytest

import des_cases as dc


@pytest.fixture(scope="module")
def host_engine():
    return dc.host_engine_factory(dc.host_library())


def test_host_engine_matches_golden_runs(host_engine):
    bad = []
    n = 0
    for group in dc.groups(dc.runs()):
        for case, (rows, rep, lat, ev) in zip(group, dc.run_group(host_engine, group)):
            n += 1
            errs = dc.check(case, rows, rep, lat, ev)
            if errs:
                bad.append((case["bundle"], case["target"], case.get("ablations"), errs[:3]))
    assert n == 69
    assert not bad, bad


def test_host_engine_capacity_retry(host_engine):
    """A replica that runs out of invocation slots (failures re-run invocations beyond the
    default 1.25 per item) is re-run with doubled capacity; the result is still exact."""
    case = next(c for c in dc.runs() if c["bundle"] == "overhead" and c.get("failure_rate"))
    spec = dc.run_spec(case)
    eng = host_engine(spec)
    eng.cap_scale = 1.0
    res = eng.run([dc.frames_of(case)], [float(case["target"])], [dc.seed_of(case)],
                  log_cap=case["expect"]["log_rows"] + 16, final_tables=True)[0]
    from paper_2102_01887_b200.engine import report_of

    rep = report_of(res, target_s=float(case["target"]), scenario_name=spec.scenario.name,
                    pipeline_name="x", seed=dc.seed_of(case), ablations=())
    assert not dc.check(case, eng.log_rows(res.log), rep, res.lat)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_host_engine_matches_live_reference_random(ref, host_engine, seed):
    """Fresh random AMBER runs (trace, target, ablations, noise / straggle / failure, profile
    scale) of the live reference engine (build container only) against the engine source."""
    import json
    import tempfile

    from slackpipe import cli, manager, pipeline, profiler, workload
    from slackpipe import scenario as scn
    from paper_2102_01887_b200.engine import RunSpec, TuningParams, report_of

    rng = np.random.default_rng(seed)
    base = "/root/reference/pkg/scenarios/branching"
    doc = json.load(open(base + "/pipeline.json"))
    dag, ops = pipeline.load_pipeline(doc)
    sc = scn.load_scenario(base + "/scenario.json")
    store = profiler.MetadataStore(tempfile.mkdtemp())
    profiles, _ = cli._ensure_profiles(store, ops, sc, sc.tuning.samples_per_config)
    paths = cli._paths_for(store, doc, dag)
    frames = workload.generate_trace(int(rng.integers(200, 700)), seed + 100,
                                     {"cars": float(rng.uniform(0.2, 1.5)), "persons": float(rng.uniform(0.2, 1.5))}, 4)
    abl = [a for a in ("fb", "dfp", "sdb", "eslc", "pbc") if rng.random() < 0.25]
    faults = dict(noise_sigma=float(rng.choice([0.0, 0.25])), failure_rate=float(rng.choice([0.0, 0.05])),
                  straggle_rate=float(rng.choice([0.0, 0.05])), straggle_factor=3.0)
    rs = sc.with_fault_overrides(**faults)
    target = float(rng.uniform(5.0, 60.0))
    scale = float(rng.choice([1.0, 0.8, 1.3]))
    tp = cli._tuning_params(rs, None)
    run = manager.PipelineRun(dag, ops, profiles, frames, rs, target, tp, ablations=frozenset(abl),
                              seed=seed, paths=paths, profile_scale=scale)
    want = run.run_to_completion()
    spec = RunSpec(dag, profiles, rs, TuningParams(tp.alpha, tp.cq_capacity, tp.dfp_count,
                                                   tp.straggler_timeout_factor, tp.smoothing_beta),
                   ablations=abl, paths=paths, profile_scale=scale)
    eng = host_engine(spec)
    res = eng.run([frames], [target], [seed], log_cap=len(run.configurator.decision_log) + 16,
                  final_tables=True, event_cap=len(run.sim.trace) + 16)[0]
    assert dc.log_digest(eng.log_rows(res.log)) == dc.log_digest(run.configurator.decision_log)
    assert dc.log_digest(eng.event_rows(res.events)) == dc.log_digest(run.sim.trace)
    got = report_of(res, target_s=target, scenario_name=rs.name, pipeline_name="x", seed=seed)
    for f in ("latency_s", "cost", "slack_met_frac", "configs_used", "failures", "duplicates",
              "invocations", "completed", "terminal_items", "decision_count"):
        assert repr(float(getattr(got, f))) == repr(float(getattr(want, f))), f
    lat = np.concatenate([run.tables[o].lat for o in sorted(run.tables)])
    assert np.array_equal(lat.view(np.uint64), res.lat.view(np.uint64))


def _wide_pipeline(n_ops: int, seed: int):
    """A synthetic pipeline of n_ops operations (chain + skip edges + one join + a predicate /
    fan-out branch), two backend kinds, hand-made profiles and ground truth."""
    from paper_2102_01887_b200.pipeline import BranchPredicate, ConfigEntry, ConfigSpec, PipelineDag
    from paper_2102_01887_b200.scenario import BackendSpec, GroundTruthModel, OpKindTruth, Scenario

    rng = np.random.default_rng(seed)
    ops = [f"s{i:02d}" for i in range(n_ops)]
    edges = [(ops[i], ops[i + 1]) for i in range(n_ops - 1)]
    edges += [(ops[3], ops[9]), (ops[12], ops[n_ops - 5])]  # skips (ops 9 / n-5 become joins)
    edges += [(ops[6], "br")]
    ops.append("br")
    preds = {(ops[6], "br"): BranchPredicate("persons", ">", 0)}
    dag = PipelineDag(vertices=tuple(ops), edges=tuple(edges), branch_predicates=preds,
                      fanout_rules={"br": "persons"})
    profiles, truth = {}, {}
    for op in ops:
        ents = []
        for kind, res_opts, bs in (("cpu", (1, 2, 4), (1, 4)), ("gpu", (4, 8), (1, 8))):
            for r in res_opts:
                for b in bs:
                    lat = float(rng.uniform(0.05, 2.0)) * (b ** 0.7) / (r ** 0.3)
                    ents.append(ConfigEntry(f"{kind}-r{r}-b{b}", kind, {}, b, r, lat, lat))
        profiles[op] = ConfigSpec(op, ents, "cpu-r1-b1")
        truth[op] = {"cpu": OpKindTruth(float(rng.uniform(0.1, 1.0)), 1, 0.3, 0.8, 0.01),
                     "gpu": OpKindTruth(float(rng.uniform(0.02, 0.2)), 4, 0.2, 0.4, 0.001)}
    sc = Scenario("wide", (BackendSpec("cpu", 8, 4, 1.32e-5), BackendSpec("gpu", 2, 8, 9e-4)),
                  GroundTruthModel(truth, noise_sigma=0.2, failure_rate=0.02), 11)
    frames = [(i, {"persons": int(x)}) for i, x in enumerate(rng.poisson(0.7, size=120))]
    return dag, profiles, sc, frames


@pytest.mark.parametrize("n_ops", [40, 63])
def test_host_engine_many_operations_vs_oracle(host_engine, n_ops):
    """Pipelines beyond the bundled 7 operations (up to 64 — ancestors as a 64-bit mask), with
    joins, a predicate / fan-out branch, noise and failures, against oracle/engine.py."""
    from oracle import engine as oe
    from paper_2102_01887_b200.engine import RunSpec, TuningParams, _paths, report_of

    dag, profiles, sc, frames = _wide_pipeline(n_ops, n_ops)
    paths = _paths(dag)
    params = TuningParams(cq_capacity=4)
    spec = RunSpec(dag, profiles, sc, params, paths=paths)
    eng = host_engine(spec)
    for target, seed in ((5.0, 1), (40.0, 2), (float("inf"), 3)):
        want = oe.Engine(dag, profiles, frames, sc, target, oe.Params(100.0, 4, 10, 1.5, 0.5),
                         seed=seed, paths=paths).run()
        res = eng.run([frames], [target], [seed], log_cap=len(want.log) + 16, final_tables=True)[0]
        assert dc.log_digest(eng.log_rows(res.log)) == dc.log_digest(want.log), target
        got = report_of(res, target_s=target, scenario_name="wide", pipeline_name="x", seed=seed)
        for f in ("latency_s", "cost", "failures", "duplicates", "invocations", "completed",
                  "terminal_items", "decision_count"):
            assert repr(float(getattr(got, f))) == repr(float(getattr(want, f))), (target, f)
