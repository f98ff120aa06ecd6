"""oracle/engine.py (the CPU restatement of the reference run engine) pinned to the reference:
against the golden runs (any box) and against the live reference on fresh random cases (build
container only)."""
from __future__ import annotations

import math
import tempfile

import numpy as np
import pytest

import des_cases as dc
from oracle import engine as oe


def _oracle_run(case, frames=None):
    doc, dag, sc, profiles, paths, bundle_frames = dc.bundle(case["bundle"])
    t = sc.tuning
    p = oe.Params(t.alpha if case.get("alpha") is None else case["alpha"], t.cq_capacity,
                  t.dfp_count, t.straggler_timeout_factor, t.smoothing_beta)
    eng = oe.Engine(dag, profiles, frames if frames is not None else dc.frames_of(case), sc,
                    float(case["target"]), p, ablations=case.get("ablations", []),
                    seed=dc.seed_of(case), paths=paths, profile_scale=case.get("profile_scale", 1.0),
                    noise_sigma=case.get("noise_sigma"), failure_rate=case.get("failure_rate"),
                    straggle_rate=case.get("straggle_rate"), straggle_factor=case.get("straggle_factor"))
    rep = eng.run()
    lat = np.concatenate([eng.t[o].lat for o in eng.ops])
    return rep, lat


# one case per behaviour: targets fast / cheap / 50 %, every ablation, noise (straggler
# duplicates), failures (retries), straggles, profile scaling, the join bundle, a config-4 replica
PICK = [0, 1, 3, 6, 7, 8, 9, 10, 12, 14, 15, 16, 18, 19, 20, 24, 25, 29]


@pytest.mark.parametrize("i", PICK)
def test_oracle_engine_matches_golden_run(i):
    case = dc.runs()[i]
    rep, lat = _oracle_run(case)
    assert not dc.check(case, rep.log, rep, lat)


def _ref_build(ref, bundle_name):
    from slackpipe import cli, pipeline, profiler
    from slackpipe import scenario as scn
    import json

    base = f"/root/reference/pkg/scenarios/{bundle_name}"
    doc = json.load(open(base + "/pipeline.json"))
    dag, ops = pipeline.load_pipeline(doc)
    sc = scn.load_scenario(base + "/scenario.json")
    store = profiler.MetadataStore(tempfile.mkdtemp())
    profiles, _ = cli._ensure_profiles(store, ops, sc, sc.tuning.samples_per_config)
    return doc, dag, ops, sc, profiles, cli._paths_for(store, doc, dag)


@pytest.mark.parametrize("seed", [101, 202])
def test_oracle_engine_matches_live_reference(ref, seed):
    from slackpipe import cli, manager, workload

    doc, dag, ops, sc, profiles, paths = _ref_build(ref, "parallel")
    rng = np.random.default_rng(seed)
    frames = workload.generate_trace(int(rng.integers(200, 600)), seed, {"persons": 0.5}, 2)
    rs = sc.with_fault_overrides(noise_sigma=float(rng.uniform(0.1, 0.4)),
                                 failure_rate=float(rng.uniform(0.0, 0.1)),
                                 straggle_rate=0.05, straggle_factor=3.0)
    target = float(rng.uniform(10, 80))
    tp = cli._tuning_params(rs, None)
    run = manager.PipelineRun(dag, ops, profiles, frames, rs, target, tp, seed=seed, paths=paths)
    want = run.run_to_completion()
    eng = oe.Engine(dag, profiles, frames, rs, target,
                    oe.Params(tp.alpha, tp.cq_capacity, tp.dfp_count, tp.straggler_timeout_factor,
                              tp.smoothing_beta), seed=seed, paths=paths)
    got = eng.run()
    assert dc.log_digest(got.log) == dc.log_digest(run.configurator.decision_log)
    for f in ("latency_s", "cost", "slack_met_frac", "failures", "duplicates", "invocations"):
        a, b = getattr(got, f), getattr(want, f)
        assert repr(float(a)) == repr(float(b)), f
