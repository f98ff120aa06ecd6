"""Replica-parallel run engine on the B200 (k_des_run) against the
reference's own runs: all 69 golden runs (tests/golden/des/runs.json) — every decision-log row,
the report and the final latency tables bit for bit — run as replicas of one launch per run
description; the PipelineRun drop-in's CSV row; fresh random cases against oracle/engine.py."""
from __future__ import annotations

import numpy as np
import pytest

import des_cases as dc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def device_engine(gpu_ctx):
    from paper_2102_01887_b200.engine import ReplicaEngine

    return lambda spec: ReplicaEngine(spec, gpu_ctx)


@pytest.mark.parametrize("mode", ["warp", "thread", "lanes8", "lanes2"])
def test_device_engine_matches_golden_runs(device_engine, gpu_ctx, mode):
    """Both execution forms: one warp per replica (default) and one thread per replica."""
    launches0 = gpu_ctx.launch_count
    bad = []
    n = 0

    def make(spec):
        eng = device_engine(spec)
        eng.set_mode(mode)
        return eng

    for group in dc.groups(dc.runs()):
        for case, (rows, rep, lat, ev) in zip(group, dc.run_group(make, group)):
            n += 1
            errs = dc.check(case, rows, rep, lat, ev)
            if errs:
                bad.append((case["bundle"], case["target"], case.get("ablations"), errs[:3]))
    assert n == 69
    assert not bad, bad
    assert gpu_ctx.launch_count > launches0


def test_pipeline_run_dropin_csv_row(gpu_ctx, tmp_path):
    from paper_2102_01887_b200.engine import PipelineRun

    case = dc.runs()[3]  # AMBER, 50 % target
    doc, dag, sc, profiles, paths, frames = dc.bundle("branching")
    spec = dc.run_spec(case)
    run = PipelineRun(dag, {}, profiles, frames, sc, float(case["target"]), spec.params, paths=paths,
                      pipeline_name=doc["name"], ctx=gpu_ctx)
    rep = run.run_to_completion()
    assert rep.csv_row().split(",")[1:] == case["expect"]["csv_row"].split(",")[1:]
    assert dc.log_digest(run.decision_log) == case["expect"]["log_sha256"]
    run.write_decision_log(str(tmp_path / "log.tsv"))
    assert sum(1 for _ in open(tmp_path / "log.tsv")) == case["expect"]["log_rows"] + 1
    assert dc.log_digest(run.sim.trace) == case["expect"]["ev_sha256"]
    run.sim.write_trace(str(tmp_path / "events.tsv"))
    assert sum(1 for _ in open(tmp_path / "events.tsv")) == case["expect"]["ev_rows"] + 1


def test_device_engine_random_cases_vs_oracle(device_engine):
    """Fresh traces / seeds / faults on the join bundle, checked by oracle/engine.py."""
    from oracle import engine as oe
    from paper_2102_01887_b200.engine import generate_trace

    rng = np.random.default_rng(5)
    base = dict(bundle="parallel", noise_sigma=0.25, failure_rate=0.08, straggle_rate=0.05,
                straggle_factor=3.0)
    spec = dc.run_spec(base)
    doc, dag, sc, profiles, paths, _ = dc.bundle("parallel")
    eng = device_engine(spec)
    traces = [generate_trace(int(rng.integers(100, 400)), 1000 + i, {"persons": 0.7}, 3) for i in range(6)]
    targets = [float(rng.uniform(10, 90)) for _ in traces]
    seeds = [int(rng.integers(0, 2**31)) for _ in traces]
    res = eng.run(traces, targets, seeds, log_cap=20000, final_tables=True)
    t = sc.tuning
    for tr, tg, sd, r in zip(traces, targets, seeds, res):
        o = oe.Engine(dag, profiles, tr, sc, tg,
                      oe.Params(t.alpha, t.cq_capacity, t.dfp_count, t.straggler_timeout_factor,
                                t.smoothing_beta), seed=sd, paths=paths, noise_sigma=0.25,
                      failure_rate=0.08, straggle_rate=0.05, straggle_factor=3.0)
        want = o.run()
        assert dc.log_digest(eng.log_rows(r.log)) == dc.log_digest(want.log)
        assert repr(r.cost) == repr(float(want.cost))
        assert (r.failures, r.duplicates, r.invocations) == (want.failures, want.duplicates, want.invocations)
        lat = np.concatenate([o.t[op].lat for op in o.ops])
        assert np.array_equal(lat.view(np.uint64), r.lat.view(np.uint64))


@pytest.mark.parametrize("mode", ["warp", "thread"])
def test_device_engine_many_operations_vs_oracle(device_engine, mode):
    """A 64-operation pipeline (entry columns + path suffixes too large for shared memory: the
    kernels read them from global memory) against oracle/engine.py."""
    from oracle import engine as oe
    from paper_2102_01887_b200.engine import RunSpec, TuningParams, _paths
    from test_engine_host import _wide_pipeline

    dag, profiles, sc, frames = _wide_pipeline(63, 63)
    paths = _paths(dag)
    spec = RunSpec(dag, profiles, sc, TuningParams(cq_capacity=4), paths=paths)
    eng = device_engine(spec)
    eng.set_mode(mode)
    targets, seeds = [5.0, 40.0, float("inf")], [1, 2, 3]
    wants = [oe.Engine(dag, profiles, frames, sc, t, oe.Params(100.0, 4, 10, 1.5, 0.5), seed=s,
                       paths=paths).run() for t, s in zip(targets, seeds)]
    res = eng.run([frames] * 3, targets, seeds, log_cap=max(len(w.log) for w in wants) + 16)
    for w, r in zip(wants, res):
        assert dc.log_digest(eng.log_rows(r.log)) == dc.log_digest(w.log)
        assert repr(r.cost) == repr(float(w.cost)) and r.invocations == w.invocations


def test_group_engine_fans_out_over_member_contexts(gpu_ctx):
    """GroupReplicaEngine over two member contexts (both on device 0 here: the same code path as
    two GPUs) gives the single-engine results for the config-4 golden runs, in replica order."""
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200.engine import GroupReplicaEngine

    cases = [c for c in dc.runs() if c.get("group") == "c4"][:10]
    grp = sp.DeviceGroup([0, 0])

    def make(spec):
        return GroupReplicaEngine(spec, grp)

    for case, (rows, rep, lat, ev) in zip(cases, dc.run_group(make, cases)):
        assert not dc.check(case, rows, rep, lat, ev), case["target"]


@pytest.mark.parametrize("target,sha16,csv_tail", [
    (142.20064921472454, "4647eeb560b36a71",
     "142.20064921472454,132.73451153109434,0.9334311218977895,0.16671542613566986,1.0,20,0,0"),
    (0.0, "04a858b09a523792", "0.0,90.41885182994682,inf,0.3916674839012888,0.0,19,0,0"),
    (float("inf"), "3a27109b8eba0deb", "inf,193.98244659950223,0.0,0.14018874269532433,1.0,15,0,0"),
])
def test_amber_dropin_reproduces_survey_goldens(gpu_ctx, tmp_path, target, sha16, csv_tail):
    """The decision-log FILE the device drop-in writes (write_decision_log, manager.py:632-646)
    has the sha256 prefix SURVEY.md §8(c) recorded from the reference CLI's own AMBER runs, and
    the report's CSV row the recorded values (run_id aside: it hashes the CLI's flag paths)."""
    import hashlib

    from paper_2102_01887_b200.engine import PipelineRun

    doc, dag, sc, profiles, paths, frames = dc.bundle("branching")
    spec = dc.run_spec(dict(bundle="branching"))
    run = PipelineRun(dag, {}, profiles, frames, sc, target, spec.params, paths=paths,
                      pipeline_name=doc["name"], ctx=gpu_ctx)
    rep = run.run_to_completion()
    assert rep.csv_row().split(",", 1)[1] == csv_tail
    p = tmp_path / "decisions.tsv"
    run.write_decision_log(str(p))
    assert hashlib.sha256(p.read_bytes()).hexdigest()[:16] == sha16
