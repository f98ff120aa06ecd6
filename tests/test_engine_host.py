"""The run engine's source (csrc/sp_des.cuh) compiled for the host — a test harness, so the
CPU suite checks the engine logic without a GPU — against the reference's own runs: every
decision-log row, the report and the final latency tables of the 69 golden runs
(tests/golden/des/runs.json: the three bundled scenarios, 5 targets, every ablation, noise /
straggle / failure injection, profile scaling, and 40 config-4 replicas), and against the live
reference on fresh random cases in the build container.  The device kernel runs the same source
(tests/test_gpu_engine.py)."""
from __future__ import annotations

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
