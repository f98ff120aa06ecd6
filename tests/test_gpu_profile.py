"""Device profile generation (csrc/sp_profile.cu, paper_2102_01887_b200/profiler.py) against
the unmodified reference: every operation of the three bundled scenarios (1 and 3 samples, with
noise, with noise and straggles — tests/golden/profile_cases.json) and the config-2 / config-5
synthetic tables (tests/golden/synth_sample.npz); the correctly rounded power against a
60-digit decimal evaluation."""
from __future__ import annotations

import hashlib
import json
import random
from decimal import Decimal, getcontext

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu


def _scenario(case):
    from paper_2102_01887_b200.scenario import BackendSpec, GroundTruthModel, OpKindTruth, Scenario

    gt = GroundTruthModel(
        per_op={op: {k: OpKindTruth(**t) for k, t in kinds.items()} for op, kinds in case["ground_truth"].items()},
        noise_sigma=case["noise_sigma"], straggle_rate=case["straggle_rate"],
        straggle_factor=case["straggle_factor"], peak_memory_per_item_mb=case["peak_memory_per_item_mb"])
    return Scenario(case["name"], tuple(BackendSpec(*b) for b in case["backends"]), gt, case["seed"])


def _op(o):
    from paper_2102_01887_b200.pipeline import Knob, KnobTemplate, OperationSpec

    t = o["template"]
    tpl = KnobTemplate(tuple(Knob(n, tuple(v)) for n, v in t["knobs"]), tuple(t["hardware_targets"]),
                       tuple(t["batch_sizes"]), {k: tuple(v) for k, v in t["resource_options"].items()})
    return OperationSpec(o["name"], o["executable_id"], tpl)


def test_profile_operation_vs_reference(gpu_ctx):
    from paper_2102_01887_b200 import profiler

    cases = json.loads((GOLDEN / "profile_cases.json").read_text())
    n = 0
    for case in cases:
        sc = _scenario(case)
        for o in case["ops"]:
            spec = profiler.profile_operation(_op(o), sc, case["samples"])
            got = [[e.config_id, e.latency_s, e.peak_memory_mb, e.schedulable] for e in spec.entries]
            assert [g[0] for g in got] == [w[0] for w in o["entries"]], (case["name"], o["name"])
            gl = np.array([g[1] for g in got])
            wl = np.array([w[1] for w in o["entries"]])
            assert np.array_equal(gl.view(np.uint64), wl.view(np.uint64)), (case["name"], o["name"])
            assert [g[2:] for g in got] == [w[2:] for w in o["entries"]]
            assert spec.reference_id == o["reference_id"]
            n += len(got)
    assert n == 588


def test_profile_enumeration_matches_host(gpu_ctx):
    """The kernel's decoded (kind, resource, batch) of every assignment = enumerate_configs."""
    from paper_2102_01887_b200 import profiler
    from paper_2102_01887_b200.pipeline import enumerate_configs

    case = json.loads((GOLDEN / "profile_cases.json").read_text())[0]
    sc = _scenario(case)
    for o in case["ops"]:
        op = _op(o)
        lat, kinds, kidx, res, bat = profiler.profile_latencies(op, sc, 1)
        asg = enumerate_configs(op.knob_template)
        assert [kinds[k] for k in kidx] == [a.backend_kind for a in asg]
        assert res.tolist() == [a.resource_request for a in asg]
        assert bat.tolist() == [a.batch_size for a in asg]


@pytest.mark.parametrize("tag,with_model", [("c2", False), ("c5", True)])
def test_profile_synthetic_tables_vs_goldens(gpu_ctx, tag, with_model):
    """Config 2 (4,096 entries) and config 5 (16,384) generated on the device and loaded into an
    OpTable: latencies and config ids equal the reference's (make_golden.py gen_synth)."""
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import profiler, synth
    from paper_2102_01887_b200.pipeline import Knob, KnobTemplate, OperationSpec
    from paper_2102_01887_b200.scenario import GroundTruthModel, OpKindTruth, Scenario

    d = golden("synth_sample")
    knobs = [Knob("sampling", synth.SAMPLING), Knob("variant", synth.VARIANT)]
    if with_model:
        knobs.append(Knob("model", synth.MODEL))
    tpl = KnobTemplate(tuple(knobs), ("cpu", "gpu"), synth.BATCHES, {"cpu": synth.CPU_RES, "gpu": synth.GPU_RES})
    tr = synth.synth_truths(with_model)
    gt = GroundTruthModel(per_op={"op": {k: OpKindTruth(v.base_seconds, v.ref_resource, v.resource_exponent,
                                                       v.batch_exponent, 0.0, v.knob_multipliers)
                                         for k, v in tr.items()}})
    sc0 = synth.synth_scenario()
    sc = Scenario("synth", sc0.backends, gt, seed=1)
    spec = profiler.profile_operation(OperationSpec("op", "synth-v1", tpl), sc, 1)
    table = sp.OpTable(spec, sc)
    assert np.array_equal(np.asarray(table.lat).view(np.uint64), d[f"{tag}_lat"].view(np.uint64))
    sha = hashlib.sha256("\n".join(e.config_id for e in table.entries).encode()).digest()
    assert np.array_equal(np.frombuffer(sha, np.uint8), d[f"{tag}_ids_sha"])
    assert table.ref_index == int(d[f"{tag}_ref_index"])


def test_pow_correctly_rounded_vs_decimal(gpu_ctx):
    from paper_2102_01887_b200 import profiler

    getcontext().prec = 60
    rnd = random.Random(3)
    xs = [rnd.uniform(1e-3, 1e3) for _ in range(1500)] + [float(2 ** k) for k in range(-20, 21)] + \
         [rnd.choice([1.0, 2.0, 4.0, 0.5, 3.0, 10.0]) for _ in range(200)]
    ys = [rnd.uniform(-3.0, 3.0) for _ in range(1500)] + [rnd.choice([0.5, -0.5, 2.0, 0.85, -0.3]) for _ in range(41)] + \
         [rnd.choice([0.5, 2.0, 3.0, -1.0, 0.25, 1.0, 0.0]) for _ in range(200)]
    got = profiler.pow_correctly_rounded(np.array(xs), np.array(ys))
    want = np.array([float((Decimal(x).ln() * Decimal(y)).exp()) if y != 0 else 1.0 for x, y in zip(xs, ys)])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
