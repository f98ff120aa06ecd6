"""Golden profiles produced by the UNMODIFIED reference's profile_operation (profiler.py:35-85),
for the device profile generator (csrc/sp_profile.cu).  Run in the build container:
    python tests/golden/make_golden_profiles.py

Cases (every operation of the bundled scenarios' pipelines):
* the three bundled scenarios (branching = AMBER, parallel, overhead) as shipped, with
  samples = 1 (the AMBER metadata's setting) and samples = 3 (the mean of identical draws);
* the branching scenario with log-normal noise (sigma 0.25), and with noise plus straggles
  (rate 0.15, factor 2.5), 3 samples each — the RNG stream of the reference drawn in its order.

Writes tests/golden/profile_cases.json: per case the scenario's ground truth / fleet / seed, the
operations' templates, and per operation the reference's entries (config id, latency, peak
memory, schedulable) and reference id.  Floats are stored with repr (exact round trip).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from slackpipe import profiler as prof  # noqa: E402
from slackpipe.pipeline import load_pipeline  # noqa: E402
from slackpipe.scenario import scenario_from_json  # noqa: E402

OUT = Path(__file__).resolve().parent / "profile_cases.json"


def template_json(t):
    return {"knobs": [[k.name, list(k.values)] for k in t.knobs],
            "hardware_targets": list(t.hardware_targets), "batch_sizes": list(t.batch_sizes),
            "resource_options": {k: list(v) for k, v in t.resource_options.items()}}


def case(name, sc_obj, pipe, samples, overrides=None):
    sc = scenario_from_json(sc_obj)
    if overrides:
        sc = sc.with_fault_overrides(**overrides)
    gt = sc.ground_truth
    ops = []
    for op in pipe.values():
        spec = prof.profile_operation(op, sc, samples)
        ops.append({
            "name": op.name, "executable_id": op.executable_id,
            "template": template_json(op.knob_template),
            "entries": [[e.config_id, e.latency_s, e.peak_memory_mb, e.schedulable] for e in spec.entries],
            "reference_id": spec.reference_id,
        })
    return {
        "name": name, "samples": samples, "seed": sc.seed,
        "backends": [[b.kind, b.instance_count, b.resources_per_instance, b.price_rate] for b in sc.backends],
        "noise_sigma": gt.noise_sigma, "straggle_rate": gt.straggle_rate,
        "straggle_factor": gt.straggle_factor, "peak_memory_per_item_mb": gt.peak_memory_per_item_mb,
        "ground_truth": {op: {k: {"base_seconds": t.base_seconds, "ref_resource": t.ref_resource,
                                  "resource_exponent": t.resource_exponent,
                                  "batch_exponent": t.batch_exponent,
                                  "per_item_seconds": t.per_item_seconds,
                                  "knob_multipliers": {kn: dict(v) for kn, v in t.knob_multipliers.items()}}
                              for k, t in kinds.items()}
                         for op, kinds in gt.per_op.items()},
        "ops": ops,
    }


def main():
    cases = []
    for scen in ("branching", "parallel", "overhead"):
        d = REF / "scenarios" / scen
        sc_obj = json.loads((d / "scenario.json").read_text())
        _, pipe = load_pipeline(json.loads((d / "pipeline.json").read_text()))
        for samples in (1, 3):
            cases.append(case(f"{scen}-s{samples}", sc_obj, pipe, samples))
        if scen == "branching":
            cases.append(case("branching-noise", sc_obj, pipe, 3, {"noise_sigma": 0.25}))
            cases.append(case("branching-noise-straggle", sc_obj, pipe, 3,
                              {"noise_sigma": 0.25, "straggle_rate": 0.15, "straggle_factor": 2.5}))
    OUT.write_text(json.dumps(cases))
    print(OUT, sum(len(o["entries"]) for c in cases for o in c["ops"]), "entries")


if __name__ == "__main__":
    main()
