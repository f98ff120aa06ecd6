"""CPU restatement of profile generation — TEST ORACLE ONLY.

Follows profiler.profile_operation (profiler.py:35-85): enumerate_configs (pipeline.py:454-475),
per assignment `samples` draws of backend.draw_actual_latency (backend.py:36-58) over
OpKindTruth.base_latency (scenario.py:68-77) with the generator seeded by
content_hash([scenario.seed, executable_id]) (pipeline.py:31-37), and the mean
float(sum(drawn) / len(drawn)).  Pure Python floats (CPython's `**` and math.exp), so it is the
reference's arithmetic exactly; pinned against tests/golden/profile_cases.json (produced by the
unmodified reference, tests/golden/make_golden_profiles.py).
"""
from __future__ import annotations

import hashlib
import itertools
import json
import math

import numpy as np


def content_hash(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def enumerate_assignments(template: dict):
    """(kind, resource, batch, knob_values) in enumerate_configs order."""
    names = [k[0] for k in template["knobs"]]
    values = [k[1] for k in template["knobs"]]
    for kind in sorted(template["hardware_targets"]):
        for r in template["resource_options"][kind]:
            for b in sorted(template["batch_sizes"]):
                for combo in itertools.product(*values):
                    yield kind, r, b, tuple(zip(names, combo))


def base_latency(t: dict, r: int, b: int, knobs) -> float:
    lat = t["base_seconds"]
    if t["resource_exponent"]:
        lat *= (r / t["ref_resource"]) ** -t["resource_exponent"]
    lat *= b ** t["batch_exponent"]
    for knob, value in knobs:
        table = t["knob_multipliers"].get(knob)
        if table:
            lat *= table.get(str(value), 1.0)
    return lat


def profile_latencies(case: dict, op: dict) -> list[float]:
    """One operation of a profile_cases.json case: the profiled latency of every assignment."""
    rng = np.random.default_rng(int(content_hash([case["seed"], op["executable_id"]])[:16], 16))
    truths = case["ground_truth"][op["name"]]
    sigma, rate, factor = case["noise_sigma"], case["straggle_rate"], case["straggle_factor"]
    out = []
    for kind, r, b, knobs in enumerate_assignments(op["template"]):
        t = truths[kind]
        drawn = []
        for _ in range(max(1, case["samples"])):
            latency = base_latency(t, r, b, knobs) + t["per_item_seconds"] * b
            if sigma > 0.0:
                latency *= math.exp(rng.normal(0.0, sigma))
            if rate > 0.0 and rng.random() < rate:
                latency *= factor
            drawn.append(latency)
        out.append(float(sum(drawn) / len(drawn)))
    return out
