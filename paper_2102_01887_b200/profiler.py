"""Profile generation with the latency law evaluated on the B200.

``profile_operation`` is the reference's ``profiler.profile_operation`` (profiler.py:35-85):
same arguments, same validation, same ``ConfigSpec`` out.  The cross product of the knob
template (pipeline.py:454-475) and the ground-truth law of every assignment (scenario.py:68-77,
backend.py:36-58, the sample mean of profiler.py:64-68) are evaluated by one kernel
(``sp_profile_configs``, csrc/sp_profile.cu).  What stays on the host is what is inherently
sequential or string-valued: the reference's RNG stream (numpy ``default_rng`` seeded by the
content hash of (scenario seed, executable id), normals through CPython's ``math.exp`` and the
straggle Bernoulli draws, in the reference's per-sample order) and the config-id strings.
"""
from __future__ import annotations

import math

import numpy as np

from ._lib import check, get_context, ptr
from .pipeline import ConfigEntry, ConfigSpec, content_hash, enumerate_configs, reference_config

DEFAULT_SAMPLES = 3  # profiler.py:31


def _rng_factors(model, n: int, samples: int, rng):
    """The multiplicative noise and straggle factors of every draw, in the order
    draw_actual_latency consumes the generator (backend.py:53-58): per assignment, per sample,
    a normal (when noise_sigma > 0) and then a uniform (when straggle_rate > 0)."""
    sigma = float(model.noise_sigma)
    rate = float(model.straggle_rate)
    if sigma <= 0.0 and rate <= 0.0:
        return None, None
    if rate <= 0.0:  # normals only: one vectorised draw is the same stream
        z = rng.normal(0.0, sigma, size=n * samples)
        return np.fromiter(map(math.exp, z.tolist()), dtype=np.float64, count=n * samples), None
    noise = np.ones(n * samples) if sigma > 0.0 else None
    strag = np.ones(n * samples)
    factor = float(model.straggle_factor)
    for j in range(n * samples):
        if sigma > 0.0:
            noise[j] = math.exp(rng.normal(0.0, sigma))
        if rng.random() < rate:
            strag[j] = factor
    return noise, strag


def profile_latencies(op, scenario, samples: int, *, ctx=None):
    """The profiled latency of every assignment of ``op``'s template, in enumeration order, from
    the device kernel; also returns (kind index, resource, batch) per assignment."""
    ctx = ctx or get_context()
    tpl = op.knob_template
    kinds = sorted(tpl.hardware_targets)
    model = scenario.ground_truth
    truths = [model.kind_truth(op.name, k) for k in kinds]
    batches = np.ascontiguousarray(sorted(int(b) for b in tpl.batch_sizes), dtype=np.int32)
    n_res = np.array([len(tpl.resource_options[k]) for k in kinds], dtype=np.int32)
    res_opts = np.ascontiguousarray([int(r) for k in kinds for r in tpl.resource_options[k]],
                                    dtype=np.int32)
    knobs = list(tpl.knobs)
    counts = np.array([len(k.values) for k in knobs], dtype=np.int32)
    mult = np.ones((len(kinds), int(counts.sum()) if knobs else 1), dtype=np.float64)
    for ki, tr in enumerate(truths):
        col = 0
        for kn in knobs:
            table = tr.knob_multipliers.get(kn.name)
            for v in kn.values:
                if table:
                    mult[ki, col] = table.get(str(v), 1.0)
                col += 1
    f64 = lambda xs: np.ascontiguousarray(xs, dtype=np.float64)
    n = int(sum(int(r) * len(batches) * int(np.prod(counts)) for r in n_res))
    samples = max(1, int(samples))
    seed_material = content_hash([scenario.seed, op.executable_id])
    rng = np.random.default_rng(int(seed_material[:16], 16))
    noise, strag = _rng_factors(model, n, samples, rng)
    lat = np.empty(n, np.float64)
    kind = np.empty(n, np.int32)
    res = np.empty(n, np.int32)
    bat = np.empty(n, np.int32)
    # (every buffer bound to a name: ptr() hands out raw addresses)
    base = f64([t.base_seconds for t in truths])
    refr = np.ascontiguousarray([int(t.ref_resource) for t in truths], dtype=np.int32)
    rexp = f64([t.resource_exponent for t in truths])
    bexp = f64([t.batch_exponent for t in truths])
    pitem = f64([t.per_item_seconds for t in truths])
    check(ctx.lib.sp_profile_configs(
        ctx.handle, len(kinds), ptr(n_res), ptr(res_opts), ptr(base), ptr(refr), ptr(rexp),
        ptr(bexp), ptr(pitem), len(batches), ptr(batches), len(knobs),
        ptr(counts) if knobs else None, ptr(mult) if knobs else None, samples, ptr(noise),
        ptr(strag), n, ptr(lat), ptr(kind), ptr(res), ptr(bat)), "sp_profile_configs")
    return lat, kinds, kind, res, bat


def profile_operation(op, scenario, samples_per_config: int = DEFAULT_SAMPLES) -> ConfigSpec:
    """profiler.py:35-85 with the per-assignment latency law on the device."""
    for kind in op.knob_template.hardware_targets:
        try:
            scenario.backend(kind)
        except KeyError:
            raise ValueError(
                f"operation {op.name!r} targets backend kind {kind!r}, "
                f"which the scenario does not provide"
            ) from None
    assignments = enumerate_configs(op.knob_template)
    lat, kinds, kidx, res, bat = profile_latencies(op, scenario, samples_per_config)
    model = scenario.ground_truth
    entries = []
    for j, a in enumerate(assignments):
        latency = float(lat[j])
        backend = scenario.backend(a.backend_kind)
        entries.append(ConfigEntry(
            config_id=a.config_id(),
            backend_kind=a.backend_kind,
            knob_values=dict(a.knob_values),
            batch_size=a.batch_size,
            resource_request=a.resource_request,
            latency_s=latency,
            latency_initial_s=latency,
            peak_memory_mb=model.peak_memory_per_item_mb * a.batch_size,
            schedulable=a.resource_request <= backend.resources_per_instance,
        ))
    draft = ConfigSpec(operation=op.name, entries=entries, reference_id=entries[0].config_id)
    draft.reference_id = reference_config(draft).config_id
    return draft


def pow_correctly_rounded(x, y, *, ctx=None) -> np.ndarray:
    """x ** y correctly rounded, evaluated on the device (the power of the profile law)."""
    ctx = ctx or get_context()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(np.broadcast_to(y, x.shape), dtype=np.float64)
    out = np.empty_like(x)
    check(ctx.lib.sp_pow_correctly_rounded(ctx.handle, int(x.size), ptr(x), ptr(y), ptr(out)),
          "sp_pow_correctly_rounded")
    return out
