"""Synthetic workloads of BASELINE.json's configs, seeded and deterministic.

Tables are produced exactly as the reference profiler would at zero noise with one sample
(profiler.py:35-85 -> backend.py:36-58 -> scenario.py:68-77), so the golden script can pin
them against the reference's own ``profile_operation``.  Invocation streams follow the
distributions written in SURVEY.md §8(d).  Nothing here is on the hot path; it only makes
inputs.
"""
from __future__ import annotations

import itertools
import math
import random
from dataclasses import dataclass

import numpy as np

from .pipeline import ConfigEntry, ConfigSpec, PipelineDag, config_id_of, reference_config
from .scenario import BackendSpec, Scenario

BATCHES = (1, 2, 4, 8, 16, 32, 64, 128)
CPU_RES = tuple(range(1, 33))
GPU_RES = tuple(range(512, 16385, 512))
SAMPLING = (1, 2, 4, 8)
VARIANT = ("a", "b")
MODEL = ("a", "b", "c", "d")
MODEL_MULT = {"a": 1.0, "b": 1.2, "c": 1.5, "d": 2.0}

KINDS = ("cpu", "gpu")


def synth_scenario() -> Scenario:
    """cpu 10 x 64 cores at 1.32e-5 $/core-s; gpu 2 x 16,384 MB at 9e-4/16,384 $/MB-s."""
    return Scenario(
        name="synth",
        backends=(BackendSpec("cpu", 10, 64, 1.32e-5), BackendSpec("gpu", 2, 16384, 9e-4 / 16384)),
    )


@dataclass(frozen=True)
class Truth:
    """OpKindTruth (scenario.py:46-77) restricted to what the synthetic tables use."""

    base_seconds: float
    ref_resource: int
    resource_exponent: float
    batch_exponent: float
    knob_multipliers: dict

    def base_latency(self, resource: int, batch: int, knobs) -> float:
        lat = self.base_seconds
        if self.resource_exponent:
            lat *= (resource / self.ref_resource) ** -self.resource_exponent
        lat *= batch ** self.batch_exponent
        for knob, value in knobs:
            table = self.knob_multipliers.get(knob)
            if table:
                lat *= table.get(str(value), 1.0)
        return lat


def synth_truths(with_model: bool) -> dict[str, Truth]:
    mult = {"sampling": {str(s): 1.0 / s ** 0.5 for s in SAMPLING}, "variant": {"a": 1.0, "b": 1.0}}
    if with_model:
        mult["model"] = {k: v for k, v in MODEL_MULT.items()}
    return {
        "cpu": Truth(2.0, 1, 0.6, 0.85, mult),
        "gpu": Truth(0.12, 4096, 0.3, 0.35, mult),
    }


def synth_spec(with_model: bool = False, operation: str = "op") -> ConfigSpec:
    """Config 2 (4,096 entries) or config 5 (16,384 entries with the `model` knob).

    Enumeration order follows enumerate_configs (pipeline.py:454-475): kinds sorted, then
    resource and batch ascending, then the knob cross product in template order."""
    knobs = [("sampling", SAMPLING), ("variant", VARIANT)]
    if with_model:
        knobs.append(("model", MODEL))
    truths = synth_truths(with_model)
    sc = synth_scenario()
    entries = []
    for kind in sorted(KINDS):
        res_opts = CPU_RES if kind == "cpu" else GPU_RES
        for r in res_opts:
            for b in BATCHES:
                for combo in itertools.product(*[v for _, v in knobs]):
                    kv = tuple(zip([k for k, _ in knobs], combo))
                    lat = truths[kind].base_latency(r, b, kv)
                    # profiler.py:64-68: one noise-free sample, mean of one value
                    lat = float(sum([lat + 0.0 * b]) / 1)
                    entries.append(ConfigEntry(
                        config_id=config_id_of(kind, r, b, kv), backend_kind=kind,
                        knob_values=dict(kv), batch_size=b, resource_request=r,
                        latency_s=lat, latency_initial_s=lat,
                        schedulable=r <= sc.backend(kind).resources_per_instance,
                    ))
    draft = ConfigSpec(operation=operation, entries=entries, reference_id=entries[0].config_id)
    draft.reference_id = reference_config(draft).config_id
    return draft


@dataclass
class Invocations:
    slack: np.ndarray      # (N, K) float64
    avail: np.ndarray      # (N,) int32
    supply: np.ndarray     # (N,) int32
    min_batch: np.ndarray  # (N,) int32
    flags: np.ndarray      # (N,) uint32  (bit0 allow_delay, bits 8.. excluded mask)
    op: np.ndarray | None = None

    @property
    def N(self) -> int:
        return int(self.slack.shape[0])

    def take(self, sl: slice) -> "Invocations":
        return Invocations(self.slack[sl], self.avail[sl], self.supply[sl], self.min_batch[sl],
                           self.flags[sl], None if self.op is None else self.op[sl])

    def nbytes(self) -> int:
        n = self.slack.nbytes + self.avail.nbytes + self.supply.nbytes + self.min_batch.nbytes + self.flags.nbytes
        return n + (0 if self.op is None else self.op.nbytes)


def synth_invocations(N: int, lat: np.ndarray, gkind: np.ndarray, seed: int = 20261017,
                      K: int = 2, max_avail: int = 128) -> Invocations:
    """slack_k ~ U(-2, 10) with 5% +inf and 2% set exactly to a
    random same-kind entry's latency (boundary => penalized); avail U{1..128}; supply
    U{0..256}; allow_delay Bern(0.5); exclude cpu 10%, gpu 10%, both 1% (-> None);
    min_batch 1 w.p. 0.8 else U{2, 4, ..., 128}."""
    rng = np.random.default_rng(seed)
    slack = rng.uniform(-2.0, 10.0, size=(N, K))
    u = rng.random((N, K))
    slack[u < 0.05] = np.inf
    eq = (u >= 0.05) & (u < 0.07)
    for k in range(K):
        pool = lat[gkind == k]
        rows = np.flatnonzero(eq[:, k])
        if len(pool) and len(rows):
            slack[rows, k] = pool[rng.integers(0, len(pool), size=len(rows))]
    avail = rng.integers(1, max_avail + 1, size=N).astype(np.int32)
    supply = rng.integers(0, 257, size=N).astype(np.int32)
    allow = (rng.random(N) < 0.5).astype(np.uint32)
    e = rng.random(N)
    excl = np.zeros(N, dtype=np.uint32)
    excl[e < 0.01] = 0b11
    excl[(e >= 0.01) & (e < 0.11)] = 0b01
    excl[(e >= 0.11) & (e < 0.21)] = 0b10
    mb = np.ones(N, dtype=np.int32)
    big = rng.random(N) >= 0.8
    mb[big] = (2 * rng.integers(1, max_avail // 2 + 1, size=int(big.sum()))).astype(np.int32)
    flags = allow | (excl << np.uint32(8))
    return Invocations(np.ascontiguousarray(slack), avail, supply, mb, flags.astype(np.uint32))


# ---- config 3: deep DAG -------------------------------------------------------------------

def deep_dag(n_ops: int = 64, max_fanout: int = 32, seed: int = 1) -> PipelineDag:
    """Ops v00..v63 in topological index order; for i < n-1, out-degree U{1..min(32, n-1-i)}
    with targets sampled from (i, n-1] (random.Random(seed))."""
    r = random.Random(seed)
    names = [f"v{i:02d}" for i in range(n_ops)]
    edges = []
    for i in range(n_ops - 1):
        deg = r.randint(1, min(max_fanout, n_ops - 1 - i))
        for j in sorted(r.sample(range(i + 1, n_ops), deg)):
            edges.append((names[i], names[j]))
    return PipelineDag(vertices=tuple(names), edges=tuple(edges))


def critical_path(dag: PipelineDag, ref: dict) -> float:
    order = dag.topological_order()
    best = {}
    for v in order:
        ps = dag.predecessors(v)
        best[v] = (max(best[p] for p in ps) if ps else 0.0) + ref[v]
    return max(best[v] for v in dag.output_vertices())


def deep_dag_instances(dag: PipelineDag, I: int, seed: int = 3, K: int = 4):
    """ref0 log-uniform(1e-3, 10); per instance ref = ref0*exp(N(0,0.3)),
    T ~ U(0.5, 10)*CP_ref, now ~ U(0, T), Q_k ~ Exp(0.05 T)."""
    rng = np.random.default_rng(seed)
    V = len(dag.vertices)
    ref0 = np.exp(rng.uniform(math.log(1e-3), math.log(10.0), size=V))
    cp = critical_path(dag, dict(zip(dag.vertices, ref0)))
    ref = ref0[None, :] * np.exp(rng.normal(0.0, 0.3, size=(I, V)))
    T = rng.uniform(0.5, 10.0, size=I) * cp
    now = rng.uniform(0.0, 1.0, size=I) * T
    Q = rng.exponential(1.0, size=(I, K)) * (0.05 * T)[:, None]
    return np.ascontiguousarray(ref), T, now, np.ascontiguousarray(Q)


# ---- config 4: latency-target sweep x replicas on the AMBER pipeline -----------------------

SWEEP_MULTS = (0.5, 1.0, 2.0, 5.0, 10.0)
SWEEP_SNAPSHOTS = 64
SWEEP_CP_MIN = 90.41885182994682  # fast-anchor latency of the AMBER run


@dataclass
class SweepInputs:
    """Instance-major inputs of config 4: instance i = ((r - r0) * 5 + m) * 64 + j."""
    ref: np.ndarray      # (I, V) reference latencies by operation (meta["ops"] order)
    target: np.ndarray   # (I,)
    now: np.ndarray      # (I,)
    Q: np.ndarray        # (I, K)
    avail: np.ndarray    # (I, V) int32
    supply: np.ndarray   # (I, V) int32


def amber_sweep(ref0: np.ndarray, K: int, r0: int, r1: int, mults=SWEEP_MULTS,
                snapshots: int = SWEEP_SNAPSHOTS, cp_min: float = SWEEP_CP_MIN) -> SweepInputs:
    """SURVEY.md §8(d) config 4 for replicas [r0, r1): target T = m * CP_min; snapshot j at
    now = j/64 * T; per (replica r, target index m) one generator seeded r*5 + m draws, in this
    order, Q (64 x K) ~ Exp(0.02 T), the reference-latency drift (64 x V) exp(N(0, 0.2)), avail
    (64 x V) U{1..64} and upstream supply (64 x V) U{0..64}.  Seeds depend on the global replica
    index, so any split of [0, R) over ranks reproduces the same global workload."""
    V = len(ref0)
    S, nm = snapshots, len(mults)
    n = (r1 - r0) * nm
    ref = np.empty((n, S, V))
    Q = np.empty((n, S, K))
    avail = np.empty((n, S, V), np.int32)
    supply = np.empty((n, S, V), np.int32)
    target = np.repeat(np.array([m * cp_min for m in mults] * (r1 - r0)), S)
    frac = np.arange(S) / S
    for u in range(n):
        r, m = r0 + u // nm, u % nm
        rng = np.random.default_rng(r * 5 + m)
        T = mults[m] * cp_min
        Q[u] = rng.exponential(0.02 * T, size=(S, K))
        ref[u] = ref0[None, :] * np.exp(rng.normal(0.0, 0.2, size=(S, V)))
        avail[u] = rng.integers(1, 65, size=(S, V))
        supply[u] = rng.integers(0, 65, size=(S, V))
    now = np.tile(frac, n) * target
    I = n * S
    return SweepInputs(ref.reshape(I, V), target, now, Q.reshape(I, K), avail.reshape(I, V),
                       supply.reshape(I, V))
