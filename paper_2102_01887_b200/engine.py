"""Replica-parallel run engine: the reference's tuned pipeline run on the device (SURVEY.md §8(f)
rank 4).

The reference executes one run at a time, single-threaded: ``PipelineRun.run_to_completion``
(manager.py:535-575) pops events from ``BackendSim`` (backend.py:125-269) and, after each, lets
the ``Configurator`` speculate, commit and fold feedback (configurator.py:368-772).  Here the whole
loop is one CUDA thread per replica (``k_des_run``, csrc/sp_des.cuh): replicas share the run
description built below (``RunSpec``: the tables ``PipelineRun.__init__`` builds, the DAG, the fleet,
the tuning parameters) and differ in trace, target and seed.  Every decision-log row, the report
and the final latency tables equal the reference's own run bit for bit (tests/test_engine*.py).

Host work here is setup only — the OpTable filter (configurator.py:166-209), profile scaling
(manager.py:187-208), the ground-truth base latency of every entry (scenario.py:68-77), and the
reference RNG stream of noisy scenarios (backend.py:52-57, 186: the per-start draws of the
replica's numpy Generator, in the reference's order).  There is no CPU fallback: without
libslackpipe_b200.so and a B200 every call raises.

``PipelineRun`` mirrors the reference class (same constructor, ``run_to_completion`` ->
``RunReport`` with the same CSV row, ``write_decision_log``); ``ReplicaEngine.run`` runs many
replicas of one ``RunSpec`` in one launch.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from statistics import mean, median
from typing import Any, Iterable, Mapping, Sequence

import numpy as np

from . import _lib
from .pipeline import content_hash, reference_config

ABLATION_TOKENS = ("fb", "dfp", "sdb", "eslc", "pbc")  # configurator.py:23
_ABL_BIT = {"fb": 1, "dfp": 2, "sdb": 4, "eslc": 8, "pbc": 16}
_CMP = {"<": 0, "<=": 1, ">": 2, ">=": 3, "==": 4, "!=": 5}
DRAW_NOISE, DRAW_STRAGGLE, DRAW_FAIL = 1, 2, 4

STATUS = {0: "ok", 1: "invocation capacity", 2: "event heap capacity", 3: "item-list capacity",
          4: "livelock", 5: "no configuration", 6: "non-finite score", 7: "draw capacity",
          8: "weight capacity", 9: "item-buffer capacity", 10: "event cap", 11: "no ground truth"}
_CAPACITY = (1, 2, 3, 7, 9)

OUT_DTYPE = np.dtype([("latency", "<f8"), ("cost", "<f8"), ("now", "<f8"),
                      ("peak_slots", "<i4"), ("peak_heap", "<i4"),
                      ("status", "<i4"), ("met", "<i4"), ("completed", "<i4"),
                      ("failures", "<i4"), ("duplicates", "<i4"), ("invocations", "<i4"),
                      ("terminal_items", "<i4"), ("n_speculate", "<i4"), ("n_commit", "<i4"),
                      ("configs_used", "<i4"), ("log_len", "<i4"), ("events", "<i4"),
                      ("event_len", "<i4"), ("pad", "<i4")])
LOG_DTYPE = np.dtype([("t", "<f8"), ("slack", "<f8"), ("obj", "<f8"), ("iid", "<i4"),
                      ("meta", "<i4")])
EVENT_DTYPE = np.dtype([("t", "<f8"), ("iid", "<i4"), ("meta", "<i4")])
_EVENT_KIND = ("start", "complete", "fail")


class _Spec(C.Structure):  # sp_des_spec (include/slackpipe_b200.h)
    _fields_ = ([(n, C.c_int32) for n in ("n_ops", "n_kinds", "n_entries", "n_attrs", "n_cfg_ids")]
                + [(n, C.c_void_p) for n in (
                    "entry_off", "lat", "lat_init", "res", "batch", "kind", "id_rank", "cfg_id",
                    "truth_base", "truth_per_item", "ref_index", "ref_latency", "succ_off", "succ",
                    "pred_attr", "pred_cmp", "pred_value", "fanout_attr", "suffix_off", "suffix_ops",
                    "instances", "inst_resources", "price", "cq_capacity")]
                + [(n, C.c_double) for n in ("alpha", "beta", "timeout_factor", "dispatch_overhead",
                                             "straggle_factor")]
                + [(n, C.c_int32) for n in ("dfp_count", "ablations", "draws")])


@dataclass(frozen=True)
class TuningParams:
    """Engine knobs (configurator.py:26-46)."""

    alpha: float = 100.0
    cq_capacity: int | None = None
    dfp_count: int = 10
    straggler_timeout_factor: float = 1.5
    smoothing_beta: float = 0.5

    def __post_init__(self) -> None:
        if self.alpha < 0:
            raise ValueError("alpha must be >= 0")
        if self.cq_capacity is not None and self.cq_capacity < 1:
            raise ValueError("cq_capacity must be >= 1")
        if self.dfp_count < 0:
            raise ValueError("dfp_count must be >= 0")
        if self.straggler_timeout_factor <= 0:
            raise ValueError("straggler_timeout_factor must be positive")
        if not (0.0 < self.smoothing_beta <= 1.0):
            raise ValueError("smoothing_beta must be in (0, 1]")


def _base_latency(truth, res: int, batch: int, knobs: Mapping[str, Any]) -> float:
    """OpKindTruth.base_latency (scenario.py:68-77) on the entry's assignment (backend.py:27-33)."""
    lat = truth.base_seconds
    if truth.resource_exponent:
        lat *= (res / truth.ref_resource) ** -truth.resource_exponent
    lat *= batch ** truth.batch_exponent
    for knob, value in sorted(knobs.items()):
        tab = truth.knob_multipliers.get(knob)
        if tab:
            lat *= tab.get(str(value), 1.0)
    return lat


def _paths(dag) -> list[tuple[str, ...]]:
    """All input -> output simple paths (pipeline.py:428-451)."""
    out: list[tuple[str, ...]] = []

    def walk(v, prefix):
        succ = dag.successors(v)
        if not succ:
            out.append(prefix)
            return
        for d in succ:
            walk(d, prefix + (d,))

    for v in dag.input_vertices():
        walk(v, (v,))
    return out


def _ancestors(dag, v) -> set:
    seen, stack = set(), list(dag.predecessors(v))
    while stack:
        u = stack.pop()
        if u not in seen:
            seen.add(u)
            stack.extend(dag.predecessors(u))
    return seen


class RunSpec:
    """Everything ``PipelineRun.__init__`` derives that all replicas share (manager.py:210-300)."""

    def __init__(self, dag, profiles: Mapping[str, Any], scenario, params: TuningParams | None = None,
                 *, ablations: Iterable[str] = (), paths=None, profile_scale: float = 1.0,
                 noise_sigma: float | None = None, failure_rate: float | None = None,
                 straggle_rate: float | None = None, straggle_factor: float | None = None):
        params = params or TuningParams()
        abl = frozenset(ablations)
        unknown = abl - set(ABLATION_TOKENS)
        if unknown:
            raise ValueError(f"unknown ablation tokens: {sorted(unknown)}")
        if profile_scale <= 0:
            raise ValueError("profile_scale must be positive")
        for v in dag.vertices:
            if v not in profiles:
                raise ValueError(f"operation {v!r} has not been profiled")
        self._check_joins(dag)
        self.dag, self.params, self.ablations = dag, params, abl
        self.scenario = scenario
        gt = scenario.ground_truth
        self.noise_sigma = gt.noise_sigma if noise_sigma is None else float(noise_sigma)
        self.failure_rate = gt.failure_rate if failure_rate is None else float(failure_rate)
        self.straggle_rate = gt.straggle_rate if straggle_rate is None else float(straggle_rate)
        self.straggle_factor = gt.straggle_factor if straggle_factor is None else float(straggle_factor)
        self.ops = sorted(dag.vertices)
        opix = {v: i for i, v in enumerate(self.ops)}
        self.kinds = list(scenario.backend_kinds())
        kpos = {k: i for i, k in enumerate(self.kinds)}
        present = set(self.kinds)

        # tables (configurator.py:166-209) over scaled profile copies (manager.py:187-208)
        cfg_names: dict[str, int] = {}
        cols = {n: [] for n in ("lat", "lat_init", "res", "batch", "kind", "id_rank", "cfg",
                                "base", "per_item")}
        self.entry_off = [0]
        self.entries: list[list] = []
        ref_index, ref_lat = [], []
        for op in self.ops:
            spec = profiles[op]
            ents = [e for e in spec.entries if e.schedulable and e.backend_kind in present
                    and e.resource_request <= scenario.backend(e.backend_kind).resources_per_instance]
            if not ents:
                raise ValueError(f"operation {op!r} has no schedulable configuration")
            order = sorted(range(len(ents)), key=lambda i: ents[i].config_id)
            rank = [0] * len(ents)
            for r, i in enumerate(order):
                rank[i] = r
            ref = reference_config(spec)
            ids = [e.config_id for e in ents]
            ri = ids.index(ref.config_id) if ref.config_id in ids else -1
            ref_index.append(ri)
            ref_lat.append(ents[ri].latency_s * profile_scale if ri >= 0 else ref.latency_s * profile_scale)
            for i, e in enumerate(ents):
                try:
                    truth = gt.kind_truth(op, e.backend_kind)
                except KeyError:  # raised by the run only if it starts such an entry (NaN marker)
                    truth = None
                cols["lat"].append(e.latency_s * profile_scale)
                cols["lat_init"].append(e.latency_initial_s * profile_scale)
                cols["res"].append(float(e.resource_request))
                cols["batch"].append(int(e.batch_size))
                cols["kind"].append(kpos[e.backend_kind])
                cols["id_rank"].append(rank[i])
                cols["cfg"].append(cfg_names.setdefault(e.config_id, len(cfg_names)))
                cols["base"].append(math.nan if truth is None else
                                    _base_latency(truth, e.resource_request, e.batch_size,
                                                  dict(e.knob_values)))
                cols["per_item"].append(math.nan if truth is None else float(truth.per_item_seconds))
            self.entries.append(ents)
            self.entry_off.append(self.entry_off[-1] + len(ents))
        self.cfg_names = list(cfg_names)
        f64 = lambda x: np.ascontiguousarray(x, dtype=np.float64)
        i32 = lambda x: np.ascontiguousarray(x, dtype=np.int32)
        self.arr = {
            "entry_off": i32(self.entry_off), "lat": f64(cols["lat"]), "lat_init": f64(cols["lat_init"]),
            "res": f64(cols["res"]), "batch": i32(cols["batch"]), "kind": i32(cols["kind"]),
            "id_rank": i32(cols["id_rank"]), "cfg_id": i32(cols["cfg"]),
            "truth_base": f64(cols["base"]), "truth_per_item": f64(cols["per_item"]),
            "ref_index": i32(ref_index), "ref_latency": f64(ref_lat),
        }
        # DAG: sorted successors, predicates, fan-outs (pipeline.py:283-326)
        preds = dict(getattr(dag, "branch_predicates", {}) or {})
        fan = dict(getattr(dag, "fanout_rules", {}) or {})
        self.attr_names = sorted({p.attr for p in preds.values()} | set(fan.values()))
        apos = {a: i for i, a in enumerate(self.attr_names)}
        succ_off, succ, pa, pc, pv = [0], [], [], [], []
        for op in self.ops:
            for d in sorted(dag.successors(op), key=lambda x: opix[x]):
                p = preds.get((op, d))
                succ.append(opix[d])
                pa.append(apos[p.attr] if p is not None else -1)
                pc.append(_CMP[p.op] if p is not None else 0)
                pv.append(int(p.value) if p is not None else 0)
            succ_off.append(len(succ))
        self.has_join = any(len(dag.predecessors(v)) > 1 for v in dag.vertices)
        paths = list(paths) if paths is not None else _paths(dag)
        suf_off, suf = [0], []
        for op in self.ops:
            for p in paths:
                if op in p:
                    s = p[p.index(op):]
                    suf.append(len(s))
                    suf.extend(opix[o] for o in s)
            if suf_off[-1] == len(suf):
                raise ValueError(f"operation {op!r} does not appear on any path")
            suf_off.append(len(suf))
        # fleet and commit-queue capacity (configurator.py:443-458)
        K = len(self.kinds)
        if params.cq_capacity is not None:
            cap = [params.cq_capacity] * K
        else:
            cap = []
            kinds_arr = self.arr["kind"]
            for k in range(K):
                on = kinds_arr == k
                cap.append(max(1, int(float(scenario.backend(self.kinds[k]).pool_resources)
                                      // int(self.arr["res"][on].min()))) if on.any() else 1)
        self.arr.update({
            "succ_off": i32(succ_off), "succ": i32(succ or [0]), "pred_attr": i32(pa or [0]),
            "pred_cmp": i32(pc or [0]), "pred_value": i32(pv or [0]),
            "fanout_attr": i32([apos[fan[o]] if o in fan else -1 for o in self.ops]),
            "suffix_off": i32(suf_off), "suffix_ops": i32(suf),
            "instances": i32([b.instance_count for b in scenario.backends]),
            "inst_resources": i32([b.resources_per_instance for b in scenario.backends]),
            "price": f64([b.price_rate for b in scenario.backends]),
            "cq_capacity": i32(cap),
        })
        self.draws = ((DRAW_NOISE if self.noise_sigma > 0.0 else 0)
                      | (DRAW_STRAGGLE if self.straggle_rate > 0.0 else 0)
                      | (DRAW_FAIL if self.failure_rate > 0.0 else 0))
        self.ablation_bits = sum(_ABL_BIT[a] for a in abl)
        self._fan_attr = [apos[fan[o]] if o in fan else -1 for o in self.ops]

    @staticmethod
    def _check_joins(dag) -> None:  # manager.py:292-299
        preds = getattr(dag, "branch_predicates", {}) or {}
        for v in dag.vertices:
            ps = dag.predecessors(v)
            if len(ps) <= 1:
                continue
            if v in (getattr(dag, "fanout_rules", {}) or {}):
                raise ValueError(f"join vertex {v!r} cannot carry a fan-out rule")
            for p in ps:
                if (p, v) in preds:
                    raise ValueError(f"edge ({p}, {v}) into join vertex cannot carry a predicate")

    def c_spec(self) -> _Spec:
        a = self.arr
        s = _Spec()
        s.n_ops, s.n_kinds = len(self.ops), len(self.kinds)
        s.n_entries, s.n_attrs, s.n_cfg_ids = int(self.entry_off[-1]), len(self.attr_names), len(self.cfg_names)
        for n in ("entry_off", "lat", "lat_init", "res", "batch", "kind", "id_rank", "cfg_id",
                  "truth_base", "truth_per_item", "ref_index", "ref_latency", "succ_off", "succ",
                  "pred_attr", "pred_cmp", "pred_value", "fanout_attr", "suffix_off", "suffix_ops",
                  "instances", "inst_resources", "price", "cq_capacity"):
            setattr(s, n, a[n].ctypes.data)
        p = self.params
        s.alpha, s.beta = float(p.alpha), float(p.smoothing_beta)
        s.timeout_factor = float(p.straggler_timeout_factor)
        s.dispatch_overhead = float(getattr(self.scenario, "dispatch_overhead_s", 0.0))
        s.straggle_factor = float(self.straggle_factor)
        s.dfp_count, s.ablations, s.draws = int(p.dfp_count), self.ablation_bits, self.draws
        return s

    # ---- per-replica inputs ------------------------------------------------------------------
    def encode_frames(self, traces: Sequence[Sequence[tuple[int, Mapping[str, int]]]]):
        """(frame_off[R+1], attrs[F, n_attrs]) with 0 where a frame lacks an attribute
        (BranchPredicate.evaluate / fan-out `attrs.get(attr, 0)`, pipeline.py:294-295,
        manager.py:405)."""
        off = [0]
        rows = []
        A = len(self.attr_names)
        for frames in traces:
            ids = set()
            for fid, attrs in frames:
                for k, v in attrs.items():
                    if not isinstance(v, (int, np.integer)) or isinstance(v, bool) or v < 0:
                        raise ValueError(f"frame {fid}: attribute {k!r} must be a non-negative int")
                if self.has_join:
                    if fid in ids:
                        raise ValueError("the run engine stages join items by frame; frame ids must be unique")
                    ids.add(fid)
                rows.append([int(attrs.get(a, 0)) for a in self.attr_names])
            off.append(off[-1] + len(frames))
        attrs = np.zeros((off[-1], max(A, 1)), dtype=np.int32)
        if A and rows:
            attrs[:, :A] = np.asarray(rows, dtype=np.int32).reshape(-1, A)
        return np.asarray(off, dtype=np.int32), np.ascontiguousarray(attrs[:, :A] if A else attrs[:, :0])

    def item_bound(self, frame_off: np.ndarray, attrs: np.ndarray) -> int:
        """Largest number of items any replica's trace can push through all buffers (the same
        bound sp_des_prepare sizes its arenas with)."""
        order = self.dag.topological_order() if hasattr(self.dag, "topological_order") else None
        if order is None:
            from .pipeline import PipelineDag
            order = PipelineDag(tuple(self.dag.vertices), tuple(self.dag.edges)).topological_order()
        opix = {v: i for i, v in enumerate(self.ops)}
        a = self.arr
        F = int(frame_off[-1])
        mult = np.zeros((len(self.ops), F), dtype=np.int64)
        for v in order:
            i = opix[v]
            if not self.dag.predecessors(v):
                mult[i] = 1
            for q in range(a["succ_off"][i], a["succ_off"][i + 1]):
                d = int(a["succ"][q])
                m = mult[i].copy()
                if a["pred_attr"][q] >= 0:
                    x = attrs[:, a["pred_attr"][q]]
                    ok = {0: x < a["pred_value"][q], 1: x <= a["pred_value"][q], 2: x > a["pred_value"][q],
                          3: x >= a["pred_value"][q], 4: x == a["pred_value"][q],
                          5: x != a["pred_value"][q]}[int(a["pred_cmp"][q])]
                    m = np.where(ok, m, 0)
                if self._fan_attr[d] >= 0:
                    m = m * np.maximum(attrs[:, self._fan_attr[d]], 0)
                mult[d] += m
        per = np.add.reduceat(mult, frame_off[:-1], axis=1) if F else np.zeros((len(self.ops), 0))
        per = per[:, np.diff(frame_off) > 0] if F else per
        return int(per.sum(axis=0).max()) if per.size else 0

    def draws_for(self, seeds: Sequence[int], cap: int):
        """The reference's per-start RNG draws (backend.py:52-57, 186) of each replica's numpy
        Generator, in stream order: exp(N(0, sigma)) (CPython's math.exp), then the straggle and
        failure Bernoulli draws — generated by sp_des_draws (PCG64 + numpy's ziggurat in C, host
        threads)."""
        R = len(seeds)
        fac = np.ones((R, cap), dtype=np.float64) if self.draws & DRAW_NOISE else None
        bits = np.zeros((R, cap), dtype=np.uint8) if self.draws & (DRAW_STRAGGLE | DRAW_FAIL) else None
        st = np.empty((R, 4), dtype=np.uint64)
        m64 = (1 << 64) - 1
        for r, seed in enumerate(seeds):
            s = np.random.default_rng(seed).bit_generator.state["state"]
            st[r] = (s["state"] >> 64, s["state"] & m64, s["inc"] >> 64, s["inc"] & m64)
        lib = _lib.load_library()
        ptr = lambda x: x.ctypes.data if x is not None else None
        _lib.check(lib.sp_des_draws(R, st.ctypes.data, int(cap), float(self.noise_sigma),
                                    float(self.straggle_rate), float(self.failure_rate), ptr(fac),
                                    ptr(bits)), "sp_des_draws")
        return fac, bits


@dataclass
class RunResult:
    latency_s: float
    cost: float
    met: int
    completed: int
    failures: int
    duplicates: int
    invocations: int
    terminal_items: int
    decision_count: int
    configs_used: int
    status: int
    log: np.ndarray | None = None
    lat: np.ndarray | None = None
    events: np.ndarray | None = None

    @property
    def slack_met_frac(self) -> float:
        return self.met / self.completed if self.completed else 1.0


class ReplicaEngine:
    """A RunSpec resident on one device; ``run`` executes R replicas in one launch."""

    def __init__(self, spec: RunSpec, ctx=None):
        self.spec = spec
        self.ctx = ctx or _lib.get_context()
        self.lib = self.ctx.lib
        h = C.c_void_p()
        cs = spec.c_spec()
        _lib.check(self.lib.sp_des_create(self.ctx.handle, C.byref(cs), C.byref(h)), "sp_des_create")
        self.handle = h
        self.cap_scale = 1.25

    def set_mode(self, mode: str) -> None:
        """"default" (32 lanes per replica below 2,048 replicas, 8 below 32,768, else 2),
        "warp" (32 lanes), "lanes16" / "lanes8" / "lanes4" / "lanes2", or "thread" (one thread per
        replica)."""
        m = {"default": 0, "thread": 1, "warp": 32, "lanes2": 2, "lanes4": 4, "lanes8": 8,
             "lanes16": 16}[mode]
        _lib.check(self.lib.sp_des_set_mode(self.handle, m), "sp_des_set_mode")

    def close(self) -> None:
        if self.handle:
            self.lib.sp_des_destroy(self.ctx.handle, self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, traces, targets, seeds=None, *, trace_of=None, log_cap: int = 0,
            final_tables: bool = False, encoded=None, event_cap: int = 0) -> list[RunResult]:
        """Run one replica per target: replica i runs trace ``trace_of[i]`` (default: trace i)
        of ``traces`` (or of ``encoded`` = encode_frames(traces)) with seed ``seeds[i]`` (default:
        the scenario seed, manager.py:240)."""
        spec = self.spec
        R = len(targets)
        frame_off, attrs = encoded if encoded is not None else spec.encode_frames(traces)
        T = len(frame_off) - 1
        trace_of = (np.arange(R, dtype=np.int32) if trace_of is None
                    else np.ascontiguousarray(trace_of, dtype=np.int32))
        if len(trace_of) != R or (R and (trace_of.min() < 0 or trace_of.max() >= T)):
            raise ValueError("trace_of must give every replica a trace")
        targets = np.ascontiguousarray(targets, dtype=np.float64)
        seeds = list(seeds) if seeds is not None else [spec.scenario.seed] * R
        results: list[RunResult | None] = [None] * R
        todo = np.arange(R)
        scale = self.cap_scale
        while len(todo):
            out, lg, lat, ev = self._launch(frame_off, attrs, np.ascontiguousarray(trace_of[todo]),
                                            targets[todo], [seeds[r] for r in todo], scale, log_cap,
                                            final_tables, event_cap)
            retry = []
            for j, r in enumerate(todo):
                st = int(out["status"][j])
                if st in _CAPACITY and scale < 64:
                    retry.append(r)
                    continue
                if st == 4:
                    raise RuntimeError("run stalled with work remaining")
                if st == 5:
                    raise RuntimeError("no configuration can re-run a retried or duplicated invocation")
                if st == 11:
                    raise KeyError("no ground truth for an operation / backend kind the run executes")
                if st != 0:
                    raise _lib.SlackpipeError(f"run engine replica {r}: {STATUS.get(st, st)}")
                o = out[j]
                results[r] = RunResult(
                    float(o["latency"]), float(o["cost"]), int(o["met"]), int(o["completed"]),
                    int(o["failures"]), int(o["duplicates"]), int(o["invocations"]),
                    int(o["terminal_items"]), int(o["n_speculate"]) + int(o["n_commit"]),
                    int(o["configs_used"]), st,
                    lg[j, :min(int(o["log_len"]), log_cap)].copy() if lg is not None else None,
                    lat[j].copy() if lat is not None else None,
                    ev[j, :min(int(o["event_len"]), event_cap)].copy() if ev is not None else None)
                if ev is not None and int(o["event_len"]) > event_cap:
                    raise ValueError(f"event trace of replica {r} has {int(o['event_len'])} rows > event_cap")
                if lg is not None and int(o["log_len"]) > log_cap:
                    raise ValueError(f"decision log of replica {r} has {int(o['log_len'])} rows > log_cap")
            todo = np.asarray(retry, dtype=np.int64)
            scale *= 2
        return results  # type: ignore[return-value]

    def _launch(self, frame_off, attrs, trace_of, targets, seeds, scale, log_cap, final_tables,
                event_cap=0):
        spec, lib, ctx = self.spec, self.lib, self.ctx
        R = len(targets)
        _lib.check(lib.sp_des_set_capacity(self.handle, float(scale)), "sp_des_set_capacity")
        draw_cap, fac, bits = 0, None, None
        if spec.draws:
            items = spec.item_bound(frame_off, attrs)
            draw_cap = int(items * scale) + 256
            fac, bits = spec.draws_for(seeds, draw_cap)
        out = np.zeros(R, dtype=OUT_DTYPE)
        lg = np.zeros((R, log_cap), dtype=LOG_DTYPE) if log_cap else None
        lat = np.zeros((R, int(spec.entry_off[-1])), dtype=np.float64) if final_tables else None
        ev = np.zeros((R, event_cap), dtype=EVENT_DTYPE) if event_cap else None
        ptr = lambda x: x.ctypes.data if x is not None else None
        _lib.check(lib.sp_des_run(ctx.handle, self.handle, R, len(frame_off) - 1, frame_off.ctypes.data,
                                  ptr(attrs), trace_of.ctypes.data, targets.ctypes.data, draw_cap,
                                  ptr(fac), ptr(bits), int(log_cap), ptr(lg), ptr(lat), out.ctypes.data,
                                  int(event_cap), ptr(ev), _lib.SP_MEM_HOST), "sp_des_run")
        return out, lg, lat, ev

    # ---- device-resident form (bench `value`): inputs already in HBM, stream-ordered, no sync
    def prepare(self, frame_off: np.ndarray, attrs: np.ndarray, R: int, *, scale: float | None = None) -> int:
        """Size the arenas for R replicas of these (host) traces; returns bytes per replica."""
        _lib.check(self.lib.sp_des_set_capacity(self.handle, float(scale or self.cap_scale)),
                   "sp_des_set_capacity")
        fo = np.ascontiguousarray(frame_off, dtype=np.int32)
        at = np.ascontiguousarray(attrs, dtype=np.int32)
        _lib.check(self.lib.sp_des_prepare(self.ctx.handle, self.handle, int(R), len(fo) - 1,
                                           fo.ctypes.data, at.ctypes.data, 0, 0), "sp_des_prepare")
        return int(self.lib.sp_des_arena_bytes(self.handle))

    def run_device(self, R: int, n_traces: int, frame_off_ptr: int, attrs_ptr: int, trace_of_ptr: int,
                   targets_ptr: int, out_ptr: int) -> None:
        """sp_des_run over device buffers (after ``prepare`` with the same traces); ``out_ptr``
        receives R OUT_DTYPE rows.  Noise-free scenarios only (no draw streams)."""
        if self.spec.draws:
            raise ValueError("run_device: scenarios with RNG draws take the host-buffer form")
        _lib.check(self.lib.sp_des_run(self.ctx.handle, self.handle, int(R), int(n_traces), frame_off_ptr,
                                       attrs_ptr, trace_of_ptr, targets_ptr, 0, None, None, 0, None,
                                       None, out_ptr, 0, None, _lib.SP_MEM_DEVICE), "sp_des_run")

    # ---- BackendSim.trace rows in the reference's tuple form (backend.py:207, 243)
    def event_rows(self, events: np.ndarray) -> list[tuple]:
        kinds = self.spec.kinds
        return [(float(ev["t"]), _EVENT_KIND[int(ev["meta"]) & 3], int(ev["iid"]),
                 kinds[(int(ev["meta"]) >> 2) & 63], int(ev["meta"]) >> 8) for ev in events]

    # ---- decision-log rows in the reference's tuple form (configurator.py:650-654, 746-749)
    def log_rows(self, log: np.ndarray) -> list[tuple]:
        spec = self.spec
        rows = []
        for rec in log:
            meta = int(rec["meta"])
            op = meta & 0xFF
            e = (meta >> 8) & 0x3FFFFF
            ent = spec.entries[op][e]
            rows.append((float(rec["t"]), "commit" if meta >> 30 & 1 else "speculate", int(rec["iid"]),
                         spec.ops[op], ent.backend_kind, ent.config_id, float(rec["slack"]),
                         float(rec["obj"])))
        return rows


class GroupReplicaEngine:
    """ReplicaEngine fanned out over a DeviceGroup from one host thread's call (SURVEY.md §8(b)
    Threading, §8(e)): the replicas are split into contiguous shards, one per member device, all in
    flight at once (a worker thread per member; the library call releases the GIL), results in
    replica order.  Replicas are independent: no collective."""

    def __init__(self, spec: RunSpec, group):
        self.spec = spec
        self.engines = [ReplicaEngine(spec, m) for m in group.members]

    def set_mode(self, mode: str) -> None:
        for e in self.engines:
            e.set_mode(mode)

    def close(self) -> None:
        for e in self.engines:
            e.close()

    def run(self, traces, targets, seeds=None, *, trace_of=None, log_cap: int = 0,
            final_tables: bool = False, encoded=None, event_cap: int = 0) -> list[RunResult]:
        import threading

        R = len(targets)
        fo, at = encoded if encoded is not None else self.spec.encode_frames(traces)
        trace_of = np.arange(R, dtype=np.int32) if trace_of is None else np.asarray(trace_of, np.int32)
        targets = np.asarray(targets, dtype=np.float64)
        seeds = list(seeds) if seeds is not None else [self.spec.scenario.seed] * R
        G = len(self.engines)
        bounds = [(g * R // G, (g + 1) * R // G) for g in range(G)]
        out: list = [None] * G
        err: list = []

        def work(g):
            a, b = bounds[g]
            try:
                out[g] = self.engines[g].run(None, targets[a:b], seeds[a:b], trace_of=trace_of[a:b],
                                             log_cap=log_cap, final_tables=final_tables,
                                             encoded=(fo, at), event_cap=event_cap) if b > a else []
            except BaseException as e:  # re-raised in the caller's thread
                err.append(e)

        th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if err:
            raise err[0]
        return [r for part in out for r in part]

    def log_rows(self, log):
        return self.engines[0].log_rows(log)

    def event_rows(self, events):
        return self.engines[0].event_rows(events)


@dataclass
class RunReport:
    """Aggregates of one pipeline run; the CSV schema is the reference's (manager.py:104-170)."""

    run_id: str
    scenario: str
    pipeline: str
    target_s: float
    latency_s: float
    normalized_latency: float
    cost: float
    slack_met_frac: float
    configs_used: int
    failures: int
    duplicates: int
    invocations: int
    completed: int
    terminal_items: int
    speculate_median_ms: float
    speculate_mean_ms: float
    commit_median_ms: float
    commit_mean_ms: float
    decision_count: int
    decisions_per_s: float
    wall_s: float
    flags: dict = field(default_factory=dict)

    CSV_COLUMNS = ("run_id", "target_s", "latency_s", "normalized_latency", "cost",
                   "slack_met_frac", "configs_used", "failures", "duplicates")

    def target_met(self) -> bool:
        return self.normalized_latency <= 1.0

    def csv_row(self) -> str:
        return ",".join([self.run_id, repr(float(self.target_s)), repr(float(self.latency_s)),
                         repr(float(self.normalized_latency)), repr(float(self.cost)),
                         repr(float(self.slack_met_frac)), str(self.configs_used),
                         str(self.failures), str(self.duplicates)])


def report_of(res: RunResult, *, target_s: float, scenario_name: str, pipeline_name: str, seed: int,
              ablations=(), flags: Mapping[str, Any] | None = None, wall_s: float = 0.0) -> RunReport:
    """manager.py:577-630 from one replica's result row."""
    lat = float(res.latency_s)
    if target_s > 0:
        norm = lat / target_s
    elif lat == 0.0:
        norm = 0.0
    else:
        norm = float("inf")
    flags = dict(flags or {})
    run_id = content_hash({"scenario": scenario_name, "pipeline": pipeline_name, "target": target_s,
                           "seed": seed, "ablations": sorted(ablations),
                           "flags": {k: str(v) for k, v in sorted(flags.items())}})[:12]
    per = wall_s / res.decision_count * 1e3 if res.decision_count else 0.0
    return RunReport(run_id, scenario_name, pipeline_name, target_s, lat, norm, res.cost,
                     res.slack_met_frac, res.configs_used, res.failures, res.duplicates,
                     res.invocations, res.completed, res.terminal_items, per, per, per, per,
                     res.decision_count, res.decision_count / wall_s if wall_s > 0 else 0.0,
                     wall_s, flags)


class _SimView:
    """The finished run's backend view: BackendSim.trace and write_trace (backend.py:264-269)."""

    def __init__(self, trace):
        self.trace = trace

    def write_trace(self, path: str) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("virtual_time\tevent_kind\tinvocation_id\tbackend\tinstance\n")
            for t, kind, inv, backend, instance in self.trace:
                fh.write(f"{t:.9f}\t{kind}\t{inv}\t{backend}\t{instance}\n")


class PipelineRun:
    """Drop-in for the reference's PipelineRun (manager.py:210-300): same constructor, the run
    executes on the device."""

    def __init__(self, dag, operations, profiles, frames, scenario, target_s: float,
                 params: TuningParams | None = None, *, ablations: Iterable[str] = (),
                 seed: int | None = None, paths=None, profile_scale: float = 1.0,
                 pipeline_name: str = "pipeline", flags: Mapping[str, Any] | None = None, ctx=None):
        self.dag = dag
        self.operations = dict(operations or {})
        self.scenario = scenario
        self.target_s = float(target_s)
        self.params = params or TuningParams()
        self.ablations = frozenset(ablations)
        self.seed = scenario.seed if seed is None else seed
        self.pipeline_name = pipeline_name
        self.flags = dict(flags or {})
        self.frames = [(int(fid), dict(attrs)) for fid, attrs in frames]
        self.spec = RunSpec(dag, profiles, scenario, self.params, ablations=self.ablations,
                            paths=paths, profile_scale=profile_scale)
        self._ctx = ctx
        self.decision_log: list[tuple] = []
        self.final_latency: np.ndarray | None = None

    def run_to_completion(self, log_cap: int | None = None) -> RunReport:
        eng = ReplicaEngine(self.spec, self._ctx)
        fo, at = self.spec.encode_frames([self.frames])
        cap = log_cap if log_cap is not None else 8 * (self.spec.item_bound(fo, at) + 64)
        t0 = time.perf_counter()
        res = eng.run(None, [self.target_s], [self.seed], log_cap=cap, final_tables=True,
                      encoded=(fo, at), event_cap=cap)[0]
        wall = time.perf_counter() - t0
        self.decision_log = eng.log_rows(res.log)
        self.final_latency = res.lat
        self.sim = _SimView(eng.event_rows(res.events))
        eng.close()
        return report_of(res, target_s=self.target_s, scenario_name=self.scenario.name,
                         pipeline_name=self.pipeline_name, seed=self.seed,
                         ablations=self.ablations, flags=self.flags, wall_s=wall)

    def write_decision_log(self, path: str) -> None:
        """manager.py:632-646."""
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("virtual_time\tdecision\tinvocation_id\toperation\tbackend"
                     "\tconfig_id\tslack_s\tobjective\n")
            for t, kind, iid, op, backend, cid, slack_s, obj in self.decision_log:
                fh.write(f"{t:.9f}\t{kind}\t{iid}\t{op}\t{backend}\t{cid}\t{slack_s:.9f}\t{obj:.9f}\n")


# ---- traces (workload.py:14-66) ------------------------------------------------------------

def load_trace(path: str) -> list[tuple[int, dict[str, int]]]:
    """One JSON object per line: frame_id plus non-negative integer attributes (workload.py:14-36)."""
    import json

    frames = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            obj = json.loads(line)
            if "frame_id" not in obj:
                raise ValueError(f"{path}:{lineno}: missing frame_id")
            attrs = {}
            for k, v in obj.get("attributes", {}).items():
                if not isinstance(v, int) or isinstance(v, bool) or v < 0:
                    raise ValueError(f"{path}:{lineno}: attribute {k!r} must be a non-negative integer")
                attrs[k] = v
            frames.append((int(obj["frame_id"]), attrs))
    return frames


def generate_trace(count: int, seed: int, attribute_rates: Mapping[str, float] | None = None,
                   max_per_attribute: int = 4) -> list[tuple[int, dict[str, int]]]:
    """Poisson attribute counts per frame, clipped (workload.py:45-66; same numpy stream)."""
    if count < 0:
        raise ValueError("count must be non-negative")
    rng = np.random.default_rng(seed)
    rates = dict(attribute_rates or {})
    return [(fid, {name: int(min(rng.poisson(rate), max_per_attribute))
                   for name, rate in sorted(rates.items())}) for fid in range(count)]
