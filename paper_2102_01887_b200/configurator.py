"""GPU-backed drop-in for the reference's configurator hot path (configurator.py).

Same class / function names, signatures, return types and error behaviour as the reference
(`slackpipe.configurator`), so that the reference's `Configurator` / `PipelineRun` can run on
top of these objects unchanged, and so the parity tests read like the reference's own tests.
Every Eq. 1 score, argmin, delay/downgrade decision, Eq. 3 ratio, Alg. 1 slack and Eq. 2 sum
is computed by libslackpipe_b200.so on the B200; this module only marshals arguments.

Batch entry points (`select_batch`, `SlackGraph.slack_batch`) expose the data-parallel form
of the same functions over many invocations / pipeline instances.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Any, Iterable, Mapping, Sequence

import numpy as np

from . import _lib
from ._lib import check, get_context, ptr
from .pipeline import ConfigEntry, reference_config

ABLATION_TOKENS = ("fb", "dfp", "sdb", "eslc", "pbc")  # configurator.py:23

_I32_MAX = 2**31 - 1


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


@dataclass(frozen=True)
class Slack:
    seconds: float
    backend_kind: str


@dataclass(frozen=True)
class AffinityScore:
    operation: str
    backend_kind: str
    ratio: float


@dataclass
class Decision:
    """Outcome of one selection pass (configurator.py:146-157)."""

    kind: str  # 'assign' or 'delay'
    entry: ConfigEntry
    entry_index: int
    fill: int
    objective_value: float
    slack_s: float
    wait_budget_s: float = 0.0


def _i32(v: int, what: str) -> int:
    v = int(v)
    if not (-(2**31) <= v <= _I32_MAX):
        raise ValueError(f"{what} out of int32 range")
    return v


class SelectResult(dict):
    """Arrays of a batched select: idx, code, fill, obj, slack, wait (+ kind_min)."""

    @property
    def kind_name(self):
        code = self["code"]
        if isinstance(code, np.ndarray):
            k = code & 3
        else:
            k = (code & 3).cpu().numpy()
        return np.array(["none", "assign", "delay", "?"])[k]


class OpTable:
    """Vectorized, device-resident view of one operation's schedulable configurations
    (configurator.py:159-318).

    Public arrays keep the reference's meaning (``lat``, ``res``, ``batch``, ``batch_int``,
    ``pool``, ``price``, ``kind_idx``, ``id_rank``, ``index_of_id``, ``ref_index``,
    ``ref_entry``, ``entries``, ``kinds``, ``max_batch``); ``lat`` is a host mirror kept
    bit-identical to the device copy the kernels read.

    ``kinds`` (keyword-only, optional) fixes the global backend-kind order used by the
    batched API; it defaults to ``scenario.backend_kinds()``.
    """

    def __init__(self, spec, scenario, *, kinds: Sequence[str] | None = None,
                 device: int | None = None) -> None:
        self.operation = spec.operation
        kinds_present = {b.kind for b in scenario.backends}
        entries = []
        for e in spec.entries:  # configurator.py:170-177
            if (
                e.schedulable
                and e.backend_kind in kinds_present
                and e.resource_request <= scenario.backend(e.backend_kind).resources_per_instance
            ):
                entries.append(e)
        if not entries:
            raise ValueError(f"operation {spec.operation!r} has no schedulable configuration")
        self.entries = entries
        self.kinds = sorted({e.backend_kind for e in entries})
        self._kind_pos = {k: i for i, k in enumerate(self.kinds)}
        n = len(entries)
        self.lat = np.array([e.latency_s for e in entries], dtype=np.float64)
        self.res = np.array([e.resource_request for e in entries], dtype=np.float64)
        self.batch = np.array([e.batch_size for e in entries], dtype=np.float64)
        self.batch_int = np.array([e.batch_size for e in entries], dtype=np.int64)
        self.pool = np.array(
            [scenario.backend(e.backend_kind).pool_resources for e in entries], dtype=np.float64
        )
        self.price = np.array(
            [scenario.backend(e.backend_kind).price_rate for e in entries], dtype=np.float64
        )
        self.kind_idx = np.array([self._kind_pos[e.backend_kind] for e in entries], dtype=np.int64)
        order = sorted(range(n), key=lambda i: entries[i].config_id)
        self.id_rank = np.empty(n, dtype=np.int64)
        for rank, i in enumerate(order):
            self.id_rank[i] = rank
        self.index_of_id = {e.config_id: i for i, e in enumerate(entries)}
        ref = reference_config(spec)
        if ref.config_id in self.index_of_id:
            self.ref_index = self.index_of_id[ref.config_id]
            self.ref_entry = entries[self.ref_index]
        else:
            self.ref_index = -1
            self.ref_entry = ref
        self.max_batch = int(self.batch_int.max())

        # ---- device table ---------------------------------------------------------------
        self.global_kinds = list(kinds) if kinds is not None else list(scenario.backend_kinds())
        gpos = {k: i for i, k in enumerate(self.global_kinds)}
        missing = [k for k in self.kinds if k not in gpos]
        if missing:
            raise ValueError(f"kinds {missing} missing from the global kind list")
        if len(self.global_kinds) > _lib.MAX_KINDS:
            raise _lib.SlackpipeError("at most 24 backend kinds are supported")
        self._gpos = gpos
        self.gkind = np.array([gpos[e.backend_kind] for e in entries], dtype=np.int32)
        self._create_device(device)

    def _device_columns(self):
        """sp_table_create's column arguments (kept alive by the caller across the call)."""
        lat_init = np.array([e.latency_initial_s for e in self.entries], dtype=np.float64)
        return (len(self.entries), self.lat, lat_init, self.res, self.batch_int.astype(np.int32),
                self.pool, self.price, self.gkind, self.id_rank.astype(np.int32))

    def _create_device(self, device) -> None:
        self._ctx = get_context(device)
        n, lat, lat_init, res, batch32, pool, price, gkind, rank32 = self._device_columns()
        h = C.c_void_p()
        check(
            self._ctx.lib.sp_table_create(
                self._ctx.handle, n, ptr(lat), ptr(lat_init), ptr(res), ptr(batch32), ptr(pool),
                ptr(price), ptr(gkind), ptr(rank32), len(self.global_kinds), self.ref_index,
                C.byref(h)),
            "sp_table_create",
        )
        self._handle = h

    # -- device plumbing ------------------------------------------------------------------
    @property
    def handle(self) -> C.c_void_p:
        return self._handle

    @property
    def K(self) -> int:
        return len(self.global_kinds)

    def close(self) -> None:
        if getattr(self, "_handle", None):
            self._ctx.lib.sp_table_destroy(self._ctx.handle, self._handle)
            self._handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def sync_from_device(self) -> None:
        """Refresh the host mirror after a device-side fold (sp_feedback_fold)."""
        out = np.empty_like(self.lat)
        check(self._ctx.lib.sp_table_get_latency(self._ctx.handle, self._handle, ptr(out)))
        self.lat[:] = out
        for e, v in zip(self.entries, out):
            e.latency_s = float(v)

    def prepare(self, alpha: float) -> None:
        check(self._ctx.lib.sp_table_prepare(self._ctx.handle, self._handle, float(alpha)))

    def prepare_many(self, alphas) -> None:
        """The plans of several alphas current for this table version: stale ones are rebuilt
        together, up to four per launch (one thread-block cluster each)."""
        a = np.ascontiguousarray(alphas, dtype=np.float64)
        check(self._ctx.lib.sp_table_prepare_many(self._ctx.handle, self._handle, len(a), ptr(a)))

    def invalidate_plans(self) -> None:
        """Every plan of the table is rebuilt by its next use (as after a latency change)."""
        check(self._ctx.lib.sp_table_invalidate(self._ctx.handle, self._handle))

    def plan_supported(self) -> bool:
        return bool(self._ctx.lib.sp_table_plan_supported(self._handle))

    def plan_bytes(self, alpha: float) -> int:
        out = C.c_int64()
        check(self._ctx.lib.sp_table_plan_bytes(self._ctx.handle, self._handle, float(alpha),
                                                C.byref(out)))
        return int(out.value)

    def plan_image(self, alpha: float, builder: str = "default") -> bytes:
        """The decision plan's byte image for alpha, built by the context default, the
        multi-kernel ("legacy") or the one-kernel cluster ("cluster") builder (diagnostic)."""
        return _plan_image(self._ctx, self._handle, alpha, builder)

    # -- reference API ----------------------------------------------------------------------
    def set_latency(self, index: int, latency_s: float) -> None:
        """configurator.py:211-213 (device copy, then the host mirror — a rejected value leaves
        both unchanged)."""
        i = np.array([index], dtype=np.int32)
        v = np.array([latency_s], dtype=np.float64)
        check(self._ctx.lib.sp_table_set_latency(self._ctx.handle, self._handle, 1, ptr(i), ptr(v)))
        self.entries[index].latency_s = latency_s
        self.lat[index] = latency_s

    def slack_array(self, slack_by_kind: Mapping[str, float]) -> np.ndarray:
        """slack_by_kind as a K-vector in global kind order.  Table kinds must be present
        (KeyError, as configurator.py:216); other kinds are unused and filled with NaN."""
        out = np.full(self.K, np.nan, dtype=np.float64)
        for k in self.kinds:
            out[self._gpos[k]] = float(slack_by_kind[k])
        for k, v in slack_by_kind.items():
            if k in self._gpos:
                out[self._gpos[k]] = float(v)
        return out

    def excluded_mask(self, excluded_kinds: Iterable[str]) -> int:
        m = 0
        for k in excluded_kinds:
            if k in self._gpos:
                m |= 1 << self._gpos[k]
        return m

    def scores(self, slack_by_kind: Mapping[str, float], alpha: float) -> tuple[np.ndarray, np.ndarray]:
        """Eq. 1 for every entry (configurator.py:219-227), computed on the device."""
        s = self.slack_array(slack_by_kind)
        score = np.empty(len(self.entries), dtype=np.float64)
        cost = np.empty(len(self.entries), dtype=np.float64)
        check(self._ctx.lib.sp_scores(self._ctx.handle, self._handle, ptr(s), float(alpha),
                                      ptr(score), ptr(cost)), "sp_scores")
        return score, cost

    def select(
        self,
        slack_by_kind: Mapping[str, float],
        alpha: float,
        available: int,
        *,
        allow_delay: bool,
        upstream_supply: int = 0,
        excluded_kinds: frozenset[str] = frozenset(),
        min_batch: int = 1,
    ) -> Decision | None:
        """configurator.py:239-300, one invocation: the per-call drop-in path.  Arguments go
        into persistent one-invocation buffers (pinned staging inside the library, one launch,
        one sync)."""
        one = self._one_call()
        flags = (_lib.SP_FLAG_ALLOW_DELAY if allow_delay else 0) | (
            self.excluded_mask(excluded_kinds) << _lib.SP_FLAG_EXCL_SHIFT)
        one["slack"][0] = self.slack_array(slack_by_kind)
        one["avail"][0] = _i32(available, "available")
        one["supply"][0] = _i32(upstream_supply, "upstream_supply")
        one["min_batch"][0] = _i32(min_batch, "min_batch")
        one["flags"][0] = flags
        check(self._ctx.lib.sp_select_batch(self._ctx.handle, 1, one["tables"], float(alpha), 1,
                                            None, *one["args"], _lib.MODES["auto"],
                                            _lib.SP_MEM_HOST), "sp_select_batch")
        return self.decision_from(one["out"], 0)

    def _one_call(self):
        one = getattr(self, "_one", None)
        if one is None:
            one = {"slack": np.zeros((1, self.K)), "avail": np.zeros(1, np.int32),
                   "supply": np.zeros(1, np.int32), "min_batch": np.zeros(1, np.int32),
                   "flags": np.zeros(1, np.uint32), "q": np.zeros(1, np.int32), "aff": np.zeros(1)}
            one["out"] = {"idx": np.zeros(1, np.int32), "code": np.zeros(1, np.int32),
                          "fill": np.zeros(1, np.int32), "obj": np.zeros(1), "slack": np.zeros(1),
                          "wait": np.zeros(1)}
            one["args"] = [ptr(one[k]) for k in ("slack", "avail", "supply", "min_batch", "flags")] + \
                          [ptr(one["out"][k]) for k in ("idx", "code", "fill", "obj", "slack", "wait")] + \
                          [C.c_void_p(0)]
            one["tables"] = C.cast((C.c_void_p * 1)(self.handle.value), C.c_void_p)
            self._one = one
        return one

    def decision_from(self, r: Mapping[str, Any], i: int) -> Decision | None:
        code = int(r["code"][i]) & 3
        if code == _lib.SP_DEC_NONE:
            return None
        if code == _lib.SP_DEC_ERROR:
            # configurator.py:236: NaN scores leave _argmin's tie set empty
            raise ValueError("min() arg is an empty sequence")
        j = int(r["idx"][i])
        return Decision(
            kind="delay" if code == _lib.SP_DEC_DELAY else "assign",
            entry=self.entries[j],
            entry_index=j,
            fill=int(r["fill"][i]),
            objective_value=float(r["obj"][i]),
            slack_s=float(r["slack"][i]),
            wait_budget_s=float(r["wait"][i]),
        )

    def affinity(self, backend_kind: str, slack_by_kind: Mapping[str, float], alpha: float) -> float | None:
        """Eq. 3 (configurator.py:302-318): unmasked per-kind minima and their ratio on the
        device, one call."""
        if backend_kind not in self._kind_pos:
            return None
        one = self._one_call()
        one["slack"][0] = self.slack_array(slack_by_kind)
        one["q"][0] = self._gpos[backend_kind]
        check(self._ctx.lib.sp_affinity_batch(self._ctx.handle, 1, one["tables"], float(alpha), 1, None,
                                              ptr(one["slack"]), ptr(one["q"]), ptr(one["aff"]),
                                              _lib.MODES["auto"]), "sp_affinity_batch")
        return float(one["aff"][0])

    def select_batch(self, slack, alpha, available, *, upstream_supply, min_batch, flags,
                     kind_min: bool = False, mode: str = "auto", out: dict | None = None) -> SelectResult:
        return select_batch([self], slack, alpha, available, upstream_supply=upstream_supply,
                            min_batch=min_batch, flags=flags, kind_min=kind_min, mode=mode,
                            out=out)


def _plan_image(ctx, handle, alpha: float, builder: str) -> bytes:
    b = {"default": 0, "legacy": 1, "cluster": 2, "current": 3}[builder]
    n = C.c_int64()
    check(ctx.lib.sp_table_plan_image(ctx.handle, handle, float(alpha), b, None, 0, C.byref(n)),
          "sp_table_plan_image")
    out = np.empty(int(n.value), np.uint8)
    check(ctx.lib.sp_table_plan_image(ctx.handle, handle, float(alpha), b, ptr(out), len(out),
                                      C.byref(n)), "sp_table_plan_image")
    return out.tobytes()


def make_flags(allow_delay, excluded_mask=0) -> np.ndarray:
    """Pack per-invocation allow_delay / excluded-kind masks into the SP_FLAG word."""
    ad = np.asarray(allow_delay).astype(np.uint32)
    ex = np.asarray(excluded_mask).astype(np.uint32)
    return (ad * np.uint32(_lib.SP_FLAG_ALLOW_DELAY)) | (ex << np.uint32(_lib.SP_FLAG_EXCL_SHIFT))


def handle_array(tables):
    """The tables' handles as a C void* array (cached on a single table: the common call)."""
    if len(tables) == 1:
        h = getattr(tables[0], "_harr", None)
        if h is None:
            h = (C.c_void_p * 1)(tables[0].handle.value)
            tables[0]._harr = h
        return h
    return (C.c_void_p * len(tables))(*[t.handle.value for t in tables])


def _is_device(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def select_batch(tables: Sequence[OpTable], slack, alpha: float, available, *, upstream_supply,
                 min_batch, flags, op=None, kind_min: bool = False, mode: str = "auto",
                 out: dict | None = None) -> SelectResult:
    """Batched OpTable.select over N invocations (K2).

    ``slack`` is (N, K) float64 in the tables' global kind order; ``available``,
    ``upstream_supply``, ``min_batch`` int32 (N,); ``flags`` uint32 (N,) from
    :func:`make_flags`; ``op`` optional int32 (N,) table index.  All numpy (host: the call
    copies in, launches, copies out and synchronises) or all torch CUDA tensors (device:
    stream-ordered on the context stream, no synchronisation).
    """
    if not tables:
        raise ValueError("select_batch: no tables")
    ctx = tables[0]._ctx
    K = tables[0].K
    device = _is_device(slack)
    N = int(slack.shape[0])
    if tuple(slack.shape) != (N, K):
        raise ValueError(f"slack must have shape (N, {K})")
    if device:
        import torch

        want = ((available, torch.int32), (upstream_supply, torch.int32), (min_batch, torch.int32))
        if slack.dtype != torch.float64 or any(a.dtype != d or a.shape != (N,) for a, d in want) \
                or flags.dtype not in (torch.int32, torch.uint32) or flags.shape != (N,) \
                or (op is not None and (op.dtype != torch.int32 or op.shape != (N,))):
            raise ValueError("select_batch: device inputs must be float64 slack (N, K) and int32 "
                             "available / upstream_supply / min_batch / flags / op (N,)")
    else:  # host inputs: the C-ABI reads raw int32 / uint32 / float64 buffers of length N
        slack = np.ascontiguousarray(slack, dtype=np.float64)
        cols = []
        for name, a, dt in (("available", available, np.int32), ("upstream_supply", upstream_supply, np.int32),
                            ("min_batch", min_batch, np.int32), ("flags", flags, np.uint32),
                            ("op", op, np.int32)):
            if a is None:
                cols.append(None)
                continue
            a = np.ascontiguousarray(a, dtype=dt)
            if a.shape != (N,):
                raise ValueError(f"select_batch: {name} must have shape ({N},)")
            cols.append(a)
        available, upstream_supply, min_batch, flags, op = cols
    if out is None:
        if device:
            import torch

            dev = slack.device
            out = {
                "idx": torch.empty(N, dtype=torch.int32, device=dev),
                "code": torch.empty(N, dtype=torch.int32, device=dev),
                "fill": torch.empty(N, dtype=torch.int32, device=dev),
                "obj": torch.empty(N, dtype=torch.float64, device=dev),
                "slack": torch.empty(N, dtype=torch.float64, device=dev),
                "wait": torch.empty(N, dtype=torch.float64, device=dev),
            }
            if kind_min:
                out["kind_min"] = torch.empty((N, K), dtype=torch.float64, device=dev)
        else:
            out = {
                "idx": np.empty(N, np.int32), "code": np.empty(N, np.int32),
                "fill": np.empty(N, np.int32), "obj": np.empty(N, np.float64),
                "slack": np.empty(N, np.float64), "wait": np.empty(N, np.float64),
            }
            if kind_min:
                out["kind_min"] = np.empty((N, K), np.float64)
    check(
        ctx.lib.sp_select_batch(
            ctx.handle, len(tables), handle_array(tables), float(alpha), N, ptr(op),
            ptr(slack), ptr(available), ptr(upstream_supply), ptr(min_batch), ptr(flags),
            ptr(out["idx"]), ptr(out["code"]), ptr(out.get("fill")), ptr(out.get("obj")),
            ptr(out.get("slack")), ptr(out.get("wait")), ptr(out.get("kind_min") if kind_min else None),
            _lib.MODES[mode], _lib.SP_MEM_DEVICE if device else _lib.SP_MEM_HOST),
        "sp_select_batch",
    )
    return SelectResult(out)


def affinity_from_minima(kind_min, query_kind, *, ctx=None):
    """Eq. 3 ratios from per-kind minima (host numpy in/out)."""
    ctx = ctx or get_context()
    km = np.ascontiguousarray(kind_min, dtype=np.float64)
    q = np.ascontiguousarray(query_kind, dtype=np.int32)
    N, K = km.shape
    outv = np.empty(N, dtype=np.float64)
    check(ctx.lib.sp_affinity_from_minima(ctx.handle, N, K, ptr(km), ptr(q), ptr(outv), None,
                                          _lib.SP_MEM_HOST), "sp_affinity_from_minima")
    return outv


# ---- spec-level functions (configurator.py:64-143, 321-357) ------------------------------

def _ordered_sum(values: Sequence[float], res: Sequence[float] | None = None,
                 pool: float = 1.0, counts: Sequence[int] | None = None, ctx=None) -> float:
    """One left-to-right device sum via sp_queueing (K=1)."""
    ctx = ctx or get_context()
    n = len(values)
    lat = np.ascontiguousarray(values, dtype=np.float64)
    r = np.ascontiguousarray(res if res is not None else np.ones(n), dtype=np.float64)
    c = None if counts is None else np.ascontiguousarray(counts, dtype=np.int32)
    p = np.array([0, n], dtype=np.int32)
    pl = np.array([pool], dtype=np.float64)
    o = np.empty(1, dtype=np.float64)
    check(ctx.lib.sp_queueing(ctx.handle, 1, ptr(p), ptr(lat), ptr(r), ptr(c), ptr(pl), ptr(o)))
    return float(o[0])


def remaining_path_latency(operation: str, path, ref_latency: Mapping[str, float]) -> float:
    """configurator.py:64-73: left-to-right sum from `operation` to the end of `path`."""
    i = path.index(operation)
    return _ordered_sum([ref_latency[o] for o in path[i:]])


def estimate_queueing(queued_entries, pool_resources: float) -> float:
    """configurator.py:109-119 (ordered device sum of lat*res/pool)."""
    es = list(queued_entries)
    return _ordered_sum([e.latency_s for e in es], [e.resource_request for e in es],
                        pool=float(pool_resources))


def objective(entry, slack_s: float, *, price_rate: float, pool_resources: float,
              alpha: float) -> float:
    """configurator.py:122-143 through the Eq. 1 kernel on a one-entry table."""
    # A one-entry table reproduces objective() exactly: pool and price are taken as given.
    tab = _RawTable(lat=[entry.latency_s], res=[entry.resource_request], batch=[entry.batch_size],
                    pool=[float(pool_resources)], price=[float(price_rate)])
    try:
        score, _ = tab.scores(np.array([float(slack_s)]), float(alpha))
    finally:
        tab.close()
    return float(score[0])


class _RawTable:
    """A device table from raw arrays (single kind), for spec-level helpers and benches."""

    def __init__(self, *, lat, res, batch, pool, price, kind=None, id_rank=None, K: int = 1,
                 ref_index: int = -1, lat_init=None, device: int | None = None, ctx=None):
        self._ctx = ctx or get_context(device)
        self.lat = np.ascontiguousarray(lat, dtype=np.float64)
        M = len(self.lat)
        self.M = M
        self.K = K
        self.res = np.ascontiguousarray(res, dtype=np.float64)
        self.batch_int = np.ascontiguousarray(batch, dtype=np.int32)
        self.pool = np.ascontiguousarray(pool, dtype=np.float64)
        self.price = np.ascontiguousarray(price, dtype=np.float64)
        self.gkind = np.ascontiguousarray(np.zeros(M) if kind is None else kind, dtype=np.int32)
        self.id_rank = np.ascontiguousarray(np.arange(M) if id_rank is None else id_rank, dtype=np.int32)
        li = self.lat if lat_init is None else np.ascontiguousarray(lat_init, dtype=np.float64)
        self.ref_index = int(ref_index)
        h = C.c_void_p()
        check(self._ctx.lib.sp_table_create(
            self._ctx.handle, M, ptr(self.lat), ptr(li), ptr(self.res), ptr(self.batch_int),
            ptr(self.pool), ptr(self.price), ptr(self.gkind), ptr(self.id_rank), K,
            self.ref_index, C.byref(h)), "sp_table_create")
        self._handle = h

    @property
    def handle(self):
        return self._handle

    def scores(self, slack_vec: np.ndarray, alpha: float):
        s = np.ascontiguousarray(slack_vec, dtype=np.float64)
        score = np.empty(self.M, np.float64)
        cost = np.empty(self.M, np.float64)
        check(self._ctx.lib.sp_scores(self._ctx.handle, self._handle, ptr(s), float(alpha),
                                      ptr(score), ptr(cost)), "sp_scores")
        return score, cost

    def set_latency(self, index, latency_s) -> None:
        """Batched configurator.py:211-213: lat[index[j]] = latency_s[j] (host mirror + device)."""
        i = np.ascontiguousarray(np.atleast_1d(index), dtype=np.int32)
        v = np.ascontiguousarray(np.atleast_1d(latency_s), dtype=np.float64)
        if i.shape != v.shape:
            raise ValueError("set_latency: index and latency_s differ in length")
        check(self._ctx.lib.sp_table_set_latency(self._ctx.handle, self._handle, len(i), ptr(i), ptr(v)))
        self.lat[i] = v  # after the device accepted the values

    def get_latency(self) -> np.ndarray:
        out = np.empty(self.M, np.float64)
        check(self._ctx.lib.sp_table_get_latency(self._ctx.handle, self._handle, ptr(out)))
        return out

    def plan_bytes(self, alpha: float) -> int:
        out = C.c_int64()
        check(self._ctx.lib.sp_table_plan_bytes(self._ctx.handle, self._handle, float(alpha),
                                                C.byref(out)))
        return int(out.value)

    def prepare(self, alpha: float) -> None:
        check(self._ctx.lib.sp_table_prepare(self._ctx.handle, self._handle, float(alpha)))

    def plan_image(self, alpha: float, builder: str = "default") -> bytes:
        return _plan_image(self._ctx, self._handle, alpha, builder)

    def prepare_many(self, alphas) -> None:
        a = np.ascontiguousarray(alphas, dtype=np.float64)
        check(self._ctx.lib.sp_table_prepare_many(self._ctx.handle, self._handle, len(a), ptr(a)))

    def invalidate_plans(self) -> None:
        check(self._ctx.lib.sp_table_invalidate(self._ctx.handle, self._handle))

    def close(self) -> None:
        if getattr(self, "_handle", None):
            self._ctx.lib.sp_table_destroy(self._ctx.handle, self._handle)
            self._handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


RawTable = _RawTable


def select_config(spec, scenario, slack_by_kind: Mapping[str, float], available: int,
                  params: TuningParams, *, allow_delay: bool = True,
                  upstream_supply: int = 0) -> Decision:
    """configurator.py:321-341."""
    table = OpTable(spec, scenario)
    try:
        decision = table.select(slack_by_kind, params.alpha, available, allow_delay=allow_delay,
                                upstream_supply=upstream_supply)
    finally:
        table.close()
    assert decision is not None
    return decision


def affinity(spec, scenario, backend_kind: str, slack_by_kind: Mapping[str, float],
             params: TuningParams) -> AffinityScore:
    """configurator.py:344-357."""
    table = OpTable(spec, scenario)
    try:
        ratio = table.affinity(backend_kind, slack_by_kind, params.alpha)
    finally:
        table.close()
    if ratio is None:
        raise ValueError(
            f"affinity undefined: {spec.operation!r} has no schedulable entry on {backend_kind!r}"
        )
    return AffinityScore(spec.operation, backend_kind, ratio)


from .slack import SlackGraph, compute_slack  # noqa: E402  (re-export, reference layout)
