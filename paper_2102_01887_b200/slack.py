"""Alg. 1 slack allotment on the device (K1): configurator.py:76-106, 493-543.

A :class:`SlackGraph` is the device form of "every decomposed path suffix that starts at an
operation":

* ``SlackGraph.from_dag(dag)`` — the pipeline DAG itself.  Every op->sink path of a DAG is a
  suffix of some input->output path returned by ``decompose_paths`` (pipeline.py:428-451),
  so the exponential path enumeration is replaced by a per-source forward DP.
* ``SlackGraph.from_paths(paths)`` — an explicit path list (what ``compute_slack`` and the
  reference ``Configurator`` receive); suffixes are merged into a trie so only the listed
  suffixes are considered, exactly as the reference iterates them.

``slack_batch`` evaluates ``slack[i, s, k] = min_suffix (ref[op_s] / total) * budget_k`` for
many pipeline instances at once, bit-identical to ``Configurator.slack_by_kind``.
"""
from __future__ import annotations

import ctypes as C
from typing import Mapping, Sequence

import numpy as np

from . import _lib
from ._lib import check, get_context, ptr


class SlackGraph:
    def __init__(self, *, pred_ptr, pred_idx, val_idx, terminal, sources, value_names,
                 source_names, device: int | None = None):
        self._ctx = get_context(device)
        self.value_names = list(value_names)
        self.source_names = list(source_names)
        self._vpos = {n: i for i, n in enumerate(self.value_names)}
        self._spos = {n: i for i, n in enumerate(self.source_names)}
        self.V = len(val_idx)
        pp = np.ascontiguousarray(pred_ptr, dtype=np.int32)
        pi = np.ascontiguousarray(pred_idx if len(pred_idx) else [0], dtype=np.int32)
        vi = np.ascontiguousarray(val_idx, dtype=np.int32)
        te = np.ascontiguousarray(terminal, dtype=np.uint8)
        so = np.ascontiguousarray(sources, dtype=np.int32)
        h = C.c_void_p()
        check(self._ctx.lib.sp_dag_create(self._ctx.handle, self.V, ptr(pp), ptr(pi), ptr(vi),
                                          ptr(te), len(so), ptr(so), C.byref(h)), "sp_dag_create")
        self._handle = h

    # -- constructors ---------------------------------------------------------------------
    @classmethod
    def from_dag(cls, dag, sources: Sequence[str] | None = None, *, device: int | None = None):
        order = dag.topological_order() if hasattr(dag, "topological_order") else _topo(dag)
        pos = {v: i for i, v in enumerate(order)}
        preds: list[list[int]] = [[] for _ in order]
        has_succ = set()
        for s, d in dag.edges:
            preds[pos[d]].append(pos[s])
            has_succ.add(s)
        pred_ptr = [0]
        pred_idx: list[int] = []
        for v in range(len(order)):
            pred_idx.extend(sorted(preds[v]))
            pred_ptr.append(len(pred_idx))
        names = list(dag.vertices)
        vpos = {n: i for i, n in enumerate(names)}
        srcs = list(sources) if sources is not None else names
        return cls(
            pred_ptr=pred_ptr, pred_idx=pred_idx,
            val_idx=[vpos[v] for v in order],
            terminal=[0 if v in has_succ else 1 for v in order],
            sources=[pos[s] for s in srcs], value_names=names, source_names=srcs,
            device=device,
        )

    @classmethod
    def from_paths(cls, paths: Sequence[Sequence[str]], sources: Sequence[str] | None = None,
                   *, device: int | None = None):
        """Suffix trie of every path containing each source (configurator.py:415-420)."""
        all_names: list[str] = []
        for p in paths:
            for o in p:
                if o not in all_names:
                    all_names.append(o)
        srcs = list(sources) if sources is not None else all_names
        # values: only operations that occur on a suffix of some source
        names: list[str] = []
        for op in srcs:
            for p in paths:
                if op in p:
                    for o in p[list(p).index(op):]:
                        if o not in names:
                            names.append(o)
        vpos = {n: i for i, n in enumerate(names)}
        pred_ptr = [0]
        pred_idx: list[int] = []
        val_idx: list[int] = []
        terminal: list[int] = []
        roots: list[int] = []
        for op in srcs:
            sufs = [tuple(p[list(p).index(op):]) for p in paths if op in p]
            if not sufs:
                raise ValueError(f"operation {op!r} does not appear on any path")
            node_of: dict[tuple, int] = {}
            for suf in sufs:
                for L in range(1, len(suf) + 1):
                    key = suf[:L]
                    if key in node_of:
                        continue
                    v = len(val_idx)
                    node_of[key] = v
                    val_idx.append(vpos[suf[L - 1]])
                    terminal.append(0)
                    if L > 1:
                        pred_idx.append(node_of[suf[: L - 1]])
                    pred_ptr.append(len(pred_idx))
                terminal[node_of[suf]] = 1
            roots.append(node_of[sufs[0][:1]])
        return cls(pred_ptr=pred_ptr, pred_idx=pred_idx, val_idx=val_idx, terminal=terminal,
                   sources=roots, value_names=names, source_names=srcs, device=device)

    # -- evaluation ---------------------------------------------------------------------------
    @property
    def handle(self):
        return self._handle

    def ref_vector(self, ref_latency: Mapping[str, float]) -> np.ndarray:
        return np.array([float(ref_latency[n]) for n in self.value_names], dtype=np.float64)

    def slack_batch(self, ref, target, now, Q, *, out=None, ratios: bool = False):
        """ref: (n_val,) shared or (I, n_val); target, now: (I,); Q: (I, K).

        Returns slack (I, n_src, K) [and ratios (I, n_src, 2) = (own/Tmax, own/Tmin)].
        numpy in -> synchronous host call; torch CUDA tensors in -> stream-ordered.
        """
        device = hasattr(target, "is_cuda") and bool(target.is_cuda)
        I = int(target.shape[0])
        K = int(Q.shape[1]) if Q.ndim == 2 else 0
        stride = 0 if ref.ndim == 1 else int(ref.shape[1])
        n_src = len(self.source_names)
        if out is None:
            if device:
                import torch

                out = {"slack": torch.empty((I, n_src, K), dtype=torch.float64, device=target.device)}
                if ratios:
                    out["ratio"] = torch.empty((I, n_src, 2), dtype=torch.float64, device=target.device)
            else:
                out = {"slack": np.empty((I, n_src, K), np.float64)}
                if ratios:
                    out["ratio"] = np.empty((I, n_src, 2), np.float64)
        check(self._ctx.lib.sp_slack_batch(
            self._ctx.handle, self._handle, I, ptr(ref), stride, ptr(target), ptr(now), K,
            ptr(Q), ptr(out["slack"]), ptr(out.get("ratio")),
            _lib.SP_MEM_DEVICE if device else _lib.SP_MEM_HOST), "sp_slack_batch")
        return out

    def slack_select_batch(self, tables: Sequence, alpha: float, ref, target, now, Q, available,
                           *, upstream_supply, min_batch, flags, out=None, kslack: bool = False):
        """K1 -> K2 fused (sp_slack_select_batch): for every instance i and source s, the Alg. 1
        slack of s is the slack_by_kind of invocation d = i * n_src + s, decided against
        ``tables[s]`` (one table per source, in ``source_names`` order).

        ``available``, ``upstream_supply``, ``min_batch``, ``flags``: (I * n_src,).  Returns the
        decision arrays of ``select_batch`` (flattened over d) and, with ``kslack``, the slack
        values (I * n_src, K).  numpy -> synchronous; torch CUDA tensors -> stream-ordered.
        """
        if len(tables) != len(self.source_names):
            raise ValueError("slack_select_batch: one table per source operation")
        device = hasattr(target, "is_cuda") and bool(target.is_cuda)
        I = int(target.shape[0])
        K = int(Q.shape[1])
        N = I * len(tables)
        stride = 0 if ref.ndim == 1 else int(ref.shape[1])
        if out is None:
            if device:
                import torch

                z = lambda shape, dt: torch.empty(shape, dtype=dt, device=target.device)
                i32, f64 = torch.int32, torch.float64
            else:
                z = lambda shape, dt: np.empty(shape, dtype=dt)
                i32, f64 = np.int32, np.float64
            out = {"idx": z(N, i32), "code": z(N, i32), "fill": z(N, i32), "obj": z(N, f64),
                   "slack": z(N, f64), "wait": z(N, f64)}
            if kslack:
                out["kslack"] = z((N, K), f64)
        arr_t = (C.c_void_p * len(tables))(*[t.handle.value for t in tables])
        check(self._ctx.lib.sp_slack_select_batch(
            self._ctx.handle, self._handle, len(tables), C.cast(arr_t, C.c_void_p), float(alpha), I,
            ptr(ref), stride, ptr(target), ptr(now), K, ptr(Q), ptr(available), ptr(upstream_supply),
            ptr(min_batch), ptr(flags), ptr(out["idx"]), ptr(out["code"]), ptr(out.get("fill")),
            ptr(out.get("obj")), ptr(out.get("slack")), ptr(out.get("wait")), ptr(out.get("kslack")),
            _lib.SP_MEM_DEVICE if device else _lib.SP_MEM_HOST), "sp_slack_select_batch")
        return out

    def slack_by_kind(self, op: str, kinds: Sequence[str], *, target_s: float, now: float,
                      queueing: Mapping[str, float], ref_latency: Mapping[str, float]) -> dict:
        """Configurator.slack_by_kind for one op (configurator.py:526-543)."""
        s = self._spos[op]
        Q = np.array([[float(queueing[k]) for k in kinds]], dtype=np.float64)
        r = self.slack_batch(self.ref_vector(ref_latency), np.array([float(target_s)]),
                             np.array([float(now)]), Q)
        return {k: float(r["slack"][0, s, j]) for j, k in enumerate(kinds)}

    def close(self) -> None:
        if getattr(self, "_handle", None):
            self._ctx.lib.sp_dag_destroy(self._ctx.handle, self._handle)
            self._handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _topo(dag) -> list[str]:
    indeg = {v: 0 for v in dag.vertices}
    for _, d in dag.edges:
        indeg[d] += 1
    ready = sorted(v for v, n in indeg.items() if n == 0)
    order = []
    while ready:
        v = ready.pop(0)
        order.append(v)
        for d in sorted(d for s, d in dag.edges if s == v):
            indeg[d] -= 1
            if indeg[d] == 0:
                ready.append(d)
                ready.sort()
    if len(order) != len(dag.vertices):
        raise ValueError("pipeline contains a cycle")
    return order


def compute_slack(operation: str, backend_kind: str, *, target_s: float, elapsed_s: float,
                  queueing_s: float, paths, ref_latency: Mapping[str, float]):
    """configurator.py:76-106 — Alg. 1 for one operation, on the device."""
    from .configurator import Slack

    if not any(operation in p for p in paths):
        raise ValueError(f"operation {operation!r} does not appear on any path")
    g = SlackGraph.from_paths(paths, [operation])
    try:
        r = g.slack_batch(g.ref_vector(ref_latency), np.array([float(target_s)]),
                          np.array([float(elapsed_s)]), np.array([[float(queueing_s)]]))
    finally:
        g.close()
    return Slack(float(r["slack"][0, 0, 0]), backend_kind)
