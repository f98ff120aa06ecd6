"""Profile feedback fold on the device (K3): manager.py:45-47, 91-101, 436-457 and
configurator.py:463-491.

``fold_observations`` replays a batch of completed invocations, in completion order, into
the device tables exactly as ``PipelineRun._apply_feedback`` does one at a time: EWMA
smoothing of the committed entry's latency, observation counts, reference completion
counts, and the one-time warm-up gate-lift rescale of never-observed entries.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import check, ptr


def _is_device(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def fold_observations(tables: Sequence, op, idx, obs, *, beta: float = 0.5,
                      dfp_count: int = 10, dfp_on: bool = True, fb_frozen: bool = False,
                      sync_host: bool = True) -> None:
    """Fold observations obs[j] of entry idx[j] of table tables[op[j]] (op may be None for
    a single table).  numpy inputs run synchronously; torch CUDA tensors stream-ordered.
    With ``sync_host`` the tables' host mirrors (``lat``) are refreshed afterwards."""
    if not tables:
        raise ValueError("fold_observations: no tables")
    ctx = tables[0]._ctx
    device = _is_device(obs)
    n = int(obs.shape[0])
    from .configurator import handle_array

    arr_t = handle_array(tables)
    if not device:
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        obs = np.ascontiguousarray(obs, dtype=np.float64)
        if op is not None:
            op = np.ascontiguousarray(op, dtype=np.int32)
    check(ctx.lib.sp_feedback_fold(
        ctx.handle, len(tables), arr_t, n, ptr(op), ptr(idx), ptr(obs),
        float(beta), int(dfp_count), 1 if dfp_on else 0, 1 if fb_frozen else 0,
        _lib.SP_MEM_DEVICE if device else _lib.SP_MEM_HOST), "sp_feedback_fold")
    if sync_host:
        if device:
            ctx.synchronize()
        for t in tables:
            if hasattr(t, "sync_from_device"):
                t.sync_from_device()


def simulate_observations(decisions, truth_base, noise, *, truth_per_item=None, out=None, ctx=None):
    """Observation records of a decision batch from the simulated backend (backend.py:36-58):
    assignments run, obs = (truth_base[idx] + truth_per_item[idx] * fill) * noise; delayed / None
    decisions give idx -1.  ``decisions``: the device output dict of ``select_batch``
    (``code``, ``idx``, ``fill``); torch CUDA tensors, stream-ordered.  Returns (obs_idx, obs)."""
    from ._lib import get_context

    code = decisions["code"]
    ctx = ctx or get_context(code.device.index)
    n = int(code.shape[0])
    if out is None:
        import torch

        out = (torch.empty(n, dtype=torch.int32, device=code.device),
               torch.empty(n, dtype=torch.float64, device=code.device))
    oi, ob = out
    check(ctx.lib.sp_simulate_observations(
        ctx.handle, n, ptr(code), ptr(decisions["idx"]), ptr(decisions.get("fill")),
        ptr(truth_base), ptr(truth_per_item), ptr(noise), ptr(oi), ptr(ob)),
        "sp_simulate_observations")
    return oi, ob


def simulate_and_fold(table, decisions, truth_base, noise, *, truth_per_item=None, out,
                      beta: float = 0.5, dfp_count: int = 10, dfp_on: bool = True,
                      fb_frozen: bool = False) -> None:
    """``simulate_observations`` then ``fold_observations`` of one table in one cooperative
    kernel (torch CUDA tensors, stream-ordered); the observation records still land in
    ``out = (obs_idx, obs)``."""
    ctx = table._ctx
    code = decisions["code"]
    oi, ob = out
    check(ctx.lib.sp_simulate_and_fold(
        ctx.handle, table.handle, int(code.shape[0]), ptr(code), ptr(decisions["idx"]),
        ptr(decisions.get("fill")), ptr(truth_base), ptr(truth_per_item), ptr(noise),
        float(beta), int(dfp_count), 1 if dfp_on else 0, 1 if fb_frozen else 0, ptr(oi), ptr(ob)),
        "sp_simulate_and_fold")


def table_counters(table) -> tuple[int, np.ndarray]:
    """(completed_ref, per-entry observation counts) of a device table."""
    ctx = table._ctx
    c = C.c_int32()
    M = len(table.lat)
    counts = np.empty(M, dtype=np.int32)
    check(ctx.lib.sp_table_get_counters(ctx.handle, table.handle, C.byref(c), ptr(counts)))
    return int(c.value), counts


def set_table_counters(table, completed_ref: int, counts: np.ndarray | None = None) -> None:
    ctx = table._ctx
    cc = None if counts is None else np.ascontiguousarray(counts, dtype=np.int32)
    check(ctx.lib.sp_table_set_counters(ctx.handle, table.handle, int(completed_ref), ptr(cc)))


def apply_feedback(old_estimate_s: float, observed_s: float, beta: float) -> float:
    """manager.py:45-47, evaluated by the fold kernel on a one-entry table."""
    from .configurator import RawTable

    t = RawTable(lat=[float(old_estimate_s)], res=[1.0], batch=[1], pool=[1.0], price=[1.0])
    try:
        fold_observations([t], None, np.zeros(1, np.int32), np.array([float(observed_s)]),
                          beta=beta, dfp_on=False, sync_host=False)
        return float(t.get_latency()[0])
    finally:
        t.close()


def observation_quantiles(tables: Sequence, op, idx, obs, q: float, *, smooth=None,
                          beta: float = 0.5) -> dict:
    """Per-entry latency percentile of an observation batch (extension of K3; the reference has
    no percentile — parity is pinned to numpy): ``quantile[e] = np.quantile(obs of entry e, q,
    method="inverted_cdf")`` (NaN without observations) and ``count[e]``, entries numbered
    across ``tables`` in order.  ``smooth`` (optional array, updated in place) receives
    ``beta * quantile + (1 - beta) * smooth`` for observed entries — the EWMA of
    manager.py:45-47 applied to the batch percentile.  numpy in -> synchronous; torch CUDA
    tensors in -> stream-ordered."""
    if not tables:
        raise ValueError("observation_quantiles: no tables")
    ctx = tables[0]._ctx
    device = _is_device(obs)
    n = int(obs.shape[0])
    total = sum(len(t.lat) for t in tables)
    arr_t = (C.c_void_p * len(tables))(*[t.handle.value for t in tables])
    if device:
        import torch

        out = {"quantile": torch.empty(total, dtype=torch.float64, device=obs.device),
               "count": torch.empty(total, dtype=torch.int32, device=obs.device)}
    else:
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        obs = np.ascontiguousarray(obs, dtype=np.float64)
        if op is not None:
            op = np.ascontiguousarray(op, dtype=np.int32)
        out = {"quantile": np.empty(total, np.float64), "count": np.empty(total, np.int32)}
    check(ctx.lib.sp_observation_quantiles(
        ctx.handle, len(tables), arr_t, n, ptr(op), ptr(idx), ptr(obs),
        float(q), float(beta), ptr(out["quantile"]), ptr(out["count"]), ptr(smooth),
        _lib.SP_MEM_DEVICE if device else _lib.SP_MEM_HOST), "sp_observation_quantiles")
    return out
