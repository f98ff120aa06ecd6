"""Speculation loop on the B200: Configurator.speculate_from_buffer.

The reference forms invocations from an operation's buffered inputs one decision at a time
(configurator.py:563-620): each iteration recomputes the op's slack from the speculative and
commit-queue weights (Eq. 2, 511-524; Alg. 1, 526-543), selects a configuration (or the
reference entry during dfp warm-up), pops ``fill`` items and adds the new invocation's weight
(553-561) — so every iteration depends on the previous one.  ``speculate_batch`` runs R such
calls (independent weight states, e.g. pipeline replicas) with one thread each on the device
(sp_spec.cuh); ``speculate_from_buffer`` is the drop-in for one reference ``Configurator`` call:
the decisions come from the device, the host replays the reference's bookkeeping (invocations,
queues, holds, wake-ups, decision log) in the same order.
"""
from __future__ import annotations

import ctypes as C
import math
import sys
import time
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import check, ptr


def speculate_batch(tables: Sequence, alpha: float, pool, op, n_buf, supply, now, target, rmin,
                    rmax, slack0, flags, w_ptr, w_tab, w_eidx, w_count, *, ctx=None,
                    out=None) -> dict:
    """R speculate_from_buffer calls (see sp_speculate_batch).

    ``slack0`` (R, K); ``w_ptr`` (2*K*R + 1,) CSR over (call, queue, kind) of the weight keys
    (``w_tab`` table index, ``w_eidx`` entry, ``w_count``); ``pool`` (K,) host values.  numpy
    arrays: host memory, the call copies in and out and synchronises; torch CUDA tensors
    (int32 / float64 / uint32 as the C header says): stream-ordered device call.  Returns
    ``off`` (R + 1,) and, per formed invocation, ``idx, fill, slack, obj``; per call ``n``
    (invocations formed) and the stopping delay ``delay_idx`` (-1: none) / ``delay_wait``.
    ``out`` (a previous result for the same n_buf) is reused without reallocating — for
    device calls that keeps the call free of host synchronisation.
    """
    ctx = ctx or tables[0]._ctx
    K = int(tables[0].K)
    pool = np.ascontiguousarray(pool, dtype=np.float64)
    handles = (C.c_void_p * len(tables))(*[t.handle.value for t in tables])
    if hasattr(op, "is_cuda") and op.is_cuda:
        import torch

        R = int(op.shape[0])
        if out is None:
            off = torch.zeros(R + 1, dtype=torch.int32, device=op.device)
            off[1:] = torch.cumsum(n_buf, 0)
            O = max(int(off[-1].item()), 1)
        z = lambda n, dt: torch.empty(n, dtype=dt, device=op.device)
        i32, f64 = torch.int32, torch.float64
        mem = _lib.SP_MEM_DEVICE
    else:
        i32c = lambda a: np.ascontiguousarray(a, dtype=np.int32)
        f64c = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        op, n_buf, supply = i32c(op), i32c(n_buf), i32c(supply)
        R = len(op)
        now, target, rmin, rmax = f64c(now), f64c(target), f64c(rmin), f64c(rmax)
        slack0 = f64c(slack0).reshape(R, K)
        flags = np.ascontiguousarray(flags, dtype=np.uint32)
        w_ptr, w_tab, w_eidx, w_count = i32c(w_ptr), i32c(w_tab), i32c(w_eidx), i32c(w_count)
        if len(w_tab) == 0:
            w_tab = w_eidx = w_count = np.zeros(1, np.int32)
        off = np.zeros(R + 1, np.int32)
        np.cumsum(n_buf, out=off[1:])
        O = max(int(off[-1]), 1)
        z = lambda n, dt: np.empty(n, dtype=dt)
        i32, f64 = np.int32, np.float64
        mem = _lib.SP_MEM_HOST
    if out is None:
        out = {"off": off, "idx": z(O, i32), "fill": z(O, i32), "slack": z(O, f64),
               "obj": z(O, f64), "n": z(R, i32), "delay_idx": z(R, i32), "delay_wait": z(R, f64)}
    off = out["off"]
    check(ctx.lib.sp_speculate_batch(
        ctx.handle, len(tables), handles, float(alpha), K, ptr(pool), R, ptr(op), ptr(n_buf),
        ptr(supply), ptr(now), ptr(target), ptr(rmin), ptr(rmax), ptr(slack0), ptr(flags),
        ptr(w_ptr), ptr(w_tab), ptr(w_eidx), ptr(w_count), ptr(off), ptr(out["idx"]),
        ptr(out["fill"]), ptr(out["slack"]), ptr(out["obj"]), ptr(out["n"]),
        ptr(out["delay_idx"]), ptr(out["delay_wait"]), mem), "sp_speculate_batch")
    return out


def pack_weights(conf, op_index, kinds):
    """The SQ / CQ weight dicts of a reference Configurator as (w_ptr, w_tab, w_eidx, w_count)
    for one call, keys in dict order (configurator.py:511-524 iterates them so)."""
    ptr_, tab, eidx, cnt = [0], [], [], []
    for table in (conf._sq_weight, conf._cq_weight):
        for k in kinds:
            for (o, e), c in table[k].items():
                tab.append(op_index[o])
                eidx.append(e)
                cnt.append(c)
            ptr_.append(len(tab))
    return ptr_, tab, eidx, cnt


def speculate_from_buffer(conf, op: str, buffer) -> int:
    """Drop-in for ``Configurator.speculate_from_buffer`` (configurator.py:563-620) on a
    reference-shaped configurator whose ``tables`` are this package's ``OpTable``s.

    The decisions come from one sp_speculate_batch call; the reference's own bookkeeping
    (``_make_invocation``, ``_enqueue_speculated``, holds, wake-ups, ``forced_counts``,
    ``speculate_times``) is replayed in the reference's order.  Returns the number of
    invocations formed.
    """
    if not buffer:
        return 0
    mod = sys.modules[type(conf).__module__]
    t0 = time.perf_counter()
    names = list(conf.tables)
    op_index = {n: i for i, n in enumerate(names)}
    tables = [conf.tables[n] for n in names]
    table = conf.tables[op]
    kinds = list(conf.kinds)
    dfp_on = "dfp" not in conf.ablations
    sdb_on = "sdb" not in conf.ablations
    forced = dfp_on and table.ref_index >= 0 and conf.completed_ref[op] < conf.params.dfp_count
    hold = conf.holds.get(op)
    now = conf._clock()
    flags = (_lib.SP_SPEC_SDB if sdb_on else 0) | (_lib.SP_SPEC_FORCED if forced else 0) | \
        (_lib.SP_SPEC_HOLD_EXPIRED if hold is not None and now >= hold.deadline_s else 0)
    ratios = conf._path_ratios(op)
    sl0 = conf.slack_by_kind(op)
    w = pack_weights(conf, op_index, kinds)
    try:
        r = speculate_batch(tables, conf.params.alpha, [conf._pool[k] for k in kinds],
                            [op_index[op]], [len(buffer)], [conf._supply(op)], [now],
                            [conf.target_s], [min(ratios)], [max(ratios)],
                            [[sl0[k] for k in kinds]], [flags], *w)
    except _lib.SlackpipeError:
        # shapes the batched kernel does not take (a table without a staircase plan): the
        # reference's own loop, whose OpTable.select calls still run on the device one at a time
        original = _ORIGINAL.get("speculate_from_buffer")
        if original is None:
            raise
        return original(conf, op, buffer)
    formed = int(r["n"][0])
    dt = (time.perf_counter() - t0) / max(1, formed + (r["delay_idx"][0] >= 0))
    for j in range(formed):
        e, fill = int(r["idx"][j]), int(r["fill"][j])
        entry = table.entries[e]
        decision = mod.Decision(kind="assign", entry=entry, entry_index=e, fill=fill,
                                objective_value=float(r["obj"][j]), slack_s=float(r["slack"][j]))
        if forced:
            conf.forced_counts[op] += 1
        conf.holds.pop(op, None)
        items = [buffer.popleft() for _ in range(fill)]
        inv = conf._make_invocation(op, items, forced)
        conf._enqueue_speculated(inv, decision)
        conf.speculate_times.append(dt)
    d = int(r["delay_idx"][0])
    if d >= 0:  # configurator.py:606-612: arm the batching hold once, then stop
        if formed:
            # the reference evaluated slack_by_kind at the top of this last iteration, after
            # the enqueues above changed the weight version: leave its cache in that state
            conf.slack_by_kind(op)
        if conf.holds.get(op) is None:
            deadline = conf._clock() + float(r["delay_wait"][0])
            conf.holds[op] = mod._Hold(deadline, table.entries[d].batch_size)
            if deadline != math.inf:
                conf._schedule_wake(deadline, ("hold", op))
        conf.speculate_times.append(dt)
    return formed


# the reference Configurator's own methods, kept by install() for the shapes the batched kernels
# do not take
_ORIGINAL: dict = {}


def install(configurator_cls) -> None:
    """Replace ``Configurator.speculate_from_buffer`` and ``Configurator.pump_commits`` of the
    reference class (slackpipe.configurator.Configurator) with the device drop-ins, keeping the
    originals as their fallback for tables without a staircase plan."""
    from . import commit as _commit

    if "speculate_from_buffer" not in _ORIGINAL:
        _ORIGINAL["speculate_from_buffer"] = configurator_cls.speculate_from_buffer
        _ORIGINAL["pump_commits"] = configurator_cls.pump_commits
    configurator_cls.speculate_from_buffer = (
        lambda self, op, buffer: speculate_from_buffer(self, op, buffer))
    configurator_cls.pump_commits = (
        lambda self, buffered_count, topup: _commit.pump_commits(self, buffered_count, topup))
