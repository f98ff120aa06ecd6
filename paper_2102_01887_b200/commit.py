"""Batched commit step: Configurator.pump_commits rounds on the B200.

The reference commits one speculated invocation per round (configurator.py:693-756): for every
operation whose speculative queue has a head it re-selects the head's configuration
(``_commit_candidate``, 657-691: ``OpTable.select`` with ``allow_delay=False``, the saturated
kinds excluded, ``min_batch = head.fill`` and ``available = head.fill + buffered``), scores the
candidate's hardware affinity (Eq. 3, ``OpTable.affinity``, 302-318) and commits the head with
the smallest priority key — ``(0, -depth, id)`` for warm-up heads, ``(1, -affinity, slack, id)``
otherwise, ``(id,)`` under the ``pbc`` ablation; ``eslc`` commits the speculated entry as is.

``commit_round`` runs R such rounds (independent queue states over the same operations) in one
library call: one K2 launch re-selects all R x n_ops heads, one kernel forms the keys and
reduces every round with a warp (sp_commit.cu).  ``commit_candidates`` is the per-round form a
GPU-backed ``Configurator.pump_commits`` calls.
"""
from __future__ import annotations

import ctypes as C
from typing import Any, Iterable, Mapping, Sequence

import numpy as np

from . import _lib
from ._lib import check, get_context, ptr

ABLATIONS = {"pbc": _lib.SP_COMMIT_FIFO, "eslc": _lib.SP_COMMIT_ESLC}


def policy_of(ablations: Iterable[str]) -> int:
    p = 0
    for a in ablations:
        p |= ABLATIONS.get(a, 0)
    return p


def _is_device(a) -> bool:
    return hasattr(a, "is_cuda") and a.is_cuda


def commit_round(tables: Sequence, slack, head_fill, buffered, head_id, depth, head_flags, *,
                 alpha: float, full_mask, policy: int = 0, spec_idx=None, spec_slack=None,
                 spec_obj=None, ctx=None) -> dict:
    """R commit rounds over the same ``tables`` (op j = tables[j]).

    Shapes: ``slack`` (R, n_ops, K); ``head_fill``, ``buffered``, ``head_id``, ``head_flags``,
    ``spec_*`` (R, n_ops); ``depth`` (n_ops,); ``full_mask`` (R,).  numpy arrays (host: the
    call copies in and out and synchronises) or torch CUDA tensors (device: stream-ordered).
    Returns ``idx, fill, slack, obj, aff`` (R, n_ops) and ``best`` (R,), see sp_commit_round.
    """
    n_ops = len(tables)
    ctx = ctx or tables[0]._ctx
    dev = _is_device(slack)
    if dev:
        import torch

        R = int(slack.shape[0])
        z = lambda shape, dt: torch.empty(shape, dtype=dt, device=slack.device)
        i32, f64 = torch.int32, torch.float64
        if spec_idx is None:
            spec_idx = torch.zeros((R, n_ops), dtype=i32, device=slack.device)
        if spec_slack is None:
            spec_slack = torch.zeros((R, n_ops), dtype=f64, device=slack.device)
        if spec_obj is None:
            spec_obj = torch.zeros((R, n_ops), dtype=f64, device=slack.device)
        mem = _lib.SP_MEM_DEVICE
    else:
        slack = np.ascontiguousarray(slack, dtype=np.float64)
        if slack.ndim == 2:
            slack = slack[None]
        R = slack.shape[0]
        shp = (R, n_ops)
        c = lambda a, dt: np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=dt), shp))
        head_fill, buffered = c(head_fill, np.int32), c(buffered, np.int32)
        head_id, head_flags = c(head_id, np.int64), c(head_flags, np.uint32)
        spec_idx = c(0 if spec_idx is None else spec_idx, np.int32)
        spec_slack = c(0.0 if spec_slack is None else spec_slack, np.float64)
        spec_obj = c(0.0 if spec_obj is None else spec_obj, np.float64)
        depth = np.ascontiguousarray(depth, dtype=np.int32)
        full_mask = np.ascontiguousarray(np.broadcast_to(np.asarray(full_mask, np.uint32), (R,)))
        z = lambda shape, dt: np.empty(shape, dtype=dt)
        i32, f64 = np.int32, np.float64
        mem = _lib.SP_MEM_HOST
    out = {"idx": z((R, n_ops), i32), "fill": z((R, n_ops), i32), "slack": z((R, n_ops), f64),
           "obj": z((R, n_ops), f64), "aff": z((R, n_ops), f64), "best": z((R,), i32)}
    handles = (C.c_void_p * n_ops)(*[t.handle.value for t in tables])
    check(ctx.lib.sp_commit_round(
        ctx.handle, R, n_ops, handles, float(alpha), ptr(slack), ptr(head_fill), ptr(buffered),
        ptr(head_id), ptr(depth), ptr(head_flags), ptr(spec_idx), ptr(spec_slack), ptr(spec_obj),
        ptr(full_mask), int(policy), ptr(out["idx"]), ptr(out["fill"]), ptr(out["slack"]),
        ptr(out["obj"]), ptr(out["aff"]), ptr(out["best"]), mem), "sp_commit_round")
    return out


def commit_candidates(tables: Sequence, slacks: Sequence[Mapping[str, float]],
                      heads: Sequence[Any | None], buffered: Sequence[int],
                      depths: Sequence[int], full_kinds: Iterable[str], alpha: float,
                      ablations: Iterable[str] = ()):
    """One pump_commits round with the reference's objects (configurator.py:693-728).

    ``heads[j]`` is op j's speculative-queue head (an object with ``fill``, ``forced``,
    ``invocation_id``, ``spec_eidx``, ``spec_slack_s``, ``spec_objective``) or None.  Returns
    ``(j, entry, entry_index, fill_target, slack_s, objective)`` for the winning op — exactly the
    tuple the reference's loop picks as ``best`` — or None when no op has a candidate.
    """
    n = len(tables)
    K = tables[0].K
    slack = np.zeros((1, n, K), dtype=np.float64)
    fill = np.zeros((1, n), np.int32)
    hid = np.zeros((1, n), np.int64)
    hf = np.zeros((1, n), np.uint32)
    sidx = np.zeros((1, n), np.int32)
    ssl = np.zeros((1, n), np.float64)
    sob = np.zeros((1, n), np.float64)
    for j, (t, h) in enumerate(zip(tables, heads)):
        if h is None:
            continue
        if slacks[j] is not None:  # else the head's candidate needs no slack (see _needs_slack)
            slack[0, j] = t.slack_array(slacks[j])
        fill[0, j] = h.fill
        hid[0, j] = h.invocation_id
        hf[0, j] = _lib.SP_HEAD_PRESENT | (_lib.SP_HEAD_FORCED if h.forced else 0)
        sidx[0, j] = max(int(h.spec_eidx), 0)
        ssl[0, j] = h.spec_slack_s
        sob[0, j] = h.spec_objective
    full = tables[0].excluded_mask(full_kinds)
    r = commit_round(tables, slack, fill, np.asarray(buffered, np.int32)[None], hid,
                     np.asarray(depths, np.int32), hf, alpha=alpha, full_mask=[full],
                     policy=policy_of(ablations), spec_idx=sidx, spec_slack=ssl, spec_obj=sob)
    j = int(r["best"][0])
    if j < 0:
        return None
    e = int(r["idx"][0, j])
    return (j, tables[j].entries[e], e, int(r["fill"][0, j]), float(r["slack"][0, j]),
            float(r["obj"][0, j]))


def _needs_slack(conf, op, head, full, fifo) -> bool:
    """Whether Configurator._commit_candidate / pump_commits (configurator.py:657-728) call
    slack_by_kind(op) for this head."""
    if head is None:
        return False
    if head.forced:
        return conf.tables[op].ref_entry.backend_kind not in full
    if "eslc" in conf.ablations:
        return head.spec_entry.backend_kind not in full and not fifo
    return True


def pump_commits(conf, buffered_count, topup) -> int:
    """Drop-in for ``Configurator.pump_commits`` (configurator.py:693-756) on a reference-shaped
    configurator whose ``tables`` are this package's ``OpTable``s.

    Every round's candidate scan and priority key (657-728: re-selection of each op's head,
    Eq. 3 affinity, the key order) is one ``commit_candidates`` call on the device; the commit
    itself — popping the head, moving its weight from the speculative to the commit queue,
    topping up, the decision log, submission (731-756) — is the reference's bookkeeping,
    replayed in the same order.  Returns the number of commits.
    """
    import time

    committed = 0
    ops = list(conf.tables)
    tabs = [conf.tables[o] for o in ops]
    depths = [conf.depths[o] for o in ops]
    fifo = "pbc" in conf.ablations
    while True:
        t0 = time.perf_counter()
        full = frozenset(k for k in conf.kinds if conf._cq_length(k) >= conf.cq_capacity[k])
        heads = [conf.sq_by_op[o][0] if conf.sq_by_op[o] else None for o in ops]
        # slack_by_kind only where the reference evaluates it (it caches by weight version, so
        # an extra call would fix a value the reference computes later, at a later clock):
        # forced heads whose reference kind has room, eslc heads whose speculated kind has room
        # and that need the affinity key (not pbc), every other head (its re-selection)
        slacks = [conf.slack_by_kind(o) if _needs_slack(conf, o, h, full, fifo) else None
                  for o, h in zip(ops, heads)]
        try:
            best = commit_candidates(tabs, slacks, heads,
                                     [buffered_count(o) if h is not None else 0
                                      for o, h in zip(ops, heads)],
                                     depths, full, conf.params.alpha, conf.ablations)
        except _lib.SlackpipeError:
            # a shape the batched kernel does not take: the reference's own loop (its
            # OpTable.select / affinity calls still run on the device) from this round on
            from .speculate import _ORIGINAL

            original = _ORIGINAL.get("pump_commits")
            if original is None:
                raise
            return committed + original(conf, buffered_count, topup)
        if best is None:
            return committed
        j, entry, eidx, fill_target, slack_s, obj = best
        op, inv = ops[j], heads[j]
        conf.sq_by_op[op].popleft()
        conf._weights_add(conf._sq_weight, inv.spec_entry.backend_kind, op, inv.spec_eidx, -1)
        if fill_target > inv.fill:
            topup(inv, fill_target - inv.fill)
        inv.state = "committed"
        inv.committed_entry = entry
        inv.committed_eidx = eidx
        inv.committed_slack_s = slack_s
        inv.committed_at = conf._clock()
        conf._weights_add(conf._cq_weight, entry.backend_kind, op, eidx, +1)
        conf.decision_log.append((conf._clock(), "commit", inv.invocation_id, op,
                                  entry.backend_kind, entry.config_id, slack_s, obj))
        conf.commit_times.append(time.perf_counter() - t0)
        committed += 1
        conf._submit(inv, entry, inv.fill)
