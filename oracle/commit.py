"""CPU restatement of one Configurator.pump_commits round — TEST ORACLE ONLY.

Follows configurator.py:657-691 (_commit_candidate) and 693-728 (the per-round candidate scan
and priority key) over oracle/optable.py tables.  Pinned against tests/golden/commit_rounds.npz
(rounds recorded from the unmodified reference engine) by tests/test_oracle_golden.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import optable


@dataclass
class Head:
    fill: int
    forced: bool
    invocation_id: int
    spec_idx: int = -1
    spec_slack: float = 0.0
    spec_obj: float = 0.0


def commit_candidate(t: optable.Arrays, slack_global, head: Head, full_mask: int, buffered: int,
                     alpha: float, eslc: bool):
    """configurator.py:657-691 -> (entry_index, fill_target, slack_s, objective) or None."""
    if head.forced:
        kind = int(t.gkind[t.ref_index])
        if (full_mask >> kind) & 1:
            return None
        return (t.ref_index, head.fill, float(slack_global[kind]), math.nan)
    if eslc:
        kind = int(t.gkind[head.spec_idx])
        if (full_mask >> kind) & 1:
            return None
        return (head.spec_idx, head.fill, head.spec_slack, head.spec_obj)
    code, i, fill, obj, s_k, _w, _f = optable.select(
        t, slack_global, alpha, head.fill + buffered, allow_delay=False,
        excluded_mask=full_mask, min_batch=head.fill)
    if code == optable.NONE:
        return None
    return (i, max(fill, head.fill), s_k, obj)


def round_winner(tables, slacks, heads, full_mask: int, buffered, depths, alpha: float,
                 fifo: bool = False, eslc: bool = False):
    """configurator.py:704-728: (op index, candidate) of the minimum key, or None."""
    best_key, best = None, None
    for j, (t, h) in enumerate(zip(tables, heads)):
        if h is None:
            continue
        cand = commit_candidate(t, slacks[j], h, full_mask, buffered[j], alpha, eslc)
        if cand is None:
            continue
        if fifo:
            key = (h.invocation_id,)
        elif h.forced:
            key = (0, -depths[j], h.invocation_id)
        else:
            aff = optable.affinity(t, int(t.gkind[cand[0]]), slacks[j], alpha)
            key = (1, -(aff if aff is not None else 0.0), cand[2], h.invocation_id)
        if best_key is None or key < best_key:
            best_key, best = key, (j, cand)
    return best


def amber_tables(meta) -> list:
    """Oracle tables of the AMBER run from tests/golden/amber_trace.npz metadata."""
    back = {k: (n * r, p) for k, n, r, p in meta["backends"]}
    kinds = meta["kinds"]
    out = []
    for name in meta["ops"]:
        m = meta["tables"][name]
        ids = m["config_id"]
        order = sorted(range(len(ids)), key=lambda i: ids[i])
        rank = np.empty(len(ids), dtype=np.int64)
        for r, i in enumerate(order):
            rank[i] = r
        out.append(optable.from_columns(
            lat=m["lat"], res=m["res"], batch=m["batch"],
            pool=[back[k][0] for k in m["kind"]], price=[back[k][1] for k in m["kind"]],
            gkind=[kinds.index(k) for k in m["kind"]], id_rank=rank, n_kinds=len(kinds),
            ref_index=m["ref_index"], lat_init=m["lat_init"]))
    return out
