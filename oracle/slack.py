"""CPU restatement of Alg. 1 slack allotment — TEST ORACLE ONLY.

* ``remaining_path_latency`` / ``compute_slack``       configurator.py:64-106
* ``decompose_paths``                                  pipeline.py:428-451 (DFS, sorted)
* ``path_ratios`` / ``slack_by_kind``                  configurator.py:415-420, 493-543
* ``dp_slack``  forward left-to-right DP restatement for DAGs whose path set cannot be
  enumerated (config 3).  SURVEY.md §8(c) validated it at 0 / 128,045 mismatches against
  ``compute_slack``; tests/test_oracle_golden.py re-runs that check on committed cases.
"""
from __future__ import annotations

from typing import Mapping, Sequence

import numpy as np


def remaining_path_latency(op: str, path: Sequence[str], ref: Mapping[str, float]) -> float:
    total = 0.0
    for o in path[list(path).index(op):]:
        total += ref[o]
    return total


def compute_slack(op: str, *, target_s: float, elapsed_s: float, queueing_s: float,
                  paths: Sequence[Sequence[str]], ref: Mapping[str, float]) -> float:
    budget = target_s - elapsed_s - queueing_s
    best = None
    for p in paths:
        if op not in p:
            continue
        v = ref[op] / remaining_path_latency(op, p, ref) * budget
        if best is None or v < best:
            best = v
    if best is None:
        raise ValueError(f"operation {op!r} does not appear on any path")
    return best


def decompose_paths(vertices: Sequence[str], edges: Sequence[tuple[str, str]]):
    succ = {v: sorted(d for s, d in edges if s == v) for v in vertices}
    has_pred = {d for _, d in edges}
    outputs = {v for v in vertices if not succ[v]}
    paths: list[tuple] = []

    def walk(v, prefix):
        prefix.append(v)
        if v in outputs:
            paths.append(tuple(prefix))
        else:
            for n in succ[v]:
                walk(n, prefix)
        prefix.pop()

    for s in sorted(v for v in vertices if v not in has_pred):
        walk(s, [])
    paths.sort()
    return tuple(paths)


def path_ratios(op: str, paths, ref: Mapping[str, float]) -> tuple:
    own = ref[op]
    out = []
    for p in paths:
        if op not in p:
            continue
        total = 0.0
        for o in p[list(p).index(op):]:
            total += ref[o]
        out.append(own / total)
    return tuple(out)


def slack_by_kind(op: str, kinds: Sequence[str], *, target_s: float, now: float,
                  queueing: Mapping[str, float], paths, ref: Mapping[str, float]) -> dict:
    ratios = path_ratios(op, paths, ref)
    out = {}
    for k in kinds:
        budget = target_s - now - queueing[k]
        s = None
        for r in ratios:
            v = r * budget
            if s is None or v < s:
                s = v
        out[k] = s
    return out


def dp_ratios(order: Sequence[int], preds: Sequence[Sequence[int]], terminal: Sequence[bool],
              ref: np.ndarray, src: int) -> tuple[float, float]:
    """(own/Tmax, own/Tmin) by the forward left-to-right DP from `src` (vertices are
    topologically numbered; preds[v] lists predecessors)."""
    V = len(preds)
    hi = [None] * V
    lo = [None] * V
    hi[src] = lo[src] = 0.0 + float(ref[src])
    for v in range(src + 1, V):
        ps = [p for p in preds[v] if hi[p] is not None]
        if not ps:
            continue
        hi[v] = max(hi[p] for p in ps) + float(ref[v])
        lo[v] = min(lo[p] for p in ps) + float(ref[v])
    tmax = max(hi[v] for v in range(V) if hi[v] is not None and terminal[v])
    tmin = min(lo[v] for v in range(V) if lo[v] is not None and terminal[v])
    own = float(ref[src])
    return own / tmax, own / tmin


def dp_slack(ratio_lo: float, ratio_hi: float, budget: float) -> float:
    return (ratio_lo if budget >= 0 else ratio_hi) * budget
