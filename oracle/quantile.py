"""CPU restatement of the batch percentile estimate — TEST ORACLE ONLY.

The reference has no percentile; this follows numpy's documented
``np.quantile(..., method="inverted_cdf")`` per entry, which is what the device kernel
(sp_quantile.cu) promises.
"""
from __future__ import annotations

import math

import numpy as np


def batch_quantiles(sizes, op, idx, obs, q: float):
    """(quantile, count) over all entries of tables with the given sizes (entries numbered
    across tables in order); idx < 0 is no observation."""
    total = int(sum(sizes))
    base = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    per: dict[int, list] = {}
    for j in range(len(idx)):
        if idx[j] < 0:
            continue
        g = int(base[0 if op is None else op[j]] + idx[j])
        per.setdefault(g, []).append(float(obs[j]))
    out = np.full(total, np.nan)
    cnt = np.zeros(total, np.int32)
    for g, v in per.items():
        out[g] = np.quantile(np.array(v), q, method="inverted_cdf")
        cnt[g] = len(v)
    return out, cnt


def order_statistic(values, q: float) -> float:
    """inverted_cdf by its definition: the ceil(q * n)-th smallest value (the smallest at q = 0)."""
    v = sorted(values)
    r = min(max(math.ceil(q * len(v)), 1), len(v))
    return v[r - 1]


def smooth(prev, cur, beta: float):
    """manager.py:45-47 EWMA applied to the batch percentile (NaN prev: start at the value)."""
    out = prev.copy()
    m = ~np.isnan(cur)
    start = m & np.isnan(prev)
    upd = m & ~np.isnan(prev)
    out[start] = cur[start]
    out[upd] = beta * cur[upd] + (1.0 - beta) * prev[upd]
    return out
