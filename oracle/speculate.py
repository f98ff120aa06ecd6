"""CPU restatement of Configurator.speculate_from_buffer's decision loop — TEST ORACLE ONLY.

Follows configurator.py:563-620 (the loop: forced warm-up decisions, the batching-hold gate, the
select call, popping `fill` items, enqueueing), 511-524 (Eq. 2 `queueing_by_kind`: SQ then CQ
weights in dict order), 526-543 (`slack_by_kind` from the op's path ratios) and 553-561
(`_weights_add`: an existing key is incremented in place, a new key appended) over
oracle/optable.py tables.  Pinned against tests/golden/speculate_calls.npz (calls recorded from
the unmodified reference engine) by tests/test_oracle_golden.py.
"""
from __future__ import annotations

import math

import numpy as np

from . import optable

SDB_ON, FORCED, HOLD_EXPIRED = 1, 2, 4


def speculate(tables, op: int, n: int, supply: int, now: float, target: float, rmin: float,
              rmax: float, pool, alpha: float, flags: int, sq, cq, slack0):
    """One speculate_from_buffer call of operation `op` with `n` buffered items.

    slack0: the op's slack_by_kind when the call starts — the reference caches it by weight
    version only (configurator.py:526-529), so it can carry an earlier clock; every later
    iteration follows an _weights_add bump and recomputes it with `now`.

    sq, cq: per global kind a list of [table, entry, count] in the weights dict's order; `sq` is
    updated in place as the reference's _weights_add does.  Returns (decisions, delay):
    decisions = [(entry, fill, slack_s, objective)] for every invocation formed, delay =
    (entry, wait_budget_s) when the loop stopped on a delay decision, else None.
    """
    t = tables[op]
    K = len(pool)
    out = []
    first = True
    while n > 0:
        # configurator.py:516-523: Eq. 2 per kind, SQ weights then CQ weights
        slack = np.array(slack0, dtype=np.float64) if first else np.empty(K)
        for k in range(K if not first else 0):
            total = 0.0
            for lst in (sq[k], cq[k]):
                for tb, e, c in lst:
                    total += c * (tables[tb].lat[e] * tables[tb].res[e])
            q = total / pool[k]
            budget = target - now - q  # configurator.py:535
            # min over the op's ratios r of r * budget (configurator.py:536-540)
            slack[k] = (rmin if budget >= 0.0 else rmax) * budget
        if flags & FORCED:  # configurator.py:571-589
            i = int(t.ref_index)
            fill = 1
            kd = int(t.gkind[i])
            s_k = float(slack[kd])
            obj = math.nan
        else:
            allow = bool(flags & SDB_ON) and not (first and (flags & HOLD_EXPIRED))
            code, i, fill, obj, s_k, wait, _ = optable.select(t, slack, alpha, n, allow_delay=allow,
                                                               upstream_supply=supply)
            if code == optable.DELAY:  # configurator.py:606-612
                return out, (i, wait)
            kd = int(t.gkind[i])
        first = False  # the hold is popped after the first formed invocation (613)
        n -= fill
        for item in sq[kd]:  # _weights_add(self._sq_weight, kind, op, eidx, +1)
            if item[0] == op and item[1] == i:
                item[2] += 1
                break
        else:
            sq[kd].append([op, i, 1])
        out.append((i, fill, s_k, obj))
    return out, None
