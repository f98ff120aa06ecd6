"""CPU restatement of Eq. 2 queueing — TEST ORACLE ONLY.

``estimate_queueing``  configurator.py:109-119 (sum of lat*res/pool, left to right)
``queueing_by_kind``   configurator.py:511-524 (sum of count*(lat*res) in SQ-then-CQ dict
                       order, divided by the pool once).  The two differ bitwise in ~36% of
                       random cases (SURVEY.md §8 rule P5); the live engine uses the latter.
"""
from __future__ import annotations


def estimate_queueing(pairs, pool: float) -> float:
    total = 0.0
    for lat, res in pairs:
        total += lat * res / pool
    return total


def queueing_by_kind(triples, pool: float) -> float:
    total = 0.0
    for lat, res, count in triples:
        total += count * (lat * res)
    return total / pool
