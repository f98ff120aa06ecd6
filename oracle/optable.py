"""CPU restatement of the reference OpTable (configurator.py:159-318) — TEST ORACLE ONLY.

Arrays follow the reference exactly (float64 numpy, same ufunc order), so the results are
bit-identical to the reference.  Two differences of form, none of substance:
  * tables are plain ``Arrays`` records (no ConfigEntry objects needed), built either from
    a ConfigSpec/Scenario (``from_spec``) or from raw SoA columns (``from_columns``);
  * ``select`` returns a small tuple instead of a Decision.
The global kind order used by the batched API is carried alongside (``gkind``).
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Iterable, Mapping, Sequence

import numpy as np

NONE, ASSIGN, DELAY = 0, 1, 2


@dataclass
class Arrays:
    lat: np.ndarray
    res: np.ndarray
    batch: np.ndarray       # float64 (configurator.py:186)
    batch_int: np.ndarray   # int64 (187)
    pool: np.ndarray
    price: np.ndarray
    kind_idx: np.ndarray    # position in the table's sorted kind list (194)
    id_rank: np.ndarray     # Python-str rank of config_id (195-198)
    kinds: list             # sorted table kinds (181)
    gkind: np.ndarray = field(default=None)  # position in the caller's global kind list
    ref_index: int = -1
    lat_init: np.ndarray = field(default=None)
    kind_global: np.ndarray = field(default=None)  # table kind position -> global kind

    def __post_init__(self):
        if self.kind_global is None and self.gkind is not None:
            kg = np.zeros(len(self.kinds), dtype=np.int64)
            for e in range(len(self.lat)):
                kg[self.kind_idx[e]] = self.gkind[e]
            self.kind_global = kg


def from_spec(spec, scenario, global_kinds: Sequence[str] | None = None) -> Arrays:
    """configurator.py:166-209 (filter + SoA build)."""
    present = {b.kind for b in scenario.backends}
    ents = [e for e in spec.entries
            if e.schedulable and e.backend_kind in present
            and e.resource_request <= scenario.backend(e.backend_kind).resources_per_instance]
    if not ents:
        raise ValueError(f"operation {spec.operation!r} has no schedulable configuration")
    kinds = sorted({e.backend_kind for e in ents})
    kpos = {k: i for i, k in enumerate(kinds)}
    order = sorted(range(len(ents)), key=lambda i: ents[i].config_id)
    id_rank = np.empty(len(ents), dtype=np.int64)
    for r, i in enumerate(order):
        id_rank[i] = r
    gk = list(global_kinds) if global_kinds is not None else list(scenario.backend_kinds())
    gpos = {k: i for i, k in enumerate(gk)}
    # reference config (pipeline.py:478-500)
    cands = [e for e in spec.entries if e.backend_kind == "cpu" and e.batch_size == 1]
    ref_index = -1
    if cands:
        ref = min(cands, key=lambda e: (e.resource_request,
                                        tuple(sorted((k, str(v)) for k, v in e.knob_values.items())),
                                        e.config_id))
        ids = [e.config_id for e in ents]
        if ref.config_id in ids:
            ref_index = ids.index(ref.config_id)
    return Arrays(
        lat=np.array([e.latency_s for e in ents], dtype=np.float64),
        res=np.array([e.resource_request for e in ents], dtype=np.float64),
        batch=np.array([e.batch_size for e in ents], dtype=np.float64),
        batch_int=np.array([e.batch_size for e in ents], dtype=np.int64),
        pool=np.array([scenario.backend(e.backend_kind).pool_resources for e in ents], dtype=np.float64),
        price=np.array([scenario.backend(e.backend_kind).price_rate for e in ents], dtype=np.float64),
        kind_idx=np.array([kpos[e.backend_kind] for e in ents], dtype=np.int64),
        id_rank=id_rank, kinds=kinds,
        gkind=np.array([gpos[e.backend_kind] for e in ents], dtype=np.int64),
        ref_index=ref_index,
        lat_init=np.array([e.latency_initial_s for e in ents], dtype=np.float64),
    )


def from_columns(*, lat, res, batch, pool, price, gkind, id_rank, n_kinds: int,
                 ref_index: int = -1, lat_init=None) -> Arrays:
    """Raw SoA columns with kinds given as global indices 0..n_kinds-1."""
    gkind = np.asarray(gkind, dtype=np.int64)
    present = sorted(set(int(k) for k in gkind))
    kpos = {k: i for i, k in enumerate(present)}
    b = np.asarray(batch, dtype=np.int64)
    lat = np.asarray(lat, dtype=np.float64)
    return Arrays(
        lat=lat.copy(), res=np.asarray(res, dtype=np.float64), batch=b.astype(np.float64),
        batch_int=b, pool=np.asarray(pool, dtype=np.float64),
        price=np.asarray(price, dtype=np.float64),
        kind_idx=np.array([kpos[int(k)] for k in gkind], dtype=np.int64),
        id_rank=np.asarray(id_rank, dtype=np.int64), kinds=present, gkind=gkind,
        ref_index=int(ref_index),
        lat_init=(lat.copy() if lat_init is None else np.asarray(lat_init, dtype=np.float64)),
    )


def scores(t: Arrays, slack_vec_by_table_kind: np.ndarray, alpha: float):
    """configurator.py:219-227; slack indexed by the table's own kind positions."""
    slack_arr = slack_vec_by_table_kind[t.kind_idx]
    cost = (t.res * t.lat) * t.price / t.batch
    penalty = alpha * ((t.lat * t.res) / (t.batch * t.pool))
    score = cost + np.where(t.lat < slack_arr, 0.0, penalty)
    return score, cost


def argmin(t: Arrays, score: np.ndarray, cost: np.ndarray, mask: np.ndarray) -> int:
    """configurator.py:229-237 — masked min, exact ties by (cost, res, id_rank)."""
    masked = np.where(mask, score, np.inf)
    best = masked.min()
    ties = np.flatnonzero(masked == best)
    if len(ties) == 1:
        return int(ties[0])
    return int(min(ties, key=lambda i: (cost[i], t.res[i], t.id_rank[i])))


def table_slack(t: Arrays, slack_global: np.ndarray) -> np.ndarray:
    """slack_by_kind as the table's per-kind vector (configurator.py:215-217)."""
    return np.asarray(slack_global, dtype=np.float64)[t.kind_global]


def select(t: Arrays, slack_global: np.ndarray, alpha: float, available: int, *,
           allow_delay: bool, upstream_supply: int = 0, excluded_mask: int = 0,
           min_batch: int = 1):
    """configurator.py:239-300.  Returns (code, idx, fill, objective, slack_s, wait, feasible)
    with code NONE / ASSIGN / DELAY; slack_global is indexed by global kind."""
    sv = table_slack(t, slack_global)
    n = len(t.lat)
    mask = np.ones(n, dtype=bool)
    if excluded_mask:
        keep = np.array([not ((excluded_mask >> int(g)) & 1) for g in t.kind_global], dtype=bool)
        mask &= keep[t.kind_idx]
    if min_batch > 1:
        mask &= t.batch_int >= min_batch
    if not mask.any():
        return (NONE, -1, 0, 0.0, 0.0, 0.0, False)
    score, cost = scores(t, sv, alpha)
    i = argmin(t, score, cost, mask)
    B = int(t.batch_int[i])
    s_k = float(sv[t.kind_idx[i]])
    if allow_delay and B > available and upstream_supply >= B - available:
        wait = s_k - float(t.lat[i])
        if wait > 0.0:
            return (DELAY, i, int(available), float(score[i]), s_k, wait, bool(t.lat[i] < s_k))
    if B > available:
        mask2 = mask & (t.batch_int <= available)
        if mask2.any():
            i = argmin(t, score, cost, mask2)
    B = int(t.batch_int[i])
    s_k = float(sv[t.kind_idx[i]])
    return (ASSIGN, i, min(B, int(available)), float(score[i]), s_k, 0.0, bool(t.lat[i] < s_k))


def kind_minima(t: Arrays, slack_global: np.ndarray, alpha: float, n_kinds: int) -> np.ndarray:
    """Per global kind, the unmasked min score (+inf if absent) — Eq. 3 operands."""
    score, _ = scores(t, table_slack(t, slack_global), alpha)
    out = np.full(n_kinds, np.inf)
    for k in range(n_kinds):
        on = t.gkind == k
        if on.any():
            out[k] = score[on].min()
    return out


def affinity(t: Arrays, kind_global: int, slack_global: np.ndarray, alpha: float):
    """configurator.py:302-318 (kind given as a global index)."""
    on = t.gkind == kind_global
    if not on.any():
        return None
    if on.all():
        return float("inf")
    score, _ = scores(t, table_slack(t, slack_global), alpha)
    return float(score[~on].min() / score[on].min())


# ---- batched driver (per-invocation loop, like the reference engine) --------------------

def select_many(tables: Sequence[Arrays], slack: np.ndarray, alpha: float, avail, supply,
                min_batch, flags, op=None, start: int = 0, stop: int | None = None):
    """Loop ``select`` over invocations [start, stop); returns SoA result arrays."""
    N = slack.shape[0]
    stop = N if stop is None else stop
    n = stop - start
    out = {
        "code": np.zeros(n, np.int32), "idx": np.full(n, -1, np.int32),
        "fill": np.zeros(n, np.int32), "obj": np.zeros(n), "slack": np.zeros(n),
        "wait": np.zeros(n), "feasible": np.zeros(n, bool),
    }
    for j, i in enumerate(range(start, stop)):
        t = tables[0 if op is None else int(op[i])]
        f = int(flags[i])
        r = select(t, slack[i], alpha, int(avail[i]), allow_delay=bool(f & 1),
                   upstream_supply=int(supply[i]), excluded_mask=(f >> 8) & 0xFFFFFF,
                   min_batch=int(min_batch[i]))
        (out["code"][j], out["idx"][j], out["fill"][j], out["obj"][j], out["slack"][j],
         out["wait"][j], out["feasible"][j]) = r
    return out


_POOL_STATE: dict = {}


def _pool_init(tables, slack, alpha, avail, supply, min_batch, flags, op):
    _POOL_STATE.update(tables=tables, slack=slack, alpha=alpha, avail=avail, supply=supply,
                       min_batch=min_batch, flags=flags, op=op)


def _pool_run(rng):
    s = _POOL_STATE
    return select_many(s["tables"], s["slack"], s["alpha"], s["avail"], s["supply"],
                       s["min_batch"], s["flags"], s["op"], rng[0], rng[1])


def select_many_parallel(tables, slack, alpha, avail, supply, min_batch, flags, op=None,
                         processes: int | None = None):
    """All host cores: contiguous invocation shards over a fork pool."""
    import multiprocessing as mp

    procs = processes or os.cpu_count() or 1
    N = slack.shape[0]
    bounds = np.linspace(0, N, procs + 1).astype(int)
    ranges = [(int(bounds[i]), int(bounds[i + 1])) for i in range(procs) if bounds[i + 1] > bounds[i]]
    ctx = mp.get_context("fork")
    with ctx.Pool(len(ranges), initializer=_pool_init,
                  initargs=(tables, slack, alpha, avail, supply, min_batch, flags, op)) as pool:
        parts = pool.map(_pool_run, ranges)
    return {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}


_POOL_TABLES: dict = {}


def _pool_tables(tables):
    _POOL_TABLES["tables"] = tables


def _pool_ready(_):
    return os.getpid()


def _pool_chunk(a):
    slack, alpha, avail, supply, min_batch, flags, op = a
    return select_many(_POOL_TABLES["tables"], slack, alpha, avail, supply, min_batch, flags, op)


class SelectPool:
    """A persistent fork pool over all host cores holding the tables: forked and warmed once, so
    timed calls pay only the per-call shipping of their (small) invocation shards, not process
    start-up (used by bench.py's CPU baseline and reference arm)."""

    def __init__(self, tables, processes: int | None = None):
        import multiprocessing as mp

        self.procs = processes or os.cpu_count() or 1
        self.pool = mp.get_context("fork").Pool(self.procs, initializer=_pool_tables, initargs=(tables,))
        self.pool.map(_pool_ready, range(4 * self.procs), chunksize=1)

    def select(self, slack, alpha, avail, supply, min_batch, flags, op=None):
        N = slack.shape[0]
        b = np.linspace(0, N, self.procs + 1).astype(int)
        jobs = [(slack[b[i]:b[i + 1]], alpha, avail[b[i]:b[i + 1]], supply[b[i]:b[i + 1]],
                 min_batch[b[i]:b[i + 1]], flags[b[i]:b[i + 1]], None if op is None else op[b[i]:b[i + 1]])
                for i in range(self.procs) if b[i + 1] > b[i]]
        parts = self.pool.map(_pool_chunk, jobs, chunksize=1)
        return {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}

    def close(self):
        self.pool.close()
        self.pool.join()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
