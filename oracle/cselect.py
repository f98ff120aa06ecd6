"""ctypes loader for select_oracle.c — TEST ORACLE ONLY.

``build()`` compiles the C restatement into oracle/_build/liboracle_select.so (git-ignored,
travels to the GPU box with gpurun).  ``select_batch`` mirrors the batched API of the
product so tests can compare arrays directly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "select_oracle.c"
OUT = HERE / "_build" / "liboracle_select.so"

_lib = None


def build(force: bool = False) -> Path:
    if OUT.exists() and not force and OUT.stat().st_mtime >= SRC.stat().st_mtime:
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
           "-o", str(OUT), str(SRC), "-lm"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return OUT


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(OUT))
        _lib.oracle_select_batch.restype = C.c_int
    return _lib


def _p(a):
    return C.c_void_p(0) if a is None else C.c_void_p(a.ctypes.data)


def select_batch(tables, slack, alpha, avail, supply, min_batch, flags, op=None, threads=None):
    """tables: sequence of oracle.optable.Arrays (gkind = global kind index)."""
    lib = _load()
    if threads is not None:
        os.environ["OMP_NUM_THREADS"] = str(threads)
    off = np.zeros(len(tables) + 1, dtype=np.int64)
    for t, a in enumerate(tables):
        off[t + 1] = off[t] + len(a.lat)
    cat = lambda name, dt: np.ascontiguousarray(np.concatenate([getattr(a, name) for a in tables]), dtype=dt)
    lat, res = cat("lat", np.float64), cat("res", np.float64)
    batch, pool, price = cat("batch_int", np.int64), cat("pool", np.float64), cat("price", np.float64)
    gkind, idr = cat("gkind", np.int64), cat("id_rank", np.int64)
    slack = np.ascontiguousarray(slack, dtype=np.float64)
    N, K = slack.shape
    avail = np.ascontiguousarray(avail, dtype=np.int32)
    supply = np.ascontiguousarray(supply, dtype=np.int32)
    min_batch = np.ascontiguousarray(min_batch, dtype=np.int32)
    flags = np.ascontiguousarray(flags, dtype=np.uint32)
    opa = None if op is None else np.ascontiguousarray(op, dtype=np.int32)
    out = {
        "code": np.empty(N, np.int32), "idx": np.empty(N, np.int32), "fill": np.empty(N, np.int32),
        "obj": np.empty(N), "slack": np.empty(N), "wait": np.empty(N), "feasible": np.empty(N, np.uint8),
    }
    max_m = int(max(len(a.lat) for a in tables))
    lib.oracle_select_batch(
        _p(off), _p(lat), _p(res), _p(batch), _p(pool), _p(price), _p(gkind), _p(idr),
        C.c_int(K), C.c_double(float(alpha)), C.c_int64(N), _p(opa), _p(slack), _p(avail),
        _p(supply), _p(min_batch), _p(flags), _p(out["code"]), _p(out["idx"]), _p(out["fill"]),
        _p(out["obj"]), _p(out["slack"]), _p(out["wait"]), _p(out["feasible"]), C.c_int64(max_m))
    out["feasible"] = out["feasible"].astype(bool)
    return out


def _sig(lib):
    lib.oracle_slack_paths.restype = C.c_int
    lib.oracle_slack_dp.restype = C.c_int
    lib.oracle_fold.restype = C.c_int


def slack_paths(ref, target, now, Q, paths_cols):
    """Alg. 1 over an explicit path list (configurator.py:415-417, 493-543) for I instances.
    ref (I, V) by column; paths_cols: sequences of columns.  Returns slack (I, V, K)."""
    lib = _load()
    _sig(lib)
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    I, V = ref.shape
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    K = Q.shape[1]
    off = np.zeros(len(paths_cols) + 1, dtype=np.int32)
    for p, cols in enumerate(paths_cols):
        off[p + 1] = off[p] + len(cols)
    nodes = np.ascontiguousarray(np.concatenate([np.asarray(c, dtype=np.int32) for c in paths_cols]))
    target = np.ascontiguousarray(target, dtype=np.float64)
    now = np.ascontiguousarray(now, dtype=np.float64)
    out = np.empty((I, V, K))
    lib.oracle_slack_paths(C.c_int64(I), C.c_int(V), C.c_int(K), _p(ref), _p(target), _p(now),
                           _p(Q), C.c_int(len(paths_cols)), _p(off), _p(nodes), _p(out))
    return out


def slack_dp(dag, ref, target, now, Q, ratios=False):
    """Forward-DP Alg. 1 (oracle/slack.py dp_ratios / dp_slack) for a PipelineDag whose path set
    cannot be enumerated.  ref (I, V) in dag.vertices column order.  Returns slack (I, V, K)
    (and ratio (I, V, 2) = (own/Tmax, own/Tmin) when ratios=True)."""
    lib = _load()
    _sig(lib)
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    I, V = ref.shape
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    K = Q.shape[1]
    order = dag.topological_order()
    pos = {v: i for i, v in enumerate(order)}
    col = np.array([dag.vertices.index(v) for v in order], dtype=np.int32)
    preds = [[pos[p] for p in dag.predecessors(v)] for v in order]
    poff = np.zeros(V + 1, dtype=np.int32)
    for s, ps in enumerate(preds):
        poff[s + 1] = poff[s] + len(ps)
    pidx = np.array([p for ps in preds for p in ps], dtype=np.int32)
    term = np.array([not dag.successors(v) for v in order], dtype=np.uint8)
    out = np.empty((I, V, K))
    rat = np.empty((I, V, 2)) if ratios else None
    lib.oracle_slack_dp(C.c_int64(I), C.c_int(V), C.c_int(K), _p(ref),
                        _p(np.ascontiguousarray(target, dtype=np.float64)),
                        _p(np.ascontiguousarray(now, dtype=np.float64)), _p(Q), _p(col), _p(poff),
                        _p(pidx), _p(term), _p(out), _p(rat))
    return (out, rat) if ratios else out


class FoldState:
    """One table's feedback state for oracle_fold (manager.py:436-457)."""

    def __init__(self, lat, lat_init, ref_index):
        self.lat = np.array(lat, dtype=np.float64)
        self.lat_init = np.ascontiguousarray(lat_init, dtype=np.float64)
        self.ref_index = int(ref_index)
        self.completed_ref = np.zeros(1, dtype=np.int64)
        self.obs_count = np.zeros(len(self.lat), dtype=np.int64)


def fold(st: FoldState, idx, obs, beta=0.5, dfp_count=10):
    """Sequential fold of one batch of observations into st (in order)."""
    lib = _load()
    _sig(lib)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    obs = np.ascontiguousarray(obs, dtype=np.float64)
    rc = lib.oracle_fold(C.c_int64(len(st.lat)), _p(st.lat), _p(st.lat_init), C.c_int64(st.ref_index),
                         _p(st.completed_ref), _p(st.obs_count), C.c_int64(len(idx)), _p(idx), _p(obs),
                         C.c_double(beta), C.c_int64(dfp_count))
    if rc != 0:
        raise ValueError("observation index out of range")
    return st
