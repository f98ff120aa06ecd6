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
