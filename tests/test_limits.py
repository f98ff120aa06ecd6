"""Shapes beyond the staircase plan — non-finite latencies (set through set_latency, as the
reference allows), more than 8 backend kinds, more than 16 batch sizes and more than 32,766
entries — against golden vectors of the unmodified reference (tests/golden/limits_cases.npz,
made by tests/golden/make_golden_limits.py): the numpy oracle on the CPU and the device's
literal scan on the B200, result by result, including the ValueError the reference raises
when NaN scores leave _argmin's tie set empty (configurator.py:229-237)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import golden
from oracle import optable

CASES = ("inf", "nan", "wide")


def _case(d, name):
    t = {k[len(name) + 3:]: v for k, v in d.items() if k.startswith(f"{name}_t_")}
    q = {k[len(name) + 3:]: v for k, v in d.items() if k.startswith(f"{name}_q_")}
    return t, q


def _arrays(t):
    return optable.from_columns(lat=t["lat"], res=t["res"], batch=t["batch"], pool=t["pool"],
                                price=t["price"], gkind=t["gkind"], id_rank=t["id_rank"],
                                n_kinds=int(t["K"]))


def _same(a, b):
    a, b = float(a), float(b)
    return (math.isnan(a) and math.isnan(b)) or np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64)


@pytest.fixture(scope="module")
def lim():
    return golden("limits_cases")


@pytest.mark.parametrize("name", CASES)
def test_numpy_oracle_matches_reference_limits(lim, name):
    t, q = _case(lim, name)
    a = _arrays(t)
    n = len(q["r_code"]) if name != "wide" else 40
    with np.errstate(all="ignore"):
        for i in range(n):
            fl = int(q["flags"][i])
            try:
                r = optable.select(a, q["slack"][i], float(q["alpha"][i]), int(q["avail"][i]),
                                   allow_delay=bool(fl & 1), upstream_supply=int(q["supply"][i]),
                                   excluded_mask=fl >> 8, min_batch=int(q["min_batch"][i]))
                code = r[0]
            except ValueError:
                code, r = 3, None
            assert code == q["r_code"][i], i
            if code in (1, 2):
                assert r[1] == q["r_idx"][i] and r[2] == q["r_fill"][i], i
                assert _same(r[3], q["r_obj"][i]) and _same(r[4], q["r_slack"][i]), i
                assert _same(r[5], q["r_wait"][i]), i


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_literal_scan_matches_reference_limits(gpu_ctx, lim, name):
    import paper_2102_01887_b200 as sp

    t, q = _case(lim, name)
    K = int(t["K"])
    tab = sp.RawTable(lat=t["lat"], res=t["res"], batch=t["batch"], pool=t["pool"],
                      price=t["price"], kind=t["gkind"], id_rank=t["id_rank"], K=K)
    n = len(q["r_code"])
    for alpha in np.unique(q["alpha"]):
        sel = np.flatnonzero(q["alpha"] == alpha)
        for mode in ("auto", "scan"):
            r = sp.select_batch([tab], np.ascontiguousarray(q["slack"][sel]), float(alpha),
                                np.ascontiguousarray(q["avail"][sel], np.int32),
                                upstream_supply=np.ascontiguousarray(q["supply"][sel], np.int32),
                                min_batch=np.ascontiguousarray(q["min_batch"][sel], np.int32),
                                flags=np.ascontiguousarray(q["flags"][sel], np.uint32), mode=mode)
            code = np.asarray(r["code"]) & 3
            assert np.array_equal(code, q["r_code"][sel]), (mode, alpha)
            ok = (q["r_code"][sel] == 1) | (q["r_code"][sel] == 2)
            assert np.array_equal(np.asarray(r["idx"])[ok], q["r_idx"][sel][ok])
            assert np.array_equal(np.asarray(r["fill"])[ok], q["r_fill"][sel][ok])
            for k in ("obj", "slack", "wait"):
                got, exp = np.asarray(r[k])[ok], q[f"r_{k}"][sel][ok]
                assert all(_same(x, y) for x, y in zip(got, exp)), k
    # affinity (configurator.py:302-318): NaN propagates through numpy's min
    qk = np.ascontiguousarray(q["aff_kind"], np.int32)
    for alpha in np.unique(q["aff_alpha"]):
        sel = np.flatnonzero(q["aff_alpha"] == alpha)
        out = np.empty(len(sel))
        from paper_2102_01887_b200 import _lib
        import ctypes as C

        arr = (C.c_void_p * 1)(tab.handle.value)
        s_in = np.ascontiguousarray(q["aff_slack"][sel])  # kept alive across the call
        q_in = np.ascontiguousarray(qk[sel])
        _lib.check(tab._ctx.lib.sp_affinity_batch(
            tab._ctx.handle, 1, C.cast(arr, C.c_void_p), float(alpha), len(sel), None,
            _lib.ptr(s_in), _lib.ptr(q_in), _lib.ptr(out), _lib.MODES["auto"]))
        bad = [j for j, (x, y) in enumerate(zip(out, q["aff_out"][sel])) if not _same(x, y)]
        assert not bad, (name, len(bad), bad[:4], out[bad[:4]].tolist(), q["aff_out"][sel][bad[:4]].tolist(),
                         qk[sel][bad[:4]].tolist())
    tab.close()


@pytest.mark.gpu
def test_object_api_raises_like_the_reference(gpu_ctx, lim):
    """OpTable.select raises ValueError exactly where the reference's _argmin does."""
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    spec = synth.synth_spec(False)
    t = sp.OpTable(spec, synth.synth_scenario())
    t.set_latency(5, math.nan)  # a cpu entry: every unmasked cpu score involving it is NaN
    with pytest.raises(ValueError):
        t.select({"cpu": 1.0, "gpu": 1.0}, 100.0, 8, allow_delay=False)
    # with the cpu kind excluded the NaN entry is masked out and the decision is normal
    d = t.select({"cpu": 1.0, "gpu": 1.0}, 100.0, 8, allow_delay=False,
                 excluded_kinds=frozenset({"cpu"}))
    assert d is not None and d.entry.backend_kind == "gpu"
    t.set_latency(5, math.inf)
    assert t.select({"cpu": 1.0, "gpu": 1.0}, 100.0, 8, allow_delay=False) is not None
    t.close()
