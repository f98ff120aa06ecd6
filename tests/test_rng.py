"""sp_des_draws (host C: PCG64 + numpy's ziggurat tables) against the reference's own draw loop
(numpy Generator + CPython math.exp, backend.py:52-57, 186) — bit-identical per start, for every
draw pattern the scenarios produce.  CPU only (the draw generator is host code)."""
from __future__ import annotations

import math

import numpy as np
import pytest


def _python_draws(seed, cap, sig, sr, fr):
    rng = np.random.default_rng(seed)
    fac = np.ones(cap)
    bits = np.zeros(cap, np.uint8)
    for k in range(cap):
        if sig > 0.0:
            fac[k] = math.exp(rng.normal(0.0, sig))
        b = 0
        if sr > 0.0 and rng.random() < sr:
            b |= 1
        if fr > 0.0 and rng.random() < fr:
            b |= 2
        bits[k] = b
    return fac, bits


@pytest.mark.parametrize("sig,sr,fr", [(0.3, 0.0, 0.0), (0.2, 0.05, 0.1), (0.0, 0.1, 0.0),
                                       (0.0, 0.0, 0.5), (1.5, 0.5, 0.5)])
def test_draws_match_numpy(sig, sr, fr):
    from paper_2102_01887_b200.engine import RunSpec

    class _Spec:  # only the draw parameters of a RunSpec
        noise_sigma, straggle_rate, failure_rate = sig, sr, fr
        draws = (1 if sig > 0 else 0) | (2 if sr > 0 else 0) | (4 if fr > 0 else 0)

    seeds = [0, 7, 12345, 2**40 + 3]
    cap = 30000  # >= 0.3 % ziggurat slow paths per normal: both rare branches are exercised
    fac, bits = RunSpec.draws_for(_Spec(), seeds, cap)
    for i, s in enumerate(seeds):
        f, b = _python_draws(s, cap, sig, sr, fr)
        if fac is not None:
            assert np.array_equal(fac[i].view(np.uint64), f.view(np.uint64)), s
        if bits is not None:
            assert np.array_equal(bits[i], b), s


def test_normals_incl_tail_match_numpy():
    """A long normal stream (the ziggurat's idx == 0 tail and the wedge rejections included)."""
    from paper_2102_01887_b200.engine import RunSpec

    class _Spec:
        noise_sigma, straggle_rate, failure_rate, draws = 1.0, 0.0, 0.0, 1

    cap = 400000
    fac, _ = RunSpec.draws_for(_Spec(), [99], cap)
    z = np.random.default_rng(99).normal(0.0, 1.0, size=cap)
    exp = np.fromiter(map(math.exp, z.tolist()), dtype=np.float64, count=cap)
    assert np.array_equal(fac[0].view(np.uint64), exp.view(np.uint64))
    assert (np.abs(z) > 3.6541528853610088).sum() > 50  # the tail branch ran
