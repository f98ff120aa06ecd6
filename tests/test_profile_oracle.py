"""The profile-generation oracle (oracle/profile.py) pinned to the unmodified reference's
profile_operation outputs (tests/golden/profile_cases.json) — CPU only."""
from __future__ import annotations

import json

import numpy as np

from conftest import GOLDEN
from oracle import profile as op_oracle


def test_profile_oracle_matches_reference_goldens():
    cases = json.loads((GOLDEN / "profile_cases.json").read_text())
    assert len(cases) == 8
    n = 0
    for case in cases:
        for op in case["ops"]:
            got = np.array(op_oracle.profile_latencies(case, op))
            want = np.array([e[1] for e in op["entries"]])
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (case["name"], op["name"])
            n += len(got)
    assert n == 588


def test_vectorised_normals_are_the_sequential_stream():
    """The device path draws a case's normals in one call when there are no straggles: the same
    values as draw_actual_latency's one-at-a-time draws (backend.py:53-54)."""
    a = np.random.default_rng(12345)
    b = np.random.default_rng(12345)
    seq = np.array([a.normal(0.0, 0.3) for _ in range(5000)])
    vec = b.normal(0.0, 0.3, size=5000)
    assert np.array_equal(seq.view(np.uint64), vec.view(np.uint64))
