"""The CPU restatement of the decision plan (oracle/plan.py) against the reference argmin:
decisions read from the restated plan equal OpTable._argmin (configurator.py:219-237) over
the masked entries (CPU, no GPU needed)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import optable, plan
from paper_2102_01887_b200 import synth


def _tables():
    t2 = optable.from_spec(synth.synth_spec(False), synth.synth_scenario(), ["cpu", "gpu"])
    yield "c2", t2, 2
    rng = np.random.default_rng(5)
    for M, nB, K in ((300, 5, 3), (120, 11, 2), (64, 2, 4)):
        bv = np.sort(rng.choice(np.arange(1, 200), size=nB, replace=False))
        lat = np.where(rng.random(M) < 0.5, rng.choice(rng.uniform(0.01, 3, M // 6), M), rng.uniform(0.01, 3, M))
        gk = rng.integers(0, K, M)
        t = optable.from_columns(lat=lat, res=rng.choice([1.0, 2.0, 4.0], M), batch=rng.choice(bv, M),
                                 pool=rng.choice([16.0, 64.0], K)[gk], price=rng.choice([1e-5, 3e-4], K)[gk],
                                 gkind=gk, id_rank=rng.permutation(M), n_kinds=K)
        yield f"rand{M}", t, K


@pytest.mark.parametrize("alpha", [0.0, 100.0])
def test_plan_restatement_reproduces_reference_argmin(alpha):
    rng = np.random.default_rng(1)
    for name, t, K in _tables():
        img = plan.plan_image(t.lat, t.res, t.batch_int, t.pool, t.price, t.gkind, t.id_rank, K, alpha)
        bvals = img["batch_vals"]
        for _ in range(300):
            s = rng.uniform(-1, 4, size=K)
            s[rng.random(K) < 0.2] = rng.choice(t.lat)
            mb = int(rng.choice(bvals)) if rng.random() < 0.5 else 1
            lane = int(np.searchsorted(bvals, mb))
            score, cost = optable.scores(t, optable.table_slack(t, s), alpha)
            mask = t.batch_int >= mb
            want = optable.argmin(t, score, cost, mask) if mask.any() else None
            got = plan.plan_argmin(img, s, lane)
            if want is None:
                assert got is None, name
            else:
                assert got is not None and got[0] == want, (name, got, want)
                assert got[1] == bool(t.lat[want] < s[t.gkind[want]])
