"""Percentile estimate of an observation batch (sp_observation_quantiles, an extension of K3:
the reference has no percentile, so parity is pinned to numpy's inverted_cdf quantile)."""
from __future__ import annotations

import numpy as np
import pytest


def _batch(seed, sizes, n):
    rng = np.random.default_rng(seed)
    op = rng.integers(0, len(sizes), size=n).astype(np.int32)
    idx = np.array([rng.integers(0, sizes[t]) for t in op], dtype=np.int32)
    hot = rng.random(n) < 0.3  # a few hot entries with long runs
    idx[hot] = 0
    idx[rng.random(n) < 0.05] = -1
    obs = np.exp(rng.normal(0.0, 0.5, size=n)) * (1 + (idx % 7))
    obs[::97] = obs[1]  # ties
    return op, idx, obs


@pytest.mark.parametrize("q", [0.0, 0.05, 0.5, 0.95, 1.0, 1 / 3])
def test_oracle_matches_definition(q):
    from oracle import quantile as oq

    sizes = [50, 7]
    op, idx, obs = _batch(3, sizes, 3000)
    out, cnt = oq.batch_quantiles(sizes, op, idx, obs, q)
    base = [0, 50]
    for g in range(57):
        t = 0 if g < 50 else 1
        vals = [obs[j] for j in range(len(idx)) if idx[j] >= 0 and op[j] == t and base[t] + idx[j] == g]
        assert cnt[g] == len(vals)
        if vals:
            assert out[g] == oq.order_statistic(vals, q)
        else:
            assert np.isnan(out[g])


@pytest.mark.gpu
@pytest.mark.parametrize("q", [0.0, 0.5, 0.95, 1.0, 1 / 3])
def test_device_quantiles_vs_oracle(gpu_ctx, q):
    import paper_2102_01887_b200 as sp
    from oracle import quantile as oq

    rng = np.random.default_rng(11)
    sizes = [300, 40, 2000]
    tabs = [sp.RawTable(lat=np.ones(m), res=np.ones(m), batch=np.ones(m, np.int32),
                        pool=np.ones(m), price=np.ones(m), K=1) for m in sizes]
    smooth = np.full(sum(sizes), np.nan)
    exp_sm = smooth.copy()
    for b in range(3):
        op, idx, obs = _batch(20 + b, sizes, 70000)
        got = sp.observation_quantiles(tabs, op, idx, obs, q, smooth=smooth, beta=0.25)
        exp, cnt = oq.batch_quantiles(sizes, op, idx, obs, q)
        assert np.array_equal(got["count"], cnt)
        assert np.array_equal(np.isnan(got["quantile"]), np.isnan(exp))
        m = ~np.isnan(exp)
        assert np.array_equal(got["quantile"][m].view(np.uint64), exp[m].view(np.uint64))
        exp_sm = oq.smooth(exp_sm, exp, 0.25)
        assert np.array_equal(np.isnan(smooth), np.isnan(exp_sm))
        m2 = ~np.isnan(exp_sm)
        assert np.array_equal(smooth[m2].view(np.uint64), exp_sm[m2].view(np.uint64))
    # empty batch: every entry NaN / 0
    e = sp.observation_quantiles(tabs, None, np.zeros(0, np.int32), np.zeros(0), 0.5)
    assert np.isnan(e["quantile"]).all() and (e["count"] == 0).all()
    for t in tabs:
        t.close()
