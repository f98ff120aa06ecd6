"""Golden vectors for the shapes the staircase plan does not cover, produced by the UNMODIFIED
reference (run in the build container: python tests/golden/make_golden_limits.py).

* "inf" / "nan": tables whose latencies were set to +inf / -inf (alpha in {0, 1, 100, inf}) or
  NaN through OpTable.set_latency (configurator.py:211-213 accepts any float): every select's
  result — including the ValueError that NaN scores raise in _argmin (configurator.py:229-237)
  — and every affinity ratio (configurator.py:302-318).
* "wide": K = 10 backend kinds, M = 40,000 entries, 32 distinct batch sizes (beyond the plan's 8
  kinds / 16 batch sizes / 32,766 entries): selects and affinities at alpha 100.

Writes tests/golden/limits_cases.npz.  Result code per select: 0 None, 1 assign, 2 delay,
3 ValueError.
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from slackpipe.configurator import OpTable  # noqa: E402
from slackpipe.pipeline import ConfigEntry, ConfigSpec  # noqa: E402
from slackpipe.scenario import BackendSpec, GroundTruthModel, Scenario  # noqa: E402

OUT = Path(__file__).resolve().parent / "limits_cases.npz"


def make_case(rng, M, K, nB, n_sel, n_aff, alphas, nonfinite):
    kinds = ["cpu"] + [f"k{i:02d}" for i in range(1, K)]
    backends = tuple(BackendSpec(k, int(rng.integers(2, 12)), int(rng.choice([8, 64, 4096])),
                                 float(rng.choice([1e-5, 3e-5, 2.5e-4]))) for k in kinds)
    sc = Scenario("limits", backends, GroundTruthModel(per_op={}))
    bvals = np.sort(rng.choice(np.arange(1, 400), size=nB, replace=False))
    bvals[0] = 1
    lat_pool = rng.uniform(0.01, 5.0, size=max(3, M // 8))
    ents = []
    for j in range(M):
        k = kinds[int(rng.integers(0, K))] if j else "cpu"
        b = int(bvals[0]) if j == 0 else int(rng.choice(bvals))
        inst = next(x for x in backends if x.kind == k).resources_per_instance
        r = int(rng.integers(1, inst + 1))
        lat = float(rng.choice(lat_pool)) if rng.random() < 0.5 else float(rng.uniform(0.01, 5.0))
        ents.append(ConfigEntry(f"{k}-r{r}-b{b}-i={j}", k, {"i": j}, b, r, lat, lat))
    spec = ConfigSpec("op", ents, ents[0].config_id)
    t = OpTable(spec, sc)
    if nonfinite == "inf":
        for j in rng.choice(np.arange(1, M), size=max(3, M // 10), replace=False):
            t.set_latency(int(j), float(rng.choice([math.inf, -math.inf])))
    elif nonfinite == "nan":  # two NaN latencies on one kind (excluded by a third of the queries)
        on = [j for j in range(1, M) if t.kind_idx[j] == t.kinds.index(kinds[-1])]
        for j in on[:2]:
            t.set_latency(int(j), math.nan)
    g = {k: i for i, k in enumerate(kinds)}
    tab = {
        "lat": t.lat.copy(), "res": t.res.copy(), "batch": t.batch_int.copy(), "pool": t.pool.copy(),
        "price": t.price.copy(), "gkind": np.array([g[t.kinds[i]] for i in t.kind_idx]),
        "id_rank": t.id_rank.copy(), "K": K,
    }
    q = {"slack": [], "alpha": [], "avail": [], "supply": [], "min_batch": [], "flags": [],
         "r_code": [], "r_idx": [], "r_fill": [], "r_obj": [], "r_slack": [], "r_wait": [],
         "aff_kind": [], "aff_slack": [], "aff_alpha": [], "aff_out": []}
    for i in range(n_sel):
        s = rng.uniform(-2.0, 6.0, size=K)
        u = rng.random(K)
        s[u < 0.08] = math.inf
        pick = u > 0.9
        s[pick] = rng.choice(t.lat[np.isfinite(t.lat)], size=int(pick.sum()))
        sbk = {k: float(s[g[k]]) for k in kinds}
        a = float(alphas[i % len(alphas)])
        av = int(rng.integers(0, 420))
        sup = int(rng.integers(0, 420))
        mb = 1 if rng.random() < 0.7 else int(rng.integers(1, 420))
        excl = int(rng.integers(0, 1 << K)) if rng.random() < 0.3 else 0
        if nonfinite == "nan" and rng.random() < 0.35:
            excl |= 1 << (K - 1)
        ad = bool(rng.random() < 0.5)
        ex = frozenset(k for k in kinds if (excl >> g[k]) & 1)
        try:
            d = t.select(sbk, a, av, allow_delay=ad, upstream_supply=sup, excluded_kinds=ex,
                         min_batch=mb)
            if d is None:
                res = (0, -1, 0, 0.0, 0.0, 0.0)
            else:
                res = (2 if d.kind == "delay" else 1, d.entry_index, d.fill, d.objective_value,
                       d.slack_s, d.wait_budget_s)
        except ValueError:
            res = (3, -1, 0, 0.0, 0.0, 0.0)
        q["slack"].append(s)
        q["alpha"].append(a)
        q["avail"].append(av)
        q["supply"].append(sup)
        q["min_batch"].append(mb)
        q["flags"].append(int(ad) | (excl << 8))
        for key, v in zip(("r_code", "r_idx", "r_fill", "r_obj", "r_slack", "r_wait"), res):
            q[key].append(v)
    with np.errstate(all="ignore"):
        for i in range(n_aff):
            s = rng.uniform(-2.0, 6.0, size=K)
            s[rng.random(K) < 0.08] = math.inf
            sbk = {k: float(s[g[k]]) for k in kinds}
            a = float(alphas[i % len(alphas)])
            kq = kinds[int(rng.integers(0, K))]
            r = t.affinity(kq, sbk, a)
            q["aff_kind"].append(g[kq])
            q["aff_slack"].append(s)
            q["aff_alpha"].append(a)
            q["aff_out"].append(math.nan if r is None else r)
            q.setdefault("aff_none", []).append(r is None)
    return tab, {k: np.array(v) for k, v in q.items()}


def main():
    rng = np.random.default_rng(20261017)
    out = {}
    cases = {"inf": dict(M=150, K=3, nB=5, n_sel=1200, n_aff=300,
                         alphas=(0.0, 1.0, 100.0, math.inf), nonfinite="inf"),
             "nan": dict(M=120, K=3, nB=4, n_sel=600, n_aff=150, alphas=(0.0, 100.0),
                         nonfinite="nan"),
             "wide": dict(M=40000, K=10, nB=32, n_sel=200, n_aff=60, alphas=(100.0,),
                          nonfinite=None)}
    for name, kw in cases.items():
        with np.errstate(all="ignore"):
            tab, q = make_case(rng, **kw)
        for k, v in tab.items():
            out[f"{name}_t_{k}"] = np.asarray(v)
        for k, v in q.items():
            out[f"{name}_q_{k}"] = v
        codes = np.bincount(q["r_code"], minlength=4)
        print(name, "select codes (none, assign, delay, error):", codes.tolist(),
              "affinity None/NaN:", int(q["aff_none"].sum()), int(np.isnan(q["aff_out"]).sum()))
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
