"""Randomised parity sweep of the run engine: N random AMBER / join-bundle runs (traces, targets,
ablations, noise / straggle / failure rates, profile scales, seeds) on the device (default
execution form) against oracle/engine.py (the Python restatement of the reference engine, pinned
to the reference) on all host cores.  Compares each run's decision log and event trace (sha256),
cost, latency, invocations, completions and final tables.

    python tools/des_parity_sweep.py [N] > profiles/.../des_parity_sweep.json
"""
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import des_cases as dc  # noqa: E402

ABL = ("fb", "dfp", "sdb", "eslc", "pbc")


def make_case(i):
    rng = np.random.default_rng(1000 + i)
    bundle = "parallel" if i % 4 == 3 else "branching"
    c = {"bundle": bundle, "seed": int(rng.integers(0, 2**31)),
         "ablations": [a for a in ABL if rng.random() < 0.15],
         "profile_scale": float(rng.choice([1.0, 1.0, 0.7, 1.4])),
         "noise_sigma": float(rng.choice([0.0, 0.0, 0.2, 0.35])),
         "failure_rate": float(rng.choice([0.0, 0.0, 0.03, 0.1])),
         "straggle_rate": float(rng.choice([0.0, 0.0, 0.05])), "straggle_factor": 3.0,
         "frames": int(rng.integers(200, 1500)), "trace_seed": int(rng.integers(0, 2**31)),
         "rates": {"cars": float(rng.uniform(0.1, 1.2)), "persons": float(rng.uniform(0.1, 1.2))},
         "target": float(rng.choice([0.0, float("inf"), rng.uniform(10, 200)]))}
    return c


def frames_of(c):
    from paper_2102_01887_b200.engine import generate_trace

    rates = c["rates"] if c["bundle"] == "branching" else {"persons": c["rates"]["persons"]}
    return generate_trace(c["frames"], c["trace_seed"], rates, 4)


def digest(rows):
    return dc.log_digest(rows)


def oracle_run(c):
    from oracle import engine as oe

    doc, dag, sc, profiles, paths, _ = dc.bundle(c["bundle"])
    t = sc.tuning
    eng = oe.Engine(dag, profiles, frames_of(c), sc, c["target"],
                    oe.Params(t.alpha, t.cq_capacity, t.dfp_count, t.straggler_timeout_factor,
                              t.smoothing_beta), ablations=c["ablations"], seed=c["seed"], paths=paths,
                    profile_scale=c["profile_scale"], noise_sigma=c["noise_sigma"],
                    failure_rate=c["failure_rate"], straggle_rate=c["straggle_rate"],
                    straggle_factor=c["straggle_factor"])
    rep = eng.run()
    lat = np.concatenate([eng.t[o].lat for o in eng.ops])
    return (digest(rep.log), repr(float(rep.cost)), repr(float(rep.latency_s)), rep.invocations,
            rep.completed, hashlib.sha256(lat.tobytes()).hexdigest(), len(rep.log))


def main():
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200.engine import ReplicaEngine

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    cases = [make_case(i) for i in range(n)]
    t0 = time.time()
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        want = pool.map(oracle_run, cases)
    t1 = time.time()
    ctx = sp.get_context(0)
    groups = {}
    for i, c in enumerate(cases):
        key = (c["bundle"], tuple(c["ablations"]), c["profile_scale"], c["noise_sigma"],
               c["failure_rate"], c["straggle_rate"])
        groups.setdefault(key, []).append(i)
    bad, runs = [], 0
    for key, idx in groups.items():
        c0 = cases[idx[0]]
        spec = dc.run_spec(dict(bundle=c0["bundle"], ablations=c0["ablations"],
                                profile_scale=c0["profile_scale"], noise_sigma=c0["noise_sigma"],
                                failure_rate=c0["failure_rate"], straggle_rate=c0["straggle_rate"],
                                straggle_factor=c0["straggle_factor"]))
        eng = ReplicaEngine(spec, ctx)
        cap = max(want[i][6] for i in idx) + 16
        res = eng.run([frames_of(cases[i]) for i in idx], [cases[i]["target"] for i in idx],
                      [cases[i]["seed"] for i in idx], log_cap=cap, final_tables=True)
        for i, r in zip(idx, res):
            got = (digest(eng.log_rows(r.log)), repr(r.cost), repr(r.latency_s), r.invocations,
                   r.completed, hashlib.sha256(r.lat.tobytes()).hexdigest(), len(r.log))
            runs += 1
            if got != want[i]:
                bad.append({"case": cases[i], "fields": [k for k, a, b in zip(
                    ("log", "cost", "latency", "invocations", "completed", "tables", "rows"), got, want[i]) if a != b]})
        eng.close()
    t2 = time.time()
    print(json.dumps({"runs": runs, "mismatches": len(bad), "bad": bad[:5],
                      "decision_rows": int(sum(w[6] for w in want)),
                      "oracle_seconds": t1 - t0, "device_seconds_incl_setup": t2 - t1,
                      "cases": "random AMBER (3/4) and join-bundle (1/4) runs: 200-1500 frames, targets "
                               "0 / inf / U(10, 200), each ablation w.p. 0.15, profile scale, noise, "
                               "failure and straggle rates, seeds"}))


if __name__ == "__main__":
    main()
