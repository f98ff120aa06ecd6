"""Golden runs of the reference engine for the replica-parallel run engine.

    python tests/golden/make_golden_des.py [--ref /root/reference/pkg/src]

Runs the UNMODIFIED reference `PipelineRun.run_to_completion` (manager.py:535-630), built the
way its CLI builds a run (cli.py:193-222: profiles through MetadataStore, decomposed paths,
fault overrides), on the three bundled scenarios and on config-4 replicas (SURVEY.md §8(d):
`generate_trace(3000, 17 + r, {"cars": 0.6, "persons": 0.8}, 3)` at m x 90.41885182994682 s),
and records per run the decision log (row count + sha256 of its rows in repr form), the backend's
event trace (BackendSim.trace, same digest), the report (CSV row and fields) and the final latency
tables (sha256).  The bundle inputs (pipeline,
scenario, trace) and the profiles the reference's MetadataStore wrote are copied next to it so
the GPU box, which has no /root/reference, can rebuild every run.  Output: tests/golden/des/.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import shutil
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = HERE / "des"
BUNDLES = Path("/root/reference/pkg/scenarios")
CP_MIN = 90.41885182994682  # the fast-anchor latency
T_AMBER = [0.0, float("inf"), 116.30975052233568, 142.20064921472454, 168.09154790711338]


def log_digest(rows) -> str:
    h = hashlib.sha256()
    for r in rows:
        h.update("\t".join(repr(float(x)) if isinstance(x, float) else str(x) for x in r).encode())
        h.update(b"\n")
    return h.hexdigest()


def lat_digest(arrs) -> str:
    return hashlib.sha256(b"".join(np.ascontiguousarray(a, dtype=np.float64).tobytes() for a in arrs)).hexdigest()


def cases():
    out = []
    for t in T_AMBER:
        out.append(dict(bundle="branching", target=t))
    t50 = T_AMBER[3]
    for ab in (["fb"], ["dfp"], ["sdb"], ["eslc"], ["pbc"], ["eslc", "pbc"], ["fb", "sdb"]):
        out.append(dict(bundle="branching", target=t50, ablations=ab))
    out.append(dict(bundle="branching", target=t50, noise_sigma=0.3))
    out.append(dict(bundle="branching", target=t50, noise_sigma=0.3, seed=7))
    out.append(dict(bundle="branching", target=t50, failure_rate=0.03))
    out.append(dict(bundle="branching", target=T_AMBER[2], noise_sigma=0.3, failure_rate=0.05))
    out.append(dict(bundle="branching", target=t50, straggle_rate=0.05, straggle_factor=4.0))
    out.append(dict(bundle="branching", target=t50, noise_sigma=0.2, straggle_rate=0.02,
                    straggle_factor=3.0, failure_rate=0.02, ablations=["eslc"]))
    out.append(dict(bundle="branching", target=t50, profile_scale=1.7))
    out.append(dict(bundle="branching", target=t50, profile_scale=0.6, alpha=1.0))
    for t in (0.0, float("inf"), 30.0, 60.0):
        out.append(dict(bundle="parallel", target=t))
    out.append(dict(bundle="parallel", target=60.0, noise_sigma=0.2, failure_rate=0.1))
    out.append(dict(bundle="parallel", target=45.0, straggle_rate=0.1, straggle_factor=5.0))
    for t in (0.0, 60.0):
        out.append(dict(bundle="overhead", target=t))
    out.append(dict(bundle="overhead", target=60.0, noise_sigma=0.2, failure_rate=0.1))
    for r in range(8):
        for m in (0.5, 1.0, 2.0, 5.0, 10.0):
            out.append(dict(bundle="branching", target=m * CP_MIN,
                            trace=dict(count=3000, seed=17 + r, rates={"cars": 0.6, "persons": 0.8},
                                       max=3), group="c4"))
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from slackpipe import cli, manager, pipeline, profiler, workload
    from slackpipe import scenario as scn

    OUT.mkdir(parents=True, exist_ok=True)
    built = {}
    for b in ("branching", "parallel", "overhead"):
        dst = OUT / b
        if dst.exists():
            shutil.rmtree(dst)
        dst.mkdir(parents=True)
        shutil.copy(BUNDLES / b / "pipeline.json", dst / "pipeline.json")
        shutil.copy(BUNDLES / b / "scenario.json", dst / "scenario.json")
        frames = workload.load_trace(str(BUNDLES / b / "trace.jsonl"))
        names = sorted({k for _, a in frames for k in a})
        np.savez_compressed(dst / "trace.npz", frame_id=np.array([f for f, _ in frames], np.int64),
                            names=np.array(names),
                            attrs=np.array([[a.get(k, 0) for k in names] for _, a in frames], np.int64))
        doc = json.load(open(BUNDLES / b / "pipeline.json"))
        dag, ops = pipeline.load_pipeline(doc)
        sc = scn.load_scenario(str(BUNDLES / b / "scenario.json"))
        md = dst / "metadata"
        store = profiler.MetadataStore(str(md))
        profiles, _ = cli._ensure_profiles(store, ops, sc, sc.tuning.samples_per_config)
        paths = cli._paths_for(store, doc, dag)
        built[b] = (doc, dag, ops, sc, profiles, paths, frames)

    runs = []
    t0 = time.time()
    for c in cases():
        doc, dag, ops, sc, profiles, paths, frames = built[c["bundle"]]
        if "trace" in c:
            tr = c["trace"]
            frames = workload.generate_trace(tr["count"], tr["seed"], tr["rates"], tr["max"])
        rs = sc.with_fault_overrides(noise_sigma=c.get("noise_sigma"), failure_rate=c.get("failure_rate"),
                                     straggle_rate=c.get("straggle_rate"),
                                     straggle_factor=c.get("straggle_factor"))
        tp = cli._tuning_params(rs, c.get("alpha"))
        run = manager.PipelineRun(dag, ops, profiles, frames, rs, c["target"], tp,
                                  ablations=frozenset(c.get("ablations", [])), seed=c.get("seed"),
                                  paths=paths, profile_scale=c.get("profile_scale", 1.0),
                                  pipeline_name=doc.get("name", "pipeline"))
        rep = run.run_to_completion()
        rows = run.configurator.decision_log
        c = dict(c)
        c["target"] = repr(float(c["target"]))
        c["expect"] = dict(
            log_rows=len(rows), log_sha256=log_digest(rows), csv_row=rep.csv_row(),
            latency_s=repr(rep.latency_s), cost=repr(float(rep.cost)), slack_met_frac=repr(rep.slack_met_frac),
            configs_used=rep.configs_used, failures=rep.failures, duplicates=rep.duplicates,
            invocations=rep.invocations, completed=rep.completed, terminal_items=rep.terminal_items,
            decision_count=rep.decision_count,
            lat_sha256=lat_digest([run.tables[o].lat for o in sorted(run.tables)]),
            ev_rows=len(run.sim.trace), ev_sha256=log_digest(run.sim.trace),
            first_rows=[[repr(float(x)) if isinstance(x, float) else x for x in r] for r in rows[:8]],
        )
        runs.append(c)
        print(f"{len(runs):3d} {c['bundle']:9s} t={c['target']:>22s} rows={len(rows):6d} "
              f"dups={rep.duplicates} fail={rep.failures} {time.time() - t0:6.1f}s", flush=True)
    with open(OUT / "runs.json", "w", encoding="utf-8") as fh:
        json.dump({"generator": "tests/golden/make_golden_des.py", "runs": runs}, fh, indent=1)


if __name__ == "__main__":
    main()
