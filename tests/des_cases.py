"""Rebuild the golden reference runs of tests/golden/des/runs.json with package types (no
reference import: usable on the GPU box).  Shared by the run-engine tests."""
from __future__ import annotations

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

DES = Path(__file__).resolve().parent / "golden" / "des"


def runs() -> list[dict]:
    with open(DES / "runs.json", encoding="utf-8") as fh:
        return json.load(fh)["runs"]


@lru_cache(maxsize=None)
def bundle(name: str):
    from paper_2102_01887_b200 import metadata
    from paper_2102_01887_b200.pipeline import dag_from_json
    from paper_2102_01887_b200.scenario import scenario_from_json

    d = DES / name
    doc = json.load(open(d / "pipeline.json"))
    dag = dag_from_json(doc)
    sc = scenario_from_json(json.load(open(d / "scenario.json")))
    profiles = metadata.load_profiles(d / "metadata", sorted(dag.vertices))
    paths = metadata.load_paths(d / "metadata")
    with np.load(d / "trace.npz") as z:
        names = [str(x) for x in z["names"]]
        frames = [(int(f), {k: int(v) for k, v in zip(names, row)})
                  for f, row in zip(z["frame_id"], z["attrs"])]
    return doc, dag, sc, profiles, paths, frames


def frames_of(case) -> list:
    from paper_2102_01887_b200.engine import generate_trace

    if "trace" in case:
        t = case["trace"]
        return generate_trace(t["count"], t["seed"], t["rates"], t["max"])
    return bundle(case["bundle"])[5]


def spec_key(case) -> tuple:
    """Cases with equal keys share one RunSpec (one launch of many replicas)."""
    return (case["bundle"], tuple(case.get("ablations", [])), case.get("noise_sigma"),
            case.get("failure_rate"), case.get("straggle_rate"), case.get("straggle_factor"),
            case.get("profile_scale", 1.0), case.get("alpha"))


def run_spec(case):
    from paper_2102_01887_b200.engine import RunSpec, TuningParams

    doc, dag, sc, profiles, paths, _ = bundle(case["bundle"])
    t = sc.tuning
    params = TuningParams(alpha=t.alpha if case.get("alpha") is None else case["alpha"],
                          cq_capacity=t.cq_capacity, dfp_count=t.dfp_count,
                          straggler_timeout_factor=t.straggler_timeout_factor,
                          smoothing_beta=t.smoothing_beta)
    return RunSpec(dag, profiles, sc, params, ablations=case.get("ablations", []), paths=paths,
                   profile_scale=case.get("profile_scale", 1.0), noise_sigma=case.get("noise_sigma"),
                   failure_rate=case.get("failure_rate"), straggle_rate=case.get("straggle_rate"),
                   straggle_factor=case.get("straggle_factor"))


def seed_of(case) -> int:
    return case.get("seed") if case.get("seed") is not None else bundle(case["bundle"])[2].seed


def log_digest(rows) -> str:
    h = hashlib.sha256()
    for r in rows:
        h.update("\t".join(repr(float(x)) if isinstance(x, float) else str(x) for x in r).encode())
        h.update(b"\n")
    return h.hexdigest()


def lat_digest(lat: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(lat, dtype=np.float64).tobytes()).hexdigest()


def check(case, rows, report, lat, events=None) -> list[str]:
    """Mismatches between one engine run and the golden reference run."""
    e = case["expect"]
    bad = []
    if events is not None and "ev_sha256" in e:
        if len(events) != e["ev_rows"]:
            bad.append(f"event rows {len(events)} != {e['ev_rows']}")
        elif log_digest(events) != e["ev_sha256"]:
            bad.append("event trace digest")
    if len(rows) != e["log_rows"]:
        bad.append(f"log rows {len(rows)} != {e['log_rows']}")
    got_first = [[repr(float(x)) if isinstance(x, float) else x for x in r] for r in rows[:8]]
    if got_first != e["first_rows"]:
        bad.append(f"first rows {got_first[:2]} != {e['first_rows'][:2]}")
    if log_digest(rows) != e["log_sha256"]:
        bad.append("decision log digest")
    for f in ("configs_used", "failures", "duplicates", "invocations", "completed",
              "terminal_items", "decision_count"):
        if getattr(report, f) != e[f]:
            bad.append(f"{f} {getattr(report, f)} != {e[f]}")
    for f in ("latency_s", "cost", "slack_met_frac"):
        if repr(float(getattr(report, f))) != e[f]:
            bad.append(f"{f} {getattr(report, f)!r} != {e[f]}")
    if lat is not None and lat_digest(lat) != e["lat_sha256"]:
        bad.append("final latency tables")
    return bad


def groups(cases) -> list[list[dict]]:
    out: dict[tuple, list] = {}
    for c in cases:
        out.setdefault(spec_key(c), []).append(c)
    return list(out.values())


def run_group(make_engine, cases):
    """Run the cases of one spec group as replicas of one launch; returns (rows, report, lat)
    per case.  make_engine(spec) -> a ReplicaEngine (device) or the host harness engine."""
    from paper_2102_01887_b200.engine import report_of

    spec = run_spec(cases[0])
    eng = make_engine(spec)
    doc = bundle(cases[0]["bundle"])[0]
    traces = [frames_of(c) for c in cases]
    targets = [float(c["target"]) for c in cases]
    seeds = [seed_of(c) for c in cases]
    cap = max(c["expect"]["log_rows"] for c in cases) + 16
    ecap = max(c["expect"].get("ev_rows", 0) for c in cases) + 16
    res = eng.run(traces, targets, seeds, log_cap=cap, final_tables=True, event_cap=ecap)
    out = []
    for c, r in zip(cases, res):
        rep = report_of(r, target_s=float(c["target"]), scenario_name=spec.scenario.name,
                        pipeline_name=doc.get("name", "pipeline"), seed=seeds[len(out)],
                        ablations=c.get("ablations", []))
        out.append((eng.log_rows(r.log), rep, r.lat, eng.event_rows(r.events)))
    return out


def host_library():
    """Compile the engine source for the host (test harness only; see tests/native/des_host.cpp)."""
    import ctypes as C
    import subprocess

    root = Path(__file__).resolve().parent
    src = root / "native" / "des_host.cpp"
    out = root / "native" / "_build" / "des_host.so"
    pkg = root.parent / "paper_2102_01887_b200" / "csrc"
    deps = [src, pkg / "sp_des.cuh", pkg / "sp_des_host.h", root.parent / "include" / "slackpipe_b200.h"]
    if not out.exists() or any(d.stat().st_mtime > out.stat().st_mtime for d in deps):
        out.parent.mkdir(parents=True, exist_ok=True)
        subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                        "-shared", "-I", str(root.parent / "include"), "-I", str(pkg), str(src),
                        "-o", str(out)], check=True, capture_output=True, text=True)
    lib = C.CDLL(str(out))
    lib.des_host_error.restype = C.c_char_p
    return lib


def host_engine_factory(lib):
    import ctypes as C

    from paper_2102_01887_b200 import engine as E

    class HostEngine(E.ReplicaEngine):
        def __init__(self, spec):
            self.spec, self.cap_scale, self.handle = spec, 1.25, None

        def close(self):
            pass

        def _launch(self, frame_off, attrs, trace_of, targets, seeds, scale, log_cap, final_tables,
                    event_cap=0):
            spec = self.spec
            R = len(targets)
            draw_cap, fac, bits = 0, None, None
            if spec.draws:
                draw_cap = int(spec.item_bound(frame_off, attrs) * scale) + 256
                fac, bits = spec.draws_for(seeds, draw_cap)
            out = np.zeros(R, dtype=E.OUT_DTYPE)
            lg = np.zeros((R, log_cap), dtype=E.LOG_DTYPE) if log_cap else None
            lat = np.zeros((R, int(spec.entry_off[-1]))) if final_tables else None
            ev = np.zeros((R, event_cap), dtype=E.EVENT_DTYPE) if event_cap else None
            ptr = lambda x: C.c_void_p(x.ctypes.data) if x is not None else None
            cs = spec.c_spec()
            rc = lib.des_host_run(C.byref(cs), C.c_double(scale), R, len(frame_off) - 1,
                                  ptr(frame_off), ptr(attrs), ptr(trace_of),
                                  ptr(np.ascontiguousarray(targets, dtype=np.float64)), draw_cap,
                                  ptr(fac), ptr(bits), log_cap, ptr(lg), ptr(lat), ptr(out),
                                  event_cap, ptr(ev))
            if rc:
                raise ValueError(lib.des_host_error().decode())
            return out, lg, lat, ev

    return HostEngine
