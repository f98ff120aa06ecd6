"""Throughput probe of the replica-parallel run engine (k_des_run) on config-4 replicas."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np

import des_cases as dc
import paper_2102_01887_b200 as sp
from paper_2102_01887_b200.engine import ReplicaEngine, generate_trace

CP_MIN = 90.41885182994682
ctx = sp.get_context(0)
case = dc.runs()[3]
spec = dc.run_spec(case)
eng = ReplicaEngine(spec, ctx)
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("R", nargs="*", type=int, default=[148, 1024, 4096])
ap.add_argument("--frames", type=int, default=3000)
ap.add_argument("--once", action="store_true")
ap.add_argument("--mode", default="warp", choices=["default", "warp", "thread", "lanes2", "lanes4", "lanes8", "lanes16"])
args = ap.parse_args()
eng.set_mode(args.mode)
for R in args.R:
    t0 = time.time()
    uniq = [generate_trace(args.frames, 17 + i, {"cars": 0.6, "persons": 0.8}, 3) for i in range(min(R, 256))]
    trace_of = [(r // 5) % len(uniq) for r in range(R)]
    targets = [(0.5, 1.0, 2.0, 5.0, 10.0)[r % 5] * CP_MIN for r in range(R)]
    fo, at = spec.encode_frames(uniq)
    t1 = time.time()
    res = eng.run(None, targets, None, trace_of=trace_of, encoded=(fo, at))
    t2 = time.time()
    if not args.once:
        res = eng.run(None, targets, None, trace_of=trace_of, encoded=(fo, at))
    t3 = time.time()
    dt = (t3 - t2) if not args.once else (t2 - t1)
    dec = sum(r.decision_count for r in res)
    print(f"{args.mode} R={R}: gen {t1-t0:.2f}s run {t2-t1:.3f}s / {t3-t2:.3f}s  {R/dt:.1f} runs/s  "
          f"{dec/dt:.3e} decisions/s  arena {eng.lib.sp_des_arena_bytes(eng.handle)/1e6:.2f} MB/replica",
          flush=True)
