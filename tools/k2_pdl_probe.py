"""Probe: K2f per-step time, (a) L2 flushed + event pair per step, (b) K back-to-back steps over
4 rotating input sets (286 MB > L2) in one event pair.  Run with and without SP_NO_PDL."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2102_01887_b200 as sp  # noqa: E402
from paper_2102_01887_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
ctx = sp.get_context(0)
ctx.set_stream(stream.cuda_stream)
table = sp.OpTable(synth.synth_spec(False), synth.synth_scenario(), device=0)
N = 1 << 20
SETS = 4
sets = []
for s in range(SETS):
    inv = synth.synth_invocations(N, table.lat, table.gkind, seed=20261017 + s)
    dd = {"slack": torch.from_numpy(inv.slack).to(dev), "avail": torch.from_numpy(inv.avail).to(dev),
          "supply": torch.from_numpy(inv.supply).to(dev), "min_batch": torch.from_numpy(inv.min_batch).to(dev),
          "flags": torch.from_numpy(inv.flags.astype(np.int32)).to(dev)}
    oo = {"idx": torch.empty(N, dtype=torch.int32, device=dev), "code": torch.empty(N, dtype=torch.int32, device=dev),
          "fill": torch.empty(N, dtype=torch.int32, device=dev), "obj": torch.empty(N, dtype=torch.float64, device=dev),
          "slack": torch.empty(N, dtype=torch.float64, device=dev), "wait": torch.empty(N, dtype=torch.float64, device=dev)}
    sets.append((dd, oo))
ALPHAS = (0.0, 1.0, 100.0, 1000.0)
for a in ALPHAS:
    table.prepare(a)
flush = torch.ones(256 << 20, dtype=torch.uint8, device=dev)
STEPS = 40


def k2(i):
    dd, oo = sets[i % SETS]
    table.select_batch(dd["slack"], ALPHAS[i % 4], dd["avail"], upstream_supply=dd["supply"],
                       min_batch=dd["min_batch"], flags=dd["flags"], out=oo)


def per_step():
    for i in range(4):
        flush.max(); k2(i)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(STEPS)]
    torch.cuda._sleep(int(2e6 + 4e5 * STEPS))
    for i in range(STEPS):
        flush.max()
        evs[i][0].record(stream)
        k2(i)
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) * 1e3 for a, b in evs]
    return statistics.median(ms)


def batched():
    for i in range(4):
        k2(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e6 + 4e5 * STEPS))
    e0.record(stream)
    for i in range(STEPS):
        k2(i)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / STEPS


tag = "nopdl" if os.environ.get("SP_NO_PDL") else "pdl"
for rep in range(2):
    print(json.dumps({"pdl": tag, "flush_per_step_us": per_step(), "rotate_batched_us": batched()}), flush=True)
