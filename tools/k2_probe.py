"""Probe: K2 per-launch time with an L2-flush kernel between steps vs. rotating input sets
larger than L2 (no kernel in between).  Prints one JSON line per mode."""
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2102_01887_b200 as sp  # noqa: E402
from paper_2102_01887_b200 import synth  # noqa: E402

N = 1 << 20
SETS = 4
STEPS = 24
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
ctx = sp.get_context(0)
ctx.set_stream(stream.cuda_stream)
table = sp.OpTable(synth.synth_spec(False), synth.synth_scenario(), device=0)
sets = []
for s in range(SETS):
    inv = synth.synth_invocations(N, table.lat, table.gkind, seed=20261017 + s)
    d = {"slack": torch.from_numpy(inv.slack).to(dev), "avail": torch.from_numpy(inv.avail).to(dev),
         "supply": torch.from_numpy(inv.supply).to(dev), "min_batch": torch.from_numpy(inv.min_batch).to(dev),
         "flags": torch.from_numpy(inv.flags.astype(np.int32)).to(dev)}
    o = {"idx": torch.empty(N, dtype=torch.int32, device=dev), "code": torch.empty(N, dtype=torch.int32, device=dev),
         "fill": torch.empty(N, dtype=torch.int32, device=dev), "obj": torch.empty(N, dtype=torch.float64, device=dev),
         "slack": torch.empty(N, dtype=torch.float64, device=dev), "wait": torch.empty(N, dtype=torch.float64, device=dev)}
    sets.append((d, o))
alpha = 100.0
table.prepare(alpha)
flush = torch.ones(256 << 20, dtype=torch.uint8, device=dev)


def step(s):
    d, o = sets[s % SETS]
    table.select_batch(d["slack"], alpha, d["avail"], upstream_supply=d["supply"],
                       min_batch=d["min_batch"], flags=d["flags"], out=o)


def run(mode):
    for i in range(6):
        if mode == "flush":
            flush.max()
        step(i)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(STEPS)]
    torch.cuda._sleep(int(2e6 + 4e5 * STEPS))
    for i in range(STEPS):
        if mode == "flush":
            flush.max()
        elif mode == "tiny":
            flush[:1].zero_()
        evs[i][0].record(stream)
        step(i)
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) * 1e3 for a, b in evs]
    return {"mode": mode, "median_us": statistics.median(ms), "min_us": min(ms), "max_us": max(ms)}


for mode in ("flush", "rotate", "tiny", "flush", "rotate"):
    print(json.dumps(run(mode)), flush=True)
