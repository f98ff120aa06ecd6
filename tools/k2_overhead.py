"""Probe: where the fixed per-step time of the K2b bench goes — event pair around a tiny kernel
with / without a preceding L2 flush, and K back-to-back launches over rotating input sets."""
import json
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
alpha = 100.0
table.prepare(alpha)
flush = torch.ones(256 << 20, dtype=torch.uint8, device=dev)
tiny = torch.zeros(1, device=dev)
STEPS = 20


def k2(i, n=N):
    dd, oo = sets[i % SETS]
    table.select_batch(dd["slack"][:n], alpha, dd["avail"][:n], upstream_supply=dd["supply"][:n],
                       min_batch=dd["min_batch"][:n], flags=dd["flags"][:n], out={k: v[:n] for k, v in oo.items()})


def per_step(fn, pre):
    for i in range(4):
        pre(); fn(i)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(STEPS)]
    torch.cuda._sleep(int(2e6 + 4e5 * STEPS))
    for i in range(STEPS):
        pre()
        evs[i][0].record(stream)
        fn(i)
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) * 1e3 for a, b in evs]
    return statistics.median(ms), min(ms)


def batched(fn):
    for i in range(4):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e6 + 4e5 * STEPS))
    e0.record(stream)
    for i in range(STEPS):
        fn(i)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / STEPS


nop = lambda: None
fl = lambda: flush.max()
small = lambda: tiny.zero_()
out = {}
out["tiny|noflush"] = per_step(lambda i: tiny.add_(1), nop)
out["tiny|flush"] = per_step(lambda i: tiny.add_(1), fl)
out["tiny|tinypre"] = per_step(lambda i: tiny.add_(1), small)
out["k2n1|noflush"] = per_step(lambda i: k2(i, 1), nop)
out["k2n1|flush"] = per_step(lambda i: k2(i, 1), fl)
out["k2|flush"] = per_step(k2, fl)
out["k2|rotate-per-step"] = per_step(k2, nop)
out["k2|rotate-batched"] = batched(k2)
out["tiny|batched"] = batched(lambda i: tiny.add_(1))
for k, v in out.items():
    print(json.dumps({"case": k, "us": v}), flush=True)
