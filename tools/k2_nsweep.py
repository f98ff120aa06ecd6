"""Probe: K2b launch time vs invocation count (L2 flushed between steps) — the intercept is the
fixed per-launch overhead (launch, plan staging, drain), the slope the per-invocation cost."""
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
NMAX = 1 << 22
inv = synth.synth_invocations(NMAX, table.lat, table.gkind, seed=20261017)
d = {"slack": torch.from_numpy(inv.slack).to(dev), "avail": torch.from_numpy(inv.avail).to(dev),
     "supply": torch.from_numpy(inv.supply).to(dev), "min_batch": torch.from_numpy(inv.min_batch).to(dev),
     "flags": torch.from_numpy(inv.flags.astype(np.int32)).to(dev)}
o = {"idx": torch.empty(NMAX, dtype=torch.int32, device=dev), "code": torch.empty(NMAX, dtype=torch.int32, device=dev),
     "fill": torch.empty(NMAX, dtype=torch.int32, device=dev), "obj": torch.empty(NMAX, dtype=torch.float64, device=dev),
     "slack": torch.empty(NMAX, dtype=torch.float64, device=dev), "wait": torch.empty(NMAX, dtype=torch.float64, device=dev)}
alpha = 100.0
table.prepare(alpha)
flush = torch.ones(256 << 20, dtype=torch.uint8, device=dev)
STEPS = 20


def run(n, what="k2"):
    dd = {k: v[:n] if k != "slack" else v[:n] for k, v in d.items()}
    oo = {k: v[:n] for k, v in o.items()}

    def step():
        if what == "k2":
            table.select_batch(dd["slack"], alpha, dd["avail"], upstream_supply=dd["supply"],
                               min_batch=dd["min_batch"], flags=dd["flags"], out=oo)
        else:
            flush[:1].zero_()
    for _ in range(4):
        flush.max(); step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(STEPS)]
    torch.cuda._sleep(int(2e6 + 4e5 * STEPS))
    for i in range(STEPS):
        flush.max()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) * 1e3 for a, b in evs]
    return {"what": what, "n": n, "median_us": statistics.median(ms), "min_us": min(ms)}


print(json.dumps(run(1, "tiny")), flush=True)
for n in (1, 148 * 1024, 1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22):
    print(json.dumps(run(n)), flush=True)
