"""Probe: K2f step time (2^20 invocations, four rotating input sets back to back, as bench.py)
against plan-image size — random K = 2, nB = 8 tables of M = 64 .. 4,096 entries, so the
difference is the per-CTA staging of the plan (296 CTAs each copy the whole image)."""
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2102_01887_b200 as sp  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
ctx = sp.get_context(0)
ctx.set_stream(stream.cuda_stream)
N, SETS, STEPS = 1 << 20, 4, 40
rng = np.random.default_rng(7)
batch_vals = np.array([1, 2, 4, 8, 16, 32, 64, 128])
sets = []
for s in range(SETS):
    sl = rng.uniform(-2, 10, size=(N, 2))
    d = {"slack": torch.from_numpy(sl).to(dev),
         "avail": torch.from_numpy(rng.integers(1, 129, N).astype(np.int32)).to(dev),
         "supply": torch.from_numpy(rng.integers(0, 257, N).astype(np.int32)).to(dev),
         "min_batch": torch.ones(N, dtype=torch.int32, device=dev),
         "flags": torch.from_numpy(sp.make_flags(rng.random(N) < 0.5, 0).astype(np.int32)).to(dev)}
    o = {"idx": torch.empty(N, dtype=torch.int32, device=dev), "code": torch.empty(N, dtype=torch.int32, device=dev),
         "fill": torch.empty(N, dtype=torch.int32, device=dev), "obj": torch.empty(N, dtype=torch.float64, device=dev),
         "slack": torch.empty(N, dtype=torch.float64, device=dev), "wait": torch.empty(N, dtype=torch.float64, device=dev)}
    sets.append((d, o))
for M in (64, 512, 2048, 4096):
    lat = rng.uniform(0.05, 8.0, size=M)
    gk = np.arange(M) % 2
    t = sp.RawTable(lat=lat, res=rng.choice([1.0, 2.0, 4.0], size=M), batch=rng.choice(batch_vals, size=M),
                    pool=np.where(gk == 0, 640.0, 32768.0), price=np.where(gk == 0, 1.3e-5, 5e-8),
                    kind=gk.astype(np.int32), id_rank=rng.permutation(M).astype(np.int32), K=2)
    t.prepare(100.0)
    pb = t.plan_bytes(100.0)

    def step(k):
        d, o = sets[k % SETS]
        sp.select_batch([t], d["slack"], 100.0, d["avail"], upstream_supply=d["supply"],
                        min_batch=d["min_batch"], flags=d["flags"], out=o)
    for k in range(6):
        step(k)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = []
    for rep in range(3):
        a.record(stream)
        for k in range(STEPS):
            step(k)
        b.record(stream)
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) * 1e3 / STEPS)
    print(json.dumps({"M": M, "plan_bytes": pb, "us_per_step": statistics.median(res)}), flush=True)
    t.close()
