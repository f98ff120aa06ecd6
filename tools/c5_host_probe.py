"""Probe: is the online-mode (config 5) loop host-bound?  Times the host enqueue of NB batches,
the wall time to completion and the device time between events."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2102_01887_b200 as sp  # noqa: E402
from paper_2102_01887_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
ctx = sp.get_context(0)
ctx.set_stream(stream.cuda_stream)
table = sp.OpTable(synth.synth_spec(True), synth.synth_scenario())
B, NB = 65536, int(sys.argv[1]) if len(sys.argv) > 1 else 48
inv = synth.synth_invocations(B * NB, table.lat, table.gkind, seed=5)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
d = {"slack": T(inv.slack), "avail": T(inv.avail), "supply": T(inv.supply), "mb": T(inv.min_batch),
     "flags": T(inv.flags.astype(np.int32))}
lat_init = T(np.array([e.latency_initial_s for e in table.entries]))
noise = torch.exp(0.3 * torch.randn(B * NB, dtype=torch.float64, device=dev))
out = {k: torch.empty(B, dtype=dt, device=dev) for k, dt in
       (("idx", torch.int32), ("code", torch.int32), ("fill", torch.int32),
        ("obj", torch.float64), ("slack", torch.float64), ("wait", torch.float64))}
obs_idx = torch.empty(B, dtype=torch.int32, device=dev)
table.prepare(100.0)
torch.cuda.synchronize()
parts = {"select": 0.0, "torch": 0.0, "fold": 0.0}


def run(nb, timed_parts=False):
    for b in range(nb):
        s = slice(b * B, (b + 1) * B)
        t0 = time.perf_counter()
        table.select_batch(d["slack"][s], 100.0, d["avail"][s], upstream_supply=d["supply"][s],
                           min_batch=d["mb"][s], flags=d["flags"][s], out=out)
        t1 = time.perf_counter()
        torch.where((out["code"] & 3) == 1, out["idx"], torch.full_like(out["idx"], -1), out=obs_idx)
        obs = lat_init[obs_idx.clamp(min=0).long()] * noise[s]
        t2 = time.perf_counter()
        sp.fold_observations([table], None, obs_idx, obs, beta=0.5, dfp_count=10, sync_host=False)
        t3 = time.perf_counter()
        if timed_parts:
            parts["select"] += t1 - t0
            parts["torch"] += t2 - t1
            parts["fold"] += t3 - t2


run(4)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
w0 = time.perf_counter()
e0.record(stream)
run(NB, True)
e1.record(stream)
w1 = time.perf_counter()
torch.cuda.synchronize()
w2 = time.perf_counter()
print(json.dumps({"enqueue_ms_per_batch": 1e3 * (w1 - w0) / NB, "wall_ms_per_batch": 1e3 * (w2 - w0) / NB,
                  "device_ms_per_batch": e0.elapsed_time(e1) / NB,
                  "host_parts_ms_per_batch": {k: 1e3 * v / NB for k, v in parts.items()},
                  "launches_per_batch": None}))
