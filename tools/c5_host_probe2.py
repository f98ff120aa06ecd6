"""Probe: host enqueue time per config-5 batch (per API call) vs the device time of the batch.
If the host needs longer to enqueue a batch than the device to run it, the loop is host-bound."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2102_01887_b200 as sp
from paper_2102_01887_b200 import synth
import bench_workloads as bw

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
ctx = sp.get_context(0); ctx.set_stream(st.cuda_stream)
tab = sp.OpTable(synth.synth_spec(True), synth.synth_scenario())
B, NB = 65536, 48
inv = synth.synth_invocations(B * NB, tab.lat, tab.gkind, seed=5)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
d = {"slack": T(inv.slack), "avail": T(inv.avail), "supply": T(inv.supply), "mb": T(inv.min_batch), "flags": T(inv.flags.astype(np.int32))}
base = T(np.array([e.latency_initial_s for e in tab.entries]))
noise = T(bw.c5_noise(B, range(NB)).reshape(-1))
out = {k: torch.empty(B, dtype=dt, device=dev) for k, dt in (("idx", torch.int32), ("code", torch.int32), ("fill", torch.int32), ("obj", torch.float64), ("slack", torch.float64), ("wait", torch.float64))}
oi = torch.empty(B, dtype=torch.int32, device=dev); ob = torch.empty(B, dtype=torch.float64, device=dev)
host = {"select": [], "observe": [], "fold": []}
def batch(bt, rec):
    s = slice(bt * B, (bt + 1) * B)
    t0 = time.perf_counter()
    tab.select_batch(d["slack"][s], 100.0, d["avail"][s], upstream_supply=d["supply"][s], min_batch=d["mb"][s], flags=d["flags"][s], out=out)
    t1 = time.perf_counter()
    sp.simulate_observations(out, base, noise[s], out=(oi, ob))
    t2 = time.perf_counter()
    sp.fold_observations([tab], None, oi, ob, beta=0.5, dfp_count=10, sync_host=False)
    t3 = time.perf_counter()
    if rec:
        host["select"].append(t1 - t0); host["observe"].append(t2 - t1); host["fold"].append(t3 - t2)
for bt in range(8):
    batch(bt, False)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
w0 = time.perf_counter(); e0.record(st)
for bt in range(NB):
    batch(bt, True)
w1 = time.perf_counter(); e1.record(st); torch.cuda.synchronize(); w2 = time.perf_counter()
print("host enqueue us/batch", round(1e6 * (w1 - w0) / NB, 1), "wall us/batch", round(1e6 * (w2 - w0) / NB, 1),
      "device us/batch", round(1e3 * e0.elapsed_time(e1) / NB, 1))
print({k: round(1e6 * float(np.median(v)), 1) for k, v in host.items()})
