"""Per-phase device time of the config-5 online batch (CUDA events; each phase timed alone)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2102_01887_b200 as sp
from paper_2102_01887_b200 import synth
import bench_workloads as bw

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
ctx = sp.get_context(0); ctx.set_stream(st.cuda_stream)
spec = synth.synth_spec(True)
tab = sp.OpTable(spec, synth.synth_scenario())
B, NB = 65536, 24
inv = synth.synth_invocations(B * NB, tab.lat, tab.gkind, seed=5)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
d = {"slack": T(inv.slack), "avail": T(inv.avail), "supply": T(inv.supply), "mb": T(inv.min_batch), "flags": T(inv.flags.astype(np.int32))}
base = T(np.array([e.latency_initial_s for e in tab.entries]))
noise = T(bw.c5_noise(B, range(NB)).reshape(-1))
out = {k: torch.empty(B, dtype=dt, device=dev) for k, dt in (("idx", torch.int32), ("code", torch.int32), ("fill", torch.int32), ("obj", torch.float64), ("slack", torch.float64), ("wait", torch.float64))}
oi = torch.empty(B, dtype=torch.int32, device=dev); ob = torch.empty(B, dtype=torch.float64, device=dev)
ph = {"rebuild": [], "select": [], "observe": [], "fold": [], "whole": []}
def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(st); return e
for bt in range(NB):
    s = slice(bt * B, (bt + 1) * B)
    torch.cuda.synchronize(); e0 = ev()
    tab.prepare(100.0)
    e1 = ev()
    tab.select_batch(d["slack"][s], 100.0, d["avail"][s], upstream_supply=d["supply"][s], min_batch=d["mb"][s], flags=d["flags"][s], out=out)
    e2 = ev()
    sp.simulate_observations(out, base, noise[s], out=(oi, ob))
    e3 = ev()
    sp.fold_observations([tab], None, oi, ob, beta=0.5, dfp_count=10, sync_host=False)
    e4 = ev(); torch.cuda.synchronize()
    if bt >= 4:
        ph["rebuild"].append(e0.elapsed_time(e1)); ph["select"].append(e1.elapsed_time(e2))
        ph["observe"].append(e2.elapsed_time(e3)); ph["fold"].append(e3.elapsed_time(e4))
# whole batches back to back
torch.cuda.synchronize(); e0 = ev()
for bt in range(NB):
    s = slice(bt * B, (bt + 1) * B)
    tab.select_batch(d["slack"][s], 100.0, d["avail"][s], upstream_supply=d["supply"][s], min_batch=d["mb"][s], flags=d["flags"][s], out=out)
    sp.simulate_observations(out, base, noise[s], out=(oi, ob))
    sp.fold_observations([tab], None, oi, ob, beta=0.5, dfp_count=10, sync_host=False)
e1 = ev(); torch.cuda.synchronize()
print({k: round(1e3 * float(np.median(v)), 1) for k, v in ph.items() if v}, "back-to-back us/batch", round(1e3 * e0.elapsed_time(e1) / NB, 1))
