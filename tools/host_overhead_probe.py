"""Host cost of the Python API calls of one config-5 batch (device tensors, kernels async):
select_batch / simulate_observations / fold_observations, each called back to back 2,000 times
without synchronising, against the bare ctypes call with pre-built arguments."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np, torch
import paper_2102_01887_b200 as sp
from paper_2102_01887_b200 import synth, _lib

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
ctx = sp.get_context(0); ctx.set_stream(st.cuda_stream)
tab = sp.OpTable(synth.synth_spec(True), synth.synth_scenario())
B = 4096
inv = synth.synth_invocations(B, tab.lat, tab.gkind, seed=5)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
d = {"slack": T(inv.slack), "avail": T(inv.avail), "supply": T(inv.supply), "mb": T(inv.min_batch), "flags": T(inv.flags.astype(np.int32))}
out = {k: torch.empty(B, dtype=dt, device=dev) for k, dt in (("idx", torch.int32), ("code", torch.int32), ("fill", torch.int32), ("obj", torch.float64), ("slack", torch.float64), ("wait", torch.float64))}
base = T(np.array([e.latency_initial_s for e in tab.entries])); noise = torch.ones(B, dtype=torch.float64, device=dev)
oi = torch.empty(B, dtype=torch.int32, device=dev); ob = torch.empty(B, dtype=torch.float64, device=dev)
tab.prepare(100.0); torch.cuda.synchronize()
def rate(f, n=2000):
    for _ in range(50): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    t1 = time.perf_counter(); torch.cuda.synchronize()
    return round(1e6 * (t1 - t0) / n, 2)
res = {}
res["select_batch (plan fresh)"] = rate(lambda: tab.select_batch(d["slack"], 100.0, d["avail"], upstream_supply=d["supply"], min_batch=d["mb"], flags=d["flags"], out=out))
arr = (C.c_void_p * 1)(tab.handle.value)
args = (ctx.handle, 1, C.cast(arr, C.c_void_p), 100.0, B, None, *[C.c_void_p(x.data_ptr()) for x in (d["slack"], d["avail"], d["supply"], d["mb"], d["flags"], out["idx"], out["code"], out["fill"], out["obj"], out["slack"], out["wait"])], None, _lib.MODES["auto"], _lib.SP_MEM_DEVICE)
res["sp_select_batch bare ctypes"] = rate(lambda: ctx.lib.sp_select_batch(*args))
res["simulate_observations"] = rate(lambda: sp.simulate_observations(out, base, noise, out=(oi, ob)))
res["fold_observations (+ select after: plan rebuild)"] = rate(lambda: (sp.fold_observations([tab], None, oi, ob, beta=0.5, dfp_count=10, sync_host=False), tab.select_batch(d["slack"], 100.0, d["avail"], upstream_supply=d["supply"], min_batch=d["mb"], flags=d["flags"], out=out)), 500)
res["torch empty launch (x.add_(0))"] = rate(lambda: ob.add_(0))
print(res)
