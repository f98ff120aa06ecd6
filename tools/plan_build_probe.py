"""Plan build time, cluster vs multi-kernel builder (CUDA events, warm, rebuilds after a
set_latency each time so every build is real)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2102_01887_b200 as sp
from paper_2102_01887_b200 import synth

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
ctx = sp.get_context(0); ctx.set_stream(st.cuda_stream)
for wm in (False, True):
    spec = synth.synth_spec(wm)
    tab = sp.OpTable(spec, synth.synth_scenario())
    for builder in ("cluster", "legacy"):
        tab.plan_image(100.0, builder)  # warm
        lib = ctx.lib
        # time prepare() after a latency bump, through the context default
        os.environ.pop("SP_PLAN_LEGACY", None)
        ts = []
        for it in range(30):
            tab.set_latency(0, float(tab.lat[0]))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            tab.prepare(100.0)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(len(tab.lat), "default builder", "median us", np.median(ts[5:]), "min", min(ts[5:]), flush=True)
        break
