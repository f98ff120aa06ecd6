"""From-scratch plan builds of the config-2 table (invalidate -> prepare), CUDA-event timed, and
with SP_PC_DEBUG=1 the cluster builder's per-phase timestamps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2102_01887_b200 as sp
from paper_2102_01887_b200 import synth

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
ctx = sp.get_context(0); ctx.set_stream(st.cuda_stream)
wm = len(sys.argv) > 1 and sys.argv[1] == "c5"
tab = sp.OpTable(synth.synth_spec(wm), synth.synth_scenario())
ts = []
for it in range(30):
    tab.invalidate_plans()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2000000)
    e0.record(st)
    tab.prepare(100.0)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(len(tab.lat), "from-scratch build us: median", np.median(ts[5:]), "min", min(ts[5:]), flush=True)
