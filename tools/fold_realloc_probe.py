"""Regression probe: the cooperative fold's buffers grown by a larger key space (here 4,096 ->
16,384 + 1 keys) right before a fold — the re-initialisation must be ordered before the kernel on
the context's (non-blocking) stream.  Fresh context per trial."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2102_01887_b200 as sp
from paper_2102_01887_b200 import _lib, synth
from oracle import feedback as ofb
bits = lambda a: np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)
spec = synth.synth_spec(True)
lat0 = np.array([e.latency_s for e in spec.entries]); M = len(lat0)
fails = 0
trials = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for trial in range(trials):
    ctx = _lib.Context(0)
    small = sp.RawTable(lat=lat0[:4096] * 0.7, res=np.ones(4096), batch=np.ones(4096, np.int32), pool=np.ones(4096),
                        price=np.ones(4096), ref_index=0, lat_init=lat0[:4096] * 0.7, ctx=ctx)
    sp.fold_observations([small], None, np.arange(100, dtype=np.int32), np.ones(100), beta=0.5, dfp_count=10, sync_host=False)
    rng = np.random.default_rng(trial)
    n = 65536
    hot = rng.choice(M, size=64, replace=False)
    idx = np.where(rng.random(n) < 0.8, rng.choice(hot, size=n), rng.integers(0, M, size=n)).astype(np.int32)
    idx[rng.random(n) < 0.01] = 0
    obs = lat0[idx] * np.exp(rng.normal(0, 0.3, size=n))
    tab = sp.RawTable(lat=lat0 * 0.7, res=np.ones(M), batch=np.ones(M, np.int32), pool=np.ones(M), price=np.ones(M),
                      ref_index=0, lat_init=lat0 * 0.7, ctx=ctx)
    st = ofb.FoldState(lat0 * 0.7, lat0 * 0.7, 0)
    sp.fold_observations([tab], None, idx, obs, beta=0.5, dfp_count=10, sync_host=False)
    ofb.fold([st], None, idx, obs, beta=0.5, dfp_count=10)
    bad = np.flatnonzero(bits(tab.get_latency()) != bits(st.lat))
    if len(bad):
        fails += 1
        print("trial", trial, "mismatching entries", len(bad), flush=True)
    del small, tab
    ctx.close() if hasattr(ctx, "close") else None
print("fails", fails, "of", trials)
