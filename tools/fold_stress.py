import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2102_01887_b200 as sp
from paper_2102_01887_b200 import synth
from oracle import feedback as ofb
bits = lambda a: np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)
spec = synth.synth_spec(True)
lat0 = np.array([e.latency_s for e in spec.entries]); M = len(lat0)
fails = 0
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    rng = np.random.default_rng(seed)
    n = 65536
    hot = rng.choice(M, size=64, replace=False)
    idx = np.where(rng.random(n) < 0.8, rng.choice(hot, size=n), rng.integers(0, M, size=n)).astype(np.int32)
    idx[rng.random(n) < 0.01] = 0
    obs = lat0[idx] * np.exp(rng.normal(0, 0.3, size=n))
    tab = sp.RawTable(lat=lat0 * 0.7, res=np.ones(M), batch=np.ones(M, np.int32), pool=np.ones(M), price=np.ones(M), ref_index=0, lat_init=lat0 * 0.7)
    st = ofb.FoldState(lat0 * 0.7, lat0 * 0.7, 0)
    for a, b in ((0, 20000), (20000, n)):
        sp.fold_observations([tab], None, idx[a:b], obs[a:b], beta=0.5, dfp_count=10, sync_host=False)
        ofb.fold([st], None, idx[a:b], obs[a:b], beta=0.5, dfp_count=10)
    g = bits(tab.get_latency()); e = bits(st.lat)
    bad = np.flatnonzero(g != e)
    if len(bad):
        fails += 1
        cnt = np.bincount(idx[idx >= 0], minlength=M)
        print('seed', seed, 'mismatch entries', len(bad), bad[:10], 'obs counts', cnt[bad[:10]], 'is hot', np.isin(bad[:10], hot), flush=True)
print('fails', fails)
