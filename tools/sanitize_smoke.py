"""Small end-to-end exercise of every kernel family for compute-sanitizer runs (memcheck,
racecheck, synccheck): K2f/K2b/K2a select, plan build (sorts, stair, finalize, graph replay),
K1 slack, K1c certified slack (with fallbacks), K3 fold, commit rounds, quantiles."""
import sys

import numpy as np

sys.path.insert(0, ".")
import __graft_entry__ as g  # noqa: E402

g.smoke()

import paper_2102_01887_b200 as sp  # noqa: E402
from paper_2102_01887_b200 import synth  # noqa: E402

table = sp.OpTable(synth.synth_spec(False), synth.synth_scenario())
inv = synth.synth_invocations(2048, table.lat, table.gkind, seed=11)
for rebuild in range(3):  # first build, captured rebuild, replayed rebuild
    r = table.select_batch(inv.slack, 100.0, inv.avail, upstream_supply=inv.supply,
                           min_batch=inv.min_batch, flags=inv.flags)
    idx = np.where((r["code"] & 3) == 1, r["idx"], -1).astype(np.int32)
    sp.fold_observations([table], None, idx, table.lat[np.maximum(idx, 0)] * 1.1, beta=0.5,
                         dfp_count=10)
r = table.select_batch(inv.slack, 100.0, inv.avail, upstream_supply=inv.supply,
                       min_batch=inv.min_batch, flags=inv.flags, kind_min=True, mode="plan")
r = table.select_batch(inv.slack[:256], 100.0, inv.avail[:256], upstream_supply=inv.supply[:256],
                       min_batch=inv.min_batch[:256], flags=inv.flags[:256], mode="scan")
tabs = [table, sp.OpTable(synth.synth_spec(False), synth.synth_scenario())]
R = 64
rng = np.random.default_rng(1)
out = sp.commit_round(tabs, rng.uniform(-1, 10, (R, 2, 2)), np.ones((R, 2), np.int32),
                      np.zeros((R, 2), np.int32), np.arange(2 * R).reshape(R, 2),
                      np.array([0, 1], np.int32), np.ones((R, 2), np.uint32), alpha=100.0,
                      full_mask=np.zeros(R, np.uint32))
# K1c: certified backward pass with ties / bad refs (per-source and whole-instance fallbacks)
import os  # noqa: E402

dag = synth.deep_dag()
ref, T, now, Q = synth.deep_dag_instances(dag, 200, seed=9, K=2)
ref = np.round(ref * 2) / 2
ref[3, 5] = -1.0
ref[7, :] = 0.0
gd = sp.SlackGraph.from_dag(dag)
a = gd.slack_batch(ref, T, now, Q, ratios=True)
sp.get_context(0).set_option("SP_K1_CERT", 1)
b = gd.slack_batch(ref, T, now, Q, ratios=True)
sp.get_context(0).set_option("SP_K1_CERT", 0)
assert np.array_equal(a["slack"].view(np.uint64), b["slack"].view(np.uint64))
# per-entry observation quantiles
idx = rng.integers(0, len(table.lat), 4000).astype(np.int32)
sp.observation_quantiles([table], None, idx, rng.uniform(0.1, 2.0, 4000), 0.9)
print("sanitize smoke ok", int((out["best"] >= 0).sum()))
# round 2: the one-kernel cluster plan builder (cached-order and re-sorted builds, config-5
# table), the literal scan with non-finite latencies and K > 8, the pinned per-call path,
# affinity batch, the simulated backend and the single-process device group
import math  # noqa: E402

t5 = sp.OpTable(synth.synth_spec(True), synth.synth_scenario())
inv5 = synth.synth_invocations(1024, t5.lat, t5.gkind, seed=3)
for step in range(3):
    r5 = t5.select_batch(inv5.slack, 100.0, inv5.avail, upstream_supply=inv5.supply,
                         min_batch=inv5.min_batch, flags=inv5.flags, mode="plan")
    t5.set_latency(int(step * 37), float(t5.lat[step * 37]) * 1.3)  # forces a re-sort
t5.plan_image(100.0, "cluster")
t5.select({"cpu": 1.0, "gpu": 2.0}, 100.0, 4, allow_delay=True, upstream_supply=3)
t5.affinity("gpu", {"cpu": 1.0, "gpu": 2.0}, 100.0)
t5.set_latency(3, math.inf)
t5.set_latency(9, math.nan)
try:
    t5.select({"cpu": 1.0, "gpu": 2.0}, 100.0, 4, allow_delay=True)
except ValueError:
    pass
rng = np.random.default_rng(2)
K10 = 10
wide = sp.RawTable(lat=rng.uniform(0.1, 3, 3000), res=rng.integers(1, 8, 3000), batch=rng.integers(1, 40, 3000),
                   pool=np.full(3000, 64.0), price=np.full(3000, 1e-5), kind=rng.integers(0, K10, 3000),
                   id_rank=rng.permutation(3000), K=K10)
sp.select_batch([wide], rng.uniform(-1, 4, (300, K10)), 100.0, np.full(300, 8, np.int32),
                upstream_supply=np.zeros(300, np.int32), min_batch=np.ones(300, np.int32),
                flags=np.zeros(300, np.uint32), kind_min=True)
import torch  # noqa: E402

d_out = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in
         (("code", np.ones(64, np.int32)), ("idx", np.arange(64, dtype=np.int32)),
          ("fill", np.ones(64, np.int32)))}
sp.simulate_observations(d_out, torch.ones(len(t5.lat), dtype=torch.float64, device="cuda"),
                         torch.ones(64, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
grp = sp.DeviceGroup([0, 0])
gt = grp.table(synth.synth_spec(False), synth.synth_scenario())
gt.select_batch(inv.slack, 100.0, inv.avail, upstream_supply=inv.supply, min_batch=inv.min_batch,
                flags=inv.flags)
print("sanitize smoke ok")
# the one-kernel cooperative fold: two chunks, a gate lifting in the second, long (narrowed-window)
# segments; the device profile generator (noise + straggles) and the correctly rounded power
rng = np.random.default_rng(4)
M = 3000
lat0 = rng.uniform(0.1, 2.0, M)
ft = sp.RawTable(lat=lat0, res=np.ones(M), batch=np.ones(M, np.int32), pool=np.ones(M),
                 price=np.ones(M), ref_index=0, lat_init=lat0)
n = 140000
idx = np.where(rng.random(n) < 0.6, rng.integers(0, 8, n), rng.integers(0, M, n)).astype(np.int32)
idx[rng.random(n) < 0.1] = -1
sp.fold_observations([ft], None, idx, rng.uniform(0.1, 3.0, n), beta=0.5, dfp_count=9000)
from paper_2102_01887_b200 import profiler  # noqa: E402
from paper_2102_01887_b200.pipeline import Knob, KnobTemplate, OperationSpec  # noqa: E402
from paper_2102_01887_b200.scenario import BackendSpec, GroundTruthModel, OpKindTruth, Scenario  # noqa: E402

tpl = KnobTemplate((Knob("m", ("a", "b")),), ("cpu", "gpu"), (1, 2, 4), {"cpu": (1, 2), "gpu": (4, 8)})
gtm = GroundTruthModel({"op": {"cpu": OpKindTruth(1.0, 1, 0.5, 0.85, 0.1, {"m": {"a": 1.2}}),
                               "gpu": OpKindTruth(0.1, 4, 0.3, 0.35)}}, noise_sigma=0.2, straggle_rate=0.1,
                       straggle_factor=2.0)
scn = Scenario("s", (BackendSpec("cpu", 2, 4, 1e-5), BackendSpec("gpu", 1, 8, 1e-4)), gtm, 3)
profiler.profile_operation(OperationSpec("op", "x", tpl), scn, 3)
profiler.pow_correctly_rounded(rng.uniform(0.01, 100, 500), rng.uniform(-2, 2, 500))
print("sanitize smoke (round 2, session 2) ok")

# session 3: the multi-plan build (one launch, four clusters) + decisions on it, the fused
# simulate-and-fold, and the replica-parallel run engine (small traces, noise / failures / joins)
t6 = sp.OpTable(synth.synth_spec(False), synth.synth_scenario())
t6.invalidate_plans()
t6.prepare_many([0.0, 1.0, 100.0, 1000.0])
for al in (0.0, 1.0, 100.0, 1000.0):
    t6.select_batch(inv.slack, al, inv.avail, upstream_supply=inv.supply, min_batch=inv.min_batch,
                    flags=inv.flags, mode="plan")
dec = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in
       (("code", np.ones(5000, np.int32)), ("idx", rng.integers(0, len(t6.lat), 5000).astype(np.int32)),
        ("fill", np.ones(5000, np.int32)))}
rec = (torch.empty(5000, dtype=torch.int32, device="cuda"), torch.empty(5000, dtype=torch.float64, device="cuda"))
sp.simulate_and_fold(t6, dec, torch.ones(len(t6.lat), dtype=torch.float64, device="cuda"),
                     torch.ones(5000, dtype=torch.float64, device="cuda"), out=rec)
torch.cuda.synchronize()
sys.path.insert(0, "tests")
import des_cases as dc  # noqa: E402
from paper_2102_01887_b200.engine import ReplicaEngine, generate_trace  # noqa: E402

for case in (dict(bundle="branching"), dict(bundle="parallel", noise_sigma=0.2, failure_rate=0.1,
                                            straggle_rate=0.05, straggle_factor=3.0)):
    eng = ReplicaEngine(dc.run_spec(case))
    traces = [generate_trace(60, 100 + i, {"cars": 0.6, "persons": 0.8}, 3) for i in range(3)]
    eng.run(traces, [30.0, 60.0, float("inf")], [1, 2, 3], log_cap=4000, final_tables=True)
print("sanitize smoke (round 2, session 3) ok")
