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
