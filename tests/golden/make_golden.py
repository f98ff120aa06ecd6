"""Generate the golden fixtures from the UNMODIFIED reference (run in the build container).

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Every expected value below is produced by calling the reference package itself
(`slackpipe`, imported read-only from /root/reference); the inputs come from seeded
generators in this file.  The resulting .npz files are committed and travel to the GPU box,
where /root/reference does not exist.  Files:

  select_cases.npz   3,000 random small OpTable instances: select / affinity / scores
  synth_sample.npz   config-2 table (4,096 entries) x 4,096 invocations x 4 alphas, plus a
                     config-5 table (16,384 entries) x 1,024 invocations (OpTable.select)
  slack_cases.npz    random DAGs (<= 12 ops) and explicit path lists: compute_slack
  feedback_cases.npz random observation streams through PipelineRun._apply_feedback
  queue_cases.npz    estimate_queueing on random lists (+ the reference's 20 fixtures)
  amber_trace.npz    every OpTable.select / affinity / set_latency call of the reference
                     AMBER (`branching`) run at the 50% target, in call order, with results
  commit_rounds.npz  every Configurator.pump_commits round (one _commit_candidate per op with a
                     speculated head, then the winner) of AMBER runs at the 50% and fast
                     targets and under the pbc / eslc ablations, interleaved in order with the
                     set_latency calls that change the tables between rounds
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import random
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

KINDS3 = ["cpu", "gpu", "lite"]


def _ref_modules(ref_src: str):
    sys.path.insert(0, ref_src)
    import slackpipe  # noqa: F401
    from slackpipe import configurator, manager, pipeline, profiler, scenario

    return configurator, manager, pipeline, profiler, scenario


# ---- 1. small select cases ------------------------------------------------------------------

def gen_select_cases(R, n_cases=3000, seed=987654321):
    conf, _, pipe, _, scen = R
    rng = random.Random(seed)
    backends = (scen.BackendSpec("cpu", 4, 4, 1.32e-5), scen.BackendSpec("gpu", 2, 8, 3.0e-4),
                scen.BackendSpec("lite", 64, 2, 8.0e-6))
    sc = scen.Scenario("golden", backends, scen.GroundTruthModel(per_op={}))
    caps = {"cpu": 4, "gpu": 8, "lite": 2}
    cols = {k: [] for k in ("kind", "res", "batch", "lat", "sched", "knob")}
    off = [0]
    params = {k: [] for k in ("alpha", "avail", "supply", "allow_delay", "excl", "min_batch")}
    slacks = []
    exp = {k: [] for k in ("code", "idx", "fill", "obj", "slack", "wait", "feas")}
    kmin = []
    aff = []
    score_cat = []
    lat_pool = [0.25, 0.5, 1.0, 2.0, 0.75]
    for case in range(n_cases):
        ents = []
        n = rng.randint(0, 15)
        # a cpu batch-1 entry most of the time (reference config), sometimes unschedulable
        first_res = rng.choice([1, 2, 8]) if rng.random() < 0.1 else rng.choice([1, 2])
        proto = [("cpu", first_res, 1, rng.uniform(0.05, 4.0), first_res <= 4, 0)]
        for i in range(n):
            kind = rng.choice(KINDS3)
            res = rng.choice([1, 2, 4, 8])
            batch = rng.choice([1, 2, 4, 8, 16])
            lat = rng.choice(lat_pool) if rng.random() < 0.3 else rng.uniform(0.01, 8.0)
            sched = res <= caps[kind] if rng.random() < 0.9 else False
            proto.append((kind, res, batch, lat, sched, i + 1))
            if rng.random() < 0.15:  # exact twin differing only by knob -> id tie-break
                proto.append((kind, res, batch, lat, sched, 100 + i))
        for kind, res, batch, lat, sched, knob in proto:
            ents.append(pipe.ConfigEntry(
                config_id=f"{kind}-r{res}-b{batch}-i={knob}", backend_kind=kind,
                knob_values={"i": knob}, batch_size=batch, resource_request=res,
                latency_s=lat, latency_initial_s=lat, schedulable=sched))
        spec = pipe.ConfigSpec("op", ents, ents[0].config_id)
        try:
            table = conf.OpTable(spec, sc)
        except ValueError:
            continue  # no schedulable entry (reference raises); skip the case
        for e in ents:
            cols["kind"].append(KINDS3.index(e.backend_kind))
            cols["res"].append(e.resource_request)
            cols["batch"].append(e.batch_size)
            cols["lat"].append(e.latency_s)
            cols["sched"].append(int(e.schedulable))
            cols["knob"].append(e.knob_values["i"])
        off.append(len(cols["kind"]))
        s = {}
        for k in KINDS3:
            u = rng.random()
            if u < 0.05:
                s[k] = math.inf
            elif u < 0.12 and table.entries:
                s[k] = rng.choice(table.entries).latency_s  # boundary: lat == slack
            else:
                s[k] = rng.uniform(-2.0, 5.0)
        alpha = rng.choice([0.0, 1.0, 100.0, 1000.0])
        avail = rng.randint(1, 20)
        supply = rng.randint(0, 20)
        allow = rng.random() < 0.5
        ex = frozenset(k for k in KINDS3 if rng.random() < 0.15)
        mb = rng.choice([1, 1, 1, 2, 4, 8, 16, 32])
        d = table.select(s, alpha, avail, allow_delay=allow, upstream_supply=supply,
                         excluded_kinds=ex, min_batch=mb)
        params["alpha"].append(alpha)
        params["avail"].append(avail)
        params["supply"].append(supply)
        params["allow_delay"].append(int(allow))
        params["excl"].append(sum(1 << KINDS3.index(k) for k in ex))
        params["min_batch"].append(mb)
        slacks.append([s[k] for k in KINDS3])
        if d is None:
            vals = (0, -1, 0, 0.0, 0.0, 0.0, 0)
        else:
            code = 2 if d.kind == "delay" else 1
            feas = int(d.entry.latency_s < s[d.entry.backend_kind])
            vals = (code, d.entry_index, d.fill, d.objective_value, d.slack_s, d.wait_budget_s, feas)
        for k, v in zip(exp, vals):
            exp[k].append(v)
        sc_, _ = table.scores(s, alpha)
        score_cat.extend(sc_.tolist())
        km, af = [], []
        for k in KINDS3:
            on = [i for i, e in enumerate(table.entries) if e.backend_kind == k]
            km.append(min(sc_[i] for i in on) if on else math.inf)
            a = table.affinity(k, s, alpha)
            af.append(math.nan if a is None else a)
        kmin.append(km)
        aff.append(af)
    out = {f"ent_{k}": np.array(v) for k, v in cols.items()}
    out["ent_lat"] = out["ent_lat"].astype(np.float64)
    out["off"] = np.array(off, dtype=np.int64)
    out.update({f"p_{k}": np.array(v) for k, v in params.items()})
    out["slack"] = np.array(slacks, dtype=np.float64)
    out.update({f"x_{k}": np.array(v) for k, v in exp.items()})
    out["x_kind_min"] = np.array(kmin, dtype=np.float64)
    out["x_affinity"] = np.array(aff, dtype=np.float64)
    out["x_scores"] = np.array(score_cat, dtype=np.float64)
    out["backends"] = np.array([[4, 4, 1.32e-5], [2, 8, 3.0e-4], [64, 2, 8.0e-6]])
    return out


# ---- 2. synthetic config-2 / config-5 samples -----------------------------------------------

def gen_synth(R):
    conf, _, pipe, prof, scen = R
    from paper_2102_01887_b200 import synth

    out = {}
    for tag, with_model, n_inv, alphas in (("c2", False, 4096, (0.0, 1.0, 100.0, 1000.0)),
                                           ("c5", True, 1024, (100.0,))):
        tr = synth.synth_truths(with_model)
        knobs = [pipe.Knob("sampling", synth.SAMPLING), pipe.Knob("variant", synth.VARIANT)]
        if with_model:
            knobs.append(pipe.Knob("model", synth.MODEL))
        tpl = pipe.KnobTemplate(knobs=tuple(knobs), hardware_targets=("cpu", "gpu"),
                                batch_sizes=synth.BATCHES,
                                resource_options={"cpu": synth.CPU_RES, "gpu": synth.GPU_RES})
        op = pipe.OperationSpec("op", "synth-v1", tpl)
        sc = scen.Scenario(
            "synth", (scen.BackendSpec("cpu", 10, 64, 1.32e-5), scen.BackendSpec("gpu", 2, 16384, 9e-4 / 16384)),
            scen.GroundTruthModel(per_op={"op": {
                k: scen.OpKindTruth(v.base_seconds, v.ref_resource, v.resource_exponent,
                                    v.batch_exponent, 0.0, v.knob_multipliers) for k, v in tr.items()}}),
            seed=1)
        spec = prof.profile_operation(op, sc, 1)
        table = conf.OpTable(spec, sc)
        out[f"{tag}_lat"] = table.lat.copy()
        out[f"{tag}_ids_sha"] = np.frombuffer(
            hashlib.sha256("\n".join(e.config_id for e in table.entries).encode()).digest(), np.uint8)
        out[f"{tag}_ref_index"] = np.array(table.ref_index)
        gk = np.array([["cpu", "gpu"].index(e.backend_kind) for e in table.entries])
        inv = synth.synth_invocations(n_inv, table.lat, gk, seed=20261017 if tag == "c2" else 5)
        for f in ("slack", "avail", "supply", "min_batch", "flags"):
            out[f"{tag}_in_{f}"] = getattr(inv, f)
        for a in alphas:
            res = {k: [] for k in ("code", "idx", "fill", "obj", "slack", "wait", "feas")}
            for i in range(n_inv):
                s = {"cpu": float(inv.slack[i, 0]), "gpu": float(inv.slack[i, 1])}
                fl = int(inv.flags[i])
                ex = frozenset(k for j, k in enumerate(("cpu", "gpu")) if (fl >> (8 + j)) & 1)
                d = table.select(s, a, int(inv.avail[i]), allow_delay=bool(fl & 1),
                                 upstream_supply=int(inv.supply[i]), excluded_kinds=ex,
                                 min_batch=int(inv.min_batch[i]))
                if d is None:
                    v = (0, -1, 0, 0.0, 0.0, 0.0, 0)
                else:
                    v = (2 if d.kind == "delay" else 1, d.entry_index, d.fill, d.objective_value,
                         d.slack_s, d.wait_budget_s, int(d.entry.latency_s < s[d.entry.backend_kind]))
                for k, x in zip(res, v):
                    res[k].append(x)
            for k, v in res.items():
                out[f"{tag}_a{int(a)}_{k}"] = np.array(v)
        # affinity on the first 256 invocations (alpha 100), both kinds
        affs = []
        for i in range(256):
            s = {"cpu": float(inv.slack[i, 0]), "gpu": float(inv.slack[i, 1])}
            affs.append([table.affinity(k, s, 100.0) for k in ("cpu", "gpu")])
        out[f"{tag}_affinity"] = np.array(affs, dtype=np.float64)
    return out


# ---- 3. slack cases ---------------------------------------------------------------------------

def gen_slack(R, n_dags=400, seed=7):
    conf, _, pipe, _, _ = R
    rng = random.Random(seed)
    e_off, e_src, e_dst = [0], [], []
    v_off, v_ref = [0], []
    q_case, q_op, q_target, q_elapsed, q_queue, q_expect = [], [], [], [], [], []
    for c in range(n_dags):
        n = rng.randint(1, 12)
        names = [f"v{i:02d}" for i in range(n)]
        perm = names[:]
        rng.shuffle(perm)
        edges = []
        for i in range(n):
            for j in range(i + 1, n):
                if rng.random() < 0.4:
                    edges.append((perm[i], perm[j]))
        dag = pipe.PipelineDag(vertices=tuple(sorted(names)), edges=tuple(edges))
        paths = pipe.decompose_paths(dag)
        ref = {v: rng.choice([rng.uniform(1e-3, 10.0), rng.choice([0.1, 0.2, 0.3, 1 / 3, 0.7])])
               for v in names}
        for s, d in edges:
            e_src.append(names.index(s))
            e_dst.append(names.index(d))
        e_off.append(len(e_src))
        v_ref.extend(ref[v] for v in names)
        v_off.append(len(v_ref))
        for op in names:
            for _ in range(3):
                u = rng.random()
                if u < 0.1:
                    tgt, el, qu = math.inf, rng.uniform(0, 5), rng.uniform(0, 2)
                elif u < 0.2:
                    tgt, el, qu = 3.0, 3.0, 0.0  # zero budget
                else:
                    tgt, el, qu = rng.uniform(0, 60), rng.uniform(0, 30), rng.uniform(0, 10)
                got = conf.compute_slack(op, "cpu", target_s=tgt, elapsed_s=el, queueing_s=qu,
                                         paths=paths, ref_latency=ref).seconds
                q_case.append(c)
                q_op.append(names.index(op))
                q_target.append(tgt)
                q_elapsed.append(el)
                q_queue.append(qu)
                q_expect.append(got)
    out = dict(e_off=np.array(e_off), e_src=np.array(e_src), e_dst=np.array(e_dst),
               v_off=np.array(v_off), v_ref=np.array(v_ref, dtype=np.float64),
               q_case=np.array(q_case), q_op=np.array(q_op), q_target=np.array(q_target),
               q_elapsed=np.array(q_elapsed), q_queue=np.array(q_queue),
               q_expect=np.array(q_expect, dtype=np.float64))
    # explicit path lists (random subsequences, as test_configurator.py:164-185 does)
    p_case_paths, p_ref, p_expect, p_op, p_budget = [], [], [], [], []
    for c in range(300):
        r2 = random.Random(1000 + c)
        ops = [f"v{i}" for i in range(r2.randint(2, 6))]
        ref = {op: r2.choice([0.25, 0.5, 1.0, 2.0, 4.0, r2.uniform(0.01, 3)]) for op in ops}
        paths = []
        for _ in range(r2.randint(1, 4)):
            k = r2.randint(1, len(ops))
            paths.append(tuple(sorted(r2.sample(ops, k), key=ops.index)))
        op = r2.choice([o for p in paths for o in p])
        budget = float(r2.randint(-8, 64)) if r2.random() < 0.7 else r2.uniform(-10, 100)
        got = conf.compute_slack(op, "cpu", target_s=budget, elapsed_s=0.0, queueing_s=0.0,
                                 paths=tuple(paths), ref_latency=ref).seconds
        p_case_paths.append([list(p) for p in paths])
        p_ref.append(ref)
        p_expect.append(got)
        p_op.append(op)
        p_budget.append(budget)
    out["paths_json"] = np.frombuffer(json.dumps(
        {"paths": p_case_paths, "ref": p_ref, "op": p_op, "budget": p_budget}).encode(), np.uint8)
    out["paths_expect"] = np.array(p_expect, dtype=np.float64)
    return out


# ---- 4. feedback streams ----------------------------------------------------------------------

class _Inv:
    def __init__(self, op, entry, eidx):
        self.operation = op
        self.committed_entry = entry
        self.committed_eidx = eidx


def gen_feedback(R, n_cases=120, seed=11):
    conf, man, pipe, prof, scen = R
    rng = random.Random(seed)
    recs = []
    arrays = {k: [] for k in ("lat0", "latinit", "obs", "obs_op", "obs_idx", "final_lat",
                              "final_cnt")}
    meta = []
    for c in range(n_cases):
        truth = {
            "a": {"cpu": scen.OpKindTruth(0.5, 1, 0.3, 1.1), "gpu": scen.OpKindTruth(0.08, 4, 0.2, 0.4)},
            "b": {"cpu": scen.OpKindTruth(0.3, 1, 0.0, 0.9), "lite": scen.OpKindTruth(0.2, 1, 0.1, 1.0)},
        }
        sc = scen.Scenario("fb", (scen.BackendSpec("cpu", 4, 4, 1.32e-5), scen.BackendSpec("gpu", 2, 8, 3e-4),
                                  scen.BackendSpec("lite", 16, 2, 8e-6)),
                           scen.GroundTruthModel(per_op=truth), seed=c)
        ops = {
            "a": pipe.OperationSpec("a", "a-v1", pipe.KnobTemplate((), ("cpu", "gpu"), (1, 2, 4), {"cpu": (1, 2), "gpu": (4,)})),
            "b": pipe.OperationSpec("b", "b-v1", pipe.KnobTemplate((), ("cpu", "lite"), (1, 4), {"cpu": (1,), "lite": (1, 2)})),
        }
        dag = pipe.PipelineDag(vertices=("a", "b"), edges=(("a", "b"),))
        profiles = {k: prof.profile_operation(o, sc, 1) for k, o in ops.items()}
        dfp = rng.choice([0, 1, 2, 3, 5])
        scale = rng.choice([0.5, 1.0, 1.7, 0.8])
        abl = rng.choice([(), (), ("fb",), ("dfp",)])
        beta = rng.choice([0.5, 0.5, 0.25, 1.0, 0.3])
        run = man.PipelineRun(dag, ops, profiles, [(0, {})], sc, 60.0,
                              conf.TuningParams(dfp_count=dfp, smoothing_beta=beta),
                              ablations=abl, profile_scale=scale)
        tabs = [run.tables["a"], run.tables["b"]]
        for t in tabs:
            arrays["lat0"].extend(t.lat.tolist())
            arrays["latinit"].extend(e.latency_initial_s for e in t.entries)
        n = rng.randint(0, 40)
        for _ in range(n):
            ti = rng.randrange(2)
            t = tabs[ti]
            if rng.random() < 0.5 and t.ref_index >= 0:
                e = t.ref_index
            else:
                e = rng.randrange(len(t.entries))
            ob = t.entries[e].latency_initial_s / scale * math.exp(rng.gauss(0, 0.2))
            run._apply_feedback(_Inv(("a", "b")[ti], t.entries[e], e), ob)
            arrays["obs"].append(ob)
            arrays["obs_op"].append(ti)
            arrays["obs_idx"].append(e)
        for ti, t in enumerate(tabs):
            arrays["final_lat"].extend(t.lat.tolist())
            arrays["final_cnt"].extend(run.feedback.observations.get((("a", "b")[ti], e.config_id), 0)
                                       for e in t.entries)
        meta.append({"n_obs": n, "sizes": [len(t.entries) for t in tabs],
                     "ref": [t.ref_index for t in tabs], "dfp": dfp, "beta": beta,
                     "fb": "fb" not in abl, "dfp_on": "dfp" not in abl,
                     "completed_ref": [run.configurator.completed_ref["a"], run.configurator.completed_ref["b"]]})
    out = {k: np.array(v, dtype=np.float64 if k in ("lat0", "latinit", "obs", "final_lat") else np.int64)
           for k, v in arrays.items()}
    out["meta_json"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    return out


# ---- 5. queueing --------------------------------------------------------------------------------

def gen_queue(R, n=500, seed=5):
    conf, _, pipe, _, _ = R
    rng = random.Random(seed)
    lat, res, off, pool, expect = [], [], [0], [], []
    for c in range(n):
        m = rng.randint(0, 12)
        ents = [pipe.ConfigEntry(f"q{i}", "cpu", {}, 1, rng.choice([1, 2, 3, 4, 8]),
                                 rng.uniform(0.01, 10.0), 1.0) for i in range(m)]
        p = rng.choice([2.0, 3.0, 16.0, 96.0, 7.0])
        expect.append(conf.estimate_queueing(ents, p))
        lat.extend(e.latency_s for e in ents)
        res.extend(e.resource_request for e in ents)
        off.append(len(lat))
        pool.append(p)
    return dict(lat=np.array(lat), res=np.array(res, dtype=np.float64), off=np.array(off),
                pool=np.array(pool), expect=np.array(expect))


# ---- 6. AMBER trace -----------------------------------------------------------------------------

def gen_amber(R, ref_root: Path, target=142.20064921472454):
    conf, man, pipe, prof, scen = R
    from slackpipe import workload

    bundle = ref_root / "scenarios" / "branching"
    dag, ops = pipe.load_pipeline(json.loads((bundle / "pipeline.json").read_text()))
    sc = scen.load_scenario(bundle / "scenario.json")
    frames = workload.load_trace(bundle / "trace.jsonl")
    profiles = {n: prof.profile_operation(o, sc, sc.tuning.samples_per_config) for n, o in ops.items()}
    kinds = sc.backend_kinds()
    rec = {"kind": [], "op": [], "slack": [], "alpha": [], "avail": [], "supply": [], "flags": [],
           "min_batch": [], "r_code": [], "r_idx": [], "r_fill": [], "r_obj": [], "r_slack": [],
           "r_wait": [], "aff_kind": [], "lat_idx": [], "lat_val": []}
    orig_select, orig_aff, orig_set = conf.OpTable.select, conf.OpTable.affinity, conf.OpTable.set_latency
    op_names = sorted(dag.vertices)

    def _slack(sl):
        return [float(sl.get(k, math.nan)) for k in kinds]

    def sel(self, slack_by_kind, alpha, available, *, allow_delay, upstream_supply=0,
            excluded_kinds=frozenset(), min_batch=1):
        d = orig_select(self, slack_by_kind, alpha, available, allow_delay=allow_delay,
                        upstream_supply=upstream_supply, excluded_kinds=excluded_kinds,
                        min_batch=min_batch)
        rec["kind"].append(0)
        rec["op"].append(op_names.index(self.operation))
        rec["slack"].append(_slack(slack_by_kind))
        rec["alpha"].append(alpha)
        rec["avail"].append(available)
        rec["supply"].append(upstream_supply)
        rec["flags"].append(int(allow_delay) | (sum(1 << kinds.index(k) for k in excluded_kinds if k in kinds) << 8))
        rec["min_batch"].append(min_batch)
        if d is None:
            v = (0, -1, 0, 0.0, 0.0, 0.0)
        else:
            v = (2 if d.kind == "delay" else 1, d.entry_index, d.fill, d.objective_value, d.slack_s,
                 d.wait_budget_s)
        for k, x in zip(("r_code", "r_idx", "r_fill", "r_obj", "r_slack", "r_wait"), v):
            rec[k].append(x)
        rec["aff_kind"].append(-1)
        rec["lat_idx"].append(-1)
        rec["lat_val"].append(0.0)
        return d

    def aff(self, backend_kind, slack_by_kind, alpha):
        a = orig_aff(self, backend_kind, slack_by_kind, alpha)
        rec["kind"].append(1)
        rec["op"].append(op_names.index(self.operation))
        rec["slack"].append(_slack(slack_by_kind))
        rec["alpha"].append(alpha)
        for k in ("avail", "supply", "flags", "min_batch", "r_code", "r_idx", "r_fill", "lat_idx"):
            rec[k].append(-1 if k in ("r_idx", "lat_idx") else 0)
        rec["r_obj"].append(math.nan if a is None else a)
        rec["r_slack"].append(0.0)
        rec["r_wait"].append(0.0)
        rec["aff_kind"].append(kinds.index(backend_kind))
        rec["lat_val"].append(0.0)
        return a

    def setl(self, index, latency_s):
        orig_set(self, index, latency_s)
        rec["kind"].append(2)
        rec["op"].append(op_names.index(self.operation))
        rec["slack"].append([math.nan] * len(kinds))
        rec["alpha"].append(0.0)
        for k in ("avail", "supply", "flags", "min_batch", "r_code", "r_idx", "r_fill"):
            rec[k].append(-1 if k == "r_idx" else 0)
        for k in ("r_obj", "r_slack", "r_wait"):
            rec[k].append(0.0)
        rec["aff_kind"].append(-1)
        rec["lat_idx"].append(index)
        rec["lat_val"].append(float(self.lat[index]))

    conf.OpTable.select, conf.OpTable.affinity, conf.OpTable.set_latency = sel, aff, setl
    try:
        paths = pipe.decompose_paths(dag)
        run = man.PipelineRun(dag, ops, profiles, frames, sc, target, conf.TuningParams(
            alpha=sc.tuning.alpha, smoothing_beta=sc.tuning.smoothing_beta,
            dfp_count=sc.tuning.dfp_count, straggler_timeout_factor=sc.tuning.straggler_timeout_factor,
            cq_capacity=sc.tuning.cq_capacity), paths=paths, pipeline_name="video_branching")
        init_tables = {}
        for n in op_names:
            t = run.tables[n]
            init_tables[n] = {
                "config_id": [e.config_id for e in t.entries],
                "kind": [e.backend_kind for e in t.entries],
                "res": [e.resource_request for e in t.entries],
                "batch": [e.batch_size for e in t.entries],
                "lat": [e.latency_s for e in t.entries],
                "lat_init": [e.latency_initial_s for e in t.entries],
                "ref_index": t.ref_index,
                "ref_id": t.ref_entry.config_id,
            }
        report = run.run_to_completion()
    finally:
        conf.OpTable.select, conf.OpTable.affinity, conf.OpTable.set_latency = orig_select, orig_aff, orig_set
    out = {k: np.array(v) for k, v in rec.items()}
    out["slack"] = np.array(rec["slack"], dtype=np.float64)
    meta = {"kinds": kinds, "ops": op_names, "tables": init_tables, "target": target,
            "backends": [[b.kind, b.instance_count, b.resources_per_instance, b.price_rate] for b in sc.backends],
            "csv_row": report.csv_row(), "paths": [list(p) for p in paths]}
    out["meta_json"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    return out



# ---- 7. commit rounds (Configurator.pump_commits) -----------------------

def gen_commit_rounds(R, ref_root: Path, max_rounds=6000):
    """Record, for AMBER runs of the reference engine, each pump_commits round: per op with a
    speculated head the inputs of _commit_candidate (head fill / forced / id / speculated entry,
    buffered items, saturated kinds, the op's slack per kind) and its result, plus the winner
    (the invocation the round committed).  set_latency calls are recorded in the same order so a
    replay can keep the tables identical.  Everything is captured by wrapping the reference's own
    methods; no reference logic is restated here."""
    conf, man, pipe, prof, scen = R
    from slackpipe import workload

    bundle = ref_root / "scenarios" / "branching"
    dag, ops = pipe.load_pipeline(json.loads((bundle / "pipeline.json").read_text()))
    sc = scen.load_scenario(bundle / "scenario.json")
    frames = workload.load_trace(bundle / "trace.jsonl")
    profiles = {n: prof.profile_operation(o, sc, sc.tuning.samples_per_config) for n, o in ops.items()}
    kinds = sc.backend_kinds()
    op_names = sorted(dag.vertices)
    paths = pipe.decompose_paths(dag)
    runs = [(142.20064921472454, ()), (0.0, ()), (142.20064921472454, ("pbc",)),
            (142.20064921472454, ("eslc",))]
    C = {k: [] for k in ("round", "op", "fill", "forced", "inv", "spec_idx", "spec_kind", "spec_slack",
                         "spec_obj", "buffered", "full_mask", "slack", "r_idx", "r_fill", "r_slack",
                         "r_obj")}
    Rd = {k: [] for k in ("run", "seq", "winner_op", "winner_inv", "first_cand", "n_cand")}
    S = {k: [] for k in ("run", "seq", "op", "idx", "val")}
    run_meta = []
    orig_cc, orig_pump, orig_set = conf.Configurator._commit_candidate, conf.Configurator.pump_commits, \
        conf.OpTable.set_latency
    state = {"run": 0, "seq": 0, "open": None, "rounds": 0}

    def close(winner_inv=None, winner_op=-1):
        o = state["open"]
        if o is not None and o["n"] > 0:
            Rd["run"].append(state["run"])
            Rd["seq"].append(state["seq"])
            Rd["winner_op"].append(winner_op)
            Rd["winner_inv"].append(-1 if winner_inv is None else winner_inv)
            Rd["first_cand"].append(o["first"])
            Rd["n_cand"].append(o["n"])
            state["seq"] += 1
            state["rounds"] += 1
        state["open"] = None

    def cc(self, op, head, full_kinds, buffered):
        r = orig_cc(self, op, head, full_kinds, buffered)
        if state["rounds"] >= max_rounds:
            return r
        if state["open"] is None:
            state["open"] = {"first": len(C["op"]), "n": 0}
        sl = self.slack_by_kind(op)
        C["round"].append(len(Rd["run"]))
        C["op"].append(op_names.index(op))
        C["fill"].append(head.fill)
        C["forced"].append(int(head.forced))
        C["inv"].append(head.invocation_id)
        C["spec_idx"].append(head.spec_eidx)
        C["spec_kind"].append(kinds.index(head.spec_entry.backend_kind) if head.spec_entry is not None else -1)
        C["spec_slack"].append(float(head.spec_slack_s))
        C["spec_obj"].append(float(head.spec_objective))
        C["buffered"].append(int(buffered))
        C["full_mask"].append(sum(1 << kinds.index(k) for k in full_kinds))
        C["slack"].append([float(sl.get(k, math.nan)) for k in kinds])
        if r is None:
            C["r_idx"].append(-1); C["r_fill"].append(0); C["r_slack"].append(0.0); C["r_obj"].append(0.0)
        else:
            C["r_idx"].append(r[1]); C["r_fill"].append(r[2]); C["r_slack"].append(float(r[3]))
            C["r_obj"].append(float(r[4]))
        state["open"]["n"] += 1
        return r

    def pump(self, buffered_count, topup):
        close()
        return orig_pump(self, buffered_count, topup)

    def setl(self, index, latency_s):
        orig_set(self, index, latency_s)
        if state["rounds"] >= max_rounds:
            return
        close()
        S["run"].append(state["run"])
        S["seq"].append(state["seq"])
        S["op"].append(op_names.index(self.operation))
        S["idx"].append(index)
        S["val"].append(float(self.lat[index]))
        state["seq"] += 1

    class Log(list):
        def append(self, e):
            super().append(e)
            if e[1] == "commit" and state["open"] is not None and state["rounds"] < max_rounds:
                close(winner_inv=e[2], winner_op=op_names.index(e[3]))

    conf.Configurator._commit_candidate, conf.Configurator.pump_commits = cc, pump
    conf.OpTable.set_latency = setl
    try:
        for ri, (target, abl) in enumerate(runs):
            state.update(run=ri, open=None, rounds=0)
            run = man.PipelineRun(dag, ops, profiles, frames, sc, target, conf.TuningParams(
                alpha=sc.tuning.alpha, smoothing_beta=sc.tuning.smoothing_beta,
                dfp_count=sc.tuning.dfp_count, straggler_timeout_factor=sc.tuning.straggler_timeout_factor,
                cq_capacity=sc.tuning.cq_capacity), ablations=abl, paths=paths,
                pipeline_name="video_branching")
            run.configurator.decision_log = Log()
            run_meta.append({"target": target, "ablations": list(abl), "alpha": run.params.alpha,
                             "depths": [run.depths[o] for o in op_names],
                             "tables": {n: {"lat": [e.latency_s for e in run.tables[n].entries],
                                            "ref_index": run.tables[n].ref_index}
                                        for n in op_names}})
            run.run_to_completion()
            close()
    finally:
        conf.Configurator._commit_candidate, conf.Configurator.pump_commits = orig_cc, orig_pump
        conf.OpTable.set_latency = orig_set
    out = {f"c_{k}": np.array(v) for k, v in C.items()}
    out["c_slack"] = np.array(C["slack"], dtype=np.float64)
    out.update({f"r_{k}": np.array(v, dtype=np.int64) for k, v in Rd.items()})
    out.update({f"s_{k}": np.array(v) for k, v in S.items()})
    out["s_val"] = np.array(S["val"], dtype=np.float64)
    meta = {"kinds": kinds, "ops": op_names, "runs": run_meta, "max_rounds": max_rounds}
    out["meta_json"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    return out


# ---- 7b. speculate_from_buffer calls ---------------------------------

def gen_speculate_calls(R, ref_root: Path, max_calls=5000):
    """Record, for AMBER runs of the reference engine, each Configurator.speculate_from_buffer
    call: its inputs (op, buffered items, upstream supply, clock, the op's path ratios, the
    forced / batching-hold state, and the SQ / CQ weight dicts in their order) and what it did
    (every invocation formed: entry, fill, slack, objective; the delay it stopped on).
    set_latency calls are recorded in the same order so a replay can keep the tables identical.
    Everything is captured by wrapping the reference's own methods."""
    conf, man, pipe, prof, scen = R
    from slackpipe import workload

    bundle = ref_root / "scenarios" / "branching"
    dag, ops = pipe.load_pipeline(json.loads((bundle / "pipeline.json").read_text()))
    sc = scen.load_scenario(bundle / "scenario.json")
    frames = workload.load_trace(bundle / "trace.jsonl")
    profiles = {n: prof.profile_operation(o, sc, sc.tuning.samples_per_config) for n, o in ops.items()}
    kinds = sc.backend_kinds()
    op_names = sorted(dag.vertices)
    paths = pipe.decompose_paths(dag)
    runs = [(142.20064921472454, ()), (116.30975052233568, ()), (142.20064921472454, ("dfp",))]
    C = {k: [] for k in ("run", "seq", "op", "n", "supply", "now", "target", "rmin", "rmax", "flags",
                         "w_first", "w_n", "d_first", "d_n", "delay_idx", "delay_wait", "slack0")}
    W = {k: [] for k in ("kind", "queue", "tab", "eidx", "count")}
    D = {k: [] for k in ("idx", "fill", "slack", "obj")}
    S = {k: [] for k in ("run", "seq", "op", "idx", "val")}
    run_meta = []
    orig_spec, orig_enq = conf.Configurator.speculate_from_buffer, conf.Configurator._enqueue_speculated
    orig_sel, orig_set = conf.OpTable.select, conf.OpTable.set_latency
    state = {"run": 0, "seq": 0, "calls": 0, "in": False, "last": None}

    def spec(self, op, buffer):
        if state["calls"] >= max_calls:
            return orig_spec(self, op, buffer)
        t = self.tables[op]
        hold = self.holds.get(op)
        now = self._clock()
        forced = ("dfp" not in self.ablations and t.ref_index >= 0
                  and self.completed_ref[op] < self.params.dfp_count)
        flags = (1 if "sdb" not in self.ablations else 0) | (2 if forced else 0) | \
                (4 if hold is not None and now >= hold.deadline_s else 0)
        ratios = self._path_ratios(op)
        # the first iteration's slack is whatever slack_by_kind returns now — its cache is keyed
        # by the weight version only, so it may carry an earlier clock (configurator.py:526-529);
        # later iterations recompute after every _weights_add bump with the current clock
        sl0 = self.slack_by_kind(op)
        C["slack0"].append([float(sl0[k]) for k in kinds])
        C["run"].append(state["run"]); C["seq"].append(state["seq"])
        C["op"].append(op_names.index(op)); C["n"].append(len(buffer))
        C["supply"].append(int(self._supply(op))); C["now"].append(float(now))
        C["target"].append(float(self.target_s)); C["rmin"].append(min(ratios))
        C["rmax"].append(max(ratios)); C["flags"].append(flags)
        C["w_first"].append(len(W["kind"]))
        for q, table in enumerate((self._sq_weight, self._cq_weight)):
            for k in kinds:
                for (o, e), c in table[k].items():
                    W["kind"].append(kinds.index(k)); W["queue"].append(q)
                    W["tab"].append(op_names.index(o)); W["eidx"].append(e); W["count"].append(c)
        C["w_n"].append(len(W["kind"]) - C["w_first"][-1])
        C["d_first"].append(len(D["idx"]))
        state["in"], state["last"] = True, None
        try:
            r = orig_spec(self, op, buffer)
        finally:
            state["in"] = False
        C["d_n"].append(len(D["idx"]) - C["d_first"][-1])
        last = state["last"]
        if buffer and last is not None and last.kind == "delay":
            C["delay_idx"].append(last.entry_index); C["delay_wait"].append(float(last.wait_budget_s))
        else:
            C["delay_idx"].append(-1); C["delay_wait"].append(0.0)
        state["seq"] += 1
        state["calls"] += 1
        return r

    def enq(self, inv, decision):
        if state["in"]:
            D["idx"].append(decision.entry_index); D["fill"].append(inv.fill)
            D["slack"].append(float(decision.slack_s)); D["obj"].append(float(decision.objective_value))
        return orig_enq(self, inv, decision)

    def sel(self, *a, **kw):
        d = orig_sel(self, *a, **kw)
        if state["in"]:
            state["last"] = d
        return d

    def setl(self, index, latency_s):
        orig_set(self, index, latency_s)
        if state["calls"] >= max_calls:
            return
        S["run"].append(state["run"]); S["seq"].append(state["seq"])
        S["op"].append(op_names.index(self.operation)); S["idx"].append(index)
        S["val"].append(float(self.lat[index]))
        state["seq"] += 1

    conf.Configurator.speculate_from_buffer, conf.Configurator._enqueue_speculated = spec, enq
    conf.OpTable.select, conf.OpTable.set_latency = sel, setl
    try:
        for ri, (target, abl) in enumerate(runs):
            state.update(run=ri, calls=0)
            run = man.PipelineRun(dag, ops, profiles, frames, sc, target, conf.TuningParams(
                alpha=sc.tuning.alpha, smoothing_beta=sc.tuning.smoothing_beta,
                dfp_count=sc.tuning.dfp_count, straggler_timeout_factor=sc.tuning.straggler_timeout_factor,
                cq_capacity=sc.tuning.cq_capacity), ablations=abl, paths=paths,
                pipeline_name="video_branching")
            run_meta.append({"target": target, "ablations": list(abl), "alpha": run.params.alpha,
                             "pool": [run.configurator._pool[k] for k in kinds],
                             "tables": {n: {"lat": [e.latency_s for e in run.tables[n].entries],
                                            "ref_index": run.tables[n].ref_index}
                                        for n in op_names}})
            run.run_to_completion()
    finally:
        conf.Configurator.speculate_from_buffer, conf.Configurator._enqueue_speculated = orig_spec, orig_enq
        conf.OpTable.select, conf.OpTable.set_latency = orig_sel, orig_set
    out = {f"c_{k}": np.array(v) for k, v in C.items()}
    for k in ("now", "target", "rmin", "rmax", "delay_wait", "slack0"):
        out[f"c_{k}"] = np.array(C[k], dtype=np.float64)
    out.update({f"w_{k}": np.array(v, dtype=np.int64) for k, v in W.items()})
    out.update({f"d_{k}": np.array(v) for k, v in D.items()})
    out["d_slack"] = np.array(D["slack"], dtype=np.float64)
    out["d_obj"] = np.array(D["obj"], dtype=np.float64)
    out.update({f"s_{k}": np.array(v) for k, v in S.items()})
    out["s_val"] = np.array(S["val"], dtype=np.float64)
    meta = {"kinds": kinds, "ops": op_names, "runs": run_meta, "max_calls": max_calls}
    out["meta_json"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    return out


# ---- 8. metadata directory (profile ingest) ---------------------------

def gen_metadata_amber(R, ref_root: Path):
    """The reference's own MetadataStore files for the AMBER pipeline: one configspec JSON per
    operation (profile_operation of the bundled scenario) and the decomposed path set."""
    conf, man, pipe, prof, scen = R
    import shutil

    bundle = ref_root / "scenarios" / "branching"
    doc = json.loads((bundle / "pipeline.json").read_text())
    dag, ops = pipe.load_pipeline(doc)
    sc = scen.load_scenario(bundle / "scenario.json")
    out_dir = HERE / "metadata_amber"
    if out_dir.exists():
        shutil.rmtree(out_dir)
    store = prof.MetadataStore(out_dir)
    for name, op in sorted(ops.items()):
        store.ensure_profile(op, sc, sc.tuning.samples_per_config)
    store.store_paths(pipe.pipeline_content_hash(doc), pipe.decompose_paths(dag))
    return None

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    R = _ref_modules(a.ref)
    ref_root = Path(a.ref).parent
    jobs = {
        "select_cases": lambda: gen_select_cases(R),
        "synth_sample": lambda: gen_synth(R),
        "slack_cases": lambda: gen_slack(R),
        "feedback_cases": lambda: gen_feedback(R),
        "queue_cases": lambda: gen_queue(R),
        "amber_trace": lambda: gen_amber(R, ref_root),
        "commit_rounds": lambda: gen_commit_rounds(R, ref_root),
        "speculate_calls": lambda: gen_speculate_calls(R, ref_root),
        "metadata_amber": lambda: gen_metadata_amber(R, ref_root),
    }
    for name, fn in jobs.items():
        if a.only and name not in a.only.split(","):
            continue
        out = fn()
        if out is None:  # job wrote its own files
            print(name, "written")
            continue
        np.savez_compressed(HERE / f"{name}.npz", **out)
        print(name, {k: v.shape for k, v in list(out.items())[:6]}, "...")


if __name__ == "__main__":
    main()
