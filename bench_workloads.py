"""BASELINE.json configs 3-5 on B200 (invoked as `python bench.py --workload c3|c4|c5`).

c3  deep DAG: 64 ops, 845 edges (~3.3e9 decomposed paths, which the reference cannot
    enumerate), 100,000 pipeline instances, 4 backend kinds: Alg. 1 slack for every
    (instance, op, kind) through K1.  CPU baseline: the exact forward-DP restatement (oracle,
    labelled "restatement, not reference") on all host cores over a 1,000-instance sample.
c4  latency-target sweep x replicas on the AMBER pipeline: 10,000 replicas x 5 targets
    (0.5x..10x the fast-anchor latency) x 64 snapshots; per snapshot K1 (7 ops x 4 kinds) feeds
    K2 directly on the device (one decision per op) — 22.4M decisions per step.
commit  batched commit step: 65,536 independent Configurator.pump_commits
    rounds over the 7 AMBER operations per call (one K2 re-selection of every head + a warp
    key reduction per round); CPU baseline: oracle/commit.py round_winner on all host cores.
c5  online mode: 2^24 invocations x 16,384 configurations in 256 batches of 65,536; every batch is
    decided against the batch-start profile snapshot, the chosen configurations produce noisy
    latency observations, and K3 folds them back (the next batch's plan is rebuilt on device).
All numbers are device time (CUDA events), inputs resident in HBM; one JSON line on stdout.
"""
from __future__ import annotations

import json
import math
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def _events(torch, n):
    return [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]


def _flush_factory(torch, dev):
    buf = torch.ones(256 << 20, dtype=torch.uint8, device=dev)
    return lambda: buf.max()


def _dist(torch):
    """(rank, world, local) — NCCL process group when launched under torchrun (one rank per GPU)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 and not torch.distributed.is_initialized():
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def _tmax(torch, t: float, dev) -> float:
    """Device time of the slowest rank."""
    if not (torch.distributed.is_available() and torch.distributed.is_initialized()):
        return t
    tt = torch.tensor([t], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    return float(tt.item())


def _barrier(torch):
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.barrier()


def _clocks(local):
    """NVML clock / throttle-reason sampler around a timed region (bench.ClockSampler)."""
    from bench import ClockSampler

    return ClockSampler(local)


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


# ---- c1: the AMBER drop-in, one call at a time ----------------------------------------------

C1_REFERENCE_DECISIONS_PER_S = 18468.0  # /root/reference/pkg/test_output.txt:171 (whole engine)


def _c1_calls():
    with np.load(ROOT / "tests" / "golden" / "amber_trace.npz") as z:
        d = {k: z[k] for k in z.files}
    meta = json.loads(bytes(d["meta_json"]).decode())
    return d, meta


def _c1_replay_cpu(d, meta, n):
    """The reference's per-call path on the CPU: the numpy restatement of OpTable.select /
    affinity / set_latency (oracle/optable.py), single-threaded like the reference engine."""
    import math

    from oracle import commit as oc
    from oracle import optable

    tabs = oc.amber_tables(meta)
    kind, op, slack, alpha = d["kind"], d["op"], d["slack"], d["alpha"]
    t0 = time.perf_counter()
    for i in range(n):
        t = tabs[op[i]]
        k = kind[i]
        if k == 2:
            t.lat[int(d["lat_idx"][i])] = float(d["lat_val"][i])
        elif k == 1:
            optable.affinity(t, int(d["aff_kind"][i]), np.nan_to_num(slack[i]), float(alpha[i]))
        else:
            fl = int(d["flags"][i])
            optable.select(t, np.nan_to_num(slack[i]), float(alpha[i]), int(d["avail"][i]),
                           allow_delay=bool(fl & 1), upstream_supply=int(d["supply"][i]),
                           excluded_mask=(fl >> 8) & 0xFF, min_batch=int(d["min_batch"][i]))
    return time.perf_counter() - t0


def run_c1(args):
    """BASELINE config 1: every OpTable call the reference engine made on the AMBER scenario at
    the 50% target (43,859 select, 9,962 affinity, 7,726 set_latency, in call order), replayed
    one at a time through the drop-in object API — the path the unmodified reference engine
    drives — on the B200; every result is compared with the recorded reference result.  Wall
    clock (the per-call host work is part of the path)."""
    import math

    import torch

    import paper_2102_01887_b200 as sp

    rank, world, local = _dist(torch)
    if rank != 0:
        return
    d, meta = _c1_calls()
    kinds = meta["kinds"]
    n = len(d["kind"])
    bits = lambda x: np.float64(x).view(np.uint64)

    def replay(check):
        tabs = _amber_tables(sp, meta)
        kind, op, slack, alpha = d["kind"], d["op"], d["slack"], d["alpha"]
        sdicts = [{k: float(v) for k, v in zip(kinds, row) if not math.isnan(v)} for row in slack]
        bad = 0
        ctx = sp.get_context(local)
        l0 = ctx.launch_count
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(n):
            t = tabs[op[i]]
            k = kind[i]
            if k == 2:
                t.set_latency(int(d["lat_idx"][i]), float(d["lat_val"][i]))
            elif k == 1:
                a = t.affinity(kinds[d["aff_kind"][i]], sdicts[i], float(alpha[i]))
                if check:
                    exp = d["r_obj"][i]
                    bad += not ((a is None and math.isnan(exp)) or (a is not None and bits(a) == bits(exp)))
            else:
                fl = int(d["flags"][i])
                ex = frozenset(kk for j, kk in enumerate(kinds) if (fl >> (8 + j)) & 1)
                dec = t.select(sdicts[i], float(alpha[i]), int(d["avail"][i]), allow_delay=bool(fl & 1),
                               upstream_supply=int(d["supply"][i]), excluded_kinds=ex,
                               min_batch=int(d["min_batch"][i]))
                if check:
                    rc = d["r_code"][i]
                    if rc == 0:
                        bad += dec is not None
                    else:
                        bad += not (dec is not None and dec.entry_index == d["r_idx"][i]
                                    and dec.fill == d["r_fill"][i]
                                    and dec.kind == ("delay" if rc == 2 else "assign")
                                    and bits(dec.objective_value) == bits(d["r_obj"][i])
                                    and bits(dec.slack_s) == bits(d["r_slack"][i])
                                    and bits(dec.wait_budget_s) == bits(d["r_wait"][i]))
        dt = time.perf_counter() - t0
        launches = ctx.launch_count - l0
        for t in tabs:
            t.close()
        return dt, bad, launches

    replay(False)  # warm-up: module load, staging allocation
    times = []
    bad = launches = 0
    for rep in range(max(1, args.steps // 10)):
        dt, b, launches = replay(rep == 0)
        bad += b
        times.append(dt)
    dt = min(times)
    n_sel = int((d["kind"] == 0).sum())
    cpu = None
    if not args.no_cpu_baseline:
        cdt = _c1_replay_cpu(d, meta, n)
        cpu = {"value": n_sel / cdt, "unit": "select decisions/s", "cores": 1, "kind": "port",
               "calls_per_s": n / cdt,
               "sample": f"all {n} calls, oracle/optable.py numpy restatement of OpTable.select / "
                         f"affinity / set_latency, one call at a time on one core (the reference "
                         f"engine is single-threaded)"}
    line = {
        "workload": "c1", "metric": "OpTable calls replayed one at a time through the drop-in API",
        "unit": "select decisions/s", "value": n_sel / dt, "calls_per_s": n / dt,
        "us_per_call": 1e6 * dt / n, "n_gpus": 1, "steps": len(times),
        "config": {"scenario": "AMBER (branching), 50% target, recorded reference OpTable calls",
                   "calls": n, "selects": n_sel, "affinity": int((d["kind"] == 1).sum()),
                   "set_latency": int((d["kind"] == 2).sum()),
                   "path": "OpTable.select / affinity / set_latency -> libslackpipe_b200 (pinned "
                           "staging block, one launch + one sync per call; AUTO takes the scan "
                           "while a set_latency has left the staircase plan stale)"},
        "parity": {"calls_checked": n - int((d["kind"] == 2).sum()), "mismatches": bad,
                   "result": "bit-identical to the recorded reference results" if bad == 0 else "MISMATCH"},
        "gpu_launches": launches,
        "reference_engine_decisions_per_s": {"value": C1_REFERENCE_DECISIONS_PER_S,
                                             "source": "reference pkg/test_output.txt:171 (whole "
                                                       "engine run, other hardware)"},
        "cpu_baseline": cpu,
        "whole_run": _c1_whole_run(args),
    }
    return line


def _c1_whole_run(args):
    """Config 1 as the reference runs it: ONE complete AMBER run at the 50 % target (3,000
    frames, 15,290 decisions), PipelineRun.run_to_completion through the device drop-in
    (engine.PipelineRun: setup, H2D, one warp running the whole event loop, D2H of the report,
    the decision log and the final tables) — wall clock, against oracle/engine.py (the Python
    restatement of the reference engine) on one core; parity against the reference's own run."""
    sys.path.insert(0, str(ROOT / "tests"))
    import des_cases as dc
    from paper_2102_01887_b200.engine import PipelineRun

    case = dc.runs()[3]
    doc, dag, sc, profiles, paths, frames = dc.bundle("branching")
    spec = dc.run_spec(case)
    times, rep, run = [], None, None
    for _ in range(4):
        run = PipelineRun(dag, {}, profiles, frames, sc, float(case["target"]), spec.params,
                          paths=paths, pipeline_name=doc["name"])
        t0 = time.perf_counter()
        rep = run.run_to_completion()
        times.append(time.perf_counter() - t0)
    ok = (dc.log_digest(run.decision_log) == case["expect"]["log_sha256"]
          and rep.csv_row().split(",")[1:] == case["expect"]["csv_row"].split(",")[1:])
    dt = min(times[1:])
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import engine as oe

        p = spec.params
        c0 = time.perf_counter()
        oe.Engine(dag, profiles, frames, sc, float(case["target"]),
                  oe.Params(p.alpha, p.cq_capacity, p.dfp_count, p.straggler_timeout_factor,
                            p.smoothing_beta), seed=sc.seed, paths=paths).run()
        cdt = time.perf_counter() - c0
        cpu = {"value": rep.decision_count / cdt, "unit": "decisions/s", "cores": 1, "kind": "port",
               "seconds_per_run": cdt,
               "sample": "the same run through oracle/engine.py (Python restatement of PipelineRun / "
                         "BackendSim / Configurator, pinned to the reference), one core"}
    return {"metric": "one complete AMBER run (PipelineRun.run_to_completion) through the device drop-in",
            "unit": "decisions/s", "value": rep.decision_count / dt, "seconds_per_run": dt,
            "decisions": rep.decision_count, "kernel": "k_des_run_warp (one warp runs the whole event loop)",
            "e2e": True, "note": "wall clock of run_to_completion: run-description upload, trace encoding, H2D, the run, D2H of "
                                 "report + 15,290-row decision log + final tables",
            "parity": {"result": "decision log sha256 and CSV row equal the reference's run" if ok
                       else "MISMATCH", "csv_row": rep.csv_row()},
            "cpu_baseline": cpu}


# ---- c3 -------------------------------------------------------------------------------------

def _c3_cpu_worker(args):
    from oracle import slack as osl

    order, preds, term, vcol, ref, T, now, Q = args
    out = []
    for i in range(len(T)):
        refo = ref[i][vcol]
        for s in range(len(order)):
            lo, hi = osl.dp_ratios(order, preds, term, refo, s)
            for k in range(Q.shape[1]):
                out.append(osl.dp_slack(lo, hi, (T[i] - now[i]) - Q[i, k]))
    return len(out)


def run_c3(args):
    import torch

    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    from paper_2102_01887_b200.shard import shard_range

    rank, world, local = _dist(torch)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = sp.get_context(local)
    ctx.set_stream(stream.cuda_stream)
    dag = synth.deep_dag()
    I, K = 100_000, 4  # instances per GPU (weak scaling): rank r owns instance rows [r*I, (r+1)*I)
    ref_all, T_all, now_all, Q_all = synth.deep_dag_instances(dag, I * world, K=K)
    a, b = shard_range(I * world, rank, world)
    ref, T, now, Q = ref_all[a:b], T_all[a:b], now_all[a:b], Q_all[a:b]
    g = sp.SlackGraph.from_dag(dag)
    V = len(dag.vertices)
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in
         (("ref", ref), ("T", T), ("now", now), ("Q", Q))}
    out = {"slack": torch.empty((I, V, K), dtype=torch.float64, device=dev)}
    flush = _flush_factory(torch, dev)
    for _ in range(args.warmup):
        g.slack_batch(d["ref"], d["T"], d["now"], d["Q"], out=out)
    torch.cuda.synchronize(dev)
    _barrier(torch)
    evs = _events(torch, args.steps)
    l0 = ctx.launch_count
    with _clocks(local) as clk:
        for i in range(args.steps):
            flush()
            evs[i][0].record(stream)
            g.slack_batch(d["ref"], d["T"], d["now"], d["Q"], out=out)
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
    ms = [x.elapsed_time(y) for x, y in evs]
    launches = ctx.launch_count - l0
    t = _tmax(torch, sum(ms) / 1e3, dev)
    vals = args.steps * I * V * K * world
    got = out["slack"].cpu().numpy()
    # checker: every slack value of this rank's launch against the C forward-DP restatement
    from oracle import cselect

    exp = cselect.slack_dp(dag, ref, T, now, Q)
    bad = torch.tensor([int(np.count_nonzero(got.view(np.uint64) != exp.view(np.uint64))), got.size],
                       dtype=torch.int64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(bad)
    bad = bad.cpu().tolist()
    parity = {"slack_values": bad[1], "mismatches": bad[0],
              "result": ("bit-identical vs oracle_slack_dp (C forward-DP restatement of Alg. 1, "
                         "SURVEY.md §8(c))" if bad[0] == 0 else "MISMATCH"),
              "checked_on": f"all {world} rank(s), every (instance, op, kind) of the step"}
    # the same step through K1's per-source forward DP (SP_K1_CERT=0), reported beside it
    ctx.set_option("SP_K1_CERT", 1)  # off
    try:
        evf = _events(torch, args.steps)
        for i in range(args.steps):
            flush()
            evf[i][0].record(stream)
            g.slack_batch(d["ref"], d["T"], d["now"], d["Q"], out=out)
            evf[i][1].record(stream)
        torch.cuda.synchronize(dev)
    finally:
        ctx.set_option("SP_K1_CERT", 0)
    fwd_ms = statistics.median([x.elapsed_time(y) for x, y in evf])
    if rank != 0:
        return
    bytes_inst = 8 * V + 16 + 8 * K + 8 * V * K
    # CPU: the exact DP restatement on all host cores over a bounded sample
    order = dag.topological_order()
    pos = {v: j for j, v in enumerate(order)}
    preds = [[pos[p] for p in dag.predecessors(v)] for v in order]
    term = [not dag.successors(v) for v in order]
    vcol = [dag.vertices.index(v) for v in order]
    cores = os.cpu_count() or 1
    S = args.c3_cpu_instances
    n_cpu, cpu_t = 0, 1.0
    if world == 1:  # the CPU baseline runs on rank 0 at N=1 only
        import multiprocessing as mp

        chunks = np.array_split(np.arange(S), cores)
        work = [(order, preds, term, vcol, ref[c], T[c], now[c], Q[c]) for c in chunks if len(c)]
        with mp.get_context("fork").Pool(len(work)) as pool:  # forked outside the timed map
            pool.map(_c3_cpu_worker, [w[:4] + tuple(x[:1] for x in w[4:]) for w in work])
            t0 = time.perf_counter()
            n_cpu = sum(pool.map(_c3_cpu_worker, work))
            cpu_t = time.perf_counter() - t0
    line = {
        "workload": "c3", "metric": "Alg. 1 slack values (instance x op x kind) / s", "unit": "slack/s",
        "value": vals / t, "ms_per_step": 1e3 * t / args.steps, "steps": args.steps, "n_gpus": world,
        "scaling": "weak",
        "config": {"ops": V, "edges": len(dag.edges), "instances_per_gpu": I, "kinds": K,
                   "decomposed_paths": "~3.3e9 (not enumerable by the reference)",
                   "parallelism": f"instances sharded over {world} GPU(s), no collective"},
        "instances_per_s": args.steps * I * world / t,
        "roofline": {"bound": "issue / shared-memory latency (K1c: one backward pass + per-source "
                              "extremal-path walks, DESIGN.md §5)",
                     "hbm_bytes_per_instance": bytes_inst,
                     "hbm_frac": (args.steps * I * world * bytes_inst / t / 1e9) / (world * _peaks())},
        "forward_dp_step_ms": fwd_ms,
        "gpu_launches": launches,
        "parity": parity,
        "cpu_baseline": None if world > 1 else {"value": n_cpu / cpu_t, "unit": "slack/s", "cores": cores,
                         "kind": "restatement (the reference cannot run this DAG)",
                         "sample": f"{S} instances, oracle/slack.py dp_ratios on {cores} processes"},
        "step_ms": {"median": statistics.median(ms), "min": min(ms), "max": max(ms)},
        "clocks": clk.summary(),
    }
    return line


# ---- c4 -------------------------------------------------------------------------------------

def _amber_tables(sp, meta):
    sc = sp.Scenario("branching", tuple(sp.BackendSpec(k, n, r, p) for k, n, r, p in meta["backends"]))
    tabs = []
    for name in meta["ops"]:
        m = meta["tables"][name]
        ents = [sp.ConfigEntry(cid, k, {}, b, r, lat, li) for cid, k, r, b, lat, li in
                zip(m["config_id"], m["kind"], m["res"], m["batch"], m["lat"], m["lat_init"])]
        if m["ref_index"] < 0:
            res = int(m["ref_id"].split("-r", 1)[1].split("-", 1)[0])
            ents.append(sp.ConfigEntry(m["ref_id"], "cpu", {}, 1, res, 1.0, 1.0, schedulable=False))
        tabs.append(sp.OpTable(sp.ConfigSpec(name, ents, m["ref_id"]), sc, kinds=meta["kinds"]))
    return tabs


def _c4_cpu_worker(a):
    """Oracle per decision: slack_by_kind (configurator.py:526-543 over the path list) of each op
    of each instance, then OpTable.select (239-300).  Returns (instances, ops, 2) of (idx, code)."""
    (meta, paths, value_names, alpha), inst, ref, target, now, Q, avail, supply = a
    from oracle import commit as oc
    from oracle import optable
    from oracle import slack as osl

    otabs = oc.amber_tables(meta)
    kinds = meta["kinds"]
    out = np.zeros((len(inst), len(meta["ops"]), 2), np.int64)
    for r in range(len(inst)):
        refmap = dict(zip(value_names, ref[r]))
        q = dict(zip(kinds, Q[r]))
        for j, op in enumerate(meta["ops"]):
            sl = osl.slack_by_kind(op, kinds, target_s=float(target[r]), now=float(now[r]),
                                   queueing=q, paths=paths, ref=refmap)
            res = optable.select(otabs[j], np.array([sl[k] for k in kinds]), alpha,
                                 int(avail[r, j]), allow_delay=True,
                                 upstream_supply=int(supply[r, j]))
            out[r, j] = (res[1], res[0])
    return out


def c4_full_parity(meta, paths_cols, ops_ref, sw, alpha, got_idx, got_code, got_obj=None):
    """Checker: every decision of a config-4 step against the C oracle — literal Alg. 1 over the
    AMBER path list (oracle_slack_paths, configurator.py:415-417, 493-543) then the literal
    OpTable.select scan (oracle_select_batch, configurator.py:239-300).  Returns a parity dict."""
    from oracle import commit as oc
    from oracle import cselect

    I, V = sw.ref.shape
    K = sw.Q.shape[1]
    sl = cselect.slack_paths(sw.ref, sw.target, sw.now, sw.Q, paths_cols)
    otabs = oc.amber_tables(meta)
    N = I * V
    exp = cselect.select_batch(otabs, sl.reshape(N, K), alpha, sw.avail.reshape(-1),
                               sw.supply.reshape(-1), np.ones(N, np.int32), np.ones(N, np.uint32),
                               op=np.tile(np.arange(V, dtype=np.int32), I))
    bad_idx = int(np.count_nonzero(exp["idx"] != got_idx))
    bad_code = int(np.count_nonzero(exp["code"] != (got_code & 3)))
    res = {"decisions": int(N), "instances": int(I), "index_mismatches": bad_idx,
           "kind_code_mismatches": bad_code}
    if got_obj is not None:
        some = exp["code"] != 0
        res["objective_mismatches"] = int(np.count_nonzero(
            exp["obj"][some].view(np.uint64) != got_obj[some].view(np.uint64)))
    res["result"] = ("bit-identical" if not any(v for k, v in res.items() if k.endswith("mismatches"))
                     else "MISMATCH")
    return res


def _c4_meta():
    with np.load(ROOT / "tests" / "golden" / "amber_trace.npz") as z:
        meta = json.loads(bytes(z["meta_json"]).decode())
    ops = meta["ops"]
    ref0 = np.array([meta["tables"][o]["lat"][meta["tables"][o]["ref_index"]]
                     if meta["tables"][o]["ref_index"] >= 0 else 1.0 for o in ops])
    paths_cols = [[ops.index(n) for n in p] for p in meta["paths"]]
    return meta, ops, ref0, paths_cols


def run_c4(args):
    import torch

    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth
    from paper_2102_01887_b200.shard import shard_range

    meta, ops, ref0, paths_cols = _c4_meta()
    rank, world, local = _dist(torch)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = sp.get_context(local)
    ctx.set_stream(stream.cuda_stream)
    tabs = _amber_tables(sp, meta)
    V, K = len(ops), len(meta["kinds"])
    g = sp.SlackGraph.from_paths([tuple(p) for p in meta["paths"]], ops)
    vpos = [ops.index(n) for n in g.value_names]  # graph value order -> op column
    mults, S = synth.SWEEP_MULTS, synth.SWEEP_SNAPSHOTS
    # strong scaling: the job is R replicas in total (BASELINE config 4: 10k replicas sharded
    # over the GPUs); rank g owns the contiguous replica range shard_range(R, g, G)
    R = args.c4_replicas
    r0, r1 = shard_range(R, rank, world)
    sw = synth.amber_sweep(ref0, K, r0, r1)
    I = (r1 - r0) * len(mults) * S
    N = I * V
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    d = {"ref": T(sw.ref[:, vpos]), "target": T(sw.target), "now": T(sw.now), "Q": T(sw.Q),
         "avail": T(sw.avail.reshape(-1)), "supply": T(sw.supply.reshape(-1)),
         "mb": T(np.ones(N, np.int32)), "flags": T(np.ones(N, np.int32)),
         "op": T(np.tile(np.arange(V, dtype=np.int32), I))}
    slack = torch.empty((I, V, K), dtype=torch.float64, device=dev)
    out = {k: torch.empty(N, dtype=dt, device=dev) for k, dt in
           (("idx", torch.int32), ("code", torch.int32), ("fill", torch.int32),
            ("obj", torch.float64), ("slack", torch.float64), ("wait", torch.float64))}
    alpha = 100.0
    for t in tabs:
        t.prepare(alpha)
    torch.cuda.synchronize(dev)

    def step_two_kernels():  # K1 writes slack[I][V][K], K2 reads it back
        g.slack_batch(d["ref"], d["target"], d["now"], d["Q"], out={"slack": slack})
        sp.select_batch(tabs, slack.view(N, K), alpha, d["avail"], upstream_supply=d["supply"],
                        min_batch=d["mb"], flags=d["flags"], op=d["op"], out=out)

    def step():  # K1 -> K2 fused: the slack never leaves registers
        g.slack_select_batch(tabs, alpha, d["ref"], d["target"], d["now"], d["Q"], d["avail"],
                             upstream_supply=d["supply"], min_batch=d["mb"], flags=d["flags"],
                             out=out)

    flush = _flush_factory(torch, dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    _barrier(torch)
    evs = _events(torch, args.steps)
    l0 = ctx.launch_count
    with _clocks(local) as clk:
        for i in range(args.steps):
            flush()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
    ms = [a.elapsed_time(b) for a, b in evs]
    t = _tmax(torch, sum(ms) / 1e3, dev)
    codes = torch.bincount(out["code"] & 3, minlength=3)
    launches = ctx.launch_count - l0
    got = {k: out[k].cpu().numpy() for k in ("idx", "code", "obj")}
    # the unfused K1 + K2 pair on the same inputs, for comparison
    for _ in range(2):
        step_two_kernels()
    ev2 = _events(torch, args.steps)
    for i in range(args.steps):
        flush()
        ev2[i][0].record(stream)
        step_two_kernels()
        ev2[i][1].record(stream)
    torch.cuda.synchronize(dev)
    ms2 = [a.elapsed_time(b) for a, b in ev2]
    # checker: every decision of this rank's shard against the C oracle (full N)
    parity = c4_full_parity(meta, paths_cols, ops, sw, alpha, got["idx"], got["code"], got["obj"])
    bad = torch.tensor([parity["index_mismatches"] + parity["kind_code_mismatches"]
                        + parity.get("objective_mismatches", 0), parity["decisions"]],
                       dtype=torch.int64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(codes)
        torch.distributed.all_reduce(bad)
    codes = codes.cpu().tolist()
    bad = bad.cpu().tolist()
    if rank != 0:
        return
    parity = {"decisions": bad[1], "mismatches": bad[0],
              "result": "bit-identical (index, kind code, objective) vs C oracle: literal "
                        "_path_ratios/slack_by_kind over the path list + OpTable.select scan"
                        if bad[0] == 0 else "MISMATCH",
              "checked_on": f"all {world} rank(s), every decision of the step"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = _c4_cpu_baseline(meta, g, alpha, sw, V)
    evals_per_inst = sum(len(x.entries) for x in tabs)
    Itot = R * len(mults) * S
    line = {
        "workload": "c4", "metric": "config decisions/s (K1 slack -> K2 select fused on device)",
        "unit": "decisions/s", "value": args.steps * Itot * V / t, "ms_per_step": 1e3 * t / args.steps,
        "steps": args.steps, "warmup": args.warmup, "n_gpus": world, "scaling": "strong",
        "evals_per_s": args.steps * Itot * evals_per_inst / t,
        "config": {"replicas": R, "targets_x_cp_min": list(mults), "snapshots": S,
                   "instances": Itot, "ops": V, "kinds": K, "decisions_per_step": Itot * V,
                   "cp_min": synth.SWEEP_CP_MIN,
                   "inputs": "synth.amber_sweep: per (replica r, target m) numpy seed r*5+m draws Q ~ "
                             "Exp(0.02 T), ref drift exp(N(0,0.2)), avail U{1..64}, supply U{0..64}",
                   "l2": "L2 flushed (256 MB read sweep) before every timed step",
                   "parallelism": f"{R} replicas sharded contiguously over {world} GPU(s); decision "
                                  "counters all-reduced"},
        "decision_mix": {"none": codes[0], "assign": codes[1], "delay": codes[2]},
        "gpu_launches": launches,
        "step_ms": {"median": statistics.median(ms), "min": min(ms), "max": max(ms)},
        "kernel": "k_slack_select (K1 -> K2 fused, sp_slack_select_batch)",
        "roofline": (lambda b: {"bound": "hbm", "achieved": b / (t / args.steps) / 1e9, "peak": _peaks(),
                                "unit": "GB/s", "frac": b / (t / args.steps) / 1e9 / _peaks(),
                                "algorithmic_bytes_per_step": b,
                                "bytes_model": "per instance 8V ref + 16 (target, now) + 8K Q, per "
                                               "decision 16 B in + 36 B out (468 B per AMBER instance)"})(
            Itot * (8 * V + 16 + 8 * K + V * (16 + 36))),
        "two_kernel_step_ms": {"median": statistics.median(ms2), "min": min(ms2),
                               "note": "k_slack then k_select_plan, slack through HBM"},
        "parity": parity,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    return line


def _c4_cpu_baseline(meta, g, alpha, sw, V):
    """The reference's per-decision CPU path (oracle restatement: slack_by_kind over the path
    list + OpTable.select per decision) on all host cores; the pool is forked and warmed
    before the timed map."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    work_meta = (meta, [tuple(p) for p in meta["paths"]], g.value_names, alpha)
    vpos = [meta["ops"].index(n) for n in g.value_names]
    S_cpu = 60 * cores
    sl = np.array_split(np.arange(S_cpu), cores)
    jobs = [(work_meta, a, sw.ref[a][:, vpos], sw.target[a], sw.now[a], sw.Q[a], sw.avail[a],
             sw.supply[a]) for a in sl if len(a)]
    with mp.get_context("fork").Pool(len(jobs)) as pool:
        pool.map(_c4_cpu_worker, [(work_meta, a[:2], *(x[:2] for x in j[2:])) for a, j in zip(sl, jobs)])
        t0 = time.perf_counter()
        n = sum(len(r) * V for r in pool.map(_c4_cpu_worker, jobs))
        dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "decisions/s", "cores": cores, "kind": "port",
            "sample": f"{S_cpu} instances x {V} ops of the same sweep: oracle slack_by_kind over the "
                      f"path list + OpTable.select per decision, {cores} worker processes (pool forked "
                      f"and warmed outside the timed map)"}


# ---- c5 -------------------------------------------------------------------------------------

def c5_noise(B: int, batches: range) -> np.ndarray:
    """Observation noise of config 5: batch bt draws exp(N(0, 0.3)) for its B
    invocations from numpy default_rng(bt), one normal per invocation in order, exponentiated
    with math.exp exactly as backend.draw_actual_latency does (backend.py:36-58; np.exp differs
    from math.exp in the last bit for ~5% of arguments)."""
    out = np.empty((len(batches), B))
    for u, bt in enumerate(batches):
        z = np.random.default_rng(bt).normal(0.0, 0.3, size=B)
        out[u] = np.fromiter(map(math.exp, z.tolist()), dtype=np.float64, count=B)
    return out


def c5_truth(table):
    """Ground truth of the synthetic scenario (synth.synth_truths; scenario.py:68-77): the per-batch
    base latency of every configuration (= its zero-noise profile, latency_initial_s) plus a
    per-item coefficient (0 in this scenario) times the invocation's item count (fill)."""
    base = np.array([e.latency_initial_s for e in table.entries])
    per_item = np.zeros(len(base))
    return base, per_item


def run_c5(args):
    import torch

    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    from paper_2102_01887_b200.shard import gather_observations, shard_range

    rank, world, local = _dist(torch)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = sp.get_context(local)
    ctx.set_stream(stream.cuda_stream)
    spec = synth.synth_spec(True)
    table = sp.OpTable(spec, synth.synth_scenario())
    M = len(table.entries)
    B, NB = 65536, args.c5_batches
    N = B * NB
    inv = synth.synth_invocations(N, table.lat, table.gkind, seed=5)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    d = {"slack": T(inv.slack), "avail": T(inv.avail), "supply": T(inv.supply),
         "mb": T(inv.min_batch), "flags": T(inv.flags.astype(np.int32))}
    base_np, per_item_np = c5_truth(table)
    base, per_item = T(base_np), T(per_item_np)
    noise = T(c5_noise(B, range(NB)).reshape(-1))
    # every batch is split contiguously over the ranks (decisions), then the observation records
    # are all-gathered so that each rank folds the whole batch in global order
    a, b = shard_range(B, rank, world)
    Bl = b - a
    out = {k: torch.empty(Bl, dtype=dt, device=dev) for k, dt in
           (("idx", torch.int32), ("code", torch.int32), ("fill", torch.int32),
            ("obj", torch.float64), ("slack", torch.float64), ("wait", torch.float64))}
    obs_idx = torch.empty(Bl, dtype=torch.int32, device=dev)
    obs_val = torch.empty(Bl, dtype=torch.float64, device=dev)
    stream_idx = torch.empty(N, dtype=torch.int32, device=dev)   # the folded stream, kept for the check
    stream_obs = torch.empty(N, dtype=torch.float64, device=dev)
    alpha = 100.0

    # per-batch argument views built once (harness plumbing, outside the timed loop)
    views = []
    for bt in range(NB):
        s = slice(bt * B + a, bt * B + b)
        g = slice(bt * B, (bt + 1) * B)
        views.append((d["slack"][s], d["avail"][s], d["supply"][s], d["mb"][s], d["flags"][s],
                      noise[s], stream_idx[g], stream_obs[g]))

    def online_batch(tab, bt):
        # decide this rank's shard of batch bt against the batch-start table; the assigned
        # configurations run (simulated backend, one kernel): obs = truth(config, items=fill) *
        # exp(N(0, 0.3)); delayed / None decisions produce no observation (idx = -1); every rank
        # folds the whole batch
        sl, av, su, mb, fl, nz, si, so = views[bt]
        tab.select_batch(sl, alpha, av, upstream_supply=su, min_batch=mb, flags=fl, out=out)
        if world > 1:
            sp.simulate_observations(out, base, nz, truth_per_item=per_item, out=(obs_idx, obs_val))
            f_idx, f_obs = gather_observations(obs_idx, obs_val, B)
            si.copy_(f_idx)
            so.copy_(f_obs)
            sp.fold_observations([tab], None, si, so, beta=0.5, dfp_count=10, sync_host=False)
        else:  # one kernel: the observations evaluated in the fold's load phase; the records
            # still land in the run's observation stream
            sp.simulate_and_fold(tab, out, base, nz, truth_per_item=per_item, out=(si, so), beta=0.5,
                                 dfp_count=10)

    # warm-up on a throw-away copy of the table (module loading, scratch allocation, plan-build
    # graph capture); the timed run starts from the untouched table
    wtab = sp.OpTable(spec, synth.synth_scenario())
    for bt in range(max(3, args.warmup)):
        online_batch(wtab, bt)
    table.prepare(alpha)
    torch.cuda.synchronize(dev)
    del wtab
    _barrier(torch)
    l0 = ctx.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with _clocks(local) as clk:
        e0.record(stream)
        h0 = time.perf_counter()
        for bt in range(NB):
            online_batch(table, bt)
        h1 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    launches = ctx.launch_count - l0
    t = _tmax(torch, e0.elapsed_time(e1) / 1e3, dev)
    # replicas must stay bit-identical: compare a checksum of the final latency table
    table.sync_from_device()
    final_lat = np.asarray(table.lat).copy()
    chk = torch.tensor([int(final_lat.view(np.uint64).astype(np.int64).sum())], dtype=torch.int64,
                       device=dev)
    identical = True
    if world > 1:
        lo, hi = chk.clone(), chk.clone()
        torch.distributed.all_reduce(lo, op=torch.distributed.ReduceOp.MIN)
        torch.distributed.all_reduce(hi, op=torch.distributed.ReduceOp.MAX)
        identical = bool(lo.item() == hi.item())
    if rank != 0:
        return
    parity = c5_parity(sp, spec, synth, inv, alpha, B, NB, base_np, per_item_np, noise, online_batch,
                       out, obs_idx, stream_idx.cpu().numpy(), stream_obs.cpu().numpy(), final_lat,
                       dev, torch, check_batches=min(8, NB) if world == 1 else 0)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = _c5_cpu_baseline(spec, synth, inv, alpha, B, parity.pop("_state"))
    else:
        parity.pop("_state", None)
    line = {
        "workload": "c5", "metric": "online config decisions/s incl. per-batch feedback fold and replanning",
        "unit": "decisions/s", "value": N / t, "evals_per_s": N * M / t, "seconds": t, "n_gpus": world,
        "scaling": "strong",
        "config": {"invocations": N, "configs": M, "batches": NB, "batch": B, "beta": 0.5, "dfp_count": 10,
                   "inputs": "synth_invocations(seed 5); obs = truth(config, fill) * math.exp(N(0,0.3)) "
                             "with numpy default_rng(batch id)",
                   "parallelism": (f"each batch split over {world} GPU(s); per batch one all-gather of the "
                                   "16-B observation records, replicated fold" if world > 1 else "1 GPU")},
        "tables_bit_identical_across_ranks": identical,
        "gpu_launches": launches,
        "per_batch_ms": 1e3 * t / NB,
        "roofline": (lambda b: {"bound": "latency (sequential chain: plan -> decisions -> fold per batch)",
                                "achieved": b / (t / NB) / 1e9, "peak": _peaks(), "unit": "GB/s",
                                "frac": b / (t / NB) / 1e9 / _peaks(), "algorithmic_bytes_per_batch": b,
                                "bytes_model": "B x (32 B in + 36 B out) + M x 40 B table + 16 B per "
                                               "observation record"})(B * (32 + 36) + M * 40 + B * 16),
        "host_enqueue_ms_per_batch": 1e3 * (h1 - h0) / NB,
        "parity": parity,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    return line


def c5_parity(sp, spec, synth, inv, alpha, B, NB, base, per_item, noise, online_batch, out, obs_idx,
              stream_idx, stream_obs, final_lat, dev, torch, check_batches=8):
    """Checker.  (1) The first `check_batches` batches replayed on a fresh table: every decision
    against the C oracle scan (oracle_select_batch on the oracle's own folded table), the
    observations recomputed on the host, and the table after each batch against the C sequential
    fold (oracle_fold, manager.py:436-457).  (2) The whole timed run: its recorded observation
    stream (all NB batches) folded sequentially by the C oracle from the initial table must give
    the device's final table bit for bit (final-table checksum)."""
    from oracle import cselect, optable

    # a pristine spec: OpTable shares its ConfigEntry objects with the spec it was built from
    # (as the reference's does, configurator.py:170-177), and sync_from_device() wrote the
    # timed run's final latencies into them
    spec = synth.synth_spec(True)
    ot = optable.from_spec(spec, synth.synth_scenario(), ["cpu", "gpu"])
    lat_init = np.ascontiguousarray(base)  # latency_initial_s of the table's entries
    st = cselect.FoldState(ot.lat.copy(), lat_init, int(ot.ref_index))
    noise_h = noise.view(NB, B)
    res = {"batches_decisions_checked": 0, "decisions": 0, "decision_mismatches": 0,
           "table_mismatches_after_batch": 0}
    if check_batches:
        vtab = sp.OpTable(spec, synth.synth_scenario())
        for bt in range(check_batches):
            s = slice(bt * B, (bt + 1) * B)
            ot.lat[:] = st.lat
            exp = cselect.select_batch([ot], inv.slack[s], alpha, inv.avail[s], inv.supply[s],
                                       inv.min_batch[s], inv.flags[s])
            online_batch(vtab, bt)
            torch.cuda.synchronize(dev)
            got = {k: out[k].cpu().numpy() for k in ("idx", "code", "fill", "obj")}
            some = exp["code"] != 0
            res["decision_mismatches"] += int(
                np.count_nonzero(got["idx"] != exp["idx"]) + np.count_nonzero((got["code"] & 3) != exp["code"])
                + np.count_nonzero(got["fill"] != exp["fill"])
                + np.count_nonzero(got["obj"][some].view(np.uint64) != exp["obj"][some].view(np.uint64)))
            keep = exp["code"] == 1
            oi = exp["idx"][keep]
            ob = (base[oi] + per_item[oi] * exp["fill"][keep].astype(np.float64)) * noise_h[bt].cpu().numpy()[keep]
            # the device's folded stream of the timed run must be this batch's observations
            si = stream_idx[s]
            want = np.where(keep, exp["idx"], -1)
            if not np.array_equal(si, want):
                res["stream_idx_mismatch_batches"] = res.get("stream_idx_mismatch_batches", []) + [bt]
                dpos = np.flatnonzero(si != want)
                res.setdefault("stream_idx_examples", []).append(
                    [int(len(dpos))] + [(int(p), int(si[p]), int(want[p]), int(exp["code"][p])) for p in dpos[:3]])
            elif not np.array_equal(stream_obs[s][keep].view(np.uint64), ob.view(np.uint64)):
                res["stream_obs_mismatch_batches"] = res.get("stream_obs_mismatch_batches", []) + [bt]
                res["stream_obs_example"] = [float(stream_obs[s][keep][0]), float(ob[0])]
            cselect.fold(st, oi, ob, beta=0.5, dfp_count=10)
            vtab.sync_from_device()
            res["table_mismatches_after_batch"] += int(np.count_nonzero(
                np.asarray(vtab.lat).view(np.uint64) != st.lat.view(np.uint64)))
            res["batches_decisions_checked"] += 1
            res["decisions"] += B
    lat0 = optable.from_spec(synth.synth_spec(True), synth.synth_scenario(), ["cpu", "gpu"]).lat
    full = cselect.FoldState(lat0, lat_init, int(ot.ref_index))
    keep = stream_idx >= 0
    cselect.fold(full, stream_idx[keep], stream_obs[keep], beta=0.5, dfp_count=10)
    res["observations_folded"] = int(keep.sum())
    res["final_table_mismatches"] = int(np.count_nonzero(full.lat.view(np.uint64) != final_lat.view(np.uint64)))
    res["final_table_checksum"] = hex(int(final_lat.view(np.uint64).astype(np.uint64).sum(dtype=np.uint64)))
    ok = not (res["decision_mismatches"] or res["table_mismatches_after_batch"] or res["final_table_mismatches"]
              or "stream_idx_mismatch_batches" in res or "stream_obs_mismatch_batches" in res)
    res["result"] = "bit-identical" if ok else "MISMATCH"
    res["_state"] = (ot, st)
    return res


def _c5_cpu_baseline(spec, synth, inv, alpha, B, state):
    """The reference's per-batch CPU semantics: OpTable.select for a
    batch on all host cores (numpy restatement, persistent pool), then the sequential fold
    (oracle/feedback.py apply_feedback + set_latency, one observation at a time)."""
    from oracle import feedback as ofb
    from oracle import optable

    ot, st = state
    cores = os.cpu_count() or 1
    s = slice(0, B)
    ot.lat[:] = st.lat
    with optable.SelectPool([ot], cores) as pool:
        t0 = time.perf_counter()
        r = pool.select(inv.slack[s], alpha, inv.avail[s], inv.supply[s], inv.min_batch[s], inv.flags[s])
        t_sel = time.perf_counter() - t0
    keep = r["code"] == 1
    fs = ofb.FoldState(ot.lat.copy(), st.lat_init.copy(), int(ot.ref_index))
    t0 = time.perf_counter()
    ofb.fold([fs], None, r["idx"][keep], np.ones(int(keep.sum())), beta=0.5, dfp_count=10)
    t_fold = time.perf_counter() - t0
    return {"value": B / (t_sel + t_fold), "unit": "decisions/s", "cores": cores, "kind": "port",
            "sample": f"one batch: {B} OpTable.select (oracle/optable.py numpy restatement, persistent "
                      f"pool of {cores} processes) + the sequential fold of its observations"}


# ---- commit rounds --------------------------------------------------------------------------

def _commit_inputs(meta, R, seed=8):
    rng = np.random.default_rng(seed)
    n_ops, K = len(meta["ops"]), len(meta["kinds"])
    refs = np.array([meta["tables"][o]["ref_index"] for o in meta["ops"]])
    present = rng.random((R, n_ops)) < 0.8
    forced = present & (rng.random((R, n_ops)) < 0.1) & (refs[None, :] >= 0)
    return {
        "slack": rng.uniform(-2.0, 20.0, size=(R, n_ops, K)),
        "fill": rng.integers(1, 5, size=(R, n_ops)).astype(np.int32),
        "buffered": rng.integers(0, 9, size=(R, n_ops)).astype(np.int32),
        "head_id": np.arange(R * n_ops, dtype=np.int64).reshape(R, n_ops)[:, rng.permutation(n_ops)],
        "flags": (present.astype(np.uint32) | (forced.astype(np.uint32) << 1)),
        "full": (rng.random((R, K)) < 0.2).astype(np.uint32) @ (1 << np.arange(K, dtype=np.uint32)),
        # PipelineDag.depths (pipeline.py:328-337): longest edge distance from a source
        "depth": np.array([max(p.index(o) for p in meta["paths"] if o in p) for o in meta["ops"]],
                          dtype=np.int32),
    }


def _commit_cpu_worker(args):
    from oracle import commit as oc

    meta, x, lo, hi, alpha = args
    tabs = oc.amber_tables(meta)
    won = 0
    for r in range(lo, hi):
        heads = [oc.Head(int(x["fill"][r, j]), bool(x["flags"][r, j] & 2), int(x["head_id"][r, j]))
                 if x["flags"][r, j] & 1 else None for j in range(len(tabs))]
        w = oc.round_winner(tabs, x["slack"][r], heads, int(x["full"][r]), x["buffered"][r],
                            x["depth"], alpha)
        won += w is not None
    return hi - lo


def run_commit(args):
    import torch

    import paper_2102_01887_b200 as sp

    with np.load(ROOT / "tests" / "golden" / "amber_trace.npz") as z:
        meta = json.loads(bytes(z["meta_json"]).decode())
    rank, world, local = _dist(torch)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = sp.get_context(local)
    ctx.set_stream(stream.cuda_stream)
    tabs = _amber_tables(sp, meta)
    R = 65536
    x = _commit_inputs(meta, R, seed=8 + rank)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    d = {k: T(v) for k, v in x.items()}
    alpha = 100.0

    def step():
        return sp.commit_round(tabs, d["slack"], d["fill"], d["buffered"], d["head_id"], d["depth"],
                               d["flags"], alpha=alpha, full_mask=d["full"])

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize(dev)
    # parity spot check against the oracle on the first rounds (checker only)
    from oracle import commit as oc

    otabs = oc.amber_tables(meta)
    best = out["best"][:64].cpu().numpy()
    for r in range(64):
        heads = [oc.Head(int(x["fill"][r, j]), bool(x["flags"][r, j] & 2), int(x["head_id"][r, j]))
                 if x["flags"][r, j] & 1 else None for j in range(len(otabs))]
        w = oc.round_winner(otabs, x["slack"][r], heads, int(x["full"][r]), x["buffered"][r],
                            x["depth"], alpha)
        assert (w[0] if w else -1) == best[r], f"commit round {r} disagrees with the oracle"
    _barrier(torch)
    evs = _events(torch, args.steps)
    l0 = ctx.launch_count
    for i in range(args.steps):
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = [a.elapsed_time(b) for a, b in evs]
    t = _tmax(torch, sum(ms) / 1e3, dev)
    if rank != 0:
        return
    cpu = None
    if world == 1:
        import multiprocessing as mp

        cores = os.cpu_count() or 1
        S = 3000 * cores
        # each worker gets only its slice of the rounds (pickling the whole batch would be
        # timed as CPU work); `depth` is per op
        work = []
        for a in np.array_split(np.arange(S), cores):
            if len(a):
                lo, hi = int(a[0]), int(a[-1]) + 1
                xs = {k: (v if k == "depth" else v[lo:hi]) for k, v in x.items()}
                work.append((meta, xs, 0, hi - lo, alpha))
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(len(work)) as pool:
            n = sum(pool.map(_commit_cpu_worker, work))
        dt = time.perf_counter() - t0
        cpu = {"value": n / dt, "unit": "rounds/s", "cores": cores, "kind": "port",
               "sample": f"{S} rounds, oracle/commit.py round_winner (configurator.py:657-728) on "
                         f"{cores} processes"}
    heads = int((x["flags"] & 1).sum())
    line = {
        "workload": "commit", "metric": "Configurator.pump_commits rounds / s (batched commit step)",
        "unit": "rounds/s", "value": args.steps * R * world / t, "ms_per_step": 1e3 * t / args.steps,
        "steps": args.steps, "n_gpus": world, "scaling": "weak",
        "heads_per_s": args.steps * heads * world / t,
        "config": {"rounds_per_call": R, "ops": len(tabs), "kinds": len(meta["kinds"]),
                   "heads_per_call": heads, "alpha": alpha,
                   "inputs": "synthetic heads (80% present, 10% forced), slack U(-2, 20), 20% kinds saturated"},
        "gpu_launches": ctx.launch_count - l0,
        "cpu_baseline": cpu,
        "step_ms": {"median": statistics.median(ms), "min": min(ms), "max": max(ms)},
    }
    return line

# ---- speculate ----------------------------------------------------------

def _spec_inputs(meta, R, seed):
    """R synthetic speculate_from_buffer calls on the AMBER tables: buffers of 1-40 items, upstream
    supply, clock / target spans from overdue to loose, path ratios, entry slack, 0-7 weight keys
    per call (60 % speculative), sdb on 80 %, forced warm-up 10 %, expired holds 10 %."""
    from oracle import commit as oc

    otabs = oc.amber_tables(meta)
    K = len(meta["kinds"])
    rng = np.random.default_rng(seed)
    ops = rng.integers(0, len(otabs), R)
    x = {"op": ops, "n": rng.integers(1, 40, R), "supply": rng.integers(0, 60, R),
         "now": rng.uniform(0, 100, R)}
    x["target"] = x["now"] + rng.uniform(-5, 80, R)
    x["rmin"] = rng.uniform(0.05, 0.5, R)
    x["rmax"] = x["rmin"] + rng.uniform(0, 0.5, R)
    ref_ok = np.array([otabs[o].ref_index >= 0 for o in ops])
    x["flags"] = ((rng.random(R) < 0.8).astype(np.uint32)
                  | np.where((rng.random(R) < 0.1) & ref_ok, 2, 0).astype(np.uint32)
                  | np.where(rng.random(R) < 0.1, 4, 0).astype(np.uint32))
    x["slack0"] = rng.uniform(-2, 60, (R, K))
    calls = []
    ptr, tab, eidx, cnt = [0], [], [], []
    for _ in range(R):
        sq = [[] for _ in range(K)]
        cq = [[] for _ in range(K)]
        for _ in range(rng.integers(0, 8)):
            tb = int(rng.integers(0, len(otabs)))
            e = int(rng.integers(0, len(otabs[tb].lat)))
            k = int(otabs[tb].gkind[e])
            lst = sq if rng.random() < 0.6 else cq
            if not any(y[0] == tb and y[1] == e for y in lst[k]):
                lst[k].append([tb, e, int(rng.integers(1, 5))])
        calls.append((sq, cq))
        for lists in (sq, cq):
            for k in range(K):
                for tb, e, c in lists[k]:
                    tab.append(tb); eidx.append(e); cnt.append(c)
                ptr.append(len(tab))
    x["w_ptr"], x["w_tab"], x["w_eidx"], x["w_count"] = ptr, tab, eidx, cnt
    pk = {k: float(n * r) for k, n, r, _ in meta["backends"]}
    return x, calls, [pk[k] for k in meta["kinds"]]


def _spec_cpu_worker(a):
    meta, x, calls, pool, lo, hi, alpha = a
    from oracle import commit as oc
    from oracle import speculate as osp

    otabs = oc.amber_tables(meta)
    n = 0
    for r in range(lo, hi):
        sq = [[list(y) for y in lst] for lst in calls[r][0]]
        osp.speculate(otabs, int(x["op"][r]), int(x["n"][r]), int(x["supply"][r]), float(x["now"][r]),
                      float(x["target"][r]), float(x["rmin"][r]), float(x["rmax"][r]), pool, alpha,
                      int(x["flags"][r]), sq, calls[r][1], x["slack0"][r])
        n += 1
    return n


def run_speculate(args):
    import torch

    import paper_2102_01887_b200 as sp

    with np.load(ROOT / "tests" / "golden" / "amber_trace.npz") as z:
        meta = json.loads(bytes(z["meta_json"]).decode())
    rank, world, local = _dist(torch)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = sp.get_context(local)
    ctx.set_stream(stream.cuda_stream)
    tabs = _amber_tables(sp, meta)
    R = 262144  # one thread per call: enough calls to fill 148 SMs
    alpha = 100.0
    x, calls, pool = _spec_inputs(meta, R, seed=21 + rank)
    T = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)
    d = {k: T(x[k], np.int32) for k in ("op", "n", "supply", "w_ptr", "w_tab", "w_eidx", "w_count")}
    d.update({k: T(x[k], np.float64) for k in ("now", "target", "rmin", "rmax", "slack0")})
    d["flags"] = T(x["flags"].astype(np.int32), np.int32)

    def step(out=None):
        return sp.speculate_batch(tabs, alpha, pool, d["op"], d["n"], d["supply"], d["now"],
                                  d["target"], d["rmin"], d["rmax"], d["slack0"], d["flags"],
                                  d["w_ptr"], d["w_tab"], d["w_eidx"], d["w_count"], out=out)

    out = step()
    for _ in range(args.warmup):
        step(out)
    torch.cuda.synchronize(dev)
    formed = int(out["n"].sum().item())
    # parity spot check against the oracle on the first calls (checker only)
    from oracle import commit as oc
    from oracle import speculate as osp

    otabs = oc.amber_tables(meta)
    n_dev = out["n"][:64].cpu().numpy()
    for r in range(64):
        sq = [[list(y) for y in lst] for lst in calls[r][0]]
        dec, _ = osp.speculate(otabs, int(x["op"][r]), int(x["n"][r]), int(x["supply"][r]),
                               float(x["now"][r]), float(x["target"][r]), float(x["rmin"][r]),
                               float(x["rmax"][r]), pool, alpha, int(x["flags"][r]), sq, calls[r][1],
                               x["slack0"][r])
        assert len(dec) == n_dev[r], f"speculate call {r} disagrees with the oracle"
    _barrier(torch)
    evs = _events(torch, args.steps)
    l0 = ctx.launch_count
    for i in range(args.steps):
        evs[i][0].record(stream)
        step(out)
        evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    launches = ctx.launch_count - l0
    ms = [a.elapsed_time(b) for a, b in evs]
    t = _tmax(torch, sum(ms) / 1e3, dev)
    # end to end: numpy inputs in host memory through the same public call (copies inside)
    hx = {k: np.ascontiguousarray(x[k]) for k in x}
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        sp.speculate_batch(tabs, alpha, pool, hx["op"], hx["n"], hx["supply"], hx["now"], hx["target"],
                           hx["rmin"], hx["rmax"], hx["slack0"], hx["flags"], hx["w_ptr"], hx["w_tab"],
                           hx["w_eidx"], hx["w_count"])
    e2e_s = (time.perf_counter() - t0) / reps
    if rank != 0:
        return
    cpu = None
    if world == 1:
        import multiprocessing as mp

        cores = os.cpu_count() or 1
        S = 400 * cores
        # each worker gets only its slice (pickling the whole batch would be timed as CPU work)
        keys = ("op", "n", "supply", "now", "target", "rmin", "rmax", "flags", "slack0")
        work = []
        for a in np.array_split(np.arange(S), cores):
            if len(a):
                lo, hi = int(a[0]), int(a[-1]) + 1
                work.append((meta, {k: x[k][lo:hi] for k in keys}, calls[lo:hi], pool, 0, hi - lo,
                             alpha))
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(len(work)) as pool_:
            n = sum(pool_.map(_spec_cpu_worker, work))
        dt = time.perf_counter() - t0
        cpu = {"value": n / dt, "unit": "calls/s", "cores": cores, "kind": "port",
               "sample": f"{S} calls, oracle/speculate.py (configurator.py:563-620) on {cores} processes"}
    line = {
        "workload": "speculate",
        "metric": "Configurator.speculate_from_buffer calls / s (replica-parallel speculation loop)",
        "unit": "calls/s", "value": args.steps * R * world / t, "ms_per_step": 1e3 * t / args.steps,
        "steps": args.steps, "n_gpus": world, "scaling": "weak",
        "invocations_formed_per_s": args.steps * formed * world / t,
        "config": {"calls_per_step": R, "ops": len(tabs), "kinds": len(meta["kinds"]), "alpha": alpha,
                   "invocations_formed_per_step": formed,
                   "inputs": "synthetic AMBER-table calls: buffers 1-40, 0-7 weight keys, sdb 80%, "
                             "forced 10%, expired holds 10%"},
        "e2e": {"value": R / e2e_s, "unit": "calls/s", "path": "speculate_batch(numpy) -> "
                "sp_speculate_batch(SP_MEM_HOST)"},
        "gpu_launches": launches,
        "cpu_baseline": cpu,
        "step_ms": {"median": statistics.median(ms), "min": min(ms), "max": max(ms)},
    }
    return line


# ---- c4runs: config 4 as complete tuned runs (replica-parallel run engine)

DES_DIR = ROOT / "tests" / "golden" / "des"


def _des_amber():
    """The AMBER bundle as the reference's CLI builds a run (profiles from its MetadataStore)."""
    from paper_2102_01887_b200 import metadata
    from paper_2102_01887_b200.engine import RunSpec, TuningParams
    from paper_2102_01887_b200.pipeline import dag_from_json
    from paper_2102_01887_b200.scenario import scenario_from_json

    d = DES_DIR / "branching"
    doc = json.loads((d / "pipeline.json").read_text())
    dag = dag_from_json(doc)
    sc = scenario_from_json(json.loads((d / "scenario.json").read_text()))
    profiles = metadata.load_profiles(d / "metadata", sorted(dag.vertices))
    paths = metadata.load_paths(d / "metadata")
    t = sc.tuning
    params = TuningParams(t.alpha, t.cq_capacity, t.dfp_count, t.straggler_timeout_factor, t.smoothing_beta)
    return doc, dag, sc, profiles, paths, params, RunSpec(dag, profiles, sc, params, paths=paths)


def c4_traces(spec, r0: int, r1: int, frames: int = 3000):
    """Replica r's trace = generate_trace(3000, 17 + r, {"cars": 0.6, "persons": 0.8}, 3)
    (workload.py:45-66), drawn vectorised: one Generator.poisson call
    over the (frame, attribute) grid consumes the stream in the reference's scalar order."""
    rates = {"cars": 0.6, "persons": 0.8}
    names = sorted(rates)
    col = [names.index(a) for a in spec.attr_names]
    T = r1 - r0
    attrs = np.empty((T * frames, len(spec.attr_names)), dtype=np.int32)
    for i, r in enumerate(range(r0, r1)):
        x = np.minimum(np.random.default_rng(17 + r).poisson([rates[n] for n in names], size=(frames, len(names))), 3)
        attrs[i * frames:(i + 1) * frames] = x[:, col]
    return np.arange(0, (T + 1) * frames, frames, dtype=np.int32), attrs


def _c4runs_cpu_worker(a):
    from oracle import engine as oe
    from paper_2102_01887_b200.engine import generate_trace

    r, m = a
    doc, dag, sc, profiles, paths, params, _ = _des_amber()
    frames = generate_trace(3000, 17 + r, {"cars": 0.6, "persons": 0.8}, 3)
    eng = oe.Engine(dag, profiles, frames, sc, m * 90.41885182994682,
                    oe.Params(params.alpha, params.cq_capacity, params.dfp_count,
                              params.straggler_timeout_factor, params.smoothing_beta), seed=sc.seed,
                    paths=paths)
    rep = eng.run()
    return (rep.decision_count, repr(float(rep.cost)), repr(float(rep.latency_s)), rep.invocations,
            rep.completed)


def run_c4runs(args):
    """BASELINE config 4 as complete tuned runs: every (replica, target) pair of the sweep — 10,000
    replicas x 5 targets = 50,000 runs of the reference engine (PipelineRun.run_to_completion on
    the AMBER pipeline, replica r's trace generate_trace(3000, 17 + r, ...)) — executed by the
    replica-parallel run engine (k_des_run, one thread per run).  Parity: the 40 golden runs of
    replicas 0-7 (tests/golden/des/runs.json, produced by the unmodified reference) must match
    bit for bit (decision-log digest, report, final tables)."""
    import multiprocessing as mp

    import torch

    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200.engine import OUT_DTYPE, ReplicaEngine, report_of
    from paper_2102_01887_b200.shard import shard_range

    sys.path.insert(0, str(ROOT / "tests"))
    import des_cases as dc

    rank, world, local = _dist(torch)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = sp.get_context(local)
    ctx.set_stream(stream.cuda_stream)
    doc, dag, sc, profiles, paths, params, spec = _des_amber()
    mults = (0.5, 1.0, 2.0, 5.0, 10.0)
    cp_min = 90.41885182994682
    R = args.c4_replicas
    r0, r1 = shard_range(R, rank, world)
    fo, at = c4_traces(spec, r0, r1)
    n = (r1 - r0) * len(mults)
    trace_of = np.repeat(np.arange(r1 - r0, dtype=np.int32), len(mults))
    targets = np.tile(np.array([m * cp_min for m in mults]), r1 - r0)
    eng = ReplicaEngine(spec, ctx)
    per_replica = eng.prepare(fo, at, n)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    d_fo, d_at, d_tr, d_tg = T(fo), T(at), T(trace_of), T(targets)
    d_out = torch.zeros(n * OUT_DTYPE.itemsize, dtype=torch.uint8, device=dev)

    def step():
        eng.run_device(n, len(fo) - 1, d_fo.data_ptr(), d_at.data_ptr(), d_tr.data_ptr(),
                       d_tg.data_ptr(), d_out.data_ptr())

    steps = max(1, min(args.steps, 2))
    warmup = 3  # full-size steps (~13 s each at 50,000 runs); the timing rules ask for >= 3
    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    _barrier(torch)
    evs = _events(torch, steps)
    l0 = ctx.launch_count
    with _clocks(local) as clk:
        for i in range(steps):
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
    launches = ctx.launch_count - l0
    ms = [a.elapsed_time(b) for a, b in evs]
    t = _tmax(torch, sum(ms) / 1e3, dev)
    out = np.frombuffer(d_out.cpu().numpy().tobytes(), dtype=OUT_DTYPE)
    status_bad = int((out["status"] != 0).sum())
    decisions = int(out["n_speculate"].sum() + out["n_commit"].sum())
    # end to end through the public API: host traces / targets in, reports out (copies and the
    # capacity planning inside the timed region), sp_des_run(SP_MEM_HOST)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    res = eng.run(None, targets, None, trace_of=trace_of, encoded=(fo, at))
    e2e_s = time.perf_counter() - t0
    same = all(repr(r.cost) == repr(float(o["cost"])) and r.decision_count == int(o["n_speculate"] + o["n_commit"])
               for r, o in zip(res, out))
    # parity: the golden runs (replicas 0-7, every target) with decision logs
    gold = [c for c in dc.runs() if c.get("group") == "c4"]
    mism = []
    if r0 == 0:
        gi = [(c["trace"]["seed"] - 17, mults.index(round(float(c["target"]) / cp_min, 6))) for c in gold]
        res_g = eng.run(None, [float(c["target"]) for c in gold], None,
                        trace_of=[i for i, _ in gi], encoded=(fo, at),
                        log_cap=max(c["expect"]["log_rows"] for c in gold) + 16, final_tables=True)
        for c, (i, mi), rr in zip(gold, gi, res_g):
            rep = report_of(rr, target_s=float(c["target"]), scenario_name=sc.name,
                            pipeline_name=doc["name"], seed=sc.seed)
            errs = dc.check(c, eng.log_rows(rr.log), rep, rr.lat)
            o = out[i * len(mults) + mi]
            if repr(float(o["cost"])) != c["expect"]["cost"]:
                errs.append("timed step cost")
            if errs:
                mism.append(errs[:2])
    bad = torch.tensor([status_bad, len(mism), int(not same), decisions, n], dtype=torch.int64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(bad)
    bad = bad.cpu().tolist()
    if rank != 0:
        return
    cpu = None
    oracle_parity = None
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        sample = [(r, m) for r in range(max(1, cores)) for m in (mults[r % 5],)]
        with mp.get_context("fork").Pool(cores) as pool:
            pool.map(_c4runs_cpu_worker, sample[:1])  # warm the pool (imports)
            c0 = time.perf_counter()
            decs = pool.map(_c4runs_cpu_worker, sample)
            cs = time.perf_counter() - c0
        # the CPU sample doubles as a parity check of the timed device step (replicas 0..cores-1)
        omis = 0
        for (r, m), (dn, cost, lat, ninv, ncomp) in zip(sample, decs):
            o = out[r * len(mults) + mults.index(m)]
            omis += (int(o["n_speculate"] + o["n_commit"]) != dn or repr(float(o["cost"])) != cost
                     or repr(float(o["latency"])) != lat or int(o["invocations"]) != ninv
                     or int(o["completed"]) != ncomp)
        oracle_parity = {"runs": len(sample), "mismatches": omis,
                         "fields": "decision count, cost, latency, invocations, completions of the "
                                   "timed step vs oracle/engine.py"}
        decs = [x[0] for x in decs]
        cpu = {"value": len(sample) / cs, "unit": "runs/s", "cores": cores, "kind": "port",
               "decisions_per_s": sum(decs) / cs,
               "sample": f"{len(sample)} complete runs (replicas 0..{len(sample) - 1}, one target each) "
                         "of oracle/engine.py (the CPU restatement of PipelineRun / BackendSim / "
                         "Configurator, pinned to the reference) on a persistent fork pool"}
    total_runs = bad[4]
    line = {
        "workload": "c4runs",
        "metric": "complete tuned pipeline runs/s (reference PipelineRun.run_to_completion semantics)",
        "unit": "runs/s", "value": steps * total_runs / t, "ms_per_step": 1e3 * t / steps,
        "decisions_per_s": steps * bad[3] / t,
        "steps": steps, "warmup": warmup, "n_gpus": world, "scaling": "strong",
        "e2e": {"value": total_runs / e2e_s if world == 1 else None, "unit": "runs/s",
                "h2d_bytes_per_step": int(fo.nbytes + at.nbytes + trace_of.nbytes + targets.nbytes),
                "d2h_bytes_per_step": int(n * OUT_DTYPE.itemsize),
                "path": "ReplicaEngine.run(host traces) -> sp_des_run(SP_MEM_HOST): arena sizing, "
                        "H2D of traces / targets, the launch, D2H of the report rows",
                "same_results_as_device_step": bool(same)},
        "config": {"replicas": R, "targets_x_cp_min": list(mults), "cp_min": cp_min, "runs": total_runs,
                   "frames_per_trace": 3000, "pipeline": "AMBER (branching bundle), alpha 100, beta 0.5, "
                   "dfp 10, cq_capacity 4, noise-free scenario",
                   "arena_bytes_per_run": per_replica,
                   "parallelism": f"{R} replicas x 5 targets sharded contiguously over {world} GPU(s), "
                                  "no data-path collective"},
        "kernel": "k_des_run_warp (a lane group per run — 2 lanes at this run count — every lane "
                  "running the run's event loop: heap, backend pools, speculation, commits, feedback "
                  "in the run's HBM arena; the OpTable scans split across the lanes)",
        "roofline": {"bound": "latency (a sequential event loop per run; throughput from runs in flight)",
                     "achieved": None, "peak": None, "unit": None, "frac": None,
                     "evidence": "profiles/r02/des/ncu_des_warp_summary.json (47% warps active, 23% "
                                 "issue active, stalls: long scoreboard and instruction fetch)"},
        "gpu_launches": launches,
        "step_ms": {"median": statistics.median(ms), "min": min(ms), "max": max(ms)},
        "parity": {"runs": len(gold), "mismatches": bad[1], "bad_status": bad[0],
                   "oracle_sample": oracle_parity if cpu is not None else None,
                   "result": ("bit-identical decision logs / reports / final tables vs the reference's own runs"
                              if bad[1] == 0 and bad[0] == 0 else "MISMATCH"),
                   "checked_on": "replicas 0-7 x 5 targets (tests/golden/des/runs.json)"},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    return line


RUNNERS = {"c1": run_c1, "c3": run_c3, "c4": run_c4, "c5": run_c5, "commit": run_commit,
           "speculate": run_speculate, "c4runs": run_c4runs}


def main(args):
    line = RUNNERS[args.workload](args)
    if line is not None:  # rank 0
        print(json.dumps(line), flush=True)
