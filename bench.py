"""Benchmark of the configurator hot path (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1]): one profile table of 4,096
configurations (sampling x variant x batch x cores / GPU memory x {cpu, gpu}) and 2^20
synthetic invocations per GPU.  A step is one batched OpTable.select pass over all 2^20
invocations (K2, staircase kernel) with alpha rotating over {0, 1, 100, 1000} by step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0:
  value     invocation x configuration evaluations / s, inputs resident in HBM and larger than
            L2: K steps back to back over 4 rotating invocation sets (4 x 71.5 MB > 126 MB L2),
            one CUDA-event pair on the launching stream around the K steps, max over ranks;
            decisions_per_s alongside.  The per-step time with an L2 flush (256 MB read sweep)
            and an event pair around every step is reported beside it (step_ms_l2_flushed).
  e2e       the same metric through the reference-facing call with HOST (pinned) buffers:
            H2D of the step's inputs, kernel, D2H of every decision, inside the timed region.
  roofline  K2 kernel: algorithmic bytes per launch / mean launch time
            vs the measured HBM copy bandwidth in MEASURED_PEAKS.json.
  cpu_baseline  the oracle restatement of OpTable.select (numpy, same ops as the reference)
            on all host cores, bounded sample (rank 0, N=1 only).
--impl reference times only that CPU implementation (rank 0; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "config decisions/sec (invocation x config evals/s) at 1/2/4/8 B200; % HBM roofline"
UNIT = "evals/s"
ALPHAS = (0.0, 1.0, 100.0, 1000.0)
SETS = 4                     # rotating invocation sets per GPU (together larger than L2)
K_KINDS = 2
B_IN = 8 * K_KINDS + 16      # slack[K] f64 + avail, supply, min_batch i32 + flags u32
B_OUT = 4 + 4 + 4 + 8 + 8 + 8  # idx, code, fill i32 + objective, slack, wait f64
B_CFG = 40                   # per configuration: lat, cost, costpen, res f64 + batch, kind|id


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(n_inv: int, M: int, mode: str, world: int) -> dict:
    return {
        "workload": "config2: 2^20 invocations x 4,096 configs per GPU "
                    "(sampling x variant x batch x cores/GPU-mem x {cpu,gpu}); SURVEY.md §8(d)",
        "invocations_per_gpu": n_inv, "configs": M, "kinds": K_KINDS, "alphas": list(ALPHAS),
        "kernel": {"plan": "k_select_fast (K2f: specialised K2b staircase, PDL launch)",
                   "scan": "k_select_scan (K2a)",
                   "auto": "k_select_fast (K2f: specialised K2b staircase, PDL launch)"}.get(mode, "CPU: oracle restatement of OpTable.select"),
        "l2": ("inputs larger than L2: steps rotate over 4 invocation sets (4 x 71.5 MB = 286 MB "
               "> 126 MB L2), K steps back to back in one event pair; step_ms_l2_flushed = the same "
               "step with a 256 MB read sweep before it and an event pair around it"),
        "sets": SETS,
        "parallelism": f"replicated tables, invocations sharded, {world} GPU(s), no data-path collective",
    }


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every 2 ms through NVML (the same
    counters nvidia-smi reports) while the timed region runs."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.rows: list[tuple[float, float, int]] = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def _run(self):
        nv = self._nvml
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), int(rs)))
            except Exception:
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            time.sleep(0.01)
        except Exception:
            self._nvml = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for n, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 2 ms period"}


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "MEASURED_PEAKS.json (burst copy)"}
    return {"hbm_gbs": 6650.0, "source": "fallback 6.65 TB/s (B200_PROFILING.md)"}


def ncu_traffic() -> tuple[float | None, str | None]:
    p = ROOT / "profiles" / "ncu_k2f_summary.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("dram_bytes_per_launch"), d.get("source")
    return None, None


# ---- CPU baseline (oracle restatement, all host cores) ----------------------------------------

def cpu_baseline(target_s: float = 12.0) -> dict:
    from oracle import optable
    from paper_2102_01887_b200 import synth

    spec = synth.synth_spec(False)
    t = optable.from_spec(spec, synth.synth_scenario(), ["cpu", "gpu"])
    M = len(t.lat)
    cores = os.cpu_count() or 1
    inv = synth.synth_invocations(1 << 20, t.lat, t.gkind)
    # calibrate on one core, then size the all-core sample for ~target_s
    t0 = time.perf_counter()
    optable.select_many([t], inv.slack, 100.0, inv.avail, inv.supply, inv.min_batch, inv.flags, None, 0, 200)
    rate1 = 200 / (time.perf_counter() - t0)
    S = int(min(len(inv.avail), max(cores * 200, rate1 * cores * target_s)))
    sub = inv.take(slice(0, S))
    with optable.SelectPool([t], cores) as pool:  # forked and warmed outside the timed call
        t0 = time.perf_counter()
        pool.select(sub.slack, 100.0, sub.avail, sub.supply, sub.min_batch, sub.flags)
        best = time.perf_counter() - t0
    return {
        "value": S * M / best, "unit": UNIT, "cores": cores, "kind": "port",
        "decisions_per_s": S / best, "single_core_decisions_per_s": rate1,
        "sample": f"{S} config-2 invocations x {M} configs (alpha=100), oracle/optable.py numpy "
                  f"restatement of OpTable.select, persistent fork pool over {cores} host cores",
    }


def reference_arm(args) -> None:
    rank, world, local = dist_env()
    if rank != 0:
        return
    from oracle import optable
    from paper_2102_01887_b200 import synth

    spec = synth.synth_spec(False)
    t = optable.from_spec(spec, synth.synth_scenario(), ["cpu", "gpu"])
    M = len(t.lat)
    cores = os.cpu_count() or 1
    inv = synth.synth_invocations(1 << 16, t.lat, t.gkind)
    t0 = time.perf_counter()
    optable.select_many([t], inv.slack, 100.0, inv.avail, inv.supply, inv.min_batch, inv.flags, None, 0, 200)
    rate1 = 200 / (time.perf_counter() - t0)
    S = int(min(len(inv.avail), max(cores * 100, rate1 * cores * args.ref_step_s)))
    times = []
    with optable.SelectPool([t], cores) as pool:  # forked and warmed before the timed steps
        for step in range(args.warmup + args.steps):
            a = ALPHAS[step % len(ALPHAS)]
            off = (step * S) % max(1, len(inv.avail) - S)
            sub = inv.take(slice(off, off + S))
            t0 = time.perf_counter()
            pool.select(sub.slack, a, sub.avail, sub.supply, sub.min_batch, sub.flags)
            dt = time.perf_counter() - t0
            if step >= args.warmup:
                times.append(dt)
    tot = sum(times)
    value = args.steps * S * M / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY.md §8(d) config 2, seed 20261017)",
        "config": workload_config(1 << 20, M, "cpu", world),
        "decisions_per_s": args.steps * S / tot,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{S} invocations per step x {M} configs, oracle/optable.py numpy "
                                   f"restatement of OpTable.select (configurator.py:239-300) over "
                                   f"a persistent pool of {cores} processes; the reference package is pure Python and "
                                   f"is not present on the GPU box"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm ------------------------------------------------------------------------------------

def our_arm(args) -> None:
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import synth

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = sp.get_context(local)
    ctx.set_stream(stream.cuda_stream)

    spec = synth.synth_spec(False)
    table = sp.OpTable(spec, synth.synth_scenario(), device=local)
    M = len(table.entries)
    N = args.n
    gk = table.gkind
    inv = synth.synth_invocations(N, table.lat, gk, seed=20261017 + rank)

    def dev_set(v):
        d = {"slack": torch.from_numpy(v.slack).to(dev), "avail": torch.from_numpy(v.avail).to(dev),
             "supply": torch.from_numpy(v.supply).to(dev), "min_batch": torch.from_numpy(v.min_batch).to(dev),
             "flags": torch.from_numpy(v.flags.astype(np.int32)).to(dev)}
        o = {"idx": torch.empty(N, dtype=torch.int32, device=dev),
             "code": torch.empty(N, dtype=torch.int32, device=dev),
             "fill": torch.empty(N, dtype=torch.int32, device=dev),
             "obj": torch.empty(N, dtype=torch.float64, device=dev),
             "slack": torch.empty(N, dtype=torch.float64, device=dev),
             "wait": torch.empty(N, dtype=torch.float64, device=dev)}
        return d, o

    sets = [dev_set(inv)] + [
        dev_set(synth.synth_invocations(N, table.lat, gk, seed=20261017 + 1000 * s + rank))
        for s in range(1, SETS)]

    # plan build for every alpha (table is static: plans are reused across steps) — timed once
    plan_ms = {}
    for a in ALPHAS:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        table.prepare(a)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        plan_ms[str(a)] = e0.elapsed_time(e1)
    plan_bytes = table.plan_bytes(100.0)

    flush = torch.ones(256 << 20, dtype=torch.uint8, device=dev)

    def flush_l2():
        # read-only sweep larger than the 126 MB L2: the previous step's dirty lines are
        # written back here, outside the timed region, and L2 is left holding clean data
        flush.max()

    def alpha_of(i):
        return ALPHAS[(i + i // SETS) % len(ALPHAS)]

    def step(i, host=None):
        a = alpha_of(i)
        if host is None:
            d, o = sets[i % SETS]
            table.select_batch(d["slack"], a, d["avail"], upstream_supply=d["supply"],
                               min_batch=d["min_batch"], flags=d["flags"], mode=args.mode, out=o)
        else:
            table.select_batch(host["slack"], a, host["avail"], upstream_supply=host["supply"],
                               min_batch=host["min_batch"], flags=host["flags"], mode=args.mode,
                               out=host["out"])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)

    # ---- timed: device-resident, K steps back to back over rotating sets ----
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count
    with ClockSampler(local) as clk:
        # hold the GPU while the host enqueues every timed step, so that host-side launch
        # jitter can never land inside the timed region
        torch.cuda._sleep(int(2e6 + 4e5 * args.steps))
        e0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    launches = ctx.launch_count - launches0
    if world > 1:
        torch.distributed.barrier()
    t_local = e0.elapsed_time(e1) / 1e3
    t_max = t_local
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_max = float(tt.item())
    evals = args.steps * N * M * world
    value = evals / t_max

    # ---- plan-inclusive: every step first rebuilds its alpha's plan (SURVEY.md §8(d) config 2,
    # "alpha in {0, 1, 100, 1000}, one launch each" with nothing precomputed) ----
    for i in range(2):
        table.invalidate_plans()
        step(i)
    torch.cuda.synchronize(dev)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lp0 = ctx.launch_count
    torch.cuda._sleep(int(2e6 + 4e5 * args.steps))
    p0.record(stream)
    for i in range(args.steps):
        table.invalidate_plans()
        step(args.warmup + i)
    p1.record(stream)
    torch.cuda.synchronize(dev)
    launches_pi1 = ctx.launch_count - lp0
    t_pi1 = p0.elapsed_time(p1) / 1e3
    # the same, but after each table change the four alphas' plans are rebuilt together: one
    # launch, one thread-block cluster per plan (sp_table_prepare_many), then the four decision
    # launches of the sweep
    def group(i):
        if i % len(ALPHAS) == 0:
            table.invalidate_plans()
            table.prepare_many([alpha_of(args.warmup + j) for j in range(i, min(i + len(ALPHAS), args.steps))])
        step(args.warmup + i)

    for i in range(len(ALPHAS)):
        group(i)
    torch.cuda.synchronize(dev)
    lp0 = ctx.launch_count
    torch.cuda._sleep(int(2e6 + 4e5 * args.steps))
    p0.record(stream)
    for i in range(args.steps):
        group(i)
    p1.record(stream)
    torch.cuda.synchronize(dev)
    launches_pi = ctx.launch_count - lp0
    t_pi = p0.elapsed_time(p1) / 1e3
    if world > 1:
        tt = torch.tensor([t_pi, t_pi1], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_pi, t_pi1 = (float(x) for x in tt.tolist())

    # ---- the same steps, one at a time: L2 flushed before, an event pair around each ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    torch.cuda._sleep(int(2e6 + 4e5 * args.steps))
    for i in range(args.steps):
        flush_l2()
        evs[i][0].record(stream)
        step(args.warmup + i)
        evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    step_ms = [a.elapsed_time(b) for a, b in evs]

    # ---- e2e: host pinned buffers through the reference-facing call ----
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    host = {"slack": pin(inv.slack), "avail": pin(inv.avail), "supply": pin(inv.supply),
            "min_batch": pin(inv.min_batch), "flags": pin(inv.flags)}
    host["out"] = {"idx": pin(np.empty(N, np.int32)), "code": pin(np.empty(N, np.int32)),
                   "fill": pin(np.empty(N, np.int32)), "obj": pin(np.empty(N)), "slack": pin(np.empty(N)),
                   "wait": pin(np.empty(N))}
    h2d = sum(host[k].nbytes for k in ("slack", "avail", "supply", "min_batch", "flags"))
    d2h = sum(v.nbytes for v in host["out"].values())
    for i in range(2):
        step(i, host)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush_l2()
        e2e_ev[i][0].record(stream)
        step(i, host)
        e2e_ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    t_e2e = sum(a.elapsed_time(b) for a, b in e2e_ev) / 1e3
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e_value = evals / t_e2e

    # ---- roofline of the K2 kernel ----
    peaks = load_peaks()
    kernel_s = t_local / args.steps
    alg_bytes = N * (B_IN + B_OUT) + M * B_CFG
    achieved = alg_bytes / kernel_s / 1e9
    traffic, traffic_src = ncu_traffic()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY.md §8(d) config 2, invocation seed 20261017 + rank)",
        "config": workload_config(N, M, args.mode, world),
        "decisions_per_s": args.steps * N * world / t_max,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "decisions_per_s": args.steps * N * world / t_e2e,
                "path": "OpTable.select_batch(numpy pinned) -> sp_select_batch(SP_MEM_HOST): pinned buffers are read and written over PCIe by the decision kernel itself (zero-copy, one launch)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_model": f"N*(B_in {B_IN} + B_out {B_OUT}) + M*{B_CFG}",
                     "kernel_ms": kernel_s * 1e3, "peak_source": peaks["source"],
                     "traffic_source": traffic_src},
        "gpu_launches": launches,
        "step_ms_l2_flushed": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms),
                               "by_alpha": {str(a): statistics.median([t for k, t in enumerate(step_ms)
                                                                       if alpha_of(args.warmup + k) == a])
                                            for a in ALPHAS
                                            if any(alpha_of(args.warmup + k) == a for k in range(args.steps))},
                               "evals_per_s": N * M * world / (statistics.median(step_ms) / 1e3)},
        "plan": {"build_ms_per_alpha": plan_ms, "bytes": plan_bytes,
                 "note": "value / roofline: staircase plan built once per (profile version, alpha), "
                         "table static in config 2; value_incl_plan: the table is invalidated before "
                         "every sweep of the four alphas and each step decides with a freshly built "
                         "plan (the sweep's four plans built by one launch); value_incl_plan_per_step: "
                         "every single step invalidates the table and builds its own plan alone"},
        "value_incl_plan": evals / t_pi,
        "value_incl_plan_per_step": {"value": evals / t_pi1, "ms_per_step": 1e3 * t_pi1 / args.steps,
                                     "gpu_launches": launches_pi1,
                                     "roofline_frac": alg_bytes / (t_pi1 / args.steps) / 1e9 / peaks["hbm_gbs"]},
        "roofline_incl_plan": {"bound": "hbm", "achieved": alg_bytes / (t_pi / args.steps) / 1e9,
                               "peak": peaks["hbm_gbs"], "unit": "GB/s",
                               "frac": alg_bytes / (t_pi / args.steps) / 1e9 / peaks["hbm_gbs"],
                               "ms_per_step": 1e3 * t_pi / args.steps,
                               "gpu_launches": launches_pi,
                               "kernels": "per sweep of 4 steps: k_plan_cluster_multi (four 16-CTA "
                                          "clusters, one plan each) + k_pc_commit_order, then the 4 "
                                          "decision launches"},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
    return line if rank == 0 else None


def run_extras(args, line) -> None:
    """The other BASELINE configs on the same GPUs, attached to the headline line under
    "configs" (each entry is that workload's own line, bench_workloads.py): config 1 (AMBER
    drop-in, per call), 3 (deep DAG), 4 (target sweep, strong scaling) and 5 (online mode,
    strong scaling).  Skipped with --no-extras."""
    import copy

    import torch

    import bench_workloads

    out = {}
    for w in ("c1", "c3", "c4", "c5", "c4runs"):
        a = copy.copy(args)
        a.workload = w
        a.steps = min(args.steps, 10)
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        r = bench_workloads.RUNNERS[w](a)
        if r is not None:
            r["wall_s"] = time.perf_counter() - t0
            out[w] = r
    if line is not None:
        line["configs"] = out


def _free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and return their exit status.  Refuses (exit 2) when
    fewer than N GPUs are visible.  NCCL communicator set-up is logged (NCCL_DEBUG=INFO,
    subsystem INIT) on stderr so the rank count of every communicator can be checked."""
    if not args.dist_selftest:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} requested but only {have} GPU(s) visible",
                  file=sys.stderr, flush=True)
            return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def dist_selftest(args) -> None:
    """CPU (gloo) exercise of the multi-rank plumbing the GPU arms use: rendezvous, the
    contiguous shard of every rank, exact counter all-reduce, max-over-ranks timing and the
    ordered all-gather of observation records (paper_2102_01887_b200/shard.py); rank 0 prints
    one JSON line."""
    import torch
    import torch.distributed as dist

    from paper_2102_01887_b200.shard import gather_observations, reduce_counters, shard_range

    rank, world, _ = dist_env()
    dist.init_process_group("gloo")
    N = 1000
    a, b = shard_range(N, rank, world)
    ids = torch.arange(a, b, dtype=torch.int64)
    counters = reduce_counters(torch.tensor([b - a, int(ids.sum())], dtype=torch.int64))
    t = torch.tensor([0.001 * (rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    idx = torch.arange(a, b, dtype=torch.int32)
    g_idx, g_obs = gather_observations(idx, idx.to(torch.float64) * 0.5, N)
    ok = (counters.tolist() == [N, N * (N - 1) // 2] and g_idx.tolist() == list(range(N))
          and bool((g_obs == torch.arange(N, dtype=torch.float64) * 0.5).all()))
    if rank == 0:
        print(json.dumps({"dist_selftest": True, "world": world, "ranks_ok": ok,
                          "t_max": float(t.item()), "backend": "gloo"}), flush=True)
    dist.destroy_process_group()
    if not ok:
        sys.exit(1)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--mode", default="plan", choices=["plan", "scan", "auto"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-s", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="c2",
                    choices=["c1", "c2", "c3", "c4", "c5", "commit", "speculate", "c4runs"],
                    help="c2 (default): BASELINE configs[1]; c3/c4/c5: bench_workloads.py")
    ap.add_argument("--c3-cpu-instances", type=int, default=1000)
    ap.add_argument("--c4-replicas", type=int, default=10000)
    ap.add_argument("--c5-batches", type=int, default=256)
    ap.add_argument("--no-extras", action="store_true",
                    help="headline line only (skip configs 1, 3, 4, 5 attached under 'configs')")
    ap.add_argument("--dist-selftest", action="store_true",
                    help="CPU/gloo check of the multi-rank plumbing (tests); no GPU work")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dist_selftest:
        dist_selftest(args)
        return
    if args.workload != "c2":
        import bench_workloads

        bench_workloads.main(args)
        return
    if args.impl == "reference":
        reference_arm(args)
        return
    line = our_arm(args)
    if not args.no_extras:
        run_extras(args, line)
    if line is not None:
        print(json.dumps(line), flush=True)
    import torch

    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
