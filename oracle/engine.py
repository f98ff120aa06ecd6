"""CPU restatement of one tuned pipeline run — TEST ORACLE ONLY.

Restates, function by function, the reference run engine that SURVEY.md §8(f) rank 4 names:
  * the backend pools (backend.py:125-269: FIFO admission with a blocking head and first-fit
    instances, the (time, code, seq) event heap, `draw_actual_latency` 36-58 with the run's
    numpy Generator, `invocation_cost` 61-63),
  * the configurator's queues and decisions (configurator.py:368-772: Eq. 2 `queueing_by_kind`,
    the per-op `slack_by_kind` cache keyed by the weight version only, `speculate_from_buffer`,
    `speculate_fixed`, `_commit_candidate`, `pump_commits`, `notify_started`, the holds),
  * the run loop (manager.py:210-575: `_pump`, `_spawn_downstream` with branch predicates,
    fan-out and join staging, `_apply_feedback` with the warm-up gate lift, completions,
    failures, straggler duplicates, `run_to_completion` with its one forced flush) and the
    report (manager.py:577-630).
Selection and affinity reuse oracle/optable.py (configurator.py:219-318, same numpy ufuncs).
Pinned against the unmodified reference engine (tests/test_engine_oracle.py: decision log,
report and final tables, bundled scenarios, ablations, faults) and its committed goldens.
The product never imports this module; it is the checker of paper_2102_01887_b200/engine.py and
the `cpu_baseline` of bench.py's replica workload.
"""
from __future__ import annotations

import heapq
import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import optable

_PRED = {"<": lambda a, b: a < b, "<=": lambda a, b: a <= b, ">": lambda a, b: a > b,
         ">=": lambda a, b: a >= b, "==": lambda a, b: a == b, "!=": lambda a, b: a != b}
_COMPLETE, _WAKE = 0, 1  # backend.py:127-128: completions pop before wakes at equal times


@dataclass
class Params:
    alpha: float = 100.0
    cq_capacity: int | None = None
    dfp_count: int = 10
    straggler_timeout_factor: float = 1.5
    smoothing_beta: float = 0.5


@dataclass
class Inv:
    iid: int
    op: str
    items: list            # shared between a unit's clones (manager.py:317-329)
    unit: int
    forced: bool = False
    state: str = "pending"
    spec_e: int = -1
    spec_slack: float = 0.0
    spec_obj: float = 0.0
    com_e: int = -1
    com_slack: float = 0.0
    started_at: float = -1.0
    threshold: float = 0.0
    dup_spawned: bool = False
    # the execution (backend.py:86-99)
    instance: int = -1
    actual: float = 0.0
    will_fail: bool = False


@dataclass
class Report:
    latency_s: float
    normalized_latency: float
    cost: float
    slack_met_frac: float
    configs_used: int
    failures: int
    duplicates: int
    invocations: int
    completed: int
    terminal_items: int
    decision_count: int
    log: list = field(default_factory=list)


def _base_latency(truth, res: int, batch: int, knobs) -> float:
    """OpKindTruth.base_latency (scenario.py:68-77)."""
    lat = truth.base_seconds
    if truth.resource_exponent:
        lat *= (res / truth.ref_resource) ** -truth.resource_exponent
    lat *= batch ** truth.batch_exponent
    for knob, value in sorted(knobs.items()):
        tab = truth.knob_multipliers.get(knob)
        if tab:
            lat *= tab.get(str(value), 1.0)
    return lat


class Engine:
    """One run: `Engine(...).run()` returns a Report (manager.py:539-575, 577-630)."""

    def __init__(self, dag, profiles, frames, scenario, target_s, params: Params, *,
                 ablations=(), seed=0, paths, profile_scale=1.0, noise_sigma=None,
                 failure_rate=None, straggle_rate=None, straggle_factor=None):
        self.dag = dag
        self.target = float(target_s)
        self.p = params
        self.abl = frozenset(ablations)
        self.kinds = list(scenario.backend_kinds())
        K = len(self.kinds)
        self.kpos = {k: i for i, k in enumerate(self.kinds)}
        self.ops = sorted(dag.vertices)  # configurator / table order (manager.py:259-261)
        gt = scenario.ground_truth
        self.sigma = gt.noise_sigma if noise_sigma is None else noise_sigma
        self.fail_rate = gt.failure_rate if failure_rate is None else failure_rate
        self.strag_rate = gt.straggle_rate if straggle_rate is None else straggle_rate
        self.strag_factor = gt.straggle_factor if straggle_factor is None else straggle_factor
        self.dispatch = float(getattr(scenario, "dispatch_overhead_s", 0.0))

        # tables (configurator.py:166-209) over profile-scaled copies (manager.py:187-208)
        self.t, self.ents, self.ref_lat0 = {}, {}, {}
        for op in self.ops:
            spec = profiles[op]
            scaled = _Scaled(spec, profile_scale)
            tab = optable.from_spec(scaled, scenario, self.kinds)
            present = {b.kind for b in scenario.backends}
            ents = [e for e in scaled.entries if e.schedulable and e.backend_kind in present
                    and e.resource_request <= scenario.backend(e.backend_kind).resources_per_instance]
            self.t[op], self.ents[op] = tab, ents
            ref = _reference(scaled)
            self.ref_lat0[op] = ents[tab.ref_index].latency_s if tab.ref_index >= 0 else ref.latency_s
            tab.base_truth = np.array([_base_latency(gt.kind_truth(op, e.backend_kind),
                                                     e.resource_request, e.batch_size,
                                                     dict(e.knob_values)) for e in ents])
            tab.per_item = np.array([gt.kind_truth(op, e.backend_kind).per_item_seconds
                                     for e in ents])
        self.pool_res = [float(b.instance_count * b.resources_per_instance) for b in scenario.backends]
        self.inst_res = [b.resources_per_instance for b in scenario.backends]
        self.price = [b.price_rate for b in scenario.backends]
        self.free = [[b.resources_per_instance] * b.instance_count for b in scenario.backends]
        self.cq = [deque() for _ in range(K)]
        # CQ capacity (configurator.py:443-458)
        if params.cq_capacity is not None:
            self.cap = [params.cq_capacity] * K
        else:
            self.cap = []
            for k in range(K):
                rs = [int(self.t[op].res[self.t[op].gkind == k].min()) for op in self.ops
                      if (self.t[op].gkind == k).any()]
                self.cap.append(max(1, int(self.pool_res[k] // min(rs))) if rs else 1)

        # structure (manager.py:262-271)
        self.succ = {v: dag.successors(v) for v in dag.vertices}
        self.indeg = {v: len(dag.predecessors(v)) for v in dag.vertices}
        self.anc = {v: sorted(_ancestors(dag, v)) for v in dag.vertices}
        self.depth = dag.depths()
        self.deep_first = sorted(dag.vertices, key=lambda v: (-self.depth[v], v))
        self.suffixes = {op: [p[p.index(op):] for p in paths if op in p] for op in self.ops}
        for op, s in self.suffixes.items():
            if not s:
                raise ValueError(f"operation {op!r} does not appear on any path")
        self.frames = [(int(f), dict(a)) for f, a in frames]

        # mutable run state
        self.rng = np.random.default_rng(seed)
        self.now = 0.0
        self.heap, self.seq, self.payload = [], 0, {}
        self.running = 0
        self.buf = {v: deque() for v in dag.vertices}
        self.staging = {v: {} for v in dag.vertices if self.indeg[v] > 1}
        self.unspawned = {v: 0 for v in dag.vertices}
        self.sq = {op: deque() for op in self.ops}
        self.w = [[{} for _ in range(K)], [{} for _ in range(K)]]  # [SQ, CQ][kind]
        self.version = 0
        self.slack_cache = {}
        self.ref_lat = dict(self.ref_lat0)
        self.completed_ref = {op: 0 for op in self.ops}
        self.holds = {}
        self.observed = set()
        self.invs, self.units = {}, {}
        self.next_id = 0
        self.total_cost, self.failures, self.dups = 0.0, 0, 0
        self.completed, self.met, self.terminal, self.last_accept = 0, 0, 0, 0.0
        self.configs_used = set()
        self.n_spec, self.n_commit = 0, 0
        self.log = []

    # ---- backend pools (backend.py:155-233) ------------------------------------------
    def _push(self, t, code, payload):
        self.seq += 1
        self.payload[self.seq] = payload
        heapq.heappush(self.heap, (t, code, self.seq))

    def _wake(self, t, tag):
        self._push(max(t, self.now), _WAKE, tag)

    def _submit(self, inv):
        k = self.kpos[self.ents[inv.op][inv.com_e].backend_kind]
        self.cq[k].append(inv)
        self._try_start(k)

    def _try_start(self, k):
        q = self.cq[k]
        while q:
            inv = q[0]
            need = int(self.t[inv.op].res[inv.com_e])
            inst = next((i for i, f in enumerate(self.free[k]) if f >= need), -1)
            if inst < 0:
                return  # the FIFO head blocks (backend.py:171-173)
            q.popleft()
            self._start(k, inv, inst, need)

    def _start(self, k, inv, inst, need):
        t = self.t[inv.op]
        e = inv.com_e
        self.free[k][inst] -= need
        fill = len(inv.items)
        lat = float(t.base_truth[e]) + float(t.per_item[e]) * fill  # backend.py:51
        if self.sigma > 0.0:
            lat *= math.exp(self.rng.normal(0.0, self.sigma))
        if self.strag_rate > 0.0 and self.rng.random() < self.strag_rate:
            lat *= self.strag_factor
        inv.will_fail = self.fail_rate > 0.0 and self.rng.random() < self.fail_rate
        inv.actual, inv.instance = lat, inst
        self.running += 1
        self._push(self.now + self.dispatch + lat, _COMPLETE, inv)
        # on_start -> PipelineRun._handle_start (manager.py:331-341)
        inv.state = "running"
        inv.started_at = self.now
        self.configs_used.add(self.ents[inv.op][e].config_id)
        self._weights(1, k, inv.op, e, -1)  # notify_started (configurator.py:758-763)
        thr = self.p.straggler_timeout_factor * float(t.lat[e])
        inv.threshold = thr
        at = self.now + thr
        self._wake(at + 1e-9 * (1.0 + abs(at)), ("timeout", inv.iid))

    # ---- configurator state (configurator.py:460-561) ----------------------------------
    def _weights(self, q, k, op, e, d):
        m = self.w[q][k]
        new = m.get((op, e), 0) + d
        if new:
            m[(op, e)] = new
        else:
            m.pop((op, e), None)
        self.version += 1

    def _slacks(self, op):
        hit = self.slack_cache.get(op)
        if hit is not None and hit[0] == self.version:
            return hit[1]
        out = np.empty(len(self.kinds))
        ref = self.ref_lat
        ratios = []
        for suf in self.suffixes[op]:
            tot = 0.0
            for o in suf:
                tot += ref[o]
            ratios.append(ref[op] / tot)
        for k in range(len(self.kinds)):
            tot = 0.0
            for m in self.w[0][k], self.w[1][k]:
                for (o, e), c in m.items():
                    tot += c * (self.t[o].lat[e] * self.t[o].res[e])
            budget = self.target - self.now - tot / self.pool_res[k]
            s = None
            for r in ratios:
                v = r * budget
                if s is None or v < s:
                    s = v
            out[k] = s
        self.slack_cache[op] = (self.version, out)
        return out

    def _supply(self, op):
        return sum(self.unspawned[a] for a in self.anc[op])

    def _new(self, op, items, forced, unit=None, attempt=0):
        self.next_id += 1
        iid = self.next_id
        inv = Inv(iid, op, items, iid if unit is None else unit, forced)
        self.invs[iid] = inv
        if unit is None:
            self.units[iid] = [False, 1]  # resolved, live count (manager.py:84-88)
        else:
            self.units[unit][1] += 1
        return inv

    def _enqueue(self, inv, e, s_k, obj):
        t = self.t[inv.op]
        inv.state, inv.spec_e, inv.spec_slack, inv.spec_obj = "speculated", e, s_k, obj
        self.sq[inv.op].append(inv)
        self._weights(0, int(t.gkind[e]), inv.op, e, +1)
        self.log.append((self.now, "speculate", inv.iid, inv.op, self.kinds[int(t.gkind[e])],
                         self.ents[inv.op][e].config_id, s_k, obj))

    def _speculate_buffer(self, op):  # configurator.py:563-620
        t = self.t[op]
        buf = self.buf[op]
        formed = 0
        while buf:
            forced = ("dfp" not in self.abl and t.ref_index >= 0
                      and self.completed_ref[op] < self.p.dfp_count)
            sl = self._slacks(op)
            if forced:
                e, fill, obj = t.ref_index, 1, float("nan")
                s_k = float(sl[t.gkind[e]])
            else:
                hold = self.holds.get(op)
                allow = "sdb" not in self.abl
                if hold is not None and self.now >= hold[0]:
                    allow = False
                code, e, fill, obj, s_k, wait, _ = optable.select(
                    t, sl, self.p.alpha, len(buf), allow_delay=allow, upstream_supply=self._supply(op))
                if code == optable.DELAY:
                    if hold is None:
                        dl = self.now + wait
                        self.holds[op] = (dl, int(t.batch_int[e]))
                        if dl != float("inf"):
                            self._wake(dl, ("hold", op))
                    self.n_spec += 1
                    break
            self.holds.pop(op, None)
            items = [buf.popleft() for _ in range(fill)]
            self._enqueue(self._new(op, items, forced), e, s_k, obj)
            self.n_spec += 1
            formed += 1
        return formed

    def _speculate_fixed(self, inv):  # configurator.py:622-637
        t = self.t[inv.op]
        code, e, fill, obj, s_k, _, _ = optable.select(
            t, self._slacks(inv.op), self.p.alpha, len(inv.items), allow_delay=False,
            min_batch=len(inv.items))
        if code == optable.NONE:
            raise RuntimeError(f"no configuration can re-run {len(inv.items)} items of {inv.op!r}")
        self._enqueue(inv, e, s_k, obj)
        self.n_spec += 1

    def _pump_commits(self):  # configurator.py:681-756
        committed = 0
        fifo = "pbc" in self.abl
        while True:
            full = 0
            for k in range(len(self.kinds)):
                if len(self.cq[k]) >= self.cap[k]:
                    full |= 1 << k
            best_key, best = None, None
            for op in self.ops:
                if not self.sq[op]:
                    continue
                head = self.sq[op][0]
                t = self.t[op]
                # _commit_candidate (configurator.py:641-679)
                if head.forced:
                    k = int(t.gkind[t.ref_index])
                    if full >> k & 1:
                        continue
                    cand = (t.ref_index, len(head.items), float(self._slacks(op)[k]), float("nan"))
                elif "eslc" in self.abl:
                    if full >> int(t.gkind[head.spec_e]) & 1:
                        continue
                    cand = (head.spec_e, len(head.items), head.spec_slack, head.spec_obj)
                else:
                    code, e, fill, obj, s_k, _, _ = optable.select(
                        t, self._slacks(op), self.p.alpha, len(head.items) + len(self.buf[op]),
                        allow_delay=False, excluded_mask=full, min_batch=len(head.items))
                    if code == optable.NONE:
                        continue
                    cand = (e, max(fill, len(head.items)), s_k, obj)
                if fifo:
                    key = (head.iid,)
                elif head.forced:
                    key = (0, -self.depth[op], head.iid)
                else:
                    aff = optable.affinity(t, int(t.gkind[cand[0]]), self._slacks(op), self.p.alpha)
                    key = (1, -(aff if aff is not None else 0.0), cand[2], head.iid)
                if best_key is None or key < best_key:
                    best_key, best = key, (op, head, cand)
            if best is None:
                return committed
            op, inv, (e, fill_target, s_k, obj) = best
            t = self.t[op]
            self.sq[op].popleft()
            self._weights(0, int(t.gkind[inv.spec_e]), op, inv.spec_e, -1)
            if fill_target > len(inv.items):  # _topup (manager.py:346-352)
                buf = self.buf[op]
                for _ in range(min(fill_target - len(inv.items), len(buf))):
                    inv.items.append(buf.popleft())
                if not buf:
                    self.holds.pop(op, None)
            inv.state, inv.com_e, inv.com_slack = "committed", e, s_k
            self._weights(1, int(t.gkind[e]), op, e, +1)
            self.log.append((self.now, "commit", inv.iid, op, self.kinds[int(t.gkind[e])],
                             self.ents[op][e].config_id, s_k, obj))
            self.n_commit += 1
            committed += 1
            self._submit(inv)

    # ---- run engine (manager.py:356-575) -----------------------------------------------
    def _pump(self):
        while True:
            formed = 0
            for op in self.deep_first:
                if self.buf[op]:
                    formed += self._speculate_buffer(op)
                    if not self.buf[op]:
                        self.holds.pop(op, None)
            committed = self._pump_commits()
            if formed == 0 and committed == 0:
                return

    def _spawn(self, inv):  # manager.py:392-434
        op = inv.op
        if not self.succ[op]:
            self.terminal += len(inv.items)
            self.unspawned[op] -= len(inv.items)
            return
        preds = self.dag.branch_predicates
        for origin, attrs in inv.items:
            for dst in self.succ[op]:
                pr = preds.get((op, dst))
                if pr is not None and not _PRED[pr.op](attrs.get(pr.attr, 0), pr.value):
                    continue
                n = int(attrs.get(self.dag.fanout_rules[dst], 0)) if dst in self.dag.fanout_rules else 1
                if n <= 0:
                    continue
                if self.indeg[dst] > 1:
                    st = self.staging[dst].setdefault(origin, {})
                    st[op] = st.get(op, 0) + n
                    while len(st) == self.indeg[dst] and all(st.values()):
                        for s in st:
                            st[s] -= 1
                        for s in [s for s, c in st.items() if c == 0]:
                            del st[s]
                        self.buf[dst].append((origin, attrs))
                        self.unspawned[dst] += 1
                        if not st:
                            del self.staging[dst][origin]
                            break
                else:
                    self.buf[dst].extend([(origin, attrs)] * n)
                    self.unspawned[dst] += n
        self.unspawned[op] -= len(inv.items)

    def _feedback(self, inv, obs):  # manager.py:436-457
        op, e, t = inv.op, inv.com_e, self.t[inv.op]
        if e == t.ref_index:
            self.completed_ref[op] += 1
        self.observed.add((op, e))
        if "fb" in self.abl:
            return
        t.lat[e] = self.p.smoothing_beta * obs + (1.0 - self.p.smoothing_beta) * float(t.lat[e])
        self.version += 1  # bump_profiles (configurator.py:463-468)
        if e == t.ref_index:
            self.ref_lat[op] = t.lat[e]
            if self.completed_ref[op] == self.p.dfp_count and "dfp" not in self.abl:
                init = self.ents[op][e].latency_initial_s  # recalibrate (470-491)
                if init > 0.0:
                    ratio = float(t.lat[e]) / init
                    for i, ent in enumerate(self.ents[op]):
                        if i != e and (op, i) not in self.observed:
                            t.lat[i] = ent.latency_initial_s * ratio
                    self.version += 1

    def _finish(self, inv, t_ev, failed):  # manager.py:459-511
        k = self.kpos[self.ents[inv.op][inv.com_e].backend_kind]
        self.free[k][inv.instance] += int(self.t[inv.op].res[inv.com_e])
        self.running -= 1
        inv.cost = self.t[inv.op].res[inv.com_e] * inv.actual * self.price[k]
        self.total_cost += inv.cost
        unit = self.units[inv.unit]
        if failed:
            self.failures += 1
            inv.state = "failed"
            unit[1] -= 1
            self._try_start(k)
            if not unit[0] and unit[1] == 0:
                self._speculate_fixed(self._new(inv.op, inv.items, False, unit=inv.unit))
            return
        unit[1] -= 1
        self._try_start(k)
        self._feedback(inv, inv.actual)
        if unit[0]:
            inv.state = "duplicated"
            return
        unit[0] = True
        inv.state = "completed"
        if inv.actual <= inv.com_slack:
            self.met += 1
        self.completed += 1
        self.last_accept = t_ev
        self._spawn(inv)

    def run(self) -> Report:
        for v in self.dag.input_vertices():
            self.buf[v].extend(self.frames)
            self.unspawned[v] += len(self.frames)
        self._pump()
        flushed = False
        while True:
            if not self.heap:
                work = (any(self.buf.values()) or any(self.sq.values())
                        or any(self.cq) or self.running)
                if not work:
                    break
                if not flushed and self.holds:
                    flushed = True
                    for op in self.holds:
                        self.holds[op] = (self.now, self.holds[op][1])
                    self._pump()
                    continue
                raise RuntimeError("run stalled with work remaining")
            flushed = False
            t_ev, code, s = heapq.heappop(self.heap)
            pay = self.payload.pop(s)
            self.now = t_ev
            if code == _WAKE:
                if pay[0] == "timeout":
                    self._straggler(pay[1])
            else:
                self._finish(pay, t_ev, pay.will_fail)
            self._pump()
        lat = float(self.last_accept)
        if self.target > 0:
            norm = lat / self.target
        else:
            norm = 0.0 if lat == 0.0 else float("inf")
        return Report(lat, norm, self.total_cost,
                      self.met / self.completed if self.completed else 1.0,
                      len(self.configs_used), self.failures, self.dups, len(self.invs),
                      self.completed, self.terminal, self.n_spec + self.n_commit, self.log)

    def _straggler(self, iid):  # manager.py:499-511
        inv = self.invs.get(iid)
        if inv is None or inv.state != "running" or inv.dup_spawned:
            return
        if self.units[inv.unit][0]:
            return
        if self.now - inv.started_at > inv.threshold:
            inv.dup_spawned = True
            self.dups += 1
            self._speculate_fixed(self._new(inv.op, inv.items, False, unit=inv.unit))


class _Scaled:
    """Profile-scaled copy of a ConfigSpec (manager.py:187-208)."""

    def __init__(self, spec, scale):
        self.operation = spec.operation
        self.reference_id = getattr(spec, "reference_id", None)
        self.entries = [_Entry(e, scale) for e in spec.entries]


class _Entry:
    def __init__(self, e, scale):
        for a in ("config_id", "backend_kind", "batch_size", "resource_request", "schedulable"):
            setattr(self, a, getattr(e, a))
        self.knob_values = dict(e.knob_values)
        self.latency_s = e.latency_s * scale
        self.latency_initial_s = e.latency_initial_s * scale


def _reference(spec):
    """pipeline.py:478-500."""
    cands = [e for e in spec.entries if e.backend_kind == "cpu" and e.batch_size == 1]
    if not cands:
        raise ValueError(f"operation {spec.operation!r} has no cpu batch-1 entry to use as reference")
    return min(cands, key=lambda e: (e.resource_request,
                                     tuple(sorted((k, str(v)) for k, v in e.knob_values.items())),
                                     e.config_id))


def _ancestors(dag, v):
    seen, stack = set(), list(dag.predecessors(v))
    while stack:
        u = stack.pop()
        if u not in seen:
            seen.add(u)
            stack.extend(dag.predecessors(u))
    return seen
