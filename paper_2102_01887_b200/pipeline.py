"""Data types the hot path consumes, mirroring the reference's pipeline module.

Only what the configurator path needs is restated here:
profiled ``ConfigEntry`` / ``ConfigSpec`` rows (pipeline.py:191-279), ``reference_config``
(pipeline.py:478-500) and the DAG structure that feeds the slack kernel
(``PipelineDag`` pipeline.py:298-337).  The reference's own objects are accepted wherever
these are (duck typing), so the GPU path is a drop-in for the reference package.
"""
from __future__ import annotations

import hashlib
import itertools
import json
from dataclasses import dataclass, field
from typing import Any, Mapping, Sequence

CPU_KIND = "cpu"  # pipeline.py:19 — reference configurations live on this kind


@dataclass
class ConfigEntry:
    """A profiled configuration (pipeline.py:191-215)."""

    config_id: str
    backend_kind: str
    knob_values: dict[str, Any]
    batch_size: int
    resource_request: int
    latency_s: float
    latency_initial_s: float
    peak_memory_mb: float = 0.0
    schedulable: bool = True

    def __post_init__(self) -> None:
        if self.batch_size < 1:
            raise ValueError(f"{self.config_id}: batch size must be >= 1")
        if self.resource_request <= 0:
            raise ValueError(f"{self.config_id}: resource request must be positive")
        if self.latency_s <= 0 or self.latency_initial_s <= 0:
            raise ValueError(f"{self.config_id}: latency must be positive")


    def to_json(self) -> dict[str, Any]:
        """pipeline.py:217-228 (same keys, knob values sorted by name)."""
        return {
            "config_id": self.config_id,
            "backend_kind": self.backend_kind,
            "knob_values": dict(sorted(self.knob_values.items())),
            "batch_size": self.batch_size,
            "resource_request": self.resource_request,
            "latency_s": self.latency_s,
            "latency_initial_s": self.latency_initial_s,
            "peak_memory_mb": self.peak_memory_mb,
            "schedulable": self.schedulable,
        }

    @staticmethod
    def from_json(obj: Mapping[str, Any]) -> "ConfigEntry":
        """pipeline.py:230-242."""
        return ConfigEntry(
            config_id=obj["config_id"],
            backend_kind=obj["backend_kind"],
            knob_values=dict(obj["knob_values"]),
            batch_size=int(obj["batch_size"]),
            resource_request=int(obj["resource_request"]),
            latency_s=float(obj["latency_s"]),
            latency_initial_s=float(obj["latency_initial_s"]),
            peak_memory_mb=float(obj.get("peak_memory_mb", 0.0)),
            schedulable=bool(obj.get("schedulable", True)),
        )


@dataclass
class ConfigSpec:
    """All profiled configurations of one operation (pipeline.py:245-258)."""

    operation: str
    entries: list[ConfigEntry]
    reference_id: str

    def __post_init__(self) -> None:
        ids = [e.config_id for e in self.entries]
        if len(set(ids)) != len(ids):
            raise ValueError(f"{self.operation}: duplicate config ids")
        if self.reference_id not in set(ids):
            raise ValueError(f"{self.operation}: reference {self.reference_id!r} not among entries")

    def to_json(self) -> dict[str, Any]:
        """pipeline.py:266-271."""
        return {"operation": self.operation, "reference_id": self.reference_id,
                "entries": [e.to_json() for e in self.entries]}

    @staticmethod
    def from_json(obj: Mapping[str, Any]) -> "ConfigSpec":
        """pipeline.py:273-279."""
        return ConfigSpec(operation=obj["operation"],
                          entries=[ConfigEntry.from_json(e) for e in obj["entries"]],
                          reference_id=obj["reference_id"])


def canonical_json(obj: Any) -> str:
    """pipeline.py:31-33 (sorted keys, fixed separators)."""
    return json.dumps(obj, sort_keys=True, separators=(",", ":"))


def content_hash(obj: Any) -> str:
    """pipeline.py:36-37."""
    return hashlib.sha256(canonical_json(obj).encode("utf-8")).hexdigest()


@dataclass(frozen=True)
class Knob:
    """One tunable dimension (pipeline.py:66-74)."""

    name: str
    values: tuple[Any, ...]


@dataclass(frozen=True)
class KnobTemplate:
    """An operation's search space (pipeline.py:93-121)."""

    knobs: tuple[Knob, ...]
    hardware_targets: tuple[str, ...]
    batch_sizes: tuple[int, ...]
    resource_options: Mapping[str, tuple[int, ...]]


@dataclass(frozen=True)
class OperationSpec:
    """A named pipeline stage and its search space (pipeline.py:167-173)."""

    name: str
    executable_id: str
    knob_template: KnobTemplate
    branching: bool = False


@dataclass(frozen=True)
class ConfigAssignment:
    """One point of the search space before profiling (pipeline.py:176-188)."""

    backend_kind: str
    resource_request: int
    batch_size: int
    knob_values: tuple[tuple[str, Any], ...]

    def config_id(self) -> str:
        return config_id_of(self.backend_kind, self.resource_request, self.batch_size, self.knob_values)


def enumerate_configs(template) -> list[ConfigAssignment]:
    """pipeline.py:454-475: kinds sorted, then resource options and batch sizes ascending, then
    the knob values in template order (the host half: the assignments' ids; the device
    enumerates the same order in sp_profile_configs)."""
    out = []
    names = [k.name for k in template.knobs]
    value_lists = [k.values for k in template.knobs]
    for kind in sorted(template.hardware_targets):
        for resource in template.resource_options[kind]:
            for batch in sorted(template.batch_sizes):
                for combo in itertools.product(*value_lists):
                    out.append(ConfigAssignment(kind, resource, batch, tuple(zip(names, combo))))
    return out


def config_id_of(kind: str, resource: int, batch: int, knobs: Sequence[tuple[str, Any]] = ()) -> str:
    """Config id format of ConfigAssignment.config_id (pipeline.py:185-188)."""
    parts = [f"{kind}-r{resource}-b{batch}"]
    parts.extend(f"{k}={v}" for k, v in knobs)
    return "-".join(parts)


def reference_config(spec) -> Any:
    """Smallest CPU batch-1 entry; ties by sorted knob strings, then id (pipeline.py:478-500)."""
    cands = [e for e in spec.entries if e.backend_kind == CPU_KIND and e.batch_size == 1]
    if not cands:
        raise ValueError(
            f"operation {spec.operation!r} has no {CPU_KIND} batch-1 entry to use as reference"
        )
    return min(
        cands,
        key=lambda e: (
            e.resource_request,
            tuple(sorted((k, str(v)) for k, v in e.knob_values.items())),
            e.config_id,
        ),
    )


_PREDICATE_OPS = ("<", "<=", ">", ">=", "==", "!=")


@dataclass(frozen=True)
class BranchPredicate:
    """Comparison over one integer input attribute, e.g. persons > 0 (pipeline.py:283-295)."""

    attr: str
    op: str
    value: int

    def __post_init__(self) -> None:
        if self.op not in _PREDICATE_OPS:
            raise ValueError(f"unknown predicate operator {self.op!r}")


@dataclass
class PipelineDag:
    """Operations wired into a DAG (pipeline.py:298-337).  Branch predicates and fan-out rules
    do not influence Alg. 1 (every decomposed path counts); the run engine (engine.py) routes
    items by them."""

    vertices: tuple[str, ...]
    edges: tuple[tuple[str, str], ...]
    branching: frozenset = frozenset()
    branch_predicates: dict = field(default_factory=dict)
    fanout_rules: dict = field(default_factory=dict)

    def successors(self, v: str) -> list[str]:
        return sorted(d for s, d in self.edges if s == v)

    def predecessors(self, v: str) -> list[str]:
        return sorted(s for s, d in self.edges if d == v)

    def input_vertices(self) -> list[str]:
        has_pred = {d for _, d in self.edges}
        return sorted(v for v in self.vertices if v not in has_pred)

    def output_vertices(self) -> list[str]:
        has_succ = {s for s, _ in self.edges}
        return sorted(v for v in self.vertices if v not in has_succ)

    def topological_order(self) -> list[str]:
        """Kahn's algorithm with a sorted ready list (pipeline.py:367-387)."""
        indeg = {v: 0 for v in self.vertices}
        succ: dict[str, list[str]] = {v: [] for v in self.vertices}
        for s, d in self.edges:
            indeg[d] += 1
            succ[s].append(d)
        ready = sorted(v for v, n in indeg.items() if n == 0)
        order: list[str] = []
        import bisect

        while ready:
            v = ready.pop(0)
            order.append(v)
            for d in sorted(succ[v]):
                indeg[d] -= 1
                if indeg[d] == 0:
                    bisect.insort(ready, d)
        if len(order) != len(self.vertices):
            raise ValueError("pipeline contains a cycle")
        return order

    def depths(self) -> dict[str, int]:
        """Longest edge distance from an input vertex (pipeline.py:328-337)."""
        depth = {v: 0 for v in self.vertices}
        for v in self.topological_order():
            for d in self.successors(v):
                depth[d] = max(depth[d], depth[v] + 1)
        return depth


def dag_from_json(obj: Mapping[str, Any]) -> PipelineDag:
    """Structure of a pipeline document (pipeline.py:503-527)."""
    names = tuple(op["name"] for op in obj["operations"])
    return PipelineDag(
        vertices=names,
        edges=tuple((e[0], e[1]) for e in obj["edges"]),
        branching=frozenset(op["name"] for op in obj["operations"] if op.get("branching")),
        branch_predicates={(p["src"], p["dst"]): BranchPredicate(p["attr"], p["op"], int(p["value"]))
                           for p in obj.get("branch_predicates", [])},
        fanout_rules=dict(obj.get("fanout_rules", {})),
    )
