"""Profile ingest: the reference's on-disk profile format straight into device tables.

The reference profiles every operation once and caches the result as JSON in a
content-addressed metadata directory (``MetadataStore``, profiler.py:106-168):
``configspec-<operation>-<key16>.json`` holds ``ConfigSpec.to_json()`` (pipeline.py:217-279,
``json.dump(..., indent=1, sort_keys=True)``) and ``paths-<hash16>.json`` the decomposed path
set of a pipeline.  This module reads that directory (no re-profiling, no reference import) and
builds the GPU-backed ``OpTable`` of every operation and the ``SlackGraph`` of a path set —
the format step in front of the decision path.
"""
from __future__ import annotations

import json
import os
import re
from pathlib import Path
from typing import Mapping, Sequence

from .pipeline import ConfigSpec

METADATA_DIR_ENV = "SLACKPIPE_METADATA_DIR"  # profiler.py:31
_PROFILE_RE = re.compile(r"^configspec-(?P<op>.+)-(?P<key>[0-9a-f]{16})\.json$")
_PATHS_RE = re.compile(r"^paths-(?P<key>[0-9a-f]{16})\.json$")


def metadata_root(root: str | os.PathLike | None = None) -> Path:
    """profiler.py:115-118: explicit root, else $SLACKPIPE_METADATA_DIR, else the default."""
    if root is None:
        root = os.environ.get(METADATA_DIR_ENV, ".slackpipe-metadata")
    return Path(root)


def load_config_spec(path: str | os.PathLike) -> ConfigSpec:
    """One cached profile (MetadataStore.load_profile, profiler.py:124-129)."""
    with open(path, "r", encoding="utf-8") as fh:
        return ConfigSpec.from_json(json.load(fh))


def dump_config_spec(spec: ConfigSpec, path: str | os.PathLike) -> None:
    """Byte-identical to MetadataStore.store_profile (profiler.py:131-136)."""
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(spec.to_json(), fh, indent=1, sort_keys=True)
        fh.write("\n")


def profile_files(root: str | os.PathLike | None = None) -> dict[str, list[Path]]:
    """Operation name -> cached profile files of the metadata directory."""
    out: dict[str, list[Path]] = {}
    for p in sorted(metadata_root(root).glob("configspec-*.json")):
        m = _PROFILE_RE.match(p.name)
        if m:
            out.setdefault(m.group("op"), []).append(p)
    return out


def load_profiles(root: str | os.PathLike | None = None,
                  operations: Sequence[str] | None = None) -> dict[str, ConfigSpec]:
    """Every cached profile (or the named operations').  An operation with several cached
    profiles (different knob templates / executables) is ambiguous without its
    OperationSpec and raises ValueError; pass ``files`` to ``load_config_spec`` instead."""
    files = profile_files(root)
    names = list(operations) if operations is not None else sorted(files)
    out = {}
    for op in names:
        got = files.get(op, [])
        if not got:
            raise KeyError(f"no cached profile for operation {op!r} under {metadata_root(root)}")
        if len(got) > 1:
            raise ValueError(f"operation {op!r} has {len(got)} cached profiles: {[g.name for g in got]}")
        spec = load_config_spec(got[0])
        if spec.operation != op:
            raise ValueError(f"{got[0].name}: holds operation {spec.operation!r}")
        out[op] = spec
    return out


def load_paths(root: str | os.PathLike | None = None, pipeline_hash: str | None = None):
    """Decomposed path set (MetadataStore.load_paths, profiler.py:141-148); without a hash the
    directory must hold exactly one path set."""
    base = metadata_root(root)
    if pipeline_hash is not None:
        p = base / f"paths-{pipeline_hash[:16]}.json"
    else:
        cands = [p for p in sorted(base.glob("paths-*.json")) if _PATHS_RE.match(p.name)]
        if len(cands) != 1:
            raise ValueError(f"{base}: expected one paths-*.json, found {len(cands)}")
        p = cands[0]
    with open(p, "r", encoding="utf-8") as fh:
        return tuple(tuple(x) for x in json.load(fh))


def tables_from_metadata(scenario, root: str | os.PathLike | None = None,
                         operations: Sequence[str] | None = None, *,
                         kinds: Sequence[str] | None = None, device: int | None = None) -> dict:
    """Device tables (``OpTable``, configurator.py:166-209 filter) of every cached profile."""
    from .configurator import OpTable

    specs = load_profiles(root, operations)
    return {op: OpTable(spec, scenario, kinds=kinds, device=device) for op, spec in specs.items()}


def slack_graph_from_metadata(root: str | os.PathLike | None = None, pipeline_hash: str | None = None,
                              sources: Sequence[str] | None = None, *, device: int | None = None):
    """K1 graph of a cached path set (SlackGraph.from_paths)."""
    from .slack import SlackGraph

    return SlackGraph.from_paths(load_paths(root, pipeline_hash), sources, device=device)


def specs_equal(a: ConfigSpec, b: Mapping) -> bool:
    """Field-wise equality with another ConfigSpec-like object (reference or ours)."""
    return json.dumps(a.to_json(), sort_keys=True) == json.dumps(
        b.to_json() if hasattr(b, "to_json") else b, sort_keys=True)
