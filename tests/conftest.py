from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and libslackpipe_b200.so (run on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running (full-size parity)")


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def golden_json(d: dict, key: str):
    return json.loads(bytes(d[key]).decode())


def reference_available() -> bool:
    return (REF_SRC / "slackpipe" / "__init__.py").exists()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference package (build container only)."""
    if not reference_available():
        pytest.skip("reference package not present (GPU box)")
    sys.path.insert(0, str(REF_SRC))
    import slackpipe

    return slackpipe


@pytest.fixture(scope="session")
def gpu_ctx():
    """The library context on cuda:0 — fails loudly (no skip) when the GPU path is missing."""
    import paper_2102_01887_b200 as sp

    return sp.get_context(0)


KINDS3 = ["cpu", "gpu", "lite"]


def select_case_specs(d: dict):
    """Rebuild (spec, scenario, case-index) triples of select_cases.npz with package types."""
    from paper_2102_01887_b200.pipeline import ConfigEntry, ConfigSpec
    from paper_2102_01887_b200.scenario import BackendSpec, Scenario

    b = d["backends"]
    sc = Scenario("golden", tuple(BackendSpec(k, int(b[i, 0]), int(b[i, 1]), float(b[i, 2]))
                                  for i, k in enumerate(KINDS3)))
    off = d["off"]
    out = []
    for c in range(len(off) - 1):
        ents = []
        for j in range(off[c], off[c + 1]):
            kind = KINDS3[int(d["ent_kind"][j])]
            res, batch, knob = int(d["ent_res"][j]), int(d["ent_batch"][j]), int(d["ent_knob"][j])
            lat = float(d["ent_lat"][j])
            ents.append(ConfigEntry(f"{kind}-r{res}-b{batch}-i={knob}", kind, {"i": knob}, batch, res,
                                    lat, lat, schedulable=bool(d["ent_sched"][j])))
        out.append(ConfigSpec("op", ents, ents[0].config_id))
    return sc, out
