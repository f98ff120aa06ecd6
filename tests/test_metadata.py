"""Profile ingest (paper_2102_01887_b200.metadata): the reference's MetadataStore directory for
the AMBER pipeline (tests/golden/metadata_amber, written by the reference itself through
tests/golden/make_golden.py) is read without the reference and turned into device tables."""
from __future__ import annotations

import json
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, golden, golden_json

MD = GOLDEN / "metadata_amber"


def test_configspec_json_round_trip_is_byte_identical(tmp_path):
    from paper_2102_01887_b200 import metadata

    files = sorted(MD.glob("configspec-*.json"))
    assert len(files) == 7
    for f in files:
        spec = metadata.load_config_spec(f)
        out = tmp_path / f.name
        metadata.dump_config_spec(spec, out)
        assert out.read_bytes() == f.read_bytes(), f.name


def test_load_profiles_and_paths_match_the_amber_run():
    from paper_2102_01887_b200 import metadata

    meta = golden_json(golden("amber_trace"), "meta_json")
    specs = metadata.load_profiles(MD)
    assert sorted(specs) == sorted(meta["ops"])
    for op, spec in specs.items():
        t = meta["tables"][op]
        assert spec.reference_id == t["ref_id"]
        by_id = {e.config_id: e for e in spec.entries}
        for cid, lat in zip(t["config_id"], t["lat"]):  # the run's schedulable entries
            assert by_id[cid].latency_s == lat
    assert [list(p) for p in metadata.load_paths(MD)] == meta["paths"]


def test_ambiguous_and_missing_profiles_raise(tmp_path):
    from paper_2102_01887_b200 import metadata

    d = tmp_path / "md"
    shutil.copytree(MD, d)
    src = sorted(d.glob("configspec-decode-*.json"))[0]
    shutil.copy(src, d / "configspec-decode-0000000000000000.json")
    with pytest.raises(ValueError):
        metadata.load_profiles(d, ["decode"])
    with pytest.raises(KeyError):
        metadata.load_profiles(d, ["nosuchop"])
    assert len(metadata.load_profiles(d, ["detect"])) == 1


def test_same_objects_as_the_reference_loader(ref):
    from paper_2102_01887_b200 import metadata

    for f in sorted(MD.glob("configspec-*.json")):
        ours = metadata.load_config_spec(f)
        theirs = ref.pipeline.ConfigSpec.from_json(json.loads(f.read_text()))
        assert metadata.specs_equal(ours, theirs)


@pytest.mark.gpu
def test_tables_from_metadata_equal_the_run_tables(gpu_ctx):
    import paper_2102_01887_b200 as sp
    from paper_2102_01887_b200 import metadata
    from test_gpu_amber import amber_tables

    meta = golden_json(golden("amber_trace"), "meta_json")
    sc = sp.Scenario("branching", tuple(sp.BackendSpec(k, n, r, p) for k, n, r, p in meta["backends"]))
    tabs = metadata.tables_from_metadata(sc, MD, kinds=meta["kinds"])
    ref_tabs = amber_tables(meta)
    rng = np.random.default_rng(3)
    for op, rt in zip(meta["ops"], ref_tabs):
        t = tabs[op]
        assert [e.config_id for e in t.entries] == [e.config_id for e in rt.entries]
        assert np.array_equal(t.lat, rt.lat) and t.ref_index == rt.ref_index
        n = 512
        slack = rng.uniform(-1, 30, size=(n, t.K))
        args = dict(upstream_supply=rng.integers(0, 9, n).astype(np.int32),
                    min_batch=np.ones(n, np.int32), flags=np.ones(n, np.uint32))
        avail = rng.integers(1, 9, n).astype(np.int32)
        a = t.select_batch(slack, 100.0, avail, **args)
        b = rt.select_batch(slack, 100.0, avail, **args)
        assert np.array_equal(a["idx"], b["idx"]) and np.array_equal(a["code"], b["code"])
    g = metadata.slack_graph_from_metadata(MD, sources=meta["ops"])
    assert g.source_names == meta["ops"]
