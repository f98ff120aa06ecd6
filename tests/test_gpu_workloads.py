"""Full-size parity of BASELINE configs 3-5 through the bench workloads (B200).

Each runs `bench.py --workload cN` once and requires the line's own full-size checker to report
bit-identical results: config 3 every slack value of the 100k-instance launch vs the C forward
DP; config 4 all 22.4M decisions vs the literal path-list Alg. 1 + OpTable.select scan in C;
config 5 the first 8 batches decision by decision and the final table after all 256 batches vs
the C sequential fold of the run's observation stream."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _run(*args):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "2", "--warmup", "3",
                        "--no-cpu-baseline", *args], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_config3_full_launch_parity():
    line = _run("--workload", "c3")
    assert line["parity"]["mismatches"] == 0 and line["parity"]["slack_values"] == 100_000 * 64 * 4


def test_config4_all_decisions_parity():
    line = _run("--workload", "c4")
    assert line["parity"]["mismatches"] == 0 and line["parity"]["decisions"] == 22_400_000


def test_config5_batches_and_final_table_parity():
    line = _run("--workload", "c5")
    p = line["parity"]
    assert p["result"] == "bit-identical", p
    assert p["batches_decisions_checked"] == 8 and p["final_table_mismatches"] == 0
    assert p["observations_folded"] > 0
