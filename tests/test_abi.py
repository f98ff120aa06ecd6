"""C-ABI boundary checks that need no GPU: the library builds for sm_100a, loads, exports
exactly the entry points include/slackpipe_b200.h declares, and refuses to run (no CPU
fallback) when no B200 is visible."""
from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "slackpipe_b200.h"


def header_functions() -> set[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(sp_[a-z_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    from paper_2102_01887_b200 import _build, _lib

    lib = _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (sp_[a-z_]+)$", out, flags=re.M))
    declared = header_functions()
    assert declared, "no declarations parsed"
    assert declared == exported
    assert declared == set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    from paper_2102_01887_b200 import _build

    lib = _build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_tma_bulk_copy_in_decision_kernel_sass():
    """K2b stages its plan with cp.async.bulk (SASS UBLKCP) — the TMA path."""
    from paper_2102_01887_b200 import _build

    lib = _build.build()
    sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
    blocks = sass.split("Function : ")
    plan = [b for b in blocks if "k_select_plan" in b.splitlines()[0]]
    assert plan and all("UBLKCP" in b for b in plan)


def test_library_loads_and_binds():
    from paper_2102_01887_b200 import _lib

    lib = _lib.load_library()
    assert lib.sp_version() == 10000
    assert lib.sp_last_error(None) is not None


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2102_01887_b200 as sp

    with pytest.raises(sp.SlackpipeError):
        sp.get_context(0)


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2102_01887_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f
