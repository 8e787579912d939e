"""The C-ABI library builds for sm_100a, loads, and exports every symbol that
include/gsvr_b200.h declares (CPU-only: no compute calls)."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "gsvr_b200.h"
LIB = ROOT / "paper_2512_11624_b200" / "_lib" / "libgsvr_b200.so"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gsvr_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        subprocess.run(["make", "-s", "-j8", "-C", str(LIB.parent.parent / "csrc")], check=True)
    from paper_2512_11624_b200 import _native
    return _native.lib()


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("gsvr_render_forward", "gsvr_train_step_backward", "gsvr_knn_build",
              "gsvr_knn_query", "gsvr_train_tiles", "gsvr_field_adamw_step",
              "gsvr_slice_adamw_step", "gsvr_eval_field", "gsvr_batch_refresh"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_bindings_cover_the_header(lib):
    from paper_2512_11624_b200 import _native
    assert set(declared_symbols()) == set(_native.exported_symbols())
    assert lib.gsvr_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(LIB)],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle."""
    pkg = ROOT / "paper_2512_11624_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f
