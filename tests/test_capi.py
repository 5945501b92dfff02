"""CPU-side checks of the drop-in boundary: the C-ABI library builds for
sm_100a, loads, and exports every symbol include/flashbutterfly.h declares;
host-side argument validation fails loudly (no compute without a GPU)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def fblib():
    from paper_2302_06646_b200 import _lib
    from paper_2302_06646_b200.build import build

    build(verbose=False)
    return _lib


def test_header_symbols_exported(fblib):
    header = (ROOT / "include" / "flashbutterfly.h").read_text()
    declared = set(re.findall(r"\b(fb_[a-z_]+)\s*\(", header))
    assert declared == set(fblib.EXPORTED)
    L = fblib.lib()
    for name in declared:
        assert hasattr(L, name), name


def test_sm100a_cubin_in_library(fblib):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(fblib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_errors_without_gpu(fblib):
    L = fblib.lib()
    assert L.fb_version() == 100
    # null output pointer -> FB_ERR_ARG; bad shapes -> FB_ERR_DIM (DimensionError)
    assert L.fb_plan_create(None, 16, 1, 1, 0, 0, 0) == fblib.FB_ERR_ARG
    h = C.c_void_p()
    assert L.fb_plan_create(C.byref(h), 0, 1, 1, 0, 0, 0) == fblib.FB_ERR_DIM
    assert b"N and H" in L.fb_last_error()
    assert L.fb_plan_create(C.byref(h), 12, 1, 0, 0, 0, 0) == fblib.FB_ERR_PLAN  # circular non-pow2


def test_python_mirror_raises_reference_error_types(fblib):
    from paper_2302_06646_b200 import DimensionError, PlanError

    with pytest.raises(DimensionError):
        fblib.check(fblib.FB_ERR_DIM)
    with pytest.raises(PlanError):
        fblib.check(fblib.FB_ERR_PLAN)
    assert issubclass(DimensionError, ValueError)


def test_no_oracle_in_product_package():
    pkg = ROOT / "paper_2302_06646_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        src = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), f
        assert "liblcoracle" not in src and "liblongconv_ref" not in src, f
