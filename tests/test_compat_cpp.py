"""The reference-shaped C++ API (include/longconv_b200.hpp, liblongconv_b200.so):
code written against the reference's longconv layer builds unchanged (CPU)
and agrees with the oracle on a B200 (GPU)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2302_06646_b200"
BIN = ROOT / "build" / "compat_test"


def build_binary():
    from oracle.oracle import LC_LIB, build_oracles
    from paper_2302_06646_b200.build import build, build_compat

    build(verbose=False)
    build_compat()
    if not LC_LIB.exists():
        build_oracles(with_ref=False)
    BIN.parent.mkdir(exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", str(ROOT / "tests" / "cpp" / "compat_test.cpp"),
           f"-I{ROOT / 'include'}", f"-L{PKG}", "-llongconv_b200", "-lflashbutterfly",
           f"-L{LC_LIB.parent}", "-llcoracle", "-L/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{PKG}:{LC_LIB.parent}", "-o", str(BIN)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return BIN


def test_reference_shaped_api_compiles():
    assert build_binary().exists()


@pytest.mark.gpu
def test_reference_shaped_api_on_device():
    b = build_binary()
    r = subprocess.run([str(b)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and "COMPAT OK" in r.stdout, r.stdout + r.stderr
