"""Build libflashbutterfly.so in-tree for sm_100a (nvcc, no JIT cache).

    python -m paper_2302_06646_b200.build        # or __graft_entry__.build()

The .so lands next to this file so it travels to the GPU box with the
repository snapshot.  Rebuilds only when a source is newer than the library.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libflashbutterfly.so"
COMPAT_SRC = CSRC / "compat" / "longconv_compat.cpp"
COMPAT_LIB = PKG / "liblongconv_b200.so"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
INCLUDE = PKG.parent / "include"

SOURCES = ["fb_capi.cu", "fb_prep.cu", "fb_single.cu", "fb_single_tc.cu", "fb_tc2.cu",
           "fb_three.cu", "fb_learned.cu", "fb_learned_tc.cu", "fb_dft.cu", "fb_shard.cu", "fb_lconv.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills"]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _stale(lib: Path, deps) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = True) -> Path:
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps += list(INCLUDE.glob("*.h"))
    if not force and not _stale(LIB, deps):
        build_compat()
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs = []
    procs = []
    for s in SOURCES:
        o = objdir / (Path(s).stem + ".o")
        objs.append(o)
        if force or _stale(o, [CSRC / s] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
                           + list(INCLUDE.glob("*.h"))):
            cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, "-I", str(INCLUDE), "-c", str(CSRC / s), "-o", str(o)]
            procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                              text=True)))
    for s, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}:\n{out}")
        if verbose and out.strip():
            print(out, file=sys.stderr)
    cmd = [_nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
    subprocess.run(cmd, check=True)
    build_compat(force=True)
    return LIB


def build_compat(force: bool = False) -> Path:
    """liblongconv_b200.so: the reference-shaped C++ API (include/longconv_b200.hpp)."""
    deps = [COMPAT_SRC, INCLUDE / "longconv_b200.hpp", INCLUDE / "flashbutterfly.h", LIB]
    if not force and not _stale(COMPAT_LIB, deps):
        return COMPAT_LIB
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", f"-I{INCLUDE}",
           f"-I{CUDA_HOME / 'include'}", str(COMPAT_SRC), f"-L{PKG}", "-lflashbutterfly",
           f"-L{CUDA_HOME / 'lib64'}", "-lcudart", "-Wl,-rpath,$ORIGIN", "-o", str(COMPAT_LIB)]
    subprocess.run(cmd, check=True)
    return COMPAT_LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
