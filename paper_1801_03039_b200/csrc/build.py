"""In-tree build of the product library ``libebic_b200.so`` (sm_100a only).

Invoked by ``__graft_entry__.build()`` and ``python paper_1801_03039_b200/csrc/build.py``
(a standalone script: importing the package itself would load the library it builds).
nvcc cross-compiles for sm_100a without a GPU.  The library statically links the
CUDA runtime so the .so that travels with gpurun is self-contained.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

CSRC = Path(__file__).resolve().parent
PKG = CSRC.parent
REPO = PKG.parent
LIB = PKG / "libebic_b200.so"
SOURCES = [CSRC / "ebic_b200.cu", CSRC / "synth.cpp", CSRC / "toprank.cpp"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + [REPO / "include" / "ebic_b200.h"]
E2E = PKG / "ebic_e2e_driver"
E2E_SRC = CSRC / "e2e_driver.cu"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -ffp-contract=off: host-side fitness/synth arithmetic must not fuse into FMAs
# (bit-exact parity with the reference's x86-64 SSE2 arithmetic).
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC,-O2,-ffp-contract=off,-fvisibility=hidden",
         "-Xptxas", "-warn-spills"] + os.environ.get("EBIC_NVCC_EXTRA", "").split()  # (experiments only)


def needs_build() -> bool:
    if not LIB.exists() or not E2E.exists() or E2E_SRC.stat().st_mtime > E2E.stat().st_mtime:
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(verbose: bool = False, force: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, *FLAGS, "-shared", "-o", str(tmp), *map(str, SOURCES)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=str(PKG))
    os.replace(tmp, LIB)
    build_e2e(verbose)
    return LIB


def build_e2e(verbose: bool = False) -> Path:
    """C++ caller of the public C ABI used by bench.py for the e2e figure."""
    cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-o", str(E2E), str(E2E_SRC), "-L", str(PKG),
           "-lebic_b200", "-Xlinker", "-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=str(PKG))
    return E2E


def ptxas_report() -> str:
    """Register / spill / shared-memory report of every kernel (-Xptxas -v)."""
    cmd = [NVCC, *ARCH, *FLAGS, "-Xptxas", "-v", "-c", "-o", "/dev/null", str(SOURCES[0])]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=str(PKG))
    return r.stderr


if __name__ == "__main__":
    if "--ptxas" in sys.argv:
        print(ptxas_report())
    else:
        print(build(verbose=True, force="--force" in sys.argv))
