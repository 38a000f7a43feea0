"""Build libkgs_b200.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2502_09537_b200.build [--force] [--checked] [--experimental]

-fmad=false keeps the reference's un-contracted fp64 arithmetic
(numba/LLVM without fastmath, dpavf/kernels.py:20) so results are bitwise
identical; -lineinfo maps ncu source pages back to kgs_device.cuh.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libkgs_b200.so"
SOURCES = [CSRC / "kgs_host.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + [REPO / "include" / "kgs_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-shared",
    f"-I{REPO / 'include'}",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS)


CHECKED_OUT = PKG / "libkgs_b200_checked.so"
EXPERIMENTAL_OUT = PKG / "libkgs_b200_exp.so"


def build(force: bool = False, verbose: bool = False, checked: bool = False,
          experimental: bool = False) -> Path:
    """checked: -DKGS_CHECKED (index asserts that trap) into
    libkgs_b200_checked.so, for tools/sanitize_run.py; experimental:
    -DKGS_EXPERIMENTAL (the slower fused one-march step, clustered /
    producer-warp march variants, kgs_debug_pass) into
    libkgs_b200_exp.so.  Neither is loaded by default (select one with
    KGS_B200_LIB)."""
    flags = (["-DKGS_CHECKED"] if checked else []) + (["-DKGS_EXPERIMENTAL"] if experimental
                                                      else [])
    out = (EXPERIMENTAL_OUT if experimental else CHECKED_OUT) if flags else OUT
    if not force and not flags and up_to_date():
        return OUT
    tmp = out.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, *flags, "-o", str(tmp), *map(str, SOURCES), "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv,
                experimental="--experimental" in sys.argv))
