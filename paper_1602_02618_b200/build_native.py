"""Build libcjt_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1602_02618_b200.build_native [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
OUT = HERE / "_lib" / "libcjt_b200.so"
SOURCES = ["cjt_capi.cu", "cjt_chirpz.cu", "cjt_recur.cu", "cjt_shift.cu", "cjt_half.cu", "cjt_umma.cu", "cjt_host.cpp", "cjt_plan_dev.cu"]
HEADERS = ["cjt_internal.cuh", "cjt_tma.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    # host code (libm angles) must not contract into FMA: the plan's x and
    # x -+ 1 values have to match the reference kernel's bit for bit
    "-Xcompiler", "-ffp-contract=off",
]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [HERE.parent / "include" / "cjt.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = True, out: Path | None = None) -> Path:
    """Compile the library (extra nvcc flags from $CJT_NVCC_EXTRA, for experiments)."""
    target = out or OUT
    if out is None and not force and not needs_build():
        return OUT
    target.parent.mkdir(parents=True, exist_ok=True)
    extra = os.environ.get("CJT_NVCC_EXTRA", "").split()
    # compile each TU separately (parallel), then link
    objs = []
    procs = []
    for s in SOURCES:
        obj = target.parent / (Path(s).stem + ".o")
        objs.append(obj)
        cmd = [_nvcc(), *[f for f in NVCC_FLAGS if f != "-shared"], *extra, "-c", "-o", str(obj),
               str(CSRC / s)]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(target),
           *map(str, objs), "-lquadmath", "-lcublas", "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    for o in objs:
        o.unlink(missing_ok=True)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv)
