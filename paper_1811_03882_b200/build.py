"""Build libacct_sm100.so in-tree (sm_100a only).

    python -m paper_1811_03882_b200.build          # incremental
    python -m paper_1811_03882_b200.build --force
    python -m paper_1811_03882_b200.build --profiling   # tools/ only

`--profiling` builds `libacct_sm100_prof.so` with `-DACCT_PROFILING`: the
pipeline-analysis knobs that skip work (ACCT_SKIP in acct_common.cuh) exist
only there; tools load it with `ACCT_LIB=<path>`.  The product library never
contains them.

CUDA sources are compiled with `-gencode arch=compute_100a,code=sm_100a
-lineinfo -O3`; the host-loop file with g++ `-O3 -march=x86-64-v3
-ffp-contract=off` (vectorized, but no FMA contraction, so host loops stay
bit-identical to the gcc-compiled C-subset program).  cudart is linked
statically; the driver API (TMA descriptors) is reached through
cudaGetDriverEntryPoint, so nothing but libcuda is needed at run time.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = REPO / "include"
BUILD = PKG / "_build"
LIB = PKG / "libacct_sm100.so"
PROF_BUILD = PKG / "_build_prof"
PROF_LIB = PKG / "libacct_sm100_prof.so"

CUDA_SOURCES = ["acct_runtime.cu", "acct_elementwise.cu", "acct_gemm_simt.cu", "acct_gemm_tc.cu"]
HOST_SOURCES = ["acct_host.cpp"]
HEADERS = ["acct_common.cuh", "acct_tc.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _newer(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return False
    t = target.stat().st_mtime
    return all(d.stat().st_mtime <= t for d in deps if d.exists())


def _run(cmd: list[str]):
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd)}")
    return proc


def build_library(force: bool = False, verbose: bool = False, profiling: bool = False) -> Path:
    build, lib = (PROF_BUILD, PROF_LIB) if profiling else (BUILD, LIB)
    defs = ["-DACCT_PROFILING"] if profiling else []
    build.mkdir(exist_ok=True)
    headers = [CSRC / h for h in HEADERS] + [INCLUDE / "acct.h"]
    objects = []
    for src in CUDA_SOURCES:
        obj = build / (src + ".o")
        if force or not _newer(obj, [CSRC / src, *headers, Path(__file__)]):
            cmd = [nvcc(), *ARCH, *defs, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v" if verbose else "-O3", f"-I{INCLUDE}", f"-I{CSRC}",
                   "-c", str(CSRC / src), "-o", str(obj)]
            out = _run(cmd)
            if verbose:
                sys.stderr.write(out.stderr)
        objects.append(obj)
    for src in HOST_SOURCES:
        obj = build / (src + ".o")
        if force or not _newer(obj, [CSRC / src, INCLUDE / "acct.h", Path(__file__)]):
            _run(["g++", "-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fPIC", "-std=c++17",
                  f"-I{INCLUDE}", "-c", str(CSRC / src), "-o", str(obj)])
        objects.append(obj)
    if force or not _newer(lib, objects):
        tmp = lib.with_suffix(".so.tmp")
        _run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(tmp),
              *[str(o) for o in objects], "-lpthread", "-ldl", "-lrt"])
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv,
                        profiling="--profiling" in sys.argv))
