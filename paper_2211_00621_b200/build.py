"""Build the sm_100a C-ABI library (libpmxb200.so) and the CPU oracle.

`nvcc -gencode arch=compute_100a,code=sm_100a` cross-compiles here without a
GPU; the .so files are written in-tree so they travel to the GPU box with the
repository snapshot. Rebuilds only what is out of date.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libpmxb200.so"
INCLUDE = ROOT / "include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    f"-I{INCLUDE}",
]


def _sources() -> list[pathlib.Path]:
    return sorted(CSRC.glob("*.cu"))


def _deps() -> list[pathlib.Path]:
    return sorted(CSRC.glob("*.cuh")) + [INCLUDE / "pmx_b200.h"]


def _stale(target: pathlib.Path, inputs: list[pathlib.Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(p.stat().st_mtime > t for p in inputs)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:4])} ...")


def build_lib(verbose: bool = False) -> pathlib.Path:
    BUILD.mkdir(exist_ok=True)
    deps = _deps()
    jobs = []
    objs = []
    for src in _sources():
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if _stale(obj, [src] + deps):
            jobs.append([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            list(ex.map(_run, jobs))
    if jobs or _stale(LIB, objs):
        # -cudart static: the library carries its own runtime and shares the
        # driver's primary context with torch.
        _run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
              "-cudart", "static", "-o", str(LIB), *map(str, objs)])
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_oracle(verbose: bool = False) -> pathlib.Path:
    odir = ROOT / "oracle"
    src = odir / "pmx_oracle.c"
    out = odir / "liboracle.so"
    if _stale(out, [src]):
        # -ffp-contract=off: no FMA contraction, CPython evaluates a*b+c as two
        # rounded operations; -fno-fast-math keeps libm and IEEE semantics.
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
              "-ffp-contract=off", "-fno-fast-math", "-o", str(out), str(src), "-lm"])
    if verbose:
        print(f"built {out}")
    return out


if __name__ == "__main__":
    build_lib(verbose=True)
    build_oracle(verbose=True)
