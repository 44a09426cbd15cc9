"""Build libmcs.so in-tree with nvcc for sm_100a (no torch JIT, no CPU fallback).

    python -m paper_2504_18056_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmcs.so")
SOURCES = ["api.cu", "kf_store.cu", "select.cu", "sweep.cu", "update.cu", "weights.cu", "dist.cu",
           "predict.cu", "diversity.cu"]
HEADERS = ["mcs_internal.cuh", "reduce.cuh", "se3.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libmcs")
    return p


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), lib: str | None = None,
          build_dir: str | None = None) -> str:
    """Compile every csrc/*.cu for sm_100a and link libmcs.so (or `lib` for experiment
    variants built with extra -D `defines` into `build_dir`)."""
    global BUILD, LIB
    saved = (BUILD, LIB)
    if lib:
        LIB, BUILD = lib, build_dir or (lib + ".build")
    try:
        return _build(force, verbose, list(defines))
    finally:
        BUILD, LIB = saved


CHECKED_LIB = os.path.join(HERE, "libmcs_checked.so")


def build_checked(force: bool = False) -> str:
    """The same library with the device-side invariant checks compiled in (-DMCS_DEVICE_CHECKS:
    index bounds, probe-loop termination, ladder/donor invariants; a failure traps).  Used by
    tests/test_gpu_checked.py; never the product path."""
    return build(force=force, defines=["MCS_DEVICE_CHECKS"], lib=CHECKED_LIB,
                 build_dir=os.path.join(HERE, "_build_checked"))


def _build(force: bool, verbose: bool, defines: list[str]) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "mcs.h"),
                                                        os.path.abspath(__file__)]
    objs = []
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            futs = [ex.submit(subprocess.run, j, capture_output=True, text=True) for j in jobs]
            for j, f in zip(jobs, futs):
                r = f.result()
                if verbose or r.returncode:
                    sys.stderr.write(r.stdout + r.stderr)
                if r.returncode:
                    raise RuntimeError(f"nvcc failed: {' '.join(j)}")
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
               "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
