"""Build the sm_100a shared library in-tree (nvcc -shared, no JIT cache).

    python -m paper_2604_20384_b200.build
produces paper_2604_20384_b200/libtn_hvp.so (the C ABI of include/tn_hvp.h)
and paper_2604_20384_b200/bin/fp64_peak (FP64 roofline probe).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libtn_hvp.so")
BIN = os.path.join(HERE, "bin")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-Xptxas", "-O3"]
SOURCES = ["zgemm.cu", "kernels.cu", "spectrum.cu", "engine.cu", "abi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "tn_hvp.h"))
    jobs = []
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if _stale(o, [s] + headers):
            jobs.append([NVCC, *ARCH, *FLAGS, "-c", s, "-o", o])
    with ThreadPoolExecutor(max_workers=min(4, max(1, len(jobs)))) as ex:
        for r in ex.map(_run, jobs):
            if verbose and r.stderr:
                print(r.stderr, file=sys.stderr)
    if _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcusolver", "-lcublas", "-lcudart"])
    os.makedirs(BIN, exist_ok=True)
    peak = os.path.join(BIN, "fp64_peak")
    src = os.path.join(CSRC, "fp64_peak.cu")
    if _stale(peak, [src]):
        _run([NVCC, *ARCH, "-O3", "-o", peak, src])
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
