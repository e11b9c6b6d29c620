"""Build recipe for the native libraries (in-tree, so the .so files travel to the GPU box).

* ``_lib/libmssz_b200.so``  — CUDA sm_100a kernels + host engine + C-ABI
  (``include/mssz_cuda.h``), from ``csrc/engine.cu``.
* ``_lib/libmssz_inputs.so`` — host-side synthetic field generators and the
  base-codec reconstruction that produce bench inputs (``csrc/inputs.cpp``).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
CUDA_SO = os.path.join(LIBDIR, "libmssz_b200.so")
INPUTS_SO = os.path.join(LIBDIR, "libmssz_inputs.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-ldl", "-lz",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def build(force: bool = False, verbose: bool = False) -> None:
    os.makedirs(LIBDIR, exist_ok=True)
    cu_deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))]
    cu_deps.append(os.path.join(ROOT, "include", "mssz_cuda.h"))
    if force or _stale(CUDA_SO, cu_deps):
        _run([_nvcc(), *NVCC_FLAGS, "-o", CUDA_SO, os.path.join(CSRC, "engine.cu")], verbose)
    in_deps = [os.path.join(CSRC, "inputs.cpp")]
    if force or _stale(INPUTS_SO, in_deps):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
              "-o", INPUTS_SO, os.path.join(CSRC, "inputs.cpp")], verbose)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
