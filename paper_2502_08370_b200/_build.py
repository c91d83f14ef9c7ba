"""Build libprs.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with gpurun)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libprs.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + \
        [os.path.join(ROOT, "include", "prs.h"), __file__]


SO_CHK = os.path.join(HERE, "libprs_chk.so")  # -DPRS_CHECKS: bounds / protocol checks (test builds)


def build(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    so = SO_CHK if checks else SO
    newest = max(os.path.getmtime(f) for f in deps())
    if not force and os.path.exists(so) and os.path.getmtime(so) >= newest:
        return so
    cmd = [NVCC] + FLAGS + (["-DPRS_CHECKS"] if checks else []) + ["-o", so + ".tmp"] + sources() + ["-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    build(force=True, verbose=True)
