#!/usr/bin/env python
"""Rounding floor of a reduced-parity twin's parareal iteration, from the CPU oracle alone
(R27).  Two fp64 implementations of the same literal algorithm that are each correct
differ by rounding in every step; the iteration carries those differences forward with its own
amplification.  This script measures that floor with the oracle itself: it compiles oracle.c a
second time with FMA contraction (gcc -O2 -mfma -ffp-contract=fast: every a*b+c of the literal
algorithm rounded once instead of twice -- the same algorithm, another correct rounding), runs
that build on the twin's problem for k = 0..kmax, digests the iterates exactly as
scripts/gen_twin_digests.py did for the stored digests (tests/golden/twins/<name>.npz, the
uncontracted build) and writes per k the largest digest difference, normalised as in the twin
test, to tests/golden/twins/<name>_floor.json.  Calls only ``oracle`` (rebuilt) and ``synth``.

    python scripts/twin_sensitivity.py c4r_DR-DR [kmax]
"""
from __future__ import annotations

import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import oracle  # noqa: E402
import synth  # noqa: E402
from gen_twin_digests import twins  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "twins")
FLAGS = ["-O2", "-mfma", "-ffp-contract=fast", "-fno-fast-math", "-std=c11"]


def contracted_oracle():
    so = os.path.join("/tmp", f"liboracle_fma_{os.getpid()}.so")
    subprocess.check_call(["gcc"] + FLAGS + ["-shared", "-fPIC", "-pthread", "-o", so] + oracle._SRC + ["-lm"])
    oracle._SO = so
    oracle.build = lambda force=False: so
    oracle._lib = None
    return so


def main(name, kmax):
    p, _, _ = twins()[name]
    ref = np.load(os.path.join(OUT, f"{name}.npz"))
    kmax = min(kmax, len(ref["upd"]))
    contracted_oracle()
    o = oracle.Oracle(p)
    oracle.set_threads(int(os.environ.get("ORACLE_THREADS", oracle.host_threads())))
    idx, signs = ref["idx"], synth.projection_signs(p.npts)
    u0 = synth.initial_state(p)
    t0 = time.time()
    traj = o.coarse_sweep(u0)
    scale0 = float(np.max(np.abs(u0)))
    floor = []
    for k in range(kmax + 1):
        if k > 0:
            traj = o.iteration(traj)
        g = synth.digest(traj, idx, signs)
        scale = max(scale0, float(np.max(ref["inf"][k])))
        es = float(np.max(np.abs(g["samples"] - ref["samples"][k]))) / scale
        ep = float(np.max(np.abs(g["proj"] - ref["proj"][k]))) / (scale * math.sqrt(p.npts))
        floor.append(max(es, ep))
        print(f"{name}: k = {k} contracted vs stored oracle digests {floor[-1]:.3e} ({time.time() - t0:.0f} s)",
              flush=True)
    meta = {"name": name, "kmax": kmax, "flags": " ".join(FLAGS), "floor": floor,
            "seconds": time.time() - t0, "script": "scripts/twin_sensitivity.py",
            "what": "max normalised digest difference between the oracle built with and without FMA contraction"}
    with open(os.path.join(OUT, f"{name}_floor.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3)
