#!/usr/bin/env python
"""Rounding sensitivity of a reduced-parity twin's parareal iteration, from the CPU oracle alone
(R27).  Two fp64 implementations that are each correct differ by rounding at every
step; the iteration carries such differences forward with its own amplification.  This script
measures that amplification directly: it runs the oracle on U_0 and on U_0 perturbed by one
relative unit of rounding (U_0 (1 + eps64 z), z = +-1 seeded), digests both runs exactly as
scripts/gen_twin_digests.py does, and writes per k the largest digest difference normalised
as in the twin test.  Calls only ``oracle`` and ``synth``.

    python scripts/twin_sensitivity.py c4r_DR-DR [kmax]
"""
from __future__ import annotations

import json
import math
import os
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


def run(o, p, u0, kmax, idx, signs):
    traj = o.coarse_sweep(u0)
    digs = [synth.digest(traj, idx, signs)]
    for _ in range(kmax):
        traj = o.iteration(traj)
        digs.append(synth.digest(traj, idx, signs))
    return digs


def main(name, kmax):
    p, _, _ = twins()[name]
    o = oracle.Oracle(p)
    oracle.set_threads(int(os.environ.get("ORACLE_THREADS", oracle.host_threads())))
    idx, signs = synth.sample_indices(p.npts), synth.projection_signs(p.npts)
    u0 = synth.initial_state(p)
    z = np.where(np.random.default_rng(12345).random(u0.shape) < 0.5, -1.0, 1.0)
    u1 = u0 * (1.0 + 2.0 ** -52 * z)
    t0 = time.time()
    a, b = run(o, p, u0, kmax, idx, signs), run(o, p, u1, kmax, idx, signs)
    scale0 = float(np.max(np.abs(u0)))
    sens = []
    for k in range(kmax + 1):
        scale = max(scale0, float(np.max(a[k]["inf"])))
        es = float(np.max(np.abs(a[k]["samples"] - b[k]["samples"]))) / scale
        ep = float(np.max(np.abs(a[k]["proj"] - b[k]["proj"]))) / (scale * math.sqrt(p.npts))
        sens.append(max(es, ep))
        print(f"{name}: k = {k} relative digest change {sens[-1]:.3e}", flush=True)
    meta = {"name": name, "kmax": kmax, "perturbation": "U_0 (1 + 2^-52 z), z = +-1 (rng 12345)",
            "sensitivity": sens, "seconds": time.time() - t0, "script": "scripts/twin_sensitivity.py"}
    with open(os.path.join(OUT, f"{name}_sens.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3)
