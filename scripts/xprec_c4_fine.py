#!/usr/bin/env python
"""The oracle's own drift over one slice's fine sweep at c4's full size (R28).

Runs F^s(U_0) of c4 (s = 64 FIE steps at delta t = 1/2048, 1024^2, 8 strips, 8-cell overlap)
twice on the CPU: with the oracle (fp64, literal algorithm) and with the extended-precision step
of tests/xprec.py (80-bit residuals, iterative refinement), saving both end states; with a
third state given (the GPU's, written by a GPU run of the same sweep) it prints each one's
distance from the extended-precision value, relative to its inf norm.

    python scripts/xprec_c4_fine.py run OUTDIR          # CPU: oracle + extended precision
    python scripts/xprec_c4_fine.py compare OUTDIR GPU.npy
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import FIE  # noqa: E402
from tests.xprec import XStep  # noqa: E402


def run(out):
    p = synth.CONFIGS["c4"]
    dt = p.T / (p.N * p.s)
    u = synth.initial_state(p)
    o, xs = oracle.Oracle(p), XStep(p)
    uo, ux = u.copy(), u.astype(np.longdouble)
    t0 = time.time()
    for j in range(p.s):
        uo = o.step(FIE, dt, (j + 1) * dt, uo)
        ux, _ = xs.step(FIE, dt, (j + 1) * dt, ux)
        if j % 8 == 7 or j == p.s - 1:
            e = float(np.max(np.abs(uo.astype(np.longdouble) - ux))) / float(np.max(np.abs(ux)))
            print(f"step {j + 1}: oracle vs extended precision {e:.3e} ({time.time() - t0:.0f} s)", flush=True)
            np.save(os.path.join(out, "c4_F_oracle.npy"), uo)
            np.save(os.path.join(out, "c4_F_xprec.npy"), ux.astype(np.float64))
            np.save(os.path.join(out, "c4_F_xprec_lo.npy"), (ux - ux.astype(np.float64).astype(np.longdouble)).astype(np.float64))
            with open(os.path.join(out, "c4_F_steps.txt"), "w") as f:
                f.write(str(j + 1))


def compare(out, gpu):
    ux = np.load(os.path.join(out, "c4_F_xprec.npy")).astype(np.longdouble) + \
        np.load(os.path.join(out, "c4_F_xprec_lo.npy")).astype(np.longdouble)
    nx = float(np.max(np.abs(ux)))
    for name, f in (("oracle", os.path.join(out, "c4_F_oracle.npy")), ("GPU", gpu)):
        v = np.load(f).astype(np.longdouble)
        print(f"{name}: {float(np.max(np.abs(v - ux))) / nx:.3e} of |F^s(U_0)| off the extended-precision sweep")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        compare(sys.argv[2], sys.argv[3])
