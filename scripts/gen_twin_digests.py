#!/usr/bin/env python
"""Write tests/golden/twins/<name>.npz: digests of the CPU oracle's parareal iterates for the
reduced-parity twins of c3 / c4 and the full-size c4 k = 0 -> 1 iterate (SURVEY.md 8(d)
"reduced parity protocol", steps 3-4).  Calls only ``oracle`` (the literal serial algorithm;
its per-slice F / G evaluations spread over threads, bitwise identical to serial) and ``synth``
(problem shapes, initial data, sample indices / projection signs).  Nothing here comes from the
CUDA path.

Per iterate k and slice end n: the values at 128 fixed sample points, 4 +-1 projections of the
whole state and its inf norm (synth.digest); per k the normalised update (R7).

    python scripts/gen_twin_digests.py [name ...]      (default: all, in order)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import DR, FIE  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "twins")


def twins():
    c4r = dict(dim=2, n=256, c=1.0, split=1, dd_strips=8, dd_overlap=8, dd_ramp=0, source=1,
               N=32, s=64, init="phi")
    return {
        # c3r: c3's recipe (variable kappa, Parareal/FIE-DR, N = 64, s = 256) at n = 256, to the stop rule
        "c3r": (synth.Problem(dim=2, n=256, c=1.0, coef=1, source=0, N=64, s=256, G=FIE, F=DR, init="modes"),
                64, 1e-10),
        # c4r: c4's DD recipe (8 strips of 32 nodes, 8-cell overlap, linear ramp), every k to N
        "c4r_FIE-FIE": (synth.Problem(G=FIE, F=FIE, **c4r), 32, 0.0),
        "c4r_FIE-DR": (synth.Problem(G=FIE, F=DR, **c4r), 32, 0.0),
        # c4 at full size: k = 0 and k = 1
        "c4_k1": (synth.CONFIGS["c4"], 1, 0.0),
        "c4r_DR-FIE": (synth.Problem(G=DR, F=FIE, **c4r), 32, 0.0),
        "c4r_DR-DR": (synth.Problem(G=DR, F=DR, **c4r), 32, 0.0),
    }


def run(name, p, kmax, tol, threads):
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    idx = synth.sample_indices(p.npts)
    signs = synth.projection_signs(p.npts)
    oracle.set_threads(threads)
    t0 = time.time()
    traj = o.coarse_sweep(u0)
    scale = float(np.max(np.abs(u0))) or 1.0
    digs, upds = [synth.digest(traj, idx, signs)], []
    for k in range(min(kmax, p.N)):
        nxt = o.iteration(traj)
        upds.append(float(np.max(np.abs(nxt - traj))) / scale)
        traj = nxt
        digs.append(synth.digest(traj, idx, signs))
        print(f"{name}: k = {k + 1} update {upds[-1]:.3e} ({time.time() - t0:.0f} s)", flush=True)
        if tol > 0.0 and upds[-1] <= tol:
            break
    meta = {"name": name, "problem": {f: getattr(p, f) for f in p.__dataclass_fields__},
            "kmax": kmax, "tol": tol, "k": len(upds), "seconds": time.time() - t0,
            "threads": threads, "script": "scripts/gen_twin_digests.py",
            "stop": "update <= tol (DESIGN.md R7) or k = min(kmax, N); tol = 0: every k"}
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), idx=idx,
                        samples=np.stack([d["samples"] for d in digs]),
                        proj=np.stack([d["proj"] for d in digs]),
                        inf=np.stack([d["inf"] for d in digs]),
                        upd=np.array(upds), meta=json.dumps(meta))
    print(f"{name}: wrote k = 0..{len(upds)} in {meta['seconds']:.0f} s", flush=True)


def main():
    os.makedirs(OUT, exist_ok=True)
    threads = int(os.environ.get("ORACLE_THREADS", oracle.host_threads()))
    all_ = twins()
    names = sys.argv[1:] or list(all_)
    for nm in names:
        p, kmax, tol = all_[nm]
        run(nm, p, kmax, tol, threads)


if __name__ == "__main__":
    main()
