#!/usr/bin/env python
"""Print the per-iterate digest errors of a reduced-parity twin (tests/golden/twins/<name>.npz)
against the GPU run, normalised as in test_twin_iterates_match_stored_oracle_digests.

    python scripts/twin_errors.py c4r_DR-DR
"""
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def main(name):
    import torch
    import paper_2502_08370_b200 as prs
    d = np.load(os.path.join(ROOT, "tests", "golden", "twins", f"{name}.npz"))
    meta = json.loads(str(d["meta"]))
    p = synth.Problem(**meta["problem"])
    idx, signs = d["idx"], synth.projection_signs(p.npts)
    u0 = synth.initial_state(p)
    ctx = prs.Context(p)
    ctx.set_initial(torch.from_numpy(u0).cuda())
    ctx.coarse_sweep()
    buf = torch.empty((p.n,) * p.dim, dtype=torch.float64, device="cuda")
    scale0 = float(np.max(np.abs(u0)))
    worst = 0.0
    for k in range(meta["k"] + 1):
        if k > 0:
            ctx.fine_sweep()
            ctx.parareal_correct()
        traj = np.stack([ctx.get_slice(n, buf).cpu().numpy().copy() for n in range(p.N + 1)])
        g = synth.digest(traj, idx, signs)
        scale = max(scale0, float(np.max(d["inf"][k])))
        es = float(np.max(np.abs(g["samples"] - d["samples"][k]))) / scale
        ep = float(np.max(np.abs(g["proj"] - d["proj"][k]))) / (scale * math.sqrt(p.npts))
        worst = max(worst, es, ep)
        print(f"{name} k={k:2d} samples {es:.2e} proj {ep:.2e} scale {scale:.3e}")
    ctx.close()
    print(f"{name}: worst {worst:.2e}")


if __name__ == "__main__":
    main(sys.argv[1])
