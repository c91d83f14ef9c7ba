"""Diagnostic (GPU box): one DD FIE step from a smooth state against the extended-precision
step (tests/xprec.py), GPU and oracle, over grid size / tau / DD stage variant."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import oracle, synth
from synth import FIE, DR
from tests.xprec import XStep
import paper_2502_08370_b200 as prs

cases = [(256, 0.5), (256, 1 / 32), (512, 1 / 32), (1024, 1 / 32), (1024, 1 / 512)]
for n, tau in cases:
    p = synth.CONFIGS["c4"].replace(n=n)
    u = synth.initial_state(p)
    t = time.time()
    ref, sc = XStep(p).step(FIE, tau, tau, u)
    want = oracle.Oracle(p).step(FIE, tau, tau, u)
    nref = float(np.max(np.abs(ref)))
    ec = float(np.max(np.abs(want.astype(np.longdouble) - ref))) / nref
    line = f"n {n:5d} tau {tau:.4g} s {tau * (n + 1) ** 2:.3g}: oracle {ec:.3e}"
    for env in ({}, {"PRS_DDREFINE": "0"}, {"PRS_DDSPLIT": "0"}):
        for k in ("PRS_DDREFINE", "PRS_DDSPLIT"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ctx = prs.Context(p.replace(N=1))
        du = torch.from_numpy(u).cuda()
        out = torch.empty_like(du)
        ctx.step(FIE, tau, tau, du, out)
        got = out.cpu().numpy()
        ctx.close()
        eg = float(np.max(np.abs(got.astype(np.longdouble) - ref))) / nref
        line += f"  GPU{env or ''} {eg:.3e}"
    print(line + f"  ({time.time() - t:.0f}s)", flush=True)
