"""Diagnostic (GPU box): where c4's full-size k = 0 iterate (32 FIE coarse steps) departs from the
stored oracle digest, and each implementation's single coarse step against the extended-precision
step (tests/xprec.py) from the same state."""
import json, math, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import oracle, synth
from synth import FIE
from tests.xprec import XStep
import paper_2502_08370_b200 as prs

d = np.load("tests/golden/twins/c4_k1.npz")
meta = json.loads(str(d["meta"]))
p = synth.Problem(**meta["problem"])
idx, signs = d["idx"], synth.projection_signs(p.npts)
u0 = synth.initial_state(p)
ctx = prs.Context(p)
ctx.set_initial(torch.from_numpy(u0).cuda())
ctx.coarse_sweep()
buf = torch.empty((p.n,) * p.dim, dtype=torch.float64, device="cuda")
traj = np.stack([ctx.get_slice(n, buf).cpu().numpy().copy() for n in range(p.N + 1)])
g = synth.digest(traj, idx, signs)
scale0 = float(np.max(np.abs(u0)))
for n in range(p.N + 1):
    es = float(np.max(np.abs(g["samples"][n] - d["samples"][0][n]))) / scale0
    print(f"slice {n:2d} inf {g['inf'][n]:.6e} sample err / |U0| {es:.3e}", flush=True)
dT = p.T / p.N
xs = XStep(p)
o = oracle.Oracle(p)
out = torch.empty_like(buf)
for n in (0, 16):
    u = traj[n]
    t = time.time()
    ref, sc = xs.step(FIE, dT, (n + 1) * dT, u)
    want = o.step(FIE, dT, (n + 1) * dT, u)
    ctx.step(FIE, dT, (n + 1) * dT, torch.from_numpy(u).cuda(), out)
    got = out.cpu().numpy()
    nref = float(np.max(np.abs(ref)))
    ec = float(np.max(np.abs(want.astype(np.longdouble) - ref))) / nref
    eg = float(np.max(np.abs(got.astype(np.longdouble) - ref))) / nref
    print(f"step from slice {n}: oracle {ec:.3e}  GPU {eg:.3e}  (of |U_n+1|; scale/|U| {sc / nref:.2f}) {time.time() - t:.0f}s", flush=True)
ctx.close()
