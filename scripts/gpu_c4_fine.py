"""GPU side of scripts/xprec_c4_fine.py: F^s(U_0) of c4 (s FIE steps at delta t) through the C ABI,
saved to gpurun_out/c4_F_gpu.npy."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import synth
from synth import FIE
import paper_2502_08370_b200 as prs

p = synth.CONFIGS["c4"]
dt = p.T / (p.N * p.s)
ctx = prs.Context(p.replace(N=1))
a = torch.from_numpy(synth.initial_state(p)).cuda()
b = torch.empty_like(a)
for j in range(p.s):
    ctx.step(FIE, dt, (j + 1) * dt, a, b)
    a, b = b, a
ctx.close()
np.save("gpurun_out/c4_F_gpu.npy", a.cpu().numpy())
print("saved F^s(U_0)")
