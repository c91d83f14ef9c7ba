#!/usr/bin/env python
"""A short program for ncu: one BASELINE config, a coarse sweep, then `--sweeps` fine sweeps
+ corrections (the bench step) on cuda:0.  Exits 0 on success.

    python scripts/prof_step.py --config c3 --sweeps 2
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--sweeps", type=int, default=2)
    ap.add_argument("--set", action="append", default=[], metavar="KEY=VALUE")
    args = ap.parse_args()
    import torch

    import paper_2502_08370_b200 as prs
    p = synth.CONFIGS[args.config]
    for kv in args.set:
        k, v = kv.split("=", 1)
        p = p.replace(**{k: type(getattr(p, k))(float(v))})
    torch.cuda.set_device(0)
    ctx = prs.Context(p, stream=torch.cuda.current_stream().cuda_stream)
    ctx.set_initial(torch.from_numpy(synth.initial_state(p)).cuda())
    ctx.coarse_sweep()
    for _ in range(args.sweeps):
        ctx.fine_sweep()
        ctx.parareal_correct()
    torch.cuda.synchronize()
    ctx.close()
    print("ok")


if __name__ == "__main__":
    main()
