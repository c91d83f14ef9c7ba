#!/usr/bin/env python
"""Benchmark: fine-propagator grid-point-updates/s of parareal with splitting propagators.

A step is one parareal iteration of the BASELINE workload (default c3: 4096^2 variable
kappa, G = FIE, F = DR, N = 64 slices x s = 256 fine steps): the batched fine sweep over
every local slice, the sequential coarse chain with the fused correction, the NCCL hand-off
between ranks and the stop-test all-reduce.  value = fine updates (n^d x N x s per step,
all ranks) / max-over-ranks device time.  One process per GPU (torchrun for N > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "fine-propagator grid-point-updates/s"
UNIT = "updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="prs", choices=["prs", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--set", action="append", default=[], metavar="KEY=VALUE",
                    help="override a Problem field of the workload (experiments; the default "
                         "run uses the BASELINE config unchanged)")
    ap.add_argument("--profile-launches", action="store_true",
                    help="under ncu: only a short run, no timing extras")
    ap.add_argument("--coarse-mode", default="owner", choices=["owner", "space"],
                    help="coarse chain: owner-G (default) or space-parallel G over P row bands "
                         "(P = GPUs; --gbands virtual bands on one GPU)")
    ap.add_argument("--gbands", type=int, default=4)
    ap.add_argument("--pipeline", type=int, default=0, metavar="BLOCKS",
                    help="pipelined parareal (prs_set_pipeline, NEXT-2): the timed steps and the "
                         "time-to-tol run as one prs_iterate over BLOCKS slice blocks (on-chip "
                         "sweep configs c0/c1/c1p; 0 = off)")
    ap.add_argument("--no-time-to-tol", action="store_true",
                    help="skip the parareal time-to-tolerance run and the sequential fine solve")
    return ap.parse_args()


def workload(args):
    p = synth.CONFIGS[args.config]
    for kv in args.set:
        k, v = kv.split("=", 1)
        cur = getattr(p, k)
        p = p.replace(**{k: type(cur)(float(v)) if not isinstance(cur, str) else v})
    return p


def stop_tol(name: str) -> float:
    """A7 / DESIGN.md R7-R8: c0 runs its fixed K = 8 (= N) iterations; c1-c4 stop at 1e-10."""
    return 0.0 if name == "c0" else 1e-10


def updates_per_step(p) -> int:
    return (p.n ** p.dim) * p.N * p.s


def workload_config(p, name, n_gpus):
    sch = {0: "FIE", 1: "DR", 2: "IE"}
    kap = {0: "1", 1: "1+0.5sin2pix sin2piy", 2: "full tensor d11=d22=1/(2+cos3pix cos2piy), d12=1/4"}[p.coef]
    return {"workload": name, "grid": f"{p.n}^{p.dim}", "kappa": kap,
            "split": "dd" if p.split else "dimensional", "pairing": f"{sch[p.G]}-{sch[p.F]}",
            "N": p.N, "s": p.s, "slices_per_gpu": p.N // n_gpus,
            "state_MiB": (p.n ** p.dim) * 8 / 2 ** 20,
            "l2": "inputs larger than L2 (state 128 MiB x 64 slices per pass)" if p.n >= 4096
            else "working set may be L2-resident"}


# --------------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi every 100 ms on a reader thread; each sample keeps its host arrival time so the
    samples of a time window (the timed region) can be picked out."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.samples = []  # (host time, line)

    def start(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                self.samples.append((time.perf_counter(), line))
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def count_since(self, t0):
        return sum(1 for t, _ in self.samples if t >= t0)

    def stop(self, t0=None, t1=None):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        lines = [ln for t, ln in self.samples if (t0 is None or t >= t0) and (t1 is None or t <= t1)]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(name):
    """dram bytes per launch of the dominant kernel from a committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", f"traffic_{name}.json")
    if os.path.exists(path):
        try:
            return json.load(open(path))
        except ValueError:
            return None
    return None


# ------------------------------------------------------------------ CPU oracle ---
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores():
    return sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count() or 1))


def oracle_sample(p, reps: int = 1):
    """Time the oracle as it stands on a bounded sample: `reps` fine steps of one slice, the
    process pinned to one host core for the sample (as taskset -c <core>)."""
    import oracle
    o = oracle.Oracle(p)
    u = synth.initial_state(p)
    dt = p.T / (p.N * p.s)
    cores = host_cores()
    pin = cores[0]
    if hasattr(os, "sched_setaffinity"):
        os.sched_setaffinity(0, {pin})
    try:
        t0 = time.perf_counter()
        for j in range(reps):
            u = o.step(p.F, dt, float(j + 1) * dt, u)
        sec = time.perf_counter() - t0
    finally:
        if hasattr(os, "sched_setaffinity"):
            os.sched_setaffinity(0, set(cores))
    upd = reps * p.n ** p.dim
    return upd / sec, sec, {"kind": "oracle", "cores": 1, "taskset": f"core {pin}", "cpu_model": cpu_model(),
                            "host_cores_available": len(cores),
                            "sample": f"{reps} fine {'DR' if p.F else 'FIE'} step(s) of one slice at "
                                      f"{p.n}^{p.dim} (serial C oracle, -O2, no FMA contraction)"}


def oracle_sample_all_cores(p, reps: int = 1):
    """The oracle's slice-parallel mode on every host core: one slice's `reps` fine steps per
    core, all cores at once (the oracle's per-slice F evaluations are independent, PAPER.md:206-210;
    ctypes releases the GIL).  Returns (aggregate updates/s, seconds, threads)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    dt = p.T / (p.N * p.s)
    th = min(len(host_cores()), 64)

    def one(b):
        u = u0 * (1.0 + b / th)
        for j in range(reps):
            u = o.step(p.F, dt, float(j + 1) * dt, u)
        return 0

    t0 = time.perf_counter()
    with ThreadPoolExecutor(th) as ex:
        list(ex.map(one, range(th)))
    sec = time.perf_counter() - t0
    return th * reps * p.n ** p.dim / sec, sec, th


def oracle_ttt_extrapolated(p, k, rate_serial, rate_all, threads):
    """Oracle parareal to k iterations, extrapolated from the measured update rates: the literal
    algorithm does N coarse steps, then per iteration N s fine + 2 N coarse steps (G(U^k_n) is
    recomputed, G(U^{k+1}_n) along the chain); the slice-parallel mode spreads the N s + N
    independent steps over the threads, the chain of N coarse steps stays serial."""
    pts = p.n ** p.dim
    serial = pts * (p.N + k * (p.N * p.s + 2 * p.N)) / rate_serial
    par_rounds = -(-p.N // max(1, threads))
    allc = pts * (p.N + k * (par_rounds * (p.s + 1) + p.N)) / (rate_all / max(1, threads))
    return {"serial_s": serial, "all_cores_s": allc, "iterations": k,
            "how": "measured oracle update rates x the work of the literal algorithm (coarse steps "
                   "counted at the fine-scheme rate)"}


def oracle_reps_for(p):
    # about 10 s of serial oracle work per sample
    per_pt = {2: 0.6e-6 if p.coef else 0.12e-6, 3: 0.15e-6}[p.dim]
    if p.split:  # band elimination of the DD strip blocks (bandwidth ~ strip width)
        per_pt = 2.5e-5
    return max(1, int(10.0 / (per_pt * p.n ** p.dim)))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    p = workload(args)
    reps = oracle_reps_for(p)
    for _ in range(args.warmup):
        oracle_sample(p, 1)
    times = []
    rates = []
    for _ in range(args.steps):
        r, sec, meta = oracle_sample(p, reps)
        times.append(sec)
        rates.append(r)
    value = float(np.median(rates))
    meta["value"] = value
    meta["unit"] = UNIT
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.median(times)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(p, args.config, 1), "cpu_baseline": meta,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm -------
def run_prs(args):
    import torch
    import torch.distributed as dist

    import paper_2502_08370_b200 as prs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p = workload(args)
    uid = None
    if world > 1:
        obj = [prs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    stream = torch.cuda.current_stream()
    ctx = prs.Context(p, rank=rank, nranks=world, nccl_uid=uid, stream=stream.cuda_stream)
    if args.coarse_mode == "space":
        ctx.set_coarse_mode(1, world if world > 1 else args.gbands)
    if args.pipeline:
        ctx.set_pipeline(args.pipeline)
    u0 = synth.initial_state(p)
    u0_host = torch.from_numpy(u0).pin_memory()
    u0_dev = u0_host.cuda()
    ctx.set_initial(u0_dev)
    ctx.coarse_sweep()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        ctx.fine_sweep()
        return ctx.parareal_correct()

    if args.pipeline:  # K pipelined iterations per call (no stop test: tol = 0)
        ctx.iterate(max(1, min(args.warmup, p.N)), 0.0)
    else:
        for _ in range(args.warmup):
            step()
    barrier()
    # timed region: the production path (CUDA-graph replays on one rank), no per-kernel events
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.5)  # nvidia-smi running before the timed region starts
    l0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    upds = []
    if args.pipeline:
        assert args.steps <= p.N, "--pipeline: steps <= N (one prs_iterate call)"
        _, upds = ctx.iterate(args.steps, 0.0)
        # (an exactly zero update -- finite termination -- stops the call early: the rate
        # counts the iterations that ran)
    else:
        for _ in range(args.steps):
            upds.append(step())
    ev1.record(stream)
    torch.cuda.synchronize()
    t_end = time.perf_counter()
    launches = ctx.launches() - l0
    ms = ev0.elapsed_time(ev1)
    # a timed region shorter than the sampling period: keep the GPU on the same (untimed) steps
    # until three samples have arrived since the region started, and report those
    t_start = t_end - ms / 1e3
    extra = 0
    while clocks.proc is not None and clocks.count_since(t_start) < 3 and extra < 100000:
        if args.pipeline:
            ctx.iterate(1, 0.0)
        else:
            step()
        extra += 1
        if extra % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop(t_start, time.perf_counter())
    if extra:
        clk["window"] = (f"timed region {ms:.1f} ms < sampling period: samples over it and {extra} "
                         "untimed steps of the same work right after it")
    # per-kernel device times for the roofline: the same steps again with CUDA events around
    # every fine-sweep launch (direct launches; not part of the timed value)
    ctx.set_profiling(True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    stats = {k: ctx.kernel_stats(k) for k in (prs.PRS_K_XPASS, prs.PRS_K_LPASS, prs.PRS_K_DD, prs.PRS_K_IE)}
    ctx.set_profiling(False)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    total_updates = updates_per_step(p) * len(upds)
    value = total_updates / (ms / 1e3)

    # ---- end to end through the C ABI with host buffers (rank-local, then max) ----
    e2e = None
    if args.e2e_steps > 0:
        out_host = torch.empty_like(u0_host).pin_memory()
        last = ctx.first + ctx.count
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            ctx.set_initial(u0_host)          # H2D of the step's input from pinned host memory
            ctx.coarse_sweep()
            ctx.fine_sweep()
            ctx.parareal_correct()            # D2H of the update norm
            ctx.get_slice(last, out_host)     # D2H of the end state this rank owns
        barrier()
        sec = time.perf_counter() - t0
        st = torch.tensor([sec], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(st, op=dist.ReduceOp.MAX)
        sec = float(st.item())
        e2e = {"value": updates_per_step(p) * args.e2e_steps / sec, "unit": UNIT,
               "h2d_bytes_per_step": int(u0.nbytes) * world,
               "d2h_bytes_per_step": (int(u0.nbytes) + 16) * world,
               "includes": "set_initial(host) + coarse_sweep + fine_sweep + correct + get_slice(host)"}

    # ---- parareal time to tolerance (the metric's second part) and the sequential fine solve
    # it competes with (same kernels, N s steps on one state, one GPU: SURVEY.md 8(d)) ----
    ttt = None
    if not args.no_time_to_tol:
        tol = stop_tol(args.config)
        barrier()
        t0 = time.perf_counter()
        ev0.record(stream)
        ctx.set_initial(u0_dev)
        ctx.coarse_sweep()
        k, hist = ctx.iterate(p.N, tol)
        ev1.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([ev0.elapsed_time(ev1) / 1e3, time.perf_counter() - t0], dtype=torch.float64,
                          device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        seq = None
        if rank == 0:
            out_dev = torch.empty_like(u0_dev)
            torch.cuda.synchronize()
            s0 = time.perf_counter()
            ctx.fine_solve(u0_dev, out_dev)
            seq = time.perf_counter() - s0
        barrier()
        ttt = {"tol": tol, "stop": "max|U^{k+1}-U^k| / ||U_0||_inf <= tol or k = N (DESIGN.md R7)",
               "iterations": k, "N": p.N, "time_to_tol_s": float(tt[0].item()),
               "wall_s": float(tt[1].item()), "updates_last": hist[-1] if hist else None,
               "sequential_fine_s": seq,
               "speedup_vs_sequential_fine": (seq / float(tt[0].item())) if seq else None,
               "sequential_fine": "prs_fine_solve: N s fine steps of one state on rank 0's GPU"}

    # ---- roofline of the dominant kernel (live CUDA events around each launch) ----
    dom = max(stats, key=lambda k: stats[k][1])
    nl, kms, kwork = stats[dom]
    names = {prs.PRS_K_XPASS: "xpass_kernel (x-line solve + fused RHS)",
             prs.PRS_K_LPASS: "lpass_kernel (strided line solve + epilogue)",
             prs.PRS_K_DD: "dd_stage_kernel (DD strip-block stage)",
             prs.PRS_K_IE: "ie_axis_kernel (unsplit IE step: 2 dim sine transforms on DMMA)"}
    flop_kinds = (prs.PRS_K_DD, prs.PRS_K_IE)
    tr = ncu_traffic(args.config)
    per_launch_s = (kms / nl) / 1e3 if nl else float("nan")
    if dom in flop_kinds:
        # the block / sine transforms run on the fp64 tensor cores (DMMA m8n8k4); fp64 peak = 148 SMs x
        # 64 FP64 FMA/clk x 2 flop x 1.965 GHz = 37.2 TF/s, DMMA and DFMA alike (measured 37.1 /
        # 35.7 TF/s on this pool's B200, profiles/r01_fp64_peak_probe.txt)
        peak, peak_src, unit, bound = (148 * 64 * 2 * 1.965e9 / 1e12,
                                       "derived: 148 SM x 64 fp64 FMA/clk x 1.965 GHz (DMMA measured 37.1 TF/s)",
                                       "TFLOP/s", "tensor")
        achieved = (kwork / nl) / per_launch_s / 1e12 if nl else 0.0
    else:
        peak, peak_src = measured_peaks()
        unit, bound = "GB/s", "hbm"
        achieved = (kwork / nl) / per_launch_s / 1e9 if nl else 0.0

    def rate(v):
        if not v[0]:
            return None
        r = (v[2] / v[0]) / ((v[1] / v[0]) / 1e3)
        return r / 1e12 if any(v is stats.get(k) for k in flop_kinds) else r / 1e9
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "traffic": (tr or {}).get(names[dom].split()[0]),
            "kernel": names[dom], "peak_source": peak_src,
            "algorithmic_work_per_launch": kwork / nl if nl else None,
            "avg_launch_ms": kms / nl if nl else None,
            "share_of_step": kms / ms if ms else None,
            "other_kernels": {names[k]: {"launches": v[0], "ms": v[1],
                                         ("TFLOPs" if k in flop_kinds else "GBps"): rate(v)}
                              for k, v in stats.items() if v[0]}}
    cpu = None
    ie_big = (p.G == 2 or p.F == 2) and p.n > 300
    if rank == 0 and world == 1 and not args.no_cpu_baseline and ie_big:
        # the oracle's IE step is a band elimination of the whole n^2 system, O(n^4) per step
        # (~10^12 flops, minutes, at n = 999): no bounded sample of this workload exists
        cpu = {"kind": "oracle", "skipped": "oracle IE step is O(n^4) band elimination: one step of "
               f"n = {p.n} exceeds the bounded-sample budget", "cores": 0, "value": None}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        reps = oracle_reps_for(p)
        v, sec, meta = oracle_sample(p, reps)
        meta.update({"value": v, "unit": UNIT, "seconds": sec})
        va, seca, th = oracle_sample_all_cores(p, max(1, reps // 2))
        meta["all_cores"] = {"value": va, "unit": UNIT, "cores": th, "seconds": seca,
                             "sample": f"{max(1, reps // 2)} fine step(s) of one slice per core, {th} cores"}
        cpu = meta
        if ttt is not None:
            ttt["oracle_extrapolated"] = oracle_ttt_extrapolated(p, ttt["iterations"], v, va, th)
    ctx.close()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": workload_config(p, args.config, world),
                "parallelism": f"time-slices x{world}",
                "coarse_mode": args.coarse_mode, "pipeline_blocks": args.pipeline,
                "updates": upds, "gpu_launches": launches, "clocks": clk, "roofline": roof,
                "cpu_baseline": cpu, "e2e": e2e, "time_to_tol": ttt}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_prs(args)


if __name__ == "__main__":
    sys.exit(main())
