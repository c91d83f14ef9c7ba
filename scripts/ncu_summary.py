#!/usr/bin/env python
"""Summarise the CSV exports of one ncu --set full capture (scripts/ncu_export.sh): speed of
light, occupancy, scheduler, warp-stall breakdown and the source lines with most stall samples.

    python scripts/ncu_summary.py gpurun_out/prof_x7f > profiles/r02_ncu_x7_fine_summary.txt
"""
import csv
import sys

WANT = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Theoretical Occupancy",
        "Achieved Active Warps Per SM", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "SM Frequency", "Compute (SM) Throughput")


def main(prefix, top=25):
    det = list(csv.reader(open(prefix + "_details.csv")))
    hdr = det[0]
    name = None
    print(f"# ncu --set full summary: {prefix}")
    for row in det[1:]:
        d = dict(zip(hdr, row))
        name = d.get("Kernel Name", name)
        if d.get("Metric Name") in WANT:
            print(f"{d['Section Name'][:28]:28s} | {d['Metric Name']:36s} | {d['Metric Value']} {d['Metric Unit']}")
    print(f"kernel: {name}")
    raw = list(csv.reader(open(prefix + "_raw.csv")))
    hdr, vals = raw[0], raw[2]
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"):
        if key in hdr:
            print(f"{key} = {vals[hdr.index(key)]} {raw[1][hdr.index(key)]}")
    items = [(h, float(v or 0)) for h, v in zip(hdr, vals)
             if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued")]
    tot = sum(v for _, v in items) or 1.0
    print("\nwarp stall samples:")
    for h, v in sorted(items, key=lambda x: -x[1])[:10]:
        print(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {100 * v / tot:5.1f} %")
    rows = list(csv.reader(open(prefix + "_source.csv")))
    cur, out = None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif len(r) > 6 and r[0].isdigit():
            out.append((int(r[4]) if r[4].isdigit() else 0, cur, int(r[0]), r[1].strip()[:90]))
    tot = sum(o[0] for o in out) or 1
    print("\nsource lines with most stall samples:")
    for smp, f, ln, src in sorted(out, reverse=True)[:top]:
        print(f"  {100 * smp / tot:5.1f} %  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1])
