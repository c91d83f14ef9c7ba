#!/usr/bin/env python
"""Count the SASS instructions that prove the tensor / async-copy / barrier paths of the hot
kernels (cuobjdump -sass of the built libprs.so): DMMA (fp64 tensor core), UTMALDG / UTMASTG
(TMA tensor load / store), UBLKCP (bulk copy), LDGSTS (cp.async), SYNCS (mbarrier), STAS
(st.async into a cluster peer), DFMA.

    python scripts/sass_evidence.py > profiles/r02_sass_evidence.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2502_08370_b200", "libprs.so")
KERNELS = ["xpass7_kernelILi1ELi1ELi0ELi1E", "xpass7_kernelILi1ELi0ELi0ELi1E", "lp8_kernelILi1ELi0ELi1ELi1E",
           "lp8_kernelILi1ELi1ELi1ELi1E", "dd_pass_kernelILi0ELi1ELi1E", "dd_pass_kernelILi0ELi1ELi2E",
           "dd_scan_kernel", "df_stage_kernelILi0ELi1E", "xy3_kernelILi1E", "sweep2_kernelILi256ELi1ELi0ELi0ELi0E",
           "lpass3_kernel"]
PAT = re.compile(r"\b(DMMA\.[0-9A-Z.]+|UTMALDG[0-9A-Z.]*|UTMASTG[0-9A-Z.]*|UBLKCP[0-9A-Z.]*|LDGSTS[0-9A-Z.]*|"
                 r"SYNCS\.[0-9A-Z.]+|STAS[0-9A-Z.]*|DFMA|DMUL|DADD|BAR\.SYNC[0-9A-Z.]*|UCGABAR_[A-Z]+)")


def main():
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
    counts, cur = collections.defaultdict(collections.Counter), None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        if cur:
            for mm in PAT.findall(line):
                counts[cur][mm] += 1
    print(f"# static SASS instruction counts per kernel, cuobjdump -sass {os.path.relpath(SO, ROOT)}")
    for k in KERNELS:
        for f, c in sorted(counts.items()):
            if k in f:
                print(f)
                print("    " + ", ".join(f"{n} {v}" for n, v in sorted(c.items())))
                break


if __name__ == "__main__":
    sys.exit(main())
