#!/bin/bash
# ncu --set full of the DD split-stage pass kernels (p1, p2) of one c4 fine step (summaries in gpurun_out/).
mkdir -p gpurun_out
for i in 1 2; do
  ncu --set full --import-source on --clock-control none -k "regex:dd_pass_kernel" --launch-skip $((140 + i)) -c 1 -o gpurun_out/prof_dd$i python scripts/prof_step.py --config c4 --sweeps 1 > /dev/null 2>&1
  bash scripts/ncu_export.sh gpurun_out/prof_dd$i
  python scripts/ncu_summary.py gpurun_out/prof_dd$i > gpurun_out/sum_dd$i.txt
  rm -f gpurun_out/prof_dd${i}_source.csv gpurun_out/prof_dd${i}_raw.csv
done
