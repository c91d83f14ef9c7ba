#!/bin/bash
# ncu --set full of the DD split-stage kernels of one c4 fine step (summaries in gpurun_out/).
mkdir -p gpurun_out
i=0
for k in "dd_pass_kernel" "dd_pass_kernel" "dd_pp_kernel"; do
  i=$((i+1)); pp=1; case "$k" in dd_pass*) pp=0;; esac
  PRS_DDPP=$pp ncu --set full --import-source on --clock-control none -k "regex:${k%%<*}" --launch-skip $((140 + i)) -c 1 -o gpurun_out/prof_dd$i python scripts/prof_step.py --config c4 --sweeps 1 > /dev/null 2>&1
  bash scripts/ncu_export.sh gpurun_out/prof_dd$i
  python scripts/ncu_summary.py gpurun_out/prof_dd$i > gpurun_out/sum_dd$i.txt
  rm -f gpurun_out/prof_dd${i}_source.csv gpurun_out/prof_dd${i}_raw.csv
done
