#!/bin/bash
# ncu --set full of one partitioned full-tensor sweep kernel of a c5 fine step (summary in gpurun_out/).
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k "regex:${K:-dfp_fwd}" --launch-skip ${SKIP:-400} -c 1 -o gpurun_out/prof_dfp python scripts/prof_step.py --config c5 --sweeps 1 > /dev/null 2>&1
bash scripts/ncu_export.sh gpurun_out/prof_dfp
python scripts/ncu_summary.py gpurun_out/prof_dfp > gpurun_out/sum_dfp.txt
rm -f gpurun_out/prof_dfp_source.csv gpurun_out/prof_dfp_raw.csv
