#!/bin/bash
# Export an ncu report to small CSVs next to it and delete the report (gpurun_out <= 64 MiB).
#   scripts/ncu_export.sh gpurun_out/prof_x7
r=$1
ncu -i $r.ncu-rep --page details --csv > ${r}_details.csv 2>/dev/null
ncu -i $r.ncu-rep --page raw --csv > ${r}_raw.csv 2>/dev/null
ncu -i $r.ncu-rep --page source --csv --print-source=cuda,sass > ${r}_source.csv 2>/dev/null
rm -f $r.ncu-rep
