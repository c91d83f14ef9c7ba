mkdir -p gpurun_out
cap() {
  ncu --set full --import-source on --clock-control none -k "regex:$3" --launch-skip $4 -c 1 -o gpurun_out/prof_$1 \
      python scripts/prof_step.py --config $2 --sweeps 1 > /dev/null 2>&1
  bash scripts/ncu_export.sh gpurun_out/prof_$1
  python scripts/ncu_summary.py gpurun_out/prof_$1 > gpurun_out/sum_$1.txt
  rm -f gpurun_out/prof_$1_source.csv gpurun_out/prof_$1_raw.csv
}
cap xy3 c2 xy3_kernel 70
