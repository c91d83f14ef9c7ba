#!/bin/bash
# One ncu --set full capture per dominant kernel of c3 / c4 / c5 (a fine-sweep launch each), summarised
# into gpurun_out/sum_<tag>.txt (profiles/ keeps the summaries).
mkdir -p gpurun_out
cap() {  # tag config kernel-regex skip
  ncu --set full --import-source on --clock-control none -k "regex:$3" --launch-skip $4 -c 1 -o gpurun_out/prof_$1 \
      python scripts/prof_step.py --config $2 --sweeps 1 > /dev/null 2>&1
  bash scripts/ncu_export.sh gpurun_out/prof_$1
  python scripts/ncu_summary.py gpurun_out/prof_$1 > gpurun_out/sum_$1.txt
  rm -f gpurun_out/prof_$1_source.csv gpurun_out/prof_$1_raw.csv
}
cap x7tma c3 xpass7 70
cap lp8t c3 "lp8_kernel" 300
cap lp8f c3 "lp8_kernel" 301
cap ddp1 c4 "dd_pass_kernel" 140
cap ddp2 c4 "dd_pass_kernel" 141
cap dfpf c5 "dfp_fwd" 400
cap dfpb c5 "dfp_bwd" 401
