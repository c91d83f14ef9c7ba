#!/bin/bash
# Round-end profiles: the c3 bench launch list (ncu gpu__time_duration per launch, clocks unlocked)
# and one ncu --set full capture per dominant kernel (scripts/ncu_round.sh).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-time-to-tol > gpurun_out/launches_c3.log 2>&1
echo "launch list rc=$?"
bash scripts/ncu_round.sh
ls gpurun_out
