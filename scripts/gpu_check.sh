#!/bin/bash
# GPU check: pytest -m gpu (optional -k filter in $K), smoke, one bench line (config $CFG).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x ${K:+-k "$K"} -p no:cacheprovider -rs --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for c in ${CFGS:-c3}; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
tail -3 gpurun_out/pytest_gpu.log
