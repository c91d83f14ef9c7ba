#!/bin/bash
# Bench lines of every config (default settings, clocks sampled in each), for profiles/.
mkdir -p gpurun_out
for c in ${CFGS:-c0 c1 c1p c2 c3 c4 c5}; do
  timeout 1200 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
