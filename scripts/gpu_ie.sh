#!/bin/bash
# IE / section-5.1 (NEXT-4) round trip: GPU parity tests ($T, default the IE file + the whole
# -m gpu suite when FULL=1), the c6 bench line, one ncu --set full capture of an ie_axis_kernel
# fine-sweep launch (summary in gpurun_out/sum_ie.txt).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ie.py -q -x -p no:cacheprovider -rs > gpurun_out/pytest_ie.log 2>&1; echo "pytest ie rc=$?"
tail -3 gpurun_out/pytest_ie.log
if [ -n "$FULL" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest all rc=$?"
  tail -3 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --config c6 ${BARGS} > gpurun_out/bench_c6.json 2> gpurun_out/bench_c6.err; echo "bench c6 rc=$?"
for c in $CFGS; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
if [ -z "$NONCU" ]; then
  ncu --set full --import-source on --clock-control none -k "regex:ie_axis" --launch-skip 85 -c 1 -o gpurun_out/prof_ie \
      python scripts/prof_step.py --config c6 --sweeps 1 > gpurun_out/ncu_ie.log 2>&1; echo "ncu rc=$?"
  bash scripts/ncu_export.sh gpurun_out/prof_ie
  python scripts/ncu_summary.py gpurun_out/prof_ie > gpurun_out/sum_ie.txt
  rm -f gpurun_out/prof_ie_source.csv gpurun_out/prof_ie_raw.csv
fi
