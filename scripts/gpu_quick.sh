#!/bin/bash
# Quick GPU iteration: optional x7 phase timing (libprs_x7t.so), a c3-shape parity subset ($K),
# and short bench lines of $CFGS without the CPU baseline / time to tolerance.
mkdir -p gpurun_out
if [ -f paper_2502_08370_b200/libprs_x7t.so ] && [ -z "$NOTIME" ]; then
  cp paper_2502_08370_b200/libprs.so /tmp/libprs_keep.so
  cp paper_2502_08370_b200/libprs_x7t.so paper_2502_08370_b200/libprs.so
  python scripts/prof_step.py --config c3 --sweeps 1 2>&1 | grep x7
  cp /tmp/libprs_keep.so paper_2502_08370_b200/libprs.so
fi
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$K" -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
fi
for c in ${CFGS:-c3}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-time-to-tol $BARGS > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err; echo "bench $c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/q_$c.json')); r=d['roofline']
print('$c', '%.4g'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'dom %.3f ms'%r['avg_launch_ms'], d['clocks']['sm_mhz'], {k:round(v['ms']/v['launches'],4) for k,v in r.get('other_kernels',{}).items()})"
done
