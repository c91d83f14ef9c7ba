#!/bin/bash
# One GPU round trip: optional diagnostics ($DIAG), pytest -m gpu (optional -k $K), quick bench lines of $CFGS.
mkdir -p gpurun_out
for d in $DIAG; do timeout 900 python $d > gpurun_out/$(basename $d .py).log 2>&1; echo "diag $d rc=$?"; done
if [ -z "$NOTEST" ]; then
  timeout 3000 python -m pytest tests -m gpu -q -x ${K:+-k "$K"} -p no:cacheprovider -rs -s --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_gpu.log
fi
for c in $CFGS; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-time-to-tol $BARGS > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err; echo "bench $c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/q_$c.json')); r=d['roofline']
print('$c', '%.4g'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'dom %.3f ms'%r['avg_launch_ms'], d['clocks']['sm_mhz'], {k:round(v['ms']/v['launches'],4) for k,v in r.get('other_kernels',{}).items()})"
done
