python -m pytest tests/test_gpu_parity.py -x -q -k "skipping or iterate or graph" > gpurun_out/pytest_skip.log 2>&1; echo "pytest rc=$?"
for c in c2 c4; do python bench.py --config $c --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${c}_skip.json 2> gpurun_out/bench_${c}_skip.err; echo "$c rc=$?"; done
python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_skip.json 2> gpurun_out/bench_c3_skip.err; echo "c3 rc=$?"
