timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pipeline or pipelined" > gpurun_out/pytest_pipe.log 2>&1; echo "pytest rc=$?"
for c in c1p c1 c0; do for g in 0 2 4 8; do timeout 300 python bench.py --config $c --steps 8 --no-cpu-baseline --e2e-steps 0 --pipeline $g > gpurun_out/bench_${c}_pipe$g.json 2> gpurun_out/bench_pipe.err; echo "bench $c $g rc=$?"; done; done
