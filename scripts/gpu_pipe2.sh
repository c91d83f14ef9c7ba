timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "pipeline or pipelined" > gpurun_out/pytest_pipe2.log 2>&1; echo "pytest rc=$?"
for g in 0 4 8; do timeout 600 python bench.py --config c2 --steps 8 --no-cpu-baseline --e2e-steps 0 --pipeline $g > gpurun_out/bench_c2_pipe$g.json 2> gpurun_out/bench_pipe2.err; echo "bench c2 $g rc=$?"; done
