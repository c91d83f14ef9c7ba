python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_l8w0.json 2> gpurun_out/bench_c3_l8w0.err; echo "bench rc=$?"
PRS_L8WIDE=1 python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_l8w1.json 2> gpurun_out/bench_c3_l8w1.err; echo "bench rc=$?"
PRS_L8WIDE=1 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or full_size or lpass or long or tiled" > gpurun_out/pytest_l8w.log 2>&1; echo "pytest rc=$?"
