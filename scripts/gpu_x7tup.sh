PRS_X7TUP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or full_size or 4096" > gpurun_out/pytest_x7tup.log 2>&1; echo "pytest rc=$?"
PRS_X7TUP=1 timeout 300 python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_tup1.json 2> gpurun_out/bench_c3_tup.err; echo "bench rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_tup0.json 2>> gpurun_out/bench_c3_tup.err; echo "bench rc=$?"
