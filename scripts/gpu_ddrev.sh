PRS_DDREV=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dd or c4 or DD" > gpurun_out/pytest_ddrev.log 2>&1; echo "pytest rc=$?"
PRS_DDREV=1 timeout 300 python bench.py --config c4 --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c4_rev1.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c4_rev0.json 2>> gpurun_out/bench_c4.err; echo "bench rc=$?"
