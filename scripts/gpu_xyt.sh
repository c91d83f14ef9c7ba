PRS_XY=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c2 or xy or 128" > gpurun_out/pytest_xyt.log 2>&1; echo "pytest rc=$?"
PRS_XY=2 timeout 300 python bench.py --config c2 --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c2_xyt.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c2_xy1.json 2>> gpurun_out/bench_c2.err; echo "bench rc=$?"
