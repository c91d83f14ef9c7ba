python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or tma_ring or full_size" > gpurun_out/pytest_x7.log 2>&1; echo "pytest rc=$?"
python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_x7.json 2> gpurun_out/bench_c3_x7.err; echo "bench rc=$?"
PRS_X7=0 python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_nox7.json 2> gpurun_out/bench_c3_nox7.err; echo "bench rc=$?"
