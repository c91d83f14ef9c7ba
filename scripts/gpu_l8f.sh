python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or n2048 or fused" > gpurun_out/pytest_l8f.log 2>&1; echo "pytest rc=$?"
python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_l8f.json 2> gpurun_out/bench_c3_l8f.err; echo "bench rc=$?"
