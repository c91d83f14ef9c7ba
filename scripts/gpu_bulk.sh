python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_tma.json 2> gpurun_out/bench_c3_bulk.err; echo "bench rc=$?"
PRS_X3TMA=0 python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_notma.json 2> gpurun_out/bench_c3_nobulk.err; echo "bench rc=$?"
