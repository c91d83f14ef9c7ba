python -m pytest tests/test_gpu_parity.py -x -q -k "dd or split or c4 or S8 or fine_solve" > gpurun_out/pytest_dd.log 2>&1; echo "pytest rc=$?"
python bench.py --config c4 --no-cpu-baseline --no-time-to-tol > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
