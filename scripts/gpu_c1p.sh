python -m pytest tests/test_gpu_parity.py -x -q -k "paper_pairing" > gpurun_out/pytest_c1p.log 2>&1; echo "pytest rc=$?"
python bench.py --config c1p --no-cpu-baseline > gpurun_out/bench_c1p.json 2> gpurun_out/bench_c1p.err; echo "bench rc=$?"
