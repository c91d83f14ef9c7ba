python -m pytest tests/test_gpu_parity.py -x -q -k "on_chip or c1 or c0 or graph or fine_solve or skipping or space_parallel or iterate or n64 or n128 or n256" > gpurun_out/pytest_chain2.log 2>&1; echo "pytest rc=$?"
for c in c0 c1 c1p; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_ch2.json 2> gpurun_out/bench_${c}_ch2.err; echo "$c rc=$?"; done
