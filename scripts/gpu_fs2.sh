python -m pytest tests/test_gpu_parity.py -x -q -k "fine_solve or on_chip" > gpurun_out/pytest_fs2.log 2>&1; echo "pytest rc=$?"
for c in c0 c1p; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_fs2.json 2> gpurun_out/bench_${c}_fs2.err; echo "$c rc=$?"; done
