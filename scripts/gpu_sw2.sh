timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep2 or c1 or c0 or chain or fine_solve or graph or skip or space" > gpurun_out/pytest_sw2.log 2>&1; echo "pytest rc=$?"
for c in c1 c1p c0; do timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${c}_msg.json 2> gpurun_out/bench_sw2.err; echo "bench $c rc=$?"; done
