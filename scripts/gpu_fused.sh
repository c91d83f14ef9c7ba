set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "fused or n1024 or n2048 or c3 or full_size" > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?"
PRS_FUSED=2 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or c3_full" > gpurun_out/pytest_fused2.log 2>&1; echo "pytest2 rc=$?"
python bench.py --no-cpu-baseline --steps 2 > gpurun_out/bench_c3_f1.json 2> gpurun_out/bench_c3_f1.err; echo "bench rc=$?"
PRS_FUSED=2 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/bench_c3_f2.json 2> gpurun_out/bench_c3_f2.err; echo "bench rc=$?"
ncu --set full --clock-control none --import-source on -k regex:xpass6 --launch-skip 64 -c 1 -o gpurun_out/x6_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_x6.log 2>&1; echo "ncu rc=$?"
