timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dd or c4 or DD" > gpurun_out/pytest_ddgx.log 2>&1; echo "pytest rc=$?"
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c4_v20.json 2> gpurun_out/bench_c4_gx2.err; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dd_stage --launch-skip 64 -c 1 -o gpurun_out/dd_v20 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-time-to-tol > gpurun_out/ncu_dd.log 2>&1; echo "ncu rc=$?"
