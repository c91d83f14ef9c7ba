python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or full_size or n2048 or fused" > gpurun_out/pytest_x3r.log 2>&1; echo "pytest rc=$?"
python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_x3r.json 2> gpurun_out/bench_c3_x3r.err; echo "bench rc=$?"
PRS_X3CONTIG=1 python bench.py --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c3_x3c.json 2> gpurun_out/bench_c3_x3c.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"xpass3" --launch-skip 64 -c 2 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-time-to-tol > gpurun_out/ncu_x3r.csv 2> gpurun_out/ncu_x3r.err; echo "ncu rc=$?"
