python -m pytest tests/test_gpu_parity.py -x -q -k "n2048 or c3 or full_size or fused" > gpurun_out/pytest_l8.log 2>&1; echo "pytest rc=$?"
python bench.py --no-cpu-baseline --no-time-to-tol --steps 2 > gpurun_out/bench_c3_l8.json 2> gpurun_out/bench_c3_l8.err; echo "bench rc=$?"
PRS_L8=0 python bench.py --no-cpu-baseline --no-time-to-tol --steps 2 > gpurun_out/bench_c3_l5.json 2> gpurun_out/bench_c3_l5.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lp8|lp5|xpass" --launch-skip 256 -c 8 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-time-to-tol > gpurun_out/ncu_l8.csv 2> gpurun_out/ncu_l8.err; echo "ncu rc=$?"
