timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c2 or xy or 128 or sweep2 or c1 or c0" > gpurun_out/pytest_xy.log 2>&1; echo "pytest rc=$?"
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c2_st.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
for c in c1p c0; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_${c}_rlx.json 2>> gpurun_out/bench_c2.err; echo "bench rc=$?"; done
