# diagnostic: rebuild the (disposable, box-side) library with -DPRS_DD_TIMING and run c4
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr -DPRS_DD_TIMING -o paper_2502_08370_b200/libprs.so paper_2502_08370_b200/csrc/prs_api.cu -ldl; echo "build rc=$?"
touch paper_2502_08370_b200/libprs.so
timeout 300 python bench.py --config c4 --steps 3 --warmup 1 --no-cpu-baseline --no-time-to-tol --e2e-steps 0 > gpurun_out/bench_c4_timing.json 2> gpurun_out/bench_c4_timing.err; echo "bench rc=$?"
