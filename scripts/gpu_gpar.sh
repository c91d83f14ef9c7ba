python -m pytest tests/test_gpu_parity.py -x -q -k "space_parallel" > gpurun_out/pytest_gpar.log 2>&1; echo "pytest rc=$?"
