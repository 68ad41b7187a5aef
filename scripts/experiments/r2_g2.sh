# round 2: census tests first, then the whole GPU suite (incl. slow multi-rank sweeps)
timeout 600 python -m pytest tests/test_gpu_census.py tests/test_gpu_verify.py -x -q 2>&1 | tail -15 > gpurun_out/r2_census.log
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r2_pytest_gpu.log
