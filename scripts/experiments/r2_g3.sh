timeout 900 python scripts/sweep_wide.py > gpurun_out/r2_sweep_wide.jsonl 2> gpurun_out/r2_sweep_wide.err
timeout 900 python -m pytest tests/test_gpu_census.py tests/test_gpu_verify.py tests/test_reference_unit_tests.py -x -q 2>&1 | tail -15 > gpurun_out/r2_census2.log
