python scripts/experiments/r2_mc_ab2.py . > gpurun_out/r2_mc_ab3.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_census.py tests/test_gpu_async.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/r2_tests_new.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_wide.py tests/test_gpu_census.py tests/test_gpu_async.py -x -q > gpurun_out/r2_sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitize_memcheck.log
timeout 1200 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_wide.py tests/test_gpu_census.py -x -q -k "not row_bands" > gpurun_out/r2_sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitize_racecheck.log
timeout 1200 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_wide.py tests/test_gpu_census.py -x -q -k "not row_bands" > gpurun_out/r2_sanitize_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitize_synccheck.log
