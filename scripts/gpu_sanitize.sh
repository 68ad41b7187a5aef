cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
K="test_random_lattice_steps_match_oracle and (37 or 64 or 96 or 1025) or test_block_and_strip or test_simulate_metrics or test_row_bands_match or test_resident_kernel_matches or test_explicit_strip or test_single_phase"
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_init.py tests/test_gpu_digest.py tests/test_snapshot.py -x -q -k "small or matches_host or band or ppm or rejection" > gpurun_out/sanitize_memcheck2.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck2.log
