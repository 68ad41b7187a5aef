cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "test_resident_kernel_matches and (64 or 256)" > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 900 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "test_resident_kernel_matches and (64 or 256) or test_random_lattice_steps_match_oracle and (37 or 96)" > gpurun_out/sanitize_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck.log
