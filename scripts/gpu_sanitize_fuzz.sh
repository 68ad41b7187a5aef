# compute-sanitizer memcheck / racecheck / synccheck over the seeded random
# configurations (tests/test_gpu_fuzz.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
    timeout 1500 $CS --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_fuzz.py -q -m gpu \
        > gpurun_out/sanitize_${tool}_fuzz.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_${tool}_fuzz.log
    tail -3 gpurun_out/sanitize_${tool}_fuzz.log
done
