# compute-sanitizer memcheck over the pitch-specialised even/odd kernel at N=32768
# (immediate row offsets, zero pad rows past the band end, 16-byte stores).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --error-exitcode 9 python scripts/eo_memcheck_big.py > gpurun_out/sanitize_eo_big_memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_eo_big_memcheck.log
tail -4 gpurun_out/sanitize_eo_big_memcheck.log
timeout 1500 bash scripts/gpu_sanitize_eo.sh
