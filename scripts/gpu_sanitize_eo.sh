# compute-sanitizer over the even/odd-layout kernel paths (round 2): the layout
# conversion kernels and step_wide_kernel<..., EO> on single bands (oracle sizes,
# torus-seam windows, narrow tails, short calls) -- memcheck, racecheck, synccheck.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='test_eo_matches_oracle and (2048 or 2112) or test_eo_short_runs or test_eo_falls_back'
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_eo.py -x -q -k "$SEL" \
    > gpurun_out/sanitize_eo_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_eo_$tool.log
  tail -3 gpurun_out/sanitize_eo_$tool.log
done
