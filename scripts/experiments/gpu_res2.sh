cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "resident or golden or simulate" -p no:cacheprovider > gpurun_out/pytest_resident.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_resident.txt
timeout 300 python scripts/sweep_resident.py > gpurun_out/sweep_resident2.jsonl 2> gpurun_out/sweep_resident2.err
