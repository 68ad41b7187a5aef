cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "resident" -p no:cacheprovider > gpurun_out/pytest_resident.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_resident.txt
timeout 300 python scripts/sweep_resident.py > gpurun_out/sweep_resident.jsonl 2> gpurun_out/sweep_resident.err
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.txt
