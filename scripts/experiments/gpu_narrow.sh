cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
L=paper_1804_07981_b200/libbml_dev.so
timeout 300 python scripts/abi_sweep.py $L --n 2048 4096 8192 16384 32768 --blocks 16 --strips 0 > gpurun_out/sweep_narrow.jsonl 2>&1
