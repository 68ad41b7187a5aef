cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/abi_sweep.py paper_1804_07981_b200/libbml_dev.so --n 128 256 512 1024 --blocks 16 8 4 --strips 0 --steps 4096 > gpurun_out/sweep_pack.jsonl 2>&1
