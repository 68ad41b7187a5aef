cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
L="paper_1804_07981_b200/libbml_dev.so build_variants/libbml_dev_v1.so"
timeout 300 python scripts/abi_sweep.py $L --n 8192 16384 32768 --blocks 16 --strips 0 > gpurun_out/sweep_v2.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 65536 --blocks 16 --strips 0 --steps 320 --reps 2 >> gpurun_out/sweep_v2.jsonl 2>&1
