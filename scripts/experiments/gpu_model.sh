cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
L=paper_1804_07981_b200/libbml_dev.so
timeout 300 python scripts/abi_sweep.py $L --n 8192 --blocks 16 --strips 0 63 64 100 128 > gpurun_out/sweep_model_8192.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 16384 --blocks 16 --strips 0 253 256 330 > gpurun_out/sweep_model_16384.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 32768 --blocks 16 --strips 0 656 863 993 1024 > gpurun_out/sweep_model_32768.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 65536 --blocks 16 --strips 0 1286 2622 3856 --steps 320 --reps 2 > gpurun_out/sweep_model_65536.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 2048 4096 --blocks 8 16 --strips 0 > gpurun_out/sweep_model_small.jsonl 2>&1
