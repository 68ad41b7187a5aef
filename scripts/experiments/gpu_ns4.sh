cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
L=paper_1804_07981_b200/libbml_dev.so
timeout 300 python scripts/abi_sweep.py $L --n 8192 --blocks 16 --strips 0 -64 -65 -66 -72 -98 -128 > gpurun_out/sweep_ns4_8192.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 16384 --blocks 16 --strips 0 -64 -65 -66 -80 -98 -128 > gpurun_out/sweep_ns4_16384.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 32768 --blocks 16 --strips 0 -33 -50 -66 > gpurun_out/sweep_ns4_32768.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 65536 --blocks 16 --strips 0 -25 -51 --steps 320 --reps 2 > gpurun_out/sweep_ns4_65536.jsonl 2>&1
