cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
L=paper_1804_07981_b200/libbml_dev.so
timeout 300 python scripts/abi_sweep.py $L --n 8192 --blocks 16 --strips 0 -64 -65 -128 -130 -131 -132 > gpurun_out/sweep_ns_8192.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 16384 --blocks 16 --strips 0 -33 -64 -65 -66 > gpurun_out/sweep_ns_16384.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 32768 --blocks 16 --strips 0 -33 -50 > gpurun_out/sweep_ns_32768.jsonl 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:step_block -s 6 -c 1 -o gpurun_out/prof_32768 -f python scripts/abi_sweep.py $L --n 32768 --blocks 16 --strips 0 --steps 64 --reps 1 > gpurun_out/prof_32768.log 2>&1
