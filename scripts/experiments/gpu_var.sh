cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_digest.py -x -q > gpurun_out/pytest_digest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_digest.log
L="paper_1804_07981_b200/libbml_dev.so build_variants/libbml_dev_r8p1.so build_variants/libbml_dev_r8p0.so build_variants/libbml_dev_r6p0.so"
timeout 300 python scripts/abi_sweep.py $L --n 8192 --blocks 16 --strips -64 -128 -131 > gpurun_out/sweep_var_8192.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 16384 --blocks 16 --strips -64 -98 > gpurun_out/sweep_var_16384.jsonl 2>&1
timeout 400 python scripts/abi_sweep.py $L --n 32768 --blocks 16 --strips -50 > gpurun_out/sweep_var_32768.jsonl 2>&1
timeout 400 python scripts/abi_sweep.py $L --n 65536 --blocks 16 --strips -25 --steps 320 --reps 2 > gpurun_out/sweep_var_65536.jsonl 2>&1
