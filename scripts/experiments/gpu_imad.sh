cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
L=paper_1804_07981_b200/libbml_dev.so
V=build_variants/libbml_dev_imad.so
timeout 900 python scripts/abi_sweep.py $L $V --n 4096 8192 16384 32768 --blocks 16 --strips 0 64 128 256 > gpurun_out/sweep_imad.jsonl 2>&1
timeout 900 python scripts/abi_sweep.py $L $V --n 32768 --blocks 16 --strips 512 655 863 > gpurun_out/sweep_imad2.jsonl 2>&1
timeout 600 python scripts/abi_sweep.py $L $V --n 65536 --blocks 16 --strips 0 --steps 320 --reps 2 > gpurun_out/sweep_imad3.jsonl 2>&1
