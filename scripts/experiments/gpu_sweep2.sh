cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1804_07981_b200/libbml_dev.so
timeout 600 python scripts/abi_sweep.py $L --n 32768 --blocks 16 --strips 256 328 400 512 600 655 700 800 1000 > gpurun_out/sweep_strips_32768.jsonl 2>&1
timeout 600 python scripts/abi_sweep.py $L --n 8192 --blocks 8 16 --strips 16 24 32 41 48 64 96 128 > gpurun_out/sweep_strips_8192.jsonl 2>&1
timeout 600 python scripts/abi_sweep.py $L --n 16384 --blocks 16 --strips 64 128 164 200 256 328 > gpurun_out/sweep_strips_16384.jsonl 2>&1
