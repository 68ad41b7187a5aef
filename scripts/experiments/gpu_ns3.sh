cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1804_07981_b200/libbml_dev.so
timeout 300 python scripts/abi_sweep.py $L --n 8192 --blocks 16 --strips 0 -64 -65 -66 -68 -72 -80 -98 -128 > gpurun_out/sweep_ns3_8192.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 16384 --blocks 16 --strips 0 -64 -65 -66 -70 -80 -98 -128 > gpurun_out/sweep_ns3_16384.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 32768 --blocks 16 --strips 0 -33 -50 -66 > gpurun_out/sweep_ns3_32768.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L build_variants/libbml_dev_skip.so build_variants/libbml_dev_noimad.so --n 1024 512 256 --blocks 16 8 --strips 0 --steps 4096 > gpurun_out/sweep_res_var.jsonl 2>&1
