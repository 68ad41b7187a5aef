cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/probe/warp_slots > gpurun_out/warp_slots.txt 2>&1
L="paper_1804_07981_b200/libbml_dev.so build_variants/libbml_dev_rpw3.so build_variants/libbml_dev_rpw6.so build_variants/libbml_dev_rpw8.so"
timeout 300 python scripts/abi_sweep.py $L --n 1024 512 --blocks 16 8 --strips 0 --steps 4096 > gpurun_out/sweep_rpw.jsonl 2>&1
