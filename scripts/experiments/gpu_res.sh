cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
L="paper_1804_07981_b200/libbml_dev.so build_variants/libbml_dev_nosplit.so"
timeout 300 python scripts/abi_sweep.py $L --n 1024 512 256 --blocks 16 8 4 --strips 0 --steps 4096 > gpurun_out/sweep_res_p2p.jsonl 2>&1
