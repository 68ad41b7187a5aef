cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python scripts/abi_sweep.py paper_1804_07981_b200/libbml_dev.so build_variants/libbml_dev_fma.so --n 8192 32768 --blocks 8 16 --strips 0 64 128 256 512 > gpurun_out/abi_sweep_v3.jsonl 2> gpurun_out/abi_sweep_v3.err
