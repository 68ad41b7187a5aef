timeout 900 python -m pytest tests/test_gpu_wide.py -x -q 2>&1 | tail -5 > gpurun_out/r2_split_tests.log
timeout 900 python scripts/sweep_wide.py --n 65536 32768 16384 8192 --variants 1 5 --check 1000 > gpurun_out/r2_sweep_split.jsonl 2> gpurun_out/r2_sweep_split.err
BML_VARIANT=5 timeout 900 python scripts/band_kernel_proxy.py --n 65536 > gpurun_out/r2_band_proxy_split.jsonl 2> gpurun_out/r2_band_proxy_split.err
