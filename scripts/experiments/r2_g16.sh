timeout 900 python scripts/sweep_wide.py --n 65536 32768 16384 8192 --variants 1 5 --check 1000 > gpurun_out/r2_sweep_split2.jsonl 2> gpurun_out/r2_sweep_split2.err
BML_VARIANT=5 timeout 900 python scripts/band_kernel_proxy.py --n 65536 > gpurun_out/r2_band_proxy_split2.jsonl 2> gpurun_out/r2_band_proxy_split2.err
