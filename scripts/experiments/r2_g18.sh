timeout 900 python scripts/band_kernel_proxy.py --n 65536 --bands 1 --strips 0 > gpurun_out/r2_band_strips.jsonl 2>&1
timeout 900 python scripts/band_kernel_proxy.py --n 65536 --bands 8 --strips 0 6 8 9 11 13 17 25 34 >> gpurun_out/r2_band_strips.jsonl 2>&1
timeout 900 python scripts/band_kernel_proxy.py --n 65536 --bands 4 --strips 0 9 13 17 25 34 >> gpurun_out/r2_band_strips.jsonl 2>&1
