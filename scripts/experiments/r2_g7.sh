timeout 900 python scripts/virtual_bands.py --blocks 8 16 > gpurun_out/r2_virtual_bands.jsonl 2> gpurun_out/r2_virtual_bands.err
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r2_pytest_gpu2.log
