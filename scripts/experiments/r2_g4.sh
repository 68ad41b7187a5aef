timeout 900 python scripts/sweep_wide.py --n 65536 32768 --variants 1 2 4 > gpurun_out/r2_sweep_wide2.jsonl 2> gpurun_out/r2_sweep_wide2.err
