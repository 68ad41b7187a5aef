python scripts/experiments/r2_mc_ab2.py scratch_r1 > gpurun_out/r2_mc_ab2.jsonl 2>&1
python scripts/experiments/r2_mc_ab2.py . >> gpurun_out/r2_mc_ab2.jsonl 2>&1
