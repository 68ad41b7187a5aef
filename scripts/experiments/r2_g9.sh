python scripts/experiments/r2_mc_ab.py scratch_r1 > gpurun_out/r2_mc_ab.jsonl 2>&1
python scripts/experiments/r2_mc_ab.py . >> gpurun_out/r2_mc_ab.jsonl 2>&1
timeout 1700 python bench.py --impl reference --steps 3 > gpurun_out/r2_ref_c4.json 2> gpurun_out/r2_ref_c4.err
