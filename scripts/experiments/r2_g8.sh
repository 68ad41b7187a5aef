timeout 600 python scripts/metrics_cost.py > gpurun_out/r2_metrics_cost.jsonl 2> gpurun_out/r2_metrics_cost.err
/usr/bin/time -v timeout 1700 python bench.py --impl reference --steps 3 > gpurun_out/r2_ref_c4.json 2> gpurun_out/r2_ref_c4.err
