timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c4_final.json 2> gpurun_out/r2_bench_c4_final.err
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_ref_c4.json 2> gpurun_out/r2_bench_ref_c4.err
for w in c3 c2ff c1; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/r2_launches_c4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:step_block -s 5 -c 1 -o gpurun_out/r2_ncu_bench_c4 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r2_ncu_bench_c4.log 2>&1
