timeout 900 python -m pytest tests/test_gpu_async.py tests/test_gpu_census.py -x -q 2>&1 | tail -5 > gpurun_out/r2_async.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r2_bench_c4_b.json 2> gpurun_out/r2_bench_c4_b.err
timeout 600 python bench.py --workload c1 --steps 20 --warmup 5 --no-cpu > gpurun_out/r2_bench_c1_b.json 2> gpurun_out/r2_bench_c1_b.err
