cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 400 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_c1.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:resident -s 1 -c 1 -o gpurun_out/prof_bench_c1 -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/prof_bench_c1.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:step_block -s 20 -c 1 -o gpurun_out/prof_bench_c3 -f python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/prof_bench_c3.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv -c 400 --log-file gpurun_out/launches_c3.csv python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_c3.log 2>&1
timeout 600 python bench.py --workload c3 --no-cpu --steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c2ff --no-cpu > gpurun_out/bench_c2ff.json 2> gpurun_out/bench_c2ff.err
timeout 600 python bench.py --workload c2jam --no-cpu > gpurun_out/bench_c2jam.json 2> gpurun_out/bench_c2jam.err
