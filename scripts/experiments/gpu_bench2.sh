cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 400 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 400 python bench.py --impl reference --steps 3 > gpurun_out/bench_ref_c1.json 2> gpurun_out/bench_ref_c1.err
timeout 400 python bench.py --workload c2ff --no-cpu > gpurun_out/bench_c2ff.json 2> gpurun_out/bench_c2ff.err
timeout 600 python bench.py --workload c3 --no-cpu --steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_c1.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:resident -c 1 -o gpurun_out/prof_resident_c1 -f python scripts/prof_step.py --n 1024 --block 16 --launches 1 > gpurun_out/prof_res.log 2>&1
