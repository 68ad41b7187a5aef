cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
for w in c2ff c2jam c3; do timeout 600 python bench.py --workload $w --no-cpu > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
timeout 900 python bench.py --workload c4 --no-cpu --steps 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
L=paper_1804_07981_b200/libbml_dev.so
timeout 300 python scripts/abi_sweep.py $L --n 8192 16384 32768 --blocks 16 --strips 0 > gpurun_out/sweep_auto.jsonl 2>&1
