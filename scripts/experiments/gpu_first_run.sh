cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_info.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 300 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 300 python bench.py --workload c2ff --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2ff.json 2> gpurun_out/bench_c2ff.err
for b in 4 8 16; do timeout 120 python bench.py --workload c2ff --steps 3 --warmup 3 --no-cpu --no-e2e --block $b > gpurun_out/bench_c2ff_b$b.json 2>&1; done
