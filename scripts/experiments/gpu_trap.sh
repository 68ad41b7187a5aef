cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
L=paper_1804_07981_b200/libbml_dev.so
V=build_variants/libbml_dev_notrap.so
timeout 900 python scripts/abi_sweep.py $L $V --n 8192 16384 32768 --blocks 16 --strips 0 32 48 64 96 128 256 > gpurun_out/sweep_trap.jsonl 2>&1
timeout 600 python scripts/abi_sweep.py $L $V --n 8192 --blocks 8 --strips 0 32 64 > gpurun_out/sweep_trap_k8.jsonl 2>&1
timeout 600 python bench.py --workload c3 --no-cpu --steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c2ff --no-cpu > gpurun_out/bench_c2ff.json 2> gpurun_out/bench_c2ff.err
