cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_init.py -x -q > gpurun_out/pytest_init.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_init.log
timeout 600 python - > gpurun_out/init_timing.log 2>&1 <<'PY'
import time, paper_1804_07981_b200 as bml
for n in (8192, 32768, 65536):
    lat = bml.DeviceLattice(n)
    t = time.perf_counter(); lat.init_random(0.35, 1); lat.synchronize(); t = time.perf_counter() - t
    print(n, "device init_random s", round(t, 3), "counts", lat.counts(), "k", bml.vehicles_per_species(n, 0.35), flush=True)
    if n <= 32768:
        t = time.perf_counter(); g = lat.download(); print(n, "digest", hex(g.digest()), "download+digest s", round(time.perf_counter() - t, 2), flush=True)
    del lat
PY
timeout 900 python bench.py --workload c3 --no-cpu --steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 1200 python bench.py --workload c4 --no-cpu --steps 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
