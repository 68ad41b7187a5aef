set -x
free -g; nproc; lscpu | grep -E "Model name|Socket|Thread|Core"
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench_c4_a.json 2> gpurun_out/r2_bench_c4_a.err; echo rc=$?
tail -3 gpurun_out/r2_bench_c4_a.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu > gpurun_out/r2_bench_c4_g2shared.json 2> gpurun_out/r2_bench_c4_g2shared.err; echo rc=$?
tail -3 gpurun_out/r2_bench_c4_g2shared.err
