cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_multi2_c1.json 2> gpurun_out/bench_multi2_c1.err
timeout 600 $R --nproc-per-node 2 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 3 --workload c2ff > gpurun_out/bench_multi2_c2.json 2> gpurun_out/bench_multi2_c2.err
timeout 600 $R --nproc-per-node 2 --master-port 29513 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_multi2_ref.json 2> gpurun_out/bench_multi2_ref.err
