# Round profiling pass: one ncu --set full capture of the dominant kernel per
# bench workload and the launch lists of the bench commands (scripts/profile_round.py
# turns them into profiles/). Never read throughput numbers from these runs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --no-cpu --no-e2e --steps 1 --warmup 1"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:resident -c 1 -o gpurun_out/ncu_c1 -f $B --workload c1 > gpurun_out/ncu_c1.log 2>&1
for w in c2ff c3 c4; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:step_block -s 20 -c 1 -o gpurun_out/ncu_$w -f $B --workload $w > gpurun_out/ncu_$w.log 2>&1
done
for w in c1 c3; do
  timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$w.csv python bench.py --no-cpu --no-e2e --steps 2 --warmup 1 --workload $w > gpurun_out/launches_$w.log 2>&1
done
