cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:step_block -s 2 -c 1 -o gpurun_out/prof_n32768_k16 -f python scripts/prof_step.py --n 32768 --block 16 --strip 256 > gpurun_out/prof1.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:step_block -s 2 -c 1 -o gpurun_out/prof_n32768_k8 -f python scripts/prof_step.py --n 32768 --block 8 --strip 256 >> gpurun_out/prof1.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:step_block -s 2 -c 1 -o gpurun_out/prof_n1024_k8 -f python scripts/prof_step.py --n 1024 --block 8 --strip 16 >> gpurun_out/prof1.log 2>&1
timeout 600 python scripts/sweep.py --n 1024 8192 32768 --blocks 8 16 --strips 16 64 128 256 512 > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err
