cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:step_block -s 10 -c 1 -o gpurun_out/prof_c3 -f python scripts/abi_sweep.py paper_1804_07981_b200/libbml_dev.so --n 32768 --blocks 16 --strips 0 --steps 256 --reps 1 > gpurun_out/prof_c3.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:step_block -s 10 -c 1 -o gpurun_out/prof_c2 -f python scripts/abi_sweep.py paper_1804_07981_b200/libbml_dev.so --n 8192 --blocks 16 --strips 0 --steps 256 --reps 1 > gpurun_out/prof_c2.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:resident -c 1 -o gpurun_out/prof_c1 -f python scripts/abi_sweep.py paper_1804_07981_b200/libbml_dev.so --n 1024 --blocks 16 --strips 0 --steps 4096 --reps 1 > gpurun_out/prof_c1.log 2>&1
