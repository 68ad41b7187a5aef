timeout 900 ncu --set full --import-source on --clock-control none -k regex:resident -c 1 -o gpurun_out/r2_ncu_c1_resident python bench.py --workload c1 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2_ncu_c1.log 2>&1
ncu -i gpurun_out/r2_ncu_c1_resident.ncu-rep --page details > gpurun_out/r2_ncu_c1_details.txt 2>&1
