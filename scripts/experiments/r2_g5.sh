for v in 1 4 2; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:step_ -s 2 -c 1 -o gpurun_out/r2_ncu_v$v python scripts/prof_variant.py --n 32768 --variant $v > gpurun_out/r2_ncu_v$v.log 2>&1
done
