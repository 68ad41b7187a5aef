cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_verify.py tests/test_snapshot.py tests/test_gpu_digest.py -x -q > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
L=paper_1804_07981_b200/libbml_dev.so
timeout 300 python scripts/abi_sweep.py $L --n 8192 --blocks 16 --strips -56 -60 -62 -63 -64 -65 -66 -68 -72 -96 -120 -128 > gpurun_out/sweep_ns2_8192.jsonl 2>&1
timeout 300 python scripts/abi_sweep.py $L --n 16384 --blocks 16 --strips -48 -56 -60 -63 -64 -65 -70 -80 -98 -128 > gpurun_out/sweep_ns2_16384.jsonl 2>&1
