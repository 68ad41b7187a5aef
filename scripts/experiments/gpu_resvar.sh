cd $GRAFT_REPO_ROOT
timeout 600 python scripts/abi_sweep.py build_variants/libbml_dev_head.so build_variants/libbml_dev_push.so build_variants/libbml_dev_skip.so --n 1024 512 --blocks 8 16 --steps 4096 > gpurun_out/abi_resvar.jsonl 2> gpurun_out/abi_resvar.err
