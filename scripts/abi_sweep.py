"""Compare engine builds through the raw C-ABI (ctypes), e.g. experimental variants.

python scripts/abi_sweep.py LIB.so [LIB2.so ...] --n 8192 32768 --blocks 8 16
Random 0/1/2 lattices (throughput does not depend on content: branch-free kernels).
"""
import argparse
import ctypes
import json

import torch

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--n", type=int, nargs="+", default=[8192, 32768])
ap.add_argument("--blocks", type=int, nargs="+", default=[16])
ap.add_argument("--strips", type=int, nargs="+", default=[0])
ap.add_argument("--steps", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
vp = ctypes.c_void_p
for n in args.n:
    host = (torch.randint(0, 3, (n * n,), dtype=torch.uint8)).pin_memory()
    steps = args.steps or max(64, min(4096, int(2e12 / (n * n))))
    for path in args.libs:
        lib = ctypes.CDLL(path)
        lib.bml_dev_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
        lib.bml_dev_upload.argtypes = [vp, vp, ctypes.c_size_t]
        lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
        lib.bml_dev_configure.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        lib.bml_dev_set_stream.argtypes = [vp, vp]
        lib.bml_dev_download.argtypes = [vp, vp, ctypes.c_size_t]
        lib.bml_dev_destroy.argtypes = [vp]
        has_ll = hasattr(lib, "bml_dev_last_launch")
        if has_ll:
            lib.bml_dev_last_launch.argtypes = [vp] + [ctypes.POINTER(ctypes.c_int)] * 3
        h = vp()
        assert lib.bml_dev_create(n, 0, ctypes.byref(h)) == 0
        stream = torch.cuda.Stream()
        lib.bml_dev_set_stream(h, vp(stream.cuda_stream))
        ref = None
        for k in args.blocks:
            for r in args.strips:
                assert lib.bml_dev_configure(h, k, r if r else -1) == 0
                assert lib.bml_dev_upload(h, vp(host.data_ptr()), n) == 0
                with torch.cuda.stream(stream):
                    lib.bml_dev_step(h, steps, None, None, None, None)
                    best = 0.0
                    for _ in range(args.reps):
                        flush.fill_(1)
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        lib.bml_dev_step(h, steps, None, None, None, None)
                        e1.record(stream)
                        e1.synchronize()
                        best = max(best, n * n * steps / (e0.elapsed_time(e1) / 1e3) / 1e9)
                out = torch.empty(n * n, dtype=torch.uint8).pin_memory()
                assert lib.bml_dev_download(h, vp(out.data_ptr()), n) == 0
                digest = int(out[: 1 << 20].sum()) + int(out.sum())
                if ref is None:
                    ref = digest
                geo = None
                if has_ll:
                    g3 = [ctypes.c_int() for _ in range(3)]
                    lib.bml_dev_last_launch(h, *[ctypes.byref(x) for x in g3])
                    geo = [x.value for x in g3]
                print(json.dumps({"lib": path.split("/")[-1], "n": n, "block": k, "strip": r,
                                  "steps": steps * (1 + args.reps), "gcups": round(best, 1),
                                  "checksum": digest, "strips_items_ctas": geo}), flush=True)
        lib.bml_dev_destroy(h)
