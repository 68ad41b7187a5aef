"""bml_dev_step with / without the fused per-step moved counters, through the raw
C-ABI of one or more builds: python scripts/metrics_abi.py LIB.so [...]"""
import ctypes
import json
import sys
import time

vp = ctypes.c_void_p
for path in sys.argv[1:]:
    lib = ctypes.CDLL(path)
    lib.bml_dev_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    lib.bml_dev_init_random.argtypes = [vp, ctypes.c_double, ctypes.c_uint64]
    lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
    lib.bml_dev_sync.argtypes = [vp]
    lib.bml_dev_destroy.argtypes = [vp]
    for n, steps in ((8192, 2000), (32768, 400), (65536, 96)):
        h = vp()
        assert lib.bml_dev_create(n, 0, ctypes.byref(h)) == 0
        assert lib.bml_dev_init_random(h, 0.35, 1) == 0
        lm = (ctypes.c_int64 * steps)()
        tm = (ctypes.c_int64 * steps)()
        res = {}
        for mode in ("bare", "moved"):
            args = (None, None) if mode == "bare" else (ctypes.cast(lm, vp), ctypes.cast(tm, vp))
            lib.bml_dev_step(h, steps, *args, None, None)
            lib.bml_dev_sync(h)
            t = time.perf_counter()
            rc = lib.bml_dev_step(h, steps, *args, None, None)
            lib.bml_dev_sync(h)
            res[mode] = n * n * steps / (time.perf_counter() - t) / 1e12
            assert rc == 0, rc
        print(json.dumps({"lib": path.split("/")[-1], "n": n, **res, "lm_last": lm[steps - 1]}), flush=True)
        lib.bml_dev_destroy(h)
