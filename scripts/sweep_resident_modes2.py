import ctypes, json, sys, torch
path = sys.argv[1]
lib = ctypes.CDLL(path); vp = ctypes.c_void_p
lib.bml_dev_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
lib.bml_dev_init_random.argtypes = [vp, ctypes.c_double, ctypes.c_uint64]
lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
lib.bml_dev_set_resident.argtypes = [vp, ctypes.c_int]
lib.bml_dev_configure.argtypes = [vp, ctypes.c_int, ctypes.c_int]
lib.bml_dev_set_stream.argtypes = [vp, vp]
for n in (1024, 512, 256):
    h = vp(); assert lib.bml_dev_create(n, 0, ctypes.byref(h)) == 0
    lib.bml_dev_init_random(h, 0.38, 1)
    s = torch.cuda.Stream(); lib.bml_dev_set_stream(h, vp(s.cuda_stream))
    for mode, blk in ((1, 8), (1, 16), (2, 8)):
        lib.bml_dev_set_resident(h, mode); lib.bml_dev_configure(h, blk, 0)
        with torch.cuda.stream(s):
            lib.bml_dev_step(h, 4096, None, None, None, None)
            best = 0
            for _ in range(5):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s); lib.bml_dev_step(h, 4096, None, None, None, None); e1.record(s); e1.synchronize()
                best = max(best, n * n * 4096 / (e0.elapsed_time(e1) / 1e3) / 1e12)
        print(json.dumps({"n": n, "mode": mode, "block": blk, "tcups": round(best, 3)}), flush=True)
