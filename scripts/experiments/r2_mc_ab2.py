import ctypes, json, os, sys, time
pkg = sys.argv[1]
sys.path.insert(0, pkg)
import paper_1804_07981_b200 as bml
lib = ctypes.CDLL(bml.LIB_DEV)
vp = ctypes.c_void_p
lib.bml_dev_enable_timing.argtypes = [vp, ctypes.c_int]
lib.bml_dev_kernel_stats.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double), ctypes.c_int]
for n, steps in ((8192, 2000), (32768, 400)):
    lat = bml.DeviceLattice(n)
    h = vp(lat.handle())
    lat.init_random(0.35, 1)
    lat.step_with_metrics(steps)
    lib.bml_dev_enable_timing(h, 1)
    L, ms = ctypes.c_int64(), ctypes.c_double()
    lib.bml_dev_kernel_stats(h, ctypes.byref(L), ctypes.byref(ms), 1)
    t = time.perf_counter(); lat.step(steps); lat.synchronize(); bare = time.perf_counter() - t
    lib.bml_dev_kernel_stats(h, ctypes.byref(L), ctypes.byref(ms), 1)
    bl, bms = L.value, ms.value
    t = time.perf_counter(); lat.step_with_metrics(steps); wm = time.perf_counter() - t
    lib.bml_dev_kernel_stats(h, ctypes.byref(L), ctypes.byref(ms), 1)
    print(json.dumps({"pkg": pkg, "n": n, "bare_wall_ms": bare*1e3, "bare_launches": bl, "bare_kernel_ms": bms,
                      "metrics_wall_ms": wm*1e3, "metrics_launches": L.value, "metrics_kernel_ms": ms.value}), flush=True)
