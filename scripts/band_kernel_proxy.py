"""Per-GPU cost of a row band, measured on ONE GPU: the N x N torus as g connected
bands, stepped one band-launch at a time with a device sync in between, so every band
kernel runs alone on the whole GPU (as it would on its own GPU) and its flags are
always already raised (its neighbours finished the previous launch). The CUDA-event
kernel time per band-launch, against the single-band launch, gives the per-GPU
efficiency of the g-GPU strong split without the time-slicing of the concurrent
virtual-band run (scripts/virtual_bands.py). Not a multi-GPU measurement: NVLink
latency and flag waits between live GPUs are not in it.

python scripts/band_kernel_proxy.py [--n 65536 32768] [--bands 1 2 4 8] [--launches 16]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07981_b200 as bml  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[65536, 32768])
ap.add_argument("--bands", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--launches", type=int, default=16)
ap.add_argument("--block", type=int, default=16, help="steps per band launch")
ap.add_argument("--strips", type=int, nargs="+", default=[0], help="-ns per band (0 = automatic)")
args = ap.parse_args()

lib = ctypes.CDLL(bml.LIB_DEV)
vp = ctypes.c_void_p
lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
lib.bml_dev_sync.argtypes = [vp]
lib.bml_dev_enable_timing.argtypes = [vp, ctypes.c_int]
lib.bml_dev_kernel_stats.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double), ctypes.c_int]
lib.bml_dev_last_launch.argtypes = [vp] + [ctypes.POINTER(ctypes.c_int)] * 3

for n in args.n:
    single = None
    ref_digest = None
    for g, ns in [(g, ns) for g in args.bands for ns in args.strips]:
        lat = bml.DeviceLattice(n, g)
        lat.configure(block_steps=args.block, strip_rows=-ns if ns > 1 else (-1 if ns == 0 else 65536))
        lat.init_random(0.35, 1)
        hs = [vp(lat.handle(b)) for b in range(g)]
        for h in hs:  # warm-up launch per band
            assert lib.bml_dev_step(h, args.block, None, None, None, None) == 0
            assert lib.bml_dev_sync(h) == 0
        for h in hs:
            lib.bml_dev_enable_timing(h, 1)
            lib.bml_dev_kernel_stats(h, None, None, 1)
        for _ in range(args.launches):
            for h in hs:
                assert lib.bml_dev_step(h, args.block, None, None, None, None) == 0
                assert lib.bml_dev_sync(h) == 0
        per_band = []
        for h in hs:
            L, ms = ctypes.c_int64(), ctypes.c_double()
            lib.bml_dev_kernel_stats(h, ctypes.byref(L), ctypes.byref(ms), 1)
            per_band.append(ms.value / L.value)
        geo = [ctypes.c_int() for _ in range(3)]
        lib.bml_dev_last_launch(hs[0], *[ctypes.byref(x) for x in geo])
        d = lat.digest()
        ref_digest = d if ref_digest is None else ref_digest
        worst = max(per_band)  # the slowest band sets the pace of a lockstep multi-GPU run
        per_gpu_tcups = n * ((n + g - 1) // g) * args.block / (worst / 1e3) / 1e12
        rec = {"n": n, "bands": g, "block": args.block, "strips_requested": ns, "band_rows": (n + g - 1) // g, "ms_per_launch_max": worst,
               "ms_per_launch_mean": sum(per_band) / g, "per_gpu_tcups": per_gpu_tcups,
               "projected_total_tcups": per_gpu_tcups * g, "geometry_band0": [x.value for x in geo],
               "digest_equal": d == ref_digest}
        if g == 1 and single is None:
            single = per_gpu_tcups
        rec["per_gpu_efficiency_vs_single"] = per_gpu_tcups / single if single else None
        print(json.dumps(rec), flush=True)
        del lat
