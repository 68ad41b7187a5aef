"""Streaming-kernel variants at the bench sizes: device init_grid, a digest check
after `--check` steps against the committed reference golden (where one exists),
then device-resident throughput of `--steps` steps (CUDA events on the handle's
stream, L2 flushed before each rep, best of `--reps`). One JSON line per (n, variant).

    python scripts/sweep_eo.py --n 65536 32768 16384 --variants 1 6 7 8
"""
import argparse
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1804_07981_b200 as bml  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[65536, 32768, 16384])
ap.add_argument("--variants", type=int, nargs="+", default=[1, 6])
ap.add_argument("--steps", type=int, default=0)
ap.add_argument("--check", type=int, default=1000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--strips", type=int, nargs="+", default=[0], help="0 auto, k > 0 exactly k strips")
args = ap.parse_args()

lib = ctypes.CDLL(bml.LIB_DEV)
lib.bml_dev_set_variant.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.bml_dev_last_launch.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int)] * 3


def golden(n, steps):
    p = os.path.join(ROOT, "tests", "golden", f"ref_n{n}_rho0.35_seed1_steps{steps}.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)["final_digest"]
    return None


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in args.n:
    lat = bml.DeviceLattice(n)
    h = ctypes.c_void_p(lat.handle())
    steps = args.steps or max(1008, min(10080, int(4.3e13 / (n * n)) // 1008 * 1008))
    stream = torch.cuda.Stream()
    lat.set_stream(stream.cuda_stream)
    ref = golden(n, args.check)
    for v, st in [(v, st) for v in args.variants for st in args.strips]:
        assert lib.bml_dev_set_variant(h, v) == 0
        lat.configure(block_steps=16, strip_rows=-st if st else -1)  # -1: auto
        lat.init_random(0.35, 1)
        lat.step(args.check)
        dig = f"0x{lat.digest():016x}"
        with torch.cuda.stream(stream):
            lat.step(steps)  # warm
            best = 0.0
            for _ in range(args.reps):
                flush.fill_(1)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                lat.step(steps)
                e1.record(stream)
                e1.synchronize()
                best = max(best, n * n * steps / (e0.elapsed_time(e1) / 1e3) / 1e9)
        ns, items, grid = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        lib.bml_dev_last_launch(h, ctypes.byref(ns), ctypes.byref(items), ctypes.byref(grid))
        print(json.dumps({"n": n, "variant": v, "strip_setting": st, "steps": steps, "gcups": round(best, 1), "digest": dig,
                          "golden_steps": args.check, "golden": ref,
                          "golden_ok": None if ref is None else dig == ref, "strips": ns.value,
                          "items": items.value, "ctas": grid.value}), flush=True)
