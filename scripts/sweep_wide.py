"""Narrow (32 cells/lane) vs wide (64 cells/lane, TMA bulk ring) streaming kernel.

For each lattice size: device init_grid, then per variant (1 narrow K16, 2 wide K14,
3 wide K12) and strip setting: the digest after `--check` steps (must agree across
variants and with the reference golden when one is committed), then the
device-resident throughput of `--steps` steps (CUDA events, L2 flushed, best of reps).
One JSON line per configuration.
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
ap.add_argument("--n", type=int, nargs="+", default=[65536, 32768, 16384, 8192])
ap.add_argument("--variants", type=int, nargs="+", default=[1, 2, 3])
ap.add_argument("--strips", type=int, nargs="+", default=[0])
ap.add_argument("--steps", type=int, default=0)
ap.add_argument("--check", type=int, default=1000)
ap.add_argument("--reps", type=int, default=3)
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
    steps = args.steps or max(112, min(4200, int(4.3e13 / (n * n)) // 84 * 84))
    stream = torch.cuda.Stream()
    lat.set_stream(stream.cuda_stream)
    ref = golden(n, args.check)
    for v in args.variants:
        for r in args.strips:
            assert lib.bml_dev_set_variant(h, v) == 0
            lat.configure(block_steps=16, strip_rows=r if r else -1)
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
            print(json.dumps({"n": n, "variant": v, "strip": r, "steps": steps, "gcups": round(best, 1),
                              "digest": dig, "golden": ref, "golden_ok": None if ref is None else dig == ref,
                              "strips": ns.value, "items": items.value, "ctas": grid.value}), flush=True)
