"""Launch a few step kernels of one streaming variant for ncu (no timing)."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07981_b200 as bml  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--variant", type=int, default=1)
ap.add_argument("--steps", type=int, default=112)
ap.add_argument("--strip", type=int, default=0)
args = ap.parse_args()
lib = ctypes.CDLL(bml.LIB_DEV)
lib.bml_dev_set_variant.argtypes = [ctypes.c_void_p, ctypes.c_int]
lat = bml.DeviceLattice(args.n)
assert lib.bml_dev_set_variant(ctypes.c_void_p(lat.handle()), args.variant) == 0
if args.strip:
    lat.configure(block_steps=16, strip_rows=args.strip)
lat.init_random(0.35, 1)
lat.step(args.steps)
lat.synchronize()
print("done", args)
