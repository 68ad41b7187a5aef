"""Launch a handful of step kernels for ncu (one config), no timing."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07981_b200 as bml  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--block", type=int, default=16)
ap.add_argument("--strip", type=int, default=256)
ap.add_argument("--launches", type=int, default=4)
ap.add_argument("--rho", type=float, default=0.35)
args = ap.parse_args()
g = bml.init_grid(args.n, args.rho, 1)
lat = bml.DeviceLattice(args.n)
lat.configure(block_steps=args.block, strip_rows=args.strip)
lat.upload(g)
lat.step(args.block * args.launches)
lat.synchronize()
print("done", args)
