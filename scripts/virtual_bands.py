"""Row-band protocol overhead on ONE GPU: an n x n torus split into g bands (each a
bml_dev band handle with in-kernel ghost-row exchange and flags, all on device 0)
against the single-band run. The bands share the GPU's SMs, so the ideal is the
single-band throughput; the gap is the cost of the band protocol (flag waits,
image copies, smaller launches). Bands step in lockstep, `block` steps per launch.

python scripts/virtual_bands.py [--sizes 8192:2048 32768:320 65536:112] [--blocks 8 16]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07981_b200 as bml  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", nargs="+", default=["8192:2048", "32768:320", "65536:112"])
ap.add_argument("--blocks", type=int, nargs="+", default=[16])
ap.add_argument("--bands", type=int, nargs="+", default=[1, 2, 4, 8])
args = ap.parse_args()

for spec in args.sizes:
    n, steps = (int(x) for x in spec.split(":"))
    for block in args.blocks:
        ref = None
        for g in args.bands:
            lat = bml.DeviceLattice(n, devices=g)
            lat.configure(block_steps=block, strip_rows=0)
            lat.init_random(0.35, 1)
            lat.step(steps)
            lat.synchronize()
            t = time.perf_counter()
            lat.step(steps)
            lat.synchronize()
            dt = time.perf_counter() - t
            d = lat.digest()
            ref = d if ref is None else ref
            print(json.dumps({"n": n, "bands": g, "block": block, "steps": steps,
                              "tcups": n * n * steps / dt / 1e12, "digest_equal": d == ref}), flush=True)
            del lat
