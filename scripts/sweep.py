"""Sweep (block_steps, strip_rows) for the step kernel at several lattice sizes.

Prints one JSON line per configuration: device-resident Gcell-updates/s measured
with CUDA events (L2 flushed before each timed run). Used to pick the defaults in
bml_dev.cu; results are summarised in profiles/.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07981_b200 as bml  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[1024, 8192, 32768])
ap.add_argument("--blocks", type=int, nargs="+", default=[4, 8, 16])
ap.add_argument("--strips", type=int, nargs="+", default=[0, 16, 32, 64, 128, 256, 512, 1000])
ap.add_argument("--steps", type=int, default=0, help="BML steps per timed run (0 = auto)")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in args.n:
    cells = bytes((i * 2654435761 >> 7) % 3 for i in range(0))  # placeholder, replaced below
    g = bml.init_grid(n, 0.35, 1) if n <= 32768 else None
    lat = bml.DeviceLattice(n)
    lat.upload(g)
    steps = args.steps or max(64, min(4096, int(2e12 / (n * n))))
    stream = torch.cuda.Stream()
    lat.set_stream(stream.cuda_stream)
    for k in args.blocks:
        for r in args.strips:
            try:
                lat.configure(block_steps=k, strip_rows=r)
            except ValueError:
                continue
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
                    ms = e0.elapsed_time(e1)
                    best = max(best, n * n * steps / (ms / 1e3) / 1e9)
            print(json.dumps({"n": n, "block": k, "strip": r, "steps": steps, "gcups": round(best, 1)}),
                  flush=True)
