"""N<=1024 cluster-resident kernel: throughput vs ghost depth (block_steps)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_07981_b200 as bml  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n, steps in ((1024, 4096), (512, 4096), (256, 4096)):
    g = bml.init_grid(n, 0.38, 1)
    lat = bml.DeviceLattice(n)
    stream = torch.cuda.Stream()
    lat.set_stream(stream.cuda_stream)
    for ghost in (1, 2, 4, 8, 16):
        for resident in (1, 2, 0):
            lat.set_resident(resident)
            lat.configure(block_steps=ghost, strip_rows=16)
            lat.upload(g)
            with torch.cuda.stream(stream):
                lat.step(steps)
                best = 0.0
                for _ in range(3):
                    flush.fill_(1)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    lat.step(steps)
                    e1.record(stream)
                    e1.synchronize()
                    best = max(best, n * n * steps / (e0.elapsed_time(e1) / 1e3) / 1e9)
            print(json.dumps({"n": n, "ghost": ghost, "resident": resident,
                              "cluster": lat.resident_cluster, "gcups": round(best, 1)}), flush=True)
