"""Cost of the fused per-step metrics: DeviceLattice.step vs
step_with_metrics (lr/tb moved every step + the vehicle census: at launch boundaries by
default, after every step with set_census(True)) on the same lattice. One JSON line per size."""
import json
import time

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1804_07981_b200 as bml  # noqa: E402

for n, steps in ((1024, 4096), (8192, 2000), (32768, 400)):
    lat = bml.DeviceLattice(n)
    lat.init_random(0.35, 1)
    lat.step(steps)
    lat.synchronize()
    t = time.perf_counter()
    lat.step(steps)
    lat.synchronize()
    bare = time.perf_counter() - t
    cu = n * n * steps
    rec = {"n": n, "steps": steps, "bare_tcups": cu / bare / 1e12}
    for strict in (False, True):
        lat.set_census(strict)
        lat.step_with_metrics(steps)
        t = time.perf_counter()
        m = lat.step_with_metrics(steps)
        with_m = time.perf_counter() - t
        key = "strict" if strict else "boundary"
        rec[f"metrics_{key}_tcups"] = cu / with_m / 1e12
        rec[f"slowdown_{key}"] = with_m / bare
    rec["last_mobility"] = m[-1].mobility
    print(json.dumps(rec), flush=True)
