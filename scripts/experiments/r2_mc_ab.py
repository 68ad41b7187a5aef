import json, os, sys, time
pkg = sys.argv[1]
sys.path.insert(0, pkg)
import paper_1804_07981_b200 as bml
print("lib", bml.__file__, file=sys.stderr)
for n, steps in ((8192, 2000), (32768, 400)):
    lat = bml.DeviceLattice(n)
    lat.init_random(0.35, 1)
    lat.step(steps); lat.synchronize()
    t = time.perf_counter(); lat.step(steps); lat.synchronize(); bare = time.perf_counter() - t
    lat.step_with_metrics(steps)
    t = time.perf_counter(); m = lat.step_with_metrics(steps); wm = time.perf_counter() - t
    print(json.dumps({"pkg": pkg, "n": n, "bare_tcups": n*n*steps/bare/1e12, "metrics_tcups": n*n*steps/wm/1e12, "slowdown": wm/bare}), flush=True)
