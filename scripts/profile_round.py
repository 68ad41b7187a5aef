"""Turn a gpu_profile.sh pass (gpurun_out/) into the committed profiles/ summaries.

python scripts/profile_round.py [--round r1]
  gpurun_out/ncu_<w>.ncu-rep   -> profiles/<round>_ncu_bench_<w>.json  (+ traffic_<w>.json)
  gpurun_out/launches_<w>.csv  -> profiles/<round>_launches_<w>.json   (+ the csv)
Needs the ncu CLI (present in the build container; no GPU required).
"""
import argparse
import collections
import csv
import json
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarise  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (WORKLOADS)

ap = argparse.ArgumentParser()
ap.add_argument("--round", default="r1")
args = ap.parse_args()

for w, (n, rho, seed, steps, desc) in bench.WORKLOADS.items():
    rep = os.path.join(OUT, f"ncu_{w}.ncu-rep")
    if not os.path.exists(rep):
        continue
    rows = summarise(rep)
    k = rows[0]
    resident = "resident" in k["kernel"]
    steps_per_launch = steps if resident else 16
    k["cell_updates_per_launch"] = n * n * steps_per_launch
    k["algorithmic_bytes_per_launch"] = bench.BYTES_PER_CELL_UPDATE * k["cell_updates_per_launch"]
    k["dram_bytes_per_cell_update"] = k["dram_bytes"] / k["cell_updates_per_launch"]
    k["workload"] = desc
    k["command"] = f"ncu --set full --clock-control none -k regex:{'resident' if resident else 'step_block'} python bench.py --workload {w} --steps 1 --warmup 1 --no-cpu --no-e2e"
    path = os.path.join(PROF, f"{args.round}_ncu_bench_{w}.json")
    with open(path, "w") as f:
        json.dump(rows, f, indent=1)
    with open(os.path.join(PROF, f"traffic_{w}.json"), "w") as f:
        json.dump({"kernel": "resident_kernel" if resident else "step_block_kernel",
                   "dram_bytes_per_launch": k["dram_bytes"],
                   "algorithmic_bytes_per_launch": k["algorithmic_bytes_per_launch"],
                   "source": f"profiles/{os.path.basename(path)} (ncu --set full, one "
                             f"{steps_per_launch}-step launch)"}, f, indent=1)
    print("wrote", path)

for w in bench.WORKLOADS:
    src = os.path.join(OUT, f"launches_{w}.csv")
    if not os.path.exists(src):
        continue
    with open(src) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"][:70]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(r["Metric Unit"], 1)
        tot[name][0] += 1
        tot[name][1] += v * scale
    total = sum(t for _, t in tot.values())
    out = {"command": f"ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --workload {w} --steps 2 --warmup 1 --no-cpu --no-e2e",
           "note": "cold-cache serialised launches: compare shares, not absolute times",
           "kernels": sorted(({"kernel": k, "launches": c, "total_ns": t, "share": t / total}
                              for k, (c, t) in tot.items()), key=lambda d: -d["total_ns"])}
    with open(os.path.join(PROF, f"{args.round}_launches_{w}.json"), "w") as f:
        json.dump(out, f, indent=1)
    shutil.copy(src, os.path.join(PROF, f"{args.round}_launches_{w}.csv"))
    print("wrote launches", w)
