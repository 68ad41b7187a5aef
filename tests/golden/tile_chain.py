"""Long goldens from the UNMODIFIED reference, run as light-cone tiles on all host cores.

TEST INFRASTRUCTURE (build container only: needs oracle/_ref/ref_driver and
oracle/build/liboracle.so). The output JSON is committed and checked on the GPU box.

Why tiles are exact. One reference step (`engine.cpp:196-199`) is an LR phase
whose new cell (i,j) reads only (i,j-1),(i,j),(i,j+1) (`horizontal_rule`,
`engine.cpp:66-80` via `lanes.cpp`), then a TB phase reading (i-1,j),(i,j),(i+1,j).
After L steps a cell depends only on the (2L+1)x(2L+1) box around it. So the
reference run (`ref_driver file`, the reference's own `run()` on a torus of side
T+2L) on the tile "owned T x T block plus an L-cell margin, cut out of the full
torus with wrap-around" gives the owned block EXACTLY after L steps: whatever the
tile's own (wrong) wrap-around injects travels at most L cells in from its edges.

Every leg's full-lattice digest is kept as a checkpoint. The scheme is pinned by
`--check` legs against the committed unbroken-reference goldens (the N=65536
1000-step golden is leg 1 of the configs[4] chain; the N=46336 chain has a digest
at every 1000 steps).

    python tests/golden/tile_chain.py N RHO STEPS LEG TILE WORKDIR [--jobs J]

Leg 0 draws the lattice with the reference's own init_grid (`ref_driver golden
steps=0`, `seeding.cpp:26-51`) and checks its digest.
"""
import argparse
import concurrent.futures as cf
import ctypes
import json
import os
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
ORACLE = os.path.join(ROOT, "oracle", "build", "liboracle.so")


def digest(g):
    lib = ctypes.CDLL(ORACLE)
    lib.orc_digest.restype = ctypes.c_uint64
    lib.orc_digest.argtypes = [ctypes.c_int, ctypes.c_void_p]
    return "0x%016x" % lib.orc_digest(g.shape[0], g.ctypes.data)


def run_tile(args):
    path_in, side, steps, path_out = args
    cmd = [DRIVER, "file", f"in={path_in}", f"n={side}", f"steps={steps}", "metrics=0",
           "backend=lanes", f"dump_final={path_out}"]
    rec = json.loads(subprocess.run(cmd, check=True, capture_output=True, text=True).stdout)
    os.remove(path_in)
    return rec["run_s"]


def leg(cur, steps, tile, margin, scratch, jobs):
    n = cur.shape[0]
    assert margin >= steps
    starts = list(range(0, n, tile))
    owned = [(r, c, min(tile, n - r), min(tile, n - c)) for r in starts for c in starts]
    nxt = np.empty_like(cur)
    cpu = 0.0

    def cut(i):
        r, c, h, w = owned[i]
        side = max(h, w) + 2 * margin
        rows = np.arange(r - margin, r - margin + side) % n
        cols = np.arange(c - margin, c - margin + side) % n
        sub = np.ascontiguousarray(cur[np.ix_(rows, cols)])
        p_in = os.path.join(scratch, f"t{i}.in")
        sub.tofile(p_in)
        return (p_in, side, steps, os.path.join(scratch, f"t{i}.out"))

    with cf.ThreadPoolExecutor(jobs) as ex:
        # keep at most 2*jobs tiles cut ahead of the workers (bounded scratch space)
        pending = {}
        i = 0
        while i < len(owned) or pending:
            while i < len(owned) and len(pending) < 2 * jobs:
                pending[ex.submit(run_tile, cut(i))] = i
                i += 1
            done, _ = cf.wait(pending, return_when=cf.FIRST_COMPLETED)
            for f in done:
                k = pending.pop(f)
                cpu += f.result()
                r, c, h, w = owned[k]
                side = max(h, w) + 2 * margin
                p_out = os.path.join(scratch, f"t{k}.out")
                out = np.fromfile(p_out, dtype=np.uint8).reshape(side, side)
                os.remove(p_out)
                nxt[r:r + h, c:c + w] = out[margin:margin + h, margin:margin + w]
    return nxt, cpu


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int)
    ap.add_argument("rho", type=float)
    ap.add_argument("steps", type=int)
    ap.add_argument("leg", type=int)
    ap.add_argument("tile", type=int)
    ap.add_argument("work")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    ap.add_argument("--check", default=None,
                    help="committed golden JSON whose checkpoints (or final digest) must match")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    os.makedirs(a.work, exist_ok=True)
    scratch = os.path.join(a.work, "tiles")
    os.makedirs(scratch, exist_ok=True)
    log = os.path.join(a.work, "legs.jsonl")
    legs = [json.loads(l) for l in open(log)] if os.path.exists(log) else []

    expect = {}
    if a.check:
        g = json.load(open(a.check))
        for cp in g.get("checkpoints", []):
            expect[cp["step"]] = cp["digest"]
        expect[g["steps"]] = g["final_digest"]

    init_path = os.path.join(a.work, "s0.bin")
    if not legs:
        if not os.path.exists(init_path):
            cmd = [DRIVER, "golden", f"n={a.n}", f"rho={a.rho}", f"seed={a.seed}", "steps=0",
                   "metrics=0", "backend=lanes", f"dump_init={init_path}"]
            print("running", " ".join(cmd), flush=True)
            rec = json.loads(subprocess.run(cmd, check=True, capture_output=True, text=True).stdout)
            with open(os.path.join(a.work, "init.json"), "w") as f:
                json.dump(rec, f)
    init = json.load(open(os.path.join(a.work, "init.json")))
    done = legs[-1]["at_step"] if legs else 0
    cur = np.fromfile(os.path.join(a.work, f"s{done}.bin"), dtype=np.uint8).reshape(a.n, a.n)
    if not legs:
        assert digest(cur) == init["init_digest"], "init dump does not match the reference digest"
    while done < a.steps:
        t0 = time.time()
        steps = min(a.leg, a.steps - done)
        cur, cpu = leg(cur, steps, a.tile, a.leg, scratch, a.jobs)
        done += steps
        d = digest(cur)
        rec = {"at_step": done, "digest": d, "wall_s": time.time() - t0, "ref_run_s": cpu}
        if done in expect:
            rec["matches_unbroken_reference"] = expect[done] == d
            if expect[done] != d:
                print("MISMATCH at", done, d, "expected", expect[done], flush=True)
                sys.exit(1)
        cur.tofile(os.path.join(a.work, f"s{done}.bin"))
        prev = os.path.join(a.work, f"s{done - steps}.bin")
        if os.path.exists(prev):
            os.remove(prev)
        with open(log, "a") as f:
            f.write(json.dumps(rec) + "\n")
        print(json.dumps(rec), flush=True)

    legs = [json.loads(l) for l in open(log)]
    lr = int(np.count_nonzero(cur == 1))
    tb = int(np.count_nonzero(cur == 2))
    out = {"n": a.n, "rho": a.rho, "seed": a.seed, "steps": a.steps, "backend": "lanes",
           "threads": 1, "k": init["k"], "init_digest": init["init_digest"],
           "final_digest": legs[-1]["digest"], "lr_count": lr, "tb_count": tb,
           "init_s": init["init_s"], "run_s": sum(r["ref_run_s"] for r in legs),
           "checkpoints": [{"step": r["at_step"], "digest": r["digest"]} for r in legs],
           "pinned_against_unbroken_reference": sorted(
               r["at_step"] for r in legs if r.get("matches_unbroken_reference")),
           "generator": ("oracle/_ref/ref_driver (unmodified reference sources, lanes backend): "
                         f"reference init_grid, then {len(legs)} legs of {a.leg} steps, each leg "
                         f"the reference's run() on light-cone tiles ({a.tile} owned + {a.leg} "
                         "margin, torus wrap) (tests/golden/tile_chain.py)")}
    path = a.out or os.path.join(
        HERE, f"ref_n{a.n}_rho{a.rho}_seed{a.seed}_steps{a.steps}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path, out["final_digest"], flush=True)


if __name__ == "__main__":
    main()
