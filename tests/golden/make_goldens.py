"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref/ref_driver).

TEST INFRASTRUCTURE. Run in the build container (where /root/reference exists and
`make -C oracle ref` has built the driver); the JSON it writes is committed so the
GPU box (which has no /root/reference) can check the CUDA path against it.

    python tests/golden/make_goldens.py small      # seconds-to-a-minute configs
    python tests/golden/make_goldens.py big        # N=8192 (~5 min each, lanes)
    python tests/golden/make_goldens.py huge       # N=32768 / N=65536 (hours, lanes)
    python tests/golden/make_goldens.py c3         # N=32768 only (~95 min, lanes)
    python tests/golden/make_goldens.py c4short    # N=65536, 1000 steps (~45 min, 43 GB RAM)
    python tests/golden/make_goldens.py c4         # N=65536, 10000 steps (~6 h, 43 GB RAM)
    python tests/golden/make_goldens.py regimes    # N=256, rho .25/.38, seeds 1-10, 4096 steps (~1 min)
    python tests/golden/make_goldens.py c4chain WORKDIR
                                                   # N=65536, 10000 steps as ten resumable 1000-step
                                                   # legs (golden leg, then `file` legs on the dumped
                                                   # lattice); same digest as `c4`, restartable
    python tests/golden/make_goldens.py chain N RHO STEPS LEG WORKDIR   # any size, same scheme

Every record holds the reference's init digest, final digest after `steps`
full steps, the vehicle counts and (where metrics=1) the observer-path sums
of moved vehicles and the last StepMetrics.
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_driver")

SMALL = [
    # SURVEY §8(c) golden table + BASELINE configs[0..1]
    dict(n=256, rho=0.3, seed=1, steps=1024, metrics=1),
    dict(n=256, rho=0.3, seed=42, steps=1024, metrics=1),
    dict(n=256, rho=0.3, seed=7, steps=1024, metrics=1),
    dict(n=1024, rho=0.38, seed=1, steps=4096, metrics=1),
    # extra coverage: non-multiple-of-32 sizes, both regimes, long runs
    dict(n=1000, rho=0.25, seed=3, steps=512, metrics=1),
    dict(n=777, rho=0.5, seed=5, steps=300, metrics=1),
    dict(n=2048, rho=0.35, seed=1, steps=256, metrics=1),
    dict(n=4096, rho=0.35, seed=2, steps=64, metrics=0),
]
BIG = [
    dict(n=8192, rho=0.25, seed=1, steps=10000, metrics=0),
    dict(n=8192, rho=0.5, seed=1, steps=10000, metrics=0),
]
HUGE = [
    dict(n=32768, rho=0.35, seed=1, steps=10000, metrics=0),
    dict(n=65536, rho=0.35, seed=1, steps=10000, metrics=0),
]


def name_of(c):
    return f"ref_n{c['n']}_rho{c['rho']}_seed{c['seed']}_steps{c['steps']}.json"


def run(c, force=False):
    out = os.path.join(HERE, name_of(c))
    if os.path.exists(out) and not force:
        print("exists", out)
        return
    args = [DRIVER, "golden"] + [f"{k}={v}" for k, v in c.items()] + ["backend=lanes"]
    print("running", " ".join(args), flush=True)
    res = subprocess.run(args, check=True, capture_output=True, text=True)
    rec = json.loads(res.stdout)
    rec["generator"] = "oracle/_ref/ref_driver (unmodified reference sources, lanes backend)"
    with open(out, "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)
    print("wrote", out, rec["final_digest"], flush=True)


# Phase-transition regimes (acceptance_main.cpp criteria 3/4):
# N=256, 4096 steps, seeds 1..10 at the free-flow and jamming densities. One
# combined file (not ref_*.json: those are single records).
REGIMES = [dict(n=256, rho=rho, seed=s, steps=4096, metrics=1) for rho in (0.25, 0.38)
           for s in range(1, 11)]


def run_regimes():
    out = os.path.join(HERE, "regimes_n256_steps4096.json")
    recs = []
    for c in REGIMES:
        args = [DRIVER, "golden"] + [f"{k}={v}" for k, v in c.items()] + ["backend=lanes"]
        print("running", " ".join(args), flush=True)
        r = json.loads(subprocess.run(args, check=True, capture_output=True, text=True).stdout)
        recs.append({k: r[k] for k in ("n", "rho", "seed", "steps", "init_digest", "final_digest",
                                       "sum_lr_moved", "sum_tb_moved", "regime")})
    with open(out, "w") as f:
        json.dump({"generator": "oracle/_ref/ref_driver (unmodified reference sources, lanes backend)",
                   "window": 64, "records": recs}, f, indent=1, sort_keys=True)
    print("wrote", out)


def run_chain(n, rho, seed, steps, leg, work):
    """One long golden as resumable legs of `leg` steps.

    Leg 0 is `ref_driver golden` (the reference's own init_grid, then `leg` steps); each
    later leg is `ref_driver file` on the previous leg's dumped interior. The reference
    stepping is a pure function of the lattice (engine.cpp:206-208), so the chained
    final digest equals an unbroken run's. Every leg's record is kept in the output as
    an intermediate checkpoint digest.
    """
    os.makedirs(work, exist_ok=True)
    log = os.path.join(work, "legs.jsonl")
    legs = []
    if os.path.exists(log):
        legs = [json.loads(l) for l in open(log) if l.strip()]
    done = len(legs) * leg
    while done < steps:
        out_bin = os.path.join(work, f"s{done + leg}.bin")
        if done == 0:
            args = [DRIVER, "golden", f"n={n}", f"rho={rho}", f"seed={seed}", f"steps={leg}",
                    "metrics=0", "backend=lanes", f"dump_final={out_bin}"]
        else:
            args = [DRIVER, "file", f"in={os.path.join(work, f's{done}.bin')}", f"n={n}",
                    f"steps={leg}", "metrics=0", "backend=lanes", f"dump_final={out_bin}"]
        print("running", " ".join(args), flush=True)
        rec = json.loads(subprocess.run(args, check=True, capture_output=True, text=True).stdout)
        rec["at_step"] = done + leg
        with open(log, "a") as f:
            f.write(json.dumps(rec) + "\n")
        legs.append(rec)
        if done > 0:
            os.remove(os.path.join(work, f"s{done}.bin"))
        done += leg
        print("leg", done, rec["final_digest"], flush=True)
    first, last = legs[0], legs[-1]
    out = {"n": n, "rho": rho, "seed": seed, "steps": steps, "backend": "lanes", "threads": 1,
           "k": first["k"], "init_digest": first["init_digest"], "final_digest": last["final_digest"],
           "lr_count": last["lr_count"], "tb_count": last["tb_count"], "init_s": first["init_s"],
           "run_s": sum(r["run_s"] for r in legs),
           "checkpoints": [{"step": r["at_step"], "digest": r["final_digest"]} for r in legs],
           "generator": ("oracle/_ref/ref_driver (unmodified reference sources, lanes backend), "
                         f"{len(legs)} chained legs of {leg} steps (make_goldens.py c4chain)")}
    path = os.path.join(HERE, name_of(dict(n=n, rho=rho, seed=seed, steps=steps)))
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path, out["final_digest"], flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "small"
    if which == "c4chain":
        run_chain(65536, 0.35, 1, 10000, 1000, sys.argv[2])
        sys.exit(0)
    if which == "chain":  # chain N RHO STEPS LEG WORKDIR (e.g. the weak-sweep sizes 23168, 46336)
        n, rho, steps, leg, work = sys.argv[2:7]
        run_chain(int(n), float(rho), 1, int(steps), int(leg), work)
        sys.exit(0)
    if which == "regimes":
        run_regimes()
        sys.exit(0)
    c4short = [dict(n=65536, rho=0.35, seed=1, steps=1000, metrics=0)]
    table = {"small": SMALL, "big": BIG, "huge": HUGE, "c3": HUGE[:1], "c4short": c4short,
             "c4": HUGE[1:]}[which]
    for c in table:
        run(c)
