#!/usr/bin/env python3
"""bench.py — BML step throughput on B200 (Gcell-updates/s), one JSON line on rank 0.

Metric (BASELINE.json): Gcell-updates/sec and % of HBM roofline vs the host-CPU
reference. 1 cell-update = one cell advanced by one full BML step (LR + TB phase).

A bench "step" = one reference-style run(): `steps` full BML steps of the whole
N x N lattice (the unit the reference's own `bml bench` times, tools/main.cpp:195-201).
Default workload = BASELINE configs[4], the metric's configuration: N=65536 (4 Gi
cells), rho=0.35, 10000 steps, seed 1. With --gpus g (torchrun, one rank per GPU) the
lattice is split into row bands of ceil(N/g) rows (the reference's only parallel
split, engine.cpp:131-137):
  --scaling strong (default)  N fixed: the literal configs[3]/[4] 1/2/4/8 sweep
  --scaling weak              configs[4]: the square weak sweep N = 23168 / 32768 /
                              46336 / 65536 at g = 1 / 2 / 4 / 8;
                              other workloads: ~g x the N=1 cells, side a multiple of 32
  parity    untimed, after the timed region: the lattice re-drawn from the reference
            RNG path and run for the golden's step count on the device; its grid_digest
            must equal the digest the UNMODIFIED reference produced
            (tests/golden/ref_*.json), and so must the e2e leg's downloaded result.

  value     device-resident throughput: lattice already in HBM, CUDA events on the
            launching stream around each bench step, L2 flushed (256 MiB write)
            between bench steps outside the events.
  e2e       the same through the C-ABI (include/bml_dev.h) with pinned HOST
            buffers: upload (H2D) + steps + download (D2H) per bench step.
  roofline  dominant kernel (step_block_kernel): algorithmic bytes 4 B per
            cell-update / its average launch time, vs the
            measured HBM copy bandwidth in MEASURED_PEAKS.json.
  cpu_baseline  the unmodified reference (oracle/_ref/ref_driver, its own bench
            method) on this host, bounded sample, rank 0 only. From N=4096 up it
            steps the device-drawn input lattice (digest-checked against the
            reference's own init digest) instead of repeating the reference's
            minutes-long init_grid.

--impl reference runs only the reference CPU implementation (best of `lanes` 1
thread and `parallel` with all host threads, after ONE reference init_grid) and
prints the same line shape.
"""
import argparse
import ctypes
import json
import math
import os
import tempfile
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
DATASHEET_HBM_GBS = 8000.0  # B200 datasheet HBM3e bandwidth per GPU

WORKLOADS = {
    # name: (n, rho, seed, steps, description)
    "c0": (256, 0.3, 1, 1024, "configs[0]: N=256 rho=0.3 1024 steps"),
    "c1": (1024, 0.38, 1, 4096, "configs[1]: N=1024 rho=0.38 4096 steps"),
    "c2ff": (8192, 0.25, 1, 10000, "configs[2]: N=8192 rho=0.25 10000 steps"),
    "c2jam": (8192, 0.5, 1, 10000, "configs[2]: N=8192 rho=0.5 10000 steps"),
    "c3": (32768, 0.35, 1, 10000, "configs[3]: N=32768 rho=0.35 10000 steps"),
    "c4": (65536, 0.35, 1, 10000, "configs[4]: N=65536 rho=0.35 10000 steps"),
}
DEVICE_INIT_N = 4096  # init_grid on the device from this side up (minutes on the host at 65536)
BYTES_PER_CELL_UPDATE = 4  # 1 B read + 1 B write per cell per phase
SQUARE_WEAK = {1: 23168, 2: 32768, 4: 46336, 8: 65536}  # SURVEY §8(d) item 5 (configs[4])
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def bench_n(workload, n1, world, scaling):
    """Lattice side for `world` ranks: fixed (strong) or the weak-scaling sweep."""
    if scaling == "strong" or world < 1:
        return n1
    if workload == "c4":
        if world in SQUARE_WEAK:
            return SQUARE_WEAK[world]
        return min(65536, int(round(23168 * math.sqrt(world) / 32.0)) * 32)
    from paper_1804_07981_b200.dist import weak_scaled_n

    return weak_scaled_n(n1, world)


def find_golden(n, rho, seed, steps):
    """The reference's own digests for (n, rho, seed): the record at `steps` if one
    is committed, else the longest one (None if there is none)."""
    best = None
    prefix = f"ref_n{n}_rho{rho}_seed{seed}_steps"
    if not os.path.isdir(GOLDEN_DIR):
        return None
    for name in os.listdir(GOLDEN_DIR):
        if not (name.startswith(prefix) and name.endswith(".json")):
            continue
        with open(os.path.join(GOLDEN_DIR, name)) as f:
            rec = json.load(f)
        rec["file"] = "tests/golden/" + name
        if rec["steps"] == steps:
            return rec
        if best is None or rec["steps"] > best["steps"]:
            best = rec
    return best


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) is polled every ~2 ms from a thread, so even a
    millisecond-scale timed region gets samples; falls back to nvidia-smi -lms.
    """

    REASONS = {  # nvmlClocksEventReason bits
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, rs))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = sorted({k for _, r in self.samples for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm for sm, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------- C-ABI (ctypes)
def load_abi():
    import paper_1804_07981_b200 as bml

    lib = ctypes.CDLL(bml.LIB_DEV)
    vp = ctypes.c_void_p
    lib.bml_dev_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    lib.bml_dev_destroy.argtypes = [vp]
    lib.bml_dev_upload.argtypes = [vp, vp, ctypes.c_size_t]
    lib.bml_dev_download.argtypes = [vp, vp, ctypes.c_size_t]
    lib.bml_dev_upload_async.argtypes = [vp, vp, ctypes.c_size_t]
    lib.bml_dev_download_async.argtypes = [vp, vp, ctypes.c_size_t]
    lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
    lib.bml_dev_set_stream.argtypes = [vp, vp]
    lib.bml_dev_sync.argtypes = [vp]
    lib.bml_dev_configure.argtypes = [vp, ctypes.c_int, ctypes.c_int]
    lib.bml_dev_enable_timing.argtypes = [vp, ctypes.c_int]
    lib.bml_dev_kernel_stats.argtypes = [vp, ctypes.POINTER(ctypes.c_int64),
                                         ctypes.POINTER(ctypes.c_double), ctypes.c_int]
    lib.bml_dev_info.argtypes = [vp] + [ctypes.POINTER(ctypes.c_int)] * 5 + [ctypes.POINTER(ctypes.c_size_t)]
    lib.bml_dev_last_launch.argtypes = [vp] + [ctypes.POINTER(ctypes.c_int)] * 3
    lib.bml_dev_last_kernel.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64)]
    lib.bml_dev_last_kernel_launch.argtypes = [vp] + [ctypes.POINTER(ctypes.c_int)] * 3
    lib.bml_dev_last_error.restype = ctypes.c_char_p
    return lib


def last_launch(abi, h):
    """Geometry of the dominant step kernel's last launch (not a run's short tail)."""
    ns, items, grid = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    abi_check(abi, abi.bml_dev_last_kernel_launch(h, ctypes.byref(ns), ctypes.byref(items), ctypes.byref(grid)),
              "last_kernel_launch")
    return {"strips": ns.value, "items": items.value, "ctas": grid.value}


def abi_check(lib, rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed rc={rc}: {lib.bml_dev_last_error().decode()}")


# ---------------------------------------------------------------- reference CPU arm
# Per kernel: ALU-pipe and issued warp-instructions per 32-cell stage (one lane,
# one step) of the innermost row loop, counted in the SASS of the built library
# (scripts/sass_inner_loop.py). The ALU pipe retires 2 and an SM
# issues 4 warp-instructions per clock, and a warp-instruction covers 32 lanes, so
# a bound is (2 or 4) / count x 1024 cell-updates per clock per SM.
KERNEL_MIX = {
    # 4 LOP3 + 2 funnel shifts (+ loop predicates); 1089 instructions / 96 stages
    "step_block_kernel": {"alu": 6.0, "issue": 11.34},
    # even/odd layout: 3.5 LOP3 + 1 funnel shift (+ loop overhead); 1571 / 168 stages
    "step_wide_kernel (even/odd layout)": {"alu": 4.6, "issue": 9.35},
    "resident_kernel": {"alu": 6.0, "issue": None},
}
KERNEL_NAMES = {1: "step_block_kernel", 2: "step_wide_kernel", 3: "step_wide_kernel (even/odd layout)",
                4: "step_split_kernel", 5: "resident_kernel"}


def last_kernel(abi, h):
    k, st = ctypes.c_int(), ctypes.c_int64()
    abi_check(abi, abi.bml_dev_last_kernel(h, ctypes.byref(k), ctypes.byref(st)), "last_kernel")
    return KERNEL_NAMES.get(k.value, "step_block_kernel")


def alu_roofline(kernel, achieved_gcups, resident_cluster, sm_max_mhz, sms=148):
    """The bound that actually limits the bit-plane kernels: the ALU
    pipe or instruction issue, whichever is lower for the kernel's SASS mix
    (KERNEL_MIX). The narrow kernel issues 6 ALU-pipe instructions per 32-cell
    stage (4 LOP3 + 2 funnel shifts; the ORs of disjoint planes go to the FMA
    pipe): 2/6 x 1024 = 341 cell-updates per clock per SM, below its issue bound.
    The even/odd-layout kernel needs 4.6 ALU but issues 9.35 instructions per
    stage, so issue binds: 4/9.35 x 1024 = 438. `achieved` is the dominant
    kernel's rate (its event-timed launches), over the SMs it runs on (the
    resident kernel: one cluster)."""
    used = resident_cluster if kernel == "resident_kernel" and resident_cluster else sms
    mhz = sm_max_mhz or 1965
    mix = KERNEL_MIX.get(kernel, KERNEL_MIX["step_block_kernel"])
    alu_peak = 2.0 / mix["alu"] * 1024 * used * mhz * 1e6 / 1e9
    issue_peak = 4.0 / mix["issue"] * 1024 * used * mhz * 1e6 / 1e9 if mix["issue"] else None
    binding = "issue" if issue_peak and issue_peak < alu_peak else "alu"
    peak = min(alu_peak, issue_peak) if issue_peak else alu_peak
    return {"bound": binding, "achieved": achieved_gcups, "peak": peak, "unit": "Gcell-updates/s",
            "frac": achieved_gcups / peak, "sms": used, "sm_mhz": mhz, "kernel": kernel,
            "alu_peak": alu_peak, "issue_peak": issue_peak,
            "alu_instructions_per_32_cell_stage": mix["alu"],
            "issued_instructions_per_32_cell_stage": mix["issue"]}


def cpu_sample_plan(n, steps, reps):
    """Bounded samples of the same workload for the reference CPU backends, as
    ref_driver `ladder` plan items backend:threads:steps:reps. lanes (1 thread, the
    reference's fastest path) gets `reps` reps of ~1-3 s; parallel (all host threads,
    scalar kernel) up to 3 reps; the paper's scalar ladder (halo, naive) one rep."""
    cells = n * n
    lanes_steps = max(1, min(steps, int(6e9 / cells)))
    par_steps = max(1, min(steps, int(1.5e9 / cells)))
    halo_steps = max(1, min(steps, int(1.5e8 / cells)))
    naive_steps = max(1, min(steps, int(0.8e8 / cells)))
    return [("lanes", 1, lanes_steps, reps), ("parallel", 0, par_steps, min(reps, 3)),
            ("halo", 1, halo_steps, 1), ("naive", 1, naive_steps, 1)]


def reference_ladder(n, rho, seed, steps, reps, input_path=None, expect_init=None):
    """ONE ref_driver process: one input lattice (the reference's own init_grid, or a
    digest-checked file), then the reference bench method per backend."""
    if not os.path.exists(REF_DRIVER):
        return None, "oracle/_ref/ref_driver not built"
    plan = ",".join(f"{b}:{t}:{st}:{r}" for b, t, st, r in cpu_sample_plan(n, steps, reps))
    cmd = [REF_DRIVER, "ladder", f"n={n}", f"rho={rho}", f"seed={seed}", f"plan={plan}"]
    if input_path:
        cmd.append(f"in={input_path}")
        if expect_init:
            cmd.append(f"expect_init={expect_init}")
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        return None, f"ref_driver ladder rc={out.returncode}: {out.stderr.strip()[:200]}"
    rec = json.loads(out.stdout)
    res = {}
    for r in rec["results"]:
        r["gcups"] = n * n * r["steps"] / r["mean_s"] / 1e9
        res[r["backend"]] = r
    res["best"] = res["lanes"] if res["lanes"]["gcups"] >= res["parallel"]["gcups"] else res["parallel"]
    res["input"] = {"source": rec["init_source"], "init_s": rec["init_s"], "digest": rec["init_digest"]}
    return res, None


def cpu_baseline_record(res, steps, reps):
    best = res["best"]
    inp = res["input"]
    where = ("reference init_grid" if inp["source"] == "init_grid" else
             "device-drawn input lattice, grid_digest checked equal to the reference init digest")
    return {"value": best["gcups"], "unit": "Gcell-updates/s", "cores": best["threads"],
            "kind": "reference",
            "sample": (f"{best['backend']} backend, {best['steps']} of {steps} steps x {best['reps']} reps, "
                       f"reference bench method (tools/main.cpp:195-214); input: {where}"),
            "host": cpu_model(), "hardware_concurrency": best["hardware_concurrency"],
            "lane_width": best["lane_width"],
            "lanes_1thread_gcups": res["lanes"]["gcups"],
            "parallel_all_threads_gcups": res["parallel"]["gcups"],
            "halo_1thread_gcups": res["halo"]["gcups"],
            "naive_1thread_gcups": res["naive"]["gcups"],
            "parallel_threads": res["parallel"]["threads"],
            "input_init_s": inp["init_s"], "input_digest": inp["digest"]}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_impl(args, wl):
    n1, rho, seed, steps, desc = wl
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    n = bench_n(args.workload, n1, max(world, args.gpus), args.scaling)
    reps = max(1, args.steps)
    res, err = reference_ladder(n, rho, seed, steps, reps)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": err}))
        return
    best = res["best"]
    value = best["gcups"]
    golden = find_golden(n, rho, seed, steps)
    line = {
        "impl": "reference",
        "metric": "Gcell-updates/sec",
        "value": value,
        "unit": "Gcell-updates/s",
        "n_gpus": args.gpus,
        "steps": reps,
        "warmup": 0,
        "ms_per_step": best["mean_s"] * 1e3 * steps / best["steps"],
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (reference init_grid seed)",
        "config": {"workload": config_block(args, desc, n, rho, seed, steps, args.gpus)["workload"],
                   "n": n, "rho": rho, "seed": seed, "steps_per_run": steps, "scaling_mode": args.scaling,
                   "parallelism": "host CPU (reference backends; rank 0 only)"},
        "cpu_baseline": cpu_baseline_record(res, steps, reps),
        "e2e": {"value": value, "unit": "Gcell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "input_check": {"init_digest": res["input"]["digest"],
                        "golden_init_digest": golden["init_digest"] if golden else None,
                        "match": (res["input"]["digest"] == golden["init_digest"]) if golden else None},
    }
    print(json.dumps(line))


def config_block(args, desc, n, rho, seed, steps, world):
    wl = desc if n == WORKLOADS[args.workload][0] else desc + f" ({args.scaling}-scaled to N={n})"
    return {"workload": wl, "n": n, "rho": rho, "seed": seed, "steps_per_run": steps,
            "scaling_mode": args.scaling,
            "parallelism": "single GPU" if world == 1 else
            f"row bands of ceil(N/{world}) rows x{world}, NVLink peer ghost rows",
            "l2": "flushed (256 MiB write) between bench steps",
            "block_steps": args.block, "strip_rows": args.strip,
            "layout": "bit-planes, 2 bits/cell"}


# ---------------------------------------------------------------- b200 arm
def run_b200(args, wl):
    import torch
    import paper_1804_07981_b200 as bml

    n1, rho, seed, steps, desc = wl
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        return run_b200_multi(args, wl)
    n = bench_n(args.workload, n1, 1, args.scaling)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    # reference RNG path (untimed input generation); large lattices draw it on the
    # device (bml_dev_init_random, bit-identical to the host shuffle)
    t_init = time.perf_counter()
    grid = bml.init_grid(n, rho, seed, on_device=n >= DEVICE_INIT_N)
    t_init = time.perf_counter() - t_init
    lat = bml.DeviceLattice(n)
    lat.configure(block_steps=args.block, strip_rows=args.strip)
    stream = torch.cuda.Stream(device=dev)
    lat.set_stream(stream.cuda_stream)
    lat.upload(grid)
    abi = load_abi()
    h = ctypes.c_void_p(lat.handle())
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    # warm-up
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            lat.step(steps)
    stream.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    abi_check(abi, abi.bml_dev_kernel_stats(h, None, None, 1), "kernel_stats reset")
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.fill_(i & 0xFF)  # evict the lattice from L2 between bench steps
                starts[i].record(stream)
                lat.step(steps)
                ends[i].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    launches = ctypes.c_int64()
    kms = ctypes.c_double()
    abi_check(abi, abi.bml_dev_kernel_stats(h, ctypes.byref(launches), ctypes.byref(kms), 1),
              "kernel_stats")
    timed_launches = launches.value  # kernels launched inside the timed region
    # Roofline pass (outside the timed region): the same bench steps again with CUDA
    # events around every step-kernel launch, for the dominant kernel's average
    # launch duration. Kept separate so per-launch events do not perturb `value`.
    abi_check(abi, abi.bml_dev_enable_timing(h, 1), "enable_timing")
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            lat.step(steps)
    stream.synchronize()
    abi_check(abi, abi.bml_dev_kernel_stats(h, ctypes.byref(launches), ctypes.byref(kms), 1),
              "kernel_stats")
    abi_check(abi, abi.bml_dev_enable_timing(h, 0), "enable_timing")
    per_step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(per_step_ms)
    cell_updates = n * n * steps * args.steps
    value = cell_updates / (total_ms / 1e3) / 1e9

    peak, peak_src = measured_peaks()
    avg_launch_ms = kms.value / max(1, launches.value)
    bytes_per_launch = BYTES_PER_CELL_UPDATE * n * n * steps * args.steps / max(1, launches.value)
    achieved = bytes_per_launch / (avg_launch_ms / 1e3) / 1e9
    kernel_share = kms.value / total_ms if total_ms else None

    kernel = "resident_kernel" if lat.resident_cluster > 0 else last_kernel(abi, h)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tpath) and n == n1:
        with open(tpath) as f:
            t = json.load(f)
        if t.get("kernel", "").startswith(kernel):
            traffic = t.get("dram_bytes_per_launch")
            traffic_src = t.get("source")

    # parity (untimed): the lattice re-drawn from the reference RNG path on the
    # device, run for the golden's step count, digested on the device
    golden = find_golden(n, rho, seed, steps)
    parity = parity_check(bml, lat, n, rho, seed, golden)

    # e2e through the C-ABI with pinned host buffers: pipelined over two handles
    # (the contract's e2e), and one synchronous call sequence at a time
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e_pipelined(abi, torch, bml, grid, n, steps, args, golden)
        e2e["sync"] = run_e2e(abi, torch, bml, grid, n, steps, args, golden)

    cpu = None
    if not args.no_cpu and rank == 0:
        cpu = cpu_baseline_b200_arm(grid, n, rho, seed, steps, golden)
    del grid

    line = {
        "metric": "Gcell-updates/sec",
        "value": value,
        "unit": "Gcell-updates/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic: reference init_grid(n, rho, seed) lattice",
        "config": config_block(args, desc, n, rho, seed, steps, 1),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": kernel, "peak_source": peak_src,
                     "frac_datasheet": achieved / DATASHEET_HBM_GBS,  # also vs 8 TB/s
                     "binding_bound": "alu pipe or instruction issue, whichever roofline_alu.bound names: "
                                      "temporal blocking keeps DRAM traffic at ~1/14-1/16 of the 4 B/cell-update "
                                      "algorithmic figure",
                     "launch_geometry": last_launch(abi, h) if kernel.startswith("step_") else None,
                     "resident_cluster": lat.resident_cluster,
                     "algorithmic_bytes_per_cell_update": BYTES_PER_CELL_UPDATE,
                     "launches": launches.value, "avg_launch_us": avg_launch_ms * 1e3,
                     "kernel_share_of_step": kernel_share},
        "roofline_alu": alu_roofline(kernel, cell_updates / (kms.value / 1e3) / 1e9,
                                     lat.resident_cluster, clocks.summary().get("sm_max_mhz")),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "parity": parity,
        # step kernels (kernel_stats) + the even/odd layout's two in-place
        # conversion kernels per bml_dev_step call when that kernel ran
        "gpu_launches": timed_launches + (2 * args.steps if "even/odd" in kernel else 0),
        "init": {"s": t_init, "where": "device" if n >= DEVICE_INIT_N else "host",
                 "note": "init_grid incl. readback into a host Grid; untimed input generation"},
        "wall_s": wall,
        "clocks": clocks.summary(),
        "gpu": torch.cuda.get_device_name(dev),
    }
    print(json.dumps(line))


def parity_check(bml, lat, n, rho, seed, golden):
    """Device digest after an untimed re-draw + golden-length run vs the reference's."""
    if golden is None:
        return {"golden": None, "match": None, "note": f"no reference golden committed for n={n}"}
    lat.init_random(rho, seed)
    init_d = lat.digest()
    lat.step(golden["steps"])
    final_d = lat.digest()
    ok = (f"0x{init_d:016x}" == golden["init_digest"] and f"0x{final_d:016x}" == golden["final_digest"])
    return {"golden": golden["file"], "steps": golden["steps"], "init_digest": f"0x{init_d:016x}",
            "final_digest": f"0x{final_d:016x}", "expected_final": golden["final_digest"], "match": ok}


def cpu_baseline_b200_arm(grid, n, rho, seed, steps, golden):
    """Reference CPU sample for this line (rank 0, N=1). Large lattices hand the
    reference the device-drawn input (checked against the reference init digest)
    rather than a second minutes-long host init_grid."""
    path = None
    try:
        expect = None
        if n >= DEVICE_INIT_N:
            fd, path = tempfile.mkstemp(prefix="bml_in_", suffix=".bin")
            with os.fdopen(fd, "wb") as f:
                f.write(grid.to_bytes())
            expect = golden["init_digest"] if golden else f"0x{grid.digest():016x}"
        res, err = reference_ladder(n, rho, seed, steps, 3, input_path=path, expect_init=expect)
    finally:
        if path:
            os.unlink(path)
    if not res:
        return {"value": None, "unavailable": err}
    return cpu_baseline_record(res, steps, 3)


def check_result(bml, n, data, golden, steps):
    """The downloaded lattice's host grid_digest against the reference golden."""
    if golden is None or golden["steps"] != steps:
        return None
    d = bml.Grid.from_bytes(n, data).digest()
    check = {"golden": golden["file"], "digest": f"0x{d:016x}", "match": f"0x{d:016x}" == golden["final_digest"]}
    assert check["match"], f"e2e result differs from the reference golden: {check}"
    return check


def run_e2e_pipelined(abi, torch, bml, grid, n, steps, args, golden):
    """Bench steps as independent jobs through the asynchronous C-ABI: job i uploads
    its input from pinned host memory, runs `steps` steps and downloads its result,
    all on handle i % 2's stream, so one job's PCIe transfers (and pack/unpack)
    overlap the other job's stepping. Every job's H2D and D2H are inside the timed
    region (host clock around all jobs, both streams synchronised at the end)."""
    vp = ctypes.c_void_p
    hs = [vp(), vp()]
    dev = torch.cuda.current_device()
    try:
        for h in hs:
            abi_check(abi, abi.bml_dev_create(n, dev, ctypes.byref(h)), "create")
            abi_check(abi, abi.bml_dev_configure(h, args.block, args.strip), "configure")
        host_in = torch.frombuffer(bytearray(grid.to_bytes()), dtype=torch.uint8).pin_memory()
        host_out = [torch.empty(n * n, dtype=torch.uint8).pin_memory() for _ in hs]

        def job(i):
            h = hs[i % 2]
            abi_check(abi, abi.bml_dev_upload_async(h, vp(host_in.data_ptr()), n), "upload_async")
            abi_check(abi, abi.bml_dev_step(h, steps, None, None, None, None), "step")
            abi_check(abi, abi.bml_dev_download_async(h, vp(host_out[i % 2].data_ptr()), n), "download_async")

        for i in range(max(2, args.warmup)):
            job(i)
        for h in hs:
            abi_check(abi, abi.bml_dev_sync(h), "sync")
        t0 = time.perf_counter()
        for i in range(args.steps):
            job(i)
        for h in hs:
            abi_check(abi, abi.bml_dev_sync(h), "sync")
        total = time.perf_counter() - t0
        check = check_result(bml, n, bytes(host_out[(args.steps - 1) % 2].numpy()), golden, steps)
        return {"value": n * n * steps * args.steps / total / 1e9, "unit": "Gcell-updates/s",
                "h2d_bytes_per_step": n * n, "d2h_bytes_per_step": n * n,
                "ms_per_step": total / args.steps * 1e3,
                "path": "C-ABI bml_dev_upload_async/step/download_async, two handles on two streams, "
                        "pinned host buffers, jobs pipelined (transfers of one overlap stepping of the other)",
                "result_check": check}
    finally:
        for h in hs:
            if h:
                abi.bml_dev_destroy(h)


def run_e2e(abi, torch, bml, grid, n, steps, args, golden):
    vp = ctypes.c_void_p
    h = vp()
    abi_check(abi, abi.bml_dev_create(n, torch.cuda.current_device(), ctypes.byref(h)), "create")
    try:
        abi_check(abi, abi.bml_dev_configure(h, args.block, args.strip), "configure")
        host_in = torch.frombuffer(bytearray(grid.to_bytes()), dtype=torch.uint8).pin_memory()
        host_out = torch.empty(n * n, dtype=torch.uint8).pin_memory()
        for _ in range(max(1, args.warmup)):
            abi_check(abi, abi.bml_dev_upload(h, vp(host_in.data_ptr()), n), "upload")
            abi_check(abi, abi.bml_dev_step(h, steps, None, None, None, None), "step")
            abi_check(abi, abi.bml_dev_download(h, vp(host_out.data_ptr()), n), "download")
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            abi_check(abi, abi.bml_dev_upload(h, vp(host_in.data_ptr()), n), "upload")
            abi_check(abi, abi.bml_dev_step(h, steps, None, None, None, None), "step")
            abi_check(abi, abi.bml_dev_download(h, vp(host_out.data_ptr()), n), "download")
            times.append(time.perf_counter() - t0)
        # what was timed is checked against the UNMODIFIED reference: the downloaded
        # lattice's host grid_digest equals the golden (when one exists at `steps`)
        check = check_result(bml, n, bytes(host_out.numpy()), golden, steps)
        total = sum(times)
        return {"value": n * n * steps * len(times) / total / 1e9, "unit": "Gcell-updates/s",
                "h2d_bytes_per_step": n * n, "d2h_bytes_per_step": n * n,
                "ms_per_step": total / len(times) * 1e3,
                "path": "C-ABI bml_dev_upload/step/download, pinned host buffers, one call at a time",
                "result_check": check}
    finally:
        abi.bml_dev_destroy(h)


def run_b200_multi(args, wl):
    """One process per GPU (torchrun): each rank owns a row band of ceil(N/g) rows of
    the lattice (N fixed for --scaling strong, the square weak sweep for weak);
    neighbours exchange ghost rows inside the step kernel over NVLink (CUDA IPC peer
    stores + flags). torch.distributed only bootstraps and reduces timings."""
    import torch
    import torch.distributed as dist

    import paper_1804_07981_b200 as bml
    from paper_1804_07981_b200.dist import BandLattice, combine_digest

    n1, rho, seed, steps, desc = wl
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    local = local % ndev  # more ranks than GPUs only in tests: ranks share a GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    shared_gpu = world > ndev
    if shared_gpu:  # NCCL refuses two ranks on one GPU; the data path does not use it anyway
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if shared_gpu else dev
    n = bench_n(args.workload, n1, world, args.scaling)
    band = BandLattice(n, rank, world, local, block_steps=args.block, strip_rows=args.strip)
    # each rank draws its rows of the same reference-RNG lattice on its own GPU; ranks
    # sharing one GPU take turns (the draw needs ~16 B per cell of scratch)
    for turn in range(world if shared_gpu else 1):
        if not shared_gpu or turn == rank:
            band.init_random(rho, seed)
        if shared_gpu:
            dist.barrier()
    band.exchange_halos()
    band_cells = band.download_rows()  # host copy of the input, for the e2e leg
    dist.barrier()  # every band's first ghost rows are published before anyone steps
    stream = torch.cuda.Stream(device=dev)
    band.set_stream(stream.cuda_stream)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            band.step(steps)
    stream.synchronize()
    band.kernel_stats(reset=True)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.fill_(i & 0xFF)
                starts[i].record(stream)
                band.step(steps)
                ends[i].record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        wall = time.perf_counter() - t0
    timed_launches, _ = band.kernel_stats(reset=True)
    band_kernel = KERNEL_NAMES.get(band.last_kernel(), "step_block_kernel")
    # roofline pass, outside the timed region: per-launch CUDA events
    band.enable_timing(True)
    dist.barrier()
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            band.step(steps)
    stream.synchronize()
    launches, kms = band.kernel_stats(reset=True)
    band.enable_timing(False)
    my_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([my_ms, kms / max(1, launches)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, avg_launch_ms = float(t[0]), float(t[1])
    value = n * n * steps * args.steps / (total_ms / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    cells_per_launch = band.rows * n * steps * args.steps / max(1, launches)
    achieved = BYTES_PER_CELL_UPDATE * cells_per_launch / (avg_launch_ms / 1e3) / 1e9
    # e2e: each rank uploads its band from pinned host memory, steps, downloads
    host_in = torch.frombuffer(bytearray(band_cells), dtype=torch.uint8).pin_memory()
    e2e_times = []
    for i in range(args.steps):
        dist.barrier()
        t1 = time.perf_counter()
        band.upload_rows(host_in.data_ptr())
        band.exchange_halos()
        band.step(steps)
        band.download_rows()
        e2e_times.append(time.perf_counter() - t1)
    et = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    # whole-torus digest and conservation after the last e2e run (device-side)
    segs = [None] * world
    dist.all_gather_object(segs, (rank, band.digest_segment(), band.counts()))
    segs.sort()
    digest = combine_digest([sg for _, sg, _ in segs])
    k_total = sum(lr for _, _, (lr, _) in segs), sum(tb for _, _, (_, tb) in segs)
    conserved = k_total == (bml.vehicles_per_species(n, rho),) * 2
    if rank == 0:
        golden = find_golden(n, rho, seed, steps)
        match = None
        if golden is not None and golden["steps"] == steps:
            match = f"0x{digest:016x}" == golden["final_digest"]
        line = {
            "metric": "Gcell-updates/sec", "value": value, "unit": "Gcell-updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u8",
            "data": "synthetic: reference init_grid(n, rho, seed) lattice",
            "config": dict(config_block(args, desc, n, rho, seed, steps, world), shared_gpu=shared_gpu),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "kernel": band_kernel,
                         "peak_source": peak_src, "launches_per_rank": launches,
                         "frac_datasheet": achieved / DATASHEET_HBM_GBS,  # per rank, like frac
                         "binding_bound": "alu (per rank; see the N=1 line's roofline_alu)",
                         "avg_launch_us": avg_launch_ms * 1e3},
            "cpu_baseline": None,
            "e2e": {"value": n * n * steps * args.steps / float(et[0]) / 1e9, "unit": "Gcell-updates/s",
                    "h2d_bytes_per_step": n * n, "d2h_bytes_per_step": n * n},
            # step kernels + the even/odd layout's 4 conversion kernels (own rows and
            # ghost rows, in and out) per rank and bml_dev_step call when it ran
            "gpu_launches": (timed_launches + (4 * args.steps if "even/odd" in band_kernel else 0)) * world,
            "wall_s": wall, "clocks": clocks.summary(),
            "parity": {"digest": f"0x{digest:016x}", "vehicles": list(k_total), "conserved": conserved,
                       "steps": steps, "golden": golden["file"] if golden else None,
                       "expected_final": golden["final_digest"] if golden and golden["steps"] == steps
                       else None, "match": match,
                       "note": "grid_digest of init_grid(n, rho, seed) after `steps` steps (the last e2e "
                               "run), combined on rank 0 from the bands' device digest segments"},
        }
        print(json.dumps(line))
    band.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="N>1: fixed N split into row bands (strong) or the weak sweep")
    ap.add_argument("--block", type=int, default=16, help="steps fused per launch / resident ghost depth")
    ap.add_argument("--strip", type=int, default=0, help="streaming-kernel rows per strip (0 = auto)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_impl(args, wl)
    else:
        run_b200(args, wl)


if __name__ == "__main__":
    main()
