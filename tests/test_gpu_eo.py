"""The even/odd-layout streaming kernel (bml_dev_set_variant 6; the default bare-loop
path once measured faster): every 64-cell group is held as its even
cells then its odd cells, converted in place around a bare-loop run of a single band.
Bit-exact with the oracle and with the unmodified reference's goldens, including the
column windows that wrap the torus seam, runs with a narrow-kernel tail (steps not a
multiple of 14), runs below the conversion threshold, and sizes the layout does not
cover (n % 64 != 0), which must fall back to the 32-cell kernel."""
import ctypes
import json
import os

import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def set_variant(gpu, lat, v, band=0):
    lib = ctypes.CDLL(gpu.LIB_DEV)
    lib.bml_dev_set_variant.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert lib.bml_dev_set_variant(ctypes.c_void_p(lat.handle(band)), v) == 0


def last_launch(gpu, lat):
    lib = ctypes.CDLL(gpu.LIB_DEV)
    lib.bml_dev_last_launch.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int)] * 3
    ns, items, grid = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert lib.bml_dev_last_launch(ctypes.c_void_p(lat.handle()), ctypes.byref(ns), ctypes.byref(items),
                                   ctypes.byref(grid)) == 0
    return ns.value, items.value, grid.value


# W = n/32 words per row: 64 (two windows, both wrap), 66 (a 6-word last window),
# 128, 192 (four windows), 258 (n = 8256, five windows, the last nearly empty)
@pytest.mark.parametrize("n,steps", [(2048, 56), (2048, 61), (2112, 70), (4096, 57), (6144, 84),
                                     (8256, 60)])
def test_eo_matches_oracle(gpu, oracle, n, steps):
    cells = oracle.init_grid(n, 0.36, n + steps)
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, 6)
    lat.upload(gpu.Grid.from_bytes(n, cells))
    lat.step(steps)
    assert lat.download().to_bytes() == oracle.run(n, cells, steps)


@pytest.mark.parametrize("rho", [0.05, 0.5, 0.9])
def test_eo_densities(gpu, oracle, rho):
    n, steps = 2048, 112
    cells = oracle.init_grid(n, rho, 3)
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, 6)
    lat.upload(gpu.Grid.from_bytes(n, cells))
    lat.step(steps)
    assert lat.download().to_bytes() == oracle.run(n, cells, steps)


@pytest.mark.parametrize("n", [2080, 2000, 1024])
def test_eo_falls_back_where_the_layout_does_not_apply(gpu, oracle, n):
    """n % 64 != 0 (odd word count, or a seam), or a resident lattice: same results."""
    cells = oracle.init_grid(n, 0.35, 9)
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, 6)
    lat.upload(gpu.Grid.from_bytes(n, cells))
    lat.step(70)
    assert lat.download().to_bytes() == oracle.run(n, cells, 70)


def test_eo_short_runs_and_repeated_calls(gpu, oracle):
    """Calls below the conversion threshold (narrow kernel) interleaved with long
    ones: the layout is converted back after every call."""
    n = 4096
    cells = oracle.init_grid(n, 0.38, 21)
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, 6)
    lat.upload(gpu.Grid.from_bytes(n, cells))
    total = 0
    for s in (3, 56, 1, 100, 55, 14 * 5):
        lat.step(s)
        total += s
    assert lat.download().to_bytes() == oracle.run(n, cells, total)
    assert lat.counts() == oracle.counts(n, cells)


@pytest.mark.parametrize("n,steps", [(2048, 60), (4096, 101)])
@pytest.mark.parametrize("strict", [False, True])
def test_eo_metrics_match_oracle(gpu, oracle, n, steps, strict):
    """Metrics calls run the even/odd kernel's counting instantiations (12 steps per
    launch; moved counts and the census are popcounts, so the layout does not
    change them), then a narrow tail."""
    cells = oracle.init_grid(n, 0.4, 5)
    _, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, 6)
    lat.set_census(strict)
    lat.upload(gpu.Grid.from_bytes(n, cells))
    ms = lat.step_with_metrics(steps)
    assert [m.lr_moved for m in ms] == lm and [m.tb_moved for m in ms] == tm
    assert [m.lr_count for m in ms] == lc and [m.tb_count for m in ms] == tc


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["ref_n8192_rho0.25_seed1_steps10000.json",
                                  "ref_n8192_rho0.5_seed1_steps10000.json",
                                  "ref_n32768_rho0.35_seed1_steps10000.json",
                                  "ref_n23168_rho0.35_seed1_steps10000.json",
                                  "ref_n46336_rho0.35_seed1_steps10000.json",
                                  "ref_n65536_rho0.35_seed1_steps1000.json",
                                  "ref_n65536_rho0.35_seed1_steps10000.json"])
def test_eo_reference_goldens(gpu, name):
    """Fully on the device (init -> steps -> digest), against the unmodified
    reference; chained goldens also at every checkpoint."""
    g = _golden(name)
    lat = gpu.DeviceLattice(g["n"])
    set_variant(gpu, lat, 6)
    lat.init_random(g["rho"], g["seed"])
    assert f"0x{lat.digest():016x}" == g["init_digest"]
    done = 0
    for cp in g.get("checkpoints", []):
        lat.step(cp["step"] - done)
        done = cp["step"]
        assert f"0x{lat.digest():016x}" == cp["digest"], cp
    lat.step(g["steps"] - done)
    assert f"0x{lat.digest():016x}" == g["final_digest"]
    assert lat.counts() == (g["lr_count"], g["tb_count"])


def last_kernel(gpu, lat):
    lib = ctypes.CDLL(gpu.LIB_DEV)
    lib.bml_dev_last_kernel.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_int64)]
    k, st = ctypes.c_int(), ctypes.c_int64()
    assert lib.bml_dev_last_kernel(ctypes.c_void_p(lat.handle()), ctypes.byref(k), ctypes.byref(st)) == 0
    return k.value, st.value


@pytest.mark.parametrize("n,steps,kernel,kernel_steps", [
    (32768, 60, 3, 56),   # automatic: the even/odd kernel from W >= 640 words (4 tail steps narrow)
    (23168, 70, 3, 70),   # the weak sweep's 1-GPU size (W = 724)
    (16384, 60, 1, 60),   # below: the narrow kernel
    (32768, 40, 1, 40),   # shorter than the conversion threshold: narrow
    (1024, 60, 5, 60),    # resident
])
def test_automatic_kernel_choice(gpu, n, steps, kernel, kernel_steps):
    lat = gpu.DeviceLattice(n)
    lat.init_random(0.35, 1)
    lat.step(steps)
    assert last_kernel(gpu, lat) == (kernel, kernel_steps)


@pytest.mark.parametrize("strict,want", [(True, 21), (False, 32)])
def test_eo_census_reports_the_fault(gpu, strict, want):
    """A vehicle removed after step 20 of a 150-step metrics call: the call splits at
    the fault, the remaining 130 steps run the even/odd kernel (12-step launches);
    strict census reports step 21, the launch-boundary census step 20 + 12."""
    import re

    n = 2048
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, 6)
    lat.set_census(strict)
    g = gpu.init_grid(n, 0.3, 4)
    lat.upload(g)
    i = g.to_bytes().index(1)
    lat.debug_fault(20, *divmod(i, n))
    with pytest.raises(RuntimeError) as ei:
        lat.step_with_metrics(150)
    m = re.search(r"conservation violated at step (\d+) of (\d+)", str(ei.value))
    assert m and int(m.group(1)) == want, str(ei.value)


def test_dominant_kernel_launch_geometry(gpu):
    """bml_dev_last_kernel_launch reports the even/odd launches of a 60-step run at
    N=32768 (65 strips x 18 windows), not the 4-step narrow tail launched last."""
    lib = ctypes.CDLL(gpu.LIB_DEV)
    for f in ("bml_dev_last_kernel_launch", "bml_dev_last_launch"):
        getattr(lib, f).argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int)] * 3
    lat = gpu.DeviceLattice(32768)
    lat.init_random(0.35, 1)
    lat.step(60)
    h = ctypes.c_void_p(lat.handle())
    dom = [ctypes.c_int() for _ in range(3)]
    last = [ctypes.c_int() for _ in range(3)]
    assert lib.bml_dev_last_kernel_launch(h, *[ctypes.byref(x) for x in dom]) == 0
    assert lib.bml_dev_last_launch(h, *[ctypes.byref(x) for x in last]) == 0
    assert last_kernel(gpu, lat) == (3, 56)
    assert dom[1].value == dom[0].value * 18 and dom[2].value == 148
    assert [x.value for x in dom] != [x.value for x in last]
