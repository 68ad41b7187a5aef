"""Per-step vehicle conservation (the reference's check in run(), src/engine.cpp:219-224),
measured inside the step kernels, exercised with the fault-injection test hook
(bml_dev_debug_fault: a cell is toggled between two launches of one bml_dev_step call).

- strict census (bml_dev_set_census(1)) and the cluster-resident kernel count after
  EVERY step, so a fault applied after step S is reported at step S+1 — the step the
  reference's run() throws at for a kernel that lost a vehicle while computing it;
- the default census of the streaming kernel is taken after each launch's last step,
  so the same fault is reported at the next launch boundary;
- run()/simulate deliver the steps before the violation, then raise.
"""
import re

import pytest

pytestmark = pytest.mark.gpu


def lattice_with(gpu, n, cells):
    """n x n lattice from {(row, col): value}."""
    data = bytearray(n * n)
    for (r, c), v in cells.items():
        data[r * n + c] = v
    return gpu.Grid.from_bytes(n, bytes(data))


def violation_step(exc):
    m = re.search(r"conservation violated at step (\d+) of (\d+)", str(exc))
    assert m, str(exc)
    return int(m.group(1))


def first_lr_cell(grid):
    data = grid.to_bytes()
    i = data.index(1)
    return divmod(i, grid.n)


@pytest.mark.parametrize("resident", [1, 0])
def test_strict_census_reports_the_exact_step(gpu, resident):
    n = 256
    grid = gpu.init_grid(n, 0.3, 1)
    lat = gpu.DeviceLattice(n)
    lat.set_resident(resident)
    lat.set_census(True)
    lat.upload(grid)
    lat.step(5)
    r, c = first_lr_cell(lat.download())
    lat.debug_fault(7, r, c)  # the LR vehicle at (r, c) vanishes after step 7 of the call
    with pytest.raises(RuntimeError) as ei:
        lat.step_with_metrics(20)
    assert violation_step(ei.value) == 8


def test_resident_kernel_census_is_per_step_by_default(gpu):
    n = 256
    lat = gpu.DeviceLattice(n)
    lat.upload(gpu.init_grid(n, 0.3, 1))
    r, c = first_lr_cell(lat.download())
    lat.debug_fault(3, r, c)
    with pytest.raises(RuntimeError) as ei:
        lat.step_with_metrics(40)
    assert lat.resident_cluster > 0
    assert violation_step(ei.value) == 4


def test_boundary_census_reports_the_next_launch_boundary(gpu):
    n = 256
    lat = gpu.DeviceLattice(n)
    lat.set_resident(0)  # streaming kernel, census after each launch's last step
    lat.upload(gpu.init_grid(n, 0.3, 1))
    r, c = first_lr_cell(lat.download())
    lat.debug_fault(7, r, c)
    with pytest.raises(RuntimeError) as ei:
        lat.step_with_metrics(20)
    # launches: steps 1-7 split 4+2+1 at the fault, then 8 (steps 8-15), 4, 1:
    # the first census after the fault is the one after step 15
    assert violation_step(ei.value) == 15


def test_self_restoring_fault_is_caught_only_per_step(gpu):
    """One LR vehicle in free flow: a second one appears after step 3 and is removed
    after step 5 (it moved two cells right). The counts differ after steps 4 and 5 only;
    the per-step census catches it at step 4."""
    n = 64
    grid = lattice_with(gpu, n, {(0, 0): 1})
    for strict, resident in ((True, 0), (False, 1)):
        lat = gpu.DeviceLattice(n)
        lat.set_resident(resident)
        lat.set_census(strict)
        lat.upload(grid)
        lat.debug_fault(3, 32, 40)  # Empty -> LR
        lat.debug_fault(5, 32, 42)  # LR -> Empty (the same vehicle, two steps on)
        with pytest.raises(RuntimeError) as ei:
            lat.step_with_metrics(12)
        assert violation_step(ei.value) == 4
    # without a fault nothing is reported, and every census equals the initial count
    lat = gpu.DeviceLattice(n)
    lat.set_resident(0)
    lat.upload(grid)
    ms = lat.step_with_metrics(40)
    assert all((m.lr_count, m.tb_count) == (1, 0) for m in ms)


def test_violation_metrics_are_returned_when_not_thrown(gpu):
    n = 128
    lat = gpu.DeviceLattice(n)
    lat.set_census(True)
    lat.upload(gpu.init_grid(n, 0.35, 2))
    lr0, tb0 = lat.counts()
    r, c = first_lr_cell(lat.download())
    lat.debug_fault(10, r, c)
    ms = lat.step_with_metrics(16, 1, False)
    assert [(m.lr_count, m.tb_count) for m in ms[:10]] == [(lr0, tb0)] * 10
    # any toggle changes one species by one: Empty -> LR, LR -> Empty or TB -> Empty
    off = (ms[10].lr_count - lr0, ms[10].tb_count - tb0)
    assert off in ((1, 0), (-1, 0), (0, -1))


def test_census_counts_match_the_oracle(gpu, oracle):
    """Strict and boundary census counts at every measured step against the oracle."""
    n, steps = 200, 37
    cells = oracle.init_grid(n, 0.4, 9)
    _, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
    for strict in (True, False):
        lat = gpu.DeviceLattice(n)
        lat.set_census(strict)
        lat.upload(gpu.Grid.from_bytes(n, cells))
        ms = lat.step_with_metrics(steps)
        assert [m.lr_moved for m in ms] == lm and [m.tb_moved for m in ms] == tm
        assert [m.lr_count for m in ms] == lc and [m.tb_count for m in ms] == tc


def test_partial_band_must_be_connected(gpu):
    import ctypes

    lib = ctypes.CDLL(gpu.LIB_DEV)
    vp = ctypes.c_void_p
    lib.bml_dev_create_band.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(vp)]
    lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
    lib.bml_dev_exchange_halos.argtypes = [vp]
    lib.bml_dev_destroy.argtypes = [vp]
    h = vp()
    assert lib.bml_dev_create_band(64, 0, 32, 0, ctypes.byref(h)) == 0
    try:
        assert lib.bml_dev_step(h, 4, None, None, None, None) == 1  # BML_EINVAL
        assert lib.bml_dev_exchange_halos(h) == 1
    finally:
        lib.bml_dev_destroy(h)


def _largest_block(remaining, cap=16):
    k = 16
    while k > 1 and (k > remaining or k > cap):
        k >>= 1
    return k


@pytest.mark.parametrize("case", range(24))
def test_census_fault_fuzz(gpu, case):
    """Seeded random lattices, step counts and fault steps: strict and resident census
    report the step right after the fault; the streaming launch-boundary census reports
    the end of the first launch after it (the call's launches split at the fault)."""
    import random

    rng = random.Random(1000 + case)
    n = rng.choice([64, 96, 128, 200, 256, 333, 512, 1024, 1056, 2048])
    steps = rng.randint(2, 90)
    fault = rng.randint(0, steps - 1)
    mode = rng.choice(["strict", "boundary"])
    resident = rng.choice([0, 1])
    lat = gpu.DeviceLattice(n)
    lat.set_resident(resident)
    lat.set_census(mode == "strict")
    lat.upload(gpu.init_grid(n, rng.choice([0.2, 0.35, 0.5]), rng.randint(1, 99)))
    lat.debug_fault(fault, rng.randrange(n), rng.randrange(n))
    with pytest.raises(RuntimeError) as ei:
        lat.step_with_metrics(steps)
    per_step = mode == "strict" or lat.resident_cluster > 0
    want = fault + 1 if per_step else fault + _largest_block(steps - fault)
    assert violation_step(ei.value) == want, (n, steps, fault, mode, resident, lat.resident_cluster)
