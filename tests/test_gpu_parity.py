"""GPU parity: the b200 engine (CUDA, sm_100a) against the oracle and the reference goldens.

Mirrors the reference's own engine tests (/root/reference/proj/tests/test_engine.cpp,
test_metrics.cpp, acceptance_main.cpp criteria 1/2/8/9) with the device backend
substituted. Integer CA: every comparison is bit-exact.
"""
import os
import random

import pytest

from conftest import load_goldens, rows_to_bytes

pytestmark = pytest.mark.gpu


def rand_lattice(seed, n):
    rng = random.Random(seed)
    return bytes(b % 3 for b in rng.randbytes(n * n))


def grid_of(bml, n, cells):
    return bml.Grid.from_bytes(n, cells)


# ----------------------------------------------------------- known answers
PHASE_CASES = [  # test_engine.cpp:63-81 / acceptance_main.cpp:234-241
    (">.>.", ".>.>"),
    (">>..", ">.>."),
    (">>>>", ">>>>"),
    (">v..", ">v.."),
]


@pytest.mark.parametrize("row,expected", PHASE_CASES)
def test_single_row_horizontal_phase(gpu, row, expected):
    bml = gpu
    g = bml.Grid.from_text(row + "\n....\n....\n....")
    out = bml.step_phase(g, bml.Phase.horizontal)
    assert out.to_text() == expected + "\n....\n....\n....\n"


def test_two_by_two_steps(gpu):  # test_engine.cpp:83-93
    bml = gpu
    assert bml.step(bml.Grid.from_text(">.\n.v"), 1).to_text() == ".>\n.v\n"
    assert bml.step(bml.Grid.from_text(">.\n.."), 2).to_text() == ">.\n..\n"
    assert bml.step(bml.Grid.from_text("..\n.."), 1).to_text() == "..\n..\n"


def test_self_neighbour_wrap(gpu):  # n=1, n=2 self-wrap cases
    bml = gpu
    assert bml.step(bml.Grid.from_text(">"), 5).to_text() == ">\n"
    assert bml.step(bml.Grid.from_text("v"), 5).to_text() == "v\n"
    assert bml.step(bml.Grid.from_text(">>\n.."), 3).to_text() == ">>\n..\n"


def test_never_blocked_orbit_metrics(gpu):  # test_metrics.cpp:62-75
    bml = gpu
    _, metrics = bml.simulate(bml.Grid.from_text(">...\n....\n.v..\n...."), 8)
    assert len(metrics) == 8
    for m in metrics:
        assert (m.lr_moved, m.tb_moved, m.mobility) == (1, 1, 1.0)


def test_vacuum_mobility_is_one(gpu):  # test_metrics.cpp:47-60
    bml = gpu
    _, metrics = bml.simulate(bml.Grid.from_text("\n".join(["." * 8] * 8)), 3)
    assert [m.mobility for m in metrics] == [1.0, 1.0, 1.0]
    assert bml.classify([m.mobility for m in metrics]) == bml.Regime.FreeFlow


# ----------------------------------------------------------- random lattices vs oracle
SIZES = list(range(1, 65)) + [65, 95, 96, 97, 127, 128, 129, 255, 256, 257, 480, 1000, 1023, 1024, 1025]


@pytest.mark.parametrize("n", SIZES)
def test_random_lattice_steps_match_oracle(gpu, oracle, n):
    bml = gpu
    cells = rand_lattice(1000 + n, n)
    steps = 1 + (n * 7) % 37 if n <= 257 else 9
    got = bml.step(grid_of(bml, n, cells), steps).to_bytes()
    assert got == oracle.run(n, cells, steps), f"n={n} steps={steps}"


@pytest.mark.parametrize("n", [1, 2, 3, 5, 16, 31, 32, 33, 63, 64, 100, 1024, 1030])
@pytest.mark.parametrize("phase", [0, 1])
def test_single_phase_and_moved_match_oracle(gpu, oracle, n, phase):
    bml = gpu
    cells = rand_lattice(7 * n + phase, n)
    lat = bml.DeviceLattice(n)
    lat.upload(grid_of(bml, n, cells))
    moved = lat.phase(bml.Phase.horizontal if phase == 0 else bml.Phase.vertical)
    got = lat.download().to_bytes()
    want = oracle.phase(n, cells, phase)
    assert got == want
    assert moved == oracle.moved(n, cells, want, phase)


@pytest.mark.parametrize("block", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("strip", [1, 3, 16, 64, 1000])
@pytest.mark.parametrize("n", [37, 64, 96, 1024, 1056])
def test_block_and_strip_configurations_agree(gpu, oracle, block, strip, n):
    bml = gpu
    cells = rand_lattice(n * 31 + block, n)
    steps = 45
    lat = bml.DeviceLattice(n)
    lat.configure(block_steps=block, strip_rows=strip)
    lat.upload(grid_of(bml, n, cells))
    lat.step(steps)
    assert lat.download().to_bytes() == oracle.run(n, cells, steps)


@pytest.mark.parametrize("n,steps", [(5, 50), (33, 40), (64, 33), (250, 20), (1024, 17)])
def test_simulate_metrics_match_oracle(gpu, oracle, n, steps):
    bml = gpu
    cells = oracle.init_grid(n, 0.35, n)
    final, metrics = bml.simulate(grid_of(bml, n, cells), steps)
    want, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
    assert final.to_bytes() == want
    assert [m.step for m in metrics] == list(range(1, steps + 1))
    assert [m.lr_moved for m in metrics] == lm
    assert [m.tb_moved for m in metrics] == tm
    assert [m.lr_count for m in metrics] == lc
    assert [m.tb_count for m in metrics] == tc


# ----------------------------------------------------------- reference goldens
def _golden_ids(g):
    return f"n{g['n']}_rho{g['rho']}_seed{g['seed']}_steps{g['steps']}"


GOLDENS = [g for g in load_goldens() if g["n"] <= 8192]


@pytest.mark.parametrize("g", GOLDENS, ids=_golden_ids)
def test_reference_golden(gpu, g):
    bml = gpu
    grid = bml.init_grid(g["n"], g["rho"], g["seed"])
    assert f"0x{grid.digest():016x}" == g["init_digest"]
    if "sum_lr_moved" in g:
        final, metrics = bml.simulate(grid, g["steps"])
        assert sum(m.lr_moved for m in metrics) == g["sum_lr_moved"]
        assert sum(m.tb_moved for m in metrics) == g["sum_tb_moved"]
        last = metrics[-1]
        assert (last.step, last.lr_moved, last.tb_moved) == (
            g["last"]["step"], g["last"]["lr_moved"], g["last"]["tb_moved"])
        assert (last.lr_count, last.tb_count) == (g["lr_count"], g["tb_count"])
    else:
        final = bml.step(grid, g["steps"])
    assert f"0x{final.digest():016x}" == g["final_digest"]
    assert bml.count_vehicles(final) == (g["lr_count"], g["tb_count"])


@pytest.mark.parametrize("g", [g for g in load_goldens() if g["n"] > 8192], ids=_golden_ids)
def test_reference_golden_huge(gpu, g):
    """BASELINE configs[3]/[4] sizes: device init_grid, device steps, device digest
    (host init would take minutes), against the unmodified reference's digests."""
    lat = gpu.DeviceLattice(g["n"])
    lat.init_random(g["rho"], g["seed"])
    assert f"0x{lat.digest():016x}" == g["init_digest"]
    done = 0
    for cp in g.get("checkpoints", []):  # chained goldens keep every leg's digest
        lat.step(cp["step"] - done)
        done = cp["step"]
        assert f"0x{lat.digest():016x}" == cp["digest"], cp
    lat.step(g["steps"] - done)
    assert f"0x{lat.digest():016x}" == g["final_digest"]
    assert lat.counts() == (g["lr_count"], g["tb_count"])


# ----------------------------------------------------------- properties (size-independent)
@pytest.mark.parametrize("n", [512, 4096])
def test_conservation_and_changed_equals_twice_moved(gpu, oracle, n):
    """test_engine.cpp:140-151 (conservation), :172-186 (changed = 2 x moved)."""
    bml = gpu
    cells = oracle.init_grid(n, 0.4, 11)
    g = grid_of(bml, n, cells)
    lat = bml.DeviceLattice(n)
    lat.upload(g)
    before = lat.download().to_bytes()
    for phase in (bml.Phase.horizontal, bml.Phase.vertical):
        moved = lat.phase(phase)
        after = lat.download().to_bytes()
        changed = sum(1 for a, b in zip(before, after) if a != b)
        assert changed == 2 * moved
        before = after
    assert lat.counts() == oracle.counts(n, cells)


@pytest.mark.parametrize("n", [23, 1024, 2000])
def test_shift_equivariance(gpu, n):
    """test_engine.cpp:188-199: step commutes with torus rotations."""
    bml = gpu
    cells = rand_lattice(n, n)
    dr, dc = n // 3, (2 * n) // 5

    def rot(b):
        out = bytearray(n * n)
        for r in range(n):
            src = b[r * n:(r + 1) * n]
            rr = (r + dr) % n
            out[rr * n:(rr + 1) * n] = src[-dc % n:] + src[:-dc % n] if dc % n else src
        return bytes(out)

    lhs = bml.step(grid_of(bml, n, rot(cells)), 7).to_bytes()
    rhs = rot(bml.step(grid_of(bml, n, cells), 7).to_bytes())
    assert lhs == rhs


def test_determinism_repeat(gpu):  # acceptance criterion 8
    bml = gpu
    g = bml.init_grid(333, 0.3, 9)
    a, ma = bml.simulate(g, 50)
    b, mb = bml.simulate(g, 50)
    assert a == b and a.digest() == b.digest()
    assert [(m.lr_moved, m.tb_moved) for m in ma] == [(m.lr_moved, m.tb_moved) for m in mb]


# ----------------------------------------------------------- row bands (virtual ranks on one GPU)
@pytest.mark.parametrize("devices", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [128, 1000, 1024])
def test_row_bands_match_single_band(gpu, oracle, devices, n):
    """GPU-count invariance: g bands with in-kernel halo exchange
    equal one band and the oracle — the ParallelRows determinism test
    (test_engine.cpp:201-211) with bands in place of threads."""
    bml = gpu
    cells = oracle.init_grid(n, 0.38, devices)
    steps = 37
    got = bml.step(grid_of(bml, n, cells), steps, devices=devices).to_bytes()
    assert got == oracle.run(n, cells, steps)
    final, metrics = bml.simulate(grid_of(bml, n, cells), steps, devices=devices)
    want, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
    assert final.to_bytes() == want
    assert [m.lr_moved for m in metrics] == lm
    assert [m.tb_moved for m in metrics] == tm
    assert [m.lr_count for m in metrics] == lc
    assert [m.tb_count for m in metrics] == tc


def test_metrics_with_tall_strips(gpu, oracle):
    """The metrics kernels pack two per-lane counters into 16-bit halves; strips
    taller than 2047 rows would overflow them, so the launch splits such strips
    even when asked for one (bml_dev.cu launch_block)."""
    bml = gpu
    n, steps = 4160, 3
    cells = oracle.init_grid(n, 0.45, 8)
    lat = bml.DeviceLattice(n)
    lat.configure(block_steps=16, strip_rows=n)  # one strip requested
    lat.upload(grid_of(bml, n, cells))
    metrics = lat.step_with_metrics(steps)
    want, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
    assert lat.download().to_bytes() == want
    assert [m.lr_moved for m in metrics] == lm and [m.tb_moved for m in metrics] == tm
    assert [m.lr_count for m in metrics] == lc and [m.tb_count for m in metrics] == tc


def test_row_bands_reject_thin_bands(gpu):
    bml = gpu
    with pytest.raises(ValueError):
        bml.DeviceLattice(40, devices=4)


# ----------------------------------------------------------- boundary behaviour / errors
def test_upload_rejects_invalid_cells(gpu):
    bml = gpu
    with pytest.raises(ValueError):
        bml.Grid.from_bytes(4, bytes([0, 1, 2, 3] * 4))


def test_zero_steps_is_identity(gpu):
    bml = gpu
    g = bml.init_grid(50, 0.5, 2)
    assert bml.step(g, 0) == g
    final, metrics = bml.simulate(g, 0)
    assert final == g and metrics == []


def test_reference_backend_names_run_on_the_device(gpu, oracle):
    """Reference call sites that name a CPU backend run unchanged on the device engine
    (same grid as b200 and as the oracle); parallel keeps its threads argument."""
    bml = gpu
    cells = oracle.init_grid(45, 0.4, 11)
    g = bml.Grid.from_bytes(45, cells)
    want = oracle.run(45, cells, 7)
    for b, threads in ((bml.Backend.naive, 1), (bml.Backend.halo, 1), (bml.Backend.parallel, 3),
                       (bml.Backend.lanes, 1)):
        assert bml.step(g, 7, backend=b, threads=threads).to_bytes() == want
        final, metrics = bml.simulate(g, 7, backend=b, threads=threads)
        assert final.to_bytes() == want and len(metrics) == 7
        h = bml.step_phase(g, bml.Phase.horizontal, backend=b)
        assert h == bml.step_phase(g, bml.Phase.horizontal)


def test_native_library_is_loaded(gpu):
    """The engine that ran is the in-tree CUDA library, not anything else."""
    bml = gpu
    bml.step(bml.Grid.from_text(">.\n.v"), 1)
    with open("/proc/self/maps") as f:
        maps = f.read()
    assert os.path.realpath(bml.LIB_DEV) in maps


# ----------------------------------------------------------- cluster-resident small-lattice kernel
@pytest.mark.parametrize("n", [32, 64, 96, 128, 160, 256, 512, 640, 992, 1024])
@pytest.mark.parametrize("ghost,mode", [(1, 1), (2, 1), (4, 1), (8, 1), (16, 1), (16, 2)])
def test_resident_kernel_matches_oracle(gpu, oracle, n, ghost, mode):
    bml = gpu
    cells = oracle.init_grid(n, 0.38, n + ghost)
    steps = 53
    lat = bml.DeviceLattice(n)
    lat.set_resident(mode)
    lat.configure(block_steps=ghost)
    lat.upload(bml.Grid.from_bytes(n, cells))
    metrics = lat.step_with_metrics(steps)
    assert lat.resident_cluster > 0, "resident kernel did not run"
    want, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
    assert lat.download().to_bytes() == want
    assert [m.lr_moved for m in metrics] == lm
    assert [m.tb_moved for m in metrics] == tm
    assert [m.lr_count for m in metrics] == lc
    assert [m.tb_count for m in metrics] == tc
    # bare loop (no counters) and the streaming kernel agree
    lat.upload(bml.Grid.from_bytes(n, cells))
    lat.step(steps)
    assert lat.download().to_bytes() == want
    lat.set_resident(0)
    lat.upload(bml.Grid.from_bytes(n, cells))
    lat.step(steps)
    assert lat.resident_cluster == 0
    assert lat.download().to_bytes() == want


def test_resident_kernel_long_run_golden(gpu):
    """configs[1] (N=1024, rho=.38, 4096 steps) through the resident kernel."""
    bml = gpu
    g = [x for x in load_goldens() if x["n"] == 1024][0]
    lat = bml.DeviceLattice(1024)
    lat.upload(bml.init_grid(1024, g["rho"], g["seed"]))
    metrics = lat.step_with_metrics(g["steps"])
    assert lat.resident_cluster > 0
    assert f"0x{lat.download().digest():016x}" == g["final_digest"]
    assert sum(m.lr_moved for m in metrics) == g["sum_lr_moved"]
    assert sum(m.tb_moved for m in metrics) == g["sum_tb_moved"]


@pytest.mark.parametrize("n,ns", [(1056, 7), (1056, 66), (2048, 2), (3000, 13)])
def test_explicit_strip_count_and_launch_geometry(gpu, oracle, n, ns):
    """strip_rows = -ns asks for exactly ns strips (include/bml_dev.h); rows are
    split evenly and the result is bit-exact whatever the split."""
    import ctypes
    bml = gpu
    cells = rand_lattice(n + ns, n)
    lat = bml.DeviceLattice(n)
    lat.set_resident(0)
    lat.configure(block_steps=16, strip_rows=-ns)
    lat.upload(grid_of(bml, n, cells))
    lat.step(19)
    lib = ctypes.CDLL(bml.LIB_DEV)
    lib.bml_dev_last_launch.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int)] * 3
    got = [ctypes.c_int() for _ in range(3)]
    assert lib.bml_dev_last_launch(ctypes.c_void_p(lat.handle()), *[ctypes.byref(x) for x in got]) == 0
    strips, items, ctas = (x.value for x in got)
    assert strips == ns and items % ns == 0 and 1 <= ctas <= 148
    assert lat.download().to_bytes() == oracle.run(n, cells, 19)


@pytest.mark.parametrize("n", [993, 1000, 1023, 1025, 1100, 2047, 3000, 4099])
@pytest.mark.parametrize("block", [1, 4, 16])
def test_seam_mode_sizes(gpu, oracle, n, block):
    """n % 32 != 0 with W >= 32 runs the kSeam mode: aligned words through the
    cp.async ring, seam windows rebuilt by shuffles (bml_kernels_common.cuh)."""
    bml = gpu
    cells = rand_lattice(n * 7 + block, n)
    lat = bml.DeviceLattice(n)
    lat.configure(block_steps=block)
    lat.upload(grid_of(bml, n, cells))
    lat.step(37)
    assert lat.download().to_bytes() == oracle.run(n, cells, 37)


@pytest.mark.parametrize("n,bands", [(1100, 2), (3000, 3)])
def test_seam_mode_bands_and_metrics(gpu, oracle, n, bands):
    bml = gpu
    cells = oracle.init_grid(n, 0.4, n)
    final, metrics = bml.simulate(grid_of(bml, n, cells), 19, devices=bands)
    want, (lm, tm, lc, tc) = oracle.run(n, cells, 19, metrics=True)
    assert final.to_bytes() == want
    assert [m.lr_moved for m in metrics] == lm and [m.tb_moved for m in metrics] == tm
    assert [m.lr_count for m in metrics] == lc and [m.tb_count for m in metrics] == tc


# ----------------------------------------------------------- the benched instantiations
def test_bare_loop_golden_c1(gpu):
    """configs[1] exactly as bench.py runs it: the bare loop (no metrics) of 4096 steps,
    through the resident kernel (COUNT=0) and through the streaming kernel, against the
    unmodified reference's final digest."""
    g = [x for x in load_goldens() if x["n"] == 1024 and x["steps"] == 4096][0]
    grid = gpu.init_grid(1024, g["rho"], g["seed"])
    for resident in (1, 0):
        lat = gpu.DeviceLattice(1024)
        lat.set_resident(resident)
        lat.upload(grid)
        lat.step(g["steps"])
        assert (lat.resident_cluster > 0) == bool(resident)
        assert f"0x{lat.digest():016x}" == g["final_digest"]


@pytest.mark.slow
@pytest.mark.parametrize("bands", [2, 4, 8])
@pytest.mark.parametrize("g", [g for g in load_goldens() if g["n"] > 8192], ids=_golden_ids)
def test_reference_golden_huge_row_bands(gpu, g, bands):
    """configs[3]/[4] goldens through `bands` row bands of ceil(N/g) rows (one GPU,
    in-kernel ghost-row exchange between the bands' buffers): the literal multi-GPU
    split, bit-exact with the unmodified reference."""
    lat = gpu.DeviceLattice(g["n"], bands)
    lat.init_random(g["rho"], g["seed"])
    assert f"0x{lat.digest():016x}" == g["init_digest"]
    lat.step(g["steps"])
    assert f"0x{lat.digest():016x}" == g["final_digest"]
    assert lat.counts() == (g["lr_count"], g["tb_count"])
