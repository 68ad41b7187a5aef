"""Device-side init_grid (csrc/bml_init.cu) against the oracle.

The reference draws the lattice with a serial descending Fisher–Yates shuffle
(/root/reference/proj/src/seeding.cpp:26-51); the device computes the same
permutation in parallel. Parity is bit-exact: every case compares the whole
lattice with oracle/bml_oracle.c's orc_init_grid (itself pinned to the
reference's KATs in test_oracle.py), and the large cases compare the FNV digest
with the init digests the unmodified reference wrote into tests/golden/.
"""
import ctypes
import os

import pytest

from conftest import load_goldens

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def abi(gpu):
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1804_07981_b200", "libbml_dev.so"))
    vp = ctypes.c_void_p
    lib.bml_dev_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    lib.bml_dev_create_band.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(vp)]
    lib.bml_dev_destroy.argtypes = [vp]
    lib.bml_dev_init_random.argtypes = [vp, ctypes.c_double, ctypes.c_uint64]
    lib.bml_dev_init_random_masked.argtypes = [vp, ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64]
    lib.bml_dev_download.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    lib.bml_dev_step.argtypes = [vp, ctypes.c_int64] + [vp] * 4
    lib.bml_dev_last_error.restype = ctypes.c_char_p
    return lib


def device_init(abi, n, rho, seed, mask=0, band=None):
    h = ctypes.c_void_p()
    if band is None:
        assert abi.bml_dev_create(n, 0, ctypes.byref(h)) == 0
        rows = n
    else:
        assert abi.bml_dev_create_band(n, band[0], band[1], 0, ctypes.byref(h)) == 0
        rows = band[1] - band[0]
    try:
        rc = abi.bml_dev_init_random_masked(h, rho, seed, mask)
        assert rc == 0, abi.bml_dev_last_error()
        out = ctypes.create_string_buffer(rows * n)
        assert abi.bml_dev_download(h, out, n) == 0, abi.bml_dev_last_error()
        return out.raw[: rows * n]
    finally:
        abi.bml_dev_destroy(h)


SMALL = [(n, rho, seed) for n in (1, 2, 3, 4, 5, 7, 31, 32, 33, 64, 100, 257)
         for rho, seed in ((0.0, 1), (0.3, 1), (0.5, 42), (1.0, 7))]


@pytest.mark.parametrize("n,rho,seed", SMALL)
def test_device_init_matches_oracle_small(abi, oracle, n, rho, seed):
    assert device_init(abi, n, rho, seed) == oracle.init_grid(n, rho, seed)


def test_device_init_pinned_lattice(gpu):  # test_seeding.cpp:70-79
    assert gpu.init_grid(4, 0.5, 42, on_device=True).to_text() == "..>.\n>.vv\nv...\n>>v.\n"


@pytest.mark.parametrize("n,rho,seed", [(1024, 0.38, 1), (1000, 0.25, 3), (2048, 0.35, 9),
                                        (4099, 0.6, 123456789)])
def test_device_init_matches_oracle_medium(abi, oracle, n, rho, seed):
    assert device_init(abi, n, rho, seed) == oracle.init_grid(n, rho, seed)


@pytest.mark.parametrize("n,mask", [(16, 0x1), (64, 0x7), (200, 0x3f), (512, 0xff)])
def test_rejection_fixup_path(abi, oracle, n, mask):
    """The TEST hook rejects extra draws; device and oracle apply the same rule,
    so this drives the multi-pass rejection fix-up (hundreds of passes)."""
    dev = device_init(abi, n, 0.4, 5, mask=mask)
    assert dev == oracle.init_grid_masked(n, 0.4, 5, mask)
    assert dev != oracle.init_grid(n, 0.4, 5)  # the hook really changed the draws


@pytest.mark.parametrize("n,bands", [(256, 3), (1000, 8)])
def test_band_init_slices(abi, oracle, n, bands):
    want = oracle.init_grid(n, 0.35, 17)
    step = (n + bands - 1) // bands
    for b in range(bands):
        r0, r1 = b * step, min(n, (b + 1) * step)
        assert device_init(abi, n, 0.35, 17, band=(r0, r1)) == want[r0 * n: r1 * n]


def test_multi_band_lattice_init_then_step(gpu, oracle):
    bml = gpu
    n, steps = 384, 37
    lat = bml.DeviceLattice(n, devices=4)
    lat.init_random(0.38, 4)
    assert lat.download().to_bytes() == oracle.init_grid(n, 0.38, 4)
    lat.step(steps)
    assert lat.download().to_bytes() == oracle.run(n, oracle.init_grid(n, 0.38, 4), steps)


GOLDENS = [g for g in load_goldens() if g["n"] >= 1000]


@pytest.mark.parametrize("g", GOLDENS, ids=lambda g: f"n{g['n']}_rho{g['rho']}_seed{g['seed']}")
def test_device_init_digest_matches_reference_golden(gpu, g):
    grid = gpu.init_grid(g["n"], g["rho"], g["seed"], on_device=True)
    assert f"0x{grid.digest():016x}" == g["init_digest"]
    assert gpu.count_vehicles(grid) == (g["k"], g["k"])


def test_device_init_equals_host_init_16384(gpu):
    host = gpu.init_grid(16384, 0.35, 1)
    dev = gpu.init_grid(16384, 0.35, 1, on_device=True)
    assert dev.digest() == host.digest()


def test_device_init_rejects_bad_arguments(abi, gpu):
    h = ctypes.c_void_p()
    assert abi.bml_dev_create(8, 0, ctypes.byref(h)) == 0
    try:
        assert abi.bml_dev_init_random(h, 1.5, 1) == 1
        assert abi.bml_dev_init_random(h, -0.1, 1) == 1
    finally:
        abi.bml_dev_destroy(h)
    with pytest.raises(ValueError):
        gpu.init_grid(8, 2.0, 1, on_device=True)
