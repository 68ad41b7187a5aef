"""Device-side grid_digest (csrc/bml_digest.cu) against the host FNV and the reference goldens.

grid_digest is FNV-1a-64 over the cells, row-major (/root/reference/proj/src/digest.cpp:5-14).
The device computes it from the bit planes with the segment algebra pinned on CPU in
test_digest_algorithm.py. Bit-exact comparisons throughout.
"""
import random

import pytest

from conftest import load_goldens

pytestmark = pytest.mark.gpu


def rand_cells(seed, n):
    rng = random.Random(seed)
    return bytes(b % 3 for b in rng.randbytes(n * n))


@pytest.mark.parametrize("n", [1, 2, 3, 7, 31, 32, 33, 63, 64, 65, 100, 257, 1000, 1024, 1056])
def test_device_digest_matches_host(gpu, oracle, n):
    bml = gpu
    cells = rand_cells(n, n)
    lat = bml.DeviceLattice(n)
    lat.upload(bml.Grid.from_bytes(n, cells))
    assert lat.digest() == oracle.digest(n, cells)
    lat.step(7)
    assert lat.digest() == lat.download().digest()


@pytest.mark.parametrize("n,bands", [(64, 2), (100, 3), (384, 4), (1000, 8)])
def test_band_digests_combine(gpu, oracle, n, bands):
    bml = gpu
    cells = oracle.init_grid(n, 0.4, bands)
    lat = bml.DeviceLattice(n, devices=bands)
    lat.upload(bml.Grid.from_bytes(n, cells))
    assert lat.digest() == oracle.digest(n, cells)
    lat.step(21)
    assert lat.digest() == oracle.digest(n, oracle.run(n, cells, 21))


GOLDENS = [g for g in load_goldens() if g["n"] >= 1000]


@pytest.mark.parametrize("g", GOLDENS, ids=lambda g: f"n{g['n']}_rho{g['rho']}_steps{g['steps']}")
def test_fully_on_device_run_reproduces_reference_golden(gpu, g):
    """Device init_grid -> device steps -> device digest, against the digests the
    unmodified reference produced (tests/golden/)."""
    lat = gpu.DeviceLattice(g["n"])
    lat.init_random(g["rho"], g["seed"])
    assert f"0x{lat.digest():016x}" == g["init_digest"]
    lat.step(g["steps"])
    assert f"0x{lat.digest():016x}" == g["final_digest"]
