"""Shared test fixtures.

The oracle (oracle/build/liboracle.so, a plain-C restatement of the reference) and
the reference driver (oracle/_ref/ref_driver, the unmodified reference sources) are
TEST INFRASTRUCTURE: they are only ever the checker here.
"""
import ctypes
import glob
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
ORACLE_SO = os.path.join(ROOT, "oracle", "build", "liboracle.so")
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


class Oracle:
    """ctypes view of oracle/bml_oracle.c (dense n*n byte lattices)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
        lib = ctypes.CDLL(path)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        lib.orc_splitmix64_next.argtypes = [u64p]
        lib.orc_splitmix64_next.restype = ctypes.c_uint64
        lib.orc_bounded.argtypes = [u64p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int)]
        lib.orc_bounded.restype = ctypes.c_uint64
        lib.orc_vehicles_per_species.argtypes = [ctypes.c_int, ctypes.c_double]
        lib.orc_vehicles_per_species.restype = ctypes.c_int64
        lib.orc_init_grid.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_uint64, ctypes.c_char_p]
        lib.orc_init_grid_masked.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                             ctypes.c_uint64, ctypes.c_char_p]
        lib.orc_phase.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int]
        lib.orc_moved.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int]
        lib.orc_moved.restype = ctypes.c_int64
        lib.orc_counts.argtypes = [ctypes.c_int, ctypes.c_char_p,
                                   ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        lib.orc_fnv1a64.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_uint64]
        lib.orc_fnv1a64.restype = ctypes.c_uint64
        lib.orc_digest.argtypes = [ctypes.c_int, ctypes.c_char_p]
        lib.orc_digest.restype = ctypes.c_uint64
        lib.orc_run.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_int64] + [ctypes.c_void_p] * 4
        lib.orc_run.restype = ctypes.c_int
        for name in ("orc_horizontal_rule", "orc_vertical_rule"):
            f = getattr(lib, name)
            f.argtypes = [ctypes.c_uint8] * 3
            f.restype = ctypes.c_uint8
        self.lib = lib

    def splitmix(self, seed, count):
        s = ctypes.c_uint64(seed)
        return [self.lib.orc_splitmix64_next(ctypes.byref(s)) for _ in range(count)]

    def init_grid(self, n, rho, seed):
        buf = ctypes.create_string_buffer(n * n)
        assert self.lib.orc_init_grid(n, rho, seed, buf) == 0
        return buf.raw[: n * n]

    def init_grid_masked(self, n, rho, seed, reject_mask):
        buf = ctypes.create_string_buffer(n * n)
        assert self.lib.orc_init_grid_masked(n, rho, seed, reject_mask, buf) == 0
        return buf.raw[: n * n]

    def phase(self, n, cells, phase):
        out = ctypes.create_string_buffer(n * n)
        self.lib.orc_phase(n, cells, out, phase)
        return out.raw[: n * n]

    def moved(self, n, before, after, phase):
        return self.lib.orc_moved(n, before, after, phase)

    def run(self, n, cells, steps, metrics=False):
        buf = ctypes.create_string_buffer(bytes(cells), n * n)
        if metrics and steps > 0:
            arrs = [(ctypes.c_int64 * steps)() for _ in range(4)]
            rc = self.lib.orc_run(n, buf, steps, *[ctypes.cast(a, ctypes.c_void_p) for a in arrs])
            assert rc == 0, rc
            return buf.raw[: n * n], [list(a) for a in arrs]
        rc = self.lib.orc_run(n, buf, steps, None, None, None, None)
        assert rc == 0, rc
        return buf.raw[: n * n]

    def digest(self, n, cells):
        return self.lib.orc_digest(n, cells)

    def counts(self, n, cells):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self.lib.orc_counts(n, cells, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value


@pytest.fixture(scope="session")
def oracle():
    return Oracle()


def load_goldens():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "ref_*.json"))):
        with open(p) as f:
            out.append(json.load(f))
    return out


def rows_to_bytes(rows):
    table = {".": 0, ">": 1, "v": 2}
    return bytes(table[c] for r in rows for c in r)


def random_cells(rng, n):
    """Uniform {0,1,2} cells, like test_util.hpp:14-21 random_halo_grid."""
    return bytes(rng.randrange(3) for _ in range(n * n))


def gpu_available():
    try:
        import paper_1804_07981_b200 as bml

        return bml.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def bml():
    import paper_1804_07981_b200 as mod

    return mod


@pytest.fixture(scope="session")
def gpu(bml):
    if bml.device_count() < 1:
        pytest.skip("no CUDA device")
    return bml
