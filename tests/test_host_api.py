"""Host-side drop-in surface (no GPU needed): the reference's Python/C++ API semantics.

Mirrors /root/reference/proj/tests/python/test_smoke.py and the grid / seeding /
metrics unit tests for everything that does not step the lattice. Stepping
through a CPU backend must fail loudly — this build has no CPU engine.
"""
import ctypes
import re

import pytest

from conftest import ROOT, rows_to_bytes


def test_version_and_lane_width(bml):
    assert bml.__version__
    assert bml.lane_width() >= 16 and bml.lane_width() % 16 == 0


def test_init_grid_counts_exact(bml):  # test_smoke.py:17-19
    assert bml.count_vehicles(bml.init_grid(n=256, rho=0.3, seed=1)) == (9830, 9830)


@pytest.mark.parametrize("n,rho,seed", [(1, 0.5, 1), (4, 0.5, 42), (17, 0.9, 3), (33, 0.4, 9),
                                        (100, 0.25, 7), (257, 0.38, 11), (1024, 0.38, 1)])
def test_init_grid_bit_identical_to_oracle(bml, oracle, n, rho, seed):
    assert bml.init_grid(n, rho, seed).to_bytes() == oracle.init_grid(n, rho, seed)


def test_pinned_lattice(bml):  # test_seeding.cpp:70-79
    assert bml.init_grid(4, 0.5, 42).to_text() == "..>.\n>.vv\nv...\n>>v.\n"


def test_init_validation(bml):  # test_seeding.cpp:81-85
    for args in ((0, 0.5, 1), (4, -0.1, 1), (4, 1.1, 1)):
        with pytest.raises(ValueError):
            bml.init_grid(*args)


def test_text_round_trip_and_errors(bml):  # test_smoke.py:22-27, test_grid.cpp:81-117
    g = bml.Grid.from_text(">.\n.v")
    assert g.n == 2 and g.to_text() == ">.\n.v\n"
    assert g.cell(0, 0) == bml.Cell.lr and g.cell(1, 1) == bml.Cell.tb
    assert bml.Grid.from_text(">.\n.v\n").to_text() == ">.\n.v\n"
    for bad in ("", ">.", ">.\n>"):
        with pytest.raises(ValueError):
            bml.Grid.from_text(bad)
    with pytest.raises(ValueError, match=r"line 2.*column 2"):
        bml.Grid.from_text(">.\n.x")
    with pytest.raises(IndexError):
        g.cell(2, 0)


def test_set_cell_and_equality(bml):
    a = bml.Grid.from_text("...\n...\n...")
    b = bml.Grid.from_text("...\n...\n...")
    assert a == b
    b.set_cell(1, 2, bml.Cell.lr)
    assert not (a == b)
    assert b.cell(1, 2) == bml.Cell.lr


def test_bytes_round_trip(bml, oracle):
    cells = oracle.init_grid(37, 0.45, 5)
    g = bml.Grid.from_bytes(37, cells)
    assert g.to_bytes() == cells
    with pytest.raises(ValueError):
        bml.Grid.from_bytes(2, bytes([0, 1, 2, 3]))
    with pytest.raises(ValueError):
        bml.Grid.from_bytes(3, bytes(8))


def test_digest_matches_oracle(bml, oracle):  # test_digest.cpp:22-34
    g = bml.Grid.from_text(">v\n..")
    assert g.digest() == oracle.digest(2, rows_to_bytes([">v", ".."]))
    cells = oracle.init_grid(64, 0.3, 2)
    assert bml.Grid.from_bytes(64, cells).digest() == oracle.digest(64, cells)


def test_moved_in_phase_and_counts(bml):  # test_metrics.cpp:10-28
    before = bml.Grid.from_text(">.>.\n....\n....\n....")
    after = bml.Grid.from_text(".>.>\n....\n....\n....")
    assert bml.moved_in_phase(before, after, bml.Phase.horizontal) == 2
    assert bml.moved_in_phase(before, after, bml.Phase.vertical) == 0
    ring = bml.Grid.from_text(">>>>\n....\n....\n....")
    assert bml.moved_in_phase(ring, ring, bml.Phase.horizontal) == 0
    with pytest.raises(ValueError):
        bml.moved_in_phase(bml.Grid.from_text("..\n.."), ring, bml.Phase.horizontal)
    assert bml.count_vehicles(bml.Grid.from_text(">.\n.v")) == (1, 1)


def test_classify_thresholds(bml):  # test_metrics.cpp:30-45
    assert bml.classify([1.0] * 10) == bml.Regime.FreeFlow
    assert bml.classify([0.0] * 10) == bml.Regime.Jammed
    assert bml.classify([0.5] * 10) == bml.Regime.Intermediate
    assert bml.classify([0.99] * 4) == bml.Regime.FreeFlow
    assert bml.classify([0.01] * 4) == bml.Regime.Jammed
    with pytest.raises(ValueError):
        bml.classify([])


def test_backend_names(bml):  # test_engine.cpp:304-307, SURVEY §4 item 3
    for name in ("naive", "halo", "parallel", "lanes", "b200"):
        assert bml.backend_from_name(name) is not None
    assert bml.backend_from_name("cuda") is None
    assert bml.backend_from_name("b200") == bml.Backend.b200


def test_reference_backend_names_route_to_the_device(bml):
    """The reference's backend names stay usable (engine.hpp:15-20): they keep the
    reference layout/thread rules and run on the device engine. Without a GPU that
    is a loud RuntimeError, never a CPU computation."""
    g = bml.Grid.from_text(">.\n.v")
    for b in (bml.Backend.naive, bml.Backend.halo, bml.Backend.parallel, bml.Backend.lanes):
        try:
            out = bml.step(g, 1, backend=b)
        except RuntimeError:
            continue  # no CUDA device on this host
        assert out == bml.step(g, 1)
    with pytest.raises(ValueError, match="threads > 1"):
        bml.step(g, 1, backend=bml.Backend.lanes, threads=4)  # engine.cpp:153-156


def test_config_validation_errors(bml):
    g = bml.Grid.from_text(">.\n.v")
    with pytest.raises(ValueError):
        bml.step(g, -1)
    with pytest.raises(ValueError):
        bml.step(g, 1, threads=2)  # only ParallelRows accepts threads > 1 (engine.cpp:53-56)
    with pytest.raises(ValueError):
        bml.step(g, 1, devices=0)


# ------------------------------------------------------------------ C-ABI
HEADER = f"{ROOT}/include/bml_dev.h"


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(bml_dev_\w+)\s*\(", text, re.M)))


def test_abi_library_exports_every_declared_symbol(bml):
    lib = ctypes.CDLL(bml.LIB_DEV)
    syms = declared_symbols()
    assert len(syms) >= 20, syms
    for s in syms:
        assert hasattr(lib, s), s


def test_abi_error_paths_without_gpu_work(bml):
    lib = ctypes.CDLL(bml.LIB_DEV)
    lib.bml_dev_last_error.restype = ctypes.c_char_p
    lib.bml_dev_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.bml_dev_version()
    h = ctypes.c_void_p()
    assert lib.bml_dev_create(0, 0, ctypes.byref(h)) == 1  # BML_EINVAL: n < 1
    assert lib.bml_dev_create(8, 0, None) == 1
    assert lib.bml_dev_step(None, 1, None, None, None, None) == 1
    assert lib.bml_dev_last_error()
    count = ctypes.c_int(-1)
    assert lib.bml_dev_device_count(ctypes.byref(count)) == 0
    assert count.value >= 0
