"""Pin the oracle (oracle/bml_oracle.c) to the reference's own known answers.

Every vector here is taken from the reference test-suite (file:line under
/root/reference/proj/tests) or from tests/golden/*.json, which the UNMODIFIED
reference produced (tests/golden/make_goldens.py). CPU only.
"""
import os
import random
import subprocess

import pytest

from conftest import REF_DRIVER, load_goldens, rows_to_bytes


def test_splitmix64_seed0_vectors(oracle):  # test_seeding.cpp:10-16
    assert oracle.splitmix(0, 4) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                     0x06C45D188009454F, 0xF88BB8A8724C81EC]


def test_bounded_cases(oracle):  # test_seeding.cpp:18-37
    import ctypes

    s = ctypes.c_uint64(1)
    for _ in range(100):
        assert oracle.lib.orc_bounded(ctypes.byref(s), 1, None) == 0
    err = ctypes.c_int(0)
    oracle.lib.orc_bounded(ctypes.byref(s), 0, ctypes.byref(err))
    assert err.value == 1
    for _ in range(100):
        assert oracle.lib.orc_bounded(ctypes.byref(s), 8, None) < 8
    s = ctypes.c_uint64(20240601)
    bins = [0, 0, 0]
    draws = 300000
    for _ in range(draws):
        bins[oracle.lib.orc_bounded(ctypes.byref(s), 3, None)] += 1
    sigma = (draws * (1 / 3) * (2 / 3)) ** 0.5
    assert all(abs(b - draws / 3) <= 3 * sigma for b in bins)


def test_vehicles_per_species(oracle):  # test_seeding.cpp:39-44
    f = oracle.lib.orc_vehicles_per_species
    assert (f(256, 0.3), f(4, 0.5), f(4, 1.0), f(1, 0.0)) == (9830, 4, 8, 0)


def test_pinned_lattice_seed42(oracle):  # test_seeding.cpp:70-79
    assert oracle.init_grid(4, 0.5, 42) == rows_to_bytes(["..>.", ">.vv", "v...", ">>v."])


def test_init_counts_exact(oracle):  # test_seeding.cpp:46-59
    assert oracle.counts(16, oracle.init_grid(16, 0.0, 3)) == (0, 0)
    assert oracle.counts(4, oracle.init_grid(4, 1.0, 3)) == (8, 8)
    assert oracle.counts(256, oracle.init_grid(256, 0.3, 1)) == (9830, 9830)


def test_fnv_vectors(oracle):  # test_digest.cpp:16-20
    f = oracle.lib.orc_fnv1a64
    basis = 0xcbf29ce484222325
    assert f(b"", 0, basis) == 0xcbf29ce484222325
    assert f(b"a", 1, basis) == 0xaf63dc4c8601ec8c
    assert f(b"foobar", 6, basis) == 0x85944171f73967e8


def test_rule_truth_tables(oracle):  # test_engine.cpp:50-61
    E, LR, TB = 0, 1, 2
    h, v = oracle.lib.orc_horizontal_rule, oracle.lib.orc_vertical_rule
    assert h(LR, E, TB) == LR and h(E, LR, E) == E and h(E, TB, E) == TB and h(LR, LR, LR) == LR
    assert v(TB, E, LR) == TB and v(E, TB, E) == E and v(TB, LR, E) == LR


@pytest.mark.parametrize("row,expected", [(">.>.", ".>.>"), (">>..", ">.>."),
                                          (">>>>", ">>>>"), (">v..", ">v..")])
def test_phase_cases(oracle, row, expected):  # test_engine.cpp:63-81
    rest = ["....", "....", "...."]
    out = oracle.phase(4, rows_to_bytes([row] + rest), 0)
    assert out == rows_to_bytes([expected] + rest)


def test_two_by_two_steps(oracle):  # test_engine.cpp:83-93
    assert oracle.run(2, rows_to_bytes([">.", ".v"]), 1) == rows_to_bytes([".>", ".v"])
    assert oracle.run(2, rows_to_bytes([">.", ".."]), 2) == rows_to_bytes([">.", ".."])
    assert oracle.run(2, rows_to_bytes(["..", ".."]), 1) == rows_to_bytes(["..", ".."])


def test_never_blocked_metrics(oracle):  # test_metrics.cpp:62-75
    cells = rows_to_bytes([">...", "....", ".v..", "...."])
    _, (lm, tm, lc, tc) = oracle.run(4, cells, 8, metrics=True)
    assert lm == [1] * 8 and tm == [1] * 8 and lc == [1] * 8 and tc == [1] * 8


@pytest.mark.parametrize("g", [g for g in load_goldens() if g["n"] <= 256],
                         ids=lambda g: f"n{g['n']}_seed{g['seed']}")
def test_oracle_reproduces_reference_goldens(oracle, g):
    cells = oracle.init_grid(g["n"], g["rho"], g["seed"])
    assert f"0x{oracle.digest(g['n'], cells):016x}" == g["init_digest"]
    final, (lm, tm, lc, tc) = oracle.run(g["n"], cells, g["steps"], metrics=True)
    assert f"0x{oracle.digest(g['n'], final):016x}" == g["final_digest"]
    assert sum(lm) == g["sum_lr_moved"] and sum(tm) == g["sum_tb_moved"]
    assert (lm[-1], tm[-1]) == (g["last"]["lr_moved"], g["last"]["tb_moved"])


def test_golden_init_digests_all_sizes(oracle):
    """The init digest of every golden (up to N=4096) is reproduced by the oracle."""
    for g in load_goldens():
        if g["n"] > 4096:
            continue
        cells = oracle.init_grid(g["n"], g["rho"], g["seed"])
        assert f"0x{oracle.digest(g['n'], cells):016x}" == g["init_digest"], g


@pytest.mark.skipif(not os.path.exists(REF_DRIVER), reason="oracle/_ref not built")
@pytest.mark.parametrize("n", [1, 2, 3, 7, 15, 16, 17, 31, 32, 33, 48, 63, 64])
def test_oracle_matches_reference_binary_on_random_grids(oracle, tmp_path, n):
    """test_engine.cpp:95-114 sizes; the oracle vs the reference's own backends."""
    rng = random.Random(0xBACCA + n)
    cells = bytes(rng.randrange(3) for _ in range(n * n))
    steps = 1 + rng.randrange(3) + n % 5
    src = tmp_path / "in.bin"
    out = tmp_path / "out.bin"
    src.write_bytes(cells)
    for backend in ("naive", "halo", "lanes"):
        subprocess.run([REF_DRIVER, "file", f"in={src}", f"n={n}", f"steps={steps}",
                        f"backend={backend}", f"dump_final={out}"], check=True,
                       capture_output=True)
        assert out.read_bytes() == oracle.run(n, cells, steps), backend
    for ph, name in ((0, "h"), (1, "v")):
        subprocess.run([REF_DRIVER, "file", f"in={src}", f"n={n}", f"phase={name}",
                        "backend=naive", f"dump_final={out}"], check=True, capture_output=True)
        assert out.read_bytes() == oracle.phase(n, cells, ph)
