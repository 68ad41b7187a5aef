"""Seeded random configurations of the device engine against the oracle.

Each case draws a lattice size from the four kernel modes' ranges (n < 32, n % 32
!= 0 narrow and wide, n % 32 == 0 up to 1056), a density, a step count, a block
depth, a strip height, the resident-kernel mode and whether per-step metrics are
requested, then compares the final lattice and (when requested) every per-step
counter with the oracle (oracle/bml_oracle.c, pinned to the reference goldens).
Integer CA: bit-exact. The case list is fixed by FUZZ_SEED, so a failure names a
reproducible configuration.
"""
import random

import pytest

pytestmark = pytest.mark.gpu

FUZZ_SEED = 0x1804_07981
N_CASES = 96


def _cases():
    rng = random.Random(FUZZ_SEED)
    out = []
    for i in range(N_CASES):
        kind = i % 4
        if kind == 0:
            n = rng.randint(1, 31)
        elif kind == 1:
            n = rng.choice([32 * rng.randint(1, 33), 32 * rng.randint(1, 8)])
        elif kind == 2:
            n = rng.randint(33, 992)
            n += n % 32 == 0
        else:
            n = rng.randint(993, 1400)
            n += n % 32 == 0
        u = rng.random()
        rho = rng.choice([0.0, 1.0]) if u < 0.12 else (rng.uniform(0.3, 0.45) if u < 0.6 else rng.random())
        u = rng.random()
        steps = rng.choice([0, 1]) if u < 0.12 else (rng.randint(2, 40) if u < 0.55 else rng.randint(41, 140))
        block = rng.choice([1, 2, 4, 8, 16, 16])  # bml_dev_configure accepts powers of two
        strip = rng.choice([0, 0, rng.randint(1, 64), rng.randint(1, max(1, n))])
        resident = rng.choice([0, 1, 1, 2])
        metrics = rng.random() < 0.5
        out.append((i, n, round(rho, 4), steps, block, strip, resident, metrics, rng.getrandbits(32)))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}_n{c[1]}_s{c[3]}_b{c[4]}_r{c[6]}")
def test_random_configuration_matches_oracle(gpu, oracle, case):
    bml = gpu
    _, n, rho, steps, block, strip, resident, metrics, seed = case
    cells = oracle.init_grid(n, rho, seed)
    lat = bml.DeviceLattice(n)
    lat.configure(block_steps=block, strip_rows=strip)
    lat.set_resident(resident)
    lat.upload(bml.Grid.from_bytes(n, cells))
    if metrics and steps > 0:
        got = lat.step_with_metrics(steps)
        want, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
        assert [m.step for m in got] == list(range(1, steps + 1))
        assert [m.lr_moved for m in got] == lm
        assert [m.tb_moved for m in got] == tm
        assert [m.lr_count for m in got] == lc
        assert [m.tb_count for m in got] == tc
    else:
        lat.step(steps)
        want = oracle.run(n, cells, steps)
    assert lat.download().to_bytes() == want
    assert lat.digest() == oracle.digest(n, want)


def _band_cases():
    rng = random.Random(FUZZ_SEED + 1)
    out = []
    while len(out) < 32:
        n = rng.choice([rng.randint(64, 700), 32 * rng.randint(2, 40), rng.randint(993, 1400)])
        devices = rng.randint(2, 4)
        if n - (devices - 1) * ((n + devices - 1) // devices) < 16:  # engine.cpp band split rule
            continue
        rho = round(rng.uniform(0.2, 0.6), 4)
        steps = rng.randint(1, 120)
        block = rng.choice([1, 2, 4, 8, 16, 16])
        strip = rng.choice([0, 0, rng.randint(16, 200)])  # connected bands: strips >= 16 rows
        metrics = rng.random() < 0.5
        out.append((len(out), n, devices, rho, steps, block, strip, metrics, rng.getrandbits(32)))
    return out


@pytest.mark.parametrize("case", _band_cases(), ids=lambda c: f"b{c[0]}_n{c[1]}_d{c[2]}_s{c[4]}_b{c[5]}")
def test_random_row_bands_match_oracle(gpu, oracle, case):
    """Row bands exchanging ghost rows inside the step kernel, all
    placed on the one visible GPU: same lattice, counters and digest as one band."""
    bml = gpu
    _, n, devices, rho, steps, block, strip, metrics, seed = case
    cells = oracle.init_grid(n, rho, seed)
    lat = bml.DeviceLattice(n, devices)
    lat.configure(block_steps=block, strip_rows=strip)
    lat.upload(bml.Grid.from_bytes(n, cells))
    if metrics:
        got = lat.step_with_metrics(steps)
        want, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
        assert [m.lr_moved for m in got] == lm
        assert [m.tb_moved for m in got] == tm
        assert [m.lr_count for m in got] == lc
        assert [m.tb_count for m in got] == tc
    else:
        lat.step(steps)
        want = oracle.run(n, cells, steps)
    assert lat.download().to_bytes() == want
    assert lat.digest() == oracle.digest(n, want)
