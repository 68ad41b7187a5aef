"""The opt-in wide-lane streaming kernel (bml_dev_set_variant 2/3/4: 64 cells per lane,
K = 14 or 12 steps per launch, TMA bulk-copy or LDGSTS row ring) is bit-exact with the
oracle: lattices, per-step moved counts and census, row bands, and the torus seam
(column 0's window starts two words before the row)."""
import ctypes

import pytest

pytestmark = pytest.mark.gpu


def set_variant(gpu, lat, v, band=0):
    lib = ctypes.CDLL(gpu.LIB_DEV)
    lib.bml_dev_set_variant.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert lib.bml_dev_set_variant(ctypes.c_void_p(lat.handle(band)), v) == 0


@pytest.mark.parametrize("variant", [2, 3, 4])
@pytest.mark.parametrize("n,steps", [(2048, 45), (2176, 29), (4096, 31)])
def test_wide_variant_matches_oracle(gpu, oracle, variant, n, steps):
    cells = oracle.init_grid(n, 0.37, n + variant)
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, variant)
    lat.upload(gpu.Grid.from_bytes(n, cells))
    lat.step(steps)
    assert lat.download().to_bytes() == oracle.run(n, cells, steps)


@pytest.mark.parametrize("variant", [2, 4])
@pytest.mark.parametrize("strict", [False, True])
def test_wide_variant_metrics(gpu, oracle, variant, strict):
    n, steps = 2048, 40
    cells = oracle.init_grid(n, 0.4, 5)
    _, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, variant)
    lat.set_census(strict)
    lat.upload(gpu.Grid.from_bytes(n, cells))
    ms = lat.step_with_metrics(steps)
    assert [m.lr_moved for m in ms] == lm and [m.tb_moved for m in ms] == tm
    assert [m.lr_count for m in ms] == lc and [m.tb_count for m in ms] == tc


def test_wide_variant_rejected_when_connected(gpu):
    lat = gpu.DeviceLattice(2048, 2)  # bands are connected at construction
    lib = ctypes.CDLL(gpu.LIB_DEV)
    lib.bml_dev_set_variant.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert lib.bml_dev_set_variant(ctypes.c_void_p(lat.handle(0)), 2) == 1  # BML_EINVAL


def test_wide_variant_row_bands(gpu, oracle):
    """Two connected bands (bml_dev_create_band + connect_local), variant set on both
    before connecting, stepped in lockstep one launch at a time (14 steps each, plus
    narrow tail launches), against the oracle."""
    lib = ctypes.CDLL(gpu.LIB_DEV)
    vp = ctypes.c_void_p
    lib.bml_dev_create_band.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(vp)]
    lib.bml_dev_set_variant.argtypes = [vp, ctypes.c_int]
    lib.bml_dev_connect_local.argtypes = [vp, vp, vp]
    lib.bml_dev_upload.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    lib.bml_dev_download.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    lib.bml_dev_exchange_halos.argtypes = [vp]
    lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
    lib.bml_dev_sync.argtypes = [vp]
    lib.bml_dev_destroy.argtypes = [vp]
    n, steps = 2048, 14 * 3 + 5
    cells = oracle.init_grid(n, 0.35, 11)
    bounds = [(0, 1024), (1024, 2048)]
    hs = [vp(), vp()]
    try:
        for h, (b, e) in zip(hs, bounds):
            assert lib.bml_dev_create_band(n, b, e, 0, ctypes.byref(h)) == 0
            assert lib.bml_dev_set_variant(h, 2) == 0
        assert lib.bml_dev_connect_local(hs[0], hs[1], hs[1]) == 0
        assert lib.bml_dev_connect_local(hs[1], hs[0], hs[0]) == 0
        for h, (b, e) in zip(hs, bounds):
            assert lib.bml_dev_upload(h, cells[b * n:e * n], n) == 0
        for h in hs:
            assert lib.bml_dev_exchange_halos(h) == 0
        done = 0
        for k in [14, 14, 14, 4, 1]:
            for h in hs:
                assert lib.bml_dev_step(h, k, None, None, None, None) == 0
            done += k
        assert done == steps
        out = b""
        for h, (b, e) in zip(hs, bounds):
            buf = ctypes.create_string_buffer((e - b) * n)
            assert lib.bml_dev_download(h, buf, n) == 0
            out += buf.raw
        assert out == oracle.run(n, cells, steps)
    finally:
        for h in hs:
            lib.bml_dev_destroy(h)


# ----------------------------------------------------------- the stage-split kernel (variant 5)
@pytest.mark.parametrize("n,steps", [(2048, 45), (4096, 37), (8192, 33)])
def test_split_variant_matches_oracle(gpu, oracle, n, steps):
    cells = oracle.init_grid(n, 0.36, n + 5)
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, 5)
    lat.upload(gpu.Grid.from_bytes(n, cells))
    lat.step(steps)
    assert lat.download().to_bytes() == oracle.run(n, cells, steps)


@pytest.mark.parametrize("strict", [False, True])
def test_split_variant_metrics(gpu, oracle, strict):
    n, steps = 2048, 40
    cells = oracle.init_grid(n, 0.4, 6)
    _, (lm, tm, lc, tc) = oracle.run(n, cells, steps, metrics=True)
    lat = gpu.DeviceLattice(n)
    set_variant(gpu, lat, 5)
    lat.set_census(strict)
    lat.upload(gpu.Grid.from_bytes(n, cells))
    ms = lat.step_with_metrics(steps)
    assert [m.lr_moved for m in ms] == lm and [m.tb_moved for m in ms] == tm
    assert [m.lr_count for m in ms] == lc and [m.tb_count for m in ms] == tc


def test_split_variant_row_bands_env(gpu, oracle):
    """Row bands built by DeviceLattice with BML_VARIANT=5 in a subprocess (the
    variant must be set before the bands connect)."""
    import os
    import subprocess
    import sys

    n, steps = 2048, 50
    code = f"""
import sys; sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import paper_1804_07981_b200 as bml
lat = bml.DeviceLattice({n}, 4)
lat.init_random(0.35, 3)
lat.step({steps})
print(hex(lat.digest()))
"""
    env = dict(os.environ, BML_VARIANT="5")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    cells = oracle.init_grid(n, 0.35, 3)
    assert int(out.stdout.strip(), 16) == oracle.digest(n, oracle.run(n, cells, steps))
