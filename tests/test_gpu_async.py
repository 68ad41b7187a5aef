"""Asynchronous upload / download through the C-ABI (bml_dev_upload_async,
bml_dev_download_async): two handles pipelined on their own streams, as bench.py's
e2e leg does, must give the same lattices as the oracle; an invalid cell in an
asynchronous upload is reported by bml_dev_sync."""
import ctypes

import pytest

pytestmark = pytest.mark.gpu


def abi(gpu):
    lib = ctypes.CDLL(gpu.LIB_DEV)
    vp = ctypes.c_void_p
    lib.bml_dev_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    lib.bml_dev_destroy.argtypes = [vp]
    lib.bml_dev_upload_async.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    lib.bml_dev_download_async.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    lib.bml_dev_step.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp]
    lib.bml_dev_sync.argtypes = [vp]
    lib.bml_dev_last_error.restype = ctypes.c_char_p
    return lib


@pytest.mark.parametrize("n,steps", [(96, 37), (1000, 20), (2048, 33)])
def test_pipelined_handles_match_oracle(gpu, oracle, n, steps):
    lib = abi(gpu)
    hs = [ctypes.c_void_p(), ctypes.c_void_p()]
    for h in hs:
        assert lib.bml_dev_create(n, 0, ctypes.byref(h)) == 0
    try:
        jobs = [oracle.init_grid(n, 0.35, seed) for seed in (1, 2, 3, 4)]
        outs = [ctypes.create_string_buffer(n * n) for _ in jobs]
        ins = [ctypes.create_string_buffer(j, n * n) for j in jobs]
        for i in range(len(jobs)):
            h = hs[i % 2]
            assert lib.bml_dev_upload_async(h, ins[i], n) == 0
            assert lib.bml_dev_step(h, steps, None, None, None, None) == 0
            assert lib.bml_dev_download_async(h, outs[i], n) == 0
        for h in hs:
            assert lib.bml_dev_sync(h) == 0, lib.bml_dev_last_error()
        for j, o in zip(jobs, outs):
            assert o.raw[: n * n] == oracle.run(n, j, steps)
    finally:
        for h in hs:
            lib.bml_dev_destroy(h)


def test_async_upload_reports_bad_cell_at_sync(gpu):
    lib = abi(gpu)
    h = ctypes.c_void_p()
    assert lib.bml_dev_create(64, 0, ctypes.byref(h)) == 0
    try:
        bad = bytearray(64 * 64)
        bad[100] = 3
        buf = ctypes.create_string_buffer(bytes(bad), 64 * 64)
        assert lib.bml_dev_upload_async(h, buf, 64) == 0
        assert lib.bml_dev_sync(h) == 1  # BML_EINVAL
        assert b"outside" in lib.bml_dev_last_error()
        good = ctypes.create_string_buffer(64 * 64)
        assert lib.bml_dev_upload_async(h, good, 64) == 0
        assert lib.bml_dev_sync(h) == 0
    finally:
        lib.bml_dev_destroy(h)
