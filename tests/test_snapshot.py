"""PPM snapshots (host encode_ppm / write_ppm, and DeviceLattice.encode_ppm on the GPU),
mirroring /root/reference/proj/tests/test_snapshot.cpp and python/test_smoke.py:67-71."""
import random
import re

import pytest


def decode_ppm(data):  # test-only decoder, independent of the encoder
    m = re.match(rb"P6\n(\d+) (\d+)\n255\n", data)
    assert m
    w, h = int(m.group(1)), int(m.group(2))
    assert w == h and len(data) == m.end() + 3 * w * h
    px = data[m.end():]
    table = {(255, 0, 0): 1, (0, 0, 255): 2, (255, 255, 255): 0}
    return w, bytes(table[tuple(px[i:i + 3])] for i in range(0, len(px), 3))


def test_one_by_one_empty(bml):  # test_snapshot.cpp:46-52
    assert bml.encode_ppm(bml.Grid.from_text(".")) == b"P6\n1 1\n255\n\xff\xff\xff"


def test_colors(bml):  # test_snapshot.cpp:54-64
    assert bml.encode_ppm(bml.Grid.from_text(">"))[-3:] == b"\xff\x00\x00"
    assert bml.encode_ppm(bml.Grid.from_text("v"))[-3:] == b"\x00\x00\xff"


@pytest.mark.parametrize("n", [1, 2, 9, 17, 40])
def test_roundtrip(bml, n):  # test_snapshot.cpp:66-84
    rng = random.Random(606 + n)
    cells = bytes(rng.randrange(3) for _ in range(n * n))
    data = bml.encode_ppm(bml.Grid.from_bytes(n, cells))
    assert decode_ppm(data) == (n, cells)


def test_ppm_bytes(bml):  # python/test_smoke.py:67-71
    data = bml.encode_ppm(bml.Grid.from_text(">v\n.."))
    assert data.startswith(b"P6\n2 2\n255\n")
    assert len(data) == 11 + 3 * 4


def test_write_ppm(bml, tmp_path):
    g = bml.Grid.from_text(">v\n..")
    p = tmp_path / "snap.ppm"
    bml.write_ppm(g, str(p))
    assert p.read_bytes() == bml.encode_ppm(g)
    with pytest.raises(RuntimeError, match="nonexistent"):
        bml.write_ppm(g, str(tmp_path / "nonexistent" / "x.ppm"))


@pytest.mark.gpu
@pytest.mark.parametrize("n,bands", [(1, 1), (33, 1), (100, 1), (1024, 1), (256, 4)])
def test_device_encode_ppm_matches_host(gpu, n, bands):
    bml = gpu
    rng = random.Random(n)
    cells = bytes(rng.randrange(3) for _ in range(n * n))
    lat = bml.DeviceLattice(n, devices=bands)
    lat.upload(bml.Grid.from_bytes(n, cells))
    lat.step(5)
    assert lat.encode_ppm() == bml.encode_ppm(lat.download())
