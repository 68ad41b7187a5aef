"""CPU check of the segment formulation behind the device grid_digest (csrc/bml_digest.cu).

The reference hashes the cell bytes serially with FNV-1a-64
(/root/reference/proj/src/digest.cpp:5-14). Because cell bytes are 0/1/2, the
hash splits into a 4-state low-bit automaton plus an affine map, so chunks can be
hashed independently for the 4 possible incoming low-bit states and composed.
This file restates that algebra in Python (same Seg layout and combine rule) and
checks it against the oracle's FNV on random lattices and on every chunking.
"""
import random

import pytest

M = (1 << 64) - 1
P = 0x100000001B3
BASIS = 0xCBF29CE484222325


def fnv(data, h=BASIS):
    for b in data:
        h = ((h ^ b) * P) & M
    return h


def identity():
    return [1, [0, 0, 0, 0], [0, 1, 2, 3]]


def combine(x, y):
    pw = (x[0] * y[0]) & M
    b, out = [0] * 4, [0] * 4
    for s in range(4):
        m = x[2][s]
        b[s] = (x[1][s] * y[0] + y[1][m]) & M
        out[s] = y[2][m]
    return [pw, b, out]


def segment(data):
    g = identity()
    st = list(g[2])
    for byte in data:
        for s in range(4):
            x = st[s] ^ byte
            g[1][s] = ((g[1][s] + (x - st[s])) * P) & M
            st[s] = (x * 3) & 3
        g[0] = (g[0] * P) & M
    g[2] = st
    return g


def finish(segs):
    acc = identity()
    for s in segs:
        acc = combine(acc, s)
    return (BASIS * acc[0] + acc[1][BASIS & 3]) & M


@pytest.mark.parametrize("length", [0, 1, 2, 5, 31, 32, 33, 100])
def test_single_segment_equals_fnv(length):
    rng = random.Random(length)
    data = bytes(rng.randrange(3) for _ in range(length))
    assert finish([segment(data)]) == fnv(data)


@pytest.mark.parametrize("seed", range(6))
def test_any_chunking_composes(seed):
    rng = random.Random(seed)
    data = bytes(rng.randrange(3) for _ in range(257))
    cuts = sorted(rng.sample(range(1, 257), rng.randrange(1, 12)))
    parts = [data[a:b] for a, b in zip([0] + cuts, cuts + [257])]
    assert finish([segment(p) for p in parts]) == fnv(data)
    # tree-shaped composition (the device's block reduction) gives the same
    segs = [segment(p) for p in parts]
    while len(segs) > 1:
        segs = [combine(segs[i], segs[i + 1]) if i + 1 < len(segs) else segs[i]
                for i in range(0, len(segs), 2)]
    assert (BASIS * segs[0][0] + segs[0][1][BASIS & 3]) & M == fnv(data)


def test_matches_oracle_grid_digest(oracle):
    n = 37
    cells = oracle.init_grid(n, 0.4, 3)
    assert finish([segment(cells[r * n:(r + 1) * n]) for r in range(n)]) == oracle.digest(n, cells)


def test_fnv_known_answers():  # test_digest.cpp:16-20
    assert fnv(b"") == 0xCBF29CE484222325
    assert fnv(b"a") == 0xAF63DC4C8601EC8C
    assert fnv(b"foobar") == 0x85944171F73967E8
