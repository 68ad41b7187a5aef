"""CPU check of the parallel init_grid formulation used by csrc/bml_init.cu.

The device computes the reference's serial descending Fisher–Yates shuffle
(/root/reference/proj/src/seeding.cpp:26-51) as four data-parallel passes:
counter-based draws with a rejection fix-up, a stable sort of (j_i, i), one
links pass (first[] and link[]), and chain resolution. This file restates those
passes in numpy — same arrays, same rules — and checks them against the serial
oracle, so the algorithm itself is pinned without a GPU; test_gpu_init.py then
pins the CUDA code against the same oracle.
"""
import numpy as np
import pytest

GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def splitmix_at(seed, counter):
    z = (seed + counter * GAMMA) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def rejected(r, m, mask):
    excess = (1 << 64) % m
    return (excess != 0 and r >= (1 << 64) - excess) or (mask != 0 and (r & mask) == 0)


def parallel_init(n, rho, seed, mask=0):
    count = n * n
    k = int(np.floor(rho * float(n) * float(n) / 2.0))
    out = np.zeros(count, np.uint8)
    if k == 0:
        return out.tobytes()
    keys = np.zeros(count - 1, np.int64)
    vals = np.arange(1, count, dtype=np.int64)
    hi, off = count - 1, 0
    while True:  # draw passes (draw_kernel); each pass is "parallel" over i <= hi
        first_rej = 0
        for i in range(1, hi + 1):
            r = splitmix_at(seed, (count - 1 - i) + off + 1)
            if rejected(r, i + 1, mask):
                first_rej = max(first_rej, i)
            keys[i - 1] = r % (i + 1)
        if first_rej == 0:
            break
        hi, off = first_rej, off + 1
    order = np.argsort(keys, kind="stable")  # cub radix sort is stable
    sk, sv = keys[order], vals[order]
    first = np.zeros(count, np.int64)
    link = np.zeros(2 * k, np.int64)
    items = count - 1
    for m in range(items):  # links_kernel
        q, i = sk[m], sv[m]
        nxt = sv[m + 1] if m + 1 < items and sk[m + 1] == q else 0
        if m == 0 or sk[m - 1] != q:
            first[q] = i if i > q else nxt
        if i < 2 * k:
            link[i] = nxt if nxt else q

    def settle(x):
        while first[x]:
            x = first[x]
        return x

    for i in range(2 * k):  # scatter_kernel
        v = settle(0) if i == 0 else (settle(link[i]) if link[i] > i else link[i])
        out[v] = 1 if i < k else 2
    return out.tobytes()


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 13, 24])
@pytest.mark.parametrize("rho,seed", [(0.3, 1), (0.5, 42), (1.0, 9)])
def test_parallel_formulation_matches_serial_shuffle(oracle, n, rho, seed):
    assert parallel_init(n, rho, seed) == oracle.init_grid(n, rho, seed)


@pytest.mark.parametrize("n,mask", [(4, 0x1), (9, 0x3), (20, 0x7)])
def test_parallel_formulation_rejection_fixup(oracle, n, mask):
    assert parallel_init(n, 0.4, 5, mask) == oracle.init_grid_masked(n, 0.4, 5, mask)


def test_masked_oracle_hook_is_identity_at_zero(oracle):
    for n in (1, 7, 64):
        assert oracle.init_grid_masked(n, 0.35, 3, 0) == oracle.init_grid(n, 0.35, 3)
    a = oracle.init_grid_masked(64, 0.35, 3, 0xF)
    assert a != oracle.init_grid(64, 0.35, 3)
    assert a.count(1) == a.count(2) == oracle.init_grid(64, 0.35, 3).count(1)


def test_pinned_lattice_seed42_parallel():  # test_seeding.cpp:70-79
    cells = parallel_init(4, 0.5, 42)
    text = "".join(".>v"[c] for c in cells)
    assert [text[i:i + 4] for i in range(0, 16, 4)] == ["..>.", ">.vv", "v...", ">>v."]
