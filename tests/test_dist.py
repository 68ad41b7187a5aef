"""Multi-rank row bands: host logic on CPU (gloo, world_size 2) and, on a GPU box,
two processes sharing one GPU through CUDA IPC (the same code path 8 GPUs use).

Model: the reference's ParallelRows determinism test (test_engine.cpp:201-211) —
results must not depend on the number of bands.
"""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

from conftest import ROOT

sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_band_rows_partition():
    from paper_1804_07981_b200.dist import band_rows, check_partition, neighbour_ranks

    for n, world in ((1024, 1), (1024, 2), (1000, 3), (65536, 8), (100, 6), (33, 2)):
        spans = [band_rows(n, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        band = (n + world - 1) // world
        assert all(e - b <= band for b, e in spans)
    check_partition(1024, 8)
    with pytest.raises(ValueError):
        check_partition(100, 8)  # 13-row bands are thinner than the 16-row ghost depth
    assert neighbour_ranks(0, 4) == (3, 1) and neighbour_ranks(3, 4) == (2, 0)
    assert neighbour_ranks(0, 1) == (0, 0)


def test_weak_scaled_n():
    from paper_1804_07981_b200.dist import weak_scaled_n

    assert weak_scaled_n(1024, 1) == 1024
    assert weak_scaled_n(1024, 4) == 2048
    for g in (2, 8):
        n = weak_scaled_n(1024, g)
        assert n % 32 == 0 and abs(n * n / (1024 * 1024 * g) - 1) < 0.03


def _gloo_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1804_07981_b200.dist import exchange_blobs, neighbour_ranks

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    blobs = exchange_blobs(f"blob-of-rank-{rank}".encode())
    up, down = neighbour_ranks(rank, world)
    out[rank] = (blobs[up].decode(), blobs[down].decode(), len(blobs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_blob_exchange_gloo(world):
    mgr = mp.get_context("spawn").Manager()  # no fork() of a CUDA-initialised process
    out = mgr.dict()
    mp.spawn(_gloo_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        up, down, count = out[r]
        assert count == world
        assert up == f"blob-of-rank-{(r - 1) % world}"
        assert down == f"blob-of-rank-{(r + 1) % world}"


def _gpu_worker(rank, world, port, n, steps, out):
    import torch
    import torch.distributed as dist

    import paper_1804_07981_b200 as bml
    from paper_1804_07981_b200.dist import BandLattice

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    cells = bml.init_grid(n, 0.38, 5).to_bytes()
    band = BandLattice(n, rank, world, device=0)
    band.upload_rows(cells[band.begin * n: band.end * n])
    band.exchange_halos()
    band.step(steps)
    band.synchronize()
    out[rank] = band.download_rows()
    dist.barrier()
    band.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_two_processes_one_gpu_ipc_bands(world, oracle):
    import paper_1804_07981_b200 as bml

    if bml.device_count() < 1:
        pytest.skip("no CUDA device")
    n, steps = 512, 45
    mgr = mp.get_context("spawn").Manager()  # no fork() of a CUDA-initialised process
    out = mgr.dict()
    mp.spawn(_gpu_worker, args=(world, _free_port(), n, steps, out), nprocs=world, join=True)
    got = b"".join(out[r] for r in range(world))
    cells = oracle.init_grid(n, 0.38, 5)
    assert got == oracle.run(n, cells, steps)
