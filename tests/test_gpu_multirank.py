"""The multi-rank bench path end to end: `bench.py --gpus 2` under
torch.distributed.run, two ranks, each owning a row band, ghost rows exchanged inside the
step kernel over CUDA-IPC peer mappings. On a one-GPU box both ranks share the GPU
(gloo bootstrap). The combined device digest of the final torus must equal a single-band
run of the same lattice (init_grid on the device, same step count)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_bench_matches_single_band(gpu):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", "bench.py", "--gpus", "2",
           "--steps", "1", "--warmup", "3"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    final = line["final"]
    assert final["conserved"]
    n, rho, seed, steps = line["config"]["n"], line["config"]["rho"], line["config"]["seed"], final["steps"]
    lat = gpu.DeviceLattice(n)
    lat.init_random(rho, seed)
    lat.step(steps)
    assert final["digest"] == f"0x{lat.digest():016x}"
    assert list(lat.counts()) == final["vehicles"]
