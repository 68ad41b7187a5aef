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


def run_bench(nproc, *args, timeout=900, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", "bench.py", "--gpus", str(nproc),
           *args]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                         env=None if env is None else {**os.environ, **env})
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])


def single_band_digest(gpu, n, rho, seed, steps):
    lat = gpu.DeviceLattice(n)
    lat.init_random(rho, seed)
    lat.step(steps)
    return f"0x{lat.digest():016x}", list(lat.counts())


def test_two_rank_bench_matches_single_band(gpu):
    line = run_bench(2, "--workload", "c1", "--scaling", "weak", "--steps", "1", "--warmup", "3")
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    par = line["parity"]
    assert par["conserved"]
    cfg = line["config"]
    assert cfg["n"] == 1440  # ~2x the cells of N=1024, side a multiple of 32
    digest, counts = single_band_digest(gpu, cfg["n"], cfg["rho"], cfg["seed"], par["steps"])
    assert par["digest"] == digest
    assert counts == par["vehicles"]


@pytest.mark.parametrize("ranks", [2, 3])
def test_even_odd_row_bands_match_single_band(gpu, ranks):
    """The even/odd-layout kernel on connected row bands (BML_VARIANT=6 forces it at
    N=8192): each rank converts its rows in place, and its ghost rows once the
    neighbours' flags say their last launch wrote them; 10000 steps per run."""
    line = run_bench(ranks, "--workload", "c2ff", "--steps", "1", "--warmup", "1", "--no-cpu",
                     env={"BML_VARIANT": "6"})
    cfg = line["config"]
    assert cfg["n"] == 8192
    par = line["parity"]
    digest, counts = single_band_digest(gpu, cfg["n"], cfg["rho"], cfg["seed"], par["steps"])
    assert par["digest"] == digest
    assert counts == par["vehicles"]


@pytest.mark.slow
@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_c4_strong_split_matches_single_band(gpu, ranks):
    """configs[4]: N=65536 split into `ranks` row bands of ceil(N/g) rows (the default
    --scaling strong), 10000 steps; the combined digest equals the single-band run."""
    line = run_bench(ranks, "--workload", "c4", "--steps", "1", "--warmup", "1", "--no-cpu")
    assert line["config"]["n"] == 65536 and line["scaling"] == "strong"
    par = line["parity"]
    assert par["conserved"] and par["steps"] == 10000
    if par["expected_final"] is not None:  # the reference's own 10000-step golden
        assert par["match"], par
    digest, _ = single_band_digest(gpu, 65536, 0.35, 1, 10000)
    assert par["digest"] == digest


@pytest.mark.slow
def test_c3_eight_bands_match_reference_golden(gpu):
    """configs[3]: N=32768 over 8 row bands, 10000 steps, against the unmodified
    reference's golden digest (tests/golden/ref_n32768_rho0.35_seed1_steps10000.json)."""
    line = run_bench(8, "--workload", "c3", "--steps", "1", "--warmup", "1", "--no-cpu")
    assert line["config"]["n"] == 32768
    par = line["parity"]
    assert par["expected_final"] is not None and par["match"], par


@pytest.mark.slow
def test_c4_weak_sweep_sizes(gpu):
    """The square weak sweep: g=2 runs N=32768 (configs[3]'s
    lattice), so its digest is pinned by the reference golden."""
    line = run_bench(2, "--workload", "c4", "--scaling", "weak", "--steps", "1", "--warmup", "1",
                     "--no-cpu")
    assert line["config"]["n"] == 32768 and line["scaling"] == "weak"
    assert line["parity"]["match"], line["parity"]
