"""bench.py's single-GPU JSON line at a small workload (configs[0], N=256): the driver
contract's keys, the roofline / cpu_baseline / e2e objects, and the in-line parity
check against the reference golden."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract_c0(gpu):
    out = subprocess.run([sys.executable, "bench.py", "--workload", "c0", "--steps", "3", "--warmup", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks", "parity"):
        assert k in line, k
    assert line["metric"] == "Gcell-updates/sec" and line["higher_is_better"] is True
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["value"] > 0
    assert line["config"]["workload"].startswith("configs[0]")
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert line["roofline_alu"]["bound"] == "alu"
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 256 * 256 and e["d2h_bytes_per_step"] == 256 * 256
    assert e["result_check"]["match"] and e["sync"]["result_check"]["match"]
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] > 0 and cb["cores"] >= 1
    assert line["parity"]["match"] is True
    assert line["gpu_launches"] >= 3
    assert "sm_mhz" in line["clocks"] and "reasons" in line["clocks"]
