"""bench.py host logic on CPU: lattice sizes of the scaling modes, golden lookup, the
reference arm's bounded sampling plan, and the reference arm end to end at configs[0]
(the unmodified reference through oracle/_ref/ref_driver's init-once ladder)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_strong_scaling_keeps_n():
    for g in (1, 2, 4, 8):
        assert bench.bench_n("c4", 65536, g, "strong") == 65536
        assert bench.bench_n("c3", 32768, g, "strong") == 32768


def test_square_weak_sweep_sizes():
    assert [bench.bench_n("c4", 65536, g, "weak") for g in (1, 2, 4, 8)] == [23168, 32768, 46336, 65536]
    assert bench.bench_n("c1", 1024, 2, "weak") == 1440  # ~2x the cells, side a multiple of 32


def test_band_split_matches_reference_parallel_rows():  # engine.cpp:131-137
    from paper_1804_07981_b200.dist import band_rows, check_partition

    for g in (2, 4, 8):
        check_partition(65536, g)
        rows = [band_rows(65536, g, r) for r in range(g)]
        assert rows[0][0] == 0 and rows[-1][1] == 65536
        assert all(e - b == 65536 // g for b, e in rows)


def test_find_golden():
    g = bench.find_golden(65536, 0.35, 1, 10000)
    assert g is not None and g["init_digest"] == "0x251caaf18a5a5a71"
    assert g["steps"] in (1000, 10000)
    assert bench.find_golden(1024, 0.38, 1, 4096)["final_digest"] == "0x1927af4d802408ce"
    assert bench.find_golden(12345, 0.35, 1, 10) is None


def test_cpu_sample_plan_is_bounded():
    plan = dict((b, (t, st, r)) for b, t, st, r in bench.cpu_sample_plan(65536, 10000, 20))
    assert plan["lanes"] == (1, 1, 20)       # one step of 4.3 Gcells per rep
    assert plan["parallel"][2] == 3 and plan["halo"][2] == 1 and plan["naive"][2] == 1
    small = dict((b, (t, st, r)) for b, t, st, r in bench.cpu_sample_plan(256, 1024, 5))
    assert small["lanes"] == (1, 1024, 5)    # the whole run when it is cheap


@pytest.mark.skipif(not os.path.exists(bench.REF_DRIVER), reason="oracle/_ref not built")
def test_reference_arm_line_c0():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c0",
                          "--steps", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["metric"] == "Gcell-updates/sec" and line["higher_is_better"]
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["input_check"]["match"] is True  # the reference's own init digest
