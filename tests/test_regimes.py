"""Phase-transition regimes, the reference's physics-level acceptance check.

acceptance_main.cpp criteria 3/4 (proj/tests/acceptance/acceptance_main.cpp:129-143):
N=256, 4096 steps, seeds 1..10; classify() over the last kClassifyWindow = 64
mobilities (metrics.hpp:41-45). The reference's recorded run
(proj/test_output.txt:7-8) shows FreeFlow in 10/10 seeds at rho=0.25
([++++++++++]) and Jammed in 4/10 at rho=0.38 ([--+--++-+-]).

tests/golden/regimes_n256_steps4096.json holds, per seed, the unmodified
reference's init/final digests, moved-vehicle sums and regime
(make_goldens.py regimes). CPU: the goldens against the recorded patterns and the
oracle. GPU: the device engine's fused-metrics path against every record.
"""
import json
import os
import re

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "regimes_n256_steps4096.json")
REF_OUTPUT = "/root/reference/proj/test_output.txt"
# proj/test_output.txt:7-8 (criteria 3 and 4 of the reference's acceptance run)
RECORDED = {0.25: ("FreeFlow", "++++++++++"), 0.38: ("Jammed", "--+--++-+-")}


def _records():
    with open(GOLDEN) as f:
        return json.load(f)["records"]


def _pattern(recs, rho, want):
    return "".join("+" if r["regime"] == want else "-"
                   for r in sorted((r for r in recs if r["rho"] == rho), key=lambda r: r["seed"]))


def test_golden_regimes_match_the_recorded_reference_run():
    recs = _records()
    assert len(recs) == 20
    for rho, (want, pattern) in RECORDED.items():
        assert _pattern(recs, rho, want) == pattern


def test_recorded_patterns_match_reference_output_file():
    if not os.path.exists(REF_OUTPUT):
        pytest.skip("reference tree not present on this host")
    with open(REF_OUTPUT) as f:
        text = f.read()
    for rho, (want, pattern) in RECORDED.items():
        m = re.search(rf"rho={rho:.2f} 4096 steps: {want} in \d+/10 seeds \[([+-]+)\]", text)
        assert m and m.group(1) == pattern


def test_oracle_reproduces_regime_init_and_final_digests(oracle):
    recs = _records()
    for r in recs:
        cells = oracle.init_grid(r["n"], r["rho"], r["seed"])
        assert f"0x{oracle.digest(r['n'], cells):016x}" == r["init_digest"]
    for r in (recs[0], recs[12]):  # one per density; 268M cell-updates each in C
        cells = oracle.init_grid(r["n"], r["rho"], r["seed"])
        final = oracle.run(r["n"], cells, r["steps"])
        assert f"0x{oracle.digest(r['n'], final):016x}" == r["final_digest"]


@pytest.mark.gpu
@pytest.mark.parametrize("rec", _records(), ids=lambda r: f"rho{r['rho']}_seed{r['seed']}")
def test_device_regimes_match_reference(gpu, rec):
    """bml.simulate (fused per-step metrics on the device) reproduces the reference's
    final lattice, moved-vehicle sums and classify() verdict for every seed."""
    bml = gpu
    grid = bml.init_grid(rec["n"], rec["rho"], rec["seed"])
    assert f"0x{grid.digest():016x}" == rec["init_digest"]
    final, metrics = bml.simulate(grid, rec["steps"])
    assert f"0x{final.digest():016x}" == rec["final_digest"]
    assert sum(m.lr_moved for m in metrics) == rec["sum_lr_moved"]
    assert sum(m.tb_moved for m in metrics) == rec["sum_tb_moved"]
    regime = bml.classify([m.mobility for m in metrics[-64:]])
    assert regime == getattr(bml.Regime, rec["regime"])
