"""The light-cone tiling that produced the configs[4] 10000-step golden
(tests/golden/tile_chain.py) is exact: run on the reference itself, with ragged and
square tiles, it reproduces the unbroken reference's committed goldens, including
the checkpoint digests of a chained golden. (The configs[4] run itself was pinned the
same way: its first 1000-step leg equals the unbroken 1000-step golden,
tests/golden/tile_chain_c4_legs.jsonl.)"""
import json
import os
import subprocess
import sys

import pytest

from conftest import REF_DRIVER, ROOT

GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.mark.skipif(not os.path.exists(REF_DRIVER), reason="oracle/_ref not built")
@pytest.mark.parametrize("n,rho,seed,steps,leg,tile", [
    (1000, 0.25, 3, 512, 100, 300),   # ragged tiles (1000 = 3 x 300 + 100), a short last leg
    (2048, 0.35, 1, 256, 64, 512),    # 16 square tiles
])
def test_tiled_reference_run_matches_the_unbroken_golden(tmp_path, n, rho, seed, steps, leg, tile):
    golden = os.path.join(GOLDEN, f"ref_n{n}_rho{rho}_seed{seed}_steps{steps}.json")
    out = tmp_path / "out.json"
    subprocess.run([sys.executable, os.path.join(GOLDEN, "tile_chain.py"), str(n), str(rho), str(steps),
                    str(leg), str(tile), str(tmp_path / "work"), "--seed", str(seed), "--jobs", "4",
                    "--check", golden, "--out", str(out)], check=True, capture_output=True, timeout=600)
    got, want = json.load(open(out)), json.load(open(golden))
    assert got["final_digest"] == want["final_digest"]
    assert (got["lr_count"], got["tb_count"]) == (want["lr_count"], want["tb_count"])
    assert got["pinned_against_unbroken_reference"] == [steps]


def test_c4_chain_leg_one_is_the_unbroken_golden():
    legs = [json.loads(l) for l in open(os.path.join(GOLDEN, "tile_chain_c4_legs.jsonl"))]
    one = json.load(open(os.path.join(GOLDEN, "ref_n65536_rho0.35_seed1_steps1000.json")))
    ten = json.load(open(os.path.join(GOLDEN, "ref_n65536_rho0.35_seed1_steps10000.json")))
    assert legs[0]["at_step"] == 1000 and legs[0]["digest"] == one["final_digest"]
    assert legs[0]["matches_unbroken_reference"] is True
    assert [c["digest"] for c in ten["checkpoints"]] == [l["digest"] for l in legs]
    assert ten["final_digest"] == legs[-1]["digest"] and ten["init_digest"] == one["init_digest"]
