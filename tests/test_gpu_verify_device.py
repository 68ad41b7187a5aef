"""verify_device: the device cross-check as its own entry point,
with every device code path including the even/odd-layout kernel; verify_backends keeps
the reference's four slots."""
import pytest

pytestmark = pytest.mark.gpu

ALL = ["b200", "b200-streaming", "b200-even-odd", "b200-phases", "b200-bands"]


@pytest.mark.parametrize("n,rho,steps,seed", [(64, 0.38, 45, 1), (2048, 0.35, 60, 2), (2112, 0.3, 70, 5),
                                              (1000, 0.5, 57, 3)])
def test_verify_device_all_paths_agree(gpu, n, rho, steps, seed):
    report = gpu.verify_device(n, rho, steps, seed)
    assert report.ok, report.mismatch
    assert list(report.digests) == ALL
    assert len(set(report.digests.values())) == 1


def test_verify_device_matches_the_reference_golden(gpu):
    """N=1024 rho=.38 4096 steps (configs[1]): every path lands on the unmodified
    reference's digest (tests/golden/ref_n1024_rho0.38_seed1_steps4096.json)."""
    import json
    import os

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                    "ref_n1024_rho0.38_seed1_steps4096.json")))
    report = gpu.verify_device(1024, 0.38, 4096, 1, ["b200", "b200-streaming", "b200-bands"])
    assert report.ok
    assert {f"0x{d:016x}" for d in report.digests.values()} == {g["final_digest"]}


def test_verify_device_subset_and_unknown_path(gpu):
    report = gpu.verify_device(2048, 0.35, 56, 1, ["b200-even-odd", "b200-streaming"])
    assert report.ok and list(report.digests) == ["b200-even-odd", "b200-streaming"]
    with pytest.raises(ValueError):
        gpu.verify_device(64, 0.3, 4, 1, ["b200", "lanes"])


def test_verify_backends_keeps_four_slots(gpu):
    report = gpu.verify_backends(2048, 0.35, 60, 1)
    assert report.ok and len(report.digests) == 4
