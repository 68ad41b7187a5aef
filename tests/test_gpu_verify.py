"""verify_backends over the device code paths (csrc/host/verify.cpp), mirroring the
reference's test_verify.cpp:8-22 and python/test_smoke.py verify case: four runs from one
init_grid lattice, per-step conservation, identical digests, cell-for-cell agreement."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,rho,steps,seed", [(33, 0.5, 20, 7), (49, 0.35, 21, 2), (64, 0.38, 45, 1),
                                              (65, 0.3, 19, 4), (66, 0.4, 17, 5), (69, 0.35, 23, 6),
                                              (100, 0.3, 33, 3), (1024, 0.38, 50, 1)])
def test_four_identical_digests(gpu, oracle, n, rho, steps, seed):
    report = gpu.verify_backends(n, rho, steps, seed, 2)
    assert report.ok and report.conserved and report.mismatch is None
    assert list(report.digests) == ["b200", "b200-streaming", "b200-phases", "b200-bands"]
    want = oracle.digest(n, oracle.run(n, oracle.init_grid(n, rho, seed), steps))
    assert set(report.digests.values()) == {want}


def test_tiny_lattice(gpu):
    report = gpu.verify_backends(2, 0.5, 5)
    assert report.ok and len(set(report.digests.values())) == 1


def test_reference_python_case(gpu):  # tests/python/test_smoke.py:60-64
    report = gpu.verify_backends(n=17, rho=0.5, steps=10, seed=3, threads=2)
    assert report.ok
    assert report.conserved
    assert len(set(report.digests.values())) == 1
