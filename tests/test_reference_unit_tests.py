"""The reference project's own C++ unit tests, run against this library.

tests/ref_unit/Makefile compiles /root/reference/proj/tests/test_{grid,digest,seeding,
metrics,snapshot,verify,engine,reference}.cpp in place — unmodified, nothing copied — against
paper_1804_07981_b200/csrc/host/include (namespace bml) and links them with
libbml_b200.so, using tests/ref_unit/doctest.h (our doctest-compatible harness).
That is the drop-in claim for the C++ surface checked by the reference's own
assertions: the same call sites compile and the same expectations hold.

test_engine.cpp additionally gets two reference-internal kernel names from
tests/ref_unit/detail_shim.{hpp,cpp} (implemented on the device step_phase).

CPU: every host-only case (grid layout, parse/render, digest, splitmix/bounded,
init_grid pinned placement, metrics, PPM, rule truth tables, validation, the
brute-force model's own cases). The 13 cases that step a lattice need the device:
they run in the GPU test from the prebuilt binary (the GPU box has no
/root/reference).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
HERE = os.path.join(ROOT, "tests", "ref_unit")
BINARY = os.path.join(HERE, "_build", "ref_unit_tests")
# cases that step a lattice; names are globs, comma separated
DEVICE_CASES = ",".join([
    "vacuum mobility is 1", "a never-blocked*", "verify_backends*",            # test_metrics, test_verify
    "horizontal phase on a single-row*", "full steps on 2x2*", "all backends agree*",  # test_engine
    "swar lane kernel*", "vehicle counts are conserved*", "phase purity*", "per phase*",
    "step commutes*", "ParallelRows is deterministic*", "run honors steps*",
])
N_DEVICE_CASES = 13


def _build():
    if not os.path.isdir(REF_TESTS):
        pytest.skip("reference sources not present on this host")
    subprocess.run(["make", "-C", HERE, "-s", f"REF={os.path.dirname(REF_TESTS)}"], check=True,
                   capture_output=True)
    return BINARY


def _run(*args):
    return subprocess.run([BINARY, *args], capture_output=True, text=True, timeout=600)


def test_harness_detects_failures_and_walks_subcases(tmp_path):
    """The harness itself: a failing CHECK fails the run; each SUBCASE runs exactly once."""
    src = tmp_path / "t.cpp"
    src.write_text(
        '#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include "doctest.h"\n#include <cstdio>\n'
        "static int entries = 0;\n"
        'TEST_CASE("subcases") { ++entries; int hits = 0;\n'
        '  SUBCASE("a") { ++hits; } SUBCASE("b") { ++hits; } SUBCASE("c") { ++hits; }\n'
        "  CHECK(hits == 1); }\n"
        'TEST_CASE("entries") { CHECK(entries == 3); }\n'
        'TEST_CASE("throws") { CHECK_THROWS_AS(throw 1, int); CHECK_NOTHROW((void)0); }\n'
        'TEST_CASE("fails") { CHECK(1 + 1 == 3); }\n')
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", f"-I{HERE}", str(src), "-o", str(exe)], check=True)
    ok = subprocess.run([str(exe), "--test-case-exclude=fails"], capture_output=True, text=True)
    assert ok.returncode == 0, ok.stdout + ok.stderr
    assert "3 passed, 0 failed, 1 skipped" in ok.stdout
    bad = subprocess.run([str(exe)], capture_output=True, text=True)
    assert bad.returncode == 1 and "1 + 1 == 3" in bad.stderr


def test_reference_host_unit_tests_pass():
    _build()
    r = _run(f"--test-case-exclude={DEVICE_CASES}")
    assert r.returncode == 0, r.stdout + r.stderr
    summary = r.stdout.strip().splitlines()[-1]
    assert f", 0 failed, {N_DEVICE_CASES} skipped" in summary, summary
    passed = int(summary.split("test cases: ")[1].split(" passed")[0])
    assert passed >= 39, summary


@pytest.mark.gpu
def test_reference_unit_tests_on_the_device(gpu):
    """All built reference cases, including the three that step lattices through run()
    and verify_backends() with the reference's backend names."""
    if not os.path.exists(BINARY):
        pytest.skip("tests/ref_unit/_build/ref_unit_tests was not prebuilt (needs /root/reference)")
    r = _run()
    assert r.returncode == 0, r.stdout + r.stderr
    summary = r.stdout.strip().splitlines()[-1]
    assert ", 0 failed, 0 skipped" in summary, summary


# ----------------------------------------------------------- the reference's Python smoke tests
REF_PY_TESTS = "/root/reference/proj/tests/python/test_smoke.py"
# cases that step a lattice (need the device); run on a B200 as recorded in
# profiles/r1_reference_python_smoke_b200.txt
REF_PY_DEVICE_CASES = "single_step_golden or backends_agree or simulate_metrics or verify_backends"


def reference_python_smoke(tmp_dir, select=None):
    """Run the reference's tests/python/test_smoke.py, unmodified and in place, with
    `import bml` resolving to this package (a one-line alias package in tmp_dir)."""
    pkg = os.path.join(tmp_dir, "bml")
    os.makedirs(pkg, exist_ok=True)
    with open(os.path.join(pkg, "__init__.py"), "w") as f:
        f.write("from paper_1804_07981_b200 import *  # noqa: F401,F403\n"
                "from paper_1804_07981_b200 import __all__, __version__  # noqa: F401\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([tmp_dir, ROOT]), PYTHONDONTWRITEBYTECODE="1")
    env.pop("BML_CLI", None)  # the reference CLI is out of scope
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", tmp_dir,
           REF_PY_TESTS]
    if select:
        cmd += ["-k", select]
    return subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=tmp_dir, timeout=600)


def test_reference_python_smoke_host_cases(tmp_path):
    if not os.path.exists(REF_PY_TESTS):
        pytest.skip("reference sources not present on this host")
    r = reference_python_smoke(str(tmp_path), select=f"not ({REF_PY_DEVICE_CASES})")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "4 passed" in r.stdout, r.stdout
