"""The reference project's own C++ unit tests, run against this library.

tests/ref_unit/Makefile compiles /root/reference/proj/tests/test_{grid,digest,seeding,
metrics,snapshot,verify}.cpp in place — unmodified, nothing copied — against
paper_1804_07981_b200/csrc/host/include (namespace bml) and links them with
libbml_b200.so, using tests/ref_unit/doctest.h (our doctest-compatible harness).
That is the drop-in claim for the C++ surface checked by the reference's own
assertions: the same call sites compile and the same expectations hold.

CPU: every host-only case (grid layout, parse/render, digest, splitmix/bounded,
init_grid pinned placement, metrics, PPM). The three cases that step a lattice
(test_metrics.cpp:47, :62 and test_verify.cpp:8) need the device: they run in the
GPU test from the prebuilt binary (the GPU box has no /root/reference).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
HERE = os.path.join(ROOT, "tests", "ref_unit")
BINARY = os.path.join(HERE, "_build", "ref_unit_tests")
DEVICE_CASES = "vacuum mobility is 1,a never-blocked*,verify_backends*"


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
    assert ", 0 failed, 3 skipped" in summary, summary
    passed = int(summary.split("test cases: ")[1].split(" passed")[0])
    assert passed >= 28, summary


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
