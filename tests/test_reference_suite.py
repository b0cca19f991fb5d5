"""CPU: the reference's OWN test suite compiled unchanged against the B200
headers (paper_2605_23389_b200/include/prefixsim) — the drop-in proof that the
batcher / scheduler / prefetcher / operator / config APIs are the reference's.

  * proj/tests/test_*.cpp (72 Catch2 cases) with the Catch2-subset shim in
    tests/cpp/catch2/catch.hpp;
  * proj/tests/acceptance.cpp (10 quantitative criteria, PASS/FAIL lines).
Skipped where /root/reference is absent (the GPU box).  Binaries are cached in
/tmp keyed by a hash of the headers and test sources.
"""
import glob
import hashlib
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference sources absent")

INCLUDES = ["-I" + os.path.join(ROOT, "tests", "cpp"), "-I" + os.path.join(ROOT, "paper_2605_23389_b200", "include"),
            "-I" + os.path.join(ROOT, "third_party", "nlohmann"), "-I" + REF_TESTS]


def _key(sources):
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(ROOT, "paper_2605_23389_b200", "include", "prefixsim", "*.hpp"))) + \
            sorted(sources) + [os.path.join(ROOT, "tests", "cpp", "catch2", "catch.hpp")]:
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def _build(name, sources, extra=()):
    out = f"/tmp/asv_reftest_{name}_{_key(sources)}"
    if not os.path.exists(out):
        cmd = ["g++", "-std=c++20", "-O1", "-ffp-contract=off", *INCLUDES, *extra, *sources, "-o", out]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_reference_unit_tests_pass_against_b200_headers():
    main = "/tmp/asv_catch_main.cpp"
    with open(main, "w") as f:
        f.write("#define CATCH_CONFIG_MAIN\n#include <catch2/catch.hpp>\n")
    srcs = sorted(glob.glob(os.path.join(REF_TESTS, "test_*.cpp")))
    exe = _build("unit", [main] + srcs, [f'-DPREFIXSIM_FIXTURE_DIR="{REF_TESTS}/fixtures"'])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-400:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "72 passed | 0 failed" in r.stdout


def test_reference_acceptance_suite_passes_against_b200_headers():
    exe = _build("acceptance", [os.path.join(REF_TESTS, "acceptance.cpp")])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0
    assert r.stdout.count("[PASS]") == 10
