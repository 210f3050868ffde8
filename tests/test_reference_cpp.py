"""The drop-in boundary, C++ side: the reference's OWN unit tests
(/root/reference/proj/tests/test_{core_model,scheduler,desim,workload,
metrics}.cpp, 66 test cases) compile unchanged against this repo's pdsim
headers (include/pdsim) and link against libdualpath.so, and pass.  doctest
is not shipped with the reference (proj/vendor is absent), so the tests build
against tests/doctest_shim/doctest.h, a restated subset of its macros.

Runs where /root/reference exists (this container); skipped elsewhere."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
LIBDIR = os.path.join(ROOT, "paper_2602_21548_b200")
CASES = {"core_model": 7, "scheduler": 19, "desim": 19, "workload": 12, "metrics": 9}


def build(src, out):
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "tests", "doctest_shim"),
           "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR, "-ldualpath",
           f"-Wl,-rpath,{LIBDIR}", "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


@pytest.mark.parametrize("name", sorted(CASES))
def test_reference_unit_tests_pass_against_this_build(tmp_path, name):
    src = os.path.join(REF_TESTS, f"test_{name}.cpp")
    if not os.path.exists(src):
        pytest.skip("/root/reference is not present here")
    exe = str(tmp_path / f"ref_{name}")
    build(src, exe)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    n = CASES[name]
    assert f"test cases: {n} | {n} passed | 0 failed" in res.stdout, res.stdout


def test_shim_reports_failures(tmp_path):
    """The shim is a checker that can fail: a failing CHECK, a REQUIRE that
    aborts its case and a wrong exception type all count."""
    src = tmp_path / "bad.cpp"
    src.write_text('#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include <doctest.h>\n'
                   'TEST_CASE("a") { CHECK(1 + 1 == 3); CHECK(2.0 == doctest::Approx(2.0 + 1e-9)); }\n'
                   'TEST_CASE("b") { REQUIRE(false); CHECK(true); }\n'
                   'TEST_CASE("c") { CHECK_THROWS_AS(throw std::runtime_error("x"), std::out_of_range); }\n'
                   'TEST_CASE("d") { CHECK(1.0 == doctest::Approx(1.1).epsilon(0.2)); }\n')
    exe = str(tmp_path / "bad")
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "tests", "doctest_shim"), str(src), "-o", exe],
                   check=True, capture_output=True)
    res = subprocess.run([exe], capture_output=True, text=True)
    assert res.returncode == 1
    assert "test cases: 4 | 1 passed | 3 failed" in res.stdout
