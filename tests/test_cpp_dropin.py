"""The drop-in C++ header compiles and links exactly as a reference user would use it;
on a GPU the acceptance program (reference acceptance.cpp pattern) must pass."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "acceptance_b200.cpp")
BIN = os.path.join(ROOT, "build", "acceptance_b200")
LIBDIR = os.path.join(ROOT, "paper_2001_05585_b200")


def compile_acceptance():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN,
                    "-L", LIBDIR, "-ltcreduce_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return BIN


def test_dropin_header_compiles_and_links():
    assert os.path.exists(compile_acceptance())


@pytest.mark.gpu
def test_acceptance_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([compile_acceptance()], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


REF_TESTS = os.path.join(ROOT, "oracle", "_ref", "ref_tests_b200")


@pytest.mark.gpu
def test_reference_unit_tests_pass_against_dropin():
    """The reference's own unit tests (proj/tests/test_reduction.cpp + test_harness.cpp, 26 test
    cases), compiled unchanged against include/tcreduce/reduction.hpp by oracle/Makefile (built
    by __graft_entry__.build() where /root/reference exists; the binary travels in oracle/_ref),
    run every reduction on the B200 and must all pass."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if not os.path.exists(REF_TESTS):
        pytest.skip("oracle/_ref/ref_tests_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([REF_TESTS], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
    assert "26 test cases, 0 failed" in r.stdout


REF_ACCEPT = os.path.join(ROOT, "oracle", "_ref", "ref_acceptance_b200")


@pytest.mark.gpu
def test_reference_acceptance_suite_against_dropin():
    """The reference's acceptance suite (proj/tests/acceptance.cpp) compiled unchanged against
    the drop-in header reproduces the reference's own run criterion by criterion, detail text
    included (tests/golden/reference_acceptance.txt, tools/make_acceptance_golden.sh): 1-4, 6-8
    and 10 PASS; 5 FAILS exactly as the reference does (its recurrence at curve_config m=4 R=5
    B=32 overflows binary16 on integer inputs: "got inf (overflow)"); 9 needs the reference CLI
    (absent CLI11, out of scope)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if not os.path.exists(REF_ACCEPT):
        pytest.skip("oracle/_ref/ref_acceptance_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([REF_ACCEPT], capture_output=True, text=True, timeout=1800)
    print(r.stdout)
    got = [ln for ln in r.stdout.splitlines() if ln.startswith("criterion")]
    want = [ln for ln in open(os.path.join(ROOT, "tests", "golden", "reference_acceptance.txt")).read().splitlines()
            if ln.startswith("criterion")]
    assert len(got) == len(want) == 10, r.stdout + r.stderr
    assert got == want
