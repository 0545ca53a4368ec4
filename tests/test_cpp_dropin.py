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
