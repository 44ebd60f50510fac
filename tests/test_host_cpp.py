"""The C++ host wrapper (paper_2410_09497_b200/host/stokesmg_b200.hpp) over the C ABI: it compiles and
links against libsmg_b200.so on CPU; under -m gpu the example caller runs and checks itself."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "host_wrapper_check.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "build", "host_wrapper_check")
LIBDIR = os.path.join(ROOT, "paper_2410_09497_b200")


def build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), SRC,
                           "-L", LIBDIR, "-lsmg_b200", f"-Wl,-rpath,{LIBDIR}", "-o", BIN])
    return BIN


def test_host_wrapper_compiles_and_links():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_host_wrapper_runs():
    out = subprocess.run([build()], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "host wrapper ok" in out.stdout
