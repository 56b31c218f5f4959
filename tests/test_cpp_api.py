"""The header-only C++ host API (include/shearlet_b200.hpp) compiles against
the C ABI, links libshearlet_b200.so, and (on the GPU) round-trips."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp")
LIBDIR = os.path.join(ROOT, "paper_1402_5670_b200")
EXE = os.path.join(ROOT, "tests", "cpp", "api_smoke")


def build_exe():
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR, "-lshearlet_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", EXE]
    subprocess.check_call(cmd)


def test_cpp_api_compiles_and_links():
    build_exe()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_api_round_trip(cuda):
    build_exe()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
