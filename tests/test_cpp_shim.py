"""The C++ drop-in header (include/scrooge_b200.hpp) compiles against the C ABI,
and on the GPU behaves like the reference API (tests/cpp/shim_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_test.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "_shim_test")


def build(sg):
    from paper_2208_09985_b200 import _ffi
    libdir = os.path.dirname(_ffi.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", f"-I{ROOT}/include", SRC,
                    f"-L{libdir}", "-lscrooge_b200", f"-Wl,-rpath,{libdir}", "-o", BIN],
                   check=True)
    return BIN


def test_cpp_shim_compiles(sg):
    assert os.path.exists(build(sg))


@pytest.mark.gpu
def test_cpp_shim_behaves_like_reference(gpu):
    out = subprocess.run([build(gpu)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ok (0 failures)" in out.stdout
