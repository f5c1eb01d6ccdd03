"""The drop-in C++ API (include/wheelsieve/*.hpp, libwheelsieve.so over the
C ABI) compiles on CPU, and its reference-mirroring test program passes on the
GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_gpu_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2310_17746_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_gpu_api")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                    SRC, "-o", exe, f"-L{LIBDIR}", "-lwheelsieve", "-lwheelsieve_cuda",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_cpp_api_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_parity(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[PASS] all checks" in r.stdout
