"""The C++ drop-in (include/admmgpu/admmgpu.hpp) compiles against the C ABI and, on a
GPU, passes the reference's restated Catch2 cases (tests/cpp/test_shim.cpp)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "tests", "cpp", "test_shim")


def build():
    subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), "liboracle.so"], check=True, capture_output=True)
    cmd = ["g++", "-std=c++17", "-O2", f"-I{REPO}/include", os.path.join(REPO, "tests", "cpp", "test_shim.cpp"),
           "-o", BIN, f"-L{REPO}/paper_1811_05571_b200", "-ladmm_b200", f"-L{REPO}/oracle", "-loracle",
           f"-Wl,-rpath,{REPO}/paper_1811_05571_b200", f"-Wl,-rpath,{REPO}/oracle"]
    subprocess.run(cmd, check=True, capture_output=True)


def test_cpp_shim_compiles():
    build()
    assert os.path.exists(BIN)


def test_cpp_shim_host_cases():
    """CMAT I/O through the shim (cmat_io.hpp names and exceptions) needs no device."""
    build()
    r = subprocess.run([BIN, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "0 failures" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_shim_reference_cases_on_device():
    build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
