"""The C++ facade (include/oomb.hpp) compiled with g++ against liboomb.so, and its test
program tests/cpp/test_facade.cpp run in both modes: host-only cases here, device cases
on a B200 (-m gpu). The oracle library is the checker."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2602_02108_b200")
BIN = os.path.join(PKG, "_build", "test_facade")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build_facade_test() -> str:
    from oracle.oracle import build_port
    from paper_2602_02108_b200.build import build
    build()
    build_port()
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    oracle_dir = os.path.join(ROOT, "oracle")
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include", f"-I{CUDA}/include",
           os.path.join(ROOT, "tests", "cpp", "test_facade.cpp"), "-o", BIN, f"-L{PKG}", "-loomb", f"-L{oracle_dir}",
           "-loomb_oracle", f"-L{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{PKG}:{oracle_dir}:{CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return BIN


@pytest.fixture(scope="module")
def facade_bin():
    return build_facade_test()


def _run(binary, mode):
    r = subprocess.run([binary, mode], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


def test_facade_cpu(facade_bin):
    _run(facade_bin, "cpu")


@pytest.mark.gpu
def test_facade_gpu(facade_bin):
    _run(facade_bin, "gpu")
