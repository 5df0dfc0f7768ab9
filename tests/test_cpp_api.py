"""The C++ host API (include/h2b200.hpp over include/h2c.h) compiles against the
library (CPU) and passes the reference's restated cases on the B200 (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "b200_api_test")


def build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O3", "-march=x86-64-v3", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
                    "-I/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "b200_api_test.cpp"),
                    "-L" + os.path.join(ROOT, "paper_2003_10173_b200", "lib"), "-lh2b200",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2003_10173_b200", "lib"),
                    "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", BIN], check=True)


def test_cpp_api_compiles_and_links():
    build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_api_reference_cases_on_b200(cuda):
    build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " 0 failures" in r.stdout
