"""The C++ host mirror (include/crt/convrot_b200.hpp) compiled with g++ and
linked against the sm_100a library: CPU-only checks here, tiny forwards
with -m gpu."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp")
PKG = os.path.join(ROOT, "paper_2512_03673_b200")
EXE = os.path.join(PKG, "_build", "test_host_api")


def build_exe():
    from paper_2512_03673_b200 import build as b
    b.build(verbose=False)
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    if os.path.exists(EXE) and os.path.getmtime(EXE) > max(
            os.path.getmtime(SRC), os.path.getmtime(b.LIB),
            os.path.getmtime(os.path.join(ROOT, "include", "crt", "convrot_b200.hpp"))):
        return EXE
    cuda = "/usr/local/cuda"
    cmd = ["g++", "-std=c++17", "-O1", SRC, "-o", EXE, "-I" + os.path.join(ROOT, "include"),
           "-I" + cuda + "/include", "-L" + PKG, "-lconvrot_b200", "-Wl,-rpath," + PKG,
           "-L" + cuda + "/lib64", "-lcudart", "-Wl,-rpath," + cuda + "/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return EXE


def test_cpp_host_api_cpu():
    r = subprocess.run([build_exe(), "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_host_api_gpu():
    r = subprocess.run([build_exe(), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
