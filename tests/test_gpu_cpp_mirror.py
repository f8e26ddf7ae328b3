"""The C++ mirror of the reference interface (include/hfmm_b200.hpp): the restated reference tests
of tests/cpp/test_dropin.cpp, compiled against libhfmm_b200.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build_cpp():
    libdir = os.path.join(ROOT, "paper_1803_09948_b200")
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.check_call([cxx, "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-o", EXE,
                           "-L", libdir, "-lhfmm_b200", f"-Wl,-rpath,{libdir}"])
    return EXE


def test_cpp_mirror_compiles_and_refuses_without_device(gpu_available):
    exe = build_cpp()
    if not gpu_available:
        r = subprocess.run([exe], capture_output=True, text=True)
        assert r.returncode == 3 and "no CUDA device" in r.stdout   # loud failure, no CPU fallback


@pytest.mark.gpu
def test_cpp_mirror_reference_cases():
    exe = build_cpp()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
