"""The reference-style C++ program tests/cpp/dropin_test.cpp compiles against
include/voxmc/ and links libvoxmc_b200.so (CPU: host parts; GPU: executor)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1711_03244_b200", "lib")
EXE = os.path.join(LIBDIR, "dropin_test")


def build_exe():
    src = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", EXE,
                    "-L", LIBDIR, "-lvoxmc_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return EXE


def test_dropin_cpu_parts():
    exe = build_exe()
    r = subprocess.run([exe, "--cpu-only"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout


@pytest.mark.gpu
def test_dropin_gpu(gpu):
    exe = build_exe()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
