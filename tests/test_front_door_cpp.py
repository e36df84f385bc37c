"""The C++ front door of the drop-in (include/voxmc/config.hpp, volume_io.hpp;
paper_1711_03244_b200/csrc/voxmc_config.cpp) agrees with the Python one
(pipeline.py, volume_io.py): the same scene hash keys the calibration cache,
and volumes written by either side read back on the other."""
import os
import subprocess

import numpy as np
import pytest

import paper_1711_03244_b200 as v
from paper_1711_03244_b200 import pipeline, volume_io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1711_03244_b200", "lib")
EXE = os.path.join(LIBDIR, "front_door_test")


@pytest.fixture(scope="module")
def exe():
    src = os.path.join(ROOT, "tests", "cpp", "front_door_test.cpp")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", EXE,
                    "-L", LIBDIR, "-lvoxmc_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return EXE


def run(exe, *args):
    return subprocess.run([exe, *args], capture_output=True, text=True, check=True).stdout.split()


@pytest.mark.parametrize("name", ["b1", "b2", "b2a"])
def test_scene_hash_same_as_python(exe, name):
    st = v.benchmark_preset(v.benchmark_from_name(name))
    assert int(run(exe, "hash", name)[0], 16) == pipeline.scene_hash(st.scene, st.config)


def test_volumes_cross_read(exe, tmp_path):
    p = str(tmp_path / "cpp.raw")
    chk = int(run(exe, "write", p)[0], 16)
    vol = volume_io.read_volume(p)  # Python reads the C++ file and verifies its checksum
    assert vol.checksum == chk and vol.dims == (7, 5, 3) and vol.seed == 99 and vol.voxel_size_mm == 0.5
    assert vol.values.sum() == pytest.approx(0.375, rel=1e-6)
    q = str(tmp_path / "py.raw")
    vals = np.arange(7 * 5 * 3, dtype=np.float32) / 8
    c2 = volume_io.write_volume(vals, (7, 5, 3), 1.0, 10, 5, q)
    out = run(exe, "read", q)  # C++ reads the Python file
    assert out[:4] == ["7", "5", "3", "5"] and int(out[4], 16) == c2
    assert float(out[5]) == pytest.approx(float(vals.sum()), rel=1e-6)
