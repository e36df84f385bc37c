"""The drop-in's one-photon step API on the host (include/voxmc: launch, advance,
handle_interface, roulette; transport.hpp:45-83) walked in run_photon order by
tests/cpp/step_api_test.cpp, photon by photon against the compiled reference
(oracle/_ref, the reference's own step functions): same steps and the same
dispositions to 1e-9 (the reference build contracts FMAs, the drop-in does
not, so a rare photon may take the other side of a tie)."""
import os
import subprocess

import numpy as np
import pytest

import paper_1711_03244_b200 as v

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1711_03244_b200", "lib")
EXE = os.path.join(LIBDIR, "step_api_test")


@pytest.fixture(scope="module")
def exe():
    src = os.path.join(ROOT, "tests", "cpp", "step_api_test.cpp")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o", EXE,
                    "-L", LIBDIR, "-lvoxmc_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return EXE


def _scene(name, seed):
    if name == "b3":
        st = v.benchmark_preset(v.Benchmark.B2)
    else:
        st = v.benchmark_preset(v.Benchmark.B1)
        if name == "b2":
            st.config.boundary_mode = v.BoundaryMode.ReflectAtMismatch
    st.config.master_seed = seed
    return st


@pytest.mark.parametrize("name,seed", [("b1", 1), ("b2", 5), ("b3", 9)])
def test_step_api_matches_reference(exe, ref, name, seed):
    n = 3000
    st = _scene(name, seed)
    st.config.photon_count = n
    out = subprocess.run([exe, name, "0", str(n), str(seed)], capture_output=True, text=True, check=True).stdout
    got = np.loadtxt(out.splitlines())
    assert got.shape == (n, 6)
    rt = ref.walk(st.scene, st.config, 0, n, threads=8, cells=False, traces=True)["traces"]
    same_steps = got[:, 5].astype(np.int64) == rt["steps"]
    assert same_steps.mean() >= 0.999
    close = np.ones(n, bool)
    for k, f in enumerate(("deposited", "escaped", "killed", "truncated")):
        close &= np.abs(got[:, 1 + k] - rt[f]) < 1e-9
    assert close.mean() >= 0.999
    # every photon's books close (deposited + escaped + killed + truncated == 1)
    assert np.abs(got[:, 1:5].sum(axis=1) - 1.0).max() < 1e-12
