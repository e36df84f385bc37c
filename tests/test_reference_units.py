"""The reference's own doctest unit files (proj/tests/test_{rng,fluence,domain,
scheduler,transport,cli_io,oracles}.cpp), compiled UNMODIFIED against the B200 drop-in headers
(include/voxmc) with the doctest stand-in tests/cpp/doctest.h and linked to
libvoxmc_b200.so (recipe: oracle/Makefile `reftests`, built by
__graft_entry__.build() where /root/reference exists; the binaries travel with
the repo snapshot). Host-side units run here; the executor cases of
test_scheduler (run_group_dynamic / run_static_split / run_multi_device) and
test_transport (simulate_photon_trace: Beer-Lambert, horizon, per-photon
accounting to 1e-9, chord lengths to 1e-9, per-voxel path lengths against the
ray-march oracle, reproducibility) and test_cli_io's run_pipeline case run on
the B200 with -m gpu. test_cli_io holds the C++ front door (include/voxmc/
config.hpp, volume_io.hpp): raw volume + checksummed sidecar, corrupted-volume
detection, config presets / overrides / explicit scenes / diagnostics, device
rosters, scene hash, calibration cache, the pipeline report."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "tests")


def run_unit(name, filt=None):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([exe] + ([filt] if filt else []), capture_output=True, text=True, timeout=900)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.parametrize("name", ["test_rng", "test_fluence", "test_domain", "test_oracles"])
def test_reference_host_units(name):
    rc, out = run_unit(name)
    assert rc == 0, out[-3000:]
    assert " 0 failed" in out


@pytest.mark.parametrize("filt", ["thread count", "S1 ", "S2 ", "S3 ", "conserve", "group counter", "replay",
                                  "calibration", "strategy names"])
def test_reference_scheduler_host_cases(filt):
    rc, out = run_unit("test_scheduler", filt)
    assert rc == 0, out[-3000:]
    assert "test cases: 0 " not in out  # the filter matched something


@pytest.mark.parametrize("filt", ["pencil launch", "launch outside", "isotropic launch", "distance to voxel",
                                  "boundary distance agrees", "Henyey-Greenstein median", "sample mean equals g",
                                  "g = 0", "unit-norm over many", "Fresnel", "roulette"])
def test_reference_transport_host_cases(filt):
    """test_transport.cpp's host-side cases: launch state, DDA distance, HG
    sampling statistics (1e6 deflections), Fresnel, roulette (1e6 draws)."""
    rc, out = run_unit("test_transport", filt)
    assert rc == 0, out[-3000:]
    assert "test cases: 0 " not in out


@pytest.mark.gpu
def test_reference_transport_unit_on_gpu(gpu):
    """All of test_transport.cpp, its walk cases through the device."""
    rc, out = run_unit("test_transport")
    assert rc == 0, out[-3000:]
    assert " 0 failed" in out


@pytest.mark.gpu
def test_reference_scheduler_unit_on_gpu(gpu):
    """All of test_scheduler.cpp, including the executor contracts on the B200:
    dynamic == static raw cells, per-thread accounting, and the multi-device
    merge == single-device raw cells (test_scheduler.cpp:157-178, 246-264)."""
    rc, out = run_unit("test_scheduler")
    assert rc == 0, out[-3000:]
    assert " 0 failed" in out


@pytest.mark.parametrize("filt", ["volume files", "corrupted volume", "benchmark preset config", "photon count defaults",
                                  "explicit scene", "bad configs", "device rosters", "host device", "scene hash",
                                  "calibration cache"])
def test_reference_cli_io_host_cases(filt):
    rc, out = run_unit("test_cli_io", filt)
    assert rc == 0, out[-3000:]
    assert "test cases: 0 " not in out


@pytest.mark.gpu
def test_reference_cli_io_unit_on_gpu(gpu):
    """All of test_cli_io.cpp, run_pipeline on the B200."""
    rc, out = run_unit("test_cli_io")
    assert rc == 0, out[-3000:]
    assert " 0 failed" in out
