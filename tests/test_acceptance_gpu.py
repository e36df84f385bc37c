"""The reference's acceptance criteria (proj/tests/acceptance.cpp)
re-run on the B200 executor (-m gpu). Criteria that are pure host scheduling
(6-9) are covered on CPU in tests/test_partition.py."""
import math

import numpy as np
import pytest

import paper_1711_03244_b200 as v

pytestmark = pytest.mark.gpu


def test_c1_energy_conservation_b1_b2_ten_seeds(gpu):
    """acceptance.cpp:56-82: |residual| < 1e-6 for B1/B2 x 10 seeds at 1e5 photons."""
    worst = 0.0
    for bench in (v.Benchmark.B1, v.Benchmark.B2):
        st = v.benchmark_preset(bench)
        st.config.photon_count = 100_000
        for seed in range(10):
            st.config.master_seed = seed
            r = gpu.run_group_dynamic(0, 100_000, 1, st.scene, st.config)
            worst = max(worst, abs(r.totals.books() - 100_000) / 100_000)
    assert worst < 1e-6


def test_c2_diffusion_agreement(gpu):
    """acceptance.cpp:86-132: isotropic source in a 100^3 B1-background cube, 1e7
    photons, radial shells r = 5..15 mm within 15 % of the infinite-medium
    diffusion Green's function exp(-mueff r)/(4 pi D r) (oracles.cpp:10-26)."""
    n = 100
    grid = v.VoxelGrid((n, n, n), 1.0, np.ones(n ** 3, np.uint8),
                       [v.OpticalProperties(0, 0, 0, 1.0), v.OpticalProperties(0.005, 1.0, 0.01, 1.37)])
    src = v.Source((50.0, 50.0, 50.0), (0.0, 0.0, 1.0), isotropic=True)
    cfg = v.SimulationConfig(photon_count=10_000_000, master_seed=20260826)
    r = gpu.run_group_dynamic(0, 10_000_000, 1, v.Scene(grid, src), cfg)
    r.map.normalize(grid)
    phi = r.map._values.reshape(n, n, n)
    mua, musp = 0.005, 1.0 * (1.0 - 0.01)
    D = 1.0 / (3.0 * (mua + musp))
    mueff = math.sqrt(3.0 * mua * (mua + musp))
    c = np.arange(n) + 0.5 - 50.0
    rr = np.sqrt(c[:, None, None] ** 2 + c[None, :, None] ** 2 + c[None, None, :] ** 2)
    shell = np.rint(rr).astype(int)
    worst = 0.0
    for b in range(5, 16):
        m = shell == b
        mc = phi[m].sum()
        dif = (np.exp(-mueff * rr[m]) / (4 * math.pi * D * rr[m])).sum()
        worst = max(worst, abs(mc / dif - 1.0))
    assert worst < 0.15, worst


def test_c10_byte_identical_across_partitions(gpu):
    """acceptance.cpp:369-395: B1 1e5 photons seed 1, strategies x device
    splits -> identical volume checksum (integer maps)."""
    from paper_1711_03244_b200.volume_io import fnv1a64
    st = v.benchmark_preset(v.Benchmark.B1)
    st.config.photon_count = 100_000
    st.config.master_seed = 1
    sums = set()
    for strat in v.Strategy:
        for slots in (1, 2, 3):
            devs = [v.DeviceProfile(name=f"s{i}", cores=1 + i, a=1e-4 * (1 + 2 * i), t0=5.0 + 15 * i, gpu=0)
                    for i in range(slots)]
            m = gpu.run_multi_device(100_000, devs, strat, st.scene, st.config)
            sums.add(fnv1a64(m.map.to_float_volume()))
    assert len(sums) == 1


def test_c11_beam_axis_peak(gpu):
    """acceptance.cpp:399-422: B1 1e6 photons: peak fluence on the beam axis, z < 5."""
    st = v.benchmark_preset(v.Benchmark.B1)
    st.config.photon_count = 1_000_000
    st.config.master_seed = 1
    r = gpu.run_group_dynamic(0, 1_000_000, 1, st.scene, st.config)
    r.map.normalize(st.grid)
    k = int(np.argmax(r.map._values.reshape(-1)))
    x, y, z = k % 60, (k // 60) % 60, k // 3600
    assert (x, y) == (30, 30) and z < 5
