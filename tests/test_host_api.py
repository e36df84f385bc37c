"""Host-side mirror of the reference's domain and accumulator API (CPU):
presets (test_domain.cpp), FluenceMap semantics (test_fluence.cpp)."""
import math

import numpy as np
import pytest

import paper_1711_03244_b200 as v
from paper_1711_03244_b200.runtime import FluenceMap, merge


def test_presets_match_reference_values():
    b1 = v.benchmark_preset(v.Benchmark.B1)
    assert b1.grid.dims == (60, 60, 60) and b1.grid.voxel_size == 1.0
    assert b1.grid.media[1] == v.OpticalProperties(0.005, 1.0, 0.01, 1.37)
    assert b1.grid.media[0] == v.OpticalProperties(0.0, 0.0, 0.0, 1.0)
    assert b1.config.boundary_mode == v.BoundaryMode.TerminateAtBoundary
    assert b1.source.position == (30.0, 30.0, 0.0)
    b2 = v.benchmark_preset(v.Benchmark.B2)
    assert b2.config.boundary_mode == v.BoundaryMode.ReflectAtMismatch
    assert b2.grid.media[2] == v.OpticalProperties(0.002, 5.0, 0.9, 1.0)
    assert v.benchmark_preset(v.Benchmark.B2a).config.accumulation_mode == v.AccumulationMode.SharedAtomic
    assert v.benchmark_from_name("b2a") == v.Benchmark.B2a and v.benchmark_from_name("x") is None


def test_sphere_voxelization_brute_force():
    """test_domain.cpp:52-73: label 2 iff the voxel centre is within 15 mm."""
    g = v.benchmark_preset(v.Benchmark.B2).grid
    lab = g.labels.reshape(60, 60, 60)
    for (x, y, z) in [(30, 30, 30), (15, 30, 30), (14, 30, 30), (44, 30, 30), (45, 30, 30), (0, 0, 0)]:
        d2 = (x + 0.5 - 30) ** 2 + (y + 0.5 - 30) ** 2 + (z + 0.5 - 30) ** 2
        assert (lab[z, y, x] == 2) == (d2 <= 225.0)
    assert int((lab == 2).sum()) > 0


def test_sphere_matches_reference_grid(ref):
    """The preset grids are byte-identical to the reference's (scene_hash input)."""
    import oracle
    st = v.benchmark_preset(v.Benchmark.B2)
    st.config.master_seed = 1
    st.config.photon_count = 2000
    a, _, _ = ref.run_group(st.scene, st.config, 0, 2000, 2)
    b = oracle.corc().walk(st.scene, st.config, 0, 2000, threads=2)["cells"]
    assert (a > 0).sum() > 0 and abs(int(a.sum()) / int(b.sum()) - 1) < 1e-3


def test_voxel_of_bounds():
    g = v.benchmark_preset(v.Benchmark.B1).grid
    assert g.voxel_of((30.0, 30.0, 1e-6)) == v.VoxelIndex(30, 30, 0)
    assert g.voxel_of((60.0, 1.0, 1.0)) is None
    assert g.voxel_of((-1e-9, 1.0, 1.0)) is None
    assert g.linear((1, 2, 3)) == 1 + 60 * (2 + 60 * 3)


def test_head_volume_labels():
    lab = v.head_labels(256)
    assert lab.shape == (256, 256, 256)
    assert set(np.unique(lab)) == {1, 2, 3, 4, 5}
    assert lab[128, 128, 128] == 5 and lab[0, 0, 0] == 1 and lab[128, 128, 20] == 3
    st = v.baseline_setup("head")
    assert st.config.ngates == 10 and st.config.boundary_mode == v.BoundaryMode.ReflectAtMismatch
    assert st.source.position == (128.0, 128.0, 0.0)


def test_fluence_map_semantics():
    """test_fluence.cpp:17-141 restated on the host FluenceMap."""
    m = FluenceMap((4, 4, 4), 100)
    assert m.quantum == math.ldexp(1.0, -(62 - 7))
    q = m.quantum
    m.cells.reshape(-1)[0] += round(0.5 / q) + round(0.25 / q)
    assert m.value(0) == pytest.approx(0.75, rel=1e-12)
    assert m.total_deposited() == pytest.approx(0.75, rel=1e-12)
    a, b = FluenceMap((4, 4, 4), 50), FluenceMap((4, 4, 4), 50)
    a.cells.reshape(-1)[1] = 7
    b.cells.reshape(-1)[2] = 9
    ab, ba = merge([a, b]), merge([b, a])
    assert np.array_equal(ab.cells, ba.cells)
    with pytest.raises(v.DimensionMismatch):
        a.add(FluenceMap((4, 4, 5), 50))
    with pytest.raises(v.DimensionMismatch):
        a.add(FluenceMap((4, 4, 4), 10**9))
    with pytest.raises(v.DimensionMismatch):
        merge([])
    g = v.VoxelGrid((4, 4, 4), 2.0, np.r_[np.ones(63, np.uint8), [2]],
                    [v.OpticalProperties(), v.OpticalProperties(0.5, 1, 0, 1), v.OpticalProperties(0, 1, 0, 1)])
    a.normalize(g)
    assert a.value(1) == pytest.approx(7 * a.quantum / (0.5 * 8.0 * 50))
    assert a.value(63) == 0.0 and a.zero_mua_voxels == 1
    with pytest.raises(v.AlreadyNormalized):
        a.normalize(g)
    with pytest.raises(v.AlreadyNormalized):
        a.add(b)
    vol = b.to_float_volume()
    assert vol.dtype == np.float32 and vol[2] == np.float32(9 * b.quantum)


def test_gated_map_cw():
    m = FluenceMap((2, 2, 2), 10, ngates=3)
    m.cells[0, 0, 0, 0] = 1
    m.cells[2, 0, 0, 0] = 2
    assert m.cw_cells()[0] == 3 and m.raw_cell(0, gate=2) == 2
