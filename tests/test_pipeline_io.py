"""Front door (config/roster/report, reference config.cpp) and raw volume I/O
(volume_io.cpp) — CPU parts; the GPU run through run_pipeline is marked gpu."""
import json
import os

import numpy as np
import pytest

import paper_1711_03244_b200 as v
from paper_1711_03244_b200 import pipeline as P
from paper_1711_03244_b200.volume_io import fnv1a64, read_volume, write_volume


def test_fnv_native_matches_reference_rule():
    import oracle
    for data in [b"", b"a", b"foobar", bytes(range(256)) * 3]:
        assert fnv1a64(np.frombuffer(data, np.uint8)) == oracle.fnv1a64(data)


def test_volume_roundtrip_and_corruption(tmp_path):
    vals = np.random.default_rng(1).random(4 * 5 * 6).astype(np.float32)
    path = str(tmp_path / "vol.raw")
    ck = write_volume(vals, (4, 5, 6), 0.5, 1000, 7, path)
    side = json.load(open(path + ".json"))
    assert side["dims"] == [4, 5, 6] and side["checksum"] == ck and side["ordering"] == "x-fastest"
    d = read_volume(path)
    assert np.array_equal(d.values, vals) and d.seed == 7 and d.photon_count == 1000
    raw = bytearray(open(path, "rb").read())
    raw[10] ^= 0xFF
    open(path, "wb").write(bytes(raw))
    with pytest.raises(v.IoError):
        read_volume(path)
    os.remove(path + ".json")
    with pytest.raises(v.IoError):
        read_volume(path)


def test_config_parsing(tmp_path):
    s = P.parse_config_text(json.dumps({"benchmark": "b1", "photons": 1234, "seed": 5, "boundary": "reflect",
                                        "mode": "atomic", "gates": 10, "strategy": "s3"}))
    assert s.config.photon_count == 1234 and s.config.master_seed == 5 and s.config.ngates == 10
    assert s.config.boundary_mode == v.BoundaryMode.ReflectAtMismatch and s.strategy == v.Strategy.S3
    explicit = {"grid": {"dims": [10, 10, 10], "voxel_size_mm": 1.0},
                "media": [{"mua": 0, "mus": 0, "g": 0, "n": 1}, {"mua": 0.01, "mus": 1, "g": 0.9, "n": 1.37}],
                "sphere": {"center": [5, 5, 5], "radius": 2, "medium": {"mua": 0.1, "mus": 2, "g": 0.5, "n": 1.4}},
                "source": {"position": [5, 5, 0], "direction": [0, 0, 2]},
                "detectors": [{"position": [5, 7, 0], "radius": 1.0}]}
    s = P.parse_config_text(json.dumps(explicit))
    assert s.scene.grid.media[2].n == 1.4 and int((s.scene.grid.labels == 2).sum()) > 0
    assert s.scene.source.direction == (0.0, 0.0, 1.0) and len(s.config.detectors) == 1
    lab = np.full(1000, 1, np.uint8)
    lab.tofile(tmp_path / "labels.raw")
    s = P.parse_config_text(json.dumps({**explicit, "labels_file": "labels.raw"}), str(tmp_path))
    with pytest.raises(v.ParseError):
        P.parse_config_text("{not json")
    with pytest.raises(v.ParseError):
        P.parse_config_text(json.dumps({"photons": 5}))
    with pytest.raises(v.ValidationError):
        P.parse_config_text(json.dumps({"benchmark": "b1", "mode": "bogus"}))
    with pytest.raises(v.ValidationError):
        P.parse_config_text(json.dumps({"benchmark": "b1", "photons": 0}))


def test_roster_parsing():
    r = P.parse_roster_text(json.dumps([{"name": "a", "kind": "simulated", "a": 1e-3, "t0": 5},
                                        {"name": "g", "kind": "gpu", "gpu": 3}]))
    assert r[0].kind == v.DeviceKind.Simulated and r[1].kind == v.DeviceKind.CudaGpu and r[1].gpu == 3
    with pytest.raises(v.ParseError):
        P.parse_roster_text("[]")
    with pytest.raises(v.ParseError):
        P.parse_roster_text(json.dumps([{"name": "x", "kind": "quantum"}]))
    with pytest.raises(v.ValidationError):
        P.parse_roster_text(json.dumps([{"name": "x", "kind": "simulated"}]))


def test_scene_hash_and_cache(tmp_path):
    a = v.baseline_setup("b1")
    b = v.baseline_setup("b2")
    ha, hb = P.scene_hash(a.scene, a.config), P.scene_hash(b.scene, b.config)
    assert ha != hb and ha == P.scene_hash(a.scene, a.config)
    c = str(tmp_path / "cache.json")
    assert P.cache_lookup(c, "gpu0", ha) is None
    P.cache_store(c, "gpu0", ha, v.Calibration(1e-6, 3.0))
    assert P.cache_lookup(c, "gpu0", ha).t0 == 3.0


def test_cli_errors_exit_codes():
    from paper_1711_03244_b200.__main__ import main
    assert main(["run", "--benchmark", "b9"]) == 1
    assert main(["run"]) == 1


@pytest.mark.gpu
def test_run_pipeline_and_normalize(gpu, tmp_path):
    import torch
    st = v.baseline_setup("b1", photons=200_000)
    out = str(tmp_path / "b1.raw")
    s = P.RunSetup(st.scene, st.config, output_path=out, report_path=str(tmp_path / "r.json"))
    r = P.run_pipeline(s)
    assert abs(r.report.conservation_residual) < 1e-6 and r.report.throughput_photons_per_ms > 0
    rep = json.load(open(tmp_path / "r.json"))
    assert rep["photon_count"] == 200_000 and rep["devices"][0]["photons"] == 200_000
    vol = read_volume(out)
    assert np.array_equal(vol.values, r.map.to_float_volume())
    # K4 on the device == host FluenceMap.normalize
    plan = gpu.Plan(st.scene, st.config)
    cells = torch.from_numpy(r.map.cells.reshape(-1).copy()).cuda()
    phi = torch.zeros(plan.ncells, dtype=torch.float32, device="cuda")
    plan.normalize_torch(cells, phi, 200_000)
    r.map.normalize(st.grid)
    host = r.map.to_float_volume()
    assert np.array_equal(phi.cpu().numpy(), host)  # same arithmetic, bit for bit


@pytest.mark.gpu
@pytest.mark.parametrize("dims,ngates", [((5, 7, 9), 3), ((4, 6, 8), 10)])
def test_normalize_kernel_odd_even_gates(gpu, dims, ngates):
    """K4 on odd / even voxel counts (pair-vectorised and scalar paths), per gate and CW."""
    import torch
    nx, ny, nz = dims
    rng = np.random.default_rng(3)
    lab = rng.integers(1, 3, nx * ny * nz).astype(np.uint8)
    media = [v.OpticalProperties(), v.OpticalProperties(0.02, 1.0, 0.5, 1.3), v.OpticalProperties(0.0, 1.0, 0.5, 1.3)]
    grid = v.VoxelGrid(dims, 0.5, lab, media)
    cfg = v.SimulationConfig(photon_count=12345, ngates=ngates)
    scene = v.Scene(grid, v.Source((1.0, 1.0, 0.0), (0.0, 0.0, 1.0)))
    plan = gpu.Plan(scene, cfg)
    cells = rng.integers(0, 1 << 40, plan.ncells).astype(np.int64)
    tc = torch.from_numpy(cells).cuda()
    per = torch.zeros(plan.ncells, dtype=torch.float32, device="cuda")
    cw = torch.zeros(grid.voxel_count, dtype=torch.float32, device="cuda")
    plan.normalize_torch(tc, per, 12345, sum_gates=False)
    plan.normalize_torch(tc, cw, 12345, sum_gates=True)
    torch.cuda.synchronize()
    fm = v.FluenceMap(dims, 12345, ngates, cells)
    fm.normalize(grid)
    assert np.array_equal(per.cpu().numpy(), fm._values.reshape(-1).astype(np.float32))
    assert np.array_equal(cw.cpu().numpy(), fm.to_float_volume())
    assert np.all(per.cpu().numpy().reshape(ngates, -1)[:, lab == 2] == 0)  # mua == 0 -> 0


def _random_map(rng, dims, ngates, photons):
    nx, ny, nz = dims
    lab = rng.integers(0, 3, nx * ny * nz).astype(np.uint8)
    media = [v.OpticalProperties(), v.OpticalProperties(0.02, 1.0, 0.5, 1.3),
             v.OpticalProperties(0.0173, 1.0, 0.5, 1.3)]
    grid = v.VoxelGrid(dims, 0.7, lab, media)
    scene = v.Scene(grid, v.Source((1.0, 1.0, 0.0), (0.0, 0.0, 1.0)))
    # magnitudes past 2^53 included (double(cell) rounds, as in the reference)
    cells = rng.integers(0, 1 << 60, ngates * grid.voxel_count).astype(np.int64) >> rng.integers(
        0, 40, ngates * grid.voxel_count)
    return scene, cells


@pytest.mark.parametrize("normalized", [True, False])
def test_host_normalize_equals_reference(ref, normalized):
    """FluenceMap.normalize / to_float_volume (runtime.py) against the compiled
    reference's FluenceMap::normalize + to_float_volume (fluence.cpp:62-90), bit
    for bit, for the CW map and for every gate of a gated map."""
    rng = np.random.default_rng(11)
    scene, cells = _random_map(rng, (7, 5, 6), 3, 987_654)
    fm = v.FluenceMap(scene.grid.dims, 987_654, 3, cells)
    if normalized:
        fm.normalize(scene.grid)
    want_cw = ref.normalize(scene, 987_654, fm.cells.sum(axis=0), normalized)
    assert np.array_equal(fm.to_float_volume(), want_cw)
    if normalized:
        for g in range(3):
            want = ref.normalize(scene, 987_654, fm.cells[g], True)
            assert np.array_equal(fm._values[g].reshape(-1).astype(np.float32), want)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,ngates", [((7, 5, 6), 3), ((8, 4, 6), 10), ((60, 60, 60), 1)])
def test_normalize_kernel_equals_reference(gpu, ref, dims, ngates):
    """K4 (vmc_plan_normalize) against the compiled reference's
    FluenceMap::normalize + to_float_volume (fluence.cpp:62-90): bit for bit,
    per gate, gate-summed, and raw (unnormalized) export."""
    import torch
    rng = np.random.default_rng(5)
    scene, cells = _random_map(rng, dims, ngates, 123_457)
    cfg = v.SimulationConfig(photon_count=123_457, ngates=ngates)
    plan = gpu.Plan(scene, cfg)
    tc = torch.from_numpy(cells).cuda()
    nvox = scene.grid.voxel_count
    for normalized in (True, False):
        per = torch.zeros(plan.ncells, dtype=torch.float32, device="cuda")
        cw = torch.zeros(nvox, dtype=torch.float32, device="cuda")
        plan.normalize_torch(tc, per, 123_457, sum_gates=False, normalized=normalized)
        plan.normalize_torch(tc, cw, 123_457, sum_gates=True, normalized=normalized)
        torch.cuda.synchronize()
        per_h = per.cpu().numpy().reshape(ngates, -1)
        c = cells.reshape(ngates, -1)
        for g in range(ngates):
            assert np.array_equal(per_h[g], ref.normalize(scene, 123_457, c[g], normalized)), (g, normalized)
        assert np.array_equal(cw.cpu().numpy(), ref.normalize(scene, 123_457, c.sum(axis=0), normalized))
    plan.close()


@pytest.mark.gpu
def test_gated_pipeline_output_keeps_reference_format(gpu, tmp_path):
    """With time gates, `output` stays the reference's nx*ny*nz float file (the
    gate-summed volume, read_volume-compatible: volume_io.cpp:60-88) and the
    gate-resolved volume goes to `<output>.gates.raw`."""
    st = v.baseline_setup("b1", photons=50_000)
    st.config.ngates = 5
    out = str(tmp_path / "g.raw")
    r = P.run_pipeline(P.RunSetup(st.scene, st.config, output_path=out))
    vol = read_volume(out)
    assert vol.gates == 1 and vol.values.size == st.grid.voxel_count
    assert os.path.getsize(out) == 4 * st.grid.voxel_count
    assert np.array_equal(vol.values, r.map.to_float_volume())
    assert "gates" not in json.load(open(out + ".json"))
    gv = read_volume(out + ".gates.raw")
    assert gv.gates == 5 and gv.values.size == 5 * st.grid.voxel_count
    assert np.array_equal(gv.values, (r.map.cells.astype(np.float64) * r.map.quantum).astype(np.float32).reshape(-1))
