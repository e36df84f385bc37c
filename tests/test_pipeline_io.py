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
    assert np.allclose(phi.cpu().numpy(), host, rtol=1e-6, atol=0)


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
    assert np.allclose(per.cpu().numpy(), fm._values.reshape(-1).astype(np.float32), rtol=1e-6)
    assert np.allclose(cw.cpu().numpy(), fm._values.sum(axis=0).reshape(-1).astype(np.float32), rtol=1e-5)
    assert np.all(per.cpu().numpy().reshape(ngates, -1)[:, lab == 2] == 0)  # mua == 0 -> 0
