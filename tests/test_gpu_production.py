"""Parity of the production kernel variants the bench lines time, at the
BASELINE sizes (run with -m gpu on a B200).

* head: 256^3 x 5 labels x 10 gates dispatches k_flight<float,1,0,0,0,0>
  (gated, multi-label, direct deposits). Its map is checked against the
  compiled reference's gated walk (oracle/ref_capi.cpp ref_walk, which
  re-drives transport.cpp:161-225 with a gate sink), and its trace
  instantiation (same body, same arithmetic) photon by photon against the
  reference's RNG stream.
* B1 at BASELINE's own N = 1e6 with SURVEY §8(c)'s 1e-4 absorbed-fraction gate.
"""
import numpy as np
import pytest

import paper_1711_03244_b200 as v

pytestmark = pytest.mark.gpu


def l2_rel(a, b, mask):
    a = a.astype(np.float64)[mask]
    b = b.astype(np.float64)[mask]
    return float(np.sqrt(((a - b) ** 2).sum() / (b ** 2).sum()))


N_HEAD = 50_000


@pytest.fixture(scope="module")
def head256():
    return v.baseline_setup("head", photons=N_HEAD, seed=1, head_n=256)


@pytest.fixture(scope="module")
def head_ref(ref, head256):
    st = head256
    return ref.walk(st.scene, st.config, 0, N_HEAD, threads=8, cells=True, counts=True)


def test_head256_dispatches_production_variant(gpu, head256):
    p = gpu.Plan(head256.scene, head256.config)
    try:
        assert p.kernel == "k_flight<float,1,0,0,0,0>", p.kernel
    finally:
        p.close()


def test_head256_run_parity(gpu, golden, head256, head_ref):
    st = head256
    gold = golden["workloads"]["head256"]
    w = head_ref
    assert w["disp"] == pytest.approx(gold["disp"], rel=1e-9)  # oracle pinned to the fixture
    g = gpu.run_group_dynamic(0, N_HEAD, 1, st.scene, st.config)
    rel = g.totals.deposited / w["disp"][0] - 1.0
    assert abs(rel) <= 5e-4, rel
    assert abs(g.totals.books() - N_HEAD) / N_HEAD <= 1e-6
    assert int(g.map.cells.sum()) == g.totals_q[0]
    mask = w["counts"] >= 100
    assert mask.sum() == gold["voxels_ge100"]
    assert l2_rel(g.map.cw_cells(), w["cells"].reshape(10, -1).sum(axis=0), mask) <= 5e-3
    # gate-resolved: every gate holding >= 0.1 % of the weight within 2 %
    gs = g.map.cells.reshape(10, -1).sum(axis=1).astype(np.float64)
    rs = np.array(gold["gate_sums"], dtype=np.float64)
    big = rs > 1e-3 * rs.sum()
    assert big.sum() >= 3
    assert np.all(np.abs(gs[big] / rs[big] - 1) < 0.02), gs[big] / rs[big]
    # per gate, voxel by voxel, on the voxels with >= 100 reference deposits:
    # the first gate holds 94 % of the weight, the second 5 %
    # (fewer deposits per voxel, so more MC noise from the diverged photons)
    gm = g.map.cells.reshape(10, -1)
    rm = w["cells"].reshape(10, -1)
    e0, e1 = l2_rel(gm[0], rm[0], mask & (rm[0] > 0)), l2_rel(gm[1], rm[1], mask & (rm[1] > 0))
    print(f"head256 per-gate L2: gate0 {e0:.2e} gate1 {e1:.2e}")
    assert e0 <= 1e-2 and e1 <= 5e-2, (e0, e1)


def test_head256_per_photon_draws(gpu, ref, head256):
    """The trace instantiation of the gated head kernel (same body and
    arithmetic as production) photon by photon against the reference walk."""
    st = head256
    n = 20_000
    tr = gpu.trace_photons(st.scene, st.config, 0, n)
    rt = ref.walk(st.scene, st.config, 0, n, threads=8, cells=False, traces=True)["traces"]
    same = (tr["draws"] == rt["draws"]).mean()
    assert same >= 0.9, same
    books = tr["deposited"] + tr["escaped"] + tr["killed"] + tr["truncated"]
    assert np.abs(books - 1.0).max() < 1e-5
    # the photons that follow the same discrete path agree in their dispositions
    s = tr["draws"] == rt["draws"]
    assert np.abs(tr["deposited"][s] - rt["deposited"][s]).max() < 2e-4


def test_head256_fp64_per_photon(gpu, ref, head256):
    """FP64 K1f on the full head volume: the reference's arithmetic, draw for draw."""
    st = v.baseline_setup("head", photons=N_HEAD, seed=1, head_n=256)
    st.config.precision = v.Precision.FP64
    n = 2_000
    p = gpu.Plan(st.scene, st.config)
    assert p.kernel.startswith("k_flight<double,1,0,0,0"), p.kernel
    tr = p.trace(0, n)
    p.close()
    rt = ref.walk(st.scene, st.config, 0, n, threads=8, cells=False, traces=True)["traces"]
    same = tr["draws"] == rt["draws"]
    assert same.mean() >= 0.995
    close = np.ones(n, bool)
    for f in ("deposited", "escaped", "killed", "truncated"):
        close &= np.abs(tr[f] - rt[f]) < 1e-9
    assert close[same].mean() >= 0.999


def test_b1_at_baseline_size(gpu, ref, golden):
    """BASELINE configs[0]: B1, 1e6 photons, seed 1. SURVEY §8(c) gate:
    |absorbed fraction - reference| / reference <= 1e-4."""
    n = 1_000_000
    st = v.baseline_setup("b1", photons=n, seed=1)
    p = gpu.Plan(st.scene, st.config)
    assert p.kernel == "k_flight<float,0,0,0,1,0>", p.kernel
    p.close()
    gold = golden["workloads"]["b1_1e6"]
    w = ref.walk(st.scene, st.config, 0, n, threads=8, cells=True, counts=True)
    assert w["disp"] == pytest.approx(gold["disp"], rel=1e-9)
    g = gpu.run_group_dynamic(0, n, 1, st.scene, st.config)
    rel = g.totals.deposited / w["disp"][0] - 1.0
    assert abs(rel) <= 1e-4, rel
    assert abs(g.totals.escaped / w["disp"][1] - 1.0) <= 1e-4
    assert abs(g.totals.books() - n) / n <= 1e-6
    mask = w["counts"] >= 100
    assert mask.sum() == gold["voxels_ge100"]
    assert l2_rel(g.map.cw_cells(), w["cells"], mask) <= 5e-3
    # beam-axis peak (acceptance.cpp:399-422)
    c = g.map.cw_cells().reshape(60, 60, 60)
    z, y, x = np.unravel_index(int(np.argmax(c)), c.shape)
    assert (x, y) == (30, 30) and z < 5


@pytest.mark.parametrize("name,kernel", [("b2", "k_flight<float,0,0,0,1,0>"),
                                         ("b3", "k_flight<float,0,1,0,0,0>")])
def test_bench_variants_dispatch(gpu, name, kernel):
    """The variants the B2 / B3 bench lines time are the ones the run-parity
    tests of test_gpu_parity.py exercise (same scene, same selection)."""
    st = v.baseline_setup(name, photons=1000)
    p = gpu.Plan(st.scene, st.config)
    try:
        assert p.kernel == kernel, p.kernel
    finally:
        p.close()


def test_label_cache_follows_in_place_edits(gpu):
    """vmc_run_range caches the label volume on the device by a digest of its
    contents (no re-upload, no re-scan for a repeated scene); an in-place edit
    of the caller's array must reach the kernel on the next call."""
    n = 20_000
    st = v.baseline_setup("b3", photons=n, seed=3)
    g1 = gpu.run_group_dynamic(0, n, 1, st.scene, st.config)
    g1b = gpu.run_group_dynamic(0, n, 1, st.scene, st.config)  # cached volume
    assert (g1.map.cells == g1b.map.cells).all() and g1.totals_q == g1b.totals_q
    lab = st.scene.grid.labels
    lab[lab == 2] = 1  # remove the sphere in place (same array, same pointer)
    g2 = gpu.run_group_dynamic(0, n, 1, st.scene, st.config)
    assert not (g2.map.cells == g1.map.cells).all()
    # the edited volume in a fresh array: the same map bit for bit
    st2 = v.baseline_setup("b3", photons=n, seed=3)
    st2.scene.grid.labels[:] = lab
    g3 = gpu.run_group_dynamic(0, n, 1, st2.scene, st2.config)
    assert (g2.map.cells == g3.map.cells).all() and g2.totals_q == g3.totals_q
    # and through a plan (always uploads)
    p = gpu.Plan(st2.scene, st2.config)
    try:
        assert p.kernel == "k_flight<float,0,1,0,1,0>", p.kernel  # now single-label
    finally:
        p.close()
