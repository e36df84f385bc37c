"""Seeded random-scene parity (tests/fuzz_scenes.py): mixed media, oblique
and isotropic sources, both boundary modes, gates and detectors drawn at
random, so branch combinations no fixed scene pins are still held to the
reference.

CPU (checker pinning): the plain-C restatement equals the compiled reference
built without FMA contraction bit for bit (continuous-wave maps and
dispositions), and K1f's flight decomposition restated in double precision
draws the reference's stream photon for photon.
GPU (-m gpu): the FP64 flight kernel photon for photon against the
reference's walk (transport.cpp:310-358 plus the derived gate / detector
sink of oracle/ref_capi.cpp), and the FP32 product kernel at run level.
"""
import numpy as np
import pytest

import oracle
import paper_1711_03244_b200 as v
from fuzz_scenes import SEEDS, random_scene

NOFMA = oracle.REF_SO.replace("libvoxmc_ref.so", "libvoxmc_ref_nofma.so")


@pytest.mark.parametrize("seed", SEEDS)
def test_fuzz_c_restatement_bit_exact_vs_nofma_reference(corc, seed):
    scene, cfg = random_scene(seed, detectors=False, gates=False)
    n = 4000
    cfg.photon_count = n
    R0 = oracle.RefLib(NOFMA)
    rc, rd, _ = R0.run_group(scene, cfg, 0, n, 4)
    out = corc.walk(scene, cfg, 0, n, threads=4)
    assert np.array_equal(out["cells"], rc)
    assert out["disp"] == pytest.approx(rd, rel=1e-13, abs=1e-9)


@pytest.mark.parametrize("seed", SEEDS)
def test_fuzz_flight_decomposition(ref, corc, seed):
    scene, cfg = random_scene(seed, detectors=False, gates=False)
    n = 3000
    f = corc.walk_flight(scene, cfg, 0, n, threads=8)["traces"]
    r = ref.walk(scene, cfg, 0, n, threads=8, cells=False, traces=True)["traces"]
    same = f["draws"] == r["draws"]
    assert same.mean() >= 0.995
    close = np.ones(n, bool)
    for fld in ("deposited", "escaped", "killed", "truncated"):
        close &= np.abs(f[fld] - r[fld]) < 1e-9
    assert close.mean() >= 0.995


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_fuzz_fp64_per_photon(gpu, ref, seed):
    scene, cfg = random_scene(seed)
    cfg.precision = v.Precision.FP64
    n = 3000
    tr = gpu.trace_photons(scene, cfg, 0, n)
    rt = ref.walk(scene, cfg, 0, n, threads=8, cells=False, traces=True)["traces"]
    same = tr["draws"] == rt["draws"]
    assert same.mean() >= 0.995, same.mean()
    for f in ("deposited", "escaped", "killed", "truncated"):
        assert np.abs(tr[f][same] - rt[f][same]).max() < 1e-6, f
    assert np.array_equal(tr["flags"][same], rt["flags"][same])


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_fuzz_fp32_run(gpu, ref, seed):
    scene, cfg = random_scene(seed)
    n = 30_000
    cfg.photon_count = n
    g = gpu.run_group_dynamic(0, n, 1, scene, cfg)
    w = ref.walk(scene, cfg, 0, n, threads=8, detectors=bool(cfg.detectors))
    assert abs(g.totals.books() - n) / n < 1e-6
    assert int(g.map.cells.sum()) == g.totals_q[0]
    for i, name in enumerate(("deposited", "escaped", "killed", "truncated")):
        # correlated streams (same seeds): channel totals agree far below MC noise
        assert abs(getattr(g.totals, name) - w["disp"][i]) <= 3e-3 * n + 1e-9, name
    # per-gate deposited sums
    q = v.quantum_for(n)
    gs = g.map.cells.reshape(cfg.ngates, -1).sum(axis=1) * q
    ws = w["cells"].reshape(cfg.ngates, -1).sum(axis=1) * q
    assert np.abs(gs - ws).max() <= 3e-3 * n + 1e-9
    if cfg.detectors:
        k = w["det_count"]
        assert abs(int(g.det_count) - k) <= max(5, 0.03 * k), (g.det_count, k)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS[:12])
def test_fuzz_fp32_per_photon(gpu, ref, seed):
    """The FP32 product kernel photon by photon: rounding can flip a discrete
    decision (a face tie, a Fresnel draw at R), after which the photon follows
    another path, so the gate is statistical; the weight books of every photon
    close exactly."""
    scene, cfg = random_scene(seed)
    n = 3000
    tr = gpu.trace_photons(scene, cfg, 0, n)
    rt = ref.walk(scene, cfg, 0, n, threads=8, cells=False, traces=True)["traces"]
    assert (tr["draws"] == rt["draws"]).mean() >= 0.98  # measured >= 0.9993 on all 24 seeds
    books = tr["deposited"] + tr["escaped"] + tr["killed"] + tr["truncated"]
    assert np.abs(books - 1.0).max() < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS[:12])
def test_fuzz_step_kernel_fp64_per_photon(gpu, ref, monkeypatch, seed):
    """The per-step kernel K1 (VMC_KERNEL=step, the A/B baseline) in FP64 on the
    same random scenes."""
    monkeypatch.setenv("VMC_KERNEL", "step")
    scene, cfg = random_scene(seed)
    cfg.precision = v.Precision.FP64
    n = 2000
    tr = gpu.trace_photons(scene, cfg, 0, n)
    rt = ref.walk(scene, cfg, 0, n, threads=8, cells=False, traces=True)["traces"]
    same = tr["draws"] == rt["draws"]
    assert same.mean() >= 0.995, same.mean()
    for f in ("deposited", "escaped", "killed", "truncated"):
        assert np.abs(tr[f][same] - rt[f][same]).max() < 1e-6, f
