"""Seeded random scenes for the fuzz parity tests (tests/test_fuzz.py).

Each seed draws a small volume that mixes what the BASELINE workloads keep
apart: 1-4 interior media with random mua / mus / g / n (zero absorption,
mus = 0 flights, isotropic g = 0, backward g < 0, equal and mismatched
refractive indices), blobs of other labels and sometimes in-grid air,
non-cubic grids with a non-integer voxel size, pencil beams at random oblique
angles or an isotropic point source, either boundary mode, short and long time
horizons, 1-4 time gates and 0-3 disk detectors on the entry face.
"""
import numpy as np

import paper_1711_03244_b200 as v

AIR = v.OpticalProperties(0.0, 0.0, 0.0, 1.0)
N_INDEX = (1.0, 1.33, 1.37, 1.45, 1.6)


def random_scene(seed: int, detectors: bool = True, gates: bool = True):
    rng = np.random.default_rng(1000 + seed)
    nx, ny, nz = (int(x) for x in rng.integers(6, 23, 3))
    h = float(rng.choice([0.5, 1.0, 0.37, 1.7]))
    nmed = int(rng.integers(1, 5))
    media = [AIR]
    for _ in range(nmed):
        u = rng.random()  # no absorption / strong absorption (roulette) / tissue-like
        mua = 0.0 if u < 0.15 else (float(rng.uniform(0.2, 1.0)) if u < 0.3 else float(rng.uniform(0.001, 0.08)))
        mus = 0.0 if rng.random() < 0.1 else float(rng.uniform(0.2, 6.0))
        g = 0.0 if rng.random() < 0.2 else float(rng.uniform(-0.5, 0.95))
        media.append(v.OpticalProperties(mua, mus, g, float(rng.choice(N_INDEX))))
    lab = np.ones((nz, ny, nx), np.uint8)
    zc, yc, xc = np.meshgrid(np.arange(nz) + 0.5, np.arange(ny) + 0.5, np.arange(nx) + 0.5, indexing="ij")
    for _ in range(int(rng.integers(0, 5))):  # spheres and boxes of the other labels
        l = int(rng.integers(1, nmed + 1))
        if rng.random() < 0.5:
            c = rng.uniform(0, 1, 3) * (nx, ny, nz)
            r = rng.uniform(1.5, 0.5 * min(nx, ny, nz))
            lab[(xc - c[0]) ** 2 + (yc - c[1]) ** 2 + (zc - c[2]) ** 2 <= r * r] = l
        else:
            lo = [int(rng.integers(0, d)) for d in (nz, ny, nx)]
            hi = [int(rng.integers(a + 1, d + 1)) for a, d in zip(lo, (nz, ny, nx))]
            lab[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = l
    if rng.random() < 0.25:  # in-grid air slab at the far side
        lab[:, :, nx - int(rng.integers(1, 3)):] = 0
    grid = v.VoxelGrid((nx, ny, nz), h, lab, media)
    if rng.random() < 0.3:  # isotropic point source strictly inside
        p = tuple(float(x) for x in rng.uniform(0.2, 0.8, 3) * (nx * h, ny * h, nz * h))
        src = v.Source(p, (0.0, 0.0, 1.0), isotropic=True)
    else:  # pencil on the entry face, random oblique direction into the volume
        p = (float(rng.uniform(0.1, 0.9) * nx * h), float(rng.uniform(0.1, 0.9) * ny * h), 0.0)
        d = np.array([rng.uniform(-0.6, 0.6), rng.uniform(-0.6, 0.6), 1.0])
        src = v.Source(p, tuple(float(x) for x in d / np.linalg.norm(d)))
    cfg = v.SimulationConfig(
        photon_count=50_000, master_seed=int(rng.integers(1, 1 << 40)),
        tmax_ns=float(rng.choice([0.05, 0.3, 1.0, 5.0])),
        boundary_mode=v.BoundaryMode.ReflectAtMismatch if rng.random() < 0.6 else v.BoundaryMode.TerminateAtBoundary)
    if gates:
        cfg.ngates = int(rng.integers(1, 5))
    if detectors and rng.random() < 0.6:
        k = int(rng.integers(1, 4))
        cfg.detectors = [v.Detector((float(rng.uniform(0, nx * h)), float(rng.uniform(0, ny * h)), 0.0),
                                    float(rng.uniform(0.3, 0.3 * min(nx, ny) * h))) for _ in range(k)]
        cfg.det_capacity = 1 << 17
    return v.Scene(grid, src), cfg


SEEDS = list(range(24))
