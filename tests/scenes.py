"""Small scenes that stress branches the BASELINE workloads rarely take
(shared by the GPU parity tests and the CPU oracle tests)."""
import numpy as np

import paper_1711_03244_b200 as v


def corner_scene(kind):
    """Small scenes that stress branches the BASELINE workloads rarely take."""
    n = 20
    lab = np.ones((n, n, n), np.uint8)
    c = (np.arange(n) + 0.5) - n / 2
    r2 = c[:, None, None] ** 2 + c[None, :, None] ** 2 + c[None, None, :] ** 2
    air = v.OpticalProperties(0, 0, 0, 1.0)
    cfg = v.SimulationConfig(photon_count=50_000, master_seed=9, tmax_ns=5.0,
                             boundary_mode=v.BoundaryMode.ReflectAtMismatch)
    src = v.Source((10.0, 10.0, 0.0), (0.0, 0.0, 1.0))
    if kind == "roulette":  # strong absorption: weights fall below 1e-4 -> roulette
        media = [air, v.OpticalProperties(0.3, 10.0, 0.0, 1.3)]
    elif kind == "horizon":  # short time horizon: most photons truncated
        media = [air, v.OpticalProperties(0.01, 2.0, 0.5, 1.4)]
        cfg.tmax_ns = 0.05
    elif kind == "backward":  # negative anisotropy, isotropic-branch medium inside
        media = [air, v.OpticalProperties(0.02, 3.0, -0.5, 1.33), v.OpticalProperties(0.01, 1.0, 0.0, 1.33)]
        lab[r2 <= 25] = 2
    elif kind == "dense_inclusion":  # high-index sphere, refraction both ways + TIR inside
        media = [air, v.OpticalProperties(0.005, 1.0, 0.8, 1.0), v.OpticalProperties(0.01, 4.0, 0.9, 1.6)]
        lab[r2 <= 36] = 2
    elif kind == "terminate_inner":  # terminate mode still resolves inner mismatches
        media = [air, v.OpticalProperties(0.01, 1.0, 0.7, 1.37), v.OpticalProperties(0.01, 1.0, 0.7, 1.0)]
        lab[r2 <= 36] = 2
        cfg.boundary_mode = v.BoundaryMode.TerminateAtBoundary
    elif kind == "oblique":  # oblique pencil off a voxel corner
        media = [air, v.OpticalProperties(0.01, 1.0, 0.9, 1.37)]
        src = v.Source((7.0, 9.0, 0.0), (0.3, -0.2, 0.9))
    elif kind == "ballistic":  # mus = 0 shell + in-grid air (label 0): long flights, same-n label changes
        media = [air, v.OpticalProperties(0.02, 2.0, 0.8, 1.37), v.OpticalProperties(0.004, 0.0, 0.0, 1.37)]
        lab[(r2 > 16) & (r2 <= 49)] = 2
        lab[:, :, n - 3:] = 0
    elif kind == "aniso_grid":  # non-cubic grid, non-integer voxel size (scaled-index decode, plane landing)
        nx, ny, nz = 17, 23, 29
        lab = np.ones((nz, ny, nx), np.uint8)
        media = [air, v.OpticalProperties(0.01, 1.5, 0.85, 1.4)]
        grid = v.VoxelGrid((nx, ny, nz), 0.37, lab, media)
        src = v.Source((17 * 0.37 / 2, 23 * 0.37 / 2, 0.0), (0.1, 0.05, 1.0))
        return v.Scene(grid, src), cfg
    elif kind == "mosaic":  # 2x2x2-voxel blocks of 5 random media (4 refractive indices): interfaces
        # in every direction, Fresnel / TIR / refraction on most faces
        rng = np.random.default_rng(17)
        blocks = rng.integers(1, 6, (n // 2, n // 2, n // 2)).astype(np.uint8)
        lab = np.repeat(np.repeat(np.repeat(blocks, 2, 0), 2, 1), 2, 2)
        media = [air, v.OpticalProperties(0.01, 1.0, 0.8, 1.37), v.OpticalProperties(0.02, 2.0, 0.5, 1.0),
                 v.OpticalProperties(0.005, 0.5, 0.9, 1.45), v.OpticalProperties(0.03, 4.0, 0.0, 1.33),
                 v.OpticalProperties(0.01, 1.5, -0.3, 1.37)]
    elif kind == "iso_layers":  # isotropic point source inside layered media of different n
        media = [air, v.OpticalProperties(0.01, 1.0, 0.9, 1.37), v.OpticalProperties(0.02, 3.0, 0.7, 1.45),
                 v.OpticalProperties(0.005, 0.2, 0.0, 1.33)]
        z = np.arange(n)[:, None, None] * np.ones((1, n, n), np.int64)
        lab = np.where(z < 7, 1, np.where(z < 13, 2, 3)).astype(np.uint8)
        src = v.Source((9.7, 10.3, 10.1), (0.0, 0.0, 1.0), isotropic=True)
    grid = v.VoxelGrid((n, n, n), 1.0, lab, media)
    return v.Scene(grid, src), cfg


CORNERS = ["roulette", "horizon", "backward", "dense_inclusion", "terminate_inner", "oblique", "ballistic",
           "aniso_grid", "mosaic", "iso_layers"]
