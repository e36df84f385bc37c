"""Raw fluence volume export (reference proj/core/src/volume_io.cpp:13-89).

Headerless little-endian float32, x fastest, plus a `<path>.json` sidecar
{dims, voxel_size_mm, photon_count, normalized, seed, checksum, ordering} where
checksum is the FNV-1a-64 of the float bytes. read_volume verifies it
(IoError on mismatch). Time-gated maps add "gates" to the sidecar and store
[gate][z][y][x].
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from .errors import IoError, ParseError


def fnv1a64(data) -> int:
    """FNV-1a 64 over raw bytes (volume_io.cpp:13-20), computed by the native
    library (vmc_fnv1a64; host code, no GPU needed)."""
    import ctypes as C

    from .runtime import lib
    arr = np.ascontiguousarray(data if isinstance(data, np.ndarray) else np.frombuffer(bytes(data), np.uint8))
    return int(lib().vmc_fnv1a64(C.c_void_p(arr.ctypes.data), arr.nbytes))


@dataclass
class VolumeData:
    dims: tuple
    voxel_size_mm: float
    photon_count: int
    normalized: bool
    seed: int
    checksum: int
    values: np.ndarray
    gates: int = 1


def write_volume(values: np.ndarray, dims, voxel_size_mm: float, photon_count: int, seed: int,
                 path: str, normalized: bool = False, gates: int = 1) -> int:
    vol = np.ascontiguousarray(values, dtype="<f4").reshape(-1)
    nx, ny, nz = dims
    if vol.size != nx * ny * nz * gates:
        raise IoError("write_volume: value count does not match dims")
    checksum = fnv1a64(vol)
    try:
        with open(path, "wb") as f:
            f.write(vol.tobytes())
        side = {"dims": [nx, ny, nz], "voxel_size_mm": voxel_size_mm, "photon_count": int(photon_count),
                "normalized": bool(normalized), "seed": int(seed), "checksum": checksum,
                "ordering": "x-fastest"}
        if gates > 1:
            side["gates"] = gates
        with open(path + ".json", "w") as f:
            json.dump(side, f, indent=2)
            f.write("\n")
    except OSError as e:
        raise IoError(f"write_volume: {e}") from e
    return checksum


def read_volume(path: str) -> VolumeData:
    side_path = path + ".json"
    if not os.path.exists(side_path):
        raise IoError(f"read_volume: missing sidecar {side_path}")
    try:
        with open(side_path) as f:
            side = json.load(f)
    except json.JSONDecodeError as e:
        raise ParseError(f"read_volume: bad sidecar: {e}") from e
    nx, ny, nz = (int(x) for x in side["dims"])
    gates = int(side.get("gates", 1))
    n = nx * ny * nz * gates
    try:
        raw = open(path, "rb").read()
    except OSError as e:
        raise IoError(f"read_volume: cannot open {path}") from e
    if len(raw) < 4 * n:
        raise IoError(f"read_volume: short read from {path}")
    vals = np.frombuffer(raw[:4 * n], dtype="<f4").copy()
    if fnv1a64(vals) != int(side["checksum"]):
        raise IoError(f"read_volume: checksum mismatch for {path}")
    return VolumeData((nx, ny, nz), float(side["voxel_size_mm"]), int(side["photon_count"]),
                      bool(side["normalized"]), int(side["seed"]), int(side["checksum"]), vals, gates)
