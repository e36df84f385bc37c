"""Host-side mirror of the reference's domain types (L1 of SURVEY.md §1).

Names, fields and validation follow the reference C++ API so that code written
against voxmc reads the same here:
  OpticalProperties  proj/core/include/voxmc/types.hpp:37-44
  VoxelGrid          types.hpp:56-92, ctor checks proj/core/src/types.cpp:7-33,
                     voxel_of types.cpp:35-42
  SimulationConfig   types.hpp:97-108, validate types.cpp:44-52
  Source / Scene     types.hpp:112-121
  benchmark_preset   types.cpp:56-95 (B1 / B2 / B2a)
plus the B200 build's additions (no reference equivalent): time gates and
disk detectors on SimulationConfig, and the BASELINE.json workloads
(baseline_setup: "b1", "b2", "b3", "head").

Validation errors raise the reference's exception types (errors.py).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .errors import SourceOutsideDomain, ValidationError

LIGHT_SPEED_MM_PER_NS = 299.792458  # types.hpp:16


class AccumulationMode(enum.IntEnum):  # types.hpp:94
    SharedAtomic = _abi.VMC_ACCUM_SHARED_ATOMIC
    PrivateMerge = _abi.VMC_ACCUM_PRIVATE_MERGE


class BoundaryMode(enum.IntEnum):  # types.hpp:95
    TerminateAtBoundary = _abi.VMC_BOUNDARY_TERMINATE
    ReflectAtMismatch = _abi.VMC_BOUNDARY_REFLECT


class Precision(enum.IntEnum):
    FP32 = _abi.VMC_PRECISION_FP32
    FP64 = _abi.VMC_PRECISION_FP64


@dataclass(frozen=True)
class OpticalProperties:
    mua: float = 0.0
    mus: float = 0.0
    g: float = 0.0
    n: float = 1.0


@dataclass(frozen=True)
class VoxelIndex:
    x: int = 0
    y: int = 0
    z: int = 0


class VoxelGrid:
    """Labeled volume; labels uint8 in x-fastest order (shape (nz, ny, nx))."""

    def __init__(self, dims: Tuple[int, int, int], voxel_size_mm: float, labels,
                 media: Sequence[OpticalProperties]):
        nx, ny, nz = (int(d) for d in dims)
        if nx < 1 or ny < 1 or nz < 1:
            raise ValidationError("VoxelGrid: all dims must be >= 1")
        if not (voxel_size_mm > 0.0):
            raise ValidationError("VoxelGrid: voxel_size must be > 0")
        lab = np.ascontiguousarray(np.asarray(labels, dtype=np.uint8).reshape(-1))
        if lab.size != nx * ny * nz:
            raise ValidationError("VoxelGrid: label array size does not match dims")
        if len(media) == 0:
            raise ValidationError("VoxelGrid: media list is empty")
        for m in media:
            if m.mua < 0.0 or m.mus < 0.0 or m.g < -1.0 or m.g > 1.0 or m.n < 1.0:
                raise ValidationError("VoxelGrid: invalid optical properties")
        if lab.size and int(lab.max()) >= len(media):
            raise ValidationError("VoxelGrid: label exceeds media list")
        self._dims = (nx, ny, nz)
        self._h = float(voxel_size_mm)
        self._labels = lab
        self._media = [OpticalProperties(*map(float, (m.mua, m.mus, m.g, m.n))) for m in media]

    @property
    def dims(self):
        return self._dims

    nx = property(lambda s: s._dims[0])
    ny = property(lambda s: s._dims[1])
    nz = property(lambda s: s._dims[2])

    @property
    def voxel_size(self) -> float:
        return self._h

    @property
    def voxel_count(self) -> int:
        return self._labels.size

    @property
    def labels(self) -> np.ndarray:
        return self._labels

    @property
    def media(self) -> List[OpticalProperties]:
        return list(self._media)

    def linear(self, v) -> int:
        x, y, z = (v.x, v.y, v.z) if isinstance(v, VoxelIndex) else v
        return x + self.nx * (y + self.ny * z)

    def contains(self, v) -> bool:
        x, y, z = (v.x, v.y, v.z) if isinstance(v, VoxelIndex) else v
        return 0 <= x < self.nx and 0 <= y < self.ny and 0 <= z < self.nz

    def label(self, v) -> int:
        return int(self._labels[self.linear(v)])

    def medium(self, lbl: int) -> OpticalProperties:
        return self._media[lbl]

    def voxel_of(self, p) -> Optional[VoxelIndex]:
        v = VoxelIndex(*(int(math.floor(c / self._h)) for c in p))
        return v if self.contains(v) else None

    def media_array(self) -> np.ndarray:
        return np.array([[m.mua, m.mus, m.g, m.n] for m in self._media], dtype=np.float64)


@dataclass
class Source:
    position: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    direction: Tuple[float, float, float] = (0.0, 0.0, 1.0)
    isotropic: bool = False


@dataclass
class Detector:
    """Disk detector (B200 addition): records exiting photons within
    `radius` mm of `position`."""
    position: Tuple[float, float, float]
    radius: float


@dataclass
class SimulationConfig:
    photon_count: int = 100_000_000
    master_seed: int = 0
    accumulation_mode: AccumulationMode = AccumulationMode.PrivateMerge
    boundary_mode: BoundaryMode = BoundaryMode.TerminateAtBoundary
    tmax_ns: float = 5.0
    roulette_threshold: float = 1e-4
    roulette_multiplier: int = 10
    workgroup_size: int = 64
    # --- B200 additions -------------------------------------------------
    ngates: int = 1
    precision: Precision = Precision.FP32
    detectors: List[Detector] = field(default_factory=list)
    det_capacity: int = 0

    def validate(self) -> None:  # types.cpp:44-52
        if self.photon_count < 1:
            raise ValidationError("photon_count must be >= 1")
        if not (self.tmax_ns > 0.0):
            raise ValidationError("tmax must be > 0")
        if not (0.0 < self.roulette_threshold < 1.0):
            raise ValidationError("roulette_threshold must be in (0, 1)")
        if self.roulette_multiplier < 2:
            raise ValidationError("roulette_multiplier must be >= 2")
        if self.workgroup_size < 1:
            raise ValidationError("workgroup_size must be >= 1")
        if self.ngates < 1:
            raise ValidationError("ngates must be >= 1")


@dataclass
class Scene:
    grid: VoxelGrid
    source: Source


@dataclass
class BenchmarkSetup:
    grid: VoxelGrid
    source: Source
    config: SimulationConfig

    @property
    def scene(self) -> Scene:
        return Scene(self.grid, self.source)


class Benchmark(enum.Enum):
    B1 = "B1"
    B2 = "B2"
    B2a = "B2a"


def benchmark_from_name(name: str) -> Optional[Benchmark]:
    return {"B1": Benchmark.B1, "b1": Benchmark.B1, "B2": Benchmark.B2, "b2": Benchmark.B2,
            "B2a": Benchmark.B2a, "b2a": Benchmark.B2a, "B2A": Benchmark.B2a}.get(name)


AIR = OpticalProperties(0.0, 0.0, 0.0, 1.0)
CUBE_BACKGROUND = OpticalProperties(0.005, 1.0, 0.01, 1.37)
CUBE_SPHERE = OpticalProperties(0.002, 5.0, 0.9, 1.0)


def _cube_labels(with_sphere: bool) -> np.ndarray:
    n = 60
    lab = np.ones((n, n, n), dtype=np.uint8)  # (z, y, x)
    if with_sphere:
        c = (np.arange(n) + 0.5) - 30.0
        r2 = c[:, None, None] ** 2 + c[None, :, None] ** 2 + c[None, None, :] ** 2
        lab[r2 <= 15.0 * 15.0] = 2
    return lab


def benchmark_preset(name: Benchmark) -> BenchmarkSetup:
    """Reference presets (types.cpp:56-95): 60^3 cube, pencil at (30,30,0) +z."""
    sphere = name != Benchmark.B1
    media = [AIR, CUBE_BACKGROUND] + ([CUBE_SPHERE] if sphere else [])
    grid = VoxelGrid((60, 60, 60), 1.0, _cube_labels(sphere), media)
    cfg = SimulationConfig(
        photon_count=100_000_000,
        boundary_mode=BoundaryMode.ReflectAtMismatch if sphere else BoundaryMode.TerminateAtBoundary,
        accumulation_mode=(AccumulationMode.SharedAtomic if name == Benchmark.B2a
                           else AccumulationMode.PrivateMerge))
    return BenchmarkSetup(grid, Source((30.0, 30.0, 0.0), (0.0, 0.0, 1.0), False), cfg)


HEAD_MEDIA = [
    AIR,
    OpticalProperties(0.019, 7.8, 0.89, 1.37),   # 1 scalp
    OpticalProperties(0.019, 7.8, 0.89, 1.37),   # 2 skull
    OpticalProperties(0.004, 0.009, 0.89, 1.37),  # 3 CSF
    OpticalProperties(0.02, 9.0, 0.89, 1.37),    # 4 gray
    OpticalProperties(0.08, 40.9, 0.84, 1.37),   # 5 white
]


def head_labels(n: int = 256) -> np.ndarray:
    """Synthetic 5-label head-like volume: shells by voxel
    centre distance from the volume centre, scaled from the 256^3 radii."""
    s = n / 256.0
    c = (np.arange(n, dtype=np.float64) + 0.5) - n / 2.0
    r = np.sqrt(c[:, None, None] ** 2 + c[None, :, None] ** 2 + c[None, None, :] ** 2)
    lab = np.full((n, n, n), 1, dtype=np.uint8)
    lab[r < 115 * s] = 2
    lab[r < 108 * s] = 3
    lab[r < 106 * s] = 4
    lab[r < 100 * s] = 5
    return lab


def b3_detectors() -> List[Detector]:
    """4 disk detectors, r = 1 mm, 10 mm from the source on the entry face."""
    return [Detector((30.0, 20.0, 0.0), 1.0), Detector((30.0, 40.0, 0.0), 1.0),
            Detector((20.0, 30.0, 0.0), 1.0), Detector((40.0, 30.0, 0.0), 1.0)]


def baseline_setup(name: str, photons: Optional[int] = None, seed: int = 1,
                   head_n: int = 256) -> BenchmarkSetup:
    """BASELINE.json workloads:
    b1   reference B1 preset (terminate at boundary), 1e6 photons;
    b2   B1 grid + Fresnel reflection at the mismatched outer boundary, 1e8, 1 gate;
    b3   reference B2 preset (15 mm sphere, reflect) + 4 detectors, 1e8;
    head 256^3 5-label volume, reflect, 10 gates x 0.5 ns, 1e8."""
    name = name.lower()
    if name == "b1":
        st = benchmark_preset(Benchmark.B1)
        st.config.photon_count = photons or 1_000_000
    elif name == "b2":
        st = benchmark_preset(Benchmark.B1)
        st.config.boundary_mode = BoundaryMode.ReflectAtMismatch
        st.config.photon_count = photons or 100_000_000
    elif name == "b3":
        st = benchmark_preset(Benchmark.B2)
        st.config.photon_count = photons or 100_000_000
        st.config.detectors = b3_detectors()
        st.config.det_capacity = 1 << 20
    elif name == "head":
        grid = VoxelGrid((head_n, head_n, head_n), 256.0 / head_n, head_labels(head_n), HEAD_MEDIA)
        cfg = SimulationConfig(photon_count=photons or 100_000_000,
                               boundary_mode=BoundaryMode.ReflectAtMismatch, ngates=10)
        st = BenchmarkSetup(grid, Source((128.0, 128.0, 0.0), (0.0, 0.0, 1.0), False), cfg)
    else:
        raise ValidationError(f"unknown baseline workload '{name}'")
    st.config.master_seed = seed
    return st


class Marshalled:
    """vmc_scene / vmc_config structs plus the numpy buffers they point at."""

    def __init__(self, scene: Scene, config: SimulationConfig):
        g = scene.grid
        self.labels = g.labels
        self.media = np.ascontiguousarray(g.media_array().reshape(-1))
        self.scene = _abi.vmc_scene()
        s = self.scene
        s.nx, s.ny, s.nz = g.dims
        s.voxel_mm = g.voxel_size
        s.labels = self.labels.ctypes.data_as(C.POINTER(C.c_uint8))
        s.nmedia = len(g.media)
        s.media = self.media.ctypes.data_as(C.POINTER(C.c_double))
        s.src_pos[:] = [float(v) for v in scene.source.position]
        s.src_dir[:] = [float(v) for v in scene.source.direction]
        s.isotropic = 1 if scene.source.isotropic else 0
        self.config = _abi.vmc_config()
        c = self.config
        c.photon_count = int(config.photon_count)
        c.master_seed = int(config.master_seed) & 0xFFFFFFFFFFFFFFFF
        c.accumulation_mode = int(config.accumulation_mode)
        c.boundary_mode = int(config.boundary_mode)
        c.tmax_ns = float(config.tmax_ns)
        c.roulette_threshold = float(config.roulette_threshold)
        c.roulette_multiplier = int(config.roulette_multiplier)
        c.workgroup_size = 0
        c.ngates = int(config.ngates)
        c.precision = int(config.precision)
        dets = config.detectors or []
        self.det = np.array([[*d.position, d.radius] for d in dets], dtype=np.float64).reshape(-1)
        c.ndet = len(dets)
        c.det = self.det.ctypes.data_as(C.POINTER(C.c_double)) if dets else None
        c.det_capacity = int(config.det_capacity)
        self.nmedia = len(g.media)
        self.ncells = g.voxel_count * int(config.ngates)


def check_source_inside(scene: Scene) -> None:
    """Pencil-source launch voxel check (transport.cpp:95-99)."""
    s = scene.source
    if s.isotropic:
        d = (0.0, 0.0, 0.0)
    else:
        nrm = math.sqrt(sum(c * c for c in s.direction))
        d = tuple(c / nrm for c in s.direction)
    p = tuple(a + b * 1e-6 for a, b in zip(s.position, d))
    if scene.grid.voxel_of(p) is None:
        raise SourceOutsideDomain("source entry point maps outside the voxel grid")
