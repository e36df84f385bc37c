"""Run front door: JSON config and device roster -> run -> energy audit ->
report + raw volume (reference proj/core/src/config.cpp:37-321,
proj/core/include/voxmc/config.hpp:16-75).

Config keys are the reference's (config.cpp:150-227): "benchmark" (b1|b2|b2a)
or "grid" {dims, voxel_size_mm} + "media" [{mua,mus,g,n}, ...] (+ optional
"sphere" {center, radius, medium|label}) + "source" {position, direction,
isotropic}; "photons", "seed", "mode" (atomic|merge), "boundary"
(terminate|reflect), "tmax_ns", "roulette_threshold", "roulette_multiplier",
"workgroup_size", "devices" (roster path or inline array), "strategy"
(s1|s2|s3), "output", "report". B200 additions: "gates", "precision"
(fp32|fp64), "detectors" [{position, radius}], "det_capacity", "labels_file"
(raw uint8 x-fastest labels matching grid.dims). Roster devices take
"kind": "gpu" (with "gpu": ordinal) in addition to the reference's kinds.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import runtime as R
from .errors import IoError, ParseError, ValidationError
from .scene import (AccumulationMode, Benchmark, BoundaryMode, Detector, OpticalProperties, Precision, Scene,
                    SimulationConfig, Source, VoxelGrid, benchmark_from_name, benchmark_preset)
from .volume_io import fnv1a64, write_volume


@dataclass
class RunSetup:
    scene: Scene
    config: SimulationConfig
    devices: List[R.DeviceProfile] = field(default_factory=list)
    strategy: R.Strategy = R.Strategy.S1
    output_path: str = ""
    report_path: str = ""


@dataclass
class DeviceReport:
    name: str
    photons: int
    wall_ms: float


@dataclass
class RunReport:
    devices: List[DeviceReport]
    makespan_ms: float
    throughput_photons_per_ms: float
    conservation_residual: float
    strategy: str
    photon_count: int
    seed: int
    mode: str
    boundary: str
    reduce_ms: float = 0.0


@dataclass
class RunResult:
    map: R.FluenceMap
    report: RunReport
    detections: Optional[np.ndarray] = None


def _vec3(j, name):
    if not isinstance(j, list) or len(j) != 3:
        raise ParseError(f"{name}: expected an array of 3 numbers")
    return tuple(float(x) for x in j)


def _medium(m) -> OpticalProperties:
    try:
        return OpticalProperties(float(m["mua"]), float(m["mus"]), float(m["g"]), float(m["n"]))
    except (KeyError, TypeError) as e:
        raise ParseError(f"medium: {e}") from e


def parse_device(j) -> R.DeviceProfile:  # config.cpp:37-58 + kind "gpu"
    try:
        name = str(j["name"])
    except (KeyError, TypeError) as e:
        raise ParseError(f"device: {e}") from e
    d = R.DeviceProfile(name=name, cores=int(j.get("cores", 1)), a=float(j.get("a", 0.0)),
                        t0=float(j.get("t0", 0.0)), jitter_sigma=float(j.get("jitter_sigma", 0.0)),
                        gpu=int(j.get("gpu", 0)))
    if d.cores < 1:
        raise ValidationError(f"device {name}: cores must be >= 1")
    kind = j.get("kind", "simulated")
    kinds = {"simulated": R.DeviceKind.Simulated, "real": R.DeviceKind.RealWorkerPool,
             "worker-pool": R.DeviceKind.RealWorkerPool, "gpu": R.DeviceKind.CudaGpu}
    if kind not in kinds:
        raise ParseError(f"device {name}: unknown kind '{kind}'")
    d.kind = kinds[kind]
    if d.kind == R.DeviceKind.Simulated and not (d.a > 0.0):
        raise ValidationError(f"device {name}: simulated devices need a > 0")
    if d.t0 < 0.0:
        raise ValidationError(f"device {name}: t0 must be >= 0")
    return d


def parse_roster_text(text: str) -> List[R.DeviceProfile]:
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ParseError(f"roster: {e}") from e
    if not isinstance(j, list) or not j:
        raise ParseError("roster: expected a non-empty array")
    return [parse_device(d) for d in j]


def load_roster(path: str) -> List[R.DeviceProfile]:
    try:
        text = open(path).read()
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    return parse_roster_text(text)


def _grid(root, base_dir: str) -> VoxelGrid:  # config.cpp:60-104
    jg, jm = root["grid"], root["media"]
    if not isinstance(jm, list) or len(jm) < 2:
        raise ParseError("media: expected an array with the exterior medium plus at least one more")
    media = [_medium(m) for m in jm]
    nx, ny, nz = (int(x) for x in jg["dims"])
    h = float(jg.get("voxel_size_mm", jg.get("voxel_size", 1.0)))
    if nx < 1 or ny < 1 or nz < 1 or not (h > 0.0):
        raise ValidationError("grid: dims must be >= 1 and voxel_size > 0")
    if "labels_file" in root:
        p = root["labels_file"]
        p = p if os.path.isabs(p) else os.path.join(base_dir, p)
        try:
            labels = np.fromfile(p, dtype=np.uint8)
        except OSError as e:
            raise IoError(f"cannot open {p}") from e
        if labels.size != nx * ny * nz:
            raise ValidationError("labels_file: size does not match grid.dims")
        labels = labels.reshape(nz, ny, nx).copy()
    else:
        labels = np.ones((nz, ny, nx), np.uint8)
    if "sphere" in root:
        js = root["sphere"]
        c = _vec3(js["center"], "sphere.center")
        r = float(js["radius"])
        if "medium" in js:
            media.append(_medium(js["medium"]))
            lbl = len(media) - 1
        else:
            lbl = int(js.get("label", len(media) - 1))
        z, y, x = np.meshgrid((np.arange(nz) + 0.5) * h, (np.arange(ny) + 0.5) * h, (np.arange(nx) + 0.5) * h,
                              indexing="ij")
        labels[(x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 <= r * r] = lbl
    return VoxelGrid((nx, ny, nz), h, labels, media)


def _source(js) -> Source:
    s = Source(position=_vec3(js["position"], "source.position"))
    if "direction" in js:
        d = _vec3(js["direction"], "source.direction")
        n = math.sqrt(sum(x * x for x in d))
        s.direction = tuple(x / n for x in d)
    s.isotropic = bool(js.get("isotropic", False))
    return s


def parse_config_obj(root, base_dir: str = ".") -> RunSetup:  # config.cpp:150-227
    try:
        preset = None
        if "benchmark" in root:
            b = benchmark_from_name(str(root["benchmark"]))
            if b is None:
                raise ParseError(f"unknown benchmark '{root['benchmark']}'")
            preset = benchmark_preset(b)
        grid = _grid(root, base_dir) if "grid" in root else None
        source = _source(root["source"]) if "source" in root else None
        if preset is None and (grid is None or source is None):
            raise ParseError('config: need either "benchmark" or explicit "grid"+"media"+"source"')
        cfg = preset.config if preset else SimulationConfig()
        if "photons" in root:
            p = int(root["photons"])
            if p < 1:
                raise ValidationError("photons must be >= 1")
            cfg.photon_count = p
        cfg.master_seed = int(root.get("seed", cfg.master_seed))
        if "mode" in root:
            m = root["mode"]
            if m not in ("atomic", "merge"):
                raise ValidationError("mode must be 'atomic' or 'merge'")
            cfg.accumulation_mode = AccumulationMode.SharedAtomic if m == "atomic" else AccumulationMode.PrivateMerge
        if "boundary" in root:
            b = root["boundary"]
            if b not in ("terminate", "reflect"):
                raise ValidationError("boundary must be 'terminate' or 'reflect'")
            cfg.boundary_mode = (BoundaryMode.TerminateAtBoundary if b == "terminate"
                                 else BoundaryMode.ReflectAtMismatch)
        cfg.tmax_ns = float(root.get("tmax_ns", cfg.tmax_ns))
        cfg.roulette_threshold = float(root.get("roulette_threshold", cfg.roulette_threshold))
        cfg.roulette_multiplier = int(root.get("roulette_multiplier", cfg.roulette_multiplier))
        cfg.workgroup_size = int(root.get("workgroup_size", cfg.workgroup_size))
        cfg.ngates = int(root.get("gates", cfg.ngates))
        if "precision" in root:
            if root["precision"] not in ("fp32", "fp64"):
                raise ValidationError("precision must be 'fp32' or 'fp64'")
            cfg.precision = Precision.FP64 if root["precision"] == "fp64" else Precision.FP32
        if "detectors" in root:
            cfg.detectors = [Detector(_vec3(d["position"], "detector.position"), float(d["radius"]))
                             for d in root["detectors"]]
            cfg.det_capacity = int(root.get("det_capacity", 1 << 20))
        cfg.validate()
        setup = RunSetup(Scene(grid if grid is not None else preset.grid,
                               source if source is not None else preset.source), cfg,
                         output_path=str(root.get("output", "")), report_path=str(root.get("report", "")))
        if "devices" in root:
            jd = root["devices"]
            if isinstance(jd, str):
                setup.devices = load_roster(jd if os.path.isabs(jd) else os.path.join(base_dir, jd))
            elif isinstance(jd, list):
                setup.devices = [parse_device(d) for d in jd]
            else:
                raise ParseError("devices: expected roster path or inline array")
        if "strategy" in root:
            s = R.strategy_from_name(str(root["strategy"]))
            if s is None:
                raise ValidationError("strategy must be one of s1, s2, s3")
            setup.strategy = s
        return setup
    except (KeyError, TypeError, ValueError) as e:
        if isinstance(e, (ValidationError, ParseError)):
            raise
        raise ParseError(f"config: {e}") from e


def parse_config_text(text: str, base_dir: str = ".") -> RunSetup:
    try:
        root = json.loads(text)
    except json.JSONDecodeError as e:
        raise ParseError(f"config: {e}") from e
    return parse_config_obj(root, base_dir)


def parse_config(path: str) -> RunSetup:
    try:
        text = open(path).read()
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    return parse_config_text(text, os.path.dirname(os.path.abspath(path)))


def gpu_roster(n: Optional[int] = None) -> List[R.DeviceProfile]:
    n = R.device_count() if n is None else n
    return [R.DeviceProfile(name=f"gpu{i}", cores=1, a=1.0, kind=R.DeviceKind.CudaGpu, gpu=i) for i in range(n)]


def scene_hash(scene: Scene, config: SimulationConfig) -> int:
    """Physics-content hash keying the calibration cache (config.cpp:249-269)."""
    g = scene.grid
    parts = [np.array(g.dims, np.int32).tobytes(), np.array([g.voxel_size], np.float64).tobytes(),
             g.labels.tobytes(), g.media_array().tobytes(),
             np.array(scene.source.position, np.float64).tobytes(),
             np.array(scene.source.direction, np.float64).tobytes(),
             bytes([1 if scene.source.isotropic else 0]),
             np.array([int(config.boundary_mode)], np.int32).tobytes(),
             np.array([config.tmax_ns], np.float64).tobytes(),
             np.array([config.ngates], np.int32).tobytes()]
    return fnv1a64(np.frombuffer(b"".join(parts), np.uint8))


def cache_lookup(cache: str, device_name: str, key: int) -> Optional[R.Calibration]:
    try:
        j = json.load(open(cache))
    except (OSError, json.JSONDecodeError):
        return None
    e = j.get(f"{device_name}@{key:016x}")
    return R.Calibration(float(e["a"]), float(e["t0"])) if e else None


def cache_store(cache: str, device_name: str, key: int, cal: R.Calibration) -> None:
    try:
        j = json.load(open(cache))
    except (OSError, json.JSONDecodeError):
        j = {}
    j[f"{device_name}@{key:016x}"] = {"a": cal.a, "t0": cal.t0}
    with open(cache, "w") as f:
        json.dump(j, f, indent=2)


def report_to_json(r: RunReport) -> str:  # config.cpp:271-286
    return json.dumps({
        "devices": [{"name": d.name, "photons": d.photons, "wall_ms": d.wall_ms} for d in r.devices],
        "makespan_ms": r.makespan_ms, "throughput_photons_per_ms": r.throughput_photons_per_ms,
        "conservation_residual": r.conservation_residual, "strategy": r.strategy,
        "photon_count": r.photon_count, "seed": r.seed, "mode": r.mode, "boundary": r.boundary,
        "reduce_ms": r.reduce_ms}, indent=2)


def run_pipeline(setup: RunSetup) -> RunResult:
    """Partition across the GPU roster, simulate, merge, audit energy conservation
    (ValidationError when |residual| > 1e-6, config.cpp:316-319), write outputs."""
    setup.config.validate()
    devices = setup.devices or gpu_roster()
    if not devices:
        raise RuntimeError("no CUDA device available (the B200 library has no CPU fallback)")
    n = setup.config.photon_count
    res = R.run_multi_device(n, devices, setup.strategy, setup.scene, setup.config)
    t = res.totals
    residual = (sum(res.totals_q) * res.map.quantum - n) / n
    rep = RunReport([DeviceReport(d.name, d.photons, d.wall_ms) for d in res.devices], res.makespan_ms,
                    n / res.makespan_ms if res.makespan_ms > 0 else 0.0, residual,
                    {R.Strategy.S1: "s1", R.Strategy.S2: "s2", R.Strategy.S3: "s3"}[setup.strategy], n,
                    setup.config.master_seed,
                    "atomic" if setup.config.accumulation_mode == AccumulationMode.SharedAtomic else "merge",
                    "terminate" if setup.config.boundary_mode == BoundaryMode.TerminateAtBoundary else "reflect",
                    res.reduce_ms)
    if abs(residual) > 1e-6:
        raise ValidationError(f"energy conservation violated: relative residual {residual}")
    del t
    if setup.output_path:
        # `output` is the reference's file: the continuous-wave volume (gates
        # summed in integers first), nx*ny*nz floats + sidecar (volume_io.cpp:
        # 26-53), readable by the reference's read_volume. Gate-resolved maps go
        # to a separate `<output>.gates.raw` (+ its own sidecar with "gates").
        g = setup.scene.grid
        write_volume(res.map.to_float_volume(), g.dims, g.voxel_size, n, setup.config.master_seed,
                     setup.output_path, normalized=False)
        if setup.config.ngates > 1:
            vol = (res.map.cells.astype(np.float64) * res.map.quantum).astype(np.float32)
            write_volume(vol, g.dims, g.voxel_size, n, setup.config.master_seed, setup.output_path + ".gates.raw",
                         normalized=False, gates=setup.config.ngates)
    if setup.report_path:
        with open(setup.report_path, "w") as f:
            f.write(report_to_json(rep) + "\n")
    return RunResult(res.map, rep, res.detections)
