"""Python host API over the C-ABI (include/vmc.h) — the reference's executor
and scheduler names (proj/core/include/voxmc/scheduler.hpp, fluence.hpp,
transport.hpp) mapped onto the B200 library.

    run_group_dynamic   scheduler.hpp:94-95 -> vmc_run_range   (one GPU)
    run_static_split    scheduler.hpp:98-99 -> vmc_run_range   (same result by construction)
    run_multi_device    scheduler.hpp:139-141 -> vmc_run_multi (contiguous ranges + NCCL reduce)
    partition_s1/s2/s3, make_partition, model_makespan -> vmc_partition / vmc_model_makespan
    calibrate           scheduler.hpp:318-320 (GPU pilots timed on the device)
    FluenceMap          fluence.hpp:26-91 (raw int64 cells + quantum; add/merge/normalize)

There is no CPU fallback: if libvoxmc_b200.so is missing or no CUDA device is
present, every compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from .errors import (AlreadyNormalized, DimensionMismatch, NonPositiveSlope, SourceOutsideDomain,
                     ValidationError)
from .scene import Marshalled, Scene, SimulationConfig, VoxelGrid

_HERE = os.path.dirname(os.path.abspath(__file__))
# VMC_LIB_PATH: load an alternative build of the same library (kernel A/B runs)
LIB_PATH = os.environ.get("VMC_LIB_PATH") or os.path.join(_HERE, "lib", "libvoxmc_b200.so")
_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Load libvoxmc_b200.so (built by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_1711_03244_b200.build` "
                               "(there is no CPU fallback)")
        l = _abi.declare(C.CDLL(LIB_PATH))
        if l.vmc_abi_version() != _abi.VMC_ABI_VERSION:
            raise RuntimeError("libvoxmc_b200.so ABI version mismatch")
        _lib = l
    return _lib


def _check(rc: int) -> None:
    if rc == _abi.VMC_OK:
        return
    msg = (lib().vmc_last_error() or b"").decode()
    if rc == _abi.VMC_ERR_VALIDATION:
        if "outside the voxel grid" in msg:
            raise SourceOutsideDomain(msg)
        raise ValidationError(msg)
    raise RuntimeError(msg)


def device_count() -> int:
    return lib().vmc_device_count()


def quantum_for(photon_count: int) -> float:
    return lib().vmc_quantum_for(photon_count)


# ---------------------------------------------------------------------------
@dataclass
class PhotonDisposition:
    """transport.hpp:89-102, in launched-weight units."""
    deposited: float = 0.0
    escaped: float = 0.0
    killed: float = 0.0
    truncated: float = 0.0

    @classmethod
    def from_quanta(cls, q: Sequence[int], quantum: float) -> "PhotonDisposition":
        return cls(*(float(int(x)) * quantum for x in q))

    def books(self) -> float:
        return self.deposited + self.escaped + self.killed + self.truncated

    def __iadd__(self, o):
        self.deposited += o.deposited
        self.escaped += o.escaped
        self.killed += o.killed
        self.truncated += o.truncated
        return self


class FluenceMap:
    """Fixed-point fluence accumulator (fluence.hpp:26-91), gate-resolved.

    cells: int64 array (ngates, nz, ny, nx); value = cell * quantum."""

    def __init__(self, dims, photon_count: int, ngates: int = 1, cells: Optional[np.ndarray] = None):
        nx, ny, nz = dims
        if nx < 1 or ny < 1 or nz < 1:
            raise ValidationError("FluenceMap: dims must be >= 1")
        if photon_count < 1:
            raise ValidationError("FluenceMap: photon_count must be >= 1")
        self.dims = (nx, ny, nz)
        self.ngates = ngates
        self.photon_count = photon_count
        self.quantum = quantum_for_host(photon_count)
        shape = (ngates, nz, ny, nx)
        self.cells = np.zeros(shape, np.int64) if cells is None else np.asarray(cells, np.int64).reshape(shape)
        self._values: Optional[np.ndarray] = None

    @property
    def voxel_count(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    @property
    def normalized(self) -> bool:
        return self._values is not None

    def raw_cell(self, cell: int, gate: int = 0) -> int:
        return int(self.cells[gate].reshape(-1)[cell])

    def cw_cells(self) -> np.ndarray:
        """Gate-summed (CW) raw cells, x-fastest flat."""
        return self.cells.sum(axis=0).reshape(-1)

    def value(self, cell: int) -> float:
        if self._values is not None:
            return float(self._cw_values.reshape(-1)[cell])
        return float(self.cw_cells()[cell]) * self.quantum

    def total_deposited(self) -> float:
        return float(int(self.cells.sum())) * self.quantum

    def add(self, other: "FluenceMap") -> None:  # fluence.cpp:52-60
        if other.dims != self.dims or other.ngates != self.ngates:
            raise DimensionMismatch("FluenceMap::add: dims differ")
        if other.quantum != self.quantum:
            raise DimensionMismatch("FluenceMap::add: quantum differs")
        if self.normalized or other.normalized:
            raise AlreadyNormalized("FluenceMap::add: normalized map")
        self.cells += other.cells

    def normalize(self, grid: VoxelGrid) -> None:  # fluence.cpp:62-84
        if self.normalized:
            raise AlreadyNormalized("FluenceMap::normalize: already normalized")
        if grid.dims != self.dims:
            raise DimensionMismatch("FluenceMap::normalize: grid dims differ")
        # the reference's order: (double(cell) * quantum) / ((mua * v) * N),
        # v = h * h * h; gate-resolved values per gate, and the CW values from
        # the gate-summed cells (the reference's single map)
        mua = grid.media_array()[:, 0][grid.labels.astype(np.int64)].reshape(self.dims[::-1])
        h = float(grid.voxel_size)
        den = mua * (h * h * h) * float(self.photon_count)
        with np.errstate(divide="ignore", invalid="ignore"):
            vals = np.where(mua > 0.0, (self.cells.astype(np.float64) * self.quantum) / den, 0.0)
            cw = np.where(mua > 0.0, (self.cells.sum(axis=0).astype(np.float64) * self.quantum) / den, 0.0)
        self.zero_mua_voxels = int((mua <= 0.0).sum())
        self._values = vals
        self._cw_values = cw

    def to_float_volume(self) -> np.ndarray:  # fluence.cpp:86-90 (CW, x fastest)
        if self._values is not None:
            return self._cw_values.astype(np.float32).reshape(-1)
        return (self.cw_cells().astype(np.float64) * self.quantum).astype(np.float32)


def quantum_for_host(n: int) -> float:
    return math.ldexp(1.0, -(62 - int(n | 1).bit_length()))


def merge(maps: Sequence[FluenceMap]) -> FluenceMap:  # fluence.cpp:92-98
    if not maps:
        raise DimensionMismatch("merge: empty map list")
    out = FluenceMap(maps[0].dims, maps[0].photon_count, maps[0].ngates)
    for m in maps:
        out.add(m)
    return out


@dataclass
class GroupRunResult:
    map: FluenceMap
    totals: PhotonDisposition
    per_thread_photons: List[int]
    wall_ms: float = 0.0
    totals_q: tuple = (0, 0, 0, 0)
    detections: Optional[np.ndarray] = None
    det_count: int = 0


def _det_buffer(m: Marshalled, config: SimulationConfig):
    if not config.detectors:
        return None
    return np.zeros(max(1, int(config.det_capacity)), dtype=_abi.det_record_dtype(m.nmedia))


def run_group_dynamic(first_index: int, quota: int, threads: int, scene: Scene,
                      config: SimulationConfig, device: int = 0, cells_out: Optional[np.ndarray] = None,
                      det_out: Optional[np.ndarray] = None) -> GroupRunResult:
    """Photons [first_index, first_index+quota) on one B200 (scheduler.cpp:321-324).

    `threads` is validated as in the reference (>= 1); the device runs its
    own persistent worker grid, so the whole quota is reported in slot 0 of
    per_thread_photons (Σ == quota, size == threads). `cells_out` / `det_out`
    may be preallocated (e.g. pinned) host buffers that are overwritten."""
    if threads < 1:
        raise ValidationError("run_group: threads must be >= 1")
    config.validate()
    m = Marshalled(scene, config)
    nx, ny, nz = scene.grid.dims
    shape = (config.ngates, nz, ny, nx)
    if cells_out is not None:
        if cells_out.dtype != np.int64 or cells_out.size != m.ncells or not cells_out.flags.c_contiguous:
            raise ValidationError("cells_out must be a contiguous int64 array of ngates*nx*ny*nz cells")
        cells = cells_out.reshape(shape)
    else:
        cells = np.zeros(shape, np.int64)
    tot = _abi.vmc_disposition()
    det = _det_buffer(m, config) if det_out is None else det_out
    ndet = C.c_uint64(0)
    wall = C.c_double(0.0)
    _check(lib().vmc_run_range(C.byref(m.scene), C.byref(m.config), first_index, quota, device,
                               cells.ctypes.data, C.byref(tot),
                               det.ctypes.data if det is not None else None, C.byref(ndet),
                               C.byref(wall)))
    fmap = FluenceMap(scene.grid.dims, config.photon_count, config.ngates, cells)
    q = (tot.deposited_q, tot.escaped_q, tot.killed_q, tot.truncated_q)
    per = [0] * threads
    per[0] = quota
    res = GroupRunResult(fmap, PhotonDisposition.from_quanta(q, tot.quantum), per, wall.value, q)
    if det is not None:
        res.det_count = ndet.value
        res.detections = det[:min(ndet.value, len(det))]
    return res


run_static_split = run_group_dynamic


def simulate_photon_trace(photon_index: int, scene: Scene, config: SimulationConfig, device: int = 0,
                          max_deposits: int = 1 << 20):
    """One photon's walk on the device in the reference's arithmetic (FP64
    flight kernel; reference simulate_photon_trace, transport.cpp:368-380):
    returns (PhotonDisposition, [(cell, dw), ...]) with one entry per step that
    deposits, in walk order."""
    m = Marshalled(scene, config)
    cells = np.zeros(max_deposits, np.int64)
    dws = np.zeros(max_deposits, np.float64)
    n = C.c_uint64()
    disp = (C.c_double * 4)()
    _check(lib().vmc_simulate_photon(C.byref(m.scene), C.byref(m.config), photon_index, device, max_deposits,
                                     cells.ctypes.data, dws.ctypes.data, C.byref(n), disp))
    k = min(n.value, max_deposits)
    return PhotonDisposition(*disp), list(zip(cells[:k].tolist(), dws[:k].tolist()))


def simulate_photon(photon_index: int, scene: Scene, config: SimulationConfig,
                    device: int = 0):
    """Reference simulate_photon (transport.cpp:362-366): the photon's walk on
    the device (FP64 flight kernel) with every step deposit added to a
    FluenceMap in the quantum of config.photon_count exactly as
    FluenceMap::deposit does (llround(dw / quantum), fluence.hpp:39-54).
    Returns (disposition, map)."""
    disp, deps = simulate_photon_trace(photon_index, scene, config, device)
    fmap = FluenceMap(scene.grid.dims, config.photon_count)
    flat = fmap.cells.reshape(-1)
    inv = 1.0 / fmap.quantum
    for cell, dw in deps:
        x = dw * inv
        flat[cell] += int(math.copysign(math.floor(abs(x) + 0.5), x))  # llround
    return disp, fmap


# ---------------------------------------------------------------------------
class DeviceKind(enum.Enum):
    RealWorkerPool = "pool"
    Simulated = "simulated"
    CudaGpu = "gpu"


@dataclass
class DeviceProfile:
    """scheduler.hpp:21-28 plus the B200 build's DeviceKind.CudaGpu."""
    name: str = "gpu"
    cores: int = 1
    a: float = 0.0
    t0: float = 0.0
    kind: DeviceKind = DeviceKind.CudaGpu
    jitter_sigma: float = 0.0
    gpu: int = 0  # CUDA ordinal for CudaGpu devices


class Strategy(enum.IntEnum):
    S1 = _abi.VMC_STRATEGY_S1
    S2 = _abi.VMC_STRATEGY_S2
    S3 = _abi.VMC_STRATEGY_S3


def strategy_from_name(name: str) -> Optional[Strategy]:
    return {"s1": Strategy.S1, "S1": Strategy.S1, "s2": Strategy.S2, "S2": Strategy.S2,
            "s3": Strategy.S3, "S3": Strategy.S3}.get(name)


@dataclass
class Partition:
    counts: List[int]

    def total(self) -> int:
        return sum(self.counts)


def _profiles(devices: Sequence[DeviceProfile]):
    arr = (_abi.vmc_device_profile * len(devices))()
    for i, d in enumerate(devices):
        arr[i].cores, arr[i].a, arr[i].t0 = int(d.cores), float(d.a), float(d.t0)
    return arr


def make_partition(total: int, devices: Sequence[DeviceProfile], strategy: Strategy) -> Partition:
    if not devices:
        raise ValidationError("partition: no devices")
    out = (C.c_uint64 * len(devices))()
    _check(lib().vmc_partition(int(strategy), total, len(devices), _profiles(devices), out))
    return Partition(list(out))


def partition_s1(total, devices):
    return make_partition(total, devices, Strategy.S1)


def partition_s2(total, devices):
    return make_partition(total, devices, Strategy.S2)


def partition_s3(total, devices):
    return make_partition(total, devices, Strategy.S3)


def model_makespan(p: Partition, devices: Sequence[DeviceProfile]) -> float:
    n = len(p.counts)
    counts = (C.c_uint64 * n)(*p.counts)
    return lib().vmc_model_makespan(n, counts, _profiles(devices))


def thread_count_heuristic(cores: int, max_concurrent_per_core: int) -> int:  # scheduler.cpp:38-43
    if cores < 1 or max_concurrent_per_core < 1:
        raise ValidationError("thread_count_heuristic: arguments must be >= 1")
    return cores * max_concurrent_per_core


@dataclass
class DeviceRunResult:
    name: str
    photons: int
    wall_ms: float = 0.0


@dataclass
class MultiDeviceResult:
    map: FluenceMap
    totals: PhotonDisposition
    partition: Partition
    devices: List[DeviceRunResult]
    makespan_ms: float = 0.0
    reduce_ms: float = 0.0
    totals_q: tuple = (0, 0, 0, 0)
    detections: Optional[np.ndarray] = None
    det_count: int = 0


def run_multi_device(total: int, devices: Sequence[DeviceProfile], strategy: Strategy, scene: Scene,
                     config: SimulationConfig, threads_per_device: int = 0) -> MultiDeviceResult:
    """scheduler.cpp:395-451 on B200s: contiguous global ranges in device
    order, shared quantum from `total`, one host thread per GPU, NCCL reduce of
    the int64 maps. CudaGpu devices run on their own GPU; the reference's host
    pools and simulated devices run their ranges on GPU 0, a simulated device
    keeping the reference's modelled wall time a*n + t0 (scheduler.cpp:441-443)."""
    if not devices:
        raise ValidationError("run_multi_device: no devices")
    part = make_partition(total, devices, strategy)
    cfg = SimulationConfig(**{**config.__dict__})
    cfg.photon_count = total  # scheduler.cpp:412-413
    cfg.validate()
    m = Marshalled(scene, cfg)
    nx, ny, nz = scene.grid.dims
    cells = np.zeros((cfg.ngates, nz, ny, nx), np.int64)
    tot = _abi.vmc_disposition()
    det = _det_buffer(m, cfg)
    ndet = C.c_uint64(0)
    nd = len(devices)
    per_ms = (C.c_double * nd)()
    red_ms = C.c_double(0.0)
    gpus = (C.c_int * nd)(*[d.gpu if d.kind == DeviceKind.CudaGpu else 0 for d in devices])
    counts = (C.c_uint64 * nd)(*part.counts)
    _check(lib().vmc_run_multi(C.byref(m.scene), C.byref(m.config), nd, gpus, counts, cells.ctypes.data,
                               C.byref(tot), det.ctypes.data if det is not None else None,
                               C.byref(ndet), per_ms, C.byref(red_ms)))
    q = (tot.deposited_q, tot.escaped_q, tot.killed_q, tot.truncated_q)
    runs = [DeviceRunResult(d.name, part.counts[i],
                            (d.a * part.counts[i] + d.t0 if d.kind == DeviceKind.Simulated else per_ms[i])
                            if part.counts[i] else 0.0)
            for i, d in enumerate(devices)]
    res = MultiDeviceResult(FluenceMap(scene.grid.dims, total, cfg.ngates, cells),
                            PhotonDisposition.from_quanta(q, tot.quantum), part, runs,
                            max([r.wall_ms for r in runs] + [0.0]) + red_ms.value, red_ms.value, q)
    if det is not None:
        res.det_count = ndet.value
        res.detections = det[:min(ndet.value, len(det))]
    return res


@dataclass
class Calibration:
    a: float = 0.0
    t0: float = 0.0


def calibrate(device: DeviceProfile, n1: int, n2: int, scene: Scene, config: SimulationConfig,
              threads: int = 1, noise_seed: int = 0) -> Calibration:
    """Two-pilot runtime model (scheduler.cpp:360-393): a = (T2-T1)/(n2-n1),
    t0 = max(0, T1 - a n1). CudaGpu devices run both pilots on the GPU with the
    quantum of n2; Simulated devices answer from their model (+ lognormal
    jitter from the reference's own xorshift stream)."""
    if not (n2 > n1 >= 1):
        raise ValidationError("calibrate: need n2 > n1 >= 1")
    if device.kind == DeviceKind.Simulated:
        t1 = device.a * n1 + device.t0
        t2 = device.a * n2 + device.t0
        if device.jitter_sigma > 0.0:
            from .rngs import HostStream
            s = HostStream(noise_seed, 0x706C6F74)

            def lognormal():
                u1 = max(s.next_unit(), 1e-300)
                u2 = s.next_unit()
                z = math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * 3.14159265358979323846 * u2)
                return math.exp(device.jitter_sigma * z)
            t1 *= lognormal()
            t2 *= lognormal()
    else:
        pilot = SimulationConfig(**{**config.__dict__})
        pilot.photon_count = n2
        t1 = run_group_dynamic(0, n1, max(1, threads), scene, pilot, device.gpu).wall_ms
        t2 = run_group_dynamic(0, n2, max(1, threads), scene, pilot, device.gpu).wall_ms
    if t2 <= t1:
        raise NonPositiveSlope("calibrate: T2 <= T1; increase n2 or rerun")
    a = (t2 - t1) / (n2 - n1)
    return Calibration(a, max(0.0, t1 - a * n1))


# ---------------------------------------------------------------------------
def rng_kat(seed: int, stream_id: int, n: int, device: int = 0) -> List[int]:
    """First n next_u64() of RngStream(seed, stream_id), computed on the GPU."""
    out = (C.c_uint64 * n)()
    _check(lib().vmc_rng_kat(seed, stream_id, n, device, out))
    return list(out)


class Plan:
    """Device-resident scene (vmc_plan): upload once, run many ranges into
    caller-owned device buffers (torch tensors or raw pointers)."""

    def __init__(self, scene: Scene, config: SimulationConfig, device: int = 0):
        config.validate()
        self._m = Marshalled(scene, config)
        self.config = config
        self.scene = scene
        self.device = device
        h = C.c_void_p()
        _check(lib().vmc_plan_create(C.byref(self._m.scene), C.byref(self._m.config), device, C.byref(h)))
        self._h = h
        self.ncells = int(lib().vmc_plan_cell_count(h))
        self.nmedia = self._m.nmedia
        self.rec_bytes = _abi.det_record_bytes(self.nmedia)

    def run(self, first: int, count: int, d_cells: int, d_totals: int, d_det: int = 0,
            d_det_count: int = 0, stream: int = 0, zero: bool = True) -> None:
        _check(lib().vmc_plan_run(self._h, first, count, C.c_void_p(d_cells), C.c_void_p(d_totals),
                                  C.c_void_p(d_det or None), C.c_void_p(d_det_count or None),
                                  C.c_void_p(stream or None), _abi.VMC_RUN_ZERO if zero else 0))

    def run_torch(self, first: int, count: int, cells, totals, det=None, det_count=None,
                  stream=None, zero: bool = True) -> None:
        """Enqueue on a torch stream with torch int64 tensors as outputs."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.run(first, count, cells.data_ptr(), totals.data_ptr(),
                 det.data_ptr() if det is not None else 0,
                 det_count.data_ptr() if det_count is not None else 0, st.cuda_stream, zero)

    def sort_records_torch(self, det, n: int, first: int, count: int, out, stream=None) -> None:
        """Sort the first n detector records in `det` (written by run_torch for
        photons [first, first+count)) by photon index into `out` (uint8 tensors)."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(lib().vmc_plan_sort_records(self._h, C.c_void_p(det.data_ptr()), n, first, count,
                                           C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)))

    def trace(self, first: int, count: int) -> np.ndarray:
        out = np.zeros(count, dtype=_abi.trace_dtype())
        _check(lib().vmc_plan_trace(self._h, first, count, out.ctypes.data))
        return out

    def normalize_torch(self, cells, out, photon_count: int, sum_gates: bool = True,
                        normalized: bool = True, stream=None) -> None:
        """K4 on the device: float32 fluence (or raw weight) from int64 cells."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(lib().vmc_plan_normalize(self._h, C.c_void_p(cells.data_ptr()), photon_count,
                                        C.c_void_p(out.data_ptr()), 1 if sum_gates else 0,
                                        1 if normalized else 0, C.c_void_p(st.cuda_stream)))

    def launches_per_run(self) -> int:
        return int(lib().vmc_plan_launches_per_run(self._h, 0))

    @property
    def kernel_name(self) -> str:
        """Mangled symbol of the transport kernel variant this plan launches."""
        return (lib().vmc_plan_kernel_name(self._h) or b"").decode()

    @property
    def kernel(self) -> str:
        """Readable variant key: 'k_flight<float,G,D,T,U,Dep>' (or k_transport<...>)."""
        return demangle_kernel(self.kernel_name)

    def close(self) -> None:
        if self._h:
            lib().vmc_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def demangle_kernel(mangled: str) -> str:
    """_ZN3vmc8k_flightIfLb1ELb0ELb0ELb0ELi0ELb0EEEvNS_10KernelArgsE -> k_flight<float,1,0,0,0,0>
    (the two kernel templates' Itanium manglings, decoded without c++filt; the
    small-run instantiation of K1f shows its trailing kSolo = 1)."""
    import re
    m = re.match(r"_ZN3vmc(\d+)(k_flight|k_transport)I([fd])((?:L[bi]n?\d+E)+)E", mangled or "")
    if not m:
        return mangled or ""
    args = ["float" if m.group(3) == "f" else "double"]
    for kind, neg, val in re.findall(r"L([bi])(n?)(\d+)E", m.group(4)):
        args.append(("-" if neg else "") + val)
    if m.group(2) == "k_flight" and len(args) == 7 and args[-1] == "0":
        args.pop()  # k_flight<..., kSolo = false>: the large-run kernel keeps its short name
    return f"{m.group(2)}<{','.join(args)}>"


def trace_photons(scene: Scene, config: SimulationConfig, first: int, count: int,
                  device: int = 0) -> np.ndarray:
    p = Plan(scene, config, device)
    try:
        return p.trace(first, count)
    finally:
        p.close()
