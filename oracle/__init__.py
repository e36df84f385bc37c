"""oracle — TEST INFRASTRUCTURE ONLY.

CPU checkers for the B200 photon-transport path. Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference)
may import this package; the product library never does.

  RefLib   : the unmodified reference core (oracle/_ref/libvoxmc_ref.so, built
             by oracle/Makefile from /root/reference/proj/core/src) behind
             ref_capi.cpp.
  COracle  : the plain-C double-precision restatement (oracle/liboracle_c.so).

Both take the same vmc_scene / vmc_config structs as the product C-ABI.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

from paper_1711_03244_b200 import _abi
from paper_1711_03244_b200.scene import Marshalled, Scene, SimulationConfig

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libvoxmc_ref.so")
C_SO = os.path.join(HERE, "liboracle_c.so")


def build(quiet: bool = True) -> None:
    """make -C oracle (reference .so only when /root/reference is present)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def fnv1a64(data: bytes) -> int:
    """FNV-1a 64 (the reference's volume checksum, volume_io.cpp:13-20)."""
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv1a64_np(buf: np.ndarray) -> int:
    """Vectorised-per-step FNV-1a over a byte buffer (same result as fnv1a64)."""
    b = np.frombuffer(np.ascontiguousarray(buf).tobytes(), dtype=np.uint8)
    h = 0xCBF29CE484222325
    p = 0x100000001B3
    # plain loop over bytes in chunks; python ints keep it exact
    for x in b.tolist():
        h = ((h ^ x) * p) & 0xFFFFFFFFFFFFFFFF
    return h


def volume_checksum(cells: np.ndarray, quantum: float) -> str:
    """FNV-1a of FluenceMap::to_float_volume() of raw cells (fluence.cpp:86-90)."""
    vol = (cells.astype(np.float64) * quantum).astype(np.float32)
    return f"{fnv1a64_np(vol):016x}"


class _Base:
    def _check(self, rc: int, err) -> None:
        if rc != 0:
            from paper_1711_03244_b200.errors import ValidationError
            msg = err().decode() if err() else "oracle error"
            raise (ValidationError if rc == 1 else RuntimeError)(msg)


class RefLib(_Base):
    """The compiled reference (voxmc_ref::) behind oracle/ref_capi.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = C.CDLL(path)
        P, vp, u64, i64 = C.POINTER, C.c_void_p, C.c_uint64, C.c_int64
        S, Cf = P(_abi.vmc_scene), P(_abi.vmc_config)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_mix64.restype = u64
        lib.ref_mix64.argtypes = [u64]
        lib.ref_rng_kat.argtypes = [u64, u64, C.c_int, P(u64), P(u64), P(C.c_double)]
        lib.ref_quantum_for.restype = C.c_double
        lib.ref_quantum_for.argtypes = [u64]
        lib.ref_run_group.argtypes = [S, Cf, u64, u64, C.c_int, vp, P(C.c_double), P(C.c_double)]
        lib.ref_run_multi.argtypes = [S, Cf, u64, C.c_int, P(_abi.vmc_device_profile), C.c_int,
                                      C.c_int, vp, P(C.c_double), P(u64)]
        lib.ref_trace.argtypes = [S, Cf, u64, C.c_int, P(i64), P(C.c_double), P(C.c_int),
                                  P(C.c_double)]
        lib.ref_walk.argtypes = [S, Cf, u64, u64, C.c_int, vp, vp, vp, vp, P(u64), P(C.c_double)]
        lib.ref_partition.argtypes = [C.c_int, u64, C.c_int, P(_abi.vmc_device_profile), P(u64),
                                      P(C.c_double)]
        lib.ref_brute_force.argtypes = [u64, C.c_int, P(_abi.vmc_device_profile), P(u64),
                                        P(C.c_double)]
        lib.ref_hg_cos_theta.restype = C.c_double
        lib.ref_hg_cos_theta.argtypes = [C.c_double, C.c_double]
        lib.ref_fresnel.restype = C.c_double
        lib.ref_fresnel.argtypes = [C.c_double, C.c_double, C.c_double]
        lib.ref_distance_to_boundary.argtypes = [S, P(C.c_double), P(C.c_double), P(C.c_double)]
        self.has_pipeline = hasattr(lib, "ref_run_pipeline")
        if self.has_pipeline:
            lib.ref_run_pipeline.argtypes = [S, Cf, C.c_int, P(C.c_double), P(C.c_double), P(C.c_double)]
            lib.ref_normalize.argtypes = [S, u64, vp, C.c_int, vp]
        self.lib = lib
        self.path = path
        self.build = os.path.basename(path)

    def _ck(self, rc):
        self._check(rc, self.lib.ref_last_error)

    def rng_kat(self, seed: int, sid: int, n: int):
        out = (C.c_uint64 * n)()
        st = (C.c_uint64 * 2)()
        u = C.c_double()
        self._ck(self.lib.ref_rng_kat(seed, sid, n, out, st, C.byref(u)))
        return list(out), (st[0], st[1]), u.value

    def quantum_for(self, n: int) -> float:
        return self.lib.ref_quantum_for(n)

    def run_group(self, scene: Scene, config: SimulationConfig, first: int, count: int,
                  threads: int, want_cells: bool = True):
        m = Marshalled(scene, config)
        cells = np.zeros(scene.grid.voxel_count, dtype=np.int64) if want_cells else None
        disp = (C.c_double * 4)()
        wall = C.c_double()
        self._ck(self.lib.ref_run_group(C.byref(m.scene), C.byref(m.config), first, count, threads,
                                        cells.ctypes.data if cells is not None else None, disp,
                                        C.byref(wall)))
        return cells, list(disp), wall.value

    def run_pipeline(self, scene: Scene, config: SimulationConfig, threads: int = 0):
        """voxmc::run_pipeline over photons [0, config.photon_count) with the
        default roster host_device(threads) (0 = all hardware threads).
        Returns (makespan_ms, e2e_ms, total deposited weight)."""
        m = Marshalled(scene, config)
        mk, e2e = C.c_double(), C.c_double()
        disp = (C.c_double * 4)()
        self._ck(self.lib.ref_run_pipeline(C.byref(m.scene), C.byref(m.config), threads, C.byref(mk),
                                           C.byref(e2e), disp))
        return mk.value, e2e.value, disp[0]

    def time_pipeline(self, scene, config, n: int, threads: int) -> float:
        """ms of run_pipeline over n photons (RunReport::makespan_ms, config.cpp:305)."""
        import copy
        cfg = copy.copy(config)
        cfg.photon_count = n
        return self.run_pipeline(scene, cfg, threads)[0]

    def time_group(self, scene, config, n: int, threads: int) -> float:
        return self.run_group(scene, config, 0, n, threads, want_cells=False)[2]

    def normalize(self, scene: Scene, photon_count: int, cells: np.ndarray, normalized: bool = True):
        """FluenceMap::normalize + to_float_volume of raw cells (fluence.cpp:62-90)."""
        c = np.ascontiguousarray(cells, dtype=np.int64).reshape(-1)
        out = np.empty(scene.grid.voxel_count, np.float32)
        m = Marshalled(scene, SimulationConfig(photon_count=photon_count))
        self._ck(self.lib.ref_normalize(C.byref(m.scene), photon_count, c.ctypes.data, 1 if normalized else 0,
                                        out.ctypes.data))
        return out

    def run_multi(self, scene, config, total, profiles, strategy, threads_per_device=1):
        m = Marshalled(scene, config)
        nd = len(profiles)
        prof = (_abi.vmc_device_profile * nd)()
        for i, (cores, a, t0) in enumerate(profiles):
            prof[i].cores, prof[i].a, prof[i].t0 = cores, a, t0
        cells = np.zeros(scene.grid.voxel_count, dtype=np.int64)
        disp = (C.c_double * 4)()
        counts = (C.c_uint64 * nd)()
        self._ck(self.lib.ref_run_multi(C.byref(m.scene), C.byref(m.config), total, nd, prof,
                                        strategy, threads_per_device, cells.ctypes.data, disp,
                                        counts))
        return cells, list(disp), list(counts)

    def trace(self, scene, config, idx: int, max_deps: int = 1 << 16):
        m = Marshalled(scene, config)
        cells = (C.c_int64 * max_deps)()
        w = (C.c_double * max_deps)()
        n = C.c_int()
        disp = (C.c_double * 4)()
        self._ck(self.lib.ref_trace(C.byref(m.scene), C.byref(m.config), idx, max_deps, cells, w,
                                    C.byref(n), disp))
        k = min(n.value, max_deps)
        return list(zip(cells[:k], w[:k])), list(disp)

    def walk(self, scene, config, first, count, threads=1, cells=True, counts=False,
             traces=False, detectors=False):
        m = Marshalled(scene, config)
        out = {}
        c_arr = np.zeros(m.ncells, dtype=np.int64) if cells else None
        n_arr = np.zeros(scene.grid.voxel_count, dtype=np.int64) if counts else None
        t_arr = np.zeros(count, dtype=_abi.trace_dtype()) if traces else None
        det_arr = None
        dcount = C.c_uint64(0)
        if detectors and config.detectors:
            det_arr = np.zeros(max(1, config.det_capacity), dtype=_abi.det_record_dtype(m.nmedia))
        disp = (C.c_double * 4)()
        self._ck(self.lib.ref_walk(
            C.byref(m.scene), C.byref(m.config), first, count, threads,
            c_arr.ctypes.data if c_arr is not None else None,
            n_arr.ctypes.data if n_arr is not None else None,
            t_arr.ctypes.data if t_arr is not None else None,
            det_arr.ctypes.data if det_arr is not None else None,
            C.byref(dcount), disp))
        out["cells"], out["counts"], out["traces"] = c_arr, n_arr, t_arr
        out["disp"] = list(disp)
        if det_arr is not None:
            out["det"] = det_arr[:min(dcount.value, len(det_arr))]
            out["det_count"] = dcount.value
        return out

    def partition(self, strategy: int, total: int, profiles):
        nd = len(profiles)
        prof = (_abi.vmc_device_profile * nd)()
        for i, (cores, a, t0) in enumerate(profiles):
            prof[i].cores, prof[i].a, prof[i].t0 = cores, a, t0
        counts = (C.c_uint64 * nd)()
        ms = C.c_double()
        self._ck(self.lib.ref_partition(strategy, total, nd, prof, counts, C.byref(ms)))
        return list(counts), ms.value

    def brute_force(self, total: int, profiles):
        nd = len(profiles)
        prof = (_abi.vmc_device_profile * nd)()
        for i, (cores, a, t0) in enumerate(profiles):
            prof[i].cores, prof[i].a, prof[i].t0 = cores, a, t0
        counts = (C.c_uint64 * nd)()
        ms = C.c_double()
        self._ck(self.lib.ref_brute_force(total, nd, prof, counts, C.byref(ms)))
        return list(counts), ms.value


class COracle(_Base):
    """Plain-C double-precision restatement (oracle/voxmc_oracle.c)."""

    def __init__(self, path: str = C_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = C.CDLL(path)
        P, vp, u64 = C.POINTER, C.c_void_p, C.c_uint64
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_mix64.restype = u64
        lib.orc_mix64.argtypes = [u64]
        lib.orc_rng_kat.argtypes = [u64, u64, C.c_int, P(u64)]
        lib.orc_quantum_for.restype = C.c_double
        lib.orc_quantum_for.argtypes = [u64]
        lib.orc_hg_cos_theta.restype = C.c_double
        lib.orc_hg_cos_theta.argtypes = [C.c_double, C.c_double]
        lib.orc_fresnel.restype = C.c_double
        lib.orc_fresnel.argtypes = [C.c_double, C.c_double, C.c_double]
        lib.orc_walk.argtypes = [P(_abi.vmc_scene), P(_abi.vmc_config), u64, u64, C.c_int, vp, vp,
                                 P(C.c_double), vp, P(u64)]
        lib.orc_walk_flight.argtypes = [P(_abi.vmc_scene), P(_abi.vmc_config), u64, u64, C.c_int, vp,
                                        P(C.c_double)]
        self.lib = lib

    def rng_kat(self, seed: int, sid: int, n: int):
        out = (C.c_uint64 * n)()
        self.lib.orc_rng_kat(seed, sid, n, out)
        return list(out)

    def quantum_for(self, n: int) -> float:
        return self.lib.orc_quantum_for(n)

    def walk(self, scene, config, first, count, threads=1, cells=True, traces=False,
             detectors=False):
        m = Marshalled(scene, config)
        c_arr = np.zeros(m.ncells, dtype=np.int64) if cells else None
        t_arr = np.zeros(count, dtype=_abi.trace_dtype()) if traces else None
        det_arr = None
        dcount = C.c_uint64(0)
        if detectors and config.detectors:
            det_arr = np.zeros(max(1, config.det_capacity), dtype=_abi.det_record_dtype(m.nmedia))
        disp = (C.c_double * 4)()
        rc = self.lib.orc_walk(C.byref(m.scene), C.byref(m.config), first, count, threads,
                               c_arr.ctypes.data if c_arr is not None else None,
                               t_arr.ctypes.data if t_arr is not None else None, disp,
                               det_arr.ctypes.data if det_arr is not None else None,
                               C.byref(dcount))
        self._check(rc, self.lib.orc_last_error)
        out = {"cells": c_arr, "traces": t_arr, "disp": list(disp)}
        if det_arr is not None:
            out["det"] = det_arr[:min(dcount.value, len(det_arr))]
            out["det_count"] = dcount.value
        return out


    def walk_flight(self, scene, config, first, count, threads=1):
        """K1f's flight decomposition in double precision (traces, dispositions)."""
        m = Marshalled(scene, config)
        t_arr = np.zeros(count, dtype=_abi.trace_dtype())
        disp = (C.c_double * 4)()
        rc = self.lib.orc_walk_flight(C.byref(m.scene), C.byref(m.config), first, count, threads,
                                      t_arr.ctypes.data, disp)
        self._check(rc, self.lib.orc_last_error)
        return {"traces": t_arr, "disp": list(disp)}


_ref_singleton: Optional[RefLib] = None
_c_singleton: Optional[COracle] = None


BENCH_ISAS = ["sapphirerapids", "emeraldrapids", "icelake-server", "znver4", "znver3", "x86-64-v4"]


def host_march() -> str:
    """What `gcc -march=native` resolves to on this host ("" if unknown)."""
    try:
        out = subprocess.run(["gcc", "-march=native", "-Q", "--help=target"], capture_output=True, text=True,
                             timeout=30).stdout
        for line in out.splitlines():
            t = line.split()
            if len(t) == 2 and t[0] == "-march=":
                return t[1]
    except Exception:
        pass
    return ""


def _cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except Exception:
        pass
    return set()


_best_singleton: Optional[RefLib] = None


def ref_best() -> RefLib:
    """The reference build for the CPU baseline: the per-ISA build matching
    this host's -march=native (the reference's own flag,
    proj/core/CMakeLists.txt:18), else x86-64-v4 when the host has AVX-512,
    else the portable x86-64-v3 test build."""
    global _best_singleton
    if _best_singleton is None:
        march = host_march()
        cand = []
        if march in BENCH_ISAS:
            cand.append(march)
        if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= _cpu_flags():
            cand.append("x86-64-v4")
        lib = None
        for isa in cand:
            p = os.path.join(HERE, "_ref", f"libvoxmc_ref_bench_{isa}.so")
            if os.path.exists(p):
                lib = RefLib(p)
                lib.build = f"reference core -O3 -march={isa}" + (
                    " (== this host's -march=native)" if isa == march else
                    f" (host -march=native is {march or 'unknown'}; widest prebuilt ISA it supports)")
                break
        if lib is None:
            lib = ref()
            lib.build = "reference core -O3 -march=x86-64-v3 (portable test build)"
        _best_singleton = lib
    return _best_singleton


def ref() -> RefLib:
    global _ref_singleton
    if _ref_singleton is None:
        _ref_singleton = RefLib()
    return _ref_singleton


def corc() -> COracle:
    global _c_singleton
    if _c_singleton is None:
        _c_singleton = COracle()
    return _c_singleton
