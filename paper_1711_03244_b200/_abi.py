"""ctypes mirror of include/vmc.h (the C-ABI boundary).

Only plain C types cross this boundary. The structs here must stay
byte-identical to include/vmc.h; tests/test_abi.py checks sizes and offsets
against the header compiled with gcc.
"""
from __future__ import annotations

import ctypes as C

VMC_ABI_VERSION = 1
VMC_OK, VMC_ERR_VALIDATION, VMC_ERR_RUNTIME = 0, 1, 2
VMC_BOUNDARY_TERMINATE, VMC_BOUNDARY_REFLECT = 0, 1
VMC_ACCUM_SHARED_ATOMIC, VMC_ACCUM_PRIVATE_MERGE = 0, 1
VMC_PRECISION_FP32, VMC_PRECISION_FP64 = 0, 1
VMC_STRATEGY_S1, VMC_STRATEGY_S2, VMC_STRATEGY_S3 = 1, 2, 3
VMC_RUN_ZERO = 1


class vmc_scene(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
        ("voxel_mm", C.c_double),
        ("labels", C.POINTER(C.c_uint8)),
        ("nmedia", C.c_int32),
        ("media", C.POINTER(C.c_double)),
        ("src_pos", C.c_double * 3),
        ("src_dir", C.c_double * 3),
        ("isotropic", C.c_int32),
    ]


class vmc_config(C.Structure):
    _fields_ = [
        ("photon_count", C.c_uint64),
        ("master_seed", C.c_uint64),
        ("accumulation_mode", C.c_int32),
        ("boundary_mode", C.c_int32),
        ("tmax_ns", C.c_double),
        ("roulette_threshold", C.c_double),
        ("roulette_multiplier", C.c_int32),
        ("workgroup_size", C.c_int32),
        ("ngates", C.c_int32),
        ("precision", C.c_int32),
        ("ndet", C.c_int32),
        ("reserved0", C.c_int32),
        ("det", C.POINTER(C.c_double)),
        ("det_capacity", C.c_uint64),
    ]


class vmc_disposition(C.Structure):
    _fields_ = [
        ("deposited_q", C.c_int64), ("escaped_q", C.c_int64),
        ("killed_q", C.c_int64), ("truncated_q", C.c_int64),
        ("quantum", C.c_double),
    ]


class vmc_device_profile(C.Structure):
    _fields_ = [("cores", C.c_int32), ("reserved0", C.c_int32),
                ("a", C.c_double), ("t0", C.c_double)]


class vmc_photon_trace(C.Structure):
    _fields_ = [
        ("draws", C.c_uint32), ("steps", C.c_uint32), ("scatters", C.c_uint32),
        ("flags", C.c_uint32),
        ("deposited", C.c_double), ("escaped", C.c_double),
        ("killed", C.c_double), ("truncated", C.c_double),
    ]


class vmc_det_record_head(C.Structure):
    _fields_ = [("photon_index", C.c_uint64), ("det_id", C.c_uint32), ("nscat", C.c_uint32),
                ("w_exit", C.c_float), ("t_exit_ns", C.c_float)]


def det_record_bytes(nmedia: int) -> int:
    raw = C.sizeof(vmc_det_record_head) + 4 * max(0, nmedia - 1)
    return (raw + 7) & ~7


def det_record_dtype(nmedia: int):
    """numpy structured dtype of one detector record (vmc.h)."""
    import numpy as np
    fields = [("photon_index", "<u8"), ("det_id", "<u4"), ("nscat", "<u4"),
              ("w_exit", "<f4"), ("t_exit_ns", "<f4")]
    if nmedia > 1:
        fields.append(("ppath_mm", "<f4", (nmedia - 1,)))
    return np.dtype({"names": [f[0] for f in fields],
                     "formats": [f[1] if len(f) == 2 else (f[1], f[2]) for f in fields],
                     "itemsize": det_record_bytes(nmedia)})


TRACE_DTYPE = None


def trace_dtype():
    import numpy as np
    return np.dtype([("draws", "<u4"), ("steps", "<u4"), ("scatters", "<u4"), ("flags", "<u4"),
                     ("deposited", "<f8"), ("escaped", "<f8"), ("killed", "<f8"),
                     ("truncated", "<f8")])


# Exported symbols of libvoxmc_b200.so, in include/vmc.h order.
EXPORTS = (
    "vmc_det_record_bytes", "vmc_abi_version", "vmc_last_error", "vmc_device_count",
    "vmc_quantum_for", "vmc_validate", "vmc_run_range", "vmc_run_multi", "vmc_partition",
    "vmc_model_makespan", "vmc_rng_kat", "vmc_plan_create", "vmc_plan_destroy",
    "vmc_plan_cell_count", "vmc_plan_run", "vmc_plan_trace", "vmc_plan_normalize", "vmc_fnv1a64",
    "vmc_plan_launches_per_run",
    "vmc_plan_kernel_name",
    "vmc_plan_sort_records",
    "vmc_simulate_photon",
)


def declare(lib: C.CDLL) -> C.CDLL:
    """Attach argtypes/restypes of every vmc.h entry point to `lib`."""
    P = C.POINTER
    vp = C.c_void_p
    u64, i64, i32, u32 = C.c_uint64, C.c_int64, C.c_int32, C.c_uint32
    sig = {
        "vmc_det_record_bytes": (C.c_size_t, [i32]),
        "vmc_abi_version": (C.c_int, []),
        "vmc_last_error": (C.c_char_p, []),
        "vmc_device_count": (C.c_int, []),
        "vmc_quantum_for": (C.c_double, [u64]),
        "vmc_validate": (C.c_int, [P(vmc_scene), P(vmc_config)]),
        "vmc_run_range": (C.c_int, [P(vmc_scene), P(vmc_config), u64, u64, C.c_int, vp,
                                    P(vmc_disposition), vp, P(u64), P(C.c_double)]),
        "vmc_run_multi": (C.c_int, [P(vmc_scene), P(vmc_config), C.c_int, P(C.c_int), P(u64),
                                    vp, P(vmc_disposition), vp, P(u64), P(C.c_double),
                                    P(C.c_double)]),
        "vmc_partition": (C.c_int, [C.c_int, u64, C.c_int, P(vmc_device_profile), P(u64)]),
        "vmc_model_makespan": (C.c_double, [C.c_int, P(u64), P(vmc_device_profile)]),
        "vmc_rng_kat": (C.c_int, [u64, u64, C.c_int, C.c_int, P(u64)]),
        "vmc_plan_create": (C.c_int, [P(vmc_scene), P(vmc_config), C.c_int, P(vp)]),
        "vmc_plan_destroy": (C.c_int, [vp]),
        "vmc_plan_cell_count": (u64, [vp]),
        "vmc_plan_run": (C.c_int, [vp, u64, u64, vp, vp, vp, vp, vp, u32]),
        "vmc_plan_trace": (C.c_int, [vp, u64, u64, vp]),
        "vmc_plan_launches_per_run": (C.c_int, [vp, u32]),
        "vmc_plan_kernel_name": (C.c_char_p, [vp]),
        "vmc_plan_sort_records": (C.c_int, [vp, vp, u64, u64, u64, vp, vp]),
        "vmc_simulate_photon": (C.c_int, [P(vmc_scene), P(vmc_config), u64, C.c_int, u64, vp, vp, vp, vp]),
        "vmc_plan_normalize": (C.c_int, [vp, vp, u64, vp, C.c_int, C.c_int, vp]),
        "vmc_fnv1a64": (u64, [vp, C.c_size_t]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
