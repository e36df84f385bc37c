"""paper_1711_03244_b200 — B200-native voxel Monte Carlo photon transport.

The hot path (launch / DDA step / Beer-Lambert deposit / Henyey-Greenstein
scatter / Fresnel boundary / roulette, fused with fixed-point fluence
accumulation) runs as one persistent sm_100a kernel in lib/libvoxmc_b200.so,
behind the C-ABI declared in include/vmc.h. This package mirrors the
reference's (voxmc) host API on top of it.
"""
from .errors import (AlreadyNormalized, DimensionMismatch, InstanceTooLarge, IoError,  # noqa: F401
                     NonPositiveRadius, NonPositiveSlope, ParseError, SourceOutsideDomain,
                     ValidationError, VoxelOutOfRange)
from .scene import (AccumulationMode, Benchmark, BenchmarkSetup, BoundaryMode, Detector,  # noqa: F401
                    OpticalProperties, Precision, Scene, SimulationConfig, Source, VoxelGrid,
                    VoxelIndex, baseline_setup, benchmark_from_name, benchmark_preset, head_labels)
from .runtime import (Calibration, DeviceKind, DeviceProfile, FluenceMap, GroupRunResult,  # noqa: F401
                      MultiDeviceResult, Partition, PhotonDisposition, Plan, Strategy, calibrate,
                      device_count, lib, make_partition, merge, model_makespan, partition_s1,
                      partition_s2, partition_s3, quantum_for, rng_kat, run_group_dynamic,
                      run_multi_device, run_static_split, simulate_photon, simulate_photon_trace, strategy_from_name,
                      thread_count_heuristic, trace_photons)
