/*
 * vmc.h — C-ABI of the B200 voxel Monte Carlo photon-transport library
 * (libvoxmc_b200.so). Plain C types only: no torch, no C++ objects.
 *
 * This is the drop-in boundary for the reference's per-device executor and
 * multi-device runner (reference = /root/reference/proj, "voxmc"):
 *
 *   vmc_run_range      replaces voxmc::run_group_dynamic
 *                      (proj/core/include/voxmc/scheduler.hpp:98-99,
 *                       impl proj/core/src/scheduler.cpp:255-324)
 *   vmc_run_multi      replaces voxmc::run_multi_device
 *                      (scheduler.hpp:143-145, scheduler.cpp:395-451)
 *   vmc_partition      replaces partition_s1/s2/s3 + make_partition
 *                      (scheduler.hpp:45-56, scheduler.cpp:49-251)
 *   vmc_rng_kat        exposes RngStream::next_u64 on the device
 *                      (proj/core/include/voxmc/rng.hpp:11-35, proj/core/src/rng.cpp:5-19)
 *   vmc_quantum_for    FluenceMap quantum rule (proj/core/src/fluence.cpp:11-14)
 *   vmc_plan_*         device-resident form of the executor (scene uploaded
 *                      once, buffers owned by the caller, e.g. torch tensors),
 *                      used for in-HBM timing and the NCCL reduce path.
 *
 * Error convention (all int-returning functions): 0 = ok;
 * VMC_ERR_VALIDATION (→ voxmc::ValidationError / SourceOutsideDomain in the
 * C++ shim, reference errors.hpp:9-59); VMC_ERR_RUNTIME (CUDA / NCCL /
 * allocation). The message of the last failure on the calling thread is
 * returned by vmc_last_error().
 *
 * Fluence cells are signed 64-bit fixed point exactly as the reference's
 * FluenceMap: value = cell * quantum, quantum = 2^-(62 - bit_width(N))
 * with N = config.photon_count (the GLOBAL photon count, not the range).
 * Layout [gate][z][y][x], x fastest (reference VoxelGrid::linear, types.hpp:68-72).
 */
#ifndef VMC_H_
#define VMC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VMC_ABI_VERSION 1

#if defined(__GNUC__)
#define VMC_API __attribute__((visibility("default")))
#else
#define VMC_API
#endif

#define VMC_OK 0
#define VMC_ERR_VALIDATION 1
#define VMC_ERR_RUNTIME 2

/* boundary_mode (reference BoundaryMode, types.hpp:95) */
#define VMC_BOUNDARY_TERMINATE 0
#define VMC_BOUNDARY_REFLECT 1

/* accumulation_mode (reference AccumulationMode, types.hpp:94). Accepted for
 * API parity; the device always accumulates with exact integer atomics, which
 * give the same raw cells as either reference mode (fluence.hpp:15-25). */
#define VMC_ACCUM_SHARED_ATOMIC 0
#define VMC_ACCUM_PRIVATE_MERGE 1

/* precision: FP32 is the product path; FP64 re-runs the reference's double
 * arithmetic on the device (parity/diagnostic mode). */
#define VMC_PRECISION_FP32 0
#define VMC_PRECISION_FP64 1

/* Labeled voxel volume + media + source (reference VoxelGrid types.hpp:56-92,
 * OpticalProperties types.hpp:37-44, Source types.hpp:112-116). */
typedef struct vmc_scene {
  int32_t nx, ny, nz;
  double voxel_mm;
  const uint8_t* labels;  /* nx*ny*nz labels, x fastest; label < nmedia */
  int32_t nmedia;
  const double* media;    /* [nmedia][4] = mua (1/mm), mus (1/mm), g, n; [0] = exterior */
  double src_pos[3];
  double src_dir[3];
  int32_t isotropic;
} vmc_scene;

/* Run parameters (reference SimulationConfig types.hpp:97-108) plus the
 * B200 build's additions: time gates and disk detectors. */
typedef struct vmc_config {
  uint64_t photon_count;       /* global N: fixes the quantum */
  uint64_t master_seed;
  int32_t accumulation_mode;   /* VMC_ACCUM_* */
  int32_t boundary_mode;       /* VMC_BOUNDARY_* */
  double tmax_ns;              /* photon time horizon */
  double roulette_threshold;
  int32_t roulette_multiplier;
  int32_t workgroup_size;      /* CUDA block size; 0 = library default */
  int32_t ngates;              /* >= 1; gate g covers [g, g+1) * tmax_ns/ngates */
  int32_t precision;           /* VMC_PRECISION_* */
  int32_t ndet;                /* number of disk detectors (0 = none) */
  int32_t reserved0;
  const double* det;           /* [ndet][4] = x, y, z, radius (mm) */
  uint64_t det_capacity;       /* max detector records stored */
} vmc_config;

/* Terminal weight bookkeeping (reference PhotonDisposition,
 * transport.hpp:89-102) in the fluence quantum: value = q * quantum. */
typedef struct vmc_disposition {
  int64_t deposited_q;
  int64_t escaped_q;
  int64_t killed_q;
  int64_t truncated_q;
  double quantum;
} vmc_disposition;

/* Device capacity for partitioning (reference DeviceProfile, scheduler.hpp:21-28). */
typedef struct vmc_device_profile {
  int32_t cores;
  int32_t reserved0;
  double a;   /* ms per photon */
  double t0;  /* ms startup overhead */
} vmc_device_profile;

#define VMC_STRATEGY_S1 1
#define VMC_STRATEGY_S2 2
#define VMC_STRATEGY_S3 3

/* Per-photon diagnostic record (tests only; no reference equivalent beyond
 * simulate_photon_trace, transport.cpp:368-380). Dispositions in launched
 * weight units; draws = RNG u64 draws consumed by the photon. */
typedef struct vmc_photon_trace {
  uint32_t draws;
  uint32_t steps;
  uint32_t scatters;
  uint32_t flags;  /* bit0 escaped, bit1 killed, bit2 truncated, bit3 detected */
  double deposited;
  double escaped;
  double killed;
  double truncated;
} vmc_photon_trace;

/* Detector record: fixed header + one float per interior label 1..nmedia-1.
 *   uint64 photon_index; uint32 det_id; uint32 nscat; float w_exit;
 *   float t_exit_ns; float ppath_mm[nmedia-1]; (padded to 8 bytes)
 * Records returned by vmc_run_range / vmc_run_multi are sorted by
 * photon_index, so output is identical for any GPU count. */
typedef struct vmc_det_record_head {
  uint64_t photon_index;
  uint32_t det_id;
  uint32_t nscat;
  float w_exit;
  float t_exit_ns;
} vmc_det_record_head;

VMC_API size_t vmc_det_record_bytes(int32_t nmedia);

VMC_API int vmc_abi_version(void);
VMC_API const char* vmc_last_error(void);
VMC_API int vmc_device_count(void);

/* Quantum for N photons: 2^-(62 - bit_width(N|1)) (fluence.cpp:11-14). */
VMC_API double vmc_quantum_for(uint64_t photon_count);

/* Validates a scene/config pair exactly as the reference does
 * (VoxelGrid ctor types.cpp:7-33, SimulationConfig::validate types.cpp:44-52,
 * launch voxel check transport.cpp:96-99). */
VMC_API int vmc_validate(const vmc_scene* scene, const vmc_config* config);

/* Per-device executor, host buffers (the reference-facing call).
 * Simulates global photons [first_index, first_index+count) on CUDA device
 * `device`; photon k uses RNG stream (master_seed, k).
 * cells_out: host [ngates*nx*ny*nz] int64, overwritten (may be NULL).
 * totals_out: may be NULL. det_out: host buffer of det_capacity records
 * (may be NULL when ndet == 0); det_count_out = records detected (may exceed
 * det_capacity; only min(count, capacity) are stored).
 * wall_ms_out: device time of the run (events around the kernels). */
VMC_API int vmc_run_range(const vmc_scene* scene, const vmc_config* config, uint64_t first_index,
                  uint64_t count, int device, int64_t* cells_out, vmc_disposition* totals_out,
                  void* det_out, uint64_t* det_count_out, double* wall_ms_out);

/* Multi-device runner inside one process: contiguous ranges counts[i] in
 * device order starting at photon 0 (reference scheduler.cpp:405-413), one
 * host thread per device, exact int64 sum of the per-device maps (NCCL
 * reduce to devices[0] when ndev > 1). per_device_ms: [ndev] (may be NULL). */
VMC_API int vmc_run_multi(const vmc_scene* scene, const vmc_config* config, int ndev, const int* devices,
                  const uint64_t* counts, int64_t* cells_out, vmc_disposition* totals_out,
                  void* det_out, uint64_t* det_count_out, double* per_device_ms,
                  double* reduce_ms);

/* Photon-count partition over devices (reference partition_s1/s2/s3). */
VMC_API int vmc_partition(int strategy, uint64_t total, int ndev, const vmc_device_profile* devices,
                  uint64_t* counts_out);
VMC_API double vmc_model_makespan(int ndev, const uint64_t* counts, const vmc_device_profile* devices);

/* First n outputs of RngStream(seed, stream_id).next_u64() computed on the device. */
VMC_API int vmc_rng_kat(uint64_t seed, uint64_t stream_id, int n, int device, uint64_t* out);

/* One photon's walk in the reference's arithmetic (FP64 flight kernel) on
 * `device`: reference simulate_photon / simulate_photon_trace
 * (proj/core/include/voxmc/transport.hpp:105-113, transport.cpp:362-380).
 * Writes the per-step deposits in walk order (linear cell, absorbed weight;
 * steps that deposit nothing are skipped, as the reference's sink never sees
 * them) into cells_out/dw_out (first max_deposits of *n_deposits) and the
 * photon's disposition {deposited, escaped, killed, truncated} into disp_out.
 * Time gates are ignored (continuous wave). Synchronous. */
VMC_API int vmc_simulate_photon(const vmc_scene* scene, const vmc_config* config, uint64_t photon_index,
                                int device, uint64_t max_deposits, int64_t* cells_out, double* dw_out,
                                uint64_t* n_deposits, double* disp_out);

/* ---- device-resident plan: scene on the GPU, caller-owned buffers ------- */
typedef struct vmc_plan vmc_plan;

VMC_API int vmc_plan_create(const vmc_scene* scene, const vmc_config* config, int device,
                    vmc_plan** out);
VMC_API int vmc_plan_destroy(vmc_plan* plan);
/* Number of int64 cells (ngates*nx*ny*nz) and the record stride. */
VMC_API uint64_t vmc_plan_cell_count(const vmc_plan* plan);

#define VMC_RUN_ZERO 1u /* zero d_cells / d_totals / d_det_count before the run */

/* Runs photons [first_index, first_index+count) on `stream` (cudaStream_t, 0 =
 * legacy default). Device buffers: d_cells [cell_count] int64 (accumulated),
 * d_totals [4] int64 (deposited/escaped/killed/truncated quanta, accumulated),
 * d_det (det_capacity records) and d_det_count [1] uint64 (may be NULL when
 * ndet == 0). Asynchronous: returns after enqueueing. Runs of one plan share
 * its claim counter and scratch maps, so each run is ordered after the
 * previous run of the same plan even across streams (an event wait). */
VMC_API int vmc_plan_run(vmc_plan* plan, uint64_t first_index, uint64_t count, int64_t* d_cells,
                 int64_t* d_totals, void* d_det, uint64_t* d_det_count, void* stream,
                 uint32_t flags);

/* Per-photon diagnostics for photons [first_index, first_index+count) into the
 * host array out[count]. Deposits are not accumulated. Synchronous. */
VMC_API int vmc_plan_trace(vmc_plan* plan, uint64_t first_index, uint64_t count, vmc_photon_trace* out);

/* K4: fluence normalization Phi = E / (mua * V * N) (reference FluenceMap::normalize,
 * fluence.cpp:62-84, and to_float_volume, :86-90) as one device pass. d_cells as
 * written by vmc_plan_run ([ngates][z][y][x]); d_out float [ngates * V] when
 * sum_gates == 0, else [V] (CW, gate-summed before normalizing). Voxels with
 * mua == 0 map to 0. normalized == 0 skips the division (raw weight = cell * quantum). */
VMC_API int vmc_plan_normalize(vmc_plan* plan, const int64_t* d_cells, uint64_t photon_count, float* d_out,
                               int sum_gates, int normalized, void* stream);

/* FNV-1a 64 of a byte buffer (the reference's volume checksum, volume_io.cpp:13-20). Host only. */
VMC_API uint64_t vmc_fnv1a64(const void* data, size_t bytes);

/* Sorts n detector records written by vmc_plan_run for photons
 * [first_index, first_index+count) by photon index into d_out (device, n
 * records, must not alias d_recs), on `stream`. Records of contiguous ranges
 * sorted this way and concatenated in range order are globally sorted, which
 * is how multi-GPU gathers stay identical for any GPU count. Requires
 * count <= 2^32. Asynchronous. */
VMC_API int vmc_plan_sort_records(vmc_plan* plan, const void* d_recs, uint64_t n, uint64_t first_index,
                                  uint64_t count, void* d_out, void* stream);

/* Mangled device symbol of the transport kernel variant this plan launches
 * (e.g. _ZN3vmc8k_flightIfLb1ELb0ELb0ELb0ELi0EEEvNS_10KernelArgsE = the FP32
 * gated multi-label K1f with direct deposits); "" when unavailable. Valid while the plan lives. */
VMC_API const char* vmc_plan_kernel_name(const vmc_plan* plan);

/* Number of kernels vmc_plan_run enqueues per call (for launch accounting). */
VMC_API int vmc_plan_launches_per_run(const vmc_plan* plan, uint32_t flags);

#ifdef __cplusplus
}
#endif

#endif /* VMC_H_ */
