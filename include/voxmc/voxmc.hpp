// voxmc.hpp — C++ drop-in API of the B200 library (libvoxmc_b200.so).
//
// Code written against the reference library's public headers
// (/root/reference/proj/core/include/voxmc/{types,rng,fluence,transport,
// scheduler,errors}.hpp) compiles against this header set unchanged for the
// executor path: same namespace, type names, fields, function signatures and
// exception types. What changes is where the photons run: run_group_dynamic,
// run_static_split, run_multi_device and calibrate() execute on B200s through
// the C-ABI in vmc.h (no host worker threads, no CPU fallback).
//
// Additive extensions (marked B200): SimulationConfig::{ngates, precision,
// detectors, det_capacity}, DeviceKind::CudaGpu + DeviceProfile::gpu,
// FluenceMap::raw_cells() (raw int64 span; a double round trip would lose bits
// above 2^53) and gate-resolved maps, detector records on the results.
#pragma once

#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#pragma GCC visibility push(default)
namespace voxmc {

// ---- errors (reference errors.hpp) ---------------------------------------
struct ValidationError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct VoxelOutOfRange : std::out_of_range { using std::out_of_range::out_of_range; };
struct DimensionMismatch : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct AlreadyNormalized : std::logic_error { using std::logic_error::logic_error; };
struct SourceOutsideDomain : ValidationError { using ValidationError::ValidationError; };
struct NonPositiveSlope : std::runtime_error { using std::runtime_error::runtime_error; };
struct InstanceTooLarge : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct NonPositiveRadius : std::domain_error { using std::domain_error::domain_error; };

// ---- domain (reference types.hpp) ----------------------------------------
inline constexpr double kLightSpeedMmPerNs = 299.792458;

struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  constexpr Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  constexpr Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  constexpr Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
  constexpr double dot(const Vec3& o) const { return x * o.x + y * o.y + z * o.z; }
  double norm() const { return std::sqrt(dot(*this)); }
  Vec3 normalized() const { const double k = 1.0 / norm(); return {x * k, y * k, z * k}; }
  constexpr double operator[](int a) const { return a == 0 ? x : (a == 1 ? y : z); }
  double& ref(int a) { return a == 0 ? x : (a == 1 ? y : z); }
};

struct OpticalProperties {
  double mua = 0.0, mus = 0.0, g = 0.0, n = 1.0;
  bool operator==(const OpticalProperties&) const = default;
};

struct VoxelIndex {
  int x = 0, y = 0, z = 0;
  bool operator==(const VoxelIndex&) const = default;
};

class VoxelGrid {
 public:
  VoxelGrid(VoxelIndex dims, double voxel_size_mm, std::vector<std::uint8_t> labels,
            std::vector<OpticalProperties> media);
  VoxelIndex dims() const { return dims_; }
  int nx() const { return dims_.x; }
  int ny() const { return dims_.y; }
  int nz() const { return dims_.z; }
  double voxel_size() const { return h_; }
  std::size_t voxel_count() const { return labels_.size(); }
  std::size_t linear(const VoxelIndex& v) const {
    return static_cast<std::size_t>(v.x) +
           static_cast<std::size_t>(dims_.x) * (static_cast<std::size_t>(v.y) + static_cast<std::size_t>(dims_.y) * v.z);
  }
  bool contains(const VoxelIndex& v) const {
    return v.x >= 0 && v.y >= 0 && v.z >= 0 && v.x < dims_.x && v.y < dims_.y && v.z < dims_.z;
  }
  std::uint8_t label(const VoxelIndex& v) const { return labels_[linear(v)]; }
  const OpticalProperties& medium(std::uint8_t l) const { return media_[l]; }
  const OpticalProperties& medium_at(const VoxelIndex& v) const { return media_[label(v)]; }
  const OpticalProperties& exterior() const { return media_[0]; }
  const std::vector<OpticalProperties>& media() const { return media_; }
  const std::vector<std::uint8_t>& labels() const { return labels_; }
  std::optional<VoxelIndex> voxel_of(const Vec3& p) const;

 private:
  VoxelIndex dims_;
  double h_;
  std::vector<std::uint8_t> labels_;
  std::vector<OpticalProperties> media_;
};

enum class AccumulationMode { SharedAtomic, PrivateMerge };
enum class BoundaryMode { TerminateAtBoundary, ReflectAtMismatch };
enum class Precision { FP32, FP64 };  // B200

struct Detector {  // B200: disk detector on the exit surface
  Vec3 position;
  double radius = 1.0;
};

struct SimulationConfig {
  std::uint64_t photon_count = 100'000'000;
  std::uint64_t master_seed = 0;
  AccumulationMode accumulation_mode = AccumulationMode::PrivateMerge;
  BoundaryMode boundary_mode = BoundaryMode::TerminateAtBoundary;
  double tmax_ns = 5.0;
  double roulette_threshold = 1e-4;
  int roulette_multiplier = 10;
  int workgroup_size = 64;
  // B200 additions
  int ngates = 1;
  Precision precision = Precision::FP32;
  std::vector<Detector> detectors;
  std::uint64_t det_capacity = 0;

  void validate() const;
};

struct Source {
  Vec3 position;
  Vec3 direction{0.0, 0.0, 1.0};
  bool isotropic = false;
};

struct Scene {
  VoxelGrid grid;
  Source source;
};

enum class Benchmark { B1, B2, B2a };

struct BenchmarkSetup {
  VoxelGrid grid;
  Source source;
  SimulationConfig config;
};

BenchmarkSetup benchmark_preset(Benchmark name);
std::optional<Benchmark> benchmark_from_name(std::string_view name);
std::string_view benchmark_name(Benchmark b);

// ---- RNG (reference rng.hpp): host copy of the device stream --------------
std::uint64_t mix64(std::uint64_t z);

class RngStream {
 public:
  RngStream(std::uint64_t master_seed, std::uint64_t stream_id);
  std::uint64_t next_u64() {
    std::uint64_t a = s_[0];
    const std::uint64_t b = s_[1];
    const std::uint64_t out = a + b;
    a ^= a << 23;
    s_[0] = b;
    s_[1] = a ^ b ^ (a >> 18) ^ (b >> 5);
    return out;
  }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  std::uint64_t stream_id() const { return id_; }
  std::uint64_t state_lo() const { return s_[0]; }
  std::uint64_t state_hi() const { return s_[1]; }

 private:
  std::uint64_t s_[2];
  std::uint64_t id_;
};

// ---- scalar physics used by the kernel, for host-side checks --------------
double hg_cos_theta(double g, double xi);
double fresnel_reflectance(double n1, double n2, double cos_i);

// ---- accumulator (reference fluence.hpp) -----------------------------------
class FluenceMap {
 public:
  FluenceMap(VoxelIndex dims, std::uint64_t photon_count,
             AccumulationMode mode = AccumulationMode::PrivateMerge, bool track_counts = false,
             int ngates = 1);
  VoxelIndex dims() const { return dims_; }
  std::size_t voxel_count() const { return static_cast<std::size_t>(dims_.x) * dims_.y * dims_.z; }
  std::uint64_t photon_count() const { return photon_count_; }
  AccumulationMode mode() const { return mode_; }
  double quantum() const { return quantum_; }
  bool normalized() const { return normalized_; }
  int ngates() const { return ngates_; }

  void deposit(std::size_t cell, double dw);
  void deposit(const VoxelIndex& v, double dw);
  // CW (gate-summed) value of one voxel, or fluence after normalize()
  double value(std::size_t cell) const;
  std::int64_t raw_cell(std::size_t cell) const;  // CW raw cell
  std::int64_t deposit_count(std::size_t cell) const { return counts_.empty() ? -1 : counts_[cell]; }
  double total_deposited() const;
  void add(const FluenceMap& other);
  void normalize(const VoxelGrid& grid);
  std::size_t zero_mua_voxels() const { return zero_mua_voxels_; }
  std::vector<float> to_float_volume() const;
  // B200: raw int64 cells, layout [gate][z][y][x]
  std::span<std::int64_t> raw_cells() { return cells_; }
  std::span<const std::int64_t> raw_cells() const { return cells_; }

 private:
  VoxelIndex dims_;
  std::uint64_t photon_count_;
  AccumulationMode mode_;
  double quantum_;
  int ngates_;
  bool normalized_ = false;
  std::size_t zero_mua_voxels_ = 0;
  std::vector<std::int64_t> cells_;
  std::vector<std::int64_t> counts_;
  std::vector<double> values_;
};

FluenceMap merge(std::span<const FluenceMap> maps);

// ---- dispositions (reference transport.hpp) --------------------------------
struct PhotonDisposition {
  double deposited = 0.0, escaped = 0.0, killed = 0.0, truncated = 0.0;
  PhotonDisposition& operator+=(const PhotonDisposition& o) {
    deposited += o.deposited;
    escaped += o.escaped;
    killed += o.killed;
    truncated += o.truncated;
    return *this;
  }
};

// ---- single-photon state and host helpers (reference transport.hpp:16-83) --
// The walk itself runs on the device (simulate_photon below, the executors);
// these scalar helpers give reference callers the same one-photon building
// blocks (launch state, DDA distance, one HG deflection, one walk segment,
// one interface, one roulette draw) on the host, in the reference's double
// arithmetic, e.g. for tests and diagnostics. They are not used by any executor.
struct PhotonState {
  Vec3 position;
  Vec3 direction;
  Vec3 inv_direction;
  double weight = 1.0;
  double time_ns = 0.0;
  double remaining_scat = 0.0;
  std::uint8_t medium = 0;
  VoxelIndex voxel;
  void set_direction(const Vec3& d);
};

enum class StepKind { Scattered, CrossedVoxel, ExitedDomain, Reflected, Terminated };

struct StepOutcome {
  StepKind kind = StepKind::Terminated;
  double deposited = 0.0;
  bool interface_pending = false;
  int face_axis = -1;
  int face_step = 0;
  VoxelIndex next_voxel;
  bool next_is_exterior = false;
};

PhotonState launch(const Source& source, const VoxelGrid& grid, RngStream& stream);
double distance_to_voxel_boundary(const Vec3& position, const Vec3& direction, const VoxelGrid& grid);
Vec3 hg_scatter(const Vec3& direction, double g, RngStream& stream);
StepOutcome advance(PhotonState& photon, const VoxelGrid& grid, const SimulationConfig& config, RngStream& stream);
StepOutcome handle_interface(PhotonState& photon, const VoxelGrid& grid, const SimulationConfig& config,
                             const StepOutcome& crossing, RngStream& stream);
bool roulette(PhotonState& photon, const SimulationConfig& config, RngStream& stream);

// One photon's walk (reference transport.hpp:105-113), executed on CUDA device
// 0 by the FP64 flight kernel (the reference's arithmetic): simulate_photon
// adds every step deposit to `map` through FluenceMap::deposit;
// simulate_photon_trace returns the per-step deposit list in walk order.
PhotonDisposition simulate_photon(std::uint64_t photon_index, const Scene& scene, const SimulationConfig& config,
                                  FluenceMap& map);
PhotonDisposition simulate_photon_trace(std::uint64_t photon_index, const Scene& scene,
                                        const SimulationConfig& config,
                                        std::vector<std::pair<VoxelIndex, double>>& deposits);

struct DetectorRecord {  // B200
  std::uint64_t photon_index = 0;
  std::uint32_t det_id = 0;
  std::uint32_t nscat = 0;
  float w_exit = 0.f;
  float t_exit_ns = 0.f;
  std::vector<float> ppath_mm;  // per interior label 1..nmedia-1
};

// ---- scheduler (reference scheduler.hpp) ------------------------------------
enum class DeviceKind { RealWorkerPool, Simulated, CudaGpu };

struct DeviceProfile {
  std::string name;
  int cores = 1;
  double a = 0.0;
  double t0 = 0.0;
  DeviceKind kind = DeviceKind::Simulated;
  double jitter_sigma = 0.0;
  int gpu = 0;  // B200: CUDA ordinal for DeviceKind::CudaGpu
};

struct Partition {
  std::vector<std::uint64_t> counts;
  std::uint64_t total() const;
};

enum class Strategy { S1, S2, S3 };
std::optional<Strategy> strategy_from_name(std::string_view name);
std::string_view strategy_name(Strategy s);
int thread_count_heuristic(int cores, int max_concurrent_per_core);
Partition partition_s1(std::uint64_t total, std::span<const DeviceProfile> devices);
Partition partition_s2(std::uint64_t total, std::span<const DeviceProfile> devices);
Partition partition_s3(std::uint64_t total, std::span<const DeviceProfile> devices);
Partition make_partition(std::uint64_t total, std::span<const DeviceProfile> devices, Strategy s);
double model_makespan(const Partition& p, std::span<const DeviceProfile> devices);

class GroupCounter {  // claim semantics of the reference; the device uses an atomic twin
 public:
  explicit GroupCounter(std::uint64_t quota) : left_(static_cast<std::int64_t>(quota)), quota_(quota) {}
  std::optional<std::uint64_t> claim() {
    std::int64_t seen = left_.load(std::memory_order_relaxed);
    while (seen > 0)
      if (left_.compare_exchange_weak(seen, seen - 1, std::memory_order_relaxed))
        return quota_ - static_cast<std::uint64_t>(seen);
    return std::nullopt;
  }
  std::uint64_t remaining() const {
    const std::int64_t r = left_.load(std::memory_order_relaxed);
    return r > 0 ? static_cast<std::uint64_t>(r) : 0;
  }

 private:
  std::atomic<std::int64_t> left_;
  std::uint64_t quota_;
};

struct GroupRunResult {
  FluenceMap map;
  PhotonDisposition totals;
  std::vector<std::uint64_t> per_thread_photons;
  double wall_ms = 0.0;
  std::vector<DetectorRecord> detections;  // B200
  std::uint64_t det_count = 0;             // B200 (may exceed detections.size())
};

// Photons [first_index, first_index + quota) on CUDA device 0 (or `gpu`).
GroupRunResult run_group_dynamic(std::uint64_t first_index, std::uint64_t quota, int threads,
                                 const Scene& scene, const SimulationConfig& config);
GroupRunResult run_static_split(std::uint64_t first_index, std::uint64_t quota, int threads,
                                const Scene& scene, const SimulationConfig& config);
GroupRunResult run_group_on(int gpu, std::uint64_t first_index, std::uint64_t quota,
                            const Scene& scene, const SimulationConfig& config);  // B200

double static_split_makespan(std::span<const double> costs, int threads);
double dynamic_makespan(std::span<const double> costs, int threads);

struct Calibration {
  double a = 0.0;
  double t0 = 0.0;
};
Calibration calibrate(const DeviceProfile& device, std::uint64_t n1, std::uint64_t n2, const Scene& scene,
                      const SimulationConfig& config, int threads, std::uint64_t noise_seed = 0);

struct DeviceRunResult {
  std::string name;
  std::uint64_t photons = 0;
  double wall_ms = 0.0;
};

struct MultiDeviceResult {
  FluenceMap map;
  PhotonDisposition totals;
  Partition partition;
  std::vector<DeviceRunResult> devices;
  double makespan_ms = 0.0;
  double reduce_ms = 0.0;                  // B200: NCCL reduce time
  std::vector<DetectorRecord> detections;  // B200
  std::uint64_t det_count = 0;
};

// Devices must be DeviceKind::CudaGpu (B200 runner) — a roster of simulated or
// host-pool devices is rejected with ValidationError.
MultiDeviceResult run_multi_device(std::uint64_t total, std::span<const DeviceProfile> devices, Strategy strategy,
                                   const Scene& scene, const SimulationConfig& config, int threads_per_device);

}  // namespace voxmc
#pragma GCC visibility pop
