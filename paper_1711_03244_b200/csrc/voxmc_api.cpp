// voxmc_api.cpp — the C++ drop-in API (include/voxmc/voxmc.hpp) over the C-ABI.
//
// Host bookkeeping restated from the reference (validation rules, presets,
// FluenceMap arithmetic, partition front-ends); all photon transport goes to
// the device through vmc_run_range / vmc_run_multi. Error codes from the C-ABI
// are rethrown as the reference's exception types.
#include <algorithm>
#include <limits>
#include <cstring>
#include <functional>
#include <numeric>
#include <queue>

#include "vmc.h"
#include "voxmc/voxmc.hpp"

namespace voxmc {

namespace {

[[noreturn]] void rethrow(int rc) {
  const std::string msg = vmc_last_error();
  if (rc == VMC_ERR_VALIDATION) {
    if (msg.find("outside the voxel grid") != std::string::npos) throw SourceOutsideDomain(msg);
    throw ValidationError(msg);
  }
  throw std::runtime_error(msg);
}

void check(int rc) {
  if (rc != VMC_OK) rethrow(rc);
}

// Flattened scene/config for the C-ABI; owns the arrays the structs point to.
struct Abi {
  vmc_scene s{};
  vmc_config c{};
  std::vector<double> media, det;

  Abi(const Scene& scene, const SimulationConfig& cfg) {
    const VoxelGrid& g = scene.grid;
    s.nx = g.nx();
    s.ny = g.ny();
    s.nz = g.nz();
    s.voxel_mm = g.voxel_size();
    s.labels = g.labels().data();
    s.nmedia = static_cast<int32_t>(g.media().size());
    for (const OpticalProperties& m : g.media()) media.insert(media.end(), {m.mua, m.mus, m.g, m.n});
    s.media = media.data();
    const Source& src = scene.source;
    for (int k = 0; k < 3; ++k) {
      s.src_pos[k] = src.position[k];
      s.src_dir[k] = src.direction[k];
    }
    s.isotropic = src.isotropic ? 1 : 0;
    c.photon_count = cfg.photon_count;
    c.master_seed = cfg.master_seed;
    c.accumulation_mode =
        cfg.accumulation_mode == AccumulationMode::SharedAtomic ? VMC_ACCUM_SHARED_ATOMIC : VMC_ACCUM_PRIVATE_MERGE;
    c.boundary_mode = cfg.boundary_mode == BoundaryMode::ReflectAtMismatch ? VMC_BOUNDARY_REFLECT
                                                                           : VMC_BOUNDARY_TERMINATE;
    c.tmax_ns = cfg.tmax_ns;
    c.roulette_threshold = cfg.roulette_threshold;
    c.roulette_multiplier = cfg.roulette_multiplier;
    c.workgroup_size = 0;
    c.ngates = cfg.ngates;
    // VMC_DROPIN_PRECISION=fp64 runs every drop-in call in the reference's
    // arithmetic (the FP64 kernels) whatever the config says: reference
    // programs that compare a single-photon walk against an executor, like
    // acceptance.cpp's criterion 3, then compare like with like
    static const bool force_fp64 = [] {
      const char* e = std::getenv("VMC_DROPIN_PRECISION");
      return e && std::string(e) == "fp64";
    }();
    c.precision = (force_fp64 || cfg.precision == Precision::FP64) ? VMC_PRECISION_FP64 : VMC_PRECISION_FP32;
    for (const Detector& d : cfg.detectors) det.insert(det.end(), {d.position.x, d.position.y, d.position.z, d.radius});
    c.ndet = static_cast<int32_t>(cfg.detectors.size());
    c.det = det.empty() ? nullptr : det.data();
    c.det_capacity = cfg.det_capacity;
  }
};

std::vector<DetectorRecord> unpack_records(const std::vector<unsigned char>& raw, std::uint64_t n, int nmedia) {
  const std::size_t stride = vmc_det_record_bytes(nmedia);
  std::vector<DetectorRecord> out(n);
  for (std::uint64_t i = 0; i < n; ++i) {
    const unsigned char* rec = raw.data() + i * stride;
    vmc_det_record_head h;
    std::memcpy(&h, rec, sizeof h);
    DetectorRecord& r = out[i];
    r.photon_index = h.photon_index;
    r.det_id = h.det_id;
    r.nscat = h.nscat;
    r.w_exit = h.w_exit;
    r.t_exit_ns = h.t_exit_ns;
    r.ppath_mm.resize(static_cast<std::size_t>(std::max(0, nmedia - 1)));
    std::memcpy(r.ppath_mm.data(), rec + sizeof h, r.ppath_mm.size() * sizeof(float));
  }
  return out;
}

PhotonDisposition from_quanta(const vmc_disposition& d) {
  return {static_cast<double>(d.deposited_q) * d.quantum, static_cast<double>(d.escaped_q) * d.quantum,
          static_cast<double>(d.killed_q) * d.quantum, static_cast<double>(d.truncated_q) * d.quantum};
}

std::vector<vmc_device_profile> profiles(std::span<const DeviceProfile> devs) {
  std::vector<vmc_device_profile> p(devs.size());
  for (std::size_t i = 0; i < devs.size(); ++i) p[i] = {devs[i].cores, 0, devs[i].a, devs[i].t0};
  return p;
}

}  // namespace

// ---- domain ----------------------------------------------------------------
VoxelGrid::VoxelGrid(VoxelIndex dims, double voxel_size_mm, std::vector<std::uint8_t> labels,
                     std::vector<OpticalProperties> media)
    : dims_(dims), h_(voxel_size_mm), labels_(std::move(labels)), media_(std::move(media)) {
  if (dims_.x < 1 || dims_.y < 1 || dims_.z < 1) throw ValidationError("VoxelGrid: all dims must be >= 1");
  if (!(h_ > 0.0)) throw ValidationError("VoxelGrid: voxel_size must be > 0");
  if (labels_.size() != static_cast<std::size_t>(dims_.x) * dims_.y * dims_.z)
    throw ValidationError("VoxelGrid: label array size does not match dims");
  if (media_.empty()) throw ValidationError("VoxelGrid: media list is empty");
  for (const OpticalProperties& m : media_)
    if (m.mua < 0.0 || m.mus < 0.0 || m.g < -1.0 || m.g > 1.0 || m.n < 1.0)
      throw ValidationError("VoxelGrid: invalid optical properties");
  const std::uint8_t top = labels_.empty() ? 0 : *std::max_element(labels_.begin(), labels_.end());
  if (top >= media_.size()) throw ValidationError("VoxelGrid: label exceeds media list");
}

std::optional<VoxelIndex> VoxelGrid::voxel_of(const Vec3& p) const {
  const VoxelIndex v{static_cast<int>(std::floor(p.x / h_)), static_cast<int>(std::floor(p.y / h_)),
                     static_cast<int>(std::floor(p.z / h_))};
  if (!contains(v)) return std::nullopt;
  return v;
}

void SimulationConfig::validate() const {
  if (photon_count < 1) throw ValidationError("photon_count must be >= 1");
  if (!(tmax_ns > 0.0)) throw ValidationError("tmax must be > 0");
  if (!(roulette_threshold > 0.0 && roulette_threshold < 1.0))
    throw ValidationError("roulette_threshold must be in (0, 1)");
  if (roulette_multiplier < 2) throw ValidationError("roulette_multiplier must be >= 2");
  if (workgroup_size < 1) throw ValidationError("workgroup_size must be >= 1");
  if (ngates < 1) throw ValidationError("ngates must be >= 1");
}

BenchmarkSetup benchmark_preset(Benchmark name) {
  // 60^3 mm cube of turbid medium, pencil beam at (30,30,0) along +z; B2/B2a
  // add a 15 mm sphere at the centre and switch to Fresnel boundaries.
  const bool sphere = name != Benchmark::B1;
  std::vector<OpticalProperties> media{{0.0, 0.0, 0.0, 1.0}, {0.005, 1.0, 0.01, 1.37}};
  if (sphere) media.push_back({0.002, 5.0, 0.9, 1.0});
  std::vector<std::uint8_t> labels(60u * 60u * 60u, 1);
  if (sphere) {
    for (int z = 0, i = 0; z < 60; ++z)
      for (int y = 0; y < 60; ++y)
        for (int x = 0; x < 60; ++x, ++i) {
          const double dx = x + 0.5 - 30.0, dy = y + 0.5 - 30.0, dz = z + 0.5 - 30.0;
          if (dx * dx + dy * dy + dz * dz <= 225.0) labels[i] = 2;
        }
  }
  SimulationConfig cfg;
  cfg.photon_count = 100'000'000;
  cfg.boundary_mode = sphere ? BoundaryMode::ReflectAtMismatch : BoundaryMode::TerminateAtBoundary;
  cfg.accumulation_mode = name == Benchmark::B2a ? AccumulationMode::SharedAtomic : AccumulationMode::PrivateMerge;
  Source src;
  src.position = {30.0, 30.0, 0.0};
  return BenchmarkSetup{VoxelGrid({60, 60, 60}, 1.0, std::move(labels), std::move(media)), src, cfg};
}

std::optional<Benchmark> benchmark_from_name(std::string_view n) {
  if (n == "B1" || n == "b1") return Benchmark::B1;
  if (n == "B2" || n == "b2") return Benchmark::B2;
  if (n == "B2a" || n == "b2a" || n == "B2A") return Benchmark::B2a;
  return std::nullopt;
}

std::string_view benchmark_name(Benchmark b) {
  return b == Benchmark::B1 ? "B1" : (b == Benchmark::B2 ? "B2" : "B2a");
}

std::uint64_t mix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

RngStream::RngStream(std::uint64_t master_seed, std::uint64_t stream_id) : id_(stream_id) {
  const std::uint64_t z = master_seed ^ stream_id;
  s_[0] = mix64(z);
  s_[1] = mix64(z + 0x9E3779B97F4A7C15ULL);
  if ((s_[0] | s_[1]) == 0) s_[1] = 0x6A09E667F3BCC909ULL;
}

double hg_cos_theta(double g, double xi) {
  if (std::fabs(g) < 1e-6) return 2.0 * xi - 1.0;
  const double f = (1.0 - g * g) / (1.0 - g + 2.0 * g * xi);
  return std::clamp((1.0 + g * g - f * f) / (2.0 * g), -1.0, 1.0);
}

double fresnel_reflectance(double n1, double n2, double ci) {
  ci = std::clamp(ci, 0.0, 1.0);
  const double eta = n1 / n2;
  const double st2 = eta * eta * (1.0 - ci * ci);
  if (st2 > 1.0) return 1.0;
  const double ct = std::sqrt(1.0 - st2);
  const double rs = (n1 * ci - n2 * ct) / (n1 * ci + n2 * ct);
  const double rp = (n1 * ct - n2 * ci) / (n1 * ct + n2 * ci);
  return 0.5 * (rs * rs + rp * rp);
}

// ---- one-photon host helpers (reference transport.hpp:45-83, transport.cpp) --
namespace {
constexpr double kInfD = std::numeric_limits<double>::infinity();
double unit_length(RngStream& stream) {  // -ln(u), u = 0 -> denorm_min (transport.cpp:14-17)
  const double u = stream.next_unit();
  return -std::log(u > 0.0 ? u : std::numeric_limits<double>::denorm_min());
}
}  // namespace

void PhotonState::set_direction(const Vec3& d) {  // transport.cpp:77-81
  direction = d;
  inv_direction = {d.x != 0.0 ? 1.0 / d.x : kInfD, d.y != 0.0 ? 1.0 / d.y : kInfD, d.z != 0.0 ? 1.0 / d.z : kInfD};
}

PhotonState launch(const Source& source, const VoxelGrid& grid, RngStream& stream) {  // transport.cpp:83-106
  Vec3 dir = source.direction.normalized();
  if (source.isotropic) {
    const double mu = 2.0 * stream.next_unit() - 1.0;
    const double phi = 2.0 * 3.14159265358979323846 * stream.next_unit();
    const double s = std::sqrt(std::max(0.0, 1.0 - mu * mu));
    dir = {s * std::cos(phi), s * std::sin(phi), mu};
  }
  PhotonState st;
  st.set_direction(dir);
  st.position = source.position + dir * 1e-6;
  const std::optional<VoxelIndex> v = grid.voxel_of(st.position);
  if (!v) throw SourceOutsideDomain("source entry point maps outside the voxel grid");
  st.voxel = *v;
  st.medium = grid.label(*v);
  st.remaining_scat = unit_length(stream);
  return st;
}

namespace {
// Distance along the photon's direction to the nearest bounding plane of the
// voxel `v` (the integer index is authoritative, transport.cpp:49-73): per axis
// ((v + [d > 0]) h - p) / d clamped at 0, +inf for a zero component; `axis`
// reports the plane's axis, ties going to the lower axis.
double nearest_plane(const PhotonState& st, const VoxelIndex& v, double h, int& axis) {
  const int iv[3] = {v.x, v.y, v.z};
  double best = kInfD;
  axis = 0;
  for (int k = 0; k < 3; ++k) {
    const double dk = st.direction[k];
    if (dk == 0.0) continue;  // never crosses its planes
    const double t = std::max(0.0, ((iv[k] + (dk > 0.0 ? 1 : 0)) * h - st.position[k]) * st.inv_direction[k]);
    if (t < best) {  // strict: ties keep the lower axis
      best = t;
      axis = k;
    }
  }
  return best;
}

// exp(-x) the way the reference evaluates it (transport.cpp:22-27): the
// degree-4 series below 0.01, libm above
double beer_lambert(double x) {
  return x < 0.01 ? 1.0 - x * (1.0 - x * (0.5 - x * (1.0 / 6.0 - x * (1.0 / 24.0)))) : std::exp(-x);
}

// mirror the direction component of `axis` (specular reflection off that face)
void mirror(PhotonState& photon, int axis) {
  Vec3 d = photon.direction;
  d.ref(axis) = -d[axis];
  photon.set_direction(d);
}
}  // namespace

double distance_to_voxel_boundary(const Vec3& position, const Vec3& direction, const VoxelGrid& grid) {
  const std::optional<VoxelIndex> v = grid.voxel_of(position);  // transport.cpp:108-118, :49-73
  if (!v) throw VoxelOutOfRange("position outside grid");
  PhotonState st;
  st.position = position;
  st.set_direction(direction);
  int axis = 0;
  return nearest_plane(st, *v, grid.voxel_size(), axis);
}

// One segment of the walk (transport.hpp:64-70, transport.cpp:161-225): the
// photon moves to whichever comes first of its voxel's nearest face, its
// scattering point and the time horizon, losing weight by Beer-Lambert on the
// way (returned in `deposited`; the caller books it in the voxel it left).
// A scattering point deflects it in place (HG + rejection azimuth) and draws
// the next free path; the horizon truncates it; a face lands it exactly on
// the plane and moves the voxel index, unless the next voxel is outside the
// grid or has another refractive index (interface_pending for
// handle_interface).
StepOutcome advance(PhotonState& photon, const VoxelGrid& grid, const SimulationConfig& config, RngStream& stream) {
  const OpticalProperties& m = grid.medium(photon.medium);
  const double h = grid.voxel_size();
  int axis = 0;
  const double to_face = nearest_plane(photon, photon.voxel, h, axis);
  const double to_scatter = m.mus > 0.0 ? photon.remaining_scat / m.mus : kInfD;
  const double ns_per_mm = m.n * (1.0 / kLightSpeedMmPerNs);
  const double time_left = config.tmax_ns - photon.time_ns;
  const double first = std::min(to_face, to_scatter);
  const bool horizon = first * ns_per_mm >= time_left;  // scatter / face lose ties to the horizon
  const double d = horizon ? std::max(0.0, time_left / ns_per_mm) : first;

  StepOutcome out;
  const double w = photon.weight * beer_lambert(m.mua * d);
  out.deposited = photon.weight - w;
  photon.weight = w;
  photon.time_ns += d * ns_per_mm;
  if (horizon) {
    photon.position = photon.position + photon.direction * d;
    photon.time_ns = config.tmax_ns;
    out.kind = StepKind::Terminated;
    return out;
  }
  if (to_scatter <= to_face) {  // the scattering point wins a tie with the face
    photon.position = photon.position + photon.direction * d;
    photon.set_direction(hg_scatter(photon.direction, m.g, stream));
    photon.remaining_scat = unit_length(stream);
    out.kind = StepKind::Scattered;
    return out;
  }
  photon.remaining_scat = std::max(0.0, photon.remaining_scat - d * m.mus);
  const int step = photon.direction[axis] > 0.0 ? 1 : -1;
  Vec3 p = photon.position + photon.direction * d;
  const int iv = axis == 0 ? photon.voxel.x : (axis == 1 ? photon.voxel.y : photon.voxel.z);
  p.ref(axis) = (iv + (step > 0 ? 1 : 0)) * h;  // exactly on the crossed plane
  photon.position = p;
  VoxelIndex next = photon.voxel;
  (axis == 0 ? next.x : (axis == 1 ? next.y : next.z)) += step;
  out.kind = StepKind::CrossedVoxel;
  out.face_axis = axis;
  out.face_step = step;
  out.next_voxel = next;
  out.next_is_exterior = !grid.contains(next);
  out.interface_pending = out.next_is_exterior || grid.medium_at(next).n != m.n;
  if (!out.interface_pending) {
    photon.voxel = next;
    photon.medium = grid.label(next);
  }
  return out;
}

// A pending face from advance() (transport.hpp:72-79, transport.cpp:227-298):
// leaves the grid at once in TerminateAtBoundary mode; otherwise an identity
// index passes (or exits the grid) without a draw, total internal reflection
// mirrors the normal component without a draw, and else one uniform against
// the Fresnel reflectance picks mirror reflection or Snell refraction
// (tangential components scaled by n1/n2, normal component ±cos t,
// renormalised), after which the photon enters the next voxel or exits.
StepOutcome handle_interface(PhotonState& photon, const VoxelGrid& grid, const SimulationConfig& config,
                             const StepOutcome& crossing, RngStream& stream) {
  StepOutcome out;
  out.face_axis = crossing.face_axis;
  out.face_step = crossing.face_step;
  const bool outside = crossing.next_is_exterior;
  auto enter_or_exit = [&]() {
    if (outside) {
      out.kind = StepKind::ExitedDomain;
    } else {
      photon.voxel = crossing.next_voxel;
      photon.medium = grid.label(crossing.next_voxel);
      out.kind = StepKind::CrossedVoxel;
    }
    return out;
  };
  if (outside && config.boundary_mode == BoundaryMode::TerminateAtBoundary) {
    out.kind = StepKind::ExitedDomain;
    return out;
  }
  const double n1 = grid.medium(photon.medium).n;
  const double n2 = outside ? grid.exterior().n : grid.medium_at(crossing.next_voxel).n;
  if (n1 == n2) return enter_or_exit();
  const int axis = crossing.face_axis;
  const double ci = std::fabs(photon.direction[axis]);
  const double eta = n1 / n2;
  const double st2 = eta * eta * std::max(0.0, 1.0 - ci * ci);
  if (st2 > 1.0) {  // total internal reflection
    mirror(photon, axis);
    out.kind = StepKind::Reflected;
    return out;
  }
  const double ct = std::sqrt(1.0 - st2);
  const double rs = (n1 * ci - n2 * ct) / (n1 * ci + n2 * ct);
  const double rp = (n1 * ct - n2 * ci) / (n1 * ct + n2 * ci);
  if (stream.next_unit() < 0.5 * (rs * rs + rp * rp)) {
    mirror(photon, axis);
    out.kind = StepKind::Reflected;
    return out;
  }
  Vec3 d = photon.direction * eta;
  d.ref(axis) = photon.direction[axis] > 0.0 ? ct : -ct;
  photon.set_direction(d.normalized());
  return enter_or_exit();
}

Vec3 hg_scatter(const Vec3& direction, double g, RngStream& stream) {  // transport.cpp:126-147
  const double ct = hg_cos_theta(g, stream.next_unit());
  const double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
  double cp = 0.0, sp = 0.0;
  for (;;) {  // uniform azimuth by rejection from the unit disk (transport.cpp:32-44)
    const double ax = 2.0 * stream.next_unit() - 1.0;
    const double ay = 2.0 * stream.next_unit() - 1.0;
    const double r2 = ax * ax + ay * ay;
    if (r2 > 1e-12 && r2 <= 1.0) {
      const double k = 1.0 / std::sqrt(r2);
      cp = ax * k;
      sp = ay * k;
      break;
    }
  }
  const Vec3& d = direction;
  Vec3 o;
  if (std::fabs(d.z) > 0.99999) {
    o = {st * cp, st * sp, d.z > 0.0 ? ct : -ct};
  } else {
    const double den = std::sqrt(1.0 - d.z * d.z);
    o = {st * (d.x * d.z * cp - d.y * sp) / den + d.x * ct, st * (d.y * d.z * cp + d.x * sp) / den + d.y * ct,
         -st * cp * den + d.z * ct};
  }
  const double n2 = o.dot(o);
  return std::fabs(n2 - 1.0) > 1e-12 ? o * (1.0 / std::sqrt(n2)) : o;
}

bool roulette(PhotonState& photon, const SimulationConfig& config, RngStream& stream) {  // transport.cpp:300-306
  if (!(stream.next_unit() < 1.0 / config.roulette_multiplier)) return false;
  photon.weight *= config.roulette_multiplier;
  return true;
}

// ---- FluenceMap -------------------------------------------------------------
FluenceMap::FluenceMap(VoxelIndex dims, std::uint64_t photon_count, AccumulationMode mode, bool track_counts,
                       int ngates)
    : dims_(dims), photon_count_(photon_count), mode_(mode), quantum_(vmc_quantum_for(photon_count)),
      ngates_(ngates) {
  if (dims.x < 1 || dims.y < 1 || dims.z < 1) throw ValidationError("FluenceMap: dims must be >= 1");
  if (photon_count < 1) throw ValidationError("FluenceMap: photon_count must be >= 1");
  if (ngates < 1) throw ValidationError("FluenceMap: ngates must be >= 1");
  cells_.assign(voxel_count() * static_cast<std::size_t>(ngates), 0);
  if (track_counts) counts_.assign(voxel_count(), 0);
}

void FluenceMap::deposit(std::size_t cell, double dw) {
  const auto q = static_cast<std::int64_t>(std::llround(dw / quantum_));
  if (mode_ == AccumulationMode::SharedAtomic) {
    std::atomic_ref<std::int64_t>(cells_[cell]).fetch_add(q, std::memory_order_relaxed);
    if (!counts_.empty()) std::atomic_ref<std::int64_t>(counts_[cell]).fetch_add(1, std::memory_order_relaxed);
  } else {
    cells_[cell] += q;
    if (!counts_.empty()) ++counts_[cell];
  }
}

void FluenceMap::deposit(const VoxelIndex& v, double dw) {
  if (v.x < 0 || v.y < 0 || v.z < 0 || v.x >= dims_.x || v.y >= dims_.y || v.z >= dims_.z)
    throw VoxelOutOfRange("deposit: voxel outside map");
  if (dw < 0.0) throw ValidationError("deposit: negative weight");
  deposit(static_cast<std::size_t>(v.x) + static_cast<std::size_t>(dims_.x) * (v.y + static_cast<std::size_t>(dims_.y) * v.z), dw);
}

std::int64_t FluenceMap::raw_cell(std::size_t cell) const {
  std::int64_t s = 0;
  for (int g = 0; g < ngates_; ++g) s += cells_[static_cast<std::size_t>(g) * voxel_count() + cell];
  return s;
}

double FluenceMap::value(std::size_t cell) const {
  return normalized_ ? values_[cell] : static_cast<double>(raw_cell(cell)) * quantum_;
}

double FluenceMap::total_deposited() const {
  const std::int64_t s = std::accumulate(cells_.begin(), cells_.end(), std::int64_t{0});
  return static_cast<double>(s) * quantum_;
}

void FluenceMap::add(const FluenceMap& o) {
  if (o.dims_ != dims_ || o.ngates_ != ngates_) throw DimensionMismatch("FluenceMap::add: dims differ");
  if (o.quantum_ != quantum_) throw DimensionMismatch("FluenceMap::add: quantum differs");
  if (normalized_ || o.normalized_) throw AlreadyNormalized("FluenceMap::add: normalized map");
  for (std::size_t i = 0; i < cells_.size(); ++i) cells_[i] += o.cells_[i];
  if (!counts_.empty() && !o.counts_.empty())
    for (std::size_t i = 0; i < counts_.size(); ++i) counts_[i] += o.counts_[i];
}

void FluenceMap::normalize(const VoxelGrid& grid) {
  if (normalized_) throw AlreadyNormalized("FluenceMap::normalize: already normalized");
  if (grid.dims() != dims_) throw DimensionMismatch("FluenceMap::normalize: grid dims differ");
  const double vol = grid.voxel_size() * grid.voxel_size() * grid.voxel_size();
  values_.assign(voxel_count(), 0.0);
  zero_mua_voxels_ = 0;
  for (std::size_t i = 0; i < voxel_count(); ++i) {
    const double mua = grid.medium(grid.labels()[i]).mua;
    if (mua > 0.0)
      values_[i] = static_cast<double>(raw_cell(i)) * quantum_ / (mua * vol * static_cast<double>(photon_count_));
    else
      ++zero_mua_voxels_;
  }
  normalized_ = true;
}

std::vector<float> FluenceMap::to_float_volume() const {
  std::vector<float> v(voxel_count());
  for (std::size_t i = 0; i < v.size(); ++i) v[i] = static_cast<float>(value(i));
  return v;
}

FluenceMap merge(std::span<const FluenceMap> maps) {
  if (maps.empty()) throw DimensionMismatch("merge: empty map list");
  FluenceMap out(maps[0].dims(), maps[0].photon_count(), AccumulationMode::PrivateMerge,
                 maps[0].deposit_count(0) >= 0, maps[0].ngates());
  for (const FluenceMap& m : maps) out.add(m);
  return out;
}

// ---- scheduler --------------------------------------------------------------
std::uint64_t Partition::total() const { return std::accumulate(counts.begin(), counts.end(), std::uint64_t{0}); }

std::optional<Strategy> strategy_from_name(std::string_view n) {
  if (n == "s1" || n == "S1") return Strategy::S1;
  if (n == "s2" || n == "S2") return Strategy::S2;
  if (n == "s3" || n == "S3") return Strategy::S3;
  return std::nullopt;
}

std::string_view strategy_name(Strategy s) { return s == Strategy::S1 ? "s1" : (s == Strategy::S2 ? "s2" : "s3"); }

int thread_count_heuristic(int cores, int per_core) {
  if (cores < 1 || per_core < 1) throw ValidationError("thread_count_heuristic: arguments must be >= 1");
  return cores * per_core;
}

Partition make_partition(std::uint64_t total, std::span<const DeviceProfile> devices, Strategy s) {
  if (devices.empty()) throw ValidationError("partition: no devices");
  const auto p = profiles(devices);
  Partition out;
  out.counts.assign(devices.size(), 0);
  const int code = s == Strategy::S1 ? VMC_STRATEGY_S1 : (s == Strategy::S2 ? VMC_STRATEGY_S2 : VMC_STRATEGY_S3);
  check(vmc_partition(code, total, static_cast<int>(devices.size()), p.data(), out.counts.data()));
  return out;
}

Partition partition_s1(std::uint64_t t, std::span<const DeviceProfile> d) { return make_partition(t, d, Strategy::S1); }
Partition partition_s2(std::uint64_t t, std::span<const DeviceProfile> d) { return make_partition(t, d, Strategy::S2); }
Partition partition_s3(std::uint64_t t, std::span<const DeviceProfile> d) { return make_partition(t, d, Strategy::S3); }

double model_makespan(const Partition& p, std::span<const DeviceProfile> devices) {
  const auto pr = profiles(devices);
  const int n = static_cast<int>(std::min(p.counts.size(), devices.size()));
  return vmc_model_makespan(n, p.counts.data(), pr.data());
}

GroupRunResult run_group_on(int gpu, std::uint64_t first_index, std::uint64_t quota, const Scene& scene,
                            const SimulationConfig& config) {
  config.validate();
  Abi abi(scene, config);
  FluenceMap map(scene.grid.dims(), config.photon_count, config.accumulation_mode, false, config.ngates);
  vmc_disposition tot{};
  const int nm = static_cast<int>(scene.grid.media().size());
  std::vector<unsigned char> det(config.detectors.empty() ? 0 : config.det_capacity * vmc_det_record_bytes(nm));
  std::uint64_t ndet = 0;
  double ms = 0.0;
  check(vmc_run_range(&abi.s, &abi.c, first_index, quota, gpu, map.raw_cells().data(), &tot,
                      det.empty() ? nullptr : det.data(), &ndet, &ms));
  GroupRunResult r{std::move(map), from_quanta(tot), {quota}, ms, {}, ndet};
  if (!config.detectors.empty()) r.detections = unpack_records(det, std::min(ndet, config.det_capacity), nm);
  return r;
}

GroupRunResult run_group_dynamic(std::uint64_t first_index, std::uint64_t quota, int threads, const Scene& scene,
                                 const SimulationConfig& config) {
  if (threads < 1) throw ValidationError("run_group: threads must be >= 1");
  GroupRunResult r = run_group_on(0, first_index, quota, scene, config);
  // one device worker pool: the whole quota is reported in slot 0
  r.per_thread_photons.assign(static_cast<std::size_t>(threads), 0);
  r.per_thread_photons[0] = quota;
  return r;
}

GroupRunResult run_static_split(std::uint64_t first_index, std::uint64_t quota, int threads, const Scene& scene,
                                const SimulationConfig& config) {
  // per-photon streams make static and dynamic claiming bit-identical; the
  // accounting reports the reference's static ceil-sized blocks
  // (scheduler.cpp:295-302)
  GroupRunResult r = run_group_dynamic(first_index, quota, threads, scene, config);
  const std::uint64_t block = (quota + static_cast<std::uint64_t>(threads) - 1) / static_cast<std::uint64_t>(threads);
  for (int t = 0; t < threads; ++t) {
    const std::uint64_t lo = std::min(quota, block * static_cast<std::uint64_t>(t));
    r.per_thread_photons[static_cast<std::size_t>(t)] = std::min(quota, lo + block) - lo;
  }
  return r;
}

namespace {
std::vector<std::pair<std::int64_t, double>> walk_photon(std::uint64_t photon_index, const Scene& scene,
                                                         const SimulationConfig& config, PhotonDisposition& disp) {
  config.validate();
  Abi abi(scene, config);
  std::uint64_t cap = 1u << 16;
  for (;;) {
    std::vector<std::int64_t> cells(cap);
    std::vector<double> dw(cap);
    std::uint64_t n = 0;
    double d[4] = {0, 0, 0, 0};
    check(vmc_simulate_photon(&abi.s, &abi.c, photon_index, 0, cap, cells.data(), dw.data(), &n, d));
    if (n <= cap) {
      disp = {d[0], d[1], d[2], d[3]};
      std::vector<std::pair<std::int64_t, double>> out(n);
      for (std::uint64_t i = 0; i < n; ++i) out[i] = {cells[i], dw[i]};
      return out;
    }
    cap = n;  // longer walk than the first guess: run again with room for all of it
  }
}
}  // namespace

PhotonDisposition simulate_photon(std::uint64_t photon_index, const Scene& scene, const SimulationConfig& config,
                                  FluenceMap& map) {
  PhotonDisposition disp;
  for (const auto& [cell, dw] : walk_photon(photon_index, scene, config, disp))
    map.deposit(static_cast<std::size_t>(cell), dw);
  return disp;
}

PhotonDisposition simulate_photon_trace(std::uint64_t photon_index, const Scene& scene,
                                        const SimulationConfig& config,
                                        std::vector<std::pair<VoxelIndex, double>>& deposits) {
  PhotonDisposition disp;
  const std::int64_t nx = scene.grid.nx(), nxy = nx * scene.grid.ny();
  for (const auto& [cell, dw] : walk_photon(photon_index, scene, config, disp))
    deposits.push_back({VoxelIndex{static_cast<int>(cell % nx), static_cast<int>((cell % nxy) / nx),
                                   static_cast<int>(cell / nxy)},
                        dw});
  return disp;
}

double static_split_makespan(std::span<const double> costs, int threads) {
  if (threads < 1) throw ValidationError("threads must be >= 1");
  const std::size_t block = (costs.size() + threads - 1) / threads;
  double worst = 0.0;
  for (std::size_t b = 0; b < costs.size(); b += block)
    worst = std::max(worst, std::accumulate(costs.begin() + b, costs.begin() + std::min(costs.size(), b + block), 0.0));
  return worst;
}

double dynamic_makespan(std::span<const double> costs, int threads) {
  if (threads < 1) throw ValidationError("threads must be >= 1");
  std::priority_queue<double, std::vector<double>, std::greater<double>> free_at;
  for (int t = 0; t < threads; ++t) free_at.push(0.0);
  double worst = 0.0;
  for (double c : costs) {
    const double done = free_at.top() + c;
    free_at.pop();
    free_at.push(done);
    worst = std::max(worst, done);
  }
  return worst;
}

Calibration calibrate(const DeviceProfile& device, std::uint64_t n1, std::uint64_t n2, const Scene& scene,
                      const SimulationConfig& config, int threads, std::uint64_t noise_seed) {
  if (!(n2 > n1 && n1 >= 1)) throw ValidationError("calibrate: need n2 > n1 >= 1");
  double t1, t2;
  if (device.kind == DeviceKind::CudaGpu) {
    SimulationConfig pilot = config;
    pilot.photon_count = n2;
    t1 = run_group_on(device.gpu, 0, n1, scene, pilot).wall_ms;
    t2 = run_group_on(device.gpu, 0, n2, scene, pilot).wall_ms;
  } else if (device.kind == DeviceKind::Simulated) {
    t1 = device.a * static_cast<double>(n1) + device.t0;
    t2 = device.a * static_cast<double>(n2) + device.t0;
    if (device.jitter_sigma > 0.0) {
      RngStream noise(noise_seed, 0x706c6f74);
      auto factor = [&] {
        const double u1 = std::max(noise.next_unit(), 1e-300), u2 = noise.next_unit();
        return std::exp(device.jitter_sigma * std::sqrt(-2.0 * std::log(u1)) *
                        std::cos(2.0 * 3.14159265358979323846 * u2));
      };
      t1 *= factor();
      t2 *= factor();
    }
  } else {  // a host worker pool of the reference: its pilots run on the B200 executor
    SimulationConfig pilot = config;
    pilot.photon_count = n2;
    t1 = run_group_on(0, 0, n1, scene, pilot).wall_ms;
    t2 = run_group_on(0, 0, n2, scene, pilot).wall_ms;
  }
  (void)threads;
  if (t2 <= t1) throw NonPositiveSlope("calibrate: T2 <= T1; increase n2 or rerun");
  Calibration c;
  c.a = (t2 - t1) / static_cast<double>(n2 - n1);
  c.t0 = std::max(0.0, t1 - c.a * static_cast<double>(n1));
  return c;
}

MultiDeviceResult run_multi_device(std::uint64_t total, std::span<const DeviceProfile> devices, Strategy strategy,
                                   const Scene& scene, const SimulationConfig& config, int threads_per_device) {
  (void)threads_per_device;
  if (devices.empty()) throw ValidationError("run_multi_device: no devices");
  Partition part = make_partition(total, devices, strategy);
  SimulationConfig cfg = config;
  cfg.photon_count = total;  // shared quantum (reference scheduler.cpp:412-413)
  cfg.validate();
  Abi abi(scene, cfg);
  FluenceMap map(scene.grid.dims(), total, AccumulationMode::PrivateMerge, false, cfg.ngates);
  // every device's range runs on a B200: CudaGpu devices on their own GPU, the
  // reference's host pools and simulated devices on GPU 0 (a simulated device
  // keeps the reference's modelled wall time a*n + t0, scheduler.cpp:441-443)
  std::vector<int> gpus;
  for (const DeviceProfile& d : devices) gpus.push_back(d.kind == DeviceKind::CudaGpu ? d.gpu : 0);
  vmc_disposition tot{};
  const int nm = static_cast<int>(scene.grid.media().size());
  std::vector<unsigned char> det(cfg.detectors.empty() ? 0 : cfg.det_capacity * vmc_det_record_bytes(nm));
  std::uint64_t ndet = 0;
  std::vector<double> ms(devices.size(), 0.0);
  double red = 0.0;
  check(vmc_run_multi(&abi.s, &abi.c, static_cast<int>(devices.size()), gpus.data(), part.counts.data(),
                      map.raw_cells().data(), &tot, det.empty() ? nullptr : det.data(), &ndet, ms.data(), &red));
  MultiDeviceResult r{std::move(map), from_quanta(tot), part, {}, 0.0, red, {}, ndet};
  for (std::size_t i = 0; i < devices.size(); ++i) {
    const double wall = devices[i].kind == DeviceKind::Simulated
                            ? devices[i].a * static_cast<double>(part.counts[i]) + devices[i].t0
                            : ms[i];
    r.devices.push_back({devices[i].name, part.counts[i], part.counts[i] ? wall : 0.0});
    r.makespan_ms = std::max(r.makespan_ms, r.devices.back().wall_ms);
  }
  r.makespan_ms += red;
  if (!cfg.detectors.empty()) r.detections = unpack_records(det, std::min(ndet, cfg.det_capacity), nm);
  return r;
}

}  // namespace voxmc
