// voxmc_config.cpp — the C++ run front door of the drop-in: JSON run
// configuration and device roster, scene hash, calibration cache, run_pipeline
// and its report (reference proj/core/include/voxmc/config.hpp:14-75), and the
// raw volume export (volume_io.hpp:13-37). Host code over the B200 executors in
// voxmc_api.cpp; the keys and file formats are those of the Python front door
// (paper_1711_03244_b200/pipeline.py, volume_io.py), so configs, calibration
// caches and volumes are interchangeable between the two.
//
// JSON: nlohmann/json (the reference's own dependency, config.cpp), from the
// copy the image vendors under cudnn_frontend/thirdparty (build.py -I).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <thread>

#include <nlohmann/json.hpp>

#include "../../include/vmc.h"
#include "voxmc/config.hpp"
#include "voxmc/volume_io.hpp"

namespace voxmc {

using json = nlohmann::json;

// ---- volume_io ------------------------------------------------------------
std::uint64_t fnv1a64(const void* data, std::size_t size) { return vmc_fnv1a64(data, size); }

std::uint64_t fnv1a64(std::span<const std::byte> bytes) { return vmc_fnv1a64(bytes.data(), bytes.size()); }

void write_volume(const FluenceMap& map, double voxel_size_mm, std::uint64_t seed,
                  const std::filesystem::path& path) {
  const std::vector<float> vol = map.to_float_volume();
  const std::size_t bytes = vol.size() * sizeof(float);
  const std::uint64_t sum = fnv1a64(vol.data(), bytes);
  {
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw IoError("write_volume: cannot open " + path.string());
    f.write(reinterpret_cast<const char*>(vol.data()), static_cast<std::streamsize>(bytes));  // little endian host
    if (!f) throw IoError("write_volume: short write to " + path.string());
  }
  const VoxelIndex d = map.dims();
  const json side = {{"dims", {d.x, d.y, d.z}},
                     {"voxel_size_mm", voxel_size_mm},
                     {"photon_count", map.photon_count()},
                     {"normalized", map.normalized()},
                     {"seed", seed},
                     {"checksum", sum},
                     {"ordering", "x-fastest"}};
  std::ofstream s(path.string() + ".json", std::ios::trunc);
  if (!s) throw IoError("write_volume: cannot open " + path.string() + ".json");
  s << side.dump(2) << "\n";
}

VolumeData read_volume(const std::filesystem::path& path) {
  const std::string side_path = path.string() + ".json";
  std::ifstream s(side_path);
  if (!s) throw IoError("read_volume: missing sidecar " + side_path);
  json side;
  try {
    s >> side;
  } catch (const json::exception& e) {
    throw ParseError(std::string("read_volume: bad sidecar: ") + e.what());
  }
  VolumeData v;
  try {
    v.dims = {side.at("dims").at(0).get<int>(), side.at("dims").at(1).get<int>(), side.at("dims").at(2).get<int>()};
    v.voxel_size_mm = side.at("voxel_size_mm").get<double>();
    v.photon_count = side.at("photon_count").get<std::uint64_t>();
    v.normalized = side.at("normalized").get<bool>();
    v.seed = side.at("seed").get<std::uint64_t>();
    v.checksum = side.at("checksum").get<std::uint64_t>();
  } catch (const json::exception& e) {
    throw ParseError(std::string("read_volume: bad sidecar: ") + e.what());
  }
  const std::size_t n = static_cast<std::size_t>(v.dims.x) * v.dims.y * v.dims.z;
  v.values.resize(n);
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("read_volume: cannot open " + path.string());
  f.read(reinterpret_cast<char*>(v.values.data()), static_cast<std::streamsize>(n * sizeof(float)));
  if (static_cast<std::size_t>(f.gcount()) != n * sizeof(float)) throw IoError("read_volume: short read");
  if (fnv1a64(v.values.data(), n * sizeof(float)) != v.checksum)
    throw IoError("read_volume: checksum mismatch for " + path.string());
  return v;
}

// ---- config ----------------------------------------------------------------
namespace {

std::string slurp(const std::filesystem::path& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open " + path.string());
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

json parse_json(const std::string& text, const char* what) {
  try {
    return json::parse(text);
  } catch (const json::parse_error& e) {
    throw ParseError(std::string(what) + ": " + e.what());
  }
}

Vec3 vec3(const json& j, const char* what) {
  if (!j.is_array() || j.size() != 3) throw ParseError(std::string(what) + ": expected an array of 3 numbers");
  return {j[0].get<double>(), j[1].get<double>(), j[2].get<double>()};
}

OpticalProperties medium_of(const json& m) {
  return {m.at("mua").get<double>(), m.at("mus").get<double>(), m.at("g").get<double>(), m.at("n").get<double>()};
}

DeviceProfile device_of(const json& j) {
  DeviceProfile d;
  d.name = j.at("name").get<std::string>();
  d.cores = j.value("cores", 1);
  d.a = j.value("a", 0.0);
  d.t0 = j.value("t0", 0.0);
  d.jitter_sigma = j.value("jitter_sigma", 0.0);
  d.gpu = j.value("gpu", 0);
  if (d.cores < 1) throw ValidationError("device " + d.name + ": cores must be >= 1");
  const std::string kind = j.value("kind", std::string("simulated"));
  if (kind == "simulated") {
    d.kind = DeviceKind::Simulated;
  } else if (kind == "real" || kind == "worker-pool") {
    d.kind = DeviceKind::RealWorkerPool;
  } else if (kind == "gpu") {
    d.kind = DeviceKind::CudaGpu;
  } else {
    throw ParseError("device " + d.name + ": unknown kind '" + kind + "'");
  }
  if (d.kind == DeviceKind::Simulated && !(d.a > 0.0))
    throw ValidationError("device " + d.name + ": simulated devices need a > 0");
  if (d.t0 < 0.0) throw ValidationError("device " + d.name + ": t0 must be >= 0");
  return d;
}

std::vector<DeviceProfile> roster_of(const json& j) {
  if (!j.is_array() || j.empty()) throw ParseError("roster: expected a non-empty array");
  std::vector<DeviceProfile> out;
  for (const json& d : j) out.push_back(device_of(d));
  return out;
}

// explicit grid: dims, voxel size, media (exterior first), optional raw
// labels file and spherical inclusion (voxel-centre test)
VoxelGrid grid_of(const json& root, const std::filesystem::path& base) {
  const json& jg = root.at("grid");
  const json& jm = root.at("media");
  if (!jm.is_array() || jm.size() < 2)
    throw ParseError("media: expected an array with the exterior medium plus at least one more");
  std::vector<OpticalProperties> media;
  for (const json& m : jm) media.push_back(medium_of(m));
  const int nx = jg.at("dims").at(0).get<int>(), ny = jg.at("dims").at(1).get<int>(),
            nz = jg.at("dims").at(2).get<int>();
  const double h = jg.contains("voxel_size_mm") ? jg["voxel_size_mm"].get<double>() : jg.value("voxel_size", 1.0);
  if (nx < 1 || ny < 1 || nz < 1 || !(h > 0.0)) throw ValidationError("grid: dims must be >= 1 and voxel_size > 0");
  const std::size_t nvox = static_cast<std::size_t>(nx) * ny * nz;
  std::vector<std::uint8_t> labels(nvox, 1);
  if (root.contains("labels_file")) {
    std::filesystem::path p = root["labels_file"].get<std::string>();
    if (p.is_relative()) p = base / p;
    std::ifstream f(p, std::ios::binary);
    if (!f) throw IoError("cannot open " + p.string());
    f.read(reinterpret_cast<char*>(labels.data()), static_cast<std::streamsize>(nvox));
    if (static_cast<std::size_t>(f.gcount()) != nvox || f.peek() != std::char_traits<char>::eof())
      throw ValidationError("labels_file: size does not match grid.dims");
  }
  if (root.contains("sphere")) {
    const json& js = root["sphere"];
    const Vec3 c = vec3(js.at("center"), "sphere.center");
    const double r = js.at("radius").get<double>();
    int lbl;
    if (js.contains("medium")) {
      media.push_back(medium_of(js["medium"]));
      lbl = static_cast<int>(media.size()) - 1;
    } else {
      lbl = js.value("label", static_cast<int>(media.size()) - 1);
    }
    for (int z = 0; z < nz; ++z)
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) {
          const double dx = (x + 0.5) * h - c.x, dy = (y + 0.5) * h - c.y, dz = (z + 0.5) * h - c.z;
          if (dx * dx + dy * dy + dz * dz <= r * r)
            labels[static_cast<std::size_t>(x) + static_cast<std::size_t>(nx) * (y + static_cast<std::size_t>(ny) * z)] =
                static_cast<std::uint8_t>(lbl);
        }
  }
  return VoxelGrid({nx, ny, nz}, h, std::move(labels), std::move(media));
}

Source source_of(const json& js) {
  Source s;
  s.position = vec3(js.at("position"), "source.position");
  if (js.contains("direction")) s.direction = vec3(js["direction"], "source.direction").normalized();
  s.isotropic = js.value("isotropic", false);
  return s;
}

RunSetup setup_of(const json& root, const std::filesystem::path& base) {
  std::optional<BenchmarkSetup> preset;
  if (root.contains("benchmark")) {
    const std::string name = root["benchmark"].get<std::string>();
    const std::optional<Benchmark> b = benchmark_from_name(name);
    if (!b) throw ParseError("unknown benchmark '" + name + "'");
    preset = benchmark_preset(*b);
  }
  std::optional<VoxelGrid> grid;
  std::optional<Source> source;
  if (root.contains("grid")) grid = grid_of(root, base);
  if (root.contains("source")) source = source_of(root["source"]);
  if (!preset && (!grid || !source))
    throw ParseError("config: need either \"benchmark\" or explicit \"grid\"+\"media\"+\"source\"");
  SimulationConfig cfg = preset ? preset->config : SimulationConfig{};
  if (root.contains("photons")) {
    const long long p = root["photons"].get<long long>();
    if (p < 1) throw ValidationError("photons must be >= 1");
    cfg.photon_count = static_cast<std::uint64_t>(p);
  }
  cfg.master_seed = root.value("seed", cfg.master_seed);
  if (root.contains("mode")) {
    const std::string m = root["mode"].get<std::string>();
    if (m != "atomic" && m != "merge") throw ValidationError("mode must be 'atomic' or 'merge'");
    cfg.accumulation_mode = m == "atomic" ? AccumulationMode::SharedAtomic : AccumulationMode::PrivateMerge;
  }
  if (root.contains("boundary")) {
    const std::string b = root["boundary"].get<std::string>();
    if (b != "terminate" && b != "reflect") throw ValidationError("boundary must be 'terminate' or 'reflect'");
    cfg.boundary_mode = b == "terminate" ? BoundaryMode::TerminateAtBoundary : BoundaryMode::ReflectAtMismatch;
  }
  cfg.tmax_ns = root.value("tmax_ns", cfg.tmax_ns);
  cfg.roulette_threshold = root.value("roulette_threshold", cfg.roulette_threshold);
  cfg.roulette_multiplier = root.value("roulette_multiplier", cfg.roulette_multiplier);
  cfg.workgroup_size = root.value("workgroup_size", cfg.workgroup_size);
  cfg.ngates = root.value("gates", cfg.ngates);
  if (root.contains("precision")) {
    const std::string p = root["precision"].get<std::string>();
    if (p != "fp32" && p != "fp64") throw ValidationError("precision must be 'fp32' or 'fp64'");
    cfg.precision = p == "fp64" ? Precision::FP64 : Precision::FP32;
  }
  if (root.contains("detectors")) {
    cfg.detectors.clear();
    for (const json& d : root["detectors"])
      cfg.detectors.push_back({vec3(d.at("position"), "detector.position"), d.at("radius").get<double>()});
    cfg.det_capacity = root.value("det_capacity", std::uint64_t{1} << 20);
  }
  cfg.validate();
  RunSetup setup{Scene{grid ? *grid : preset->grid, source ? *source : preset->source}, cfg, {}, Strategy::S1,
                 root.value("output", std::string()), root.value("report", std::string())};
  if (root.contains("devices")) {
    const json& jd = root["devices"];
    if (jd.is_string()) {
      std::filesystem::path p = jd.get<std::string>();
      setup.devices = load_roster(p.is_relative() ? base / p : p);
    } else if (jd.is_array()) {
      setup.devices = roster_of(jd);
    } else {
      throw ParseError("devices: expected roster path or inline array");
    }
  }
  if (root.contains("strategy")) {
    const std::optional<Strategy> s = strategy_from_name(root["strategy"].get<std::string>());
    if (!s) throw ValidationError("strategy must be one of s1, s2, s3");
    setup.strategy = *s;
  }
  return setup;
}

// json type errors (a string where a number belongs, a missing key) are
// configuration errors; ValidationError / ParseError / IoError pass through
template <class F>
auto as_parse_error(const char* what, F&& f) {
  try {
    return f();
  } catch (const json::exception& e) {
    throw ParseError(std::string(what) + ": " + e.what());
  }
}

void append(std::vector<unsigned char>& out, const void* p, std::size_t n) {
  const auto* b = static_cast<const unsigned char*>(p);
  out.insert(out.end(), b, b + n);
}

}  // namespace

RunSetup parse_config_text(const std::string& json_text) {
  const json root = parse_json(json_text, "config");
  return as_parse_error("config", [&] { return setup_of(root, std::filesystem::current_path()); });
}

RunSetup parse_config(const std::filesystem::path& path) {
  const json root = parse_json(slurp(path), "config");
  return as_parse_error("config", [&] { return setup_of(root, std::filesystem::absolute(path).parent_path()); });
}

std::vector<DeviceProfile> parse_roster_text(const std::string& json_text) {
  const json j = parse_json(json_text, "roster");
  return as_parse_error("roster", [&] { return roster_of(j); });
}

std::vector<DeviceProfile> load_roster(const std::filesystem::path& path) { return parse_roster_text(slurp(path)); }

DeviceProfile host_device(int threads) {
  DeviceProfile d;
  d.name = "host";
  d.cores = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  d.kind = DeviceKind::RealWorkerPool;
  return d;
}

std::uint64_t scene_hash(const Scene& scene, const SimulationConfig& config) {
  // the byte layout of pipeline.scene_hash: dims (int32 x3), voxel size (f64),
  // labels, media (f64 x4 each), source position / direction (f64 x3),
  // isotropic (1 byte), boundary mode (int32), horizon (f64), gates (int32)
  const VoxelGrid& g = scene.grid;
  std::vector<unsigned char> b;
  const std::int32_t dims[3] = {g.nx(), g.ny(), g.nz()};
  append(b, dims, sizeof dims);
  const double h = g.voxel_size();
  append(b, &h, sizeof h);
  append(b, g.labels().data(), g.labels().size());
  for (const OpticalProperties& m : g.media()) {
    const double v[4] = {m.mua, m.mus, m.g, m.n};
    append(b, v, sizeof v);
  }
  const double pos[3] = {scene.source.position.x, scene.source.position.y, scene.source.position.z};
  const double dir[3] = {scene.source.direction.x, scene.source.direction.y, scene.source.direction.z};
  append(b, pos, sizeof pos);
  append(b, dir, sizeof dir);
  const unsigned char iso = scene.source.isotropic ? 1 : 0;
  append(b, &iso, 1);
  const std::int32_t mode = config.boundary_mode == BoundaryMode::ReflectAtMismatch ? VMC_BOUNDARY_REFLECT
                                                                                      : VMC_BOUNDARY_TERMINATE;
  append(b, &mode, sizeof mode);
  append(b, &config.tmax_ns, sizeof config.tmax_ns);
  const std::int32_t gates = config.ngates;
  append(b, &gates, sizeof gates);
  return fnv1a64(b.data(), b.size());
}

std::string report_to_json(const RunReport& r) {
  json devs = json::array();
  for (const DeviceReport& d : r.devices) devs.push_back({{"name", d.name}, {"photons", d.photons}, {"wall_ms", d.wall_ms}});
  const json j = {{"devices", devs},
                  {"makespan_ms", r.makespan_ms},
                  {"throughput_photons_per_ms", r.throughput_photons_per_ms},
                  {"conservation_residual", r.conservation_residual},
                  {"strategy", r.strategy},
                  {"photon_count", r.photon_count},
                  {"seed", r.seed},
                  {"mode", r.mode},
                  {"boundary", r.boundary}};
  return j.dump(2);
}

RunResult run_pipeline(const RunSetup& setup, int threads_per_device) {
  setup.config.validate();
  std::vector<DeviceProfile> devices = setup.devices;
  if (devices.empty()) devices.push_back(host_device(threads_per_device));  // runs on GPU 0
  const std::uint64_t n = setup.config.photon_count;
  MultiDeviceResult m =
      run_multi_device(n, devices, setup.strategy, setup.scene, setup.config, std::max(1, threads_per_device));
  // energy audit in the accumulator's integer quanta (deposited + escaped +
  // killed + truncated == n photons, config.cpp:316-319)
  const PhotonDisposition& t = m.totals;
  const double residual = (t.deposited + t.escaped + t.killed + t.truncated - static_cast<double>(n)) / n;
  RunReport rep;
  for (const DeviceRunResult& d : m.devices) rep.devices.push_back({d.name, d.photons, d.wall_ms});
  rep.makespan_ms = m.makespan_ms;
  rep.throughput_photons_per_ms = m.makespan_ms > 0.0 ? n / m.makespan_ms : 0.0;
  rep.conservation_residual = residual;
  rep.strategy = std::string(strategy_name(setup.strategy));
  rep.photon_count = n;
  rep.seed = setup.config.master_seed;
  rep.mode = setup.config.accumulation_mode == AccumulationMode::SharedAtomic ? "atomic" : "merge";
  rep.boundary = setup.config.boundary_mode == BoundaryMode::TerminateAtBoundary ? "terminate" : "reflect";
  if (std::fabs(residual) > 1e-6)
    throw ValidationError("energy conservation violated: relative residual " + std::to_string(residual));
  if (!setup.output_path.empty())
    write_volume(m.map, setup.scene.grid.voxel_size(), setup.config.master_seed, setup.output_path);
  if (!setup.report_path.empty()) {
    std::ofstream f(setup.report_path, std::ios::trunc);
    if (!f) throw IoError("cannot open " + setup.report_path);
    f << report_to_json(rep) << "\n";
  }
  return RunResult{std::move(m.map), std::move(rep)};
}

namespace {
json read_cache(const std::filesystem::path& cache) {
  std::ifstream f(cache);
  if (!f) return json::object();
  try {
    json j;
    f >> j;
    return j.is_object() ? j : json::object();
  } catch (const json::exception&) {
    return json::object();
  }
}

std::string cache_key(const std::string& device, std::uint64_t key) {
  char hex[17];
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(key));
  return device + "@" + hex;
}
}  // namespace

std::optional<Calibration> cache_lookup(const std::filesystem::path& cache, const std::string& device_name,
                                        std::uint64_t scene_key) {
  const json j = read_cache(cache);
  const auto it = j.find(cache_key(device_name, scene_key));
  if (it == j.end()) return std::nullopt;
  try {
    return Calibration{it->at("a").get<double>(), it->at("t0").get<double>()};
  } catch (const json::exception&) {
    return std::nullopt;
  }
}

void cache_store(const std::filesystem::path& cache, const std::string& device_name, std::uint64_t scene_key,
                 const Calibration& cal) {
  json j = read_cache(cache);
  j[cache_key(device_name, scene_key)] = {{"a", cal.a}, {"t0", cal.t0}};
  std::ofstream f(cache, std::ios::trunc);
  if (!f) throw IoError("cannot open " + cache.string());
  f << j.dump(2) << "\n";
}

}  // namespace voxmc
