// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A C-ABI veneer over the UNMODIFIED reference library (voxmc), compiled from
// the sources under /root/reference/proj/core/src with -Dvoxmc=voxmc_ref by
// oracle/Makefile, so that Python tests, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg can call the reference's own
// code path:
//   ref_run_group  -> voxmc::run_group_dynamic   (proj/core/src/scheduler.cpp:321-324)
//   ref_run_multi  -> voxmc::run_multi_device    (proj/core/src/scheduler.cpp:395-451)
//   ref_trace      -> voxmc::simulate_photon_trace (proj/core/src/transport.cpp:368-380)
//   ref_partition  -> voxmc::make_partition      (proj/core/src/scheduler.cpp:244-251)
//   ref_rng_kat    -> voxmc::RngStream           (proj/core/include/voxmc/rng.hpp:11-35)
//   ref_run_pipeline -> voxmc::run_pipeline      (proj/core/src/config.cpp:288-321; the
//                     reference's own front door, timed as the CPU baseline)
//   ref_normalize  -> voxmc::FluenceMap::normalize + to_float_volume
//                     (proj/core/src/fluence.cpp:62-90; the checker of K4)
// plus ONE derived oracle, ref_walk, for the features the reference lacks
// (time gates, disk detectors, per-photon RNG draw counts). ref_walk re-drives
// the reference's public step API (launch / advance / handle_interface /
// roulette, proj/core/include/voxmc/transport.hpp:45-83) in the order of
// run_photon (transport.cpp:310-358); with one gate and no detectors it
// produces the same per-photon dispositions and deposits as
// simulate_photon_trace (checked by tests/test_oracle_ref.py).
//
// Nothing here is copied from the reference; it only calls it.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "voxmc/config.hpp"
#include "voxmc/fluence.hpp"
#include "voxmc/oracles.hpp"
#include "voxmc/scheduler.hpp"
#include "voxmc/transport.hpp"
#include "vmc.h"

namespace R = voxmc_ref;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const R::ValidationError& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

R::Scene make_scene(const vmc_scene* s) {
  const std::size_t nvox = static_cast<std::size_t>(s->nx) * s->ny * s->nz;
  std::vector<std::uint8_t> labels(s->labels, s->labels + nvox);
  std::vector<R::OpticalProperties> media(static_cast<std::size_t>(s->nmedia));
  for (int m = 0; m < s->nmedia; ++m) {
    media[m] = {s->media[4 * m + 0], s->media[4 * m + 1], s->media[4 * m + 2], s->media[4 * m + 3]};
  }
  R::VoxelGrid grid({s->nx, s->ny, s->nz}, s->voxel_mm, std::move(labels), std::move(media));
  R::Source src;
  src.position = {s->src_pos[0], s->src_pos[1], s->src_pos[2]};
  src.direction = {s->src_dir[0], s->src_dir[1], s->src_dir[2]};
  src.isotropic = s->isotropic != 0;
  return R::Scene{std::move(grid), src};
}

R::SimulationConfig make_config(const vmc_config* c) {
  R::SimulationConfig cfg;
  cfg.photon_count = c->photon_count;
  cfg.master_seed = c->master_seed;
  cfg.accumulation_mode = c->accumulation_mode == VMC_ACCUM_SHARED_ATOMIC
                              ? R::AccumulationMode::SharedAtomic
                              : R::AccumulationMode::PrivateMerge;
  cfg.boundary_mode = c->boundary_mode == VMC_BOUNDARY_REFLECT ? R::BoundaryMode::ReflectAtMismatch
                                                               : R::BoundaryMode::TerminateAtBoundary;
  cfg.tmax_ns = c->tmax_ns;
  cfg.roulette_threshold = c->roulette_threshold;
  cfg.roulette_multiplier = c->roulette_multiplier;
  cfg.workgroup_size = c->workgroup_size > 0 ? c->workgroup_size : 64;
  return cfg;
}

void put_disp(const R::PhotonDisposition& d, double* out4) {
  if (!out4) return;
  out4[0] = d.deposited;
  out4[1] = d.escaped;
  out4[2] = d.killed;
  out4[3] = d.truncated;
}

// Number of next_u64 draws separating a fresh (seed, id) stream from `end`.
std::uint32_t draws_between(std::uint64_t seed, std::uint64_t id, const R::RngStream& end) {
  R::RngStream probe(seed, id);
  std::uint32_t n = 0;
  while (!(probe.state_lo() == end.state_lo() && probe.state_hi() == end.state_hi())) {
    probe.next_u64();
    if (++n > (1u << 26)) return 0xffffffffu;
  }
  return n;
}

struct WalkSink {
  // outputs (any may be null)
  std::int64_t* cells = nullptr;   // [ngates * V]
  std::int64_t* counts = nullptr;  // [V] deposit counts
  double inv_quantum = 0.0;
};

struct DetHit {
  std::uint64_t photon;
  std::uint32_t det;
  std::uint32_t nscat;
  float w;
  float t;
  std::vector<float> ppath;
};

// One photon through the reference's public step API, mirroring run_photon
// (transport.cpp:310-358) and adding the gate / detector / draw-count sinks.
R::PhotonDisposition walk_one(std::uint64_t idx, const R::Scene& scene,
                              const R::SimulationConfig& cfg, const vmc_config* c,
                              const WalkSink& sink, vmc_photon_trace* tr,
                              std::vector<DetHit>* hits) {
  const R::VoxelGrid& grid = scene.grid;
  const int ngates = c->ngates > 0 ? c->ngates : 1;
  const double gate_w = cfg.tmax_ns / ngates;
  const std::size_t nvox = grid.voxel_count();
  const int nmedia = static_cast<int>(grid.media().size());
  std::vector<double> ppath(static_cast<std::size_t>(std::max(0, nmedia - 1)), 0.0);

  R::RngStream stream(cfg.master_seed, idx);
  R::PhotonState ph = R::launch(scene.source, grid, stream);
  R::PhotonDisposition disp;
  std::uint32_t steps = 0, scatters = 0, flags = 0;

  for (;;) {
    const R::VoxelIndex at = ph.voxel;
    const std::uint8_t med_at = ph.medium;
    const double t_before = ph.time_ns;
    const R::Vec3 p_before = ph.position;
    const R::StepOutcome out = R::advance(ph, grid, cfg, stream);
    ++steps;
    if (hits && med_at >= 1) {
      // Path length of this step: every step is a straight segment from
      // p_before to the post-step position (before any reflection flip).
      const R::Vec3 dp = ph.position - p_before;
      ppath[med_at - 1] += std::sqrt(dp.dot(dp));
    }
    if (out.deposited != 0.0) {
      const std::size_t cell = grid.linear(at);
      int gate = static_cast<int>(std::floor(t_before / gate_w));
      gate = std::min(std::max(gate, 0), ngates - 1);
      if (sink.cells) sink.cells[static_cast<std::size_t>(gate) * nvox + cell] +=
          static_cast<std::int64_t>(std::llround(out.deposited * sink.inv_quantum));
      if (sink.counts) sink.counts[cell] += 1;
      disp.deposited += out.deposited;
    }
    bool done = false;
    switch (out.kind) {
      case R::StepKind::Terminated:
        disp.truncated += ph.weight;
        flags |= 4u;
        done = true;
        break;
      case R::StepKind::Scattered:
        ++scatters;
        if (ph.weight < cfg.roulette_threshold) {
          const double before = ph.weight;
          if (!R::roulette(ph, cfg, stream)) {
            disp.killed += before;
            flags |= 2u;
            done = true;
            break;
          }
          disp.killed += before - ph.weight;
        }
        break;
      case R::StepKind::CrossedVoxel:
        if (out.interface_pending) {
          const R::StepOutcome res = R::handle_interface(ph, grid, cfg, out, stream);
          if (res.kind == R::StepKind::ExitedDomain) {
            disp.escaped += ph.weight;
            flags |= 1u;
            done = true;
            if (hits) {
              for (int k = 0; k < c->ndet; ++k) {
                const double* dd = c->det + 4 * k;
                const double dx = ph.position.x - dd[0], dy = ph.position.y - dd[1],
                             dz = ph.position.z - dd[2];
                if (dx * dx + dy * dy + dz * dz <= dd[3] * dd[3]) {
                  DetHit h{idx, static_cast<std::uint32_t>(k), scatters,
                           static_cast<float>(ph.weight), static_cast<float>(ph.time_ns), {}};
                  h.ppath.assign(ppath.begin(), ppath.end());
                  hits->push_back(std::move(h));
                  flags |= 8u;
                  break;
                }
              }
            }
          }
        }
        break;
      default:
        break;
    }
    if (done) break;
  }
  if (tr) {
    tr->draws = draws_between(cfg.master_seed, idx, stream);
    tr->steps = steps;
    tr->scatters = scatters;
    tr->flags = flags;
    tr->deposited = disp.deposited;
    tr->escaped = disp.escaped;
    tr->killed = disp.killed;
    tr->truncated = disp.truncated;
  }
  return disp;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

std::uint64_t ref_mix64(std::uint64_t z) { return R::mix64(z); }

int ref_rng_kat(std::uint64_t seed, std::uint64_t id, int n, std::uint64_t* out,
                std::uint64_t* state2, double* first_unit) {
  return guarded([&] {
    R::RngStream s(seed, id);
    if (state2) {
      state2[0] = s.state_lo();
      state2[1] = s.state_hi();
    }
    if (first_unit) {
      R::RngStream u(seed, id);
      *first_unit = u.next_unit();
    }
    for (int i = 0; i < n; ++i) out[i] = s.next_u64();
  });
}

double ref_quantum_for(std::uint64_t n) {
  R::FluenceMap m({1, 1, 1}, n);
  return m.quantum();
}

// run_group_dynamic over [first, first+count) with `threads` workers.
int ref_run_group(const vmc_scene* s, const vmc_config* c, std::uint64_t first,
                  std::uint64_t count, int threads, std::int64_t* cells_out, double* disp4,
                  double* wall_ms) {
  return guarded([&] {
    const R::Scene scene = make_scene(s);
    const R::SimulationConfig cfg = make_config(c);
    R::GroupRunResult r = R::run_group_dynamic(first, count, threads, scene, cfg);
    if (cells_out) {
      for (std::size_t i = 0; i < r.map.voxel_count(); ++i) cells_out[i] = r.map.raw_cell(i);
    }
    put_disp(r.totals, disp4);
    if (wall_ms) *wall_ms = r.wall_ms;
  });
}

// run_multi_device with `ndev` simulated devices (the reference's own fake
// backend, scheduler.hpp:16-28): real physics on host threads.
int ref_run_multi(const vmc_scene* s, const vmc_config* c, std::uint64_t total, int ndev,
                  const vmc_device_profile* profs, int strategy, int threads_per_device,
                  std::int64_t* cells_out, double* disp4, std::uint64_t* counts_out) {
  return guarded([&] {
    const R::Scene scene = make_scene(s);
    const R::SimulationConfig cfg = make_config(c);
    std::vector<R::DeviceProfile> devs(static_cast<std::size_t>(ndev));
    for (int i = 0; i < ndev; ++i) {
      devs[i].name = "dev" + std::to_string(i);
      devs[i].cores = profs[i].cores;
      devs[i].a = profs[i].a;
      devs[i].t0 = profs[i].t0;
      devs[i].kind = R::DeviceKind::Simulated;
    }
    const R::Strategy st = strategy == 1 ? R::Strategy::S1
                           : strategy == 2 ? R::Strategy::S2
                                           : R::Strategy::S3;
    R::MultiDeviceResult r = R::run_multi_device(total, devs, st, scene, cfg, threads_per_device);
    if (cells_out) {
      for (std::size_t i = 0; i < r.map.voxel_count(); ++i) cells_out[i] = r.map.raw_cell(i);
    }
    if (counts_out) {
      for (int i = 0; i < ndev; ++i) counts_out[i] = r.partition.counts[i];
    }
    put_disp(r.totals, disp4);
  });
}

// simulate_photon_trace for one photon: deposits as (linear cell, weight).
int ref_trace(const vmc_scene* s, const vmc_config* c, std::uint64_t idx, int max_deps,
              std::int64_t* cells, double* weights, int* ndeps, double* disp4) {
  return guarded([&] {
    const R::Scene scene = make_scene(s);
    const R::SimulationConfig cfg = make_config(c);
    std::vector<std::pair<R::VoxelIndex, double>> deps;
    const R::PhotonDisposition d = R::simulate_photon_trace(idx, scene, cfg, deps);
    const int n = static_cast<int>(deps.size());
    *ndeps = n;
    for (int i = 0; i < n && i < max_deps; ++i) {
      cells[i] = static_cast<std::int64_t>(scene.grid.linear(deps[i].first));
      weights[i] = deps[i].second;
    }
    put_disp(d, disp4);
  });
}

// Derived oracle: photons [first, first+count) through the public step API
// with per-step llround deposits into gate-resolved cells (quantum from
// config.photon_count), optional deposit counts, per-photon traces and
// detector records (sorted by photon index). `threads` host threads.
int ref_walk(const vmc_scene* s, const vmc_config* c, std::uint64_t first, std::uint64_t count,
             int threads, std::int64_t* cells_out, std::int64_t* counts_out,
             vmc_photon_trace* traces, void* det_out, std::uint64_t* det_count, double* disp4) {
  return guarded([&] {
    const R::Scene scene = make_scene(s);
    const R::SimulationConfig cfg = make_config(c);
    cfg.validate();
    const int ngates = c->ngates > 0 ? c->ngates : 1;
    const std::size_t nvox = scene.grid.voxel_count();
    const std::size_t ncell = nvox * static_cast<std::size_t>(ngates);
    const double inv_q = 1.0 / ref_quantum_for(cfg.photon_count);
    const int nt = std::max(1, threads);
    const bool want_det = c->ndet > 0 && (det_out || det_count);

    std::vector<std::vector<std::int64_t>> cells(nt), counts(nt);
    std::vector<R::PhotonDisposition> disp(nt);
    std::vector<std::vector<DetHit>> hits(nt);
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) {
      pool.emplace_back([&, t] {
        WalkSink sink;
        if (cells_out) {
          cells[t].assign(ncell, 0);
          sink.cells = cells[t].data();
        }
        if (counts_out) {
          counts[t].assign(nvox, 0);
          sink.counts = counts[t].data();
        }
        sink.inv_quantum = inv_q;
        const std::uint64_t lo = count * t / nt, hi = count * (t + 1) / nt;
        for (std::uint64_t k = lo; k < hi; ++k) {
          disp[t] += walk_one(first + k, scene, cfg, c, sink, traces ? traces + k : nullptr,
                              want_det ? &hits[t] : nullptr);
        }
      });
    }
    for (auto& th : pool) th.join();

    if (cells_out) {
      std::fill(cells_out, cells_out + ncell, 0);
      for (int t = 0; t < nt; ++t)
        for (std::size_t i = 0; i < ncell; ++i) cells_out[i] += cells[t][i];
    }
    if (counts_out) {
      std::fill(counts_out, counts_out + nvox, 0);
      for (int t = 0; t < nt; ++t)
        for (std::size_t i = 0; i < nvox; ++i) counts_out[i] += counts[t][i];
    }
    R::PhotonDisposition tot;
    for (int t = 0; t < nt; ++t) tot += disp[t];
    put_disp(tot, disp4);
    if (want_det) {
      // threads own contiguous ascending ranges -> concatenation is sorted
      const int nm = static_cast<int>(scene.grid.media().size());
      const std::size_t stride = vmc_det_record_bytes(nm);
      std::uint64_t n = 0;
      for (int t = 0; t < nt; ++t) {
        for (const DetHit& h : hits[t]) {
          if (det_out && n < c->det_capacity) {
            auto* rec = static_cast<unsigned char*>(det_out) + n * stride;
            std::memset(rec, 0, stride);
            vmc_det_record_head head{h.photon, h.det, h.nscat, h.w, h.t};
            std::memcpy(rec, &head, sizeof head);
            std::memcpy(rec + sizeof head, h.ppath.data(), h.ppath.size() * sizeof(float));
          }
          ++n;
        }
      }
      if (det_count) *det_count = n;
    }
  });
}

size_t vmc_det_record_bytes(int32_t nmedia) {
  const size_t raw = sizeof(vmc_det_record_head) + sizeof(float) * (nmedia > 1 ? nmedia - 1 : 0);
  return (raw + 7) & ~static_cast<size_t>(7);
}

int ref_partition(int strategy, std::uint64_t total, int ndev, const vmc_device_profile* profs,
                  std::uint64_t* counts_out, double* makespan) {
  return guarded([&] {
    std::vector<R::DeviceProfile> devs(static_cast<std::size_t>(ndev));
    for (int i = 0; i < ndev; ++i) {
      devs[i].cores = profs[i].cores;
      devs[i].a = profs[i].a;
      devs[i].t0 = profs[i].t0;
    }
    const R::Strategy st = strategy == 1 ? R::Strategy::S1
                           : strategy == 2 ? R::Strategy::S2
                                           : R::Strategy::S3;
    const R::Partition p = R::make_partition(total, devs, st);
    for (int i = 0; i < ndev; ++i) counts_out[i] = p.counts[i];
    if (makespan) *makespan = R::model_makespan(p, devs);
  });
}

int ref_brute_force(std::uint64_t total, int ndev, const vmc_device_profile* profs,
                    std::uint64_t* counts_out, double* makespan) {
  return guarded([&] {
    std::vector<R::DeviceProfile> devs(static_cast<std::size_t>(ndev));
    for (int i = 0; i < ndev; ++i) {
      devs[i].cores = profs[i].cores;
      devs[i].a = profs[i].a;
      devs[i].t0 = profs[i].t0;
    }
    const auto r = R::oracles::brute_force_partition(total, devs);
    for (int i = 0; i < ndev; ++i) counts_out[i] = r.partition.counts[i];
    if (makespan) *makespan = r.makespan;
  });
}

// run_pipeline with the default roster (one host_device(threads) worker pool;
// threads = 0 -> std::thread::hardware_concurrency, config.cpp:118-125).
// Photons [0, config.photon_count). makespan_ms = RunReport::makespan_ms (the
// pool's wall time, config.cpp:305), e2e_ms = the whole call (map allocation,
// partition, merge, energy audit) on a steady clock.
int ref_run_pipeline(const vmc_scene* s, const vmc_config* c, int threads, double* makespan_ms,
                     double* e2e_ms, double* disp4) {
  return guarded([&] {
    R::RunSetup setup{make_scene(s), make_config(c), {}, R::Strategy::S1, "", ""};
    const auto t0 = std::chrono::steady_clock::now();
    R::RunResult r = R::run_pipeline(setup, threads);
    const auto t1 = std::chrono::steady_clock::now();
    if (makespan_ms) *makespan_ms = r.report.makespan_ms;
    if (e2e_ms) *e2e_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (disp4) {
      disp4[0] = r.map.total_deposited();
      disp4[1] = disp4[2] = disp4[3] = 0.0;
    }
  });
}

// FluenceMap(dims, photon_count) holding raw cells `cells` (set through
// deposit() in chunks the quantum represents exactly), then normalize(grid)
// (when `normalized`) and to_float_volume() into out[V].
int ref_normalize(const vmc_scene* s, std::uint64_t photon_count, const std::int64_t* cells, int normalized,
                  float* out) {
  return guarded([&] {
    const R::Scene scene = make_scene(s);
    R::FluenceMap map(scene.grid.dims(), photon_count);
    const double q = map.quantum();
    const std::int64_t chunk = std::int64_t{1} << 52;  // |chunk| * q and back are exact
    for (std::size_t i = 0; i < map.voxel_count(); ++i) {
      std::int64_t c = cells[i];
      while (c != 0) {
        const std::int64_t part = c > chunk ? chunk : (c < -chunk ? -chunk : c);
        map.deposit(i, static_cast<double>(part) * q);
        c -= part;
      }
    }
    if (normalized) map.normalize(scene.grid);
    const std::vector<float> v = map.to_float_volume();
    std::copy(v.begin(), v.end(), out);
  });
}

double ref_hg_cos_theta(double g, double xi) { return R::hg_cos_theta(g, xi); }
double ref_fresnel(double n1, double n2, double cos_i) { return R::fresnel_reflectance(n1, n2, cos_i); }
int ref_distance_to_boundary(const vmc_scene* s, const double* pos, const double* dir,
                             double* out) {
  return guarded([&] {
    const R::Scene scene = make_scene(s);
    *out = R::distance_to_voxel_boundary({pos[0], pos[1], pos[2]}, {dir[0], dir[1], dir[2]},
                                         scene.grid);
  });
}

}  // extern "C"
