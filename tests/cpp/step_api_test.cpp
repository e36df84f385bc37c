// Drives the drop-in's one-photon step API (launch / advance / handle_interface /
// roulette, include/voxmc) in the order of the reference's run_photon
// (transport.cpp:310-358) on the host and prints one line per photon:
//   index deposited escaped killed truncated steps
// tests/test_step_api.py compares the lines with the compiled reference's walk
// of the same photons (oracle/_ref, traces).
//
// usage: step_api_test <b1|b2|b3> <first> <count> <seed>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "voxmc/voxmc.hpp"

using namespace voxmc;

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s <b1|b2|b3> <first> <count> <seed>\n", argv[0]);
    return 2;
  }
  const std::string name = argv[1];
  const unsigned long long first = std::strtoull(argv[2], nullptr, 10);
  const unsigned long long count = std::strtoull(argv[3], nullptr, 10);
  BenchmarkSetup st = benchmark_preset(name == "b3" ? Benchmark::B2 : Benchmark::B1);
  if (name == "b2") st.config.boundary_mode = BoundaryMode::ReflectAtMismatch;
  st.config.master_seed = std::strtoull(argv[4], nullptr, 10);
  st.config.photon_count = first + count;
  const VoxelGrid& grid = st.grid;
  const Source& src = st.source;
  const SimulationConfig& cfg = st.config;
  for (unsigned long long i = first; i < first + count; ++i) {
    RngStream stream(cfg.master_seed, i);
    PhotonState ph = launch(src, grid, stream);
    PhotonDisposition d;
    long steps = 0;
    for (bool alive = true; alive;) {
      const StepOutcome out = advance(ph, grid, cfg, stream);
      ++steps;
      d.deposited += out.deposited;
      switch (out.kind) {
        case StepKind::Terminated:
          d.truncated += ph.weight;
          alive = false;
          break;
        case StepKind::Scattered:
          if (ph.weight < cfg.roulette_threshold) {
            const double before = ph.weight;
            if (!roulette(ph, cfg, stream)) {
              d.killed += before;
              alive = false;
            } else {
              d.killed += before - ph.weight;
            }
          }
          break;
        case StepKind::CrossedVoxel:
          if (out.interface_pending &&
              handle_interface(ph, grid, cfg, out, stream).kind == StepKind::ExitedDomain) {
            d.escaped += ph.weight;
            alive = false;
          }
          break;
        default:
          break;
      }
    }
    std::printf("%llu %.17g %.17g %.17g %.17g %ld\n", i, d.deposited, d.escaped, d.killed, d.truncated, steps);
  }
  return 0;
}
