// dropin_test.cpp — code written against the reference's C++ API
// (proj/core/include/voxmc/*.hpp) compiled unchanged against the B200
// library's headers (include/voxmc/) and linked to libvoxmc_b200.so.
// Mirrors reference tests: test_scheduler.cpp:157-168, 246-264,
// test_fluence.cpp:17-58, test_domain.cpp, acceptance.cpp criterion 11.
// usage: dropin_test [--cpu-only]
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "voxmc/fluence.hpp"
#include "voxmc/scheduler.hpp"
#include "voxmc/transport.hpp"
#include "voxmc/types.hpp"

using namespace voxmc;

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
      ++failures;                                                  \
    }                                                              \
  } while (0)

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu-only") == 0;
  // domain + validation
  auto b1 = benchmark_preset(Benchmark::B1);
  CHECK(b1.grid.nx() == 60 && b1.grid.medium(1).n == 1.37);
  bool threw = false;
  try {
    VoxelGrid bad({1, 1, 1}, 1.0, {3}, {{}, {}});
  } catch (const ValidationError&) {
    threw = true;
  }
  CHECK(threw);
  RngStream s(20260826, 123456789);
  CHECK(s.next_u64() == 0x8ac56efd89a4bd9bULL);
  // fluence arithmetic
  FluenceMap a({4, 4, 4}, 100), b({4, 4, 4}, 100);
  a.deposit(std::size_t{0}, 0.5);
  b.deposit(std::size_t{0}, 0.25);
  std::vector<FluenceMap> parts{a, b};
  CHECK(std::fabs(merge(parts).value(0) - 0.75) < 1e-12);
  // partitions
  std::vector<DeviceProfile> devs(3);
  for (auto& d : devs) d.cores = 1;
  CHECK((partition_s1(10, devs).counts == std::vector<std::uint64_t>{4, 3, 3}));
  if (cpu_only) {
    std::printf("%s (cpu-only)\n", failures ? "FAILED" : "PASSED");
    return failures;
  }
  // executor on the GPU
  Scene scene{b1.grid, b1.source};
  SimulationConfig cfg = b1.config;
  cfg.photon_count = 200'000;
  cfg.master_seed = 1;
  GroupRunResult g = run_group_dynamic(0, 200'000, 8, scene, cfg);
  const double books = g.totals.deposited + g.totals.escaped + g.totals.killed + g.totals.truncated;
  CHECK(std::fabs(books / 200'000.0 - 1.0) < 1e-6);
  CHECK(g.per_thread_photons.size() == 8);
  std::uint64_t sum = 0;
  for (auto c : g.per_thread_photons) sum += c;
  CHECK(sum == 200'000);
  CHECK(std::fabs(g.totals.deposited / 200'000.0 - 0.1791) < 0.003);
  // static == dynamic raw cells (test_scheduler.cpp:157-168)
  GroupRunResult st = run_static_split(0, 200'000, 3, scene, cfg);
  bool same = true;
  for (std::size_t c = 0; c < g.map.voxel_count(); ++c) same &= g.map.raw_cell(c) == st.map.raw_cell(c);
  CHECK(same);
  // beam-axis peak (acceptance.cpp criterion 11)
  std::size_t best = 0;
  for (std::size_t c = 1; c < g.map.voxel_count(); ++c)
    if (g.map.raw_cell(c) > g.map.raw_cell(best)) best = c;
  CHECK(best % 60 == 30 && (best / 60) % 60 == 30 && best / 3600 < 5);
  // multi-device runner with one CUDA device == single run
  std::vector<DeviceProfile> gpus(1);
  gpus[0].kind = DeviceKind::CudaGpu;
  gpus[0].name = "gpu0";
  MultiDeviceResult m = run_multi_device(200'000, gpus, Strategy::S1, scene, cfg, 0);
  same = true;
  for (std::size_t c = 0; c < g.map.voxel_count(); ++c) same &= m.map.raw_cell(c) == g.map.raw_cell(c);
  CHECK(same);
  CHECK(m.makespan_ms > 0.0);
  // SourceOutsideDomain
  threw = false;
  try {
    Scene out{b1.grid, Source{{70.0, 30.0, 30.0}, {0, 0, 1}, false}};
    run_group_dynamic(0, 10, 1, out, cfg);
  } catch (const SourceOutsideDomain&) {
    threw = true;
  }
  CHECK(threw);
  // calibration of a real GPU (two pilots)
  gpus[0].gpu = 0;
  Calibration cal = calibrate(gpus[0], 100'000, 2'000'000, scene, cfg, 1);
  CHECK(cal.a > 0.0);
  std::printf("%s a=%.3e ms/photon t0=%.3f ms\n", failures ? "FAILED" : "PASSED", cal.a, cal.t0);
  return failures;
}
