// Cross-checks the C++ front door (include/voxmc/config.hpp, volume_io.hpp)
// against the Python one (paper_1711_03244_b200/pipeline.py, volume_io.py):
//   front_door_test hash <b1|b2|b2a>     -> scene_hash of the preset (hex)
//   front_door_test write <path>         -> writes a small volume, prints its checksum
//   front_door_test read <path>          -> reads a volume, prints dims / seed / checksum / sum
#include <cstdio>
#include <string>

#include "voxmc/config.hpp"
#include "voxmc/volume_io.hpp"

using namespace voxmc;

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const std::string cmd = argv[1];
  if (cmd == "hash") {
    const BenchmarkSetup st = benchmark_preset(*benchmark_from_name(argv[2]));
    std::printf("%016llx\n", static_cast<unsigned long long>(scene_hash(Scene{st.grid, st.source}, st.config)));
  } else if (cmd == "write") {
    FluenceMap map({7, 5, 3}, 1000);
    map.deposit(VoxelIndex{1, 2, 0}, 0.25);
    map.deposit(VoxelIndex{6, 4, 2}, 0.125);
    write_volume(map, 0.5, 99, argv[2]);
    std::printf("%016llx\n", static_cast<unsigned long long>(read_volume(argv[2]).checksum));
  } else if (cmd == "read") {
    const VolumeData v = read_volume(argv[2]);
    double sum = 0.0;
    for (float x : v.values) sum += x;
    std::printf("%d %d %d %llu %016llx %.9g\n", v.dims.x, v.dims.y, v.dims.z, static_cast<unsigned long long>(v.seed),
                static_cast<unsigned long long>(v.checksum), sum);
  }
  return 0;
}
