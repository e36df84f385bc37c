// partition.hpp — host-side photon partitioning (see partition.cpp).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace vmc {

struct DeviceModel {
  int cores = 1;
  double a = 0.0;   // ms per photon
  double t0 = 0.0;  // ms fixed overhead
};

struct PartitionError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// strategy 1 = S1 (cores), 2 = S2 (1/a), 3 = S3 (exact minimax)
std::vector<uint64_t> partition_photons(int strategy, uint64_t total, const std::vector<DeviceModel>& dev);
double model_makespan(const std::vector<uint64_t>& n, const std::vector<DeviceModel>& dev);

}  // namespace vmc
