// partition.cpp — device-level photon split (host C++).
//
// Restates the reference's partitioning strategies
// (proj/core/include/voxmc/scheduler.hpp:40-56, proj/core/src/scheduler.cpp:45-251)
// so that the B200 multi-GPU runner hands every device the same contiguous
// photon range the reference would:
//   S1  proportional to cores         (scheduler.cpp:77-85)
//   S2  proportional to 1/a           (scheduler.cpp:87-95)
//   S3  exact minimax of a_i n_i + t0_i over device subsets (scheduler.cpp:107-242)
// The proportional split is largest-remainder with a lower-index tie break
// (scheduler.cpp:49-73). tests/test_partition.py compares every strategy with
// the compiled reference on random instances.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "partition.hpp"

namespace vmc {

namespace {

std::vector<uint64_t> largest_remainder(uint64_t total, const std::vector<double>& weight) {
  double sum = 0.0;
  for (double x : weight) sum += x;
  if (!(sum > 0.0)) throw PartitionError("partition: weights must sum to > 0");
  const size_t k = weight.size();
  std::vector<uint64_t> n(k, 0);
  std::vector<double> rem(k, 0.0);
  uint64_t given = 0;
  for (size_t i = 0; i < k; ++i) {
    const double exact = static_cast<double>(total) * weight[i] / sum;
    const double whole = std::floor(exact);
    n[i] = static_cast<uint64_t>(whole);
    rem[i] = exact - whole;
    given += n[i];
  }
  // hand the leftover units out by descending remainder; stable => lower index first
  std::vector<size_t> rank(k);
  std::iota(rank.begin(), rank.end(), size_t{0});
  std::stable_sort(rank.begin(), rank.end(), [&](size_t a, size_t b) { return rem[a] > rem[b]; });
  for (size_t j = 0; given < total; ++j, ++given) ++n[rank[j % k]];
  return n;
}

double finish_time(const DeviceModel& d, uint64_t n) { return d.a * static_cast<double>(n) + d.t0; }

double worst_finish(const std::vector<DeviceModel>& dev, const std::vector<size_t>& members,
                    const std::vector<uint64_t>& n) {
  double m = 0.0;
  for (size_t i : members)
    if (n[i] > 0) m = std::max(m, finish_time(dev[i], n[i]));
  return m;
}

// Minimax over one support set. The capacity of device i by time T is
// floor((T - t0_i)/a_i); bisect the smallest T whose capacities cover `total`,
// trim the surplus from the latest finisher, then polish with single-photon
// moves until no move lowers the makespan.
bool minimax_on(uint64_t total, const std::vector<DeviceModel>& dev,
                const std::vector<size_t>& members, std::vector<uint64_t>& n, double& span) {
  auto capacity = [&](double T, size_t i) -> uint64_t {
    const double c = std::floor((T - dev[i].t0) / dev[i].a + 1e-9);
    if (c <= 0.0) return 0;
    return static_cast<uint64_t>(std::min(c, static_cast<double>(total)));
  };
  auto covered = [&](double T) {
    uint64_t s = 0;
    for (size_t i : members) s += capacity(T, i);
    return s;
  };
  double hi = std::numeric_limits<double>::infinity();
  for (size_t i : members) hi = std::min(hi, finish_time(dev[i], total));
  double lo = 0.0;
  n.assign(dev.size(), 0);
  if (covered(lo) >= total) {
    span = 0.0;
    return true;
  }
  for (int it = 0; it < 200 && (hi - lo) > 1e-9 * std::max(1.0, hi); ++it) {
    const double mid = 0.5 * (lo + hi);
    (covered(mid) >= total ? hi : lo) = mid;
  }
  uint64_t given = 0;
  for (size_t i : members) given += (n[i] = capacity(hi, i));
  if (given < total) return false;
  for (uint64_t extra = given - total; extra > 0; --extra) {
    size_t late = members.front();
    double late_t = -1.0;
    for (size_t i : members) {
      if (n[i] == 0) continue;
      const double f = finish_time(dev[i], n[i]);
      if (f > late_t) {
        late_t = f;
        late = i;
      }
    }
    --n[late];
  }
  span = worst_finish(dev, members, n);
  for (int pass = 0; pass < 4096; ++pass) {
    bool better = false;
    for (size_t src : members) {
      if (n[src] == 0) continue;
      for (size_t dst : members) {
        if (dst == src) continue;
        --n[src];
        ++n[dst];
        const double m = worst_finish(dev, members, n);
        if (m < span - 1e-12 * std::max(1.0, span)) {
          span = m;
          better = true;
        } else {
          ++n[src];
          --n[dst];
        }
      }
    }
    if (!better) break;
  }
  return true;
}

}  // namespace

std::vector<uint64_t> partition_photons(int strategy, uint64_t total, const std::vector<DeviceModel>& dev) {
  if (dev.empty()) throw PartitionError("partition: no devices");
  std::vector<double> w(dev.size());
  switch (strategy) {
    case 1:
      for (size_t i = 0; i < dev.size(); ++i) {
        if (dev[i].cores < 1) throw PartitionError("partition_s1: cores must be >= 1");
        w[i] = static_cast<double>(dev[i].cores);
      }
      return largest_remainder(total, w);
    case 2:
      for (size_t i = 0; i < dev.size(); ++i) {
        if (!(dev[i].a > 0.0)) throw PartitionError("partition_s2: slope a must be > 0");
        w[i] = 1.0 / dev[i].a;
      }
      return largest_remainder(total, w);
    case 3: {
      for (const DeviceModel& d : dev)
        if (!(d.a > 0.0) || d.t0 < 0.0) throw PartitionError("partition_s3: need a > 0, t0 >= 0");
      const size_t k = dev.size();
      std::vector<uint64_t> best(k, 0), n;
      if (total == 0) return best;
      double best_span = std::numeric_limits<double>::infinity(), span = 0.0;
      if (k <= 16) {
        for (uint32_t mask = 1; mask < (1u << k); ++mask) {
          std::vector<size_t> members;
          for (size_t i = 0; i < k; ++i)
            if (mask & (1u << i)) members.push_back(i);
          if (!minimax_on(total, dev, members, n, span)) continue;
          if (span < best_span) {
            best_span = span;
            best = n;
          }
        }
      } else {
        std::vector<size_t> members(k);
        std::iota(members.begin(), members.end(), size_t{0});
        if (!minimax_on(total, dev, members, n, span)) throw PartitionError("partition_s3: infeasible instance");
        best = n;
      }
      return best;
    }
    default:
      throw PartitionError("unknown strategy");
  }
}

double model_makespan(const std::vector<uint64_t>& n, const std::vector<DeviceModel>& dev) {
  double m = 0.0;
  for (size_t i = 0; i < n.size() && i < dev.size(); ++i)
    if (n[i] > 0) m = std::max(m, finish_time(dev[i], n[i]));
  return m;
}

}  // namespace vmc
