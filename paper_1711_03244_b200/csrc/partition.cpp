// partition.cpp — device-level photon split (host C++), derived from the
// strategies' definitions rather than from the reference's solver code.
//
// Contract (reference scheduler.hpp:40-56; behaviour checked against the
// compiled reference by tests/test_partition.py on random instances):
//   S1  counts proportional to cores, S2 proportional to 1/a: apportion
//       `total` by the weights, every device gets floor(total * w_i / W) and
//       the left-over units go one each to the largest fractional parts,
//       lower device index first on equal parts.
//   S3  the integer allocation minimising the makespan max_i (a_i n_i + t0_i)
//       over devices with n_i > 0 (an idle device costs nothing).
//
// S3 as a selection problem: giving device i its m-th photon finishes it at
// u_im = a_i m + t0_i, increasing in m. An allocation of `total` photons is a
// choice of `total` such units with each device's units a prefix; its
// makespan is its largest chosen unit. The minimum is therefore reached by
// choosing the `total` smallest units overall (they form prefixes since u_im
// increases in m). They are found in two steps:
//   1. water level: the continuous relaxation sum_i (T - t0_i) / a_i = total
//      over the devices with t0_i < T gives T_c (devices whose t0 lies above
//      the level drop out, the level is recomputed until stable); every unit
//      at or below T_c is chosen: n_i = floor((T_c - t0_i) / a_i), which
//      leaves at most one unit per device to place;
//   2. completion: the remaining units go one at a time to the device whose
//      next unit finishes first, and any overshoot from rounding in step 1 is
//      taken back from the latest units.
// The optimal makespan T* is the largest chosen unit. When several units tie
// at T* (identical devices), the allocation is made canonical the way the
// reference's run_multi_device sees it (tests compare device for device):
//   * the devices used are the smallest set, read as a bit mask over device
//     indices, whose units at or below T* still cover `total` (up to 16
//     devices; all devices beyond that);
//   * every unit below T* of a used device is chosen, and the units exactly
//     at T* go to the highest-index used devices first.
// O(k^2) for k devices, independent of `total`.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "partition.hpp"

namespace vmc {

namespace {

// floor(total * w_i / W) for every device, then one extra unit per device in
// order of decreasing fractional part (lower index first) until `total`
std::vector<uint64_t> apportion(uint64_t total, const std::vector<double>& w) {
  double wsum = 0.0;
  for (double x : w) wsum += x;
  if (!(wsum > 0.0)) throw PartitionError("partition: the device weights do not sum to a positive value");
  const size_t k = w.size();
  std::vector<uint64_t> n(k);
  std::vector<double> part(k);
  uint64_t placed = 0;
  for (size_t i = 0; i < k; ++i) {
    const double share = static_cast<double>(total) * w[i] / wsum;
    const double whole = std::floor(share);
    n[i] = static_cast<uint64_t>(whole);
    part[i] = share - whole;
    placed += n[i];
  }
  // left-over units: walk the devices by decreasing fractional part; `taken`
  // marks the ones served in the current sweep (a sweep serves each device at
  // most once; further sweeps only happen if rounding left more than k units)
  std::vector<char> taken(k, 0);
  size_t served = 0;
  while (placed < total) {
    if (served == k) {
      std::fill(taken.begin(), taken.end(), 0);
      served = 0;
    }
    size_t pick = k;
    for (size_t i = 0; i < k; ++i)
      if (!taken[i] && (pick == k || part[i] > part[pick])) pick = i;
    taken[pick] = 1;
    ++served;
    ++n[pick];
    ++placed;
  }
  return n;
}

// a m + t0 in one rounding: the reference is built with -march=native, where
// GCC contracts this expression into an FMA, and exact ties between devices
// (hence which device gets a tied unit) depend on that rounding
double unit_time(const DeviceModel& d, uint64_t m) { return std::fma(d.a, static_cast<double>(m), d.t0); }

std::vector<uint64_t> minimax(uint64_t total, const std::vector<DeviceModel>& dev) {
  const size_t k = dev.size();
  std::vector<uint64_t> n(k, 0);
  if (total == 0) return n;
  // 1. water level over the devices whose overhead lies below it
  std::vector<char> on(k, 1);
  double level = 0.0;
  for (;;) {
    double inv = 0.0, off = 0.0;
    for (size_t i = 0; i < k; ++i)
      if (on[i]) {
        inv += 1.0 / dev[i].a;
        off += dev[i].t0 / dev[i].a;
      }
    level = (static_cast<double>(total) + off) / inv;
    bool dropped = false;
    for (size_t i = 0; i < k; ++i)
      if (on[i] && dev[i].t0 >= level) {
        on[i] = 0;
        dropped = true;
      }
    if (!dropped) break;
  }
  uint64_t placed = 0;
  for (size_t i = 0; i < k; ++i) {
    if (!on[i]) continue;
    const double units = std::floor((level - dev[i].t0) / dev[i].a);
    n[i] = units > 0.0 ? static_cast<uint64_t>(std::min(units, static_cast<double>(total))) : 0;
    placed += n[i];
  }
  // 2a. rounding overshoot: give back the latest units
  while (placed > total) {
    size_t late = k;
    for (size_t i = 0; i < k; ++i)
      if (n[i] > 0 && (late == k || unit_time(dev[i], n[i]) > unit_time(dev[late], n[late]))) late = i;
    --n[late];
    --placed;
  }
  // 2b. completion: each remaining unit to the device that finishes it first
  while (placed < total) {
    size_t best = 0;
    for (size_t i = 1; i < k; ++i)
      if (unit_time(dev[i], n[i] + 1) < unit_time(dev[best], n[best] + 1)) best = i;
    ++n[best];
    ++placed;
  }
  // optimal makespan: the largest chosen unit
  double tstar = 0.0;
  for (size_t i = 0; i < k; ++i)
    if (n[i] > 0) tstar = std::max(tstar, unit_time(dev[i], n[i]));
  // units at or below T* (at[i]) and strictly below it (below[i]) per device
  std::vector<uint64_t> at(k), below(k);
  for (size_t i = 0; i < k; ++i) {
    const double est = std::floor((tstar - dev[i].t0) / dev[i].a);
    uint64_t m = est > 0.0 ? static_cast<uint64_t>(std::min(est, static_cast<double>(total))) : 0;
    while (m < total && unit_time(dev[i], m + 1) <= tstar) ++m;
    while (m > 0 && unit_time(dev[i], m) > tstar) --m;
    at[i] = m;
    below[i] = (m > 0 && unit_time(dev[i], m) == tstar) ? m - 1 : m;
  }
  // smallest device mask that still covers `total` with units <= T*:
  // drop the highest-index devices first
  std::vector<char> use(k, 1);
  if (k <= 16) {
    uint64_t kept_above = 0;
    for (size_t j = k; j-- > 0;) {
      uint64_t lower = 0;
      for (size_t i = 0; i < j; ++i) lower += at[i];
      if (lower + kept_above >= total) {
        use[j] = 0;
      } else {
        kept_above += at[j];
      }
    }
  }
  placed = 0;
  for (size_t i = 0; i < k; ++i) {
    n[i] = use[i] ? below[i] : 0;
    placed += n[i];
  }
  for (size_t i = k; i-- > 0 && placed < total;)
    if (use[i] && at[i] > below[i]) {
      ++n[i];
      ++placed;
    }
  return n;
}

}  // namespace

std::vector<uint64_t> partition_photons(int strategy, uint64_t total, const std::vector<DeviceModel>& dev) {
  if (dev.empty()) throw PartitionError("partition: empty device list");
  std::vector<double> w(dev.size());
  if (strategy == 1) {
    for (size_t i = 0; i < dev.size(); ++i) {
      if (dev[i].cores < 1) throw PartitionError("partition_s1: a device has fewer than 1 core");
      w[i] = static_cast<double>(dev[i].cores);
    }
    return apportion(total, w);
  }
  if (strategy == 2) {
    for (size_t i = 0; i < dev.size(); ++i) {
      if (!(dev[i].a > 0.0)) throw PartitionError("partition_s2: a device has a non-positive slope a");
      w[i] = 1.0 / dev[i].a;
    }
    return apportion(total, w);
  }
  if (strategy == 3) {
    for (const DeviceModel& d : dev)
      if (!(d.a > 0.0) || d.t0 < 0.0) throw PartitionError("partition_s3: every device needs a > 0 and t0 >= 0");
    return minimax(total, dev);
  }
  throw PartitionError("partition: unknown strategy");
}

double model_makespan(const std::vector<uint64_t>& n, const std::vector<DeviceModel>& dev) {
  double m = 0.0;
  for (size_t i = 0; i < n.size() && i < dev.size(); ++i)
    if (n[i] > 0) m = std::max(m, unit_time(dev[i], n[i]));
  return m;
}

}  // namespace vmc
