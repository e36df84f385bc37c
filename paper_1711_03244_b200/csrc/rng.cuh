// rng.cuh — device xorshift128+ streams, bit-compatible with the reference.
//
// Seeding follows proj/core/src/rng.cpp:5-19 (splitmix64 finalizer of
// seed ^ stream_id, all-zero state remapped) and next() follows
// proj/core/include/voxmc/rng.hpp:15-23; every u64 the device draws is the
// u64 the reference draws for the same (master_seed, photon index).
//
// Uniform deviates:
//   unit<double>  = (u >> 11) * 2^-53          (rng.hpp:26, exact reference)
//   unit<float>   = (u >> 40) * 2^-24          (same u64 stream, top 24 bits)
#pragma once
#include <cstdint>

namespace vmc {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <bool kCount>
struct Xs128p {
  uint64_t a, b;      // reference s_[0], s_[1]
  uint32_t draws;     // only maintained when kCount

  __device__ __forceinline__ void seed(uint64_t master, uint64_t stream) {
    const uint64_t z = master ^ stream;
    a = mix64(z);
    b = mix64(z + 0x9E3779B97F4A7C15ull);
    if ((a | b) == 0) b = 0x6A09E667F3BCC909ull;
    if (kCount) draws = 0;
  }

  __device__ __forceinline__ uint64_t next() {
    uint64_t x = a;
    const uint64_t y = b;
    const uint64_t r = x + y;
    a = y;
    x ^= x << 23;
    b = x ^ y ^ (x >> 18) ^ (y >> 5);
    if (kCount) ++draws;
    return r;
  }

  template <typename Real>
  __device__ __forceinline__ Real unit();

  // top 24 bits of the next u64 as a float in [0, 2^24): unit<float>() * 2^24,
  // for callers that fold the 2^-24 scale into an FMA
  __device__ __forceinline__ float u24() { return static_cast<float>(static_cast<uint32_t>(next() >> 40)); }
};

template <>
template <>
__device__ __forceinline__ float Xs128p<false>::unit<float>() {
  return static_cast<float>(static_cast<uint32_t>(next() >> 40)) * 0x1p-24f;
}
template <>
template <>
__device__ __forceinline__ float Xs128p<true>::unit<float>() {
  return static_cast<float>(static_cast<uint32_t>(next() >> 40)) * 0x1p-24f;
}
template <>
template <>
__device__ __forceinline__ double Xs128p<false>::unit<double>() {
  return static_cast<double>(next() >> 11) * 0x1p-53;
}
template <>
template <>
__device__ __forceinline__ double Xs128p<true>::unit<double>() {
  return static_cast<double>(next() >> 11) * 0x1p-53;
}

}  // namespace vmc
