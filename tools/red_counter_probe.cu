// red_counter_probe.cu — what does ncu's lts__t_requests_op_red count for
// red.global.add.u64? Launches with a KNOWN number of warp-level red
// instructions and lanes per pattern; ncu reads the L1 / L2 counters next to
// it (tools/gpu_red_probe.sh). Patterns (one launch each, 148*8 CTAs x 256
// threads, K reds per thread):
//   0 scattered  every lane its own 128-B line, lines spread over 16 MB
//   1 coalesced  the 32 lanes of a warp on 32 consecutive u64 (2 lines)
//   2 same       all lanes of a warp on one u64 (one per warp)
//   3 cube60     lanes on uniform-random cells of a 1.73 MB map (the K1f map size)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void k_red(unsigned long long* m, int pattern, int K) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t warp = tid >> 5, lane = tid & 31;
  for (int k = 0; k < K; ++k) {
    uint64_t idx;
    switch (pattern) {
      case 0: idx = (static_cast<uint64_t>(hash32(tid * 131 + k)) % (1u << 17)) * 16; break;  // 128 B apart
      case 1: idx = (static_cast<uint64_t>(hash32(warp * 977 + k)) % (1u << 14)) * 32 + lane; break;
      case 2: idx = static_cast<uint64_t>(hash32(warp * 977 + k)) % (1u << 18); break;
      default: idx = hash32(tid * 7919 + k) % 216000u; break;
    }
    atomicAdd(m + idx, 1ull);
  }
}

int main() {
  unsigned long long* m;
  cudaMalloc(&m, (1u << 21) * 8);
  cudaMemset(m, 0, (1u << 21) * 8);
  const int grid = 148 * 8, block = 256, K = 16;
  for (int p = 0; p < 4; ++p) {
    k_red<<<grid, block>>>(m, p, K);
    cudaDeviceSynchronize();
    const double lanes = static_cast<double>(grid) * block * K;
    std::printf("pattern %d: %.0f lane reds, %.0f warp red instructions\n", p, lanes, lanes / 32);
  }
  return 0;
}
