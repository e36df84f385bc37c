// atomics_bench.cu — L2 red.global.add.u64 throughput on this GPU, for the
// transport kernel's secondary (L2-atomic) roofline.
//
// Every thread issues K fire-and-forget 64-bit integer adds (the instruction
// the transport kernels deposit with) into an int64 map of the cube60 size
// (60^3 cells = 1.73 MB, L2-resident), with four address streams:
//   uniform   cells drawn uniformly over the map
//   source    a cube60-B1-like hot spot: |dx|,|dy| ~ geometric around (30,30),
//             z ~ geometric from the entry face, so a few voxels take most adds
//   source/8  the same stream into 8 replicas (CTA b -> replica b mod 8), as K1f
//   single    every add to one cell (same-address serialisation bound)
//   replay    (optional, argv[2] = file of int32 cell indices) cells drawn from a
//             recorded deposit distribution -- tools/atomics_roofline.py samples
//             the B1 per-voxel deposit counts of the compiled reference
//   replay/R  the same into R = 8, 16, 32 replicas
// Output: one JSON line with adds/s per stream.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomics_bench atomics_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace {

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// geometric(|k|) from a 32-bit hash: P(k) ~ 2^-k, sign from one bit
__device__ __forceinline__ int geo(uint32_t r, int maxk) {
  const int k = __clz(static_cast<int>(r | 1u));  // P(k) = 2^-(k+1)
  return min(k, maxk);
}

__global__ void k_red(unsigned long long* cells, int mode, int ncells, int nrep, int iters,
                      const int* __restrict__ stream, uint32_t stream_mask) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long* base = cells + static_cast<long long>(blockIdx.x % nrep) * ncells;
  for (int k = 0; k < iters; ++k) {
    const uint32_t r = hash32(tid * 0x9E3779B9u + static_cast<uint32_t>(k) * 0x85EBCA6Bu + 1u);
    int c;
    if (mode == 0) {
      c = static_cast<int>(r % static_cast<uint32_t>(ncells));
    } else if (mode == 1) {
      const uint32_t r2 = hash32(r);
      const int dx = geo(r, 25) * ((r2 & 1) ? 1 : -1);
      const int dy = geo(r2, 25) * ((r & 1) ? 1 : -1);
      const int z = geo(hash32(r2), 59);
      c = (30 + dx) + 60 * ((30 + dy) + 60 * z);
    } else if (mode == 2) {
      c = 30 + 60 * 30;
    } else {
      c = __ldg(stream + (r & stream_mask));
    }
    atomicAdd(base + c, 1ull);
  }
}

}  // namespace

int main(int argc, char** argv) {
  const int iters = argc > 1 ? std::atoi(argv[1]) : 256;
  const int ncells = 60 * 60 * 60, nrep_max = 32;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, static_cast<size_t>(ncells) * nrep_max * sizeof(unsigned long long)) != cudaSuccess) {
    std::fprintf(stderr, "cudaMalloc failed\n");
    return 2;
  }
  const int block = 256, grid = sms * 8;
  const double adds = static_cast<double>(grid) * block * iters;
  // optional replay stream (power-of-two length)
  int* d_stream = nullptr;
  uint32_t stream_mask = 0;
  int nruns = 4;
  if (argc > 2) {
    FILE* f = std::fopen(argv[2], "rb");
    if (!f) {
      std::fprintf(stderr, "cannot open %s\n", argv[2]);
      return 2;
    }
    std::fseek(f, 0, SEEK_END);
    size_t n = static_cast<size_t>(std::ftell(f)) / sizeof(int);
    std::fseek(f, 0, SEEK_SET);
    size_t p2 = 1;
    while (p2 * 2 <= n) p2 *= 2;
    int* h = static_cast<int*>(std::malloc(p2 * sizeof(int)));
    if (std::fread(h, sizeof(int), p2, f) != p2) return 2;
    std::fclose(f);
    cudaMalloc(&d_stream, p2 * sizeof(int));
    cudaMemcpy(d_stream, h, p2 * sizeof(int), cudaMemcpyHostToDevice);
    std::free(h);
    stream_mask = static_cast<uint32_t>(p2 - 1);
    nruns = 8;
  }
  struct { const char* name; int mode, nrep; } runs[] = {
      {"uniform", 0, 1}, {"source", 1, 1}, {"source_rep8", 1, 8}, {"single", 2, 1},
      {"replay", 3, 1}, {"replay_rep8", 3, 8}, {"replay_rep16", 3, 16}, {"replay_rep32", 3, 32}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::printf("{\"sms\": %d, \"threads\": %d, \"adds_per_run\": %.0f", sms, grid * block, adds);
  for (int ri = 0; ri < nruns; ++ri) {
    const auto& r = runs[ri];
    const int it = r.mode == 2 ? iters / 16 : iters;  // the single-address stream is slow
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemset(d, 0, static_cast<size_t>(ncells) * nrep_max * sizeof(unsigned long long));
      cudaEventRecord(e0);
      k_red<<<grid, block>>>(d, r.mode, ncells, r.nrep, it, d_stream, stream_mask);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    const double n = static_cast<double>(grid) * block * it;
    std::printf(", \"%s\": %.4e", r.name, n / (best * 1e-3));
  }
  std::printf(", \"unit\": \"red.global.add.u64 per second\"}\n");
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    std::fprintf(stderr, "%s\n", cudaGetErrorString(err));
    return 2;
  }
  return 0;
}
