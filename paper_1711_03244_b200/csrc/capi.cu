// capi.cu — implementation of the C-ABI in include/vmc.h.
//
// Host-side executor for one B200: validates the scene exactly as the
// reference does, stages labels (packed uint8) and the media table in HBM,
// sizes a persistent grid by occupancy, and launches K1. The synchronous
// entry points (vmc_run_range / vmc_run_multi) are the drop-in for
// run_group_dynamic / run_multi_device (proj/core/src/scheduler.cpp:255-451).
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <dlfcn.h>

#include <algorithm>
#include <map>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vmc.h"
#include "partition.hpp"
#include "transport.cuh"

namespace vmc {
const void* transport_kernel_float(bool gates, bool det, bool trace, bool uniform);
const void* transport_kernel_double(bool gates, bool det, bool trace, bool uniform);
const void* flight_kernel_float(bool gates, bool det, bool trace, bool uniform, int dep, bool solo = false);
const void* flight_kernel_double(bool gates, bool det, bool trace, bool uniform);
}  // namespace vmc

namespace {

thread_local std::string g_last_error;

struct VmcError : std::runtime_error {
  int code;
  VmcError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail_validation(const std::string& m) { throw VmcError(VMC_ERR_VALIDATION, m); }
[[noreturn]] void fail_runtime(const std::string& m) { throw VmcError(VMC_ERR_RUNTIME, m); }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail_runtime(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return VMC_OK;
  } catch (const VmcError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const vmc::PartitionError& e) {
    g_last_error = e.what();
    return VMC_ERR_VALIDATION;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return VMC_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return VMC_ERR_RUNTIME;
  }
}

int bit_width_u64(uint64_t v) {
  int w = 0;
  while (v) {
    ++w;
    v >>= 1;
  }
  return w;
}

// FluenceMap quantum rule (proj/core/src/fluence.cpp:11-14): power-of-two
// quantum so N unit-weight photons cannot overflow 63 bits.
int quantum_bits(uint64_t n) { return 62 - bit_width_u64(n | 1u); }

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

struct HostLaunch {
  double dir[3];
  double pos[3];
  int v[3];
};

// Pencil launch geometry in double on the host (transport.cpp:83-106,
// VoxelGrid::voxel_of types.cpp:35-42); throws like SourceOutsideDomain.
HostLaunch pencil_launch(const vmc_scene* s) {
  HostLaunch L;
  const double n = std::sqrt(s->src_dir[0] * s->src_dir[0] + s->src_dir[1] * s->src_dir[1] +
                             s->src_dir[2] * s->src_dir[2]);
  const double inv = 1.0 / n;
  for (int k = 0; k < 3; ++k) {
    L.dir[k] = s->src_dir[k] * inv;
    L.pos[k] = s->src_pos[k] + L.dir[k] * 1e-6;
    L.v[k] = static_cast<int>(std::floor(L.pos[k] / s->voxel_mm));
  }
  return L;
}

bool inside(const vmc_scene* s, const int* v) {
  return v[0] >= 0 && v[1] >= 0 && v[2] >= 0 && v[0] < s->nx && v[1] < s->ny && v[2] < s->nz;
}

// Label-volume facts every call needs (the largest label for validation, and
// whether the volume is single-label for the kernel choice), cached by a
// 64-bit digest of the volume: a repeated call on the same volume reads the
// labels once (the digest pass) instead of three times, and vmc_run_range
// skips the label upload when the device already holds that volume.
struct LabelInfo {
  uint64_t digest = 0;
  uint8_t max = 0;
  bool uniform = false;
};

uint64_t label_digest(const uint8_t* p, size_t n) {
  // four independent multiply-xor chains over 8-byte words, then the tail
  uint64_t h[4] = {0x243F6A8885A308D3ull, 0x13198A2E03707344ull, 0xA4093822299F31D0ull, 0x082EFA98EC4E6C89ull};
  const size_t nw = n / 8;
  size_t i = 0;
  for (; i + 4 <= nw; i += 4) {
    for (int k = 0; k < 4; ++k) {
      uint64_t w;
      std::memcpy(&w, p + 8 * (i + k), 8);
      h[k] = (h[k] ^ w) * 0x9E3779B97F4A7C15ull;
      h[k] ^= h[k] >> 29;
    }
  }
  for (; i < nw; ++i) {
    uint64_t w;
    std::memcpy(&w, p + 8 * i, 8);
    h[0] = (h[0] ^ w) * 0x9E3779B97F4A7C15ull;
    h[0] ^= h[0] >> 29;
  }
  for (size_t j = 8 * nw; j < n; ++j) h[1] = (h[1] ^ p[j]) * 0x100000001B3ull;
  uint64_t r = n;
  for (int k = 0; k < 4; ++k) r = vmc::mix64(r ^ h[k]);
  return r;
}

LabelInfo label_info(const vmc_scene* s) {
  const size_t nvox = static_cast<size_t>(s->nx) * s->ny * s->nz;
  LabelInfo li;
  li.digest = label_digest(s->labels, nvox);
  static std::mutex mu;
  static LabelInfo recent[8];
  static size_t recent_n[8] = {};
  static int next = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (int k = 0; k < 8; ++k)
      if (recent_n[k] == nvox && recent[k].digest == li.digest) return recent[k];
  }
  uint8_t mx = 0;
  bool uni = true;
  const uint8_t l0 = s->labels[0];
  for (size_t i = 0; i < nvox; ++i) {
    const uint8_t b = s->labels[i];
    mx = std::max(mx, b);
    uni = uni && b == l0;
  }
  li.max = mx;
  li.uniform = uni;
  std::lock_guard<std::mutex> lock(mu);
  recent[next] = li;
  recent_n[next] = nvox;
  next = (next + 1) % 8;
  return li;
}

void validate(const vmc_scene* s, const vmc_config* c, LabelInfo* info = nullptr) {
  if (!s || !c) fail_validation("null scene/config");
  // VoxelGrid ctor, types.cpp:7-33
  if (s->nx < 1 || s->ny < 1 || s->nz < 1) fail_validation("VoxelGrid: all dims must be >= 1");
  if (!(s->voxel_mm > 0.0)) fail_validation("VoxelGrid: voxel_size must be > 0");
  if (s->nmedia < 1 || !s->media) fail_validation("VoxelGrid: media list is empty");
  if (s->nmedia > 256) fail_validation("VoxelGrid: at most 256 media (uint8 labels)");
  if (!s->labels) fail_validation("VoxelGrid: label array size does not match dims");
  for (int m = 0; m < s->nmedia; ++m) {
    const double* p = s->media + 4 * m;
    if (p[0] < 0.0 || p[1] < 0.0 || p[2] < -1.0 || p[2] > 1.0 || p[3] < 1.0 || std::isnan(p[0]) ||
        std::isnan(p[1]) || std::isnan(p[2]) || std::isnan(p[3]))
      fail_validation("VoxelGrid: invalid optical properties");
  }
  const size_t nvox = static_cast<size_t>(s->nx) * s->ny * s->nz;
  const LabelInfo li = label_info(s);
  if (info) *info = li;
  if (li.max >= s->nmedia) fail_validation("VoxelGrid: label exceeds media list");
  // SimulationConfig::validate, types.cpp:44-52
  if (c->photon_count < 1) fail_validation("photon_count must be >= 1");
  if (!(c->tmax_ns > 0.0)) fail_validation("tmax must be > 0");
  if (!(c->roulette_threshold > 0.0 && c->roulette_threshold < 1.0))
    fail_validation("roulette_threshold must be in (0, 1)");
  if (c->roulette_multiplier < 2) fail_validation("roulette_multiplier must be >= 2");
  if (c->workgroup_size < 0) fail_validation("workgroup_size must be >= 1");
  // B200 additions
  if (c->ngates < 1) fail_validation("ngates must be >= 1");
  if (c->precision != VMC_PRECISION_FP32 && c->precision != VMC_PRECISION_FP64)
    fail_validation("precision must be VMC_PRECISION_FP32 or VMC_PRECISION_FP64");
  if (c->boundary_mode != VMC_BOUNDARY_TERMINATE && c->boundary_mode != VMC_BOUNDARY_REFLECT)
    fail_validation("boundary must be 'terminate' or 'reflect'");
  if (c->ndet < 0 || c->ndet > vmc::kMaxDet) fail_validation("ndet must be in [0, 16]");
  if (c->ndet > 0) {
    if (!c->det) fail_validation("detector array is null");
    if (s->nmedia - 1 > vmc::kMaxDetMedia) fail_validation("detectors support at most 8 interior media");
    for (int k = 0; k < c->ndet; ++k)
      if (!(c->det[4 * k + 3] > 0.0)) fail_validation("detector radius must be > 0");
  }
  if (nvox >= (1ull << 31)) fail_validation("volume must have fewer than 2^31 voxels");
  if (static_cast<unsigned long long>(nvox) * static_cast<unsigned>(c->ngates) > (1ull << 40))
    fail_validation("volume x gates too large");
  // launch point (transport.cpp:95-99)
  if (!s->isotropic) {
    const double n2 = s->src_dir[0] * s->src_dir[0] + s->src_dir[1] * s->src_dir[1] + s->src_dir[2] * s->src_dir[2];
    if (!(n2 > 0.0)) fail_validation("source direction must be nonzero");
    const HostLaunch L = pencil_launch(s);
    if (!inside(s, L.v)) throw VmcError(VMC_ERR_VALIDATION, "source entry point maps outside the voxel grid");
  } else {
    // every launch direction must keep the nudged point inside the grid
    for (int corner = 0; corner < 8; ++corner) {
      int v[3];
      for (int k = 0; k < 3; ++k) {
        const double p = s->src_pos[k] + ((corner >> k) & 1 ? 1e-6 : -1e-6);
        v[k] = static_cast<int>(std::floor(p / s->voxel_mm));
      }
      if (!inside(s, v)) fail_validation("source entry point maps outside the voxel grid");
    }
  }
}

template <typename Real>
std::vector<vmc::Medium<Real>> build_media(const vmc_scene* s) {
  std::vector<vmc::Medium<Real>> out(static_cast<size_t>(s->nmedia));
  for (int m = 0; m < s->nmedia; ++m) {
    const double mua = s->media[4 * m], mus = s->media[4 * m + 1], g = s->media[4 * m + 2],
                 n = s->media[4 * m + 3];
    vmc::Medium<Real>& M = out[m];
    std::memset(&M, 0, sizeof M);
    M.mua = static_cast<Real>(mua);
    M.mus = static_cast<Real>(mus);
    M.inv_mus = mus > 0.0 ? static_cast<Real>(1.0 / mus) : std::numeric_limits<Real>::infinity();
    const double nspm = n * (1.0 / vmc::kLightMmPerNs);  // advance(), transport.cpp:169
    M.ns_per_mm = static_cast<Real>(nspm);
    M.mm_per_ns = static_cast<Real>(1.0 / nspm);
    M.n = static_cast<Real>(n);
    M.g = static_cast<Real>(g);
    M.iso = std::fabs(g) < 1e-6 ? 1 : 0;  // hg_cos_theta, transport.cpp:121
    M.ka = static_cast<Real>(-mua * 1.4426950408889634);
    if (!M.iso) {
      M.hg_a = static_cast<Real>((1.0 + g * g) / (2.0 * g));
      M.hg_b = static_cast<Real>(1.0 / (2.0 * g));
      M.hg_c = static_cast<Real>(1.0 - g * g);
      M.hg_d = static_cast<Real>(1.0 - g);
      M.hg_e = static_cast<Real>(2.0 * g);
    }
    // refractive-index class: exact double comparison of n (transport.cpp:218, 242)
    M.nclass = m;
    for (int j = 0; j < m; ++j)
      if (s->media[4 * j + 3] == n) {
        M.nclass = out[j].nclass;
        break;
      }
  }
  return out;
}

// Device allocation. Owning by default; `borrow` points at a cached buffer
// (RangeCache) that outlives the call, so nothing is freed.
struct DevBuf {
  void* p = nullptr;
  int dev = -1;
  size_t cap = 0;
  bool owned = true;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p && owned) {
      int cur = -1;
      cudaGetDevice(&cur);
      if (dev >= 0 && cur != dev) cudaSetDevice(dev);
      cudaFree(p);
      if (dev >= 0 && cur >= 0 && cur != dev) cudaSetDevice(cur);
    }
    p = nullptr;
    cap = 0;
  }
  void alloc(size_t bytes, int device) {
    release();
    dev = device;
    owned = true;
    cap = bytes ? bytes : 16;
    ck(cudaMalloc(&p, cap), "cudaMalloc");
  }
  // grow-only: keep the allocation when it is large enough
  void ensure(size_t bytes, int device) {
    if (!p || cap < bytes || dev != device) alloc(bytes, device);
  }
  void borrow(const DevBuf& from) {
    release();
    p = from.p;
    dev = from.dev;
    cap = from.cap;
    owned = false;
  }
};

// Per-device buffers reused across vmc_run_range calls: cudaMalloc/cudaFree
// churn (measured 10-700 ms of host time per call on B200 boxes) is kept out
// of the executor; the scene itself is still uploaded on every call.
// Scratch of the on-device detector-record sort (sort_records_device).
struct RecSort {
  DevBuf k0, k1, v0, v1, tmp, out;
};

struct RangeCache {
  std::mutex mu;
  DevBuf labels, media, mua, claim, err, cells, totals, det, detn, rep;
  uint64_t labels_digest = 0;  // the volume `labels` holds (valid when labels_n > 0)
  size_t labels_n = 0;
  RecSort rs;
};

RangeCache& range_cache(int device) {
  static RangeCache* caches = new RangeCache[64];  // never destroyed: no cudaFree after CUDA teardown
  if (device < 0 || device >= 64) fail_validation("device index out of range");
  return caches[device];
}

}  // namespace

struct vmc_plan {
  int device = 0;
  vmc_config cfg{};
  int nx = 0, ny = 0, nz = 0, nmedia = 0;
  uint64_t ncells = 0;
  size_t rec_stride = 0;
  DevBuf labels, media, claim, err, mua;
  double voxel_mm = 1.0;
  vmc::KernelArgs args{};
  int sms = 0;
  int block = vmc::kBlock;
  size_t smem = 0, smem_trace = 0;
  int grid = 0, grid_trace = 0;
  bool grid_adaptive = true;  // launch-time grid by photons per thread (VMC_ADAPTIVE_GRID=0: off)
  const void* kern = nullptr;
  const void* kern_trace = nullptr;
  const void* kern_solo = nullptr;  // small-run instantiation of `kern` (K1f FP32 production variants)
  std::string kern_name;  // mangled device symbol of `kern` (cudaFuncGetName)
  int dep = 0;            // deposit path of `kern` (vmc::kDepDirect / kDepWarp / kDepHotBox)
  // fluence-map scratch: nrep replicas (nrep > 1 for small maps) the transport
  // kernel deposits into, folded into the caller's map after each launch. K1f
  // always deposits into the scratch: the fold also books the deposited channel
  int nrep = 1;
  bool scratch = false, fold_books_deposited = false;
  DevBuf rep;
  // runs of one plan share the claim counter and the replica scratch, so each
  // enqueue waits for the previous one (any stream) to finish with them
  cudaEvent_t done = nullptr;
  bool done_valid = false;
  RecSort rs;  // scratch of vmc_plan_sort_records
  DevBuf den;  // K4: (mua * V) * N per label for the photon count den_n

  uint64_t den_n = 0;
  ~vmc_plan() {
    if (done) cudaEventDestroy(done);
  }
};

namespace {

void plan_init(vmc_plan* P, const vmc_scene* s, const vmc_config* c, int device, RangeCache* cache = nullptr) {
  LabelInfo li;
  validate(s, c, &li);
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) fail_validation("device index out of range");
  ck(cudaSetDevice(device), "cudaSetDevice");
  P->device = device;
  P->cfg = *c;
  P->cfg.det = nullptr;
  P->nx = s->nx;
  P->ny = s->ny;
  P->nz = s->nz;
  P->nmedia = s->nmedia;
  const size_t nvox = static_cast<size_t>(s->nx) * s->ny * s->nz;
  P->ncells = static_cast<uint64_t>(nvox) * static_cast<uint64_t>(c->ngates);
  P->rec_stride = vmc_det_record_bytes(s->nmedia);

  auto get = [&](DevBuf& own, DevBuf* shared, size_t bytes) {
    if (shared) {
      shared->ensure(bytes, device);
      own.borrow(*shared);
    } else {
      own.alloc(bytes, device);
    }
  };
  if (cache && cache->labels.p && cache->labels.dev == device && cache->labels.cap >= nvox && cache->labels_n == nvox &&
      cache->labels_digest == li.digest) {
    P->labels.borrow(cache->labels);  // the device already holds this volume
  } else {
    get(P->labels, cache ? &cache->labels : nullptr, nvox);
    if (cache) cache->labels_n = 0;  // invalid until the upload completes
    ck(cudaMemcpy(P->labels.p, s->labels, nvox, cudaMemcpyHostToDevice), "upload labels");
    if (cache) {
      cache->labels_n = nvox;
      cache->labels_digest = li.digest;
    }
  }
  const bool f64 = c->precision == VMC_PRECISION_FP64;
  size_t media_bytes;
  if (f64) {
    auto m = build_media<double>(s);
    media_bytes = m.size() * sizeof(m[0]);
    get(P->media, cache ? &cache->media : nullptr, media_bytes);
    ck(cudaMemcpy(P->media.p, m.data(), media_bytes, cudaMemcpyHostToDevice), "upload media");
  } else {
    auto m = build_media<float>(s);
    media_bytes = m.size() * sizeof(m[0]);
    get(P->media, cache ? &cache->media : nullptr, media_bytes);
    ck(cudaMemcpy(P->media.p, m.data(), media_bytes, cudaMemcpyHostToDevice), "upload media");
  }
  {
    std::vector<double> mua(static_cast<size_t>(s->nmedia));
    for (int m = 0; m < s->nmedia; ++m) mua[m] = s->media[4 * m];
    get(P->mua, cache ? &cache->mua : nullptr, mua.size() * sizeof(double));
    ck(cudaMemcpy(P->mua.p, mua.data(), mua.size() * sizeof(double), cudaMemcpyHostToDevice), "upload mua");
  }
  P->voxel_mm = s->voxel_mm;
  get(P->claim, cache ? &cache->claim : nullptr, sizeof(unsigned long long));
  get(P->err, cache ? &cache->err : nullptr, sizeof(int));
  ck(cudaMemset(P->err.p, 0, sizeof(int)), "cudaMemset");
  ck(cudaEventCreateWithFlags(&P->done, cudaEventDisableTiming), "event");

  vmc::KernelArgs& A = P->args;
  std::memset(&A, 0, sizeof A);
  A.labels = static_cast<const uint8_t*>(P->labels.p);
  A.nx = s->nx;
  A.ny = s->ny;
  A.nz = s->nz;
  A.nxy = static_cast<long long>(s->nx) * s->ny;
  A.nvox = static_cast<long long>(nvox);
  A.h = s->voxel_mm;
  A.nmedia = s->nmedia;
  A.iso_source = s->isotropic ? 1 : 0;
  A.media = P->media.p;
  for (int k = 0; k < 3; ++k) A.src_pos[k] = s->src_pos[k];
  if (!s->isotropic) {
    const HostLaunch L = pencil_launch(s);
    for (int k = 0; k < 3; ++k) {
      A.dir0[k] = L.dir[k];
      A.pos0[k] = L.pos[k];
      A.dir0f[k] = static_cast<float>(L.dir[k]);
      A.pos0f[k] = static_cast<float>(L.pos[k]);
      A.v0[k] = L.v[k];
    }
    A.lab0 = s->labels[static_cast<size_t>(L.v[0]) + static_cast<size_t>(s->nx) * (L.v[1] + static_cast<size_t>(s->ny) * L.v[2])];
  }
  A.seed = c->master_seed;
  A.tmax = c->tmax_ns;
  A.rthr = c->roulette_threshold;
  A.rmult = c->roulette_multiplier;
  A.inv_rmult = 1.0 / c->roulette_multiplier;  // roulette(), transport.cpp:301
  A.reflect = c->boundary_mode == VMC_BOUNDARY_REFLECT ? 1 : 0;
  A.ngates = c->ngates;
  A.inv_gate_w = static_cast<double>(c->ngates) / c->tmax_ns;
  A.qscale = std::ldexp(1.0, quantum_bits(c->photon_count));
  A.claim = static_cast<unsigned long long*>(P->claim.p);
  A.error_flag = static_cast<int*>(P->err.p);

  A.hf = static_cast<float>(A.h);
  A.tmaxf = static_cast<float>(A.tmax);
  A.rthrf = static_cast<float>(A.rthr);
  A.rmultf = static_cast<float>(A.rmult);
  A.inv_rmultf = static_cast<float>(A.inv_rmult);
  A.inv_gate_wf = static_cast<float>(A.inv_gate_w);
  A.gate_wf = static_cast<float>(c->tmax_ns / c->ngates);
  A.qscalef = static_cast<float>(A.qscale);
  A.scatter_pct = env_int("VMC_SCATTER_PCT", 50);
  A.refill_min = env_int("VMC_REFILL_MIN", 1);  // measured: 1 >= 2 > 3 > 4
  A.ndet = c->ndet;
  A.nppath = std::max(0, s->nmedia - 1);
  A.rec_stride = static_cast<int>(P->rec_stride);
  for (int k = 0; k < c->ndet; ++k)
    for (int j = 0; j < 4; ++j) A.det[k][j] = c->det[4 * k + j];
  for (int k = 0; k < c->ndet; ++k) {
    for (int j = 0; j < 3; ++j) A.detf[k][j] = static_cast<float>(c->det[4 * k + j]);
    A.detf[k][3] = static_cast<float>(c->det[4 * k + 3] * c->det[4 * k + 3]);
  }
  A.det_cap = c->det_capacity;

  const bool gates = c->ngates > 1, det = c->ndet > 0;
  bool uniform = li.uniform;  // single-label volume -> specialised kernel (identical results)
  {
    const uint8_t l0 = s->labels[0];
    const char* ku = std::getenv("VMC_UNIFORM_FASTPATH");
    if (ku && ku[0] == '0') uniform = false;
    if (uniform && l0 < s->nmedia) {
      A.uni_f = build_media<float>(s)[l0];
      A.uni_d = build_media<double>(s)[l0];
    } else {
      uniform = false;
    }
  }
  // measured: 70-80 flat, 75 best by 0.3 %; clamped so a warp always walks while >= 1 lane of 32 does
  A.event_pct = std::min(100, std::max(4, env_int("VMC_EVENT_PCT", 75)));
  A.walk_keep = (32 * (100 - A.event_pct)) / 100;
  {
    // scatter chain for strongly scattering volumes (max mus * h >= 10: most
    // flights end in their voxel); VMC_SCATTER_CHAIN overrides the lane count
    double mx = 0.0;
    for (int m = 0; m < s->nmedia; ++m) mx = std::max(mx, s->media[4 * m + 1] * s->voxel_mm);
    A.chain_min = std::max(0, std::min(32, env_int("VMC_SCATTER_CHAIN", mx >= 10.0 ? 22 : 0)));
  }
  // K1f (flight.cuh) in the launch's precision unless VMC_KERNEL=step selects
  // the per-step K1 (transport.cuh) for A/B runs. FP64 K1f is the
  // exact-arithmetic pin of the product kernel's structure.
  const char* kk = std::getenv("VMC_KERNEL");
  const bool step_kernel = kk && std::strcmp(kk, "step") == 0;
  if (step_kernel) {
    P->kern = f64 ? vmc::transport_kernel_double(gates, det, false, uniform)
                  : vmc::transport_kernel_float(gates, det, false, uniform);
    P->kern_trace = f64 ? vmc::transport_kernel_double(gates, det, true, uniform)
                        : vmc::transport_kernel_float(gates, det, true, uniform);
  } else if (f64) {
    P->kern = vmc::flight_kernel_double(gates, det, false, uniform);
    P->kern_trace = vmc::flight_kernel_double(gates, det, true, uniform);
  } else {
    // VMC_DEPOSIT=warp|hotbox: the warp-aggregated / SM-local hot-box deposit
    // paths (A/B; built for the production variants, direct elsewhere)
    const char* dp = std::getenv("VMC_DEPOSIT");
    int dep = vmc::kDepDirect;
    if (dp && std::strcmp(dp, "warp") == 0) dep = vmc::kDepWarp;
    if (dp && std::strcmp(dp, "hotbox") == 0 && s->nx >= vmc::kHotBoxN && s->ny >= vmc::kHotBoxN &&
        s->nz >= vmc::kHotBoxN)
      dep = vmc::kDepHotBox;
    P->kern = dep != vmc::kDepDirect ? vmc::flight_kernel_float(gates, det, false, uniform, dep) : nullptr;
    if (P->kern) {
      P->dep = dep;
    } else {
      P->kern = vmc::flight_kernel_float(gates, det, false, uniform, vmc::kDepDirect);
    }
    P->kern_trace = vmc::flight_kernel_float(gates, det, true, uniform, vmc::kDepDirect);
    if (P->dep == vmc::kDepDirect && env_int("VMC_SOLO", 1) != 0)
      P->kern_solo = vmc::flight_kernel_float(gates, det, false, uniform, vmc::kDepDirect, true);
    if (P->dep == vmc::kDepHotBox) {
      // 16^3 box around the source voxel, clamped into the grid
      const int n3[3] = {s->nx, s->ny, s->nz};
      for (int k = 0; k < 3; ++k) {
        const double p = s->isotropic ? s->src_pos[k] / s->voxel_mm : static_cast<double>(A.v0[k]);
        const int c = static_cast<int>(std::floor(p)) - vmc::kHotBoxN / 2;
        A.hb0[k] = std::max(0, std::min(c, n3[k] - vmc::kHotBoxN));
      }
    }
  }
  {
    const char* nm = nullptr;
    if (cudaFuncGetName(&nm, P->kern) == cudaSuccess && nm) P->kern_name = nm;
    else cudaGetLastError();
  }
  // media table, plus per-thread per-label path lengths in detector mode (one
  // slot per interior label; K1 and K1f both place them after the media)
  P->smem = ((media_bytes + 15) & ~static_cast<size_t>(15)) +
            (det ? static_cast<size_t>(std::max(1, s->nmedia - 1)) * vmc::kBlock * (f64 ? sizeof(double) : sizeof(float))
                 : 0);
  // K1f adds its per-thread disposition slots and per-warp seed stashes (the
  // kernel places them at compile-time offsets in front of the media table)
  P->smem = ((P->smem + 15) & ~static_cast<size_t>(15)) + 3 * vmc::kBlock * sizeof(long long) +
            (vmc::kBlock / 32) * vmc::flight_stash_bytes(f64 ? sizeof(double) : sizeof(float));
  P->smem_trace = P->smem;
  if (P->dep == vmc::kDepHotBox) P->smem += vmc::kHotBoxBytes;
  ck(cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, device), "sm count");
  ck(cudaFuncSetAttribute(P->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P->smem)), "smem attr");
  ck(cudaFuncSetAttribute(P->kern_trace, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P->smem_trace)),
     "smem attr");
  if (P->kern_solo)
    ck(cudaFuncSetAttribute(P->kern_solo, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P->smem)),
       "smem attr");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, P->kern, P->block, P->smem), "occupancy");
  {
    const int cap = env_int("VMC_CTAS_PER_SM", 0);  // A/B knob: fewer resident CTAs per SM
    if (cap > 0) per_sm = std::min(per_sm, cap);
    P->grid_adaptive = env_int("VMC_ADAPTIVE_GRID", 1) != 0 && cap <= 0;
  }
  P->grid = std::max(1, per_sm) * P->sms;
  {
    // Shared-memory carveout: just what the resident CTAs need, so the rest of
    // the SM's L1/shared array caches the label volume (read through __ldg on
    // every face of multi-label volumes). Left to itself the driver picked the
    // 132 KB configuration for B3's 4 x 21 KB (ncu launch__shared_mem_config_size).
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    const int pct_env = env_int("VMC_SMEM_CARVEOUT", -1);
    if (max_smem > 0 && pct_env != 0) {
      const long need = static_cast<long>(std::max(1, per_sm)) * (static_cast<long>(P->smem) + 1024);
      int pct = pct_env > 0 ? pct_env : static_cast<int>((need * 100 + max_smem - 1) / max_smem);
      pct = std::max(1, std::min(100, pct));
      cudaFuncSetAttribute(P->kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      cudaFuncSetAttribute(P->kern_trace, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      if (P->kern_solo) cudaFuncSetAttribute(P->kern_solo, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      cudaGetLastError();
    }
  }
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, P->kern_trace, P->block, P->smem_trace), "occupancy");
  P->grid_trace = std::max(1, per_sm) * P->sms;

  // Fluence-map replicas. The deposits of all photons funnel through the few
  // voxels next to the source, and same-address red.add throughput in L2 is
  // what limits a cube60 launch (measured: the kernel time moved by 35 % with
  // the map's base address alone). Each CTA therefore adds into one of nrep
  // copies of the map (CTA index mod nrep); one fold kernel sums them into
  // the caller's map. Integer adds: the result is bit-identical for any nrep.
  // Only small maps are replicated (nrep * map <= 64 MB, well inside L2).
  {
    const size_t map_bytes = static_cast<size_t>(P->ncells) * sizeof(int64_t);
    int r = env_int("VMC_MAP_REPLICAS", -1);
    if (r < 0) {
      r = 8;  // measured: 4, 8 and 16 equal on cube60, 1 up to 35 % slower
      while (r > 1 && static_cast<size_t>(r) * map_bytes > (64u << 20)) r >>= 1;
    }
    int p2 = 1;
    while (p2 * 2 <= std::max(1, r)) p2 *= 2;
    P->nrep = p2;
    P->fold_books_deposited = !step_kernel;  // K1f keeps no deposited accumulator
    P->scratch = P->nrep > 1 || P->fold_books_deposited;
    if (P->scratch) get(P->rep, cache ? &cache->rep : nullptr, static_cast<size_t>(P->nrep) * map_bytes);
    A.rep_mask = P->nrep - 1;
    A.rep_stride = static_cast<long long>(P->ncells);
    if (static_cast<uint64_t>(P->nrep - 1) * P->ncells >= (1ull << 31)) fail_runtime("replica offsets overflow");
  }
}

// cells (+)= sum of the nrep scratch replicas; with `book`, the sum of every
// added quantum goes to totals[0] (the deposited channel, exact in integers)
__global__ void k_fold_replicas(unsigned long long* __restrict__ cells, const unsigned long long* __restrict__ rep,
                                int nrep, uint64_t ncells, int overwrite, unsigned long long* totals, int book) {
  unsigned long long part = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < ncells;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned long long acc = 0;
    for (int r = 0; r < nrep; ++r) acc += __ldcs(rep + static_cast<uint64_t>(r) * ncells + i);
    cells[i] = overwrite ? acc : cells[i] + acc;
    part += acc;
  }
  if (!book) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  __shared__ unsigned long long warp_sum[32];
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += warp_sum[w];
    if (t) atomicAdd(totals, t);
  }
}

struct DepLog {
  long long* cells = nullptr;
  double* w = nullptr;
  unsigned long long* n = nullptr;
  unsigned long long cap = 0;
};

void plan_enqueue(vmc_plan* P, uint64_t first, uint64_t count, int64_t* d_cells, int64_t* d_totals,
                  void* d_det, uint64_t* d_det_count, cudaStream_t st, uint32_t flags, bool trace,
                  vmc_photon_trace* d_trace, const DepLog* log = nullptr) {
  if (!d_cells || !d_totals) fail_validation("device cells/totals buffers are required");
  if (P->cfg.ndet > 0 && P->cfg.det_capacity > 0 && !d_det) fail_validation("detector buffer is required");
  if (P->cfg.ndet > 0 && !d_det_count) fail_validation("detector count buffer is required");
  if (first + count < first) fail_validation("photon range overflows");
  ck(cudaSetDevice(P->device), "cudaSetDevice");
  // serialise with the previous run of this plan (shared claim counter and
  // replica scratch), whatever stream it was enqueued on
  if (P->done_valid) ck(cudaStreamWaitEvent(st, P->done, 0), "wait previous run");
  const bool zero = (flags & VMC_RUN_ZERO) != 0;
  if (zero) {
    // with a scratch map the fold overwrites the caller's cells instead
    if (!P->scratch || count == 0) ck(cudaMemsetAsync(d_cells, 0, P->ncells * sizeof(int64_t), st), "zero cells");
    ck(cudaMemsetAsync(d_totals, 0, 4 * sizeof(int64_t), st), "zero totals");
    if (d_det_count) ck(cudaMemsetAsync(d_det_count, 0, sizeof(uint64_t), st), "zero det count");
  }
  if (count == 0) return;
  ck(cudaMemsetAsync(P->claim.p, 0, sizeof(unsigned long long), st), "zero claim");
  vmc::KernelArgs A = P->args;
  A.first = first;
  A.count = count;
  A.cells = reinterpret_cast<long long*>(d_cells);
  if (P->scratch) {
    ck(cudaMemsetAsync(P->rep.p, 0, static_cast<size_t>(P->nrep) * P->ncells * sizeof(int64_t), st), "zero replicas");
    A.cells = static_cast<long long*>(P->rep.p);
  }
  A.totals = reinterpret_cast<long long*>(d_totals);
  A.det_out = static_cast<unsigned char*>(d_det);
  A.det_count = reinterpret_cast<unsigned long long*>(d_det_count);
  A.trace = d_trace;
  if (trace && log) {  // vmc_simulate_photon: per-step deposit log
    A.dep_cells = log->cells;
    A.dep_w = log->w;
    A.dep_n = log->n;
    A.dep_cap = log->cap;
  }
  // never launch more persistent threads than photons need
  const uint64_t need_blocks = (count + P->block - 1) / P->block;
  int full = trace ? P->grid_trace : P->grid;
  // Small runs: fewer resident CTAs per SM. With only a few photons per
  // resident thread the run ends when the longest horizon-truncated photon
  // chain does (~1150 dependent scatters in B1), and that chain advances
  // faster on a less contended SM. Measured on B200 (profiles/README.md,
  // "small photon counts"): of 4 CTAs/SM, 2 are best below ~7 photons per
  // full-grid thread (B1 at 1e6: +19 %), 3 below ~30, all 4 above.
  const void* kern = trace ? P->kern_trace : P->kern;
  if (!trace && P->grid_adaptive && full >= 4 * P->sms) {
    const int per = full / P->sms;
    const double r = static_cast<double>(count) / (static_cast<double>(full) * P->block);
    const int c = r < 7.0 ? per / 2 : (r < 30.0 ? per - per / 4 : per);
    full = c * P->sms;
    // ... and the small-run instantiation (lane-local loop for a warp's last
    // photon once the claims have run out); identical results
    if (r < 30.0 && P->kern_solo) kern = P->kern_solo;
  }
  const int grid = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(full), std::max<uint64_t>(1, need_blocks)));
  {
    void* argv[] = {&A};
    ck(cudaLaunchKernel(kern, dim3(grid), dim3(P->block), argv,
                        trace ? P->smem_trace : P->smem, st),
       "launch transport");
  }
  if (P->scratch) {
    const int fb = static_cast<int>(std::min<uint64_t>((P->ncells + 255) / 256, static_cast<uint64_t>(P->sms) * 8));
    k_fold_replicas<<<fb, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(d_cells),
                                        static_cast<const unsigned long long*>(P->rep.p), P->nrep, P->ncells,
                                        zero ? 1 : 0, reinterpret_cast<unsigned long long*>(d_totals),
                                        P->fold_books_deposited ? 1 : 0);
    ck(cudaGetLastError(), "fold replicas");
  }
  ck(cudaEventRecord(P->done, st), "record run");
  P->done_valid = true;
}

void check_launch_errors(vmc_plan* P) {
  int h = 0;
  ck(cudaMemcpy(&h, P->err.p, sizeof(int), cudaMemcpyDeviceToHost), "read error flag");
  if (h) {
    cudaMemset(P->err.p, 0, sizeof(int));
    fail_validation("source entry point maps outside the voxel grid");
  }
}

// Sort packed detector records by photon index (deterministic output for any
// device count / claim order). Host fallback for ranges wider than 2^32.
void sort_records(unsigned char* recs, uint64_t n, size_t stride) {
  if (n < 2) return;
  std::vector<uint64_t> order(n);
  std::iota(order.begin(), order.end(), uint64_t{0});
  auto key = [&](uint64_t i) {
    uint64_t k;
    std::memcpy(&k, recs + i * stride, sizeof k);
    return k;
  };
  std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return key(a) < key(b); });
  std::vector<unsigned char> tmp(n * stride);
  for (uint64_t i = 0; i < n; ++i) std::memcpy(tmp.data() + i * stride, recs + order[i] * stride, stride);
  std::memcpy(recs, tmp.data(), n * stride);
}

__global__ void k_rec_keys(const unsigned char* __restrict__ recs, uint32_t n, uint32_t stride, uint64_t first,
                           uint32_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    keys[i] = static_cast<uint32_t>(*reinterpret_cast<const uint64_t*>(recs + static_cast<size_t>(i) * stride) - first);
    idx[i] = i;
  }
}

// one 32-bit word per thread: record r = w / words_per_record (stride % 4 == 0)
__global__ void k_rec_gather(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                             const uint32_t* __restrict__ order, uint64_t nwords, uint32_t wpr) {
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < nwords;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = w / wpr, k = w - r * wpr;
    dst[w] = src[static_cast<uint64_t>(order[r]) * wpr + k];
  }
}

// Sort n records (photon indices in [first, first + count), count <= 2^32) on
// the device: radix sort of the 32-bit index offsets (only the bits count
// needs) carrying record positions, then a gather into `out` (R.out when
// null). Returns the sorted records.
const void* sort_records_device(const void* d_recs, uint64_t n, size_t stride, uint64_t first, uint64_t count,
                                RecSort& R, int device, cudaStream_t st, void* out = nullptr) {
  if (n < 2) {
    if (out && n) ck(cudaMemcpyAsync(out, d_recs, n * stride, cudaMemcpyDeviceToDevice, st), "copy records");
    return out && n ? out : d_recs;
  }
  const uint32_t n32 = static_cast<uint32_t>(n);
  R.k0.ensure(n * 4, device);
  R.k1.ensure(n * 4, device);
  R.v0.ensure(n * 4, device);
  R.v1.ensure(n * 4, device);
  if (!out) {
    R.out.ensure(n * stride, device);
    out = R.out.p;
  }
  int end_bit = 1;
  while (end_bit < 32 && (count - 1) >> end_bit) ++end_bit;
  auto* k0 = static_cast<uint32_t*>(R.k0.p);
  auto* k1 = static_cast<uint32_t*>(R.k1.p);
  auto* v0 = static_cast<uint32_t*>(R.v0.p);
  auto* v1 = static_cast<uint32_t*>(R.v1.p);
  size_t tb = 0;
  ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, static_cast<int>(n32), 0, end_bit, st), "cub sort");
  R.tmp.ensure(tb, device);
  k_rec_keys<<<(n32 + 255) / 256, 256, 0, st>>>(static_cast<const unsigned char*>(d_recs), n32,
                                                 static_cast<uint32_t>(stride), first, k0, v0);
  ck(cub::DeviceRadixSort::SortPairs(R.tmp.p, tb, k0, k1, v0, v1, static_cast<int>(n32), 0, end_bit, st), "cub sort");
  const uint64_t nwords = n * (stride / 4);
  const int grid = static_cast<int>(std::min<uint64_t>((nwords + 255) / 256, 148ull * 16));
  k_rec_gather<<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(d_recs), static_cast<uint32_t*>(out), v1, nwords,
                                     static_cast<uint32_t>(stride / 4));
  ck(cudaGetLastError(), "record sort");
  return out;
}

// ---- one device, host buffers ---------------------------------------------
struct RangeResult {
  std::vector<int64_t> cells;
  int64_t totals[4] = {0, 0, 0, 0};
  std::vector<unsigned char> det;
  uint64_t det_count = 0;
  double ms = 0.0;
};

// VMC_DEBUG_TIMING=1 prints the host-side phases of vmc_run_range to stderr.
struct PhaseClock {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  PhaseClock() : on(std::getenv("VMC_DEBUG_TIMING") != nullptr) { t0 = last = std::chrono::steady_clock::now(); }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[vmc] %-12s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  }
};

void run_range_device(const vmc_scene* s, const vmc_config* c, uint64_t first, uint64_t count, int device,
                      int64_t* cells_out, int64_t* totals_out, unsigned char* det_out, uint64_t* det_count_out,
                      double* ms_out) {
  PhaseClock clk;
  RangeCache& C = range_cache(device);
  std::lock_guard<std::mutex> lock(C.mu);  // one in-flight call per device
  vmc_plan P;
  plan_init(&P, s, c, device, &C);
  clk.mark("plan_init");
  const uint64_t cap = c->ndet > 0 ? c->det_capacity : 0;
  C.cells.ensure(P.ncells * sizeof(int64_t), device);
  C.totals.ensure(4 * sizeof(int64_t), device);
  C.det.ensure(cap * P.rec_stride, device);
  C.detn.ensure(sizeof(uint64_t), device);
  DevBuf& cells = C.cells;
  DevBuf& totals = C.totals;
  DevBuf& det = C.det;
  DevBuf& detn = C.detn;
  cudaStream_t st;
  ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  clk.mark("alloc");
  try {
    ck(cudaEventRecord(e0, st), "event record");
    plan_enqueue(&P, first, count, static_cast<int64_t*>(cells.p), static_cast<int64_t*>(totals.p), det.p,
                 static_cast<uint64_t*>(detn.p), st, VMC_RUN_ZERO, false, nullptr);
    clk.mark("enqueue");
    ck(cudaEventRecord(e1, st), "event record");
    if (cells_out)
      ck(cudaMemcpyAsync(cells_out, cells.p, P.ncells * sizeof(int64_t), cudaMemcpyDeviceToHost, st), "download");
    if (totals_out) ck(cudaMemcpyAsync(totals_out, totals.p, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, st), "download");
    uint64_t n = 0;
    ck(cudaMemcpyAsync(&n, detn.p, sizeof n, cudaMemcpyDeviceToHost, st), "download");
    ck(cudaStreamSynchronize(st), "run");
    clk.mark("sync");
    if (c->ndet > 0) {
      const uint64_t keep = std::min(n, cap);
      if (det_out && keep) {
        if (count <= (1ull << 32) && P.rec_stride % 4 == 0 && keep < (1ull << 31)) {
          const void* sorted = sort_records_device(det.p, keep, P.rec_stride, first, count, C.rs, device, st);
          ck(cudaMemcpyAsync(det_out, sorted, keep * P.rec_stride, cudaMemcpyDeviceToHost, st), "download det");
          ck(cudaStreamSynchronize(st), "sort det");
        } else {
          ck(cudaMemcpy(det_out, det.p, keep * P.rec_stride, cudaMemcpyDeviceToHost), "download det");
          sort_records(det_out, keep, P.rec_stride);
        }
      }
    }
    if (det_count_out) *det_count_out = c->ndet > 0 ? n : 0;
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    if (ms_out) *ms_out = ms;
    check_launch_errors(&P);
  } catch (...) {
    cudaStreamDestroy(st);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    throw;
  }
  cudaStreamDestroy(st);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  clk.mark("finish");
}

// ---- NCCL, loaded on demand (only vmc_run_multi with ndev > 1 needs it) ----
struct Nccl {
  void* h = nullptr;
  int (*CommInitAll)(void** comms, int ndev, const int* devlist) = nullptr;
  int (*CommDestroy)(void* comm) = nullptr;
  int (*Reduce)(const void*, void*, size_t, int, int, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(dlsym(n.h, "ncclCommInitAll"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(n.h, "ncclCommDestroy"));
    n.Reduce = reinterpret_cast<decltype(n.Reduce)>(dlsym(n.h, "ncclReduce"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(n.h, "ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(n.h, "ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(n.h, "ncclGetErrorString"));
  });
  if (!n.h || !n.CommInitAll || !n.Reduce || !n.GroupStart || !n.GroupEnd)
    fail_runtime("NCCL (libnccl.so.2) is required for multi-GPU runs and could not be loaded");
  return n;
}


void nck(int r, const char* what) {
  if (r != 0) {
    Nccl& n = nccl();
    fail_runtime(std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "nccl error"));
  }
}

// Communicators per device list, created once (ncclCommInitAll costs far more
// than a cube60 reduce) and kept for the life of the process.
std::vector<void*>& nccl_comms(const int* devices, int ndev) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<void*>>* cache = new std::map<std::vector<int>, std::vector<void*>>;
  std::lock_guard<std::mutex> lock(mu);
  std::vector<int> key(devices, devices + ndev);
  auto it = cache->find(key);
  if (it != cache->end()) return it->second;
  Nccl& N = nccl();
  std::vector<void*> comms(ndev, nullptr);
  nck(N.CommInitAll(comms.data(), ndev, devices), "ncclCommInitAll");
  return cache->emplace(std::move(key), std::move(comms)).first->second;
}

constexpr int kNcclInt64 = 4;  // ncclInt64
constexpr int kNcclSum = 0;    // ncclSum

}  // namespace

namespace {
// K4: normalize (fluence.cpp:62-90). HBM-streaming pass: each thread handles a
// PAIR of consecutive voxels (16-byte int64x2 loads, 8-byte float2 stores);
// up to 8 gate loads are in flight before the first store. The arithmetic is
// the reference's, operation for operation, so the f32 volume is bit-identical
// to FluenceMap::normalize + to_float_volume:
//   value = (double(cell) * quantum) / den[label],  den = (mua * V) * N
// (den per label precomputed on the host in the reference's order; den == 0
// for mua == 0 voxels -> 0); raw mode: value = double(cell) * quantum.
// Gate-summed (CW) output sums the int64 cells first, like the reference's
// single map.
__device__ __forceinline__ float k4_value(long long c, double q, double den, int normalized) {
  const double raw = static_cast<double>(c) * q;
  if (!normalized) return static_cast<float>(raw);
  return den > 0.0 ? static_cast<float>(raw / den) : 0.0f;
}

__global__ void k_normalize(const long long* __restrict__ cells, const uint8_t* __restrict__ labels,
                            const double* __restrict__ den, long long nvox, int ngates, int sum_gates,
                            int normalized, double q, float* __restrict__ out) {
  const long long npair = nvox >> 1;
  const bool vec = (nvox & 1) == 0;  // pairs never straddle a gate boundary
  const long long nwork = vec ? npair : nvox;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nwork;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int per = vec ? 2 : 1;
    const long long v0 = i * per;
    double d[2] = {0.0, 0.0};
    if (normalized)
      for (int j = 0; j < per; ++j) d[j] = den[__ldg(labels + v0 + j)];
    if (sum_gates) {
      long long raw[2] = {0, 0};
      for (int g = 0; g < ngates; ++g) {
        if (vec) {
          const longlong2 c = __ldcs(reinterpret_cast<const longlong2*>(cells + v0 + g * nvox));
          raw[0] += c.x;
          raw[1] += c.y;
        } else {
          raw[0] += __ldcs(cells + v0 + g * nvox);
        }
      }
      if (vec)
        __stcs(reinterpret_cast<float2*>(out + v0),
               make_float2(k4_value(raw[0], q, d[0], normalized), k4_value(raw[1], q, d[1], normalized)));
      else
        out[v0] = k4_value(raw[0], q, d[0], normalized);
    } else {
      for (int g0 = 0; g0 < ngates; g0 += 8) {
        longlong2 buf[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (g0 + k < ngates) {
            if (vec) buf[k] = __ldcs(reinterpret_cast<const longlong2*>(cells + v0 + (g0 + k) * nvox));
            else buf[k] = make_longlong2(__ldcs(cells + v0 + (g0 + k) * nvox), 0);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (g0 + k < ngates) {
            const float a = k4_value(buf[k].x, q, d[0], normalized);
            if (vec) {
              const float b = k4_value(buf[k].y, q, d[1], normalized);
              __stcs(reinterpret_cast<float2*>(out + v0 + (g0 + k) * nvox), make_float2(a, b));
            } else {
              __stcs(out + v0 + (g0 + k) * nvox, a);
            }
          }
        }
      }
    }
  }
}

// K3 fallback: dst += src over int64 cells (exact integer sum, order-free).
__global__ void k_add_i64(long long* __restrict__ dst, const long long* __restrict__ src, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}

void add_i64(int64_t* dst, const int64_t* src, uint64_t n, cudaStream_t st) {
  const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, 148ull * 8));
  k_add_i64<<<std::max(grid, 1), 256, 0, st>>>(reinterpret_cast<long long*>(dst),
                                               reinterpret_cast<const long long*>(src), static_cast<long long>(n));
  ck(cudaGetLastError(), "launch add_i64");
}

__global__ void k_rng_kat(uint64_t seed, uint64_t stream, int n, uint64_t* out) {
  vmc::Xs128p<false> r;
  r.seed(seed, stream);
  for (int i = 0; i < n; ++i) out[i] = r.next();
}
}  // namespace

// ============================================================================
extern "C" {

int vmc_rng_kat(uint64_t seed, uint64_t stream_id, int n, int device, uint64_t* out) {
  return guarded([&] {
    if (n < 0 || (n > 0 && !out)) fail_validation("rng_kat: bad output");
    ck(cudaSetDevice(device), "cudaSetDevice");
    DevBuf d;
    d.alloc(static_cast<size_t>(n) * sizeof(uint64_t), device);
    k_rng_kat<<<1, 1>>>(seed, stream_id, n, static_cast<uint64_t*>(d.p));
    ck(cudaGetLastError(), "launch rng_kat");
    ck(cudaMemcpy(out, d.p, static_cast<size_t>(n) * sizeof(uint64_t), cudaMemcpyDeviceToHost), "download");
  });
}

size_t vmc_det_record_bytes(int32_t nmedia) {
  const size_t raw = sizeof(vmc_det_record_head) + sizeof(float) * static_cast<size_t>(nmedia > 1 ? nmedia - 1 : 0);
  return (raw + 7) & ~static_cast<size_t>(7);
}

int vmc_abi_version(void) { return VMC_ABI_VERSION; }

const char* vmc_last_error(void) { return g_last_error.c_str(); }

int vmc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

double vmc_quantum_for(uint64_t photon_count) { return std::ldexp(1.0, -quantum_bits(photon_count)); }

int vmc_validate(const vmc_scene* scene, const vmc_config* config) {
  return guarded([&] { validate(scene, config); });
}

int vmc_run_range(const vmc_scene* scene, const vmc_config* config, uint64_t first_index, uint64_t count,
                  int device, int64_t* cells_out, vmc_disposition* totals_out, void* det_out,
                  uint64_t* det_count_out, double* wall_ms_out) {
  return guarded([&] {
    int64_t tot[4] = {0, 0, 0, 0};
    run_range_device(scene, config, first_index, count, device, cells_out, tot,
                     static_cast<unsigned char*>(det_out), det_count_out, wall_ms_out);
    if (totals_out) {
      totals_out->deposited_q = tot[0];
      totals_out->escaped_q = tot[1];
      totals_out->killed_q = tot[2];
      totals_out->truncated_q = tot[3];
      totals_out->quantum = vmc_quantum_for(config->photon_count);
    }
  });
}

int vmc_run_multi(const vmc_scene* scene, const vmc_config* config, int ndev, const int* devices,
                  const uint64_t* counts, int64_t* cells_out, vmc_disposition* totals_out, void* det_out,
                  uint64_t* det_count_out, double* per_device_ms, double* reduce_ms) {
  return guarded([&] {
    validate(scene, config);
    if (ndev < 1 || !devices || !counts) fail_validation("run_multi: no devices");
    std::vector<uint64_t> first(ndev);
    uint64_t next = 0;  // contiguous ranges in device order (scheduler.cpp:405-410)
    for (int i = 0; i < ndev; ++i) {
      first[i] = next;
      next += counts[i];
    }
    const size_t stride = vmc_det_record_bytes(scene->nmedia);
    const uint64_t cap = config->ndet > 0 ? config->det_capacity : 0;

    struct Slot {
      std::unique_ptr<vmc_plan> plan;
      DevBuf cells, totals, det, detn;
      RecSort rs;
      cudaStream_t st = nullptr;
      double ms = 0.0;
      uint64_t ndet = 0;
      std::string err;
      int code = 0;
    };
    std::vector<Slot> slot(ndev);
    auto worker = [&](int i) {
      Slot& S = slot[i];
      S.code = guarded([&] {
        const int dev = devices[i];
        S.plan.reset(new vmc_plan);
        plan_init(S.plan.get(), scene, config, dev);
        S.cells.alloc(S.plan->ncells * sizeof(int64_t), dev);
        S.totals.alloc(4 * sizeof(int64_t), dev);
        S.det.alloc(cap * stride, dev);
        S.detn.alloc(sizeof(uint64_t), dev);
        ck(cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking), "stream");
        cudaEvent_t e0, e1;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        ck(cudaEventRecord(e0, S.st), "event");
        plan_enqueue(S.plan.get(), first[i], counts[i], static_cast<int64_t*>(S.cells.p),
                     static_cast<int64_t*>(S.totals.p), S.det.p, static_cast<uint64_t*>(S.detn.p), S.st,
                     VMC_RUN_ZERO, false, nullptr);
        ck(cudaEventRecord(e1, S.st), "event");
        ck(cudaStreamSynchronize(S.st), "run");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        S.ms = ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        ck(cudaMemcpy(&S.ndet, S.detn.p, sizeof(uint64_t), cudaMemcpyDeviceToHost), "det count");
        check_launch_errors(S.plan.get());
      });
      if (S.code) S.err = g_last_error;
    };
    std::vector<std::thread> pool;
    for (int i = 0; i < ndev; ++i) pool.emplace_back(worker, i);
    for (auto& th : pool) th.join();
    auto cleanup = [&] {
      for (auto& S : slot)
        if (S.st) {
          cudaSetDevice(S.plan ? S.plan->device : 0);
          cudaStreamDestroy(S.st);
          S.st = nullptr;
        }
    };
    for (int i = 0; i < ndev; ++i)
      if (slot[i].code) {
        cleanup();
        throw VmcError(slot[i].code, slot[i].err);
      }
    const uint64_t ncells = slot[0].plan->ncells;
    double red_ms = 0.0;
    try {
      bool distinct = true;
      for (int i = 0; i < ndev; ++i)
        for (int j = 0; j < i; ++j) distinct &= devices[i] != devices[j];
      const char* mode = std::getenv("VMC_MULTI_REDUCE");
      const bool want_peer = !distinct || (mode && std::strcmp(mode, "peer") == 0);
      if (ndev > 1 && want_peer) {
        // device-side reduce without NCCL (repeated devices, or forced): peer copy
        // of each partial map into a scratch buffer on devices[0] + an int64 add
        // kernel there. Same integer sums as the NCCL path.
        cudaSetDevice(devices[0]);
        DevBuf scratch;
        scratch.alloc((ncells + 4) * sizeof(int64_t), devices[0]);
        cudaEvent_t r0, r1;
        ck(cudaEventCreate(&r0), "event");
        ck(cudaEventCreate(&r1), "event");
        ck(cudaEventRecord(r0, slot[0].st), "event");
        for (int i = 1; i < ndev; ++i) {
          int64_t* sc = static_cast<int64_t*>(scratch.p);
          ck(cudaMemcpyPeerAsync(sc, devices[0], slot[i].cells.p, devices[i], ncells * sizeof(int64_t), slot[0].st),
             "peer copy");
          ck(cudaMemcpyPeerAsync(sc + ncells, devices[0], slot[i].totals.p, devices[i], 4 * sizeof(int64_t),
                                 slot[0].st),
             "peer copy");
          add_i64(static_cast<int64_t*>(slot[0].cells.p), sc, ncells, slot[0].st);
          add_i64(static_cast<int64_t*>(slot[0].totals.p), sc + ncells, 4, slot[0].st);
        }
        ck(cudaEventRecord(r1, slot[0].st), "event");
        ck(cudaStreamSynchronize(slot[0].st), "reduce");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r0, r1);
        red_ms = ms;
        cudaEventDestroy(r0);
        cudaEventDestroy(r1);
      } else if (ndev > 1) {
        // one exchange step: NCCL reduce of the int64 maps + totals onto devices[0]
        Nccl& N = nccl();
        static std::mutex reduce_mu;  // cached communicators: one reduce at a time
        std::lock_guard<std::mutex> reduce_lock(reduce_mu);
        std::vector<void*>& comms = nccl_comms(devices, ndev);
        cudaSetDevice(devices[0]);
        cudaEvent_t r0, r1;
        ck(cudaEventCreate(&r0), "event");
        ck(cudaEventCreate(&r1), "event");
        ck(cudaEventRecord(r0, slot[0].st), "event");
        nck(N.GroupStart(), "ncclGroupStart");
        for (int i = 0; i < ndev; ++i) {
          cudaSetDevice(devices[i]);
          nck(N.Reduce(slot[i].cells.p, slot[i].cells.p, ncells, kNcclInt64, kNcclSum, 0, comms[i], slot[i].st),
              "ncclReduce");
          nck(N.Reduce(slot[i].totals.p, slot[i].totals.p, 4, kNcclInt64, kNcclSum, 0, comms[i], slot[i].st),
              "ncclReduce");
        }
        nck(N.GroupEnd(), "ncclGroupEnd");
        cudaSetDevice(devices[0]);
        ck(cudaEventRecord(r1, slot[0].st), "event");
        for (int i = 0; i < ndev; ++i) {
          cudaSetDevice(devices[i]);
          ck(cudaStreamSynchronize(slot[i].st), "reduce");
        }
        float ms = 0.f;
        cudaSetDevice(devices[0]);
        cudaEventElapsedTime(&ms, r0, r1);
        red_ms = ms;
        cudaEventDestroy(r0);
        cudaEventDestroy(r1);
      }
      cudaSetDevice(devices[0]);
      if (cells_out)
        ck(cudaMemcpy(cells_out, slot[0].cells.p, ncells * sizeof(int64_t), cudaMemcpyDeviceToHost), "download");
      int64_t tot[4];
      ck(cudaMemcpy(tot, slot[0].totals.p, sizeof tot, cudaMemcpyDeviceToHost), "download");
      if (totals_out) {
        totals_out->deposited_q = tot[0];
        totals_out->escaped_q = tot[1];
        totals_out->killed_q = tot[2];
        totals_out->truncated_q = tot[3];
        totals_out->quantum = vmc_quantum_for(config->photon_count);
      }
      // detector records: gather in device order, then sort by photon index
      uint64_t total_det = 0, stored = 0;
      bool host_sort = false;
      for (int i = 0; i < ndev; ++i) {
        total_det += slot[i].ndet;
        const uint64_t keep = std::min(slot[i].ndet, cap);
        if (det_out && keep) {
          const uint64_t room = cap > stored ? cap - stored : 0;
          const uint64_t take = std::min(keep, room);
          if (take) {
            cudaSetDevice(devices[i]);
            // each device sorts its own records; ranges ascend in device order,
            // so the concatenation is sorted by photon index
            const bool dev_sort = counts[i] <= (1ull << 32) && stride % 4 == 0 && keep < (1ull << 31);
            if (!dev_sort) host_sort = true;
            const void* src = dev_sort ? sort_records_device(slot[i].det.p, keep, stride, first[i], counts[i],
                                                             slot[i].rs, devices[i], slot[i].st)
                                       : slot[i].det.p;
            ck(cudaMemcpyAsync(static_cast<unsigned char*>(det_out) + stored * stride, src, take * stride,
                               cudaMemcpyDeviceToHost, slot[i].st),
               "download det");
            ck(cudaStreamSynchronize(slot[i].st), "download det");
            stored += take;
          }
        }
      }
      if (det_out && host_sort) sort_records(static_cast<unsigned char*>(det_out), stored, stride);
      if (det_count_out) *det_count_out = config->ndet > 0 ? total_det : 0;
      for (int i = 0; i < ndev; ++i)
        if (per_device_ms) per_device_ms[i] = slot[i].ms;
      if (reduce_ms) *reduce_ms = red_ms;
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

int vmc_partition(int strategy, uint64_t total, int ndev, const vmc_device_profile* devices, uint64_t* counts_out) {
  return guarded([&] {
    if (ndev < 1 || !devices) fail_validation("partition: no devices");
    std::vector<vmc::DeviceModel> dev(ndev);
    for (int i = 0; i < ndev; ++i) dev[i] = {devices[i].cores, devices[i].a, devices[i].t0};
    const std::vector<uint64_t> n = vmc::partition_photons(strategy, total, dev);
    std::copy(n.begin(), n.end(), counts_out);
  });
}

double vmc_model_makespan(int ndev, const uint64_t* counts, const vmc_device_profile* devices) {
  std::vector<vmc::DeviceModel> dev(ndev);
  for (int i = 0; i < ndev; ++i) dev[i] = {devices[i].cores, devices[i].a, devices[i].t0};
  return vmc::model_makespan(std::vector<uint64_t>(counts, counts + ndev), dev);
}

int vmc_plan_create(const vmc_scene* scene, const vmc_config* config, int device, vmc_plan** out) {
  return guarded([&] {
    if (!out) fail_validation("null plan output");
    std::unique_ptr<vmc_plan> P(new vmc_plan);
    plan_init(P.get(), scene, config, device);
    *out = P.release();
  });
}

int vmc_plan_destroy(vmc_plan* plan) {
  return guarded([&] {
    if (!plan) return;
    cudaSetDevice(plan->device);
    delete plan;
  });
}

uint64_t vmc_plan_cell_count(const vmc_plan* plan) { return plan ? plan->ncells : 0; }

int vmc_plan_run(vmc_plan* plan, uint64_t first_index, uint64_t count, int64_t* d_cells, int64_t* d_totals,
                 void* d_det, uint64_t* d_det_count, void* stream, uint32_t flags) {
  return guarded([&] {
    if (!plan) fail_validation("null plan");
    plan_enqueue(plan, first_index, count, d_cells, d_totals, d_det, d_det_count, static_cast<cudaStream_t>(stream),
                 flags, false, nullptr);
  });
}

int vmc_plan_trace(vmc_plan* plan, uint64_t first_index, uint64_t count, vmc_photon_trace* out) {
  return guarded([&] {
    if (!plan) fail_validation("null plan");
    ck(cudaSetDevice(plan->device), "cudaSetDevice");
    DevBuf cells, totals, det, detn, tr;
    cells.alloc(plan->ncells * sizeof(int64_t), plan->device);
    totals.alloc(4 * sizeof(int64_t), plan->device);
    const uint64_t cap = plan->cfg.ndet > 0 ? plan->cfg.det_capacity : 0;
    det.alloc(cap * plan->rec_stride, plan->device);
    detn.alloc(sizeof(uint64_t), plan->device);
    tr.alloc(count * sizeof(vmc_photon_trace), plan->device);
    plan_enqueue(plan, first_index, count, static_cast<int64_t*>(cells.p), static_cast<int64_t*>(totals.p), det.p,
                 static_cast<uint64_t*>(detn.p), nullptr, VMC_RUN_ZERO, true, static_cast<vmc_photon_trace*>(tr.p));
    ck(cudaDeviceSynchronize(), "trace run");
    if (count) ck(cudaMemcpy(out, tr.p, count * sizeof(vmc_photon_trace), cudaMemcpyDeviceToHost), "download trace");
    check_launch_errors(plan);
  });
}

namespace {
// vmc_simulate_photon is a per-photon call (reference callers loop over it, e.g.
// acceptance.cpp's criterion 3: 1e6 calls), so its plan and buffers are kept
// per device and reused while the scene and the config stay the same (key: the
// label digest plus every other input byte); a call is then one launch, one
// sync and four small copies instead of a plan build, allocations and frees.
struct SimContext {
  std::mutex mu;
  uint64_t key = 0;
  std::unique_ptr<vmc_plan> P;
  DevBuf cells, totals, det, detn, tr, lc, lw, ln;
};

SimContext& sim_context(int device) {
  static SimContext* ctx = new SimContext[64];  // never destroyed: no cudaFree after CUDA teardown
  if (device < 0 || device >= 64) fail_validation("device index out of range");
  return ctx[device];
}

uint64_t sim_key(const vmc_scene* s, const vmc_config* c, uint64_t labels) {
  std::vector<unsigned char> b;
  auto put = [&](const void* p, size_t n) {
    const auto* q = static_cast<const unsigned char*>(p);
    b.insert(b.end(), q, q + n);
  };
  put(&labels, sizeof labels);
  const int32_t dims[4] = {s->nx, s->ny, s->nz, s->nmedia};
  put(dims, sizeof dims);
  put(&s->voxel_mm, sizeof s->voxel_mm);
  put(s->media, sizeof(double) * 4 * static_cast<size_t>(std::max(0, s->nmedia)));
  put(s->src_pos, sizeof s->src_pos);
  put(s->src_dir, sizeof s->src_dir);
  put(&s->isotropic, sizeof s->isotropic);
  vmc_config cc = *c;
  cc.det = nullptr;
  put(&cc, sizeof cc);
  if (c->ndet > 0 && c->det) put(c->det, sizeof(double) * 4 * static_cast<size_t>(c->ndet));
  return vmc_fnv1a64(b.data(), b.size());
}
}  // namespace

int vmc_simulate_photon(const vmc_scene* scene, const vmc_config* config, uint64_t photon_index, int device,
                        uint64_t max_deposits, int64_t* cells_out, double* dw_out, uint64_t* n_deposits,
                        double* disp_out) {
  return guarded([&] {
    if (max_deposits && (!cells_out || !dw_out)) fail_validation("simulate_photon: null deposit buffers");
    LabelInfo li;
    validate(scene, config, &li);
    vmc_config c = *config;
    c.precision = VMC_PRECISION_FP64;  // the reference's arithmetic (FP64 flight kernel)
    c.ngates = 1;
    SimContext& X = sim_context(device);
    std::lock_guard<std::mutex> lock(X.mu);
    const uint64_t key = sim_key(scene, &c, li.digest);
    if (!X.P || X.key != key) {
      X.P.reset();
      auto P = std::make_unique<vmc_plan>();
      plan_init(P.get(), scene, &c, device);
      X.cells.ensure(P->ncells * sizeof(int64_t), device);
      X.totals.ensure(4 * sizeof(int64_t), device);
      X.det.ensure(std::max<uint64_t>(1, c.ndet > 0 ? c.det_capacity : 0) * P->rec_stride, device);
      X.detn.ensure(sizeof(uint64_t), device);
      X.tr.ensure(sizeof(vmc_photon_trace), device);
      X.ln.ensure(sizeof(unsigned long long), device);
      X.P = std::move(P);
      X.key = key;
    }
    vmc_plan* P = X.P.get();
    ck(cudaSetDevice(device), "cudaSetDevice");
    X.lc.ensure(std::max<uint64_t>(1, max_deposits) * sizeof(long long), device);
    X.lw.ensure(std::max<uint64_t>(1, max_deposits) * sizeof(double), device);
    ck(cudaMemsetAsync(X.ln.p, 0, sizeof(unsigned long long), nullptr), "zero log");
    DepLog log{static_cast<long long*>(X.lc.p), static_cast<double*>(X.lw.p),
               static_cast<unsigned long long*>(X.ln.p), max_deposits};
    plan_enqueue(P, photon_index, 1, static_cast<int64_t*>(X.cells.p), static_cast<int64_t*>(X.totals.p), X.det.p,
                 static_cast<uint64_t*>(X.detn.p), nullptr, VMC_RUN_ZERO, true,
                 static_cast<vmc_photon_trace*>(X.tr.p), &log);
    vmc_photon_trace t;
    unsigned long long n = 0;
    ck(cudaMemcpy(&t, X.tr.p, sizeof t, cudaMemcpyDeviceToHost), "download trace");
    ck(cudaMemcpy(&n, X.ln.p, sizeof n, cudaMemcpyDeviceToHost), "download log count");
    check_launch_errors(P);
    const uint64_t keep = std::min<uint64_t>(n, max_deposits);
    if (keep) {
      ck(cudaMemcpy(cells_out, X.lc.p, keep * sizeof(long long), cudaMemcpyDeviceToHost), "download log");
      ck(cudaMemcpy(dw_out, X.lw.p, keep * sizeof(double), cudaMemcpyDeviceToHost), "download log");
    }
    if (n_deposits) *n_deposits = n;
    if (disp_out) {
      disp_out[0] = t.deposited;
      disp_out[1] = t.escaped;
      disp_out[2] = t.killed;
      disp_out[3] = t.truncated;
    }
  });
}

int vmc_plan_normalize(vmc_plan* plan, const int64_t* d_cells, uint64_t photon_count, float* d_out, int sum_gates,
                       int normalized, void* stream) {
  return guarded([&] {
    if (!plan || !d_cells || !d_out) fail_validation("normalize: null argument");
    if (photon_count < 1) fail_validation("normalize: photon_count must be >= 1");
    ck(cudaSetDevice(plan->device), "cudaSetDevice");
    const long long nvox = static_cast<long long>(plan->nx) * plan->ny * plan->nz;
    const double q = vmc_quantum_for(plan->cfg.photon_count);
    // den per label in FluenceMap::normalize's order: (mua * v_voxel) * N,
    // v_voxel = h * h * h (fluence.cpp:66,73-74)
    const double v = plan->voxel_mm * plan->voxel_mm * plan->voxel_mm;
    if (plan->den_n != photon_count) {
      std::vector<double> mua(static_cast<size_t>(plan->nmedia)), den(mua.size());
      ck(cudaMemcpy(mua.data(), plan->mua.p, mua.size() * sizeof(double), cudaMemcpyDeviceToHost), "mua");
      for (size_t m = 0; m < mua.size(); ++m)
        den[m] = mua[m] > 0.0 ? mua[m] * v * static_cast<double>(photon_count) : 0.0;
      plan->den.ensure(den.size() * sizeof(double), plan->device);
      ck(cudaMemcpy(plan->den.p, den.data(), den.size() * sizeof(double), cudaMemcpyHostToDevice), "den");
      plan->den_n = photon_count;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, plan->device);
    const long long work = (nvox & 1) ? nvox : nvox / 2;  // voxel pairs when nvox is even
    const int grid = static_cast<int>(std::min<long long>((work + 255) / 256, static_cast<long long>(sms) * 16));
    k_normalize<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const long long*>(d_cells), static_cast<const uint8_t*>(plan->labels.p),
        static_cast<const double*>(plan->den.p), nvox, plan->cfg.ngates, sum_gates, normalized, q, d_out);
    ck(cudaGetLastError(), "launch normalize");
  });
}

uint64_t vmc_fnv1a64(const void* data, size_t bytes) {
  const unsigned char* b = static_cast<const unsigned char*>(data);
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < bytes; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

int vmc_plan_sort_records(vmc_plan* plan, const void* d_recs, uint64_t n, uint64_t first_index, uint64_t count,
                          void* d_out, void* stream) {
  return guarded([&] {
    if (!plan) fail_validation("null plan");
    if (n && (!d_recs || !d_out)) fail_validation("sort_records: null buffer");
    if (d_recs == d_out && n > 1) fail_validation("sort_records: output must not alias the input");
    if (count > (1ull << 32) || plan->rec_stride % 4 != 0 || n >= (1ull << 31))
      fail_validation("sort_records: range wider than 2^32 photons or more than 2^31 records");
    ck(cudaSetDevice(plan->device), "cudaSetDevice");
    sort_records_device(d_recs, n, plan->rec_stride, first_index, count, plan->rs, plan->device,
                        static_cast<cudaStream_t>(stream), d_out);
  });
}

const char* vmc_plan_kernel_name(const vmc_plan* plan) { return plan ? plan->kern_name.c_str() : ""; }

int vmc_plan_launches_per_run(const vmc_plan* plan, uint32_t flags) {
  (void)flags;
  return plan ? 1 + (plan->scratch ? 1 : 0) : 0;  // transport (+ replica fold)
}

}  // extern "C"
