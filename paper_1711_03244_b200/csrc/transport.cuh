// transport.cuh — K1, the persistent photon-transport kernel (sm_100a).
//
// One CUDA thread = one photon stream at a time. Persistent CTAs (grid = SMs x
// resident CTAs); when a lane's photon terminates, the warp claims the next
// global photon indices with ONE atomicAdd on a device counter and relaunches
// in place (the GPU form of GroupCounter::claim + the run_group worker loop,
// proj/core/include/voxmc/scheduler.hpp:64-86, proj/core/src/scheduler.cpp:286-305).
//
// The walk restates run_photon (proj/core/src/transport.cpp:310-358) with
// advance (:161-225), boundary_distance (:49-73), hg_scatter (:120-147),
// handle_interface (:227-298) and roulette (:300-306), consuming the RNG in
// exactly the reference's order, so photon k draws the
// same u64 stream as the reference photon k.
//
// Two arithmetic instantiations:
//   float  — the product path. Deposits are coalesced per (voxel, gate) run:
//            the run's absorbed weight is w_run_start - w (exact by Sterbenz
//            for the usual case), quantized once, and added with one integer
//            atomic. Per-photon dispositions are kept in the same fixed-point
//            quanta, so the energy identity closes in integers.
//   double — parity mode: per-step llround deposits and double dispositions,
//            operation-for-operation the reference (compiled with --fmad=false
//            so it matches the reference built without FMA contraction up to
//            libm-vs-CUDA log/exp rounding).
//
// Fluence cells are int64 fixed point in the reference quantum
// (proj/core/src/fluence.cpp:11-14); the device adds them with
// red.global.add.u64 (the map is L2-resident for the cube60 phantoms).
//
// Warp scheduling (see the loop below): scatters are deferred and run as a
// warp phase once enough lanes wait, with one azimuth rejection try per phase;
// dead lanes are refilled in groups. Photons are independent, so scheduling
// never changes a photon's arithmetic or its RNG draw order.
#pragma once

#include <cstdint>
#include <type_traits>

#include "../../include/vmc.h"
#include "rng.cuh"

namespace vmc {

constexpr int kBlock = 256;  // threads per CTA of K1
#ifndef VMC_AZ_UNROLL
#define VMC_AZ_UNROLL 2  // azimuth rejection tries per scatter phase (unrolled; 2 measured best)
#endif
constexpr int kMaxDet = 16;
constexpr int kMaxDetMedia = 8;
constexpr double kLightMmPerNs = 299.792458;  // types.hpp:16

// K1f deposit paths (flight.cuh, flight_body's kDep) and the hot-box edge
constexpr int kDepDirect = 0, kDepWarp = 1, kDepHotBox = 2;
constexpr int kHotBoxN = 16;
constexpr int kHotBoxBytes = kHotBoxN * kHotBoxN * kHotBoxN * 8;

// K1f per-warp seed stash: 32 x {u64 a, u64 b}, 32 first free paths (Real), header
__host__ __device__ constexpr int flight_stash_bytes(unsigned long real_bytes) {
  return static_cast<int>(32 * 16 + 32 * real_bytes + 16);
}

// Per-label optical data, staged in shared memory at CTA start.
template <typename Real>
struct alignas(16) Medium {
  Real mua, mus, inv_mus, ns_per_mm;  // ns_per_mm = n / c
  Real mm_per_ns, n, g, hg_a;         // hg_a = (1+g^2)/(2g)
  Real hg_b, hg_c, hg_d, hg_e;        // hg_b = 1/(2g), hg_c = 1-g^2, hg_d = 1-g, hg_e = 2g
  int nclass;                          // media with equal (double) n share a class
  int iso;                             // |g| < 1e-6
  Real ka;                             // -mua * log2(e): K1f's exp2-form absorb
};

struct KernelArgs {
  const uint8_t* labels;
  int nx, ny, nz, pad0;
  long long nxy, nvox;
  double h;
  int nmedia, iso_source;
  const void* media;  // Medium<Real>[nmedia]
  double src_pos[3];
  double dir0[3];      // normalized pencil direction
  double pos0[3];      // nudged pencil launch point
  int v0[3];           // pencil launch voxel
  int lab0;
  uint64_t seed, first, count;
  unsigned long long* claim;  // photon-claim counter (zeroed before launch)
  double tmax, rthr, inv_rmult;
  int rmult, reflect;
  int ngates, pad1;
  double inv_gate_w;
  double qscale;  // 1 / quantum
  long long* cells;
  long long* totals;  // [4] deposited, escaped, killed, truncated quanta
  // float copies of the hot constants (no FP64 conversion inside the loop)
  float hf, tmaxf, rthrf, rmultf, inv_rmultf, inv_gate_wf, qscalef, pad4;
  // detectors
  int ndet, nppath, rec_stride, pad3;
  // warp scheduling: scatter phase when >= scatter_pct % of live lanes wait;
  // refill when >= refill_min lanes are empty
  int scatter_pct, refill_min;
  double det[kMaxDet][4];
  unsigned char* det_out;
  unsigned long long* det_count;
  unsigned long long det_cap;
  vmc_photon_trace* trace;
  // trace launches only (vmc_simulate_photon): per-step deposit log
  // {cell, dw} in walk order, like simulate_photon_trace's deposit list
  long long* dep_cells;
  double* dep_w;
  unsigned long long* dep_n;
  unsigned long long dep_cap;
  int* error_flag;  // set to 1 when a launch point falls outside the grid
  // single-label volumes (kUni): the one interior medium, read straight from
  // the parameter bank (constant operands, no shared-memory address math)
  Medium<float> uni_f;
  Medium<double> uni_d;
  // K1f (flight.cuh): the event-phase trigger (percent of live lanes that
  // must have finished their flight before the warp runs the event phase)
  int pad11;
  float gate_wf;  // K1f: gate width tmax / ngates (FP32)
  int event_pct;
  int pad14;
  // fluence-map replicas: CTA b deposits into cells + (b & rep_mask) * rep_stride
  // (the host folds the replicas into the caller's map after the launch)
  long long rep_stride;
  int rep_mask;
  int walk_keep;  // K1f: a full warp walks while more than (32 * (100 - event_pct)) / 100 lanes walk
  int pad10, pad7;
  float detf[kMaxDet][4];  // K1f: detector disks as {x, y, z, r^2} in FP32
  int hb0[3];              // K1f hot-box deposits: box origin voxel (16^3 box around the source)
  int chain_min;  // K1f scatter chain: >= chain_min lanes ending their new flight in-voxel (0 = off)
  float dir0f[3], pos0f[3];  // K1f FP32: the pencil launch state, converted once on the host
};


// ---------------------------------------------------------------------------
// small helpers

template <typename Real>
struct RealTraits;
template <>
struct RealTraits<float> {
  static __device__ __forceinline__ float inf() { return __int_as_float(0x7f800000); }
  // MUFU.RCP (<= 1 ulp): the cached inverse direction only feeds the DDA
  // plane distances, where one ulp is far below the voxel-landing tolerance.
  static __device__ __forceinline__ float rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
  }
  static __device__ __forceinline__ float sqrt_(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
  }
  static __device__ __forceinline__ float rsqrt(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
  }
  // natural log via MUFU.LG2 (argument is a normal float here)
  static __device__ __forceinline__ float ln(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r * 0.69314718055994531f;
  }
  // exp(-x), x >= 0, via MUFU.EX2
  static __device__ __forceinline__ float exp_neg(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x * -1.4426950408889634f));
    return r;
  }
};
template <>
struct RealTraits<double> {
  static __device__ __forceinline__ double inf() { return __longlong_as_double(0x7ff0000000000000ll); }
  static __device__ __forceinline__ double rcp(double x) { return 1.0 / x; }
  static __device__ __forceinline__ double sqrt_(double x) { return sqrt(x); }
  static __device__ __forceinline__ double rsqrt(double x) { return 1.0 / sqrt(x); }
  static __device__ __forceinline__ double ln(double x) { return log(x); }
  static __device__ __forceinline__ double exp_neg(double x) { return exp(-x); }
};

// Dynamic shared memory of K1, referenced through the symbol (not a generic
// pointer) so every access compiles to LDS with a constant window base.
extern __shared__ __align__(16) unsigned char vmc_smem[];

// kUni: every voxel carries the same label (homogeneous phantoms such as the
// cube60 benchmarks): an interior neighbour is then always the same medium,
// so the neighbour-label load and refractive-class compare are skipped.
// Results are identical to the general path.
template <typename Real, bool kGates, bool kDet, bool kTrace, bool kUni = false>
__device__ __forceinline__ void transport_body(const KernelArgs& A) {
  unsigned char* smem = vmc_smem;
  using Tr = RealTraits<Real>;
  constexpr bool kF32 = std::is_same<Real, float>::value;
  using Rng = Xs128p<kTrace>;
  // optical data of the photon's current medium
  auto medium = [&](int l) -> const Medium<Real>& {
    if constexpr (kUni) {
      if constexpr (kF32) {
        return A.uni_f;
      } else {
        return A.uni_d;
      }
    } else {
      return reinterpret_cast<const Medium<Real>*>(smem)[l];
    }
  };

  // ---- shared memory: media table ---------------------------------------
  Medium<Real>* sm_media = reinterpret_cast<Medium<Real>*>(smem);
  {
    const Medium<Real>* gm = static_cast<const Medium<Real>*>(A.media);
    const int nwords = static_cast<int>(sizeof(Medium<Real>) / 4) * A.nmedia;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x)
      reinterpret_cast<int*>(sm_media)[i] = reinterpret_cast<const int*>(gm)[i];
  }
  __syncthreads();

  const int nx = A.nx, ny = A.ny, nz = A.nz;
  const int nxy32 = static_cast<int>(A.nxy);
  const Real h = kF32 ? Real(A.hf) : Real(A.h);
  const Real tmax = kF32 ? Real(A.tmaxf) : Real(A.tmax);
  const Real rthr = kF32 ? Real(A.rthrf) : Real(A.rthr);
  const Real rmult = kF32 ? Real(A.rmultf) : Real(A.rmult);
  const Real inv_rmult = kF32 ? Real(A.inv_rmultf) : Real(A.inv_rmult);
  const Real inv_gate_w = kF32 ? Real(A.inv_gate_wf) : Real(A.inv_gate_w);
  const float qscale_f = A.qscalef;
  const int lane = threadIdx.x & 31;
  const unsigned lanemask_lt = (1u << lane) - 1u;

  // per-thread fixed-point disposition totals
  long long acc_dep = 0, acc_esc = 0, acc_kill = 0, acc_trunc = 0;

  // photon state
  // 0 = ready to step, 1 = at a scattering point (scatter deferred to a scatter
  // phase), 2 = no photon (lane waits for a refill), 3 = scatter in progress,
  // waiting for another azimuth rejection-sampling try (ct/st kept in sct/sst)
  int phase = 2;
  Real sct = 0, sst = 0;
  bool exhausted = false;  // warp-uniform: counter ran past `count`
  uint64_t idx = 0;
  Rng rng;
  rng.a = rng.b = 0;
  Real px = 0, py = 0, pz = 0, dx = 0, dy = 0, dz = 0, ix = 0, iy = 0, iz = 0;
  Real w = 0, t = 0, rs = 0;
  int vx = 0, vy = 0, vz = 0, lab = 0;
  int cell = 0;  // x + nx*(y + ny*z); volumes are < 2^31 voxels (validated)
  int gate = 0;
  Real run_w0 = 0;          // float path: weight at the start of the current run
  double pd_dep = 0, pd_esc = 0, pd_kill = 0, pd_trunc = 0;  // per-photon (double path / trace)
  uint32_t steps = 0, nscat = 0;
  bool detected = false;
  // detector mode: path length in the current medium accumulates in `seg` and
  // is flushed into this thread's per-label slots in shared memory
  // (pp_sm[m * kBlock + tid], bank-conflict free) only when the label changes
  // or the photon exits, so a step costs one add
  Real seg = 0;
  Real* pp_sm = reinterpret_cast<Real*>(smem + ((sizeof(Medium<Real>) * A.nmedia + 15) & ~static_cast<size_t>(15))) +
                threadIdx.x;
  auto flush_seg = [&]() {
    if constexpr (kDet) {
      if (lab >= 1) pp_sm[(lab - 1) * kBlock] += seg;
      seg = 0;
    }
  };

  // one fixed-point add per deposit run (red.global.add.u64; the map is L2-resident)
  unsigned long long* const cbase =
      reinterpret_cast<unsigned long long*>(A.cells) + (blockIdx.x & A.rep_mask) * A.rep_stride;
  auto deposit = [&](int c, int gt, long long q) {
    if (q != 0) atomicAdd(cbase + (static_cast<long long>(c) + A.nvox * gt), static_cast<unsigned long long>(q));
  };
  auto quant = [&](Real x) -> long long {
    if constexpr (kF32) {
      return __float2ll_rn(x * qscale_f);
    } else {
      return llround(x * A.qscale);
    }
  };
  auto gate_of = [&](Real tt) -> int {
    if constexpr (kGates) {
      int g = static_cast<int>(tt * inv_gate_w);  // tt >= 0: truncation == floor
      return g < A.ngates - 1 ? g : A.ngates - 1;
    } else {
      return 0;
    }
  };
  auto set_dir = [&](Real ax_, Real ay_, Real az_) {  // transport.cpp:77-81
    dx = ax_;
    dy = ay_;
    dz = az_;
    ix = ax_ != Real(0) ? Tr::rcp(ax_) : Tr::inf();
    iy = ay_ != Real(0) ? Tr::rcp(ay_) : Tr::inf();
    iz = az_ != Real(0) ? Tr::rcp(az_) : Tr::inf();
  };
  auto scat_len = [&]() -> Real {  // transport.cpp:14-17
    const Real u = rng.template unit<Real>();
    if constexpr (kF32) {
      // u == 0 (p = 2^-24) stands for the reference's [0, 2^-24) cell: use 2^-25.
      return -Tr::ln(u > 0.0f ? u : 0x1p-25f);  // MUFU.LG2: abs. error ~1e-7
    } else {
      return -log(u > 0.0 ? u : 4.9406564584124654e-324);
    }
  };
  auto finish = [&](int kind) {  // 0 escaped 1 killed 2 truncated
    if constexpr (kTrace) {
      vmc_photon_trace tr;
      tr.draws = rng.draws;
      tr.steps = steps;
      tr.scatters = nscat;
      tr.flags = (kind == 0 ? 1u : (kind == 1 ? 2u : 4u)) | (detected ? 8u : 0u);
      detected = false;
      tr.deposited = pd_dep;
      tr.escaped = pd_esc;
      tr.killed = pd_kill;
      tr.truncated = pd_trunc;
      A.trace[idx - A.first] = tr;
    }
    if constexpr (!kF32) {
      acc_dep += llround(pd_dep * A.qscale);
      acc_esc += llround(pd_esc * A.qscale);
      acc_kill += llround(pd_kill * A.qscale);
      acc_trunc += llround(pd_trunc * A.qscale);
    }
    phase = 2;
  };

  // one advance() step (transport.cpp:161-225) and the face / interface /
  // exit handling that follows it in run_photon (transport.cpp:322-357)
  auto step = [&]() {
    // ---- one advance() step, transport.cpp:161-225 ----
    const Medium<Real>& M = medium(lab);
    if constexpr (kTrace) ++steps;
    // boundary_distance, transport.cpp:49-73
    Real tb0, tb1, tb2;
    {
      const Real plx = static_cast<Real>(vx + (dx > Real(0) ? 1 : 0)) * h;
      const Real ply = static_cast<Real>(vy + (dy > Real(0) ? 1 : 0)) * h;
      const Real plz = static_cast<Real>(vz + (dz > Real(0) ? 1 : 0)) * h;
      const Real t0_ = (plx - px) * ix, t1_ = (ply - py) * iy, t2_ = (plz - pz) * iz;
      tb0 = dx != Real(0) ? (t0_ > Real(0) ? t0_ : Real(0)) : Tr::inf();
      tb1 = dy != Real(0) ? (t1_ > Real(0) ? t1_ : Real(0)) : Tr::inf();
      tb2 = dz != Real(0) ? (t2_ > Real(0) ? t2_ : Real(0)) : Tr::inf();
    }
    // select-style argmin (ties -> lower axis), carrying the crossed axis'
    // direction component, voxel coordinate, extent and cell stride along
    int axis = 0;
    Real d_b = tb0, dax = dx;
    int vax = vx, nax = nx, stride = 1;
    if (tb1 < d_b) {
      d_b = tb1;
      axis = 1;
      dax = dy;
      vax = vy;
      nax = ny;
      stride = nx;
    }
    if (tb2 < d_b) {
      d_b = tb2;
      axis = 2;
      dax = dz;
      vax = vz;
      nax = nz;
      stride = nxy32;
    }
    // neighbour across the nearest face; its label load is issued here so the
    // L1/L2 latency overlaps the rest of the step (used only if the step crosses)
    const int stp = dax > Real(0) ? 1 : -1;
    const int nvax = vax + stp;
    const int ncell = stp > 0 ? cell + stride : cell - stride;
    const bool exterior = static_cast<unsigned>(nvax) >= static_cast<unsigned>(nax);
    const int nlab_pf = kUni ? lab : static_cast<int>(__ldg(A.labels + (exterior ? cell : ncell)));
    Real d_s;
    if constexpr (kF32) {
      d_s = M.mus > 0.0f ? rs * M.inv_mus : Tr::inf();  // rs may be 0 after a clamp
    } else {
      d_s = M.mus > 0.0 ? rs / M.mus : Tr::inf();
    }
    const Real ns = M.ns_per_mm;
    const Real remaining = tmax - t;
    Real d = d_b < d_s ? d_b : d_s;  // std::min(d_boundary, d_scatter)
    const bool horizon = d * ns >= remaining;
    if (horizon) {
      if constexpr (kF32) {
        d = fmaxf(0.0f, remaining * M.mm_per_ns);
      } else {
        d = fmax(0.0, remaining / ns);
      }
    }
    // Beer-Lambert, exp_neg transport.cpp:22-27
    Real w1;
    {
      const Real x = M.mua * d;
      Real e;
      const Real taylor = Real(1) - x * (Real(1) - x * (Real(0.5) - x * (Real(1.0 / 6.0) - x * Real(1.0 / 24.0))));
      if constexpr (kF32) {
        e = x < 0.01f ? taylor : Tr::exp_neg(x);  // branch-free select
      } else {
        e = x < 0.01 ? taylor : exp(-x);
      }
      w1 = w * e;
    }
    const Real t_start = t;
    if constexpr (!kF32) {
      // per-step deposit into the pre-step voxel (transport.cpp:323-327)
      const Real dw = w - w1;
      if (dw != 0.0) {
        deposit(cell, gate_of(t_start), llround(dw * A.qscale));
        pd_dep += dw;
      }
    } else if constexpr (kTrace) {
      pd_dep += static_cast<double>(w - w1);
    }
    w = w1;
    t += d * ns;
    if constexpr (kDet) seg += d;

    if (horizon) {  // StepKind::Terminated
      t = tmax;
      if constexpr (kF32) {
        const long long q = quant(run_w0 - w);
        deposit(cell, gate, q);
        acc_dep += q;
        acc_trunc += quant(w);
      }
      pd_trunc += w;
      finish(2);
      return;
    }

    if (d_s <= d_b) {  // StepKind::Scattered: move to the scattering point
      px += dx * d;
      py += dy * d;
      pz += dz * d;
      if constexpr (kGates && kF32) {
        const int ng = gate_of(t);
        if (ng != gate) {
          const long long q = quant(run_w0 - w);
          deposit(cell, gate, q);
          acc_dep += q;
          run_w0 = w;
          gate = ng;
        }
      }
      phase = 1;  // hg_scatter + new length + roulette run in a scatter phase
      return;
    }

    // ---- land exactly on the face (transport.cpp:197-211) ----
    if constexpr (kF32) {
      rs = fmaxf(0.0f, rs - d * M.mus);
    } else {
      rs = fmax(0.0, rs - d * M.mus);
    }
    {
      // land exactly on the crossed plane; the other two coordinates advance
      const Real plane = static_cast<Real>(vax + (stp > 0 ? 1 : 0)) * h;
      px = axis == 0 ? plane : px + dx * d;
      py = axis == 1 ? plane : py + dy * d;
      pz = axis == 2 ? plane : pz + dz * d;
    }
    const int nlab = exterior ? 0 : nlab_pf;
    const int c1 = M.nclass, c2 = (kUni && !exterior) ? c1 : sm_media[nlab].nclass;
    bool move = false, exited = false;
    if (!exterior && c1 == c2) {
      move = true;  // same refractive index: inline update (transport.cpp:218-223)
    } else if (exterior && !A.reflect) {
      exited = true;  // TerminateAtBoundary (transport.cpp:234-237)
    } else if (c1 == c2) {
      exited = exterior;  // identity interface, n1 == n2 (transport.cpp:242-252)
      move = !exterior;
    } else {
      // Fresnel / TIR, handle_interface transport.cpp:254-297
      const Real n1 = M.n, n2 = sm_media[nlab].n;
      const Real ci = dax < Real(0) ? -dax : dax;
      Real si2 = Real(1) - ci * ci;
      si2 = si2 > Real(0) ? si2 : Real(0);
      const Real eta = n1 / n2;
      const Real st2 = eta * eta * si2;
      if (st2 > Real(1)) {  // total internal reflection: deterministic flip
        set_dir(axis == 0 ? -dx : dx, axis == 1 ? -dy : dy, axis == 2 ? -dz : dz);
      } else {
        Real cost;
        if constexpr (kF32) {
          cost = sqrtf(1.0f - st2);
        } else {
          cost = sqrt(1.0 - st2);
        }
        const Real rsp = (n1 * ci - n2 * cost) / (n1 * ci + n2 * cost);
        const Real rpp = (n1 * cost - n2 * ci) / (n1 * cost + n2 * ci);
        const Real R = Real(0.5) * (rsp * rsp + rpp * rpp);
        if (rng.template unit<Real>() < R) {
          set_dir(axis == 0 ? -dx : dx, axis == 1 ? -dy : dy, axis == 2 ? -dz : dz);
        } else {
          Real qx = axis == 0 ? (dax > Real(0) ? cost : -cost) : dx * eta;
          Real qy = axis == 1 ? (dax > Real(0) ? cost : -cost) : dy * eta;
          Real qz = axis == 2 ? (dax > Real(0) ? cost : -cost) : dz * eta;
          Real k;
          if constexpr (kF32) {
            k = Tr::rsqrt(qx * qx + qy * qy + qz * qz);
          } else {
            k = 1.0 / sqrt(qx * qx + qy * qy + qz * qz);
          }
          set_dir(qx * k, qy * k, qz * k);
          exited = exterior;
          move = !exterior;
        }
      }
    }

    if (exited) {  // ExitedDomain: escaped += w (transport.cpp:348-350)
      if constexpr (kF32) {
        const long long q = quant(run_w0 - w);
        deposit(cell, gate, q);
        acc_dep += q;
        acc_esc += quant(w);
      }
      pd_esc += w;
      if constexpr (kDet) {
        flush_seg();
        int hit = -1;
        for (int k = 0; k < A.ndet; ++k) {
          const double ex = static_cast<double>(px) - A.det[k][0];
          const double ey = static_cast<double>(py) - A.det[k][1];
          const double ez = static_cast<double>(pz) - A.det[k][2];
          if (ex * ex + ey * ey + ez * ez <= A.det[k][3] * A.det[k][3]) {
            hit = k;
            break;
          }
        }
        const unsigned am = __activemask();
        const unsigned hm = __ballot_sync(am, hit >= 0);
        if constexpr (kTrace) detected = hit >= 0;
        if (hm) {
          const int leader = __ffs(hm) - 1;
          unsigned long long base = 0;
          if (lane == leader) base = atomicAdd(A.det_count, static_cast<unsigned long long>(__popc(hm)));
          base = __shfl_sync(am, base, leader);
          if (hit >= 0) {
            const unsigned long long slot = base + __popc(hm & lanemask_lt);
            if (slot < A.det_cap) {
              unsigned char* rec = A.det_out + slot * static_cast<unsigned long long>(A.rec_stride);
              vmc_det_record_head hd;
              hd.photon_index = idx;
              hd.det_id = static_cast<uint32_t>(hit);
              hd.nscat = nscat;
              hd.w_exit = static_cast<float>(w);
              hd.t_exit_ns = static_cast<float>(t);
              *reinterpret_cast<vmc_det_record_head*>(rec) = hd;
              float* pp = reinterpret_cast<float*>(rec + sizeof(vmc_det_record_head));
              for (int m = 0; m < A.nppath; ++m) pp[m] = static_cast<float>(pp_sm[m * kBlock]);
            }
          }
        }
      }
      finish(0);
      return;
    }
    if (move) {
      if constexpr (kF32) {
        const int ng = gate_of(t);
        // a new voxel (or gate) closes the current deposit run
        const long long q = quant(run_w0 - w);
        deposit(cell, gate, q);
        acc_dep += q;
        run_w0 = w;
        gate = ng;
      }
      vx += axis == 0 ? stp : 0;
      vy += axis == 1 ? stp : 0;
      vz += axis == 2 ? stp : 0;
      cell = ncell;
      if constexpr (kDet) {
        if (nlab != lab) flush_seg();
      }
      lab = nlab;
    } else if constexpr (kGates && kF32) {
      const int ng = gate_of(t);
      if (ng != gate) {
        const long long q = quant(run_w0 - w);
        deposit(cell, gate, q);
        acc_dep += q;
        run_w0 = w;
        gate = ng;
      }
    }
  };

  // hg_scatter (transport.cpp:126-147) + new free path (:14-17) + roulette
  // (:300-306, called at :333-343) for a lane at a scattering point
  auto scatter = [&]() {
    const Medium<Real>& M = medium(lab);
    if (phase == 1) {  // first visit: Henyey-Greenstein cos(theta) (transport.cpp:120-124)
      if constexpr (kTrace || kDet) ++nscat;
      const Real xi = rng.template unit<Real>();
      Real ct;
      if (M.iso) {
        ct = Real(2) * xi - Real(1);
      } else if constexpr (kF32) {
        const float f = __fdividef(M.hg_c, M.hg_d + M.hg_e * xi);
        ct = fminf(1.0f, fmaxf(-1.0f, M.hg_a - f * f * M.hg_b));
      } else {
        const double g = M.g;
        const double tmp = (1.0 - g * g) / (1.0 - g + 2.0 * g * xi);
        ct = (1.0 + g * g - tmp * tmp) / (2.0 * g);
        ct = ct < -1.0 ? -1.0 : (ct > 1.0 ? 1.0 : ct);
      }
      sct = ct;
      if constexpr (kF32) {
        sst = Tr::sqrt_(fmaxf(0.0f, 1.0f - ct * ct));
      } else {
        sst = sqrt(fmax(0.0, 1.0 - ct * ct));
      }
    }
    // one try of the rejection azimuth (transport.cpp:32-44); a rejected lane
    // keeps cos/sin(theta) and retries in the next scatter phase, so the warp
    // never loops on its unluckiest lane
    Real ax_ = 0, ay_ = 0, r2 = 0;
    bool ok = false;
#pragma unroll
    for (int k = 0; k < VMC_AZ_UNROLL; ++k) {
      if (k == 0 || !ok) {
        ax_ = Real(2) * rng.template unit<Real>() - Real(1);
        ay_ = Real(2) * rng.template unit<Real>() - Real(1);
        r2 = ax_ * ax_ + ay_ * ay_;
        ok = r2 > Real(1e-12) && r2 <= Real(1);
      }
    }
    if (!ok) {
      phase = 3;
      return;
    }
    phase = 0;
    const Real k = Tr::rsqrt(r2);
    const Real cp = ax_ * k, sp = ay_ * k;
    const Real ct = sct, st = sst;
    // rotate into the frame of the old direction (transport.cpp:133-141)
    Real ox, oy, oz;
    if ((dz < Real(0) ? -dz : dz) > Real(0.99999)) {
      ox = st * cp;
      oy = st * sp;
      oz = dz > Real(0) ? ct : -ct;
    } else if constexpr (kF32) {
      const float one_m = 1.0f - dz * dz;
      const float rden = Tr::rsqrt(one_m);
      const float sr = st * rden;
      ox = sr * (dx * dz * cp - dy * sp) + dx * ct;
      oy = sr * (dy * dz * cp + dx * sp) + dy * ct;
      oz = -st * cp * (one_m * rden) + dz * ct;
    } else {
      const double den = sqrt(1.0 - dz * dz);
      ox = st * (dx * dz * cp - dy * sp) / den + dx * ct;
      oy = st * (dy * dz * cp + dx * sp) / den + dy * ct;
      oz = -st * cp * den + dz * ct;
    }
    // renormalize (transport.cpp:142-145; 1e-6 in FP32, the reference's 1e-12 in FP64)
    const Real n2 = ox * ox + oy * oy + oz * oz;
    if ((n2 - Real(1) < Real(0) ? Real(1) - n2 : n2 - Real(1)) > (kF32 ? Real(1e-6) : Real(1e-12))) {
      const Real kk = Tr::rsqrt(n2);
      ox *= kk;
      oy *= kk;
      oz *= kk;
    }
    set_dir(ox, oy, oz);
    rs = scat_len();
    // roulette after a scatter only (transport.cpp:333-343, 300-306)
    if (w < rthr) {
      const Real before = w;
      const bool survive = rng.template unit<Real>() < inv_rmult;
      if constexpr (kF32) {
        const long long q = quant(run_w0 - w);  // close the deposit run
        deposit(cell, gate, q);
        acc_dep += q;
      }
      if (!survive) {
        if constexpr (kF32) acc_kill += quant(before);
        pd_kill += before;
        finish(1);
        return;
      }
      w *= rmult;
      if constexpr (kF32) {
        acc_kill += quant(before) - quant(w);
        run_w0 = w;
      }
      pd_kill += before - w;
    }
  };

  unsigned dead = 0xffffffffu;  // lanes without a photon (warp-uniform view)
  for (;;) {
    // Warp-level phase scheduler. Photons are independent, so the order in
    // which a warp interleaves their events never changes any photon's
    // arithmetic or RNG sequence; it only decides which lanes run together:
    //   step phase     every lane whose photon is ready to advance
    //   scatter phase  lanes at a scattering point (phase 1) or waiting for an
    //                  azimuth retry (phase 3); run once they are >= scatter_pct %
    //                  of the live lanes, one rejection-sampling try per phase
    //   refill         dead lanes (phase 2) relaunch in groups of refill_min
    if (!exhausted && dead && (__popc(dead) >= A.refill_min || dead == 0xffffffffu)) {
      const unsigned need = dead;
      {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(A.claim, static_cast<unsigned long long>(__popc(need)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base + __popc(need) >= A.count) exhausted = true;
        if (phase == 2) {
          const unsigned long long my = base + __popc(need & lanemask_lt);
          if (my < A.count) {
            // ---- launch, transport.cpp:83-106 ----
            idx = A.first + my;
            rng.seed(A.seed, idx);
            Real ux, uy, uz;
            if (A.iso_source) {
              const Real ct = Real(2) * rng.template unit<Real>() - Real(1);
              const Real u2 = rng.template unit<Real>();
              Real st, cphi, sphi;
              if constexpr (kF32) {
                st = sqrtf(fmaxf(0.0f, 1.0f - ct * ct));
                sincospif(2.0f * u2, &sphi, &cphi);
              } else {
                st = sqrt(fmax(0.0, 1.0 - ct * ct));
                const double phi = 2.0 * 3.14159265358979323846 * u2;
                sincos(phi, &sphi, &cphi);
              }
              ux = st * cphi;
              uy = st * sphi;
              uz = ct;
              // nudge + voxel_of in double (the 1e-6 mm nudge is below FP32 ulp)
              const double qx = A.src_pos[0] + static_cast<double>(ux) * 1e-6;
              const double qy = A.src_pos[1] + static_cast<double>(uy) * 1e-6;
              const double qz = A.src_pos[2] + static_cast<double>(uz) * 1e-6;
              vx = static_cast<int>(floor(qx / A.h));
              vy = static_cast<int>(floor(qy / A.h));
              vz = static_cast<int>(floor(qz / A.h));
              px = static_cast<Real>(qx);
              py = static_cast<Real>(qy);
              pz = static_cast<Real>(qz);
              if (vx < 0 || vy < 0 || vz < 0 || vx >= nx || vy >= ny || vz >= nz) {
                atomicExch(A.error_flag, 1);
                vx = vy = vz = 0;
                ux = uy = 0;
                uz = 1;
              }
              lab = __ldg(A.labels + (vx + nx * (vy + static_cast<long long>(ny) * vz)));
            } else {
              ux = static_cast<Real>(A.dir0[0]);
              uy = static_cast<Real>(A.dir0[1]);
              uz = static_cast<Real>(A.dir0[2]);
              px = static_cast<Real>(A.pos0[0]);
              py = static_cast<Real>(A.pos0[1]);
              pz = static_cast<Real>(A.pos0[2]);
              vx = A.v0[0];
              vy = A.v0[1];
              vz = A.v0[2];
              lab = A.lab0;
            }
            set_dir(ux, uy, uz);
            cell = vx + nx * (vy + ny * vz);
            w = Real(1);
            t = Real(0);
            rs = scat_len();
            gate = 0;
            run_w0 = Real(1);
            steps = nscat = 0;
            pd_dep = pd_esc = pd_kill = pd_trunc = 0;
            if constexpr (kDet) {
              seg = 0;
              for (int m = 0; m < A.nppath; ++m) pp_sm[m * kBlock] = Real(0);
            }
            phase = 0;
          }
        }
      }
      dead = __ballot_sync(0xffffffffu, phase == 2);
    }
    if (dead == 0xffffffffu) {
      if (exhausted) break;
      continue;
    }
    // ---- step phase: every lane holding a photon that is not at a scattering
    // point advances by one step (two steps per iteration measured slower)
    if (phase == 0) step();
    // ---- scatter phase: run the deferred scatters once at least half of the
    // lanes holding a photon are at a scattering point (or nobody can step) ----
    {
      const unsigned pend = __ballot_sync(0xffffffffu, (phase & 1) != 0);
      dead = __ballot_sync(0xffffffffu, phase == 2);
      const unsigned live = ~dead;
      if (pend != 0u && (pend == live || 100 * __popc(pend) >= A.scatter_pct * __popc(live))) {
        if (phase & 1) scatter();
        dead = __ballot_sync(0xffffffffu, phase == 2);  // roulette may have killed
      }
    }
  }

  // ---- epilogue: dispositions (warp reduce) -------------------------------
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc_dep += __shfl_xor_sync(0xffffffffu, acc_dep, o);
    acc_esc += __shfl_xor_sync(0xffffffffu, acc_esc, o);
    acc_kill += __shfl_xor_sync(0xffffffffu, acc_kill, o);
    acc_trunc += __shfl_xor_sync(0xffffffffu, acc_trunc, o);
  }
  if (lane == 0) {
    unsigned long long* tot = reinterpret_cast<unsigned long long*>(A.totals);
    if (acc_dep) atomicAdd(tot + 0, static_cast<unsigned long long>(acc_dep));
    if (acc_esc) atomicAdd(tot + 1, static_cast<unsigned long long>(acc_esc));
    if (acc_kill) atomicAdd(tot + 2, static_cast<unsigned long long>(acc_kill));
    if (acc_trunc) atomicAdd(tot + 3, static_cast<unsigned long long>(acc_trunc));
  }

}

}  // namespace vmc
