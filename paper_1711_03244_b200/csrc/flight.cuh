// flight.cuh — K1f, the FP32 photon-transport kernel organised by free flight (sm_100a).
//
// Same photons, same RNG draws in the same order, same discrete decisions as
// run_photon (proj/core/src/transport.cpp:310-358); what changes is how a warp
// spends its issue slots.
//
// The reference advances a photon one voxel face at a time: every advance()
// (transport.cpp:161-225) recomputes the three face distances
// (boundary_distance, :49-73), the scattering distance, the horizon test and a
// Beer-Lambert factor. Between two RNG-consuming events (scatter, Fresnel
// draw, roulette) nothing but the voxel index changes, so K1f splits the walk
// into
//
//   flight setup   once per free flight (after launch / scatter / interface):
//                  face distances tm and per-voxel increments td of an
//                  incremental DDA, the flight length
//                  L = min(remaining_scat / mus, horizon distance)
//                  (horizon iff d_scatter * n/c >= tmax - t, :169-175), the
//                  signed cell strides of the three axes;
//   walk step      per voxel face (the common, cheap event). A lane walks only
//                  while its next face s = min(tm) comes before L (checked at
//                  setup and after every face; scatter / horizon win ties,
//                  :175,191), so every lane in a walk step crosses: the
//                  segment's absorbed weight w (1 - exp(-mua ds)) closes the
//                  voxel's deposit run with one fixed-point red.add (deposit
//                  into the pre-step voxel, :323-327), the voxel index steps,
//                  the moved axis is tested against the exterior and
//                  (multi-label volumes) the neighbour label is read — a label
//                  change ends the flight at the face (interface, :214-223);
//   event phase    end of flight, scatter (hg_scatter + new free path +
//                  roulette, :126-147, :333-343), interface (handle_interface,
//                  :227-298), horizon, exit, refill, next flight's setup — run
//                  by the warp once >= event_pct % of its live lanes wait for one.
//
// A face costs ~40 SASS instructions instead of a full advance() step, and
// the expensive scatter/interface code runs on mostly full warps. Floating
// point differs from the step kernel only at the ulp level (face distances
// accumulated from the flight start instead of recomputed per face), which moves no
// discrete decision beyond the per-photon draw-count gates of the parity tests.
//
// Deposits go into one of KernelArgs::rep_mask + 1 replicas of the map (CTA
// index mod replicas): the voxels next to the source take every photon's
// first deposits, and spreading them over replicas keeps the same-address
// L2 red.add rate off the critical path. The host folds the replicas into the
// caller's map and books the deposited channel as the exact sum of the quanta
// it adds, so the kernel keeps no deposited accumulator.
//
// Voxel coordinates are kept as integers per axis; the linear cell index is
// two IMADs (FMA pipe) where a deposit or label read needs it.
#pragma once

#include <cstdio>

#include "transport.cuh"

namespace vmc {

#ifdef VMC_STATS
// debug build only (-DVMC_STATS): warp-scheduling counters, printed by the
// last CTA to finish
__device__ unsigned long long vmc_flight_stats[12];
__device__ unsigned int vmc_flight_done;
#endif

// kAbs: -1 = absorb() picks its series per launch (KernelArgs::absorb_mode);
// 0 / 1 = compiled for absorb_mode 0 (every mua * h * sqrt(3) < 0.012, the
// cube60 phantoms) / 1 (< 0.15, the head phantom), which drops the warp-uniform
// mode tests from every absorb()
template <bool kGates, bool kDet, bool kTrace, bool kUni, int kAbs = -1>
__device__ __forceinline__ void flight_body(const KernelArgs& A) {
  using Tr = RealTraits<float>;
  using Rng = Xs128p<kTrace>;
  constexpr int WALK = 0, SCAT = 1, DEAD = 2, RETRY = 3, FACE = 4, SETUP = 5, ENDF = 6;
  unsigned char* smem = vmc_smem;
  // Shared-memory layout at compile-time offsets (cheap to rematerialise):
  // per-thread disposition slots | per-warp seed stashes | per-thread path
  // lengths (detector kernels) | media table
  constexpr int kAccOff = 0;                                       // 3 x kBlock x int64
  constexpr int kStashOff = kAccOff + 3 * kBlock * 8;              // kBlock / 32 x (32 x 20 + 16) B
  constexpr int kPpOff = kStashOff + (kBlock / 32) * (32 * 20 + 16);
  constexpr int kMediaOff = kPpOff + (kDet ? kMaxDetMedia * kBlock * 4 : 0);
  static_assert(kStashOff % 16 == 0 && kPpOff % 16 == 0 && kMediaOff % 16 == 0, "smem alignment");

  // ---- shared memory: media table (exterior n is needed even when kUni) ----
  Medium<float>* sm_media = reinterpret_cast<Medium<float>*>(smem + kMediaOff);
  {
    const Medium<float>* gm = static_cast<const Medium<float>*>(A.media);
    const int nwords = static_cast<int>(sizeof(Medium<float>) / 4) * A.nmedia;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x)
      reinterpret_cast<int*>(sm_media)[i] = reinterpret_cast<const int*>(gm)[i];
  }
  __syncthreads();
  auto medium = [&](int l) -> const Medium<float>& {
    if constexpr (kUni) {
      return A.uni_f;
    } else {
      return sm_media[l];
    }
  };

  const int nx = A.nx;
  const int ny = A.ny, nz = A.nz;
  const int nxy = static_cast<int>(A.nxy);
  const float h = A.hf;
  const float tmax = A.tmaxf;
  const float qscale = A.qscalef;
  const int lane = threadIdx.x & 31;
  const unsigned lanemask_lt = (1u << lane) - 1u;

  // escaped / killed / truncated quanta change once per photon, so they live in
  // this thread's shared-memory slots (acc_sm[k * kBlock]: 0 escaped, 1 killed,
  // 2 truncated), not in registers; the deposited channel is booked by the fold
  long long* const acc_sm = reinterpret_cast<long long*>(smem + kAccOff) + threadIdx.x;
  acc_sm[0] = acc_sm[kBlock] = acc_sm[2 * kBlock] = 0;

  int phase = DEAD;
  bool exhausted = false;
  uint64_t idx = 0;
  Rng rng;
  rng.a = rng.b = 0;
  // photon state at the start of the current flight
  float px = 0, py = 0, pz = 0, dx = 0, dy = 0, dz = 1;
  float w = 0, tf = 0, rs = 0;  // weight at distance s0 along the flight; time and
                                // remaining scattering length at the flight start
  float s0 = 0;      // distance along the flight of the last face (or the flight start)
  float run_w0 = 0;  // weight at the start of the open deposit run (one voxel, one gate)
  float L = 0;       // flight length; sign bit set = the flight ends at the horizon.
                     // FACE: distance of the face event
  // incremental DDA
  float tmx = 0, tmy = 0, tmz = 0, tdx = 0, tdy = 0, tdz = 0;
  int vx = 0, vy = 0, vz = 0;  // voxel coordinates
  int sx = 0, sy = 0, sz = 0;  // +-1: direction of travel per axis
  int lab = 0, fax = 0;
  int gate = 0;
  float gate_end = 0;  // gated launches: the time at which `gate` ends (+inf for the last)
  // this CTA's replica of the fluence map (see KernelArgs::rep_mask); the host
  // keeps rep_mask * rep_stride < 2^31, so the offset is a 32-bit cell index
  const int roff = (static_cast<int>(blockIdx.x) & A.rep_mask) * static_cast<int>(A.rep_stride);
  unsigned long long* const cbase = reinterpret_cast<unsigned long long*>(A.cells) + roff;
  unsigned long long* gmap = cbase;  // cells of `gate` (gated launches)
  float fmua = 0, fns = 0;  // current medium (multi-label volumes): mua, n / c
  float sct = 0, sst = 0;  // scatter: cos/sin theta kept across azimuth retries
  uint32_t steps = 0, nscat = 0;
  double pd_dep = 0, pd_esc = 0, pd_kill = 0, pd_trunc = 0;  // trace only
  bool detected = false;
  float* pp_sm = reinterpret_cast<float*>(smem + kPpOff) + threadIdx.x;

  auto quant = [&](float x) -> long long { return __float2ll_rn(x * qscale); };
  auto gate_of = [&](float tt) -> int {
    const int g = static_cast<int>(tt * A.inv_gate_wf);  // tt >= 0: truncation == floor
    return g < A.ngates - 1 ? g : A.ngates - 1;
  };
  auto mua_ = [&]() -> float {
    if constexpr (kUni) {
      return A.uni_f.mua;
    } else {
      return fmua;
    }
  };
  auto nsmm_ = [&]() -> float {
    if constexpr (kUni) {
      return A.uni_f.ns_per_mm;
    } else {
      return fns;
    }
  };
  // Beer-Lambert over the segment [s0, s] of the flight (exp_neg,
  // transport.cpp:22-27): w -= w (1 - exp(-x)) in one rounding, with
  // 1 - exp(-x) from its Taylor series, so a run's deposit run_w0 - w (exact
  // by Sterbenz) keeps the step kernel's precision and the weights telescope
  // exactly. The series order is chosen per launch (warp-uniform branch) from
  // the largest mua * h * sqrt(3) of the volume: x^3 below 0.012, x^5 below
  // 0.15 (truncation < 1e-7 relative), else x^5 with a MUFU.EX2 fallback
  auto absorb = [&](float s) {
    const float x = mua_() * (s - s0);
    float f;
    if (kAbs == 0 || (kAbs < 0 && A.absorb_mode == 0)) {
      f = x * (1.0f - x * (0.5f - x * (1.0f / 6.0f)));
    } else {
      f = x * (1.0f - x * (0.5f - x * (1.0f / 6.0f - x * (1.0f / 24.0f - x * (1.0f / 120.0f)))));
      if (kAbs < 0 && A.absorb_mode == 2 && x >= 0.15f) {
        float e;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * -1.4426950408889634f));
        f = 1.0f - e;
      }
    }
    w = fmaf(-w, f, w);
    s0 = s;
  };
  auto cell = [&]() -> int { return vx + nx * vy + nxy * vz; };  // x-fastest linear index (two IMAD)
  // close the open deposit run at weight w_new: one fixed-point add into the
  // voxel the run belongs to (the map is L2-resident for cube60)
  auto deposit_run = [&]() {
    const float dw = run_w0 - w;
    const long long q = quant(dw);
    // q == 0 only if mua == 0; ungated launches index from the parameter-bank
    // base (one IMAD.WIDE), gated ones from the gate's pointer
    if constexpr (kGates) {
      atomicAdd(gmap + cell(), static_cast<unsigned long long>(q));
    } else {
      atomicAdd(reinterpret_cast<unsigned long long*>(A.cells) + (roff + cell()),
                static_cast<unsigned long long>(q));
    }
    if constexpr (kTrace) pd_dep += static_cast<double>(dw);
    run_w0 = w;
  };
  // The gate only changes when t passes gate_end, so the common case is one
  // compare; the gate index itself (gate_of, the semantics) is recomputed only
  // then. Returns true when the gate changed.
  auto set_gate = [&](float tt) -> bool {
    if constexpr (kGates) {
      if (tt >= gate_end) {
        const int g = gate_of(tt);
        const bool changed = g != gate;
        gate = g;
        gmap = cbase + static_cast<long long>(g) * A.nvox;
        const float e = static_cast<float>(g + 1) * A.gate_wf;
        // next boundary; one ulp further if rounding put tt past it in the same gate
        gate_end = g >= A.ngates - 1 ? Tr::inf() : (e > tt ? e : nextafterf(tt, Tr::inf()));
        return changed;
      }
    }
    return false;
  };
  auto add_path = [&](float s) {
    if constexpr (kDet) {
      if (lab >= 1) pp_sm[(lab - 1) * kBlock] += s;
    }
  };
  auto scat_len_of = [&](Rng& r) -> float {  // transport.cpp:14-17
    const float u = r.template unit<float>();
    return -Tr::ln(u > 0.0f ? u : 0x1p-25f);
  };
  auto scat_len = [&]() -> float { return scat_len_of(rng); };
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
    phase = DEAD;
  };

  // ---- flight setup: DDA state and flight length from the current state ----
  auto setup = [&]() {
    const Medium<float>& M = medium(lab);
    if constexpr (!kUni) {
      fmua = M.mua;
      fns = M.ns_per_mm;
    }
    s0 = 0.0f;
    const float ix = Tr::rcp(dx), iy = Tr::rcp(dy), iz = Tr::rcp(dz);  // +-inf for 0
    const int ux = vx, uy = vy, uz = vz;
    const float t0 = (static_cast<float>(ux + (dx > 0.0f ? 1 : 0)) * h - px) * ix;
    const float t1 = (static_cast<float>(uy + (dy > 0.0f ? 1 : 0)) * h - py) * iy;
    const float t2 = (static_cast<float>(uz + (dz > 0.0f ? 1 : 0)) * h - pz) * iz;
    tmx = dx != 0.0f ? fmaxf(t0, 0.0f) : Tr::inf();
    tmy = dy != 0.0f ? fmaxf(t1, 0.0f) : Tr::inf();
    tmz = dz != 0.0f ? fmaxf(t2, 0.0f) : Tr::inf();
    tdx = h * fabsf(ix);
    tdy = h * fabsf(iy);
    tdz = h * fabsf(iz);
    sx = dx > 0.0f ? 1 : -1;
    sy = dy > 0.0f ? 1 : -1;
    sz = dz > 0.0f ? 1 : -1;
    const float ds = M.mus > 0.0f ? rs * M.inv_mus : Tr::inf();  // rs may be 0 after a clamp
    const float rem = tmax - tf;
    const float dh = fmaxf(0.0f, rem * M.mm_per_ns);
    L = ds * M.ns_per_mm >= rem ? -dh : ds;  // horizon (transport.cpp:173-175) marked by the sign
    // a flight that ends before the first face skips the walk (short flights:
    // most of them in the head phantom's white matter)
    phase = fminf(tmx, fminf(tmy, tmz)) >= fabsf(L) ? ENDF : WALK;
  };

  // ---- the flight ended inside the current voxel (ENDF, event phase):
  // scattering point or horizon ----
  auto end_flight = [&]() {
    if constexpr (kTrace) ++steps;
    const float Ls = fabsf(L);
    absorb(Ls);
    px += dx * Ls;
    py += dy * Ls;
    pz += dz * Ls;
    const float te = tf + Ls * nsmm_();
    add_path(Ls);
    if (__float_as_int(L) < 0) {  // StepKind::Terminated (transport.cpp:181-187, 330-332)
      deposit_run();
      acc_sm[2 * kBlock] += quant(w);
      if constexpr (kTrace) pd_trunc += w;
      finish(2);
      return;
    }
    tf = te;
    rs = 0.0f;
    if constexpr (kGates) {
      if (te >= gate_end && gate_of(te) != gate) deposit_run();  // a new gate closes the run
      set_gate(te);
    }
    phase = SCAT;
  };

  // ---- one walk step of a lane in flight: the next face, or the end of the
  // flight. Branch-free apart from the rare interface / exit tail, so the
  // lanes of a warp stay converged ----
  // A lane is WALK only while its next face comes before the end of the
  // flight (checked at setup and after every face, scatter / horizon win ties,
  // transport.cpp:175, 191), so every lane that enters a walk step crosses.
  auto walk = [&]() {
    const float s = fminf(tmx, fminf(tmy, tmz));
    absorb(s);
    if constexpr (kTrace) ++steps;
    deposit_run();  // the voxel left behind
    const bool a0 = tmx == s;  // ties -> lower axis (boundary_distance)
    const bool a1 = !a0 && tmy == s;
    const bool a2 = !a0 && !a1;
    // predicated updates of the one axis that moves
    if (a0) vx += sx;
    if (a1) vy += sy;
    if (a2) vz += sz;
    if (a0) tmx += tdx;
    if (a1) tmy += tdy;
    if (a2) tmz += tdz;
    const bool ext = static_cast<unsigned>(vx) >= static_cast<unsigned>(nx) ||
                     static_cast<unsigned>(vy) >= static_cast<unsigned>(ny) ||
                     static_cast<unsigned>(vz) >= static_cast<unsigned>(nz);
    if constexpr (kGates) set_gate(tf + s * nsmm_());
    bool ev = ext;
    if constexpr (!kUni) {
      if (!ext) ev = static_cast<int>(__ldg(A.labels + cell())) != lab;
    }
    if (ev) {
      if (!kDet && ext && !A.reflect) {  // TerminateAtBoundary: ExitedDomain at once
        acc_sm[0] += quant(w);
        if constexpr (kTrace) pd_esc += w;
        finish(0);
      } else {
        phase = FACE;
        L = s;
        fax = a0 ? 0 : (a1 ? 1 : 2);
      }
    } else if (fminf(tmx, fminf(tmy, tmz)) >= fabsf(L)) {
      phase = ENDF;  // the flight ends in this voxel
    }
  };

  // ---- hg_scatter + new free path + roulette (transport.cpp:126-147, 14-17, 333-343) ----
  auto scatter = [&]() {
    const Medium<float>& M = medium(lab);
    if (phase == SCAT) {  // Henyey-Greenstein cos(theta) (transport.cpp:120-124)
      if constexpr (kTrace || kDet) ++nscat;
      const float xi = rng.template unit<float>();
      float ct;
      if (M.iso) {
        ct = 2.0f * xi - 1.0f;
      } else {
        const float f = M.hg_c * Tr::rcp(M.hg_d + M.hg_e * xi);
        ct = fminf(1.0f, fmaxf(-1.0f, M.hg_a - f * f * M.hg_b));
      }
      sct = ct;
      sst = Tr::sqrt_(fmaxf(0.0f, 1.0f - ct * ct));
    }
    // rejection azimuth (transport.cpp:32-44), VMC_AZ_UNROLL tries per event
    // phase; a lane rejected every time keeps cos/sin(theta) and retries in the
    // next event phase
    float ax_ = 0, ay_ = 0, r2 = 0;
    bool ok = false;
#pragma unroll
    for (int k = 0; k < VMC_AZ_UNROLL; ++k) {
      if (k == 0 || !ok) {
        ax_ = fmaf(rng.u24(), 0x1p-23f, -1.0f);  // 2u - 1, exact
        ay_ = fmaf(rng.u24(), 0x1p-23f, -1.0f);
        r2 = ax_ * ax_ + ay_ * ay_;
        ok = r2 > 1e-12f && r2 <= 1.0f;
      }
    }
    if (!ok) {
      phase = RETRY;
      return;
    }
    const float k = Tr::rsqrt(r2);
    const float cp = ax_ * k, sp = ay_ * k;
    const float ct = sct, st = sst;
    float ox, oy, oz;
    if (fabsf(dz) > 0.99999f) {  // transport.cpp:133-136
      ox = st * cp;
      oy = st * sp;
      oz = dz > 0.0f ? ct : -ct;
    } else {
      const float one_m = 1.0f - dz * dz;
      const float rden = Tr::rsqrt(one_m);
      const float sr = st * rden;
      ox = sr * (dx * dz * cp - dy * sp) + dx * ct;
      oy = sr * (dy * dz * cp + dx * sp) + dy * ct;
      oz = -st * cp * (one_m * rden) + dz * ct;
    }
    const float n2 = ox * ox + oy * oy + oz * oz;  // renormalize (1e-6 in FP32)
    if (fabsf(n2 - 1.0f) > 1e-6f) {
      const float kk = Tr::rsqrt(n2);
      ox *= kk;
      oy *= kk;
      oz *= kk;
    }
    dx = ox;
    dy = oy;
    dz = oz;
    rs = scat_len();
    phase = SETUP;
    if (w < A.rthrf) {  // roulette after a scatter only (transport.cpp:300-306)
      const bool survive = rng.template unit<float>() < A.inv_rmultf;
      deposit_run();  // close the deposit run before the weight jumps
      const long long qb = quant(w);
      if constexpr (kTrace) pd_kill += w;
      if (!survive) {
        acc_sm[kBlock] += qb;
        finish(1);
        return;
      }
      w *= A.rmultf;
      acc_sm[kBlock] += qb - quant(w);
      if constexpr (kTrace) pd_kill -= w;
      run_w0 = w;
    }
  };

  // ---- interface / exterior face at distance L (handle_interface, transport.cpp:227-298) ----
  auto face = [&]() {
    const float s = L;
    const int ax = fax;
    const float t = tf + s * nsmm_();
    {
      // land exactly on the crossed plane (transport.cpp:197-204); the voxel
      // index has already moved, so the plane is its near face
      const int u = ax == 0 ? vx : (ax == 1 ? vy : vz);
      const float dax = ax == 0 ? dx : (ax == 1 ? dy : dz);
      const float plane = static_cast<float>(dax > 0.0f ? u : u + 1) * h;
      px = ax == 0 ? plane : px + dx * s;
      py = ax == 1 ? plane : py + dy * s;
      pz = ax == 2 ? plane : pz + dz * s;
    }
    add_path(s);
    const Medium<float>& M = medium(lab);
    rs = fmaxf(0.0f, rs - s * M.mus);
    const bool ext = static_cast<unsigned>(vx) >= static_cast<unsigned>(nx) ||
                     static_cast<unsigned>(vy) >= static_cast<unsigned>(ny) ||
                     static_cast<unsigned>(vz) >= static_cast<unsigned>(nz);
    const int nl = ext ? 0 : static_cast<int>(__ldg(A.labels + cell()));
    bool exited = false, back = false;
    if (ext && !A.reflect) {
      exited = true;  // TerminateAtBoundary (transport.cpp:234-237)
    } else {
      const int c1 = M.nclass, c2 = sm_media[nl].nclass;
      if (c1 == c2) {
        exited = ext;  // n1 == n2: identity interface / same-n move (:218-223, 242-252)
      } else {
        const float dax = ax == 0 ? dx : (ax == 1 ? dy : dz);
        const float n1 = M.n, n2 = sm_media[nl].n;
        const float ci = fabsf(dax);
        const float si2 = fmaxf(0.0f, 1.0f - ci * ci);
        // MUFU reciprocal / sqrt: R only meets a 24-bit uniform, and the
        // interface code runs on few lanes at a time, so its length is its cost
        const float eta = n1 * Tr::rcp(n2);
        const float st2 = eta * eta * si2;
        if (st2 > 1.0f) {
          back = true;  // total internal reflection: deterministic flip
        } else {
          const float cost = Tr::sqrt_(1.0f - st2);
          const float rsp = (n1 * ci - n2 * cost) * Tr::rcp(n1 * ci + n2 * cost);
          const float rpp = (n1 * cost - n2 * ci) * Tr::rcp(n1 * cost + n2 * ci);
          const float R = 0.5f * (rsp * rsp + rpp * rpp);
          if (rng.template unit<float>() < R) {
            back = true;
          } else {  // Snell refraction, tangential components scaled by n1/n2
            const float nc = dax > 0.0f ? cost : -cost;
            const float qx = ax == 0 ? nc : dx * eta;
            const float qy = ax == 1 ? nc : dy * eta;
            const float qz = ax == 2 ? nc : dz * eta;
            const float k = Tr::rsqrt(qx * qx + qy * qy + qz * qz);
            dx = qx * k;
            dy = qy * k;
            dz = qz * k;
            exited = ext;
          }
        }
      }
    }
    if (exited) {  // ExitedDomain: escaped += w (transport.cpp:348-350)
      acc_sm[0] += quant(w);
      if constexpr (kTrace) pd_esc += w;
      if constexpr (kDet) {
        int hit = -1;
        for (int k = 0; k < A.ndet; ++k) {
          // FP32 like the exit position itself (detf = {x, y, z, r^2})
          const float ex = px - A.detf[k][0], ey = py - A.detf[k][1], ez = pz - A.detf[k][2];
          if (ex * ex + ey * ey + ez * ez <= A.detf[k][3]) {
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
              hd.w_exit = w;
              hd.t_exit_ns = t;
              *reinterpret_cast<vmc_det_record_head*>(rec) = hd;
              float* pp = reinterpret_cast<float*>(rec + sizeof(vmc_det_record_head));
              for (int m = 0; m < A.nppath; ++m) pp[m] = pp_sm[m * kBlock];
            }
          }
        }
      }
      finish(0);
      return;
    }
    if (back) {  // reflected: stay in the voxel, flip the normal component
      if (ax == 0) {
        vx -= sx;
        dx = -dx;
      } else if (ax == 1) {
        vy -= sy;
        dy = -dy;
      } else {
        vz -= sz;
        dz = -dz;
      }
    } else {
      lab = nl;
    }
    tf = t;
    phase = SETUP;
  };

  // ---- launch (transport.cpp:83-106) ----
  // the caller has set idx and seeded rng (from the warp's seed stash)
  auto launch = [&]() {
    int ux, uy, uz;
    if (A.iso_source) {
      const float ct = 2.0f * rng.template unit<float>() - 1.0f;
      const float u2 = rng.template unit<float>();
      float st, cphi, sphi;
      st = sqrtf(fmaxf(0.0f, 1.0f - ct * ct));
      sincospif(2.0f * u2, &sphi, &cphi);
      dx = st * cphi;
      dy = st * sphi;
      dz = ct;
      // nudge + voxel_of in double (the 1e-6 mm nudge is below FP32 ulp)
      const double qx = A.src_pos[0] + static_cast<double>(dx) * 1e-6;
      const double qy = A.src_pos[1] + static_cast<double>(dy) * 1e-6;
      const double qz = A.src_pos[2] + static_cast<double>(dz) * 1e-6;
      ux = static_cast<int>(floor(qx / A.h));
      uy = static_cast<int>(floor(qy / A.h));
      uz = static_cast<int>(floor(qz / A.h));
      px = static_cast<float>(qx);
      py = static_cast<float>(qy);
      pz = static_cast<float>(qz);
      if (ux < 0 || uy < 0 || uz < 0 || ux >= nx || uy >= A.ny || uz >= A.nz) {
        atomicExch(A.error_flag, 1);
        ux = uy = uz = 0;
        dx = dy = 0.0f;
        dz = 1.0f;
      }
      lab = __ldg(A.labels + (ux + nx * (uy + static_cast<long long>(A.ny) * uz)));
    } else {
      dx = static_cast<float>(A.dir0[0]);
      dy = static_cast<float>(A.dir0[1]);
      dz = static_cast<float>(A.dir0[2]);
      px = static_cast<float>(A.pos0[0]);
      py = static_cast<float>(A.pos0[1]);
      pz = static_cast<float>(A.pos0[2]);
      ux = A.v0[0];
      uy = A.v0[1];
      uz = A.v0[2];
      lab = A.lab0;
    }
    vx = ux;
    vy = uy;
    vz = uz;
    w = 1.0f;
    tf = 0.0f;
    run_w0 = 1.0f;
    if (A.iso_source) rs = scat_len();  // pencil: drawn in the seed batch
    if constexpr (kGates) {
      gate = 0;
      gmap = cbase;
      gate_end = A.ngates > 1 ? A.gate_wf : Tr::inf();
    }
    if constexpr (kTrace) {
      steps = nscat = 0;
      pd_dep = pd_esc = pd_kill = pd_trunc = 0;
    }
    if constexpr (kDet) {
      nscat = 0;
      for (int m = 0; m < A.nppath; ++m) pp_sm[m * kBlock] = 0.0f;
    }
    phase = SETUP;
  };

  // per-warp seed stash in shared memory: 32 seeded RNG states of the photons
  // st_base + 0..31 and a header {next unused slot, valid slots}; st_base and
  // st_claimed_all are warp-uniform registers
  const int warp = threadIdx.x >> 5;
  unsigned char* const stash = smem + kStashOff + warp * (32 * 20 + 16);
  uint64_t* const st_a = reinterpret_cast<uint64_t*>(stash);
  uint64_t* const st_b = st_a + 32;
  float* const st_rs = reinterpret_cast<float*>(stash + 32 * 16);  // pencil sources: first free path
  int* const st_hdr = reinterpret_cast<int*>(stash + 32 * 16 + 32 * 4);
  if (lane == 0) st_hdr[0] = st_hdr[1] = 0;
  __syncwarp();
  unsigned long long st_base = 0;
  bool st_claimed_all = false;

#ifdef VMC_STATS
  unsigned long long st_[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define VMC_ST(i, v) st_[i] += exhausted ? 0 : (v)  // steady state only (no drain tail)
#else
#define VMC_ST(i, v)
#endif
  for (;;) {
    // ================= event phase =================
#ifdef VMC_STATS
    VMC_ST(0, 1);
    VMC_ST(1, __popc(__ballot_sync(0xffffffffu, phase == WALK)));
    VMC_ST(2, __popc(__ballot_sync(0xffffffffu, phase == ENDF)));
    VMC_ST(3, __popc(__ballot_sync(0xffffffffu, phase == RETRY)));
    VMC_ST(4, __popc(__ballot_sync(0xffffffffu, phase == DEAD)));
    VMC_ST(5, __popc(__ballot_sync(0xffffffffu, phase == FACE)));
#endif
    {
      const unsigned dead = __ballot_sync(0xffffffffu, phase == DEAD);
      if (dead && !exhausted) {
        // Refill from the warp's seed stash: photons are claimed 32 at a time
        // (GroupCounter::claim, one atomicAdd) and all 32 lanes seed them at once
        // (two splitmix64 finalizers each, rng.cpp:5-19), so a relaunch no longer
        // runs the seeding on the one or two lanes that happen to be free.
        const int nd = __popc(dead);
        const int rank = __popc(dead & lanemask_lt);
        const int next = st_hdr[0], valid = st_hdr[1];
        const int take1 = min(nd, valid - next);
        int slot = -1;
        unsigned long long pid = 0;
        if (phase == DEAD && rank < take1) {
          slot = next + rank;
          pid = st_base + static_cast<unsigned long long>(slot);
          rng.a = st_a[slot];
          rng.b = st_b[slot];
          rs = st_rs[slot];
        }
        int new_next = next + take1;
        if (nd > take1 && !st_claimed_all) {  // claim and seed a new batch of 32
          unsigned long long base = 0;
          if (lane == 0) base = atomicAdd(A.claim, 32ull);
          base = __shfl_sync(0xffffffffu, base, 0);
          const int nvalid = base >= A.count ? 0 : static_cast<int>(min(32ull, A.count - base));
          if (base + 32 >= A.count) st_claimed_all = true;
          __syncwarp();
          if (lane < nvalid) {
            Rng sr;
            sr.seed(A.seed, A.first + base + lane);
            if (!A.iso_source) st_rs[lane] = scat_len_of(sr);  // a pencil's first draw (transport.cpp:105)
            st_a[lane] = sr.a;
            st_b[lane] = sr.b;
          }
          __syncwarp();
          const int take2 = min(nd - take1, nvalid);
          if (phase == DEAD && rank >= take1 && rank - take1 < take2) {
            slot = rank - take1;
            pid = base + static_cast<unsigned long long>(slot);
            rng.a = st_a[slot];
            rng.b = st_b[slot];
            rs = st_rs[slot];
          }
          st_base = base;
          new_next = take2;
          if (lane == 0) st_hdr[1] = nvalid;
        }
        if (lane == 0) st_hdr[0] = new_next;
        __syncwarp();
        if (st_claimed_all && st_hdr[0] == st_hdr[1]) exhausted = true;
        if (slot >= 0) {
          idx = A.first + pid;
          if constexpr (kTrace) rng.draws = A.iso_source ? 0 : 1;
          launch();
        }
      }
    }
    // multi-label kernels: reconverge after the refill (+3 % B3, +1.5 % head;
    // the single-label kernel is ~0.4 % faster without)
    if constexpr (!kUni) __syncwarp();
    if (phase == ENDF) end_flight();
    if (phase == SCAT || phase == RETRY) scatter();
    if (phase == FACE) face();
    __syncwarp();  // reconverge before the shared flight setup (face() has warp-level votes)
    if (phase == SETUP) setup();
    // ================= walk phase =================
    // every lane in flight crosses faces until at most (100 - event_pct) % of
    // the live lanes are still walking; the others wait for the event phase
    // walk_keep, scaled to the live lanes once the photons have run out
    int keep = A.walk_keep;
    if (exhausted) {
      const unsigned dead = __ballot_sync(0xffffffffu, phase == DEAD);
      if (dead == 0xffffffffu) break;
      keep = ((32 - __popc(dead)) * A.walk_keep) >> 5;
    }
    // After an event phase nearly every lane walks in the cube60 kernels, so
    // their first vote is skipped (+1 %); in the strongly scattering head most
    // new flights end in their voxel, so the gated kernel votes first
    // (three steps per vote amortise the loop control; 2 and 4 measured slower)
    if constexpr (kGates) {
      while (__popc(__ballot_sync(0xffffffffu, phase == WALK)) > keep) {
        VMC_ST(6, 1);
        if (phase == WALK) walk();
        if (phase == WALK) walk();
        if (phase == WALK) walk();
      }
    } else {
      do {
        VMC_ST(6, 1);
        if (phase == WALK) walk();
        if (phase == WALK) walk();
        if (phase == WALK) walk();
      } while (__popc(__ballot_sync(0xffffffffu, phase == WALK)) > keep);
    }
  }

  // ---- epilogue: dispositions (warp reduce) ----
  long long acc_esc = acc_sm[0], acc_kill = acc_sm[kBlock], acc_trunc = acc_sm[2 * kBlock];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc_esc += __shfl_xor_sync(0xffffffffu, acc_esc, o);
    acc_kill += __shfl_xor_sync(0xffffffffu, acc_kill, o);
    acc_trunc += __shfl_xor_sync(0xffffffffu, acc_trunc, o);
  }
#ifdef VMC_STATS
  if (lane == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(&vmc_flight_stats[i], st_[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&vmc_flight_done, 1u) == gridDim.x - 1) {
      const double ev = static_cast<double>(vmc_flight_stats[0]), wi = static_cast<double>(vmc_flight_stats[6]);
      printf("[vmc stats] event phases %llu: walking %.2f endf %.2f retry %.2f dead %.2f face %.2f | walk iters %llu"
             " (%.2f per event phase), walking lanes %.2f\n",
             vmc_flight_stats[0], vmc_flight_stats[1] / ev, vmc_flight_stats[2] / ev, vmc_flight_stats[3] / ev,
             vmc_flight_stats[4] / ev, vmc_flight_stats[5] / ev, vmc_flight_stats[6], wi / ev,
             vmc_flight_stats[7] / wi);
      for (int i = 0; i < 12; ++i) vmc_flight_stats[i] = 0;
      vmc_flight_done = 0;
    }
  }
#undef VMC_ST
#endif
  if (lane == 0) {
    unsigned long long* tot = reinterpret_cast<unsigned long long*>(A.totals);
    if (acc_esc) atomicAdd(tot + 1, static_cast<unsigned long long>(acc_esc));
    if (acc_kill) atomicAdd(tot + 2, static_cast<unsigned long long>(acc_kill));
    if (acc_trunc) atomicAdd(tot + 3, static_cast<unsigned long long>(acc_trunc));
  }
}

}  // namespace vmc
