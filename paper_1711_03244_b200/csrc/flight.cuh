// flight.cuh — K1f, the photon-transport kernel organised by free flight (sm_100a).
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
// Two arithmetic instantiations of the same body:
//   float  — the product path (MUFU transcendentals, FP32 Taylor absorb,
//            deposits coalesced per (voxel, gate) run, u = top 24 bits);
//   double — the exact-arithmetic pin of the product kernel's structure
//            (compiled with --fmad=false): the reference's own formulas op for
//            op (exp_neg, hg_cos_theta, the azimuth rejection, Fresnel, Snell,
//            u = top 53 bits, libm-style log/exp/sqrt) and one llround deposit
//            per step like FluenceMap::deposit, so each photon's dispositions
//            match the reference to ~1e-12 whenever its discrete path does.
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

// The arithmetic that differs between the FP32 product path and the FP64 pin.
template <typename Real>
struct FlightOps;

template <>
struct FlightOps<float> {
  static constexpr bool kF32 = true;
  using Tr = RealTraits<float>;
  static __device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
  static __device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
  static __device__ __forceinline__ float vabs(float a) { return fabsf(a); }
  static __device__ __forceinline__ bool neg(float a) { return __float_as_int(a) < 0; }
  static __device__ __forceinline__ float up(float a) { return nextafterf(a, Tr::inf()); }
  static __device__ __forceinline__ float pick(float f, double) { return f; }
  static __device__ __forceinline__ long long quant(float x, float qscale) { return __float2ll_rn(x * qscale); }
  // 2u - 1 for the rejection azimuth, exact from the top 24 bits
  template <class Rng>
  static __device__ __forceinline__ float two_u_m1(Rng& r) {
    return fmaf(r.u24(), 0x1p-23f, -1.0f);
  }
  // -log(u) (transport.cpp:14-17); u = 0 (p = 2^-24) stands for [0, 2^-24): 2^-25
  template <class Rng>
  static __device__ __forceinline__ float scat_len(Rng& r) {
    const float u = r.template unit<float>();
    return -Tr::ln(u > 0.0f ? u : 0x1p-25f);
  }
};

template <>
struct FlightOps<double> {
  static constexpr bool kF32 = false;
  using Tr = RealTraits<double>;
  static __device__ __forceinline__ double vmin(double a, double b) { return fmin(a, b); }
  static __device__ __forceinline__ double vmax(double a, double b) { return fmax(a, b); }
  static __device__ __forceinline__ double vabs(double a) { return fabs(a); }
  static __device__ __forceinline__ bool neg(double a) { return __double_as_longlong(a) < 0; }
  static __device__ __forceinline__ double up(double a) { return nextafter(a, Tr::inf()); }
  static __device__ __forceinline__ double pick(float, double d) { return d; }
  static __device__ __forceinline__ long long quant(double x, double qscale) { return llround(x * qscale); }
  template <class Rng>
  static __device__ __forceinline__ double two_u_m1(Rng& r) {
    return 2.0 * r.template unit<double>() - 1.0;
  }
  template <class Rng>
  static __device__ __forceinline__ double scat_len(Rng& r) {
    const double u = r.template unit<double>();
    return -log(u > 0.0 ? u : 4.9406564584124654e-324);
  }
};

// kDep: how a closed deposit run reaches the fluence map (all three give the
// same integer sums, so bit-identical maps):
//   kDepDirect  one red.global.add.u64 per run into the CTA's map replica;
//   kDepWarp    warp-aggregated: lanes of one deposit instruction that hit
//               the same cell (__match_any_sync) sum their quanta by pointer
//               jumping along the peer list and the lowest lane issues one
//               red; a warp whose lanes all hit distinct cells takes the
//               direct path after one vote;
//   kDepHotBox  an SM-local accumulator: runs inside a 16^3 box around the
//               source voxel (36 % of B1's deposits) add into
//               a per-CTA shared-memory box (u64 as a lo/hi u32 pair with an
//               exact carry: native ATOMS.ADD instead of a 64-bit CAS loop),
//               flushed to the map with one red per non-empty cell at CTA
//               exit (the reference's private-map merge, scheduler.cpp:
//               268-275,312-314, at CTA granularity). Ungated kernels only.
// (kDepDirect / kDepWarp / kDepHotBox, kHotBoxN: transport.cuh)

// kSolo: the small-run instantiation (host: launches below ~30 photons per
// full-grid thread). Once the claims have run out, a warp's last live photon
// finishes in a lane-local loop (no votes, no event-phase dispatch); a
// separate instantiation so the large-run kernel's code is untouched.
template <typename Real, bool kGates, bool kDet, bool kTrace, bool kUni, int kDep = kDepDirect, bool kSolo = false>
__device__ __forceinline__ void flight_body(const KernelArgs& A) {
  using Tr = RealTraits<Real>;
  using F = FlightOps<Real>;
  constexpr bool kF32 = F::kF32;
  using Rng = Xs128p<kTrace>;
  constexpr int WALK = 0, SCAT = 1, DEAD = 2, RETRY = 3, FACE = 4, SETUP = 5, ENDF = 6;
  unsigned char* smem = vmc_smem;
  // Shared-memory layout at compile-time offsets (cheap to rematerialise):
  // per-thread disposition slots | per-warp seed stashes | [hot box] | media
  // table | per-thread path lengths (detector kernels, after the media)
  constexpr int kStashBytes = flight_stash_bytes(sizeof(Real));
  constexpr int kAccOff = 0;                                       // 3 x kBlock x int64
  constexpr int kStashOff = kAccOff + 3 * kBlock * 8;              // kBlock / 32 x kStashBytes
  constexpr int kHbOff = kStashOff + (kBlock / 32) * kStashBytes;
  constexpr int kMediaOff = kHbOff + (kDep == kDepHotBox ? kHotBoxBytes : 0);
  static_assert(kStashOff % 16 == 0 && kHbOff % 16 == 0 && kMediaOff % 16 == 0, "smem alignment");
  // detector kernels: per-thread per-label path lengths after the media table,
  // sized by the volume's interior labels (nppath x kBlock), not the maximum,
  // so the L1 keeps the rest of the SM's 256 KB for the label volume
  static_assert(kDep != kDepHotBox || !kGates, "the hot box serves ungated kernels");
  constexpr int kHbCells = kHotBoxN * kHotBoxN * kHotBoxN;
  unsigned* const hb_lo = reinterpret_cast<unsigned*>(smem + kHbOff);
  unsigned* const hb_hi = hb_lo + kHbCells;
  if constexpr (kDep == kDepHotBox) {
    for (int i = threadIdx.x; i < 2 * kHbCells; i += blockDim.x) hb_lo[i] = 0u;
  }

  // ---- shared memory: media table (exterior n is needed even when kUni) ----
  Medium<Real>* sm_media = reinterpret_cast<Medium<Real>*>(smem + kMediaOff);
  {
    const Medium<Real>* gm = static_cast<const Medium<Real>*>(A.media);
    const int nwords = static_cast<int>(sizeof(Medium<Real>) / 4) * A.nmedia;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x)
      reinterpret_cast<int*>(sm_media)[i] = reinterpret_cast<const int*>(gm)[i];
  }
  __syncthreads();
  auto medium = [&](int l) -> const Medium<Real>& {
    if constexpr (kUni) {
      if constexpr (kF32) {
        return A.uni_f;
      } else {
        return A.uni_d;
      }
    } else {
      return sm_media[l];
    }
  };

  const int nx = A.nx;
  const int ny = A.ny, nz = A.nz;
  const int nxy = static_cast<int>(A.nxy);
  const Real h = F::pick(A.hf, A.h);
  const Real tmax = F::pick(A.tmaxf, A.tmax);
  const Real qscale = F::pick(A.qscalef, A.qscale);
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
  Real px = 0, py = 0, pz = 0, dx = 0, dy = 0, dz = 1;
  Real w = 0, tf = 0, rs = 0;  // weight at distance s0 along the flight; time and
                               // remaining scattering length at the flight start
  Real s0 = 0;      // distance along the flight of the last face (or the flight start)
  Real w_fl = 0;    // FP32: weight at the flight start
  Real run_w0 = 0;  // weight at the start of the open deposit run (one voxel, one gate)
  Real L = 0;       // flight length; sign bit set = the flight ends at the horizon.
                    // FACE: distance of the face event
  // incremental DDA
  Real tmx = 0, tmy = 0, tmz = 0, tdx = 0, tdy = 0, tdz = 0;
  int vx = 0, vy = 0, vz = 0;  // voxel coordinates
  int sx = 0, sy = 0, sz = 0;  // +-1: direction of travel per axis
  int lab = 0, fax = 0;
  int gate = 0;
  Real gate_end = 0;  // gated launches: the time at which `gate` ends (+inf for the last)
  // this CTA's replica of the fluence map (see KernelArgs::rep_mask); the host
  // keeps rep_mask * rep_stride < 2^31, so the offset is a 32-bit cell index
  const int roff = (static_cast<int>(blockIdx.x) & A.rep_mask) * static_cast<int>(A.rep_stride);
  unsigned long long* const cbase = reinterpret_cast<unsigned long long*>(A.cells) + roff;
  unsigned long long* gmap = cbase;  // cells of `gate` (gated launches)
  Real fmua = 0, fns = 0;  // current medium (multi-label volumes): mua, n / c
  Real fka = 0;            // FP32 multi-label volumes: -mua log2(e) of the current medium
  Real sct = 0, sst = 0;  // scatter: cos/sin theta kept across azimuth retries
  uint32_t steps = 0, nscat = 0;
  double pd_dep = 0, pd_esc = 0, pd_kill = 0, pd_trunc = 0;  // trace only
  bool detected = false;
  Real* pp_sm = reinterpret_cast<Real*>(
                    smem + kMediaOff + ((static_cast<int>(sizeof(Medium<Real>)) * A.nmedia + 15) & ~15)) +
                threadIdx.x;
  Real seg = 0;  // detector kernels: path length in the current medium since the last flush

  auto quant = [&](Real x) -> long long { return F::quant(x, qscale); };
  auto gate_of = [&](Real tt) -> int {
    const int g = static_cast<int>(tt * F::pick(A.inv_gate_wf, A.inv_gate_w));  // tt >= 0: truncation == floor
    return g < A.ngates - 1 ? g : A.ngates - 1;
  };
  auto mua_ = [&]() -> Real {
    if constexpr (kUni) {
      return medium(0).mua;
    } else {
      return fmua;
    }
  };
  auto nsmm_ = [&]() -> Real {
    if constexpr (kUni) {
      return medium(0).ns_per_mm;
    } else {
      return fns;
    }
  };
  // Beer-Lambert along the flight (exp_neg, transport.cpp:22-27).
  // FP32: w(s) = w_fl 2^(ka s), ka = -mua log2(e), from the weight at the
  // flight start in one MUFU.EX2 (3 instructions per face instead of a Taylor
  // chain on the segment); a run's deposit run_w0 - w is an exact difference
  // of two stored weights, so the deposits along a flight telescope exactly
  // (A/B on B200: +1.9 % B1/B2, +3.2 % B3 against the Taylor-3 chain).
  // FP64: w *= exp_neg(x) per segment, the reference's degree-4 series below
  // 0.01, else exp.
  auto absorb = [&](Real s) {
    if constexpr (kF32) {
      float e;
      const float ka = kUni ? medium(0).ka : fka;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(ka * s));
      w = w_fl * e;
    } else {
      const double x = mua_() * (s - s0);
      const double e = x < 0.01 ? 1.0 - x * (1.0 - x * (0.5 - x * (1.0 / 6.0 - x * (1.0 / 24.0)))) : exp(-x);
      w = w * e;
    }
    s0 = s;
  };
  auto cell = [&]() -> int { return vx + nx * vy + nxy * vz; };  // x-fastest linear index (two IMAD)
  // one fixed-point add of q quanta into the current voxel's cell
  auto red_cell = [&](unsigned long long q) {
    // ungated launches index from the parameter-bank base (one IMAD.WIDE),
    // gated ones from the gate's pointer
    if constexpr (kGates) {
      atomicAdd(gmap + cell(), q);
    } else {
      atomicAdd(reinterpret_cast<unsigned long long*>(A.cells) + (roff + cell()), q);
    }
  };
  auto add_quanta = [&](unsigned long long q) {
    if constexpr (kDep == kDepHotBox) {
      const unsigned ux = static_cast<unsigned>(vx - A.hb0[0]), uy = static_cast<unsigned>(vy - A.hb0[1]),
                     uz = static_cast<unsigned>(vz - A.hb0[2]);
      if ((ux | uy | uz) < static_cast<unsigned>(kHotBoxN)) {
        const int i = static_cast<int>(ux + kHotBoxN * (uy + kHotBoxN * uz));
        const unsigned lo = static_cast<unsigned>(q);
        const unsigned old = atomicAdd(hb_lo + i, lo);
        const unsigned hi = static_cast<unsigned>(q >> 32) + (old + lo < old ? 1u : 0u);  // exact carry
        if (hi) atomicAdd(hb_hi + i, hi);
        return;
      }
      red_cell(q);
    } else if constexpr (kDep == kDepWarp) {
      const unsigned am = __activemask();
      // the cell's offset in the (gated) map: lanes of different gates never merge
      unsigned peers;
      if constexpr (kGates) {
        peers = __match_any_sync(am, static_cast<unsigned long long>(gmap - cbase) + cell());
      } else {
        peers = __match_any_sync(am, cell());
      }
      if (__all_sync(am, peers == (1u << lane))) {
        red_cell(q);
        return;
      }
      // suffix sums along each peer list by pointer jumping: after five
      // rounds every lane holds the sum of itself and the peers above it,
      // so the lowest peer holds its group's total
      const unsigned above = peers & (0xfffffffeu << lane);
      int nxt = above ? __ffs(above) - 1 : -1;
      unsigned long long v = q;
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        const int src = nxt >= 0 ? nxt : lane;
        const unsigned long long o = __shfl_sync(am, v, src);
        const int n2 = __shfl_sync(am, nxt, src);
        if (nxt >= 0) {
          v += o;
          nxt = n2;
        }
      }
      if ((peers & lanemask_lt) == 0) red_cell(v);
    } else {
      red_cell(q);
    }
  };
  // close the open deposit run at weight w: one fixed-point add into the
  // voxel the run belongs to (the map is L2-resident for cube60)
  auto deposit_run = [&]() {
    const Real dw = run_w0 - w;
    const long long q = quant(dw);
    // FP32: q == 0 only if mua == 0. FP64: one run per step; empty steps add
    // nothing (run_photon :325-328)
    if (kF32 || q != 0) add_quanta(static_cast<unsigned long long>(q));
    if constexpr (kTrace) {
      if (A.dep_n && dw != Real(0)) {  // the reference's sink sees every nonzero step deposit
        const unsigned long long k = atomicAdd(A.dep_n, 1ull);
        if (k < A.dep_cap) {
          A.dep_cells[k] = cell();
          A.dep_w[k] = static_cast<double>(dw);
        }
      }
    }
    if constexpr (kTrace) pd_dep += static_cast<double>(dw);
    run_w0 = w;
  };
  // The gate only changes when t passes gate_end, so the common case is one
  // compare; the gate index itself (gate_of, the semantics) is recomputed only
  // then. Returns true when the gate changed.
  auto set_gate = [&](Real tt) -> bool {
    if constexpr (kGates) {
      if (tt >= gate_end) {
        const int g = gate_of(tt);
        const bool changed = g != gate;
        gate = g;
        gmap = cbase + static_cast<long long>(g) * A.nvox;
        const Real e = static_cast<Real>(g + 1) * F::pick(A.gate_wf, A.tmax / A.ngates);
        // next boundary; one ulp further if rounding put tt past it in the same gate
        gate_end = g >= A.ngates - 1 ? Tr::inf() : (e > tt ? e : F::up(tt));
        return changed;
      }
    }
    return false;
  };
  // detector kernels: path length in the current medium accumulates in a
  // register and goes to this thread's per-label slot in shared memory only
  // when the label changes or the photon exits (B3: ~3.5 label changes against
  // ~160 flight segments per photon)
  auto add_path = [&](Real s) {
    if constexpr (kDet) seg += s;
  };
  auto flush_path = [&]() {
    if constexpr (kDet) {
      if (lab >= 1) pp_sm[(lab - 1) * kBlock] += seg;
      seg = Real(0);
    }
  };
  auto scat_len = [&]() -> Real { return F::scat_len(rng); };
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
    const Medium<Real>& M = medium(lab);
    if constexpr (!kUni) {
      fmua = M.mua;
      fns = M.ns_per_mm;
      fka = M.ka;
    }
    s0 = Real(0);
    w_fl = w;
    const Real ix = Tr::rcp(dx), iy = Tr::rcp(dy), iz = Tr::rcp(dz);  // +-inf for 0
    const int ux = vx, uy = vy, uz = vz;
    const Real t0 = (static_cast<Real>(ux + (dx > Real(0) ? 1 : 0)) * h - px) * ix;
    const Real t1 = (static_cast<Real>(uy + (dy > Real(0) ? 1 : 0)) * h - py) * iy;
    const Real t2 = (static_cast<Real>(uz + (dz > Real(0) ? 1 : 0)) * h - pz) * iz;
    tmx = dx != Real(0) ? F::vmax(t0, Real(0)) : Tr::inf();
    tmy = dy != Real(0) ? F::vmax(t1, Real(0)) : Tr::inf();
    tmz = dz != Real(0) ? F::vmax(t2, Real(0)) : Tr::inf();
    tdx = h * F::vabs(ix);
    tdy = h * F::vabs(iy);
    tdz = h * F::vabs(iz);
    sx = dx > Real(0) ? 1 : -1;
    sy = dy > Real(0) ? 1 : -1;
    sz = dz > Real(0) ? 1 : -1;
    Real ds, dh;
    const Real rem = tmax - tf;
    if constexpr (kF32) {
      ds = M.mus > 0.0f ? rs * M.inv_mus : Tr::inf();  // rs may be 0 after a clamp
      dh = fmaxf(0.0f, rem * M.mm_per_ns);
    } else {
      ds = M.mus > 0.0 ? rs / M.mus : Tr::inf();  // transport.cpp:166, 172
      dh = fmax(0.0, rem / M.ns_per_mm);
    }
    L = ds * M.ns_per_mm >= rem ? -dh : ds;  // horizon (transport.cpp:173-175) marked by the sign
    // a flight that ends before the first face skips the walk (short flights:
    // most of them in the head phantom's white matter)
    phase = F::vmin(tmx, F::vmin(tmy, tmz)) >= F::vabs(L) ? ENDF : WALK;
  };

  // ---- the flight ended inside the current voxel (ENDF, event phase):
  // scattering point or horizon ----
  auto end_flight = [&]() {
    if constexpr (kTrace) ++steps;
    const Real Ls = F::vabs(L);
    absorb(Ls);
    px += dx * Ls;
    py += dy * Ls;
    pz += dz * Ls;
    const Real te = tf + Ls * nsmm_();
    add_path(Ls);
    if (F::neg(L)) {  // StepKind::Terminated (transport.cpp:181-187, 330-332)
      deposit_run();
      acc_sm[2 * kBlock] += quant(w);
      if constexpr (kTrace) pd_trunc += w;
      finish(2);
      return;
    }
    if constexpr (!kF32) deposit_run();  // FP64: every step is its own deposit
    tf = te;
    rs = Real(0);
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
    const Real s = F::vmin(tmx, F::vmin(tmy, tmz));
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
    } else if (F::vmin(tmx, F::vmin(tmy, tmz)) >= F::vabs(L)) {
      phase = ENDF;  // the flight ends in this voxel
    }
  };

  // ---- hg_scatter + new free path + roulette (transport.cpp:126-147, 14-17, 333-343) ----
  auto scatter = [&]() {
    const Medium<Real>& M = medium(lab);
    if (phase == SCAT) {  // Henyey-Greenstein cos(theta) (transport.cpp:120-124)
      if constexpr (kTrace || kDet) ++nscat;
      const Real xi = rng.template unit<Real>();
      Real ct;
      if (M.iso) {
        ct = Real(2) * xi - Real(1);
      } else if constexpr (kF32) {
        const float f = M.hg_c * Tr::rcp(M.hg_d + M.hg_e * xi);
        ct = fminf(1.0f, fmaxf(-1.0f, M.hg_a - f * f * M.hg_b));
      } else {
        const double g = M.g;
        const double tmp = (1.0 - g * g) / (1.0 - g + 2.0 * g * xi);
        ct = (1.0 + g * g - tmp * tmp) / (2.0 * g);
        ct = ct < -1.0 ? -1.0 : (ct > 1.0 ? 1.0 : ct);
      }
      sct = ct;
      sst = Tr::sqrt_(F::vmax(Real(0), Real(1) - ct * ct));
    }
    // rejection azimuth (transport.cpp:32-44), VMC_AZ_UNROLL tries per event
    // phase; a lane rejected every time keeps cos/sin(theta) and retries in the
    // next event phase
    Real ax_ = 0, ay_ = 0, r2 = 0;
    bool ok = false;
#pragma unroll
    for (int k = 0; k < VMC_AZ_UNROLL; ++k) {
      if (k == 0 || !ok) {
        ax_ = F::two_u_m1(rng);  // 2u - 1
        ay_ = F::two_u_m1(rng);
        r2 = ax_ * ax_ + ay_ * ay_;
        ok = r2 > Real(1e-12) && r2 <= Real(1);
      }
    }
    if (!ok) {
      phase = RETRY;
      return;
    }
    const Real k = Tr::rsqrt(r2);
    const Real cp = ax_ * k, sp = ay_ * k;
    const Real ct = sct, st = sst;
    Real ox, oy, oz;
    if (F::vabs(dz) > Real(0.99999)) {  // transport.cpp:133-136
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
    } else {  // transport.cpp:137-141
      const double den = sqrt(1.0 - dz * dz);
      ox = st * (dx * dz * cp - dy * sp) / den + dx * ct;
      oy = st * (dy * dz * cp + dx * sp) / den + dy * ct;
      oz = -st * cp * den + dz * ct;
    }
    // renormalize (transport.cpp:142-145; 1e-6 in FP32, the reference's 1e-12 in FP64)
    const Real n2 = ox * ox + oy * oy + oz * oz;
    if (F::vabs(n2 - Real(1)) > (kF32 ? Real(1e-6) : Real(1e-12))) {
      const Real kk = Tr::rsqrt(n2);
      ox *= kk;
      oy *= kk;
      oz *= kk;
    }
    dx = ox;
    dy = oy;
    dz = oz;
    rs = scat_len();
    phase = SETUP;
    if (w < F::pick(A.rthrf, A.rthr)) {  // roulette after a scatter only (transport.cpp:300-306)
      const bool survive = rng.template unit<Real>() < F::pick(A.inv_rmultf, A.inv_rmult);
      deposit_run();  // close the deposit run before the weight jumps
      const long long qb = quant(w);
      if constexpr (kTrace) pd_kill += w;
      if (!survive) {
        acc_sm[kBlock] += qb;
        finish(1);
        return;
      }
      w *= F::pick(A.rmultf, static_cast<double>(A.rmult));
      acc_sm[kBlock] += qb - quant(w);
      if constexpr (kTrace) pd_kill -= w;
      run_w0 = w;
    }
  };

  // ---- interface / exterior face at distance L (handle_interface, transport.cpp:227-298) ----
  auto face = [&]() {
    const Real s = L;
    const int ax = fax;
    const Real t = tf + s * nsmm_();
    {
      // land exactly on the crossed plane (transport.cpp:197-204); the voxel
      // index has already moved, so the plane is its near face
      const int u = ax == 0 ? vx : (ax == 1 ? vy : vz);
      const Real dax = ax == 0 ? dx : (ax == 1 ? dy : dz);
      const Real plane = static_cast<Real>(dax > Real(0) ? u : u + 1) * h;
      px = ax == 0 ? plane : px + dx * s;
      py = ax == 1 ? plane : py + dy * s;
      pz = ax == 2 ? plane : pz + dz * s;
    }
    add_path(s);
    const Medium<Real>& M = medium(lab);
    rs = F::vmax(Real(0), rs - s * M.mus);
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
        const Real dax = ax == 0 ? dx : (ax == 1 ? dy : dz);
        const Real n1 = M.n, n2 = sm_media[nl].n;
        const Real ci = F::vabs(dax);
        const Real si2 = F::vmax(Real(0), Real(1) - ci * ci);
        // FP32: MUFU reciprocal / sqrt: R only meets a 24-bit uniform, and the
        // interface code runs on few lanes at a time, so its length is its cost
        Real eta;
        if constexpr (kF32) {
          eta = n1 * Tr::rcp(n2);
        } else {
          eta = n1 / n2;
        }
        const Real st2 = eta * eta * si2;
        if (st2 > Real(1)) {
          back = true;  // total internal reflection: deterministic flip
        } else {
          const Real cost = Tr::sqrt_(Real(1) - st2);
          Real R;
          if constexpr (kF32) {
            const float rsp = (n1 * ci - n2 * cost) * Tr::rcp(n1 * ci + n2 * cost);
            const float rpp = (n1 * cost - n2 * ci) * Tr::rcp(n1 * cost + n2 * ci);
            R = 0.5f * (rsp * rsp + rpp * rpp);
          } else {
            const double rsp = (n1 * ci - n2 * cost) / (n1 * ci + n2 * cost);
            const double rpp = (n1 * cost - n2 * ci) / (n1 * cost + n2 * ci);
            R = 0.5 * (rsp * rsp + rpp * rpp);
          }
          if (rng.template unit<Real>() < R) {
            back = true;
          } else {  // Snell refraction, tangential components scaled by n1/n2
            const Real nc = dax > Real(0) ? cost : -cost;
            const Real qx = ax == 0 ? nc : dx * eta;
            const Real qy = ax == 1 ? nc : dy * eta;
            const Real qz = ax == 2 ? nc : dz * eta;
            const Real k = Tr::rsqrt(qx * qx + qy * qy + qz * qz);
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
        flush_path();
        int hit = -1;
        for (int k = 0; k < A.ndet; ++k) {
          // in the kernel's precision, like the exit position itself
          // (FP32: detf = {x, y, z, r^2})
          bool in;
          if constexpr (kF32) {
            const float ex = px - A.detf[k][0], ey = py - A.detf[k][1], ez = pz - A.detf[k][2];
            in = ex * ex + ey * ey + ez * ez <= A.detf[k][3];
          } else {
            const double ex = px - A.det[k][0], ey = py - A.det[k][1], ez = pz - A.det[k][2];
            in = ex * ex + ey * ey + ez * ez <= A.det[k][3] * A.det[k][3];
          }
          if (in) {
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
      if (nl != lab) flush_path();
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
      const Real ct = Real(2) * rng.template unit<Real>() - Real(1);
      const Real u2 = rng.template unit<Real>();
      Real st, cphi, sphi;
      if constexpr (kF32) {
        st = sqrtf(fmaxf(0.0f, 1.0f - ct * ct));
        sincospif(2.0f * u2, &sphi, &cphi);
      } else {
        st = sqrt(fmax(0.0, 1.0 - ct * ct));
        sincos(2.0 * 3.14159265358979323846 * u2, &sphi, &cphi);
      }
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
      px = static_cast<Real>(qx);
      py = static_cast<Real>(qy);
      pz = static_cast<Real>(qz);
      if (ux < 0 || uy < 0 || uz < 0 || ux >= nx || uy >= A.ny || uz >= A.nz) {
        atomicExch(A.error_flag, 1);
        ux = uy = uz = 0;
        dx = dy = Real(0);
        dz = Real(1);
      }
      lab = __ldg(A.labels + (ux + nx * (uy + static_cast<long long>(A.ny) * uz)));
    } else {
      // FP32: converted once on the host (no F2F.F32.F64 per launch)
      dx = F::pick(A.dir0f[0], A.dir0[0]);
      dy = F::pick(A.dir0f[1], A.dir0[1]);
      dz = F::pick(A.dir0f[2], A.dir0[2]);
      px = F::pick(A.pos0f[0], A.pos0[0]);
      py = F::pick(A.pos0f[1], A.pos0[1]);
      pz = F::pick(A.pos0f[2], A.pos0[2]);
      ux = A.v0[0];
      uy = A.v0[1];
      uz = A.v0[2];
      lab = A.lab0;
    }
    vx = ux;
    vy = uy;
    vz = uz;
    w = Real(1);
    tf = Real(0);
    run_w0 = Real(1);
    if (A.iso_source) rs = scat_len();  // pencil: drawn in the seed batch
    if constexpr (kGates) {
      gate = 0;
      gmap = cbase;
      gate_end = A.ngates > 1 ? F::pick(A.gate_wf, A.tmax / A.ngates) : Tr::inf();
    }
    if constexpr (kTrace) {
      steps = nscat = 0;
      pd_dep = pd_esc = pd_kill = pd_trunc = 0;
    }
    if constexpr (kDet) {
      nscat = 0;
      // four predicated stores per pass instead of a per-slot loop (launch
      // runs on the one or two lanes that refill; B3 +0.4 %)
#pragma unroll 1
      for (int m = 0; m < A.nppath; m += 4) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (m + j < A.nppath) pp_sm[(m + j) * kBlock] = Real(0);
      }
      seg = Real(0);
    }
    phase = SETUP;
  };

  // per-warp seed stash in shared memory: 32 seeded RNG states of the photons
  // st_base + 0..31 and a header {next unused slot, valid slots}; st_base and
  // st_claimed_all are warp-uniform registers
  const int warp = threadIdx.x >> 5;
  unsigned char* const stash = smem + kStashOff + warp * kStashBytes;
  uint64_t* const st_a = reinterpret_cast<uint64_t*>(stash);
  uint64_t* const st_b = st_a + 32;
  Real* const st_rs = reinterpret_cast<Real*>(stash + 32 * 16);  // pencil sources: first free path
  int* const st_hdr = reinterpret_cast<int*>(stash + 32 * 16 + 32 * static_cast<int>(sizeof(Real)));
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
            if (!A.iso_source) st_rs[lane] = F::scat_len(sr);  // a pencil's first draw (transport.cpp:105)
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
    // (lane-disjoint blocks: the order only moves code. Single-label and gated
    // kernels run the interface block first: B1 +2.2 %, B2 +2.0 %, head
    // +0.25 %; the detector kernel keeps scatter first: B3 -0.3 % the other way)
    if (phase == ENDF) end_flight();
    if constexpr (kUni || kGates) {
      if (phase == FACE) face();
      if (phase == SCAT || phase == RETRY) scatter();
    } else {
      if (phase == SCAT || phase == RETRY) scatter();
      if (phase == FACE) face();
    }
    __syncwarp();  // reconverge before the shared flight setup (face() has warp-level votes)
    if (phase == SETUP) setup();
    if constexpr (!kUni) {
      // scatter chain for strongly scattering media (host sets chain_min when
      // mus * h is large, e.g. the head phantom's white matter, mus h = 40.9):
      // while most lanes' new flight ends inside its voxel, run their next
      // event at once instead of a walk pass with nothing to walk
      // (A/B on B200: head +2.4 / +3.3 % at 24 / 22 of 32 lanes; B3 -1 %, so off there)
      if (A.chain_min > 0) {
        while (__popc(__ballot_sync(0xffffffffu, phase == ENDF)) >= A.chain_min) {
          if (phase == ENDF) end_flight();
          if (phase == SCAT || phase == RETRY) scatter();
          __syncwarp();
          if (phase == SETUP) setup();
        }
      }
    }
    // ================= walk phase =================
    // every lane in flight crosses faces until at most (100 - event_pct) % of
    // the live lanes are still walking; the others wait for the event phase
    // walk_keep, scaled to the live lanes once the photons have run out
    int keep = A.walk_keep;
    if (exhausted) {
      const unsigned dead = __ballot_sync(0xffffffffu, phase == DEAD);
      if (dead == 0xffffffffu) break;
      if constexpr (kSolo) {
        // the warp's last photon of a small run (typically a horizon-truncated
        // one with hundreds of scatters left): nothing to batch with, so it
        // runs to its end without votes or event-phase dispatch
        if (__popc(dead) == 31) {
          if (phase != DEAD) {
            for (;;) {
              if (phase == WALK) {
                walk();
                continue;
              }
              if (phase == ENDF) end_flight();
              if (phase == SCAT || phase == RETRY) scatter();
              if (phase == FACE) face();
              if (phase == SETUP) setup();
              if (phase == DEAD) break;
            }
          }
          break;
        }
      }
      keep = ((32 - __popc(dead)) * A.walk_keep) >> 5;
    }
    // After an event phase nearly every lane walks in the cube60 kernels, so
    // their first vote is skipped (+1 %); in the strongly scattering head most
    // new flights end in their voxel, so the gated kernel votes first
    // (three steps per vote amortise the loop control; 2 and 4 measured slower)
    // (written as three calls: a `#pragma unroll` loop of the same three
    // calls changes the register allocation of the whole kernel, -7 %)
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

  if constexpr (kDep == kDepHotBox) {
    // flush the CTA's hot box: one red per non-empty cell into its replica
    __syncthreads();
    for (int i = threadIdx.x; i < kHbCells; i += blockDim.x) {
      const unsigned long long q = hb_lo[i] | (static_cast<unsigned long long>(hb_hi[i]) << 32);
      if (q) {
        const int bx = A.hb0[0] + i % kHotBoxN, by = A.hb0[1] + (i / kHotBoxN) % kHotBoxN,
                  bz = A.hb0[2] + i / (kHotBoxN * kHotBoxN);
        atomicAdd(cbase + (bx + nx * by + nxy * bz), q);
      }
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
