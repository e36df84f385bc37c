// transport_pool.cuh — K1 v2, the FP32 product kernel: a per-warp photon pool.
//
// Same physics and RNG consumption as the reference's run_photon
// (proj/core/src/transport.cpp:310-358; see transport.cuh for the v1 kernel
// and the FP64 parity instantiation). What changes is the SIMT schedule.
//
// Each lane owns K photon slots in shared memory (structure-of-arrays, 16-byte
// groups, conflict-free). Every warp iteration runs ONE event type for all
// lanes that have a photon in that state:
//   LAUNCH   claim indices (one atomicAdd per warp) and start photons in empty slots
//   STEP     one advance(): DDA, Beer-Lambert, deposit run bookkeeping, face
//            landing / interface / exit / horizon (transport.cpp:161-298)
//   SCATTER  hg_scatter + new free path + roulette (transport.cpp:126-147, 300-306)
// With K photons per lane almost every lane has one photon ready for the chosen
// event, so the two big code paths (step, scatter) no longer share warp issue
// slots with each other. Photons are independent: the interleaving never changes
// any photon's arithmetic or its RNG draw order.
#pragma once

#include "transport.cuh"

namespace vmc {

// slot groups (float4 / uint4 per slot)
enum PoolGroup : int {
  kGP = 0,  // px, py, pz, w
  kGD,      // dx, dy, dz, t
  kGI,      // ix, iy, iz, rs
  kGC,      // cell, lab | gate << 8, run_w0 (bits), nscat
  kGR,      // rng a.lo, a.hi, b.lo, b.hi
  kGV,      // vx, vy, vz, photon offset (idx - first)
  kGBase    // number of always-present groups
};
constexpr int kGPath = kGBase;  // + 2 groups of path lengths (detector mode)
constexpr int kGTrace = kGBase; // + trace groups (after path groups when both)

template <bool kDet, bool kTrace>
struct PoolLayout {
  static constexpr int kPath = kDet ? 2 : 0;        // 8 floats of per-label path length
  static constexpr int kTr = kTrace ? 2 : 0;        // draws/steps/flags + pd_dep, pd_kill (double)
  static constexpr int kGroups = kGBase + kPath + kTr;
  static constexpr int kPathBase = kGBase;
  static constexpr int kTrBase = kGBase + kPath;
};

constexpr int kPoolK = 2;  // photon slots per lane

template <bool kGates, bool kDet, bool kTrace>
__device__ __forceinline__ void pool_body(const KernelArgs& A, unsigned char* smem) {
  using L = PoolLayout<kDet, kTrace>;
  constexpr int K = kPoolK;
  constexpr int S = 32 * K;  // slots per warp
  constexpr unsigned FULL = 0xffffffffu;

  // ---- shared memory: media table, then per-warp slot arrays -------------
  Medium<float>* sm_media = reinterpret_cast<Medium<float>*>(smem);
  const int media_bytes = static_cast<int>(sizeof(Medium<float>)) * A.nmedia;
  float4* pool_base = reinterpret_cast<float4*>(smem + ((media_bytes + 15) & ~15));
  {
    const Medium<float>* gm = static_cast<const Medium<float>*>(A.media);
    const int nwords = static_cast<int>(sizeof(Medium<float>) / 4) * A.nmedia;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x)
      reinterpret_cast<int*>(sm_media)[i] = reinterpret_cast<const int*>(gm)[i];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const unsigned lanemask_lt = (1u << lane) - 1u;
  float4* pool = pool_base + static_cast<size_t>(warp) * L::kGroups * S;
  auto grp = [&](int g, int slot) -> float4* { return pool + g * S + slot; };
  auto grpu = [&](int g, int slot) -> uint4* { return reinterpret_cast<uint4*>(pool + g * S + slot); };

  const int nx = A.nx, ny = A.ny, nz = A.nz;
  const int nxy = static_cast<int>(A.nxy);
  const float h = static_cast<float>(A.h);
  const float tmax = static_cast<float>(A.tmax);
  const float rthr = static_cast<float>(A.rthr);
  const float rmult = static_cast<float>(A.rmult);
  const float inv_rmult = static_cast<float>(A.inv_rmult);
  const float inv_gate_w = static_cast<float>(A.inv_gate_w);
  const float qscale = static_cast<float>(A.qscale);
  const float kInf = __int_as_float(0x7f800000);

  long long acc_dep = 0, acc_esc = 0, acc_kill = 0, acc_trunc = 0;
  unsigned slot_state = 0;  // 2 bits per slot k: 0 empty, 1 step, 2 scatter
  bool exhausted = false;

  auto rcp = [](float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
  };
  auto fsqrt = [](float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
  };
  auto quant = [&](float x) -> long long { return __float2ll_rn(x * qscale); };
  auto deposit = [&](int c, int gt, long long q) {
    if (q != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(A.cells) + (static_cast<long long>(c) + A.nvox * gt),
                static_cast<unsigned long long>(q));
  };
  auto gate_of = [&](float tt) -> int {
    if constexpr (kGates) {
      const int g = static_cast<int>(tt * inv_gate_w);
      return g < A.ngates - 1 ? g : A.ngates - 1;
    } else {
      return 0;
    }
  };
  auto set_state = [&](int k, unsigned v) { slot_state = (slot_state & ~(3u << (2 * k))) | (v << (2 * k)); };

  for (;;) {
    // ---- per-lane availability, warp-wide phase choice -----------------
    int k_empty = -1, k_step = -1, k_scat = -1;
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
      const unsigned sk = (slot_state >> (2 * k)) & 3u;
      if (sk == 0u) k_empty = k;
      if (sk == 1u) k_step = k;
      if (sk == 2u) k_scat = k;
    }
    const unsigned m_empty = __ballot_sync(FULL, k_empty >= 0);
    const unsigned m_step = __ballot_sync(FULL, k_step >= 0);
    const unsigned m_scat = __ballot_sync(FULL, k_scat >= 0);
    const int n_step = __popc(m_step), n_scat = __popc(m_scat);

    if (!exhausted && m_empty && (__popc(m_empty) >= A.refill_min || (m_step | m_scat) == 0u)) {
      // ================= LAUNCH (transport.cpp:83-106) =================
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(A.claim, static_cast<unsigned long long>(__popc(m_empty)));
      base = __shfl_sync(FULL, base, 0);
      if (base + __popc(m_empty) >= A.count) exhausted = true;
      if (k_empty >= 0) {
        const unsigned long long my = base + __popc(m_empty & lanemask_lt);
        if (my < A.count) {
          const int slot = k_empty * 32 + lane;
          const uint64_t idx = A.first + my;
          Xs128p<kTrace> rng;
          rng.seed(A.seed, idx);
          float ux, uy, uz, px, py, pz;
          int vx, vy, vz, lab;
          if (A.iso_source) {
            const float ct = 2.0f * rng.template unit<float>() - 1.0f;
            const float u2 = rng.template unit<float>();
            float sphi, cphi;
            const float st = fsqrt(fmaxf(0.0f, 1.0f - ct * ct));
            sincospif(2.0f * u2, &sphi, &cphi);
            ux = st * cphi;
            uy = st * sphi;
            uz = ct;
            const double qx = A.src_pos[0] + static_cast<double>(ux) * 1e-6;
            const double qy = A.src_pos[1] + static_cast<double>(uy) * 1e-6;
            const double qz = A.src_pos[2] + static_cast<double>(uz) * 1e-6;
            vx = static_cast<int>(floor(qx / A.h));
            vy = static_cast<int>(floor(qy / A.h));
            vz = static_cast<int>(floor(qz / A.h));
            px = static_cast<float>(qx);
            py = static_cast<float>(qy);
            pz = static_cast<float>(qz);
            if (vx < 0 || vy < 0 || vz < 0 || vx >= nx || vy >= ny || vz >= nz) {
              atomicExch(A.error_flag, 1);
              vx = vy = vz = 0;
              ux = uy = 0.0f;
              uz = 1.0f;
            }
            lab = __ldg(A.labels + (vx + nx * (vy + ny * vz)));
          } else {
            ux = static_cast<float>(A.dir0[0]);
            uy = static_cast<float>(A.dir0[1]);
            uz = static_cast<float>(A.dir0[2]);
            px = static_cast<float>(A.pos0[0]);
            py = static_cast<float>(A.pos0[1]);
            pz = static_cast<float>(A.pos0[2]);
            vx = A.v0[0];
            vy = A.v0[1];
            vz = A.v0[2];
            lab = A.lab0;
          }
          const float u = rng.template unit<float>();
          const float rs = -__logf(u > 0.0f ? u : 0x1p-25f);
          *grp(kGP, slot) = make_float4(px, py, pz, 1.0f);
          *grp(kGD, slot) = make_float4(ux, uy, uz, 0.0f);
          *grp(kGI, slot) = make_float4(ux != 0.0f ? rcp(ux) : kInf, uy != 0.0f ? rcp(uy) : kInf,
                                        uz != 0.0f ? rcp(uz) : kInf, rs);
          *grpu(kGC, slot) = make_uint4(static_cast<unsigned>(vx + nx * (vy + ny * vz)), static_cast<unsigned>(lab),
                                        __float_as_uint(1.0f), 0u);
          *grpu(kGR, slot) = make_uint4(static_cast<unsigned>(rng.a), static_cast<unsigned>(rng.a >> 32),
                                        static_cast<unsigned>(rng.b), static_cast<unsigned>(rng.b >> 32));
          *grpu(kGV, slot) = make_uint4(static_cast<unsigned>(vx), static_cast<unsigned>(vy),
                                        static_cast<unsigned>(vz), static_cast<unsigned>(my));
          if constexpr (kDet) {
            *grp(L::kPathBase, slot) = make_float4(0.f, 0.f, 0.f, 0.f);
            *grp(L::kPathBase + 1, slot) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          if constexpr (kTrace) {
            *grpu(L::kTrBase, slot) = make_uint4(rng.draws, 0u, 0u, 0u);
            *grpu(L::kTrBase + 1, slot) = make_uint4(0u, 0u, 0u, 0u);
          }
          set_state(k_empty, 1u);
        }
      }
      continue;
    }
    if ((m_step | m_scat) == 0u) {
      if (exhausted) break;
      continue;
    }

    if (n_scat > 0 && n_scat * 100 >= n_step * A.scatter_pct) {
      // ================= SCATTER (transport.cpp:126-147, 14-17, 300-306) =================
      if (k_scat >= 0) {
        const int slot = k_scat * 32 + lane;
        float4 gd = *grp(kGD, slot);
        float4 gi = *grp(kGI, slot);
        uint4 gc = *grpu(kGC, slot);
        const uint4 gr = *grpu(kGR, slot);
        Xs128p<kTrace> rng;
        rng.a = (static_cast<uint64_t>(gr.y) << 32) | gr.x;
        rng.b = (static_cast<uint64_t>(gr.w) << 32) | gr.z;
        if constexpr (kTrace) rng.draws = grpu(L::kTrBase, slot)->x;
        const int lab = static_cast<int>(gc.y & 0xffu);
        const Medium<float>& M = sm_media[lab];
        float dx = gd.x, dy = gd.y, dz = gd.z;
        // Henyey-Greenstein cos(theta) (transport.cpp:120-124)
        const float xi = rng.template unit<float>();
        float ct;
        if (M.iso) {
          ct = 2.0f * xi - 1.0f;
        } else {
          const float f = __fdividef(M.hg_c, M.hg_d + M.hg_e * xi);
          ct = fminf(1.0f, fmaxf(-1.0f, M.hg_a - f * f * M.hg_b));
        }
        const float st = fsqrt(fmaxf(0.0f, 1.0f - ct * ct));
        float cp, sp;
        for (;;) {  // rejection azimuth (transport.cpp:32-44)
          const float ax = 2.0f * rng.template unit<float>() - 1.0f;
          const float ay = 2.0f * rng.template unit<float>() - 1.0f;
          const float r2 = ax * ax + ay * ay;
          if (r2 > 1e-12f && r2 <= 1.0f) {
            const float k = rsqrtf(r2);
            cp = ax * k;
            sp = ay * k;
            break;
          }
        }
        float ox, oy, oz;
        if (fabsf(dz) > 0.99999f) {
          ox = st * cp;
          oy = st * sp;
          oz = dz > 0.0f ? ct : -ct;
        } else {
          const float one_m = 1.0f - dz * dz;
          const float rden = rsqrtf(one_m);
          const float sr = st * rden;
          ox = sr * (dx * dz * cp - dy * sp) + dx * ct;
          oy = sr * (dy * dz * cp + dx * sp) + dy * ct;
          oz = -st * cp * (one_m * rden) + dz * ct;
        }
        const float n2 = ox * ox + oy * oy + oz * oz;
        if (fabsf(n2 - 1.0f) > 1e-6f) {
          const float k = rsqrtf(n2);
          ox *= k;
          oy *= k;
          oz *= k;
        }
        const float u = rng.template unit<float>();
        const float rs = -__logf(u > 0.0f ? u : 0x1p-25f);
        gd.x = ox;
        gd.y = oy;
        gd.z = oz;
        gi = make_float4(ox != 0.0f ? rcp(ox) : kInf, oy != 0.0f ? rcp(oy) : kInf, oz != 0.0f ? rcp(oz) : kInf, rs);
        unsigned next = 1u;
        if constexpr (kDet) gc.w += 1u;  // scatter count for detector records
        // roulette after a scatter (transport.cpp:333-343, 300-306)
        float4 gp = *grp(kGP, slot);
        const float w = gp.w;
        if (w < rthr) {
          const bool survive = rng.template unit<float>() < inv_rmult;
          const int cell = static_cast<int>(gc.x);
          const int gate = static_cast<int>(gc.y >> 8);
          const long long q = quant(__uint_as_float(gc.z) - w);  // close the deposit run
          deposit(cell, gate, q);
          acc_dep += q;
          if (!survive) {
            acc_kill += quant(w);
            next = 0u;
            if constexpr (kTrace) {
              uint4 t0 = *grpu(L::kTrBase, slot);
              const uint4 t1 = *grpu(L::kTrBase + 1, slot);
              vmc_photon_trace tr;
              tr.draws = rng.draws;
              tr.steps = t0.y;
              tr.scatters = t0.z + 1u;
              tr.flags = 2u;
              tr.deposited = __hiloint2double(static_cast<int>(t1.y), static_cast<int>(t1.x));
              tr.escaped = 0.0;
              tr.killed = __hiloint2double(static_cast<int>(t1.w), static_cast<int>(t1.z)) + w;
              tr.truncated = 0.0;
              A.trace[grpu(kGV, slot)->w] = tr;
            }
          } else {
            const float wb = w * rmult;
            acc_kill += quant(w) - quant(wb);
            gp.w = wb;
            gc.z = __float_as_uint(wb);
            *grp(kGP, slot) = gp;
            if constexpr (kTrace) {
              uint4 t1 = *grpu(L::kTrBase + 1, slot);
              const double k0 = __hiloint2double(static_cast<int>(t1.w), static_cast<int>(t1.z)) + (w - wb);
              t1.z = static_cast<unsigned>(__double2loint(k0));
              t1.w = static_cast<unsigned>(__double2hiint(k0));
              *grpu(L::kTrBase + 1, slot) = t1;
            }
          }
        }
        if (next) {
          *grp(kGD, slot) = gd;
          *grp(kGI, slot) = gi;
          *grpu(kGC, slot) = gc;
          *grpu(kGR, slot) = make_uint4(static_cast<unsigned>(rng.a), static_cast<unsigned>(rng.a >> 32),
                                        static_cast<unsigned>(rng.b), static_cast<unsigned>(rng.b >> 32));
          if constexpr (kTrace) {
            uint4* t0 = grpu(L::kTrBase, slot);
            t0->x = rng.draws;
            t0->z += 1u;
          }
        }
        set_state(k_scat, next);
      }
      continue;
    }

    // ================= STEP: one advance() (transport.cpp:161-225) =================
    if (k_step < 0) continue;
    const int slot = k_step * 32 + lane;
    float4 gp = *grp(kGP, slot);
    float4 gd = *grp(kGD, slot);
    float4 gi = *grp(kGI, slot);
    uint4 gc = *grpu(kGC, slot);
    uint4 gv = *grpu(kGV, slot);
    int vx = static_cast<int>(gv.x), vy = static_cast<int>(gv.y), vz = static_cast<int>(gv.z);
    int cell = static_cast<int>(gc.x);
    int lab = static_cast<int>(gc.y & 0xffu);
    int gate = static_cast<int>(gc.y >> 8);
    float run_w0 = __uint_as_float(gc.z);
    float px = gp.x, py = gp.y, pz = gp.z, w = gp.w;
    const float dx = gd.x, dy = gd.y, dz = gd.z;
    float t = gd.w, rs = gi.w;
    const Medium<float>& M = sm_media[lab];
    // boundary_distance (transport.cpp:49-73)
    const float t0_ = (static_cast<float>(vx + (dx > 0.0f ? 1 : 0)) * h - px) * gi.x;
    const float t1_ = (static_cast<float>(vy + (dy > 0.0f ? 1 : 0)) * h - py) * gi.y;
    const float t2_ = (static_cast<float>(vz + (dz > 0.0f ? 1 : 0)) * h - pz) * gi.z;
    const float tb0 = dx != 0.0f ? fmaxf(t0_, 0.0f) : kInf;
    const float tb1 = dy != 0.0f ? fmaxf(t1_, 0.0f) : kInf;
    const float tb2 = dz != 0.0f ? fmaxf(t2_, 0.0f) : kInf;
    int axis = 0;
    float d_b = tb0;
    if (tb1 < d_b) {
      d_b = tb1;
      axis = 1;
    }
    if (tb2 < d_b) {
      d_b = tb2;
      axis = 2;
    }
    const float d_s = M.mus > 0.0f ? rs * M.inv_mus : kInf;
    const float ns = M.ns_per_mm;
    const float remaining = tmax - t;
    float d = d_b < d_s ? d_b : d_s;
    const bool horizon = d * ns >= remaining;
    if (horizon) d = fmaxf(0.0f, remaining * M.mm_per_ns);
    float w1;
    {  // exp_neg (transport.cpp:22-27), branch-free
      const float x = M.mua * d;
      const float taylor = 1.0f - x * (1.0f - x * (0.5f - x * (1.0f / 6.0f - x * (1.0f / 24.0f))));
      w1 = w * (x < 0.01f ? taylor : __expf(-x));
    }
    if constexpr (kTrace) {
      uint4 t1 = *grpu(L::kTrBase + 1, slot);
      const double pd = __hiloint2double(static_cast<int>(t1.y), static_cast<int>(t1.x)) + static_cast<double>(w - w1);
      t1.x = static_cast<unsigned>(__double2loint(pd));
      t1.y = static_cast<unsigned>(__double2hiint(pd));
      *grpu(L::kTrBase + 1, slot) = t1;
      grpu(L::kTrBase, slot)->y += 1u;
    }
    w = w1;
    t += d * ns;
    if constexpr (kDet) {
      float4 p0 = *grp(L::kPathBase, slot), p1 = *grp(L::kPathBase + 1, slot);
      p0.x += lab == 1 ? d : 0.f;
      p0.y += lab == 2 ? d : 0.f;
      p0.z += lab == 3 ? d : 0.f;
      p0.w += lab == 4 ? d : 0.f;
      p1.x += lab == 5 ? d : 0.f;
      p1.y += lab == 6 ? d : 0.f;
      p1.z += lab == 7 ? d : 0.f;
      p1.w += lab == 8 ? d : 0.f;
      *grp(L::kPathBase, slot) = p0;
      *grp(L::kPathBase + 1, slot) = p1;
    }

    unsigned next = 1u;
    int term = -1;  // 0 escaped, 2 truncated
    if (horizon) {  // StepKind::Terminated
      const long long q = quant(run_w0 - w);
      deposit(cell, gate, q);
      acc_dep += q;
      acc_trunc += quant(w);
      next = 0u;
      term = 2;
    } else if (d_s <= d_b) {  // StepKind::Scattered: move to the scattering point
      px += dx * d;
      py += dy * d;
      pz += dz * d;
      if constexpr (kGates) {
        const int ng = gate_of(t);
        if (ng != gate) {
          const long long q = quant(run_w0 - w);
          deposit(cell, gate, q);
          acc_dep += q;
          run_w0 = w;
          gate = ng;
        }
      }
      next = 2u;
    } else {
      // land exactly on the face (transport.cpp:197-211)
      rs = fmaxf(0.0f, rs - d * M.mus);
      const float dax = axis == 0 ? dx : (axis == 1 ? dy : dz);
      const int stp = dax > 0.0f ? 1 : -1;
      const int vax = axis == 0 ? vx : (axis == 1 ? vy : vz);
      const float plane = static_cast<float>(vax + (stp > 0 ? 1 : 0)) * h;
      px = axis == 0 ? plane : px + dx * d;
      py = axis == 1 ? plane : py + dy * d;
      pz = axis == 2 ? plane : pz + dz * d;
      const int nvx = vx + (axis == 0 ? stp : 0);
      const int nvy = vy + (axis == 1 ? stp : 0);
      const int nvz = vz + (axis == 2 ? stp : 0);
      const int stride = axis == 0 ? 1 : (axis == 1 ? nx : nxy);
      const int ncell = stp > 0 ? cell + stride : cell - stride;
      const bool exterior = static_cast<unsigned>(nvx) >= static_cast<unsigned>(nx) ||
                            static_cast<unsigned>(nvy) >= static_cast<unsigned>(ny) ||
                            static_cast<unsigned>(nvz) >= static_cast<unsigned>(nz);
      const int nlab = exterior ? 0 : static_cast<int>(__ldg(A.labels + ncell));
      const int c1 = M.nclass, c2 = sm_media[nlab].nclass;
      bool move = false, exited = false;
      if (!exterior && c1 == c2) {
        move = true;  // same refractive index (transport.cpp:218-223)
      } else if (exterior && !A.reflect) {
        exited = true;  // TerminateAtBoundary (transport.cpp:234-237)
      } else if (c1 == c2) {
        exited = exterior;  // identity interface (transport.cpp:242-252)
        move = !exterior;
      } else {
        // Fresnel / TIR (transport.cpp:254-297): one draw unless TIR
        const float n1 = M.n, n2 = sm_media[nlab].n;
        const float ci = fabsf(dax);
        const float si2 = fmaxf(0.0f, 1.0f - ci * ci);
        const float eta = n1 / n2;
        const float st2 = eta * eta * si2;
        float ndx = dx, ndy = dy, ndz = dz;
        bool flip = true;
        if (st2 <= 1.0f) {
          const uint4 gr = *grpu(kGR, slot);
          Xs128p<kTrace> rng;
          rng.a = (static_cast<uint64_t>(gr.y) << 32) | gr.x;
          rng.b = (static_cast<uint64_t>(gr.w) << 32) | gr.z;
          if constexpr (kTrace) rng.draws = grpu(L::kTrBase, slot)->x;
          const float cost = sqrtf(1.0f - st2);
          const float rsp = (n1 * ci - n2 * cost) / (n1 * ci + n2 * cost);
          const float rpp = (n1 * cost - n2 * ci) / (n1 * cost + n2 * ci);
          const float R = 0.5f * (rsp * rsp + rpp * rpp);
          flip = rng.template unit<float>() < R;
          *grpu(kGR, slot) = make_uint4(static_cast<unsigned>(rng.a), static_cast<unsigned>(rng.a >> 32),
                                        static_cast<unsigned>(rng.b), static_cast<unsigned>(rng.b >> 32));
          if constexpr (kTrace) grpu(L::kTrBase, slot)->x = rng.draws;
          if (!flip) {  // Snell refraction: tangential x eta, normal +-cos_t, renormalize
            ndx = axis == 0 ? (dax > 0.0f ? cost : -cost) : dx * eta;
            ndy = axis == 1 ? (dax > 0.0f ? cost : -cost) : dy * eta;
            ndz = axis == 2 ? (dax > 0.0f ? cost : -cost) : dz * eta;
            const float k = rsqrtf(ndx * ndx + ndy * ndy + ndz * ndz);
            ndx *= k;
            ndy *= k;
            ndz *= k;
            exited = exterior;
            move = !exterior;
          }
        }
        if (flip) {  // specular reflection or TIR: negate the normal component
          if (axis == 0) ndx = -dx;
          if (axis == 1) ndy = -dy;
          if (axis == 2) ndz = -dz;
        }
        gd.x = ndx;
        gd.y = ndy;
        gd.z = ndz;
        *grp(kGD, slot) = gd;  // .w (t) rewritten below
        gi.x = ndx != 0.0f ? rcp(ndx) : kInf;
        gi.y = ndy != 0.0f ? rcp(ndy) : kInf;
        gi.z = ndz != 0.0f ? rcp(ndz) : kInf;
        *grp(kGI, slot) = gi;
      }
      if (exited) {  // ExitedDomain: escaped += w (transport.cpp:348-350)
        const long long q = quant(run_w0 - w);
        deposit(cell, gate, q);
        acc_dep += q;
        acc_esc += quant(w);
        next = 0u;
        term = 0;
        if constexpr (kDet) {
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
          if (hit >= 0) {
            // records are rare: one atomic per record keeps the code simple
            const unsigned long long s = atomicAdd(A.det_count, 1ull);
            if (s < A.det_cap) {
              unsigned char* rec = A.det_out + s * static_cast<unsigned long long>(A.rec_stride);
              vmc_det_record_head hd;
              hd.photon_index = A.first + gv.w;
              hd.det_id = static_cast<uint32_t>(hit);
              hd.nscat = gc.w;
              hd.w_exit = w;
              hd.t_exit_ns = t;
              *reinterpret_cast<vmc_det_record_head*>(rec) = hd;
              const float4 p0 = *grp(L::kPathBase, slot), p1 = *grp(L::kPathBase + 1, slot);
              const float pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
              float* dst = reinterpret_cast<float*>(rec + sizeof(vmc_det_record_head));
#pragma unroll
              for (int m = 0; m < kMaxDetMedia; ++m)
                if (m < A.nppath) dst[m] = pp[m];
            }
            if constexpr (kTrace) grpu(L::kTrBase, slot)->w = 8u;
          }
        }
      } else if (move) {
        const int ng = gate_of(t);
        const long long q = quant(run_w0 - w);  // a new voxel closes the deposit run
        deposit(cell, gate, q);
        acc_dep += q;
        run_w0 = w;
        gate = ng;
        vx = nvx;
        vy = nvy;
        vz = nvz;
        cell = ncell;
        lab = nlab;
      } else if constexpr (kGates) {
        const int ng = gate_of(t);
        if (ng != gate) {
          const long long q = quant(run_w0 - w);
          deposit(cell, gate, q);
          acc_dep += q;
          run_w0 = w;
          gate = ng;
        }
      }
    }
    if (next) {
      *grp(kGP, slot) = make_float4(px, py, pz, w);
      grp(kGD, slot)->w = t;
      grp(kGI, slot)->w = rs;
      *grpu(kGC, slot) = make_uint4(static_cast<unsigned>(cell), static_cast<unsigned>(lab) | (static_cast<unsigned>(gate) << 8),
                                    __float_as_uint(run_w0), gc.w);
      *grpu(kGV, slot) = make_uint4(static_cast<unsigned>(vx), static_cast<unsigned>(vy), static_cast<unsigned>(vz), gv.w);
    } else if constexpr (kTrace) {
      const uint4 t0 = *grpu(L::kTrBase, slot);
      const uint4 t1 = *grpu(L::kTrBase + 1, slot);
      vmc_photon_trace tr;
      tr.draws = t0.x;
      tr.steps = t0.y;
      tr.scatters = t0.z;
      tr.flags = (term == 0 ? 1u : 4u) | t0.w;
      tr.deposited = __hiloint2double(static_cast<int>(t1.y), static_cast<int>(t1.x));
      tr.escaped = term == 0 ? static_cast<double>(w) : 0.0;
      tr.killed = __hiloint2double(static_cast<int>(t1.w), static_cast<int>(t1.z));
      tr.truncated = term == 2 ? static_cast<double>(w) : 0.0;
      A.trace[gv.w] = tr;
    }
    set_state(k_step, next);
  }

  // ---- epilogue: dispositions (warp reduce) -------------------------------
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc_dep += __shfl_xor_sync(FULL, acc_dep, o);
    acc_esc += __shfl_xor_sync(FULL, acc_esc, o);
    acc_kill += __shfl_xor_sync(FULL, acc_kill, o);
    acc_trunc += __shfl_xor_sync(FULL, acc_trunc, o);
  }
  if (lane == 0) {
    unsigned long long* tot = reinterpret_cast<unsigned long long*>(A.totals);
    if (acc_dep) atomicAdd(tot + 0, static_cast<unsigned long long>(acc_dep));
    if (acc_esc) atomicAdd(tot + 1, static_cast<unsigned long long>(acc_esc));
    if (acc_kill) atomicAdd(tot + 2, static_cast<unsigned long long>(acc_kill));
    if (acc_trunc) atomicAdd(tot + 3, static_cast<unsigned long long>(acc_trunc));
  }
}

template <bool kDet, bool kTrace>
constexpr int pool_smem_per_warp() {
  return PoolLayout<kDet, kTrace>::kGroups * 32 * kPoolK * 16;
}

}  // namespace vmc
