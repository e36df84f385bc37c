/* oracle/voxmc_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the
 * product path; the B200 library neither links nor calls this file).
 *
 * Plain-C double-precision restatement of the reference hot path
 * (/root/reference/proj). Each function names the reference lines it follows.
 * Compiled with -ffp-contract=off; the reference is compiled with GCC's
 * default FMA contraction, so results agree to rounding, not bit for bit —
 * tests/test_oracle_ref.py pins this restatement against the compiled
 * reference (oracle/_ref) and against the golden vectors of SURVEY.md
 * Appendix A / proj/test_output.txt:25.
 *
 * Time gates and disk detectors have no reference implementation; their
 * semantics here are the ones fixed in DESIGN.md ("Oracle") and are shared with
 * oracle/ref_capi.cpp's ref_walk:
 *   gate of a deposit = clamp(floor(t_step_start / (tmax/ngates)), 0, ngates-1);
 *   a photon that exits the domain is recorded by the first detector k with
 *   |exit_pos - c_k| <= r_k, with its weight, time, scatter count and the
 *   per-label path length accumulated over its steps.
 */
#include "voxmc_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

const char* orc_last_error(void) { return g_err; }

/* ---- RNG: rng.cpp:5-19, rng.hpp:15-26 -------------------------------- */

uint64_t orc_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void orc_rng_seed(orc_rng* r, uint64_t seed, uint64_t stream_id) {
  const uint64_t z = seed ^ stream_id;
  r->lo = orc_mix64(z);
  r->hi = orc_mix64(z + 0x9E3779B97F4A7C15ULL);
  if (r->lo == 0 && r->hi == 0) r->hi = 0x6A09E667F3BCC909ULL;
}

uint64_t orc_rng_next(orc_rng* r) {
  uint64_t a = r->lo;
  const uint64_t b = r->hi;
  const uint64_t out = a + b;
  a ^= a << 23;
  r->lo = b;
  r->hi = a ^ b ^ (a >> 18) ^ (b >> 5);
  return out;
}

double orc_rng_unit(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

void orc_rng_kat(uint64_t seed, uint64_t stream_id, int n, uint64_t* out) {
  orc_rng r;
  orc_rng_seed(&r, seed, stream_id);
  for (int i = 0; i < n; ++i) out[i] = orc_rng_next(&r);
}

/* ---- fluence quantum: fluence.cpp:11-14 --------------------------------- */

double orc_quantum_for(uint64_t n) {
  uint64_t v = n | 1u;
  int width = 0;
  while (v) {
    ++width;
    v >>= 1;
  }
  return ldexp(1.0, -(62 - width));
}

/* ---- scalar physics: transport.cpp ------------------------------------- */

static const double kC = 299.792458; /* types.hpp:16 */
static const double kPi = 3.14159265358979323846;

static double scat_len(orc_rng* r) { /* transport.cpp:14-17 */
  const double u = orc_rng_unit(r);
  return -log(u > 0.0 ? u : DBL_TRUE_MIN);
}

static double exp_neg(double x) { /* transport.cpp:22-27 */
  if (x < 0.01) return 1.0 - x * (1.0 - x * (0.5 - x * (1.0 / 6.0 - x * (1.0 / 24.0))));
  return exp(-x);
}

static void azimuth(orc_rng* r, double* c, double* s) { /* transport.cpp:32-44 */
  for (;;) {
    const double ax = 2.0 * orc_rng_unit(r) - 1.0;
    const double ay = 2.0 * orc_rng_unit(r) - 1.0;
    const double rr = ax * ax + ay * ay;
    if (rr > 1e-12 && rr <= 1.0) {
      const double k = 1.0 / sqrt(rr);
      *c = ax * k;
      *s = ay * k;
      return;
    }
  }
}

double orc_hg_cos_theta(double g, double xi) { /* transport.cpp:120-124 */
  if (fabs(g) < 1e-6) return 2.0 * xi - 1.0;
  const double f = (1.0 - g * g) / (1.0 - g + 2.0 * g * xi);
  double ct = (1.0 + g * g - f * f) / (2.0 * g);
  if (ct < -1.0) ct = -1.0;
  if (ct > 1.0) ct = 1.0;
  return ct;
}

double orc_fresnel(double n1, double n2, double ci) { /* transport.cpp:149-159 */
  if (ci < 0.0) ci = 0.0;
  if (ci > 1.0) ci = 1.0;
  const double eta = n1 / n2;
  const double st2 = eta * eta * (1.0 - ci * ci);
  if (st2 > 1.0) return 1.0;
  const double ct = sqrt(1.0 - st2);
  const double rs = (n1 * ci - n2 * ct) / (n1 * ci + n2 * ct);
  const double rp = (n1 * ct - n2 * ci) / (n1 * ct + n2 * ci);
  return 0.5 * (rs * rs + rp * rp);
}

/* photon state, transport.hpp:16-27 */
typedef struct {
  double p[3], d[3], inv[3];
  double w, t, rs;
  int v[3];
  int label;
} photon_t;

static void set_dir(photon_t* ph, const double* d) { /* transport.cpp:77-81 */
  for (int k = 0; k < 3; ++k) {
    ph->d[k] = d[k];
    ph->inv[k] = d[k] != 0.0 ? 1.0 / d[k] : INFINITY;
  }
}

static void hg_rotate(photon_t* ph, double g, orc_rng* r) { /* transport.cpp:126-147 */
  const double ct = orc_hg_cos_theta(g, orc_rng_unit(r));
  const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
  double cp, sp;
  azimuth(r, &cp, &sp);
  const double* d = ph->d;
  double o[3];
  if (fabs(d[2]) > 0.99999) {
    o[0] = st * cp;
    o[1] = st * sp;
    o[2] = d[2] > 0.0 ? ct : -ct;
  } else {
    const double den = sqrt(1.0 - d[2] * d[2]);
    o[0] = st * (d[0] * d[2] * cp - d[1] * sp) / den + d[0] * ct;
    o[1] = st * (d[1] * d[2] * cp + d[0] * sp) / den + d[1] * ct;
    o[2] = -st * cp * den + d[2] * ct;
  }
  const double n2 = o[0] * o[0] + o[1] * o[1] + o[2] * o[2];
  if (fabs(n2 - 1.0) > 1e-12) {
    const double k = 1.0 / sqrt(n2);
    o[0] *= k;
    o[1] *= k;
    o[2] *= k;
  }
  set_dir(ph, o);
}

typedef struct {
  const vmc_scene* s;
  const vmc_config* c;
  int ngates;
  double gate_w;
  double inv_q;
  size_t nvox;
} ctx_t;

static int in_grid(const vmc_scene* s, const int* v) {
  return v[0] >= 0 && v[1] >= 0 && v[2] >= 0 && v[0] < s->nx && v[1] < s->ny && v[2] < s->nz;
}

static size_t lin(const vmc_scene* s, const int* v) {
  return (size_t)v[0] + (size_t)s->nx * ((size_t)v[1] + (size_t)s->ny * (size_t)v[2]);
}

static int launch(const ctx_t* cx, orc_rng* r, photon_t* ph) { /* transport.cpp:83-106 */
  const vmc_scene* s = cx->s;
  double d[3];
  if (s->isotropic) {
    const double ct = 2.0 * orc_rng_unit(r) - 1.0;
    const double phi = 2.0 * kPi * orc_rng_unit(r);
    const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
    d[0] = st * cos(phi);
    d[1] = st * sin(phi);
    d[2] = ct;
  } else {
    const double* sd = s->src_dir;
    const double k = 1.0 / sqrt(sd[0] * sd[0] + sd[1] * sd[1] + sd[2] * sd[2]);
    d[0] = sd[0] * k;
    d[1] = sd[1] * k;
    d[2] = sd[2] * k;
  }
  set_dir(ph, d);
  for (int k = 0; k < 3; ++k) {
    ph->p[k] = s->src_pos[k] + d[k] * 1e-6;
    ph->v[k] = (int)floor(ph->p[k] / s->voxel_mm); /* types.cpp:35-42 */
  }
  if (!in_grid(s, ph->v)) return -1;
  ph->label = s->labels[lin(s, ph->v)];
  ph->w = 1.0;
  ph->t = 0.0;
  ph->rs = scat_len(r);
  return 0;
}

typedef struct {
  double dep, esc, kill, trunc;
} disp_t;

typedef struct {
  uint64_t photon;
  uint32_t det, nscat;
  float w, t;
  float ppath[255];
} hit_t;

typedef struct {
  hit_t* v;
  size_t n, cap;
} hits_t;

/* One photon: run_photon (transport.cpp:310-358) with advance (161-225),
 * handle_interface (227-298) and roulette (300-306) inlined. */
static int walk_one(const ctx_t* cx, uint64_t idx, int64_t* cells, vmc_photon_trace* tr,
                    disp_t* acc, hits_t* hits) {
  const vmc_scene* s = cx->s;
  const vmc_config* c = cx->c;
  const double h = s->voxel_mm;
  const double* M = s->media;
  orc_rng r;
  orc_rng_seed(&r, c->master_seed, idx);
  photon_t ph;
  if (launch(cx, &r, &ph) != 0) return -1;
  disp_t dp = {0, 0, 0, 0};
  uint32_t steps = 0, nscat = 0, flags = 0;
  double path[256];
  if (hits) memset(path, 0, sizeof path);
  const double tmax = c->tmax_ns;

  for (;;) {
    const int lab = ph.label;
    const double mua = M[4 * lab], mus = M[4 * lab + 1], g = M[4 * lab + 2], n = M[4 * lab + 3];
    const size_t cell_at = lin(s, ph.v);
    const double t0 = ph.t;
    ++steps;
    /* boundary_distance, transport.cpp:49-73 */
    double tb[3];
    for (int k = 0; k < 3; ++k) {
      const double plane = (ph.v[k] + (ph.d[k] > 0.0 ? 1 : 0)) * h;
      const double tk = (plane - ph.p[k]) * ph.inv[k];
      tb[k] = ph.d[k] != 0.0 ? (tk > 0.0 ? tk : 0.0) : INFINITY;
    }
    int ax = 0;
    double db = tb[0];
    if (tb[1] < db) {
      db = tb[1];
      ax = 1;
    }
    if (tb[2] < db) {
      db = tb[2];
      ax = 2;
    }
    const double ds = mus > 0.0 ? ph.rs / mus : INFINITY;
    const double nspm = n * (1.0 / kC);
    const double left = tmax - ph.t;
    double d = ds < db ? ds : db;
    const int horizon = d * nspm >= left;
    if (horizon) d = fmax(0.0, left / nspm);
    const double w1 = ph.w * exp_neg(mua * d);
    const double dw = ph.w - w1;
    ph.w = w1;
    ph.t += d * nspm;
    if (hits && lab >= 1) path[lab - 1] += d;
    if (dw != 0.0) {
      if (cells) {
        int gate = (int)floor(t0 / cx->gate_w);
        if (gate < 0) gate = 0;
        if (gate > cx->ngates - 1) gate = cx->ngates - 1;
        cells[(size_t)gate * cx->nvox + cell_at] += (int64_t)llround(dw * cx->inv_q);
      }
      dp.dep += dw;
    }
    if (horizon) {
      for (int k = 0; k < 3; ++k) ph.p[k] += ph.d[k] * d;
      ph.t = tmax;
      dp.trunc += ph.w;
      flags |= 4u;
      break;
    }
    if (ds <= db) { /* scatter */
      for (int k = 0; k < 3; ++k) ph.p[k] += ph.d[k] * d;
      hg_rotate(&ph, g, &r);
      ph.rs = scat_len(&r);
      ++nscat;
      if (ph.w < c->roulette_threshold) {
        const double before = ph.w;
        if (orc_rng_unit(&r) < 1.0 / c->roulette_multiplier) {
          ph.w *= c->roulette_multiplier;
          dp.kill += before - ph.w;
        } else {
          dp.kill += before;
          flags |= 2u;
          break;
        }
      }
      continue;
    }
    /* land on the face (transport.cpp:197-211) */
    ph.rs = fmax(0.0, ph.rs - d * mus);
    const int step = ph.d[ax] > 0.0 ? 1 : -1;
    for (int k = 0; k < 3; ++k) ph.p[k] += ph.d[k] * d;
    ph.p[ax] = (ph.v[ax] + (step > 0 ? 1 : 0)) * h;
    int nv[3] = {ph.v[0], ph.v[1], ph.v[2]};
    nv[ax] += step;
    const int exterior = !in_grid(s, nv);
    const int nlab = exterior ? 0 : s->labels[lin(s, nv)];
    const double n2 = M[4 * nlab + 3];
    if (!exterior && n2 == n) { /* same index: inline update (218-223) */
      ph.v[0] = nv[0];
      ph.v[1] = nv[1];
      ph.v[2] = nv[2];
      ph.label = nlab;
      continue;
    }
    /* handle_interface (227-298) */
    int exited = 0;
    if (exterior && c->boundary_mode == VMC_BOUNDARY_TERMINATE) {
      exited = 1;
    } else if (n == n2) {
      exited = exterior;
    } else {
      const double ci = fabs(ph.d[ax]);
      const double si2 = fmax(0.0, 1.0 - ci * ci);
      const double eta = n / n2;
      const double st2 = eta * eta * si2;
      double nd[3] = {ph.d[0], ph.d[1], ph.d[2]};
      if (st2 > 1.0) { /* TIR */
        nd[ax] = -nd[ax];
        set_dir(&ph, nd);
        continue;
      }
      const double ct = sqrt(1.0 - st2);
      const double rs = (n * ci - n2 * ct) / (n * ci + n2 * ct);
      const double rp = (n * ct - n2 * ci) / (n * ct + n2 * ci);
      const double R = 0.5 * (rs * rs + rp * rp);
      if (orc_rng_unit(&r) < R) {
        nd[ax] = -nd[ax];
        set_dir(&ph, nd);
        continue;
      }
      for (int k = 0; k < 3; ++k)
        if (k != ax) nd[k] = ph.d[k] * eta;
      nd[ax] = ph.d[ax] > 0.0 ? ct : -ct;
      const double kk = 1.0 / sqrt(nd[0] * nd[0] + nd[1] * nd[1] + nd[2] * nd[2]);
      nd[0] *= kk;
      nd[1] *= kk;
      nd[2] *= kk;
      set_dir(&ph, nd);
      exited = exterior;
    }
    if (exited) {
      dp.esc += ph.w;
      flags |= 1u;
      if (hits) {
        for (int k = 0; k < c->ndet; ++k) {
          const double* D = c->det + 4 * k;
          const double dx = ph.p[0] - D[0], dy = ph.p[1] - D[1], dz = ph.p[2] - D[2];
          if (dx * dx + dy * dy + dz * dz <= D[3] * D[3]) {
            if (hits->n == hits->cap) {
              hits->cap = hits->cap ? 2 * hits->cap : 64;
              hits->v = (hit_t*)realloc(hits->v, hits->cap * sizeof(hit_t));
            }
            hit_t* hh = &hits->v[hits->n++];
            hh->photon = idx;
            hh->det = (uint32_t)k;
            hh->nscat = nscat;
            hh->w = (float)ph.w;
            hh->t = (float)ph.t;
            for (int m = 0; m + 1 < s->nmedia && m < 255; ++m) hh->ppath[m] = (float)path[m];
            flags |= 8u;
            break;
          }
        }
      }
      break;
    }
    ph.v[0] = nv[0];
    ph.v[1] = nv[1];
    ph.v[2] = nv[2];
    ph.label = nlab;
  }

  if (tr) {
    orc_rng probe;
    orc_rng_seed(&probe, c->master_seed, idx);
    uint32_t k = 0;
    while (!(probe.lo == r.lo && probe.hi == r.hi) && k < (1u << 26)) {
      orc_rng_next(&probe);
      ++k;
    }
    tr->draws = k;
    tr->steps = steps;
    tr->scatters = nscat;
    tr->flags = flags;
    tr->deposited = dp.dep;
    tr->escaped = dp.esc;
    tr->killed = dp.kill;
    tr->truncated = dp.trunc;
  }
  acc->dep += dp.dep;
  acc->esc += dp.esc;
  acc->kill += dp.kill;
  acc->trunc += dp.trunc;
  return 0;
}

/* The same photon walked in K1f's decomposition (csrc/flight.cuh), in double
 * precision: one setup per free flight (incremental-DDA face distances tm,
 * increments td, flight length L = min(remaining_scat / mus, horizon
 * distance)), faces walked from the flight start (tm += td, the face at s ends
 * the flight when the neighbour label differs or is exterior), and the
 * scatter / interface / horizon events of run_photon (transport.cpp:310-358)
 * between flights. In exact arithmetic this is the reference's walk; the test
 * (tests/test_oracle_ref.py) checks that in double precision it draws the same
 * RNG stream per photon as the compiled reference, i.e. that the flight
 * decomposition changes nothing but rounding. Traces only. */
static int walk_one_flight(const ctx_t* cx, uint64_t idx, vmc_photon_trace* tr, disp_t* acc) {
  const vmc_scene* s = cx->s;
  const vmc_config* c = cx->c;
  const double h = s->voxel_mm;
  const double* M = s->media;
  orc_rng r;
  orc_rng_seed(&r, c->master_seed, idx);
  photon_t ph;
  if (launch(cx, &r, &ph) != 0) return -1;
  disp_t dp = {0, 0, 0, 0};
  uint32_t steps = 0, nscat = 0, flags = 0;
  const double tmax = c->tmax_ns;
  for (;;) {
    /* ---- flight setup ---- */
    const int lab = ph.label;
    const double mua = M[4 * lab], mus = M[4 * lab + 1], g = M[4 * lab + 2], n = M[4 * lab + 3];
    const double nspm = n * (1.0 / kC);
    double tm[3], td[3];
    int sg[3];
    for (int k = 0; k < 3; ++k) {
      const double plane = (ph.v[k] + (ph.d[k] > 0.0 ? 1 : 0)) * h;
      const double tk = (plane - ph.p[k]) * ph.inv[k];
      tm[k] = ph.d[k] != 0.0 ? (tk > 0.0 ? tk : 0.0) : INFINITY;
      td[k] = h * fabs(ph.inv[k]);
      sg[k] = ph.d[k] > 0.0 ? 1 : -1;
    }
    const double ds = mus > 0.0 ? ph.rs / mus : INFINITY;
    const double left = tmax - ph.t;
    const int horizon = ds * nspm >= left;
    const double L = horizon ? fmax(0.0, left / nspm) : ds;
    double s0 = 0.0;
    /* ---- walk faces while the next one comes before L ---- */
    int face = 0, ax = 0;
    double sf = 0.0;
    for (;;) {
      int a = 0;
      double sm = tm[0];
      if (tm[1] < sm) {
        sm = tm[1];
        a = 1;
      }
      if (tm[2] < sm) {
        sm = tm[2];
        a = 2;
      }
      if (sm >= L) break; /* scatter / horizon win ties (transport.cpp:175, 191) */
      ++steps;
      const double w1 = ph.w * exp_neg(mua * (sm - s0));
      dp.dep += ph.w - w1;
      ph.w = w1;
      s0 = sm;
      ph.v[a] += sg[a];
      tm[a] += td[a];
      const int ext = !in_grid(s, ph.v);
      if (ext || s->labels[lin(s, ph.v)] != lab) {
        face = 1;
        ax = a;
        sf = sm;
        break;
      }
    }
    if (!face) { /* the flight ends inside the voxel at L */
      ++steps;
      const double w1 = ph.w * exp_neg(mua * (L - s0));
      dp.dep += ph.w - w1;
      ph.w = w1;
      for (int k = 0; k < 3; ++k) ph.p[k] += ph.d[k] * L;
      if (horizon) {
        ph.t = tmax;
        dp.trunc += ph.w;
        flags |= 4u;
        break;
      }
      ph.t += L * nspm;
      hg_rotate(&ph, g, &r);
      ph.rs = scat_len(&r);
      ++nscat;
      if (ph.w < c->roulette_threshold) {
        const double before = ph.w;
        if (orc_rng_unit(&r) < 1.0 / c->roulette_multiplier) {
          ph.w *= c->roulette_multiplier;
          dp.kill += before - ph.w;
        } else {
          dp.kill += before;
          flags |= 2u;
          break;
        }
      }
      continue;
    }
    /* ---- interface at the face sf (handle_interface, transport.cpp:227-298) ---- */
    ph.t += sf * nspm;
    ph.rs = fmax(0.0, ph.rs - sf * mus);
    for (int k = 0; k < 3; ++k) ph.p[k] += ph.d[k] * sf;
    ph.p[ax] = (ph.v[ax] + (sg[ax] > 0 ? 0 : 1)) * h; /* the moved index's near face */
    const int exterior = !in_grid(s, ph.v);
    const int nlab = exterior ? 0 : s->labels[lin(s, ph.v)];
    const double n2 = M[4 * nlab + 3];
    int exited = 0, back = 0;
    if (exterior && c->boundary_mode == VMC_BOUNDARY_TERMINATE) {
      exited = 1;
    } else if (n == n2) {
      exited = exterior;
    } else {
      const double ci = fabs(ph.d[ax]);
      const double si2 = fmax(0.0, 1.0 - ci * ci);
      const double eta = n / n2;
      const double st2 = eta * eta * si2;
      if (st2 > 1.0) {
        back = 1;
      } else {
        const double ct = sqrt(1.0 - st2);
        const double rsp = (n * ci - n2 * ct) / (n * ci + n2 * ct);
        const double rpp = (n * ct - n2 * ci) / (n * ct + n2 * ci);
        if (orc_rng_unit(&r) < 0.5 * (rsp * rsp + rpp * rpp)) {
          back = 1;
        } else {
          double nd[3];
          for (int k = 0; k < 3; ++k) nd[k] = k == ax ? (ph.d[ax] > 0.0 ? ct : -ct) : ph.d[k] * eta;
          const double kk = 1.0 / sqrt(nd[0] * nd[0] + nd[1] * nd[1] + nd[2] * nd[2]);
          for (int k = 0; k < 3; ++k) nd[k] *= kk;
          set_dir(&ph, nd);
          exited = exterior;
        }
      }
    }
    if (exited) {
      dp.esc += ph.w;
      flags |= 1u;
      break;
    }
    if (back) {
      double nd[3] = {ph.d[0], ph.d[1], ph.d[2]};
      nd[ax] = -nd[ax];
      set_dir(&ph, nd);
      ph.v[ax] -= sg[ax];
    } else {
      ph.label = nlab;
    }
  }
  if (tr) {
    orc_rng probe;
    orc_rng_seed(&probe, c->master_seed, idx);
    uint32_t k = 0;
    while (!(probe.lo == r.lo && probe.hi == r.hi) && k < (1u << 26)) {
      orc_rng_next(&probe);
      ++k;
    }
    tr->draws = k;
    tr->steps = steps;
    tr->scatters = nscat;
    tr->flags = flags;
    tr->deposited = dp.dep;
    tr->escaped = dp.esc;
    tr->killed = dp.kill;
    tr->truncated = dp.trunc;
  }
  acc->dep += dp.dep;
  acc->esc += dp.esc;
  acc->kill += dp.kill;
  acc->trunc += dp.trunc;
  return 0;
}

typedef struct {
  const ctx_t* cx;
  uint64_t first, lo, hi;
  int64_t* cells;
  vmc_photon_trace* traces;
  disp_t disp;
  hits_t hits;
  int want_hits;
  int flight;
  int status;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  for (uint64_t k = j->lo; k < j->hi; ++k) {
    const int rc = j->flight ? walk_one_flight(j->cx, j->first + k, j->traces ? j->traces + k : NULL, &j->disp)
                             : walk_one(j->cx, j->first + k, j->cells, j->traces ? j->traces + k : NULL, &j->disp,
                                        j->want_hits ? &j->hits : NULL);
    if (rc != 0) {
      j->status = 1;
      return NULL;
    }
  }
  return NULL;
}

static int walk_jobs(const vmc_scene* s, const vmc_config* c, uint64_t first, uint64_t count,
                     int threads, int64_t* cells_out, vmc_photon_trace* traces, double* disp4,
                     void* det_out, uint64_t* det_count, int flight) {
  if (s->nx < 1 || s->ny < 1 || s->nz < 1 || !(s->voxel_mm > 0.0) || s->nmedia < 1 ||
      s->nmedia > 256) {
    snprintf(g_err, sizeof g_err, "invalid grid");
    return 1;
  }
  ctx_t cx;
  cx.s = s;
  cx.c = c;
  cx.ngates = c->ngates > 0 ? c->ngates : 1;
  cx.gate_w = c->tmax_ns / cx.ngates;
  cx.inv_q = 1.0 / orc_quantum_for(c->photon_count);
  cx.nvox = (size_t)s->nx * s->ny * s->nz;
  const size_t ncell = cx.nvox * (size_t)cx.ngates;
  if (threads < 1) threads = 1;
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const int want_hits = c->ndet > 0 && (det_out || det_count);
  for (int t = 0; t < threads; ++t) {
    jobs[t].cx = &cx;
    jobs[t].first = first;
    jobs[t].lo = count * (uint64_t)t / (uint64_t)threads;
    jobs[t].hi = count * (uint64_t)(t + 1) / (uint64_t)threads;
    jobs[t].cells = cells_out ? (int64_t*)calloc(ncell, sizeof(int64_t)) : NULL;
    jobs[t].traces = traces;
    jobs[t].want_hits = want_hits;
    jobs[t].flight = flight;
    pthread_create(&tids[t], NULL, run_job, &jobs[t]);
  }
  int status = 0;
  for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
  disp_t tot = {0, 0, 0, 0};
  if (cells_out) memset(cells_out, 0, ncell * sizeof(int64_t));
  const size_t stride = vmc_det_record_bytes(s->nmedia);
  uint64_t nrec = 0;
  for (int t = 0; t < threads; ++t) {
    if (jobs[t].status) status = 1;
    tot.dep += jobs[t].disp.dep;
    tot.esc += jobs[t].disp.esc;
    tot.kill += jobs[t].disp.kill;
    tot.trunc += jobs[t].disp.trunc;
    if (cells_out) {
      for (size_t i = 0; i < ncell; ++i) cells_out[i] += jobs[t].cells[i];
      free(jobs[t].cells);
    }
    for (size_t i = 0; i < jobs[t].hits.n; ++i, ++nrec) {
      if (det_out && nrec < c->det_capacity) {
        unsigned char* rec = (unsigned char*)det_out + nrec * stride;
        const hit_t* hh = &jobs[t].hits.v[i];
        memset(rec, 0, stride);
        vmc_det_record_head head = {hh->photon, hh->det, hh->nscat, hh->w, hh->t};
        memcpy(rec, &head, sizeof head);
        memcpy(rec + sizeof head, hh->ppath, sizeof(float) * (size_t)(s->nmedia - 1));
      }
    }
    free(jobs[t].hits.v);
  }
  if (det_count) *det_count = nrec;
  if (disp4) {
    disp4[0] = tot.dep;
    disp4[1] = tot.esc;
    disp4[2] = tot.kill;
    disp4[3] = tot.trunc;
  }
  free(jobs);
  free(tids);
  if (status) {
    snprintf(g_err, sizeof g_err, "source entry point maps outside the voxel grid");
    return 1;
  }
  return 0;
}

int orc_walk(const vmc_scene* s, const vmc_config* c, uint64_t first, uint64_t count,
             int threads, int64_t* cells_out, vmc_photon_trace* traces, double* disp4,
             void* det_out, uint64_t* det_count) {
  return walk_jobs(s, c, first, count, threads, cells_out, traces, disp4, det_out, det_count, 0);
}

int orc_walk_flight(const vmc_scene* s, const vmc_config* c, uint64_t first, uint64_t count,
                    int threads, vmc_photon_trace* traces, double* disp4) {
  return walk_jobs(s, c, first, count, threads, NULL, traces, disp4, NULL, NULL, 1);
}

size_t vmc_det_record_bytes(int32_t nmedia) {
  const size_t raw = sizeof(vmc_det_record_head) + sizeof(float) * (size_t)(nmedia > 1 ? nmedia - 1 : 0);
  return (raw + 7) & ~(size_t)7;
}
