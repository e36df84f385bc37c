/* oracle/voxmc_oracle.h — TEST INFRASTRUCTURE ONLY.
 * Plain-C, double-precision restatement of the reference's photon-transport
 * hot path (see voxmc_oracle.c for the file:line each function follows).
 * Used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as
 * the checker; never linked into or called by the product library. */
#ifndef VOXMC_ORACLE_H_
#define VOXMC_ORACLE_H_

#include <stdint.h>

#include "../include/vmc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_rng {
  uint64_t lo, hi;
} orc_rng;

uint64_t orc_mix64(uint64_t z);
void orc_rng_seed(orc_rng* r, uint64_t seed, uint64_t stream_id);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_unit(orc_rng* r);
void orc_rng_kat(uint64_t seed, uint64_t stream_id, int n, uint64_t* out);
double orc_quantum_for(uint64_t photon_count);
double orc_hg_cos_theta(double g, double xi);
double orc_fresnel(double n1, double n2, double cos_i);

/* Photons [first, first+count): per-step deposits (llround in the quantum of
 * config->photon_count) into cells_out[ngates*V] (may be NULL), per-photon
 * traces (may be NULL), summed dispositions disp4 (may be NULL), detector
 * records sorted by photon index. Returns 0, 1 (validation) or 2. */
int orc_walk(const vmc_scene* scene, const vmc_config* config, uint64_t first, uint64_t count,
             int threads, int64_t* cells_out, vmc_photon_trace* traces, double* disp4,
             void* det_out, uint64_t* det_count);

/* The same photons walked in the flight kernel's decomposition (K1f,
 * csrc/flight.cuh) in double precision: per-photon traces and dispositions. */
int orc_walk_flight(const vmc_scene* scene, const vmc_config* config, uint64_t first, uint64_t count,
                    int threads, vmc_photon_trace* traces, double* disp4);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
