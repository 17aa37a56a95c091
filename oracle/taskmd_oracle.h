/*
 * TEST INFRASTRUCTURE ONLY — the CPU checker for libtmd_gpu.so, never the
 * product. Plain-C restatement of the reference engine's LJ hot path
 * (/root/reference/proj/include/taskmd/), written from the reference's
 * published behaviour; every function cites the file:line it restates.
 *
 * What it adds over the reference (SURVEY §8c "what a restatement must add"):
 *   - the virial W = sum over in-cut pairs of ff * r^2;
 *   - compensated (Neumaier, long double) sums for PE, W, KE and per-particle
 *     forces, so 1e-12-relative energy comparisons have a trustworthy anchor
 *     (the reference's single running double sum drifts ~1e-12 relative);
 *   - the FCC lattice generator of the BASELINE configs.
 * Pinned against the reference itself (oracle/_ref) through the golden
 * vectors in tests/golden (oracle/make_golden.py, tests/test_oracle_golden.py).
 * Compiled with -ffp-contract=off so every rounding is the reference's.
 */
#ifndef TASKMD_ORACLE_H_
#define TASKMD_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tmo_lj {
  double sigma2, rc2, eps4, eps24, shift;
} tmo_lj;

void tmo_lj_prepare(double eps, double sigma, double rc, int shifted, tmo_lj* out);
void tmo_lj_eval(double r2, const tmo_lj* p, double* energy, double* force_factor);
double tmo_wrap1(double p, double length);
int tmo_cell_grid(const double box[3], double r_cut, double r_skin, int dims[3],
                  double cell_len[3]);
int tmo_cell_of(const double p[3], const int dims[3], const double cell_len[3]);
void tmo_counter_uniform3(uint64_t seed, uint64_t ctx, uint64_t step, uint64_t id,
                          double out[3]);
void tmo_counter_normal3(uint64_t seed, uint64_t ctx, uint64_t step, uint64_t id,
                         double out[3]);
void tmo_thermal_velocities(int64_t n, const int64_t* id, const double* mass,
                            double temperature, uint64_t seed, double* vel);
int tmo_gen_fcc(int cells, double rho, double offset, int64_t* id, double* pos,
                double box[3]);

typedef struct tmo_system tmo_system;

/* status: 0 ok, 1 config, 2 physics (same codes as include/tmd_gpu.h) */
tmo_system* tmo_create(int64_t n, const int64_t* id, const double* mass,
                       const double* pos, const double* vel, const double box[3],
                       double eps, double sigma, double r_cut, int shifted,
                       double r_skin, double dt, int* status);
int tmo_step(tmo_system* s, int64_t nsteps);
/* {step, kinetic, potential, virial, temperature} */
void tmo_observe(const tmo_system* s, double out[5]);
int64_t tmo_pairs(const tmo_system* s, int64_t* out, int64_t cap);
void tmo_cell_of_all(const tmo_system* s, int64_t* id, int32_t* cell);
void tmo_forces(const tmo_system* s, int64_t* id, double* f);
void tmo_flatten(const tmo_system* s, int64_t* id, double* pos, double* vel);
uint64_t tmo_rebuild_count(const tmo_system* s);
int64_t tmo_size(const tmo_system* s);
const char* tmo_error(const tmo_system* s);
void tmo_destroy(tmo_system* s);

#ifdef __cplusplus
}
#endif

#endif
