/*
 * ckmpm_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C (C11) restatement of the reference CK-MPM per-substep path,
 * Simulation<double>::step in its deterministic (serial scatter) mode
 * (/root/reference/proj/include/ckmpm/simulation.hpp:150-188), with every
 * function citing the reference file:line it restates.  Compiled without FMA
 * contraction (-ffp-contract=off; x86-64 baseline, like the reference build)
 * and with the reference's operation order, so on the same machine it is
 * bit-identical to the reference engine (pinned by tests/test_oracle_pin.py
 * against oracle/_ref/libckref.so and the committed golden fixtures).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it — as the checker, never as the product.
 */
#ifndef CKMPM_ORACLE_H_
#define CKMPM_ORACLE_H_

#include <stdint.h>

#include "../include/ckmpm_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ckor_sim ckor_sim;

ckor_sim* ckor_create(const ckg_config* cfg, const ckg_particle_f64* particles, uint64_t n);
void ckor_destroy(ckor_sim* s);
/* One substep; 0 or 2/3 with the reference's message in err. */
int32_t ckor_step(ckor_sim* s, double dt, ckg_step_out* out, char* err, int32_t cap);
/* Runs phases up to stop_after (CKG_PHASE_*), like ckg_step_phases. */
int32_t ckor_step_phases(ckor_sim* s, double dt, int32_t stop_after, ckg_step_out* out, char* err,
                         int32_t cap);
uint64_t ckor_count(const ckor_sim* s);
void ckor_particles(const ckor_sim* s, ckg_particle_f64* out);
double ckor_cfl_dt(const ckor_sim* s, double cfl, double max_dt, double remaining);
double ckor_vmax(const ckor_sim* s);
uint64_t ckor_active_blocks(const ckor_sim* s);
/* First-touch block order, nodes nb*128*4 {mass, p}. */
void ckor_grid(const ckor_sim* s, int32_t* coords, double* nodes, uint64_t nb);
/* Stable sort of the current state without modifying it. */
void ckor_sort(const ckor_sim* s, uint32_t* keys, uint32_t* order);
void ckor_diagnostics(const ckor_sim* s, ckg_diagnostics* out);

/* Kernel-level restatements (kernel.hpp:77-137). */
double ckor_ck_weight_1d(double u);
double ckor_ck_grad_1d(double u);
void ckor_axis_pair(double x, int32_t k, double dx, int32_t* base, double* f_w0_w1_g0_g1);
void ckor_polar_rotation(const double* F, double* R);
void ckor_svd3(const double* F, double* U, double* sigma, double* V);

#ifdef __cplusplus
}
#endif

#endif
