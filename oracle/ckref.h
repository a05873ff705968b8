/*
 * ckref.h — TEST INFRASTRUCTURE ONLY.  C entry points of oracle/_ref/libckref.so,
 * the reference CK-MPM CPU engine (/root/reference/proj/include/ckmpm/*.hpp)
 * compiled unmodified, with its own Release flags, behind a thin extern "C"
 * shim (oracle/ref_shim.cpp).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 */
#ifndef CKREF_H_
#define CKREF_H_

#include <stdint.h>

#include "../include/ckmpm_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* BodySpec<T> + ShapeSpec<T> (scene.hpp:24-40, :140-149) flattened. */
typedef struct ckref_body {
  int32_t kind; /* 0 sphere, 1 box, 2 cylinder (ShapeKind, scene.hpp:16) */
  int32_t axis;
  double center[3];
  double radius, inner_radius, half_length;
  double lo[3], hi[3];
  uint32_t material;
  int32_t ppc;
  uint64_t seed;
  double velocity[3];
  double shear_slope;
  double omega[3];
} ckref_body;

/* Extra SimConfig fields the step itself does not need. */
typedef struct ckref_extra {
  double cfl, frame_dt, max_dt;
  int32_t threads; /* 0 = hardware concurrency */
  int32_t _pad;
} ckref_extra;

/* Reference finalize_material<T> (material.hpp:61-88): fills mu/lambda/dp_alpha. */
int32_t ckref_finalize_material(ckg_material* m, int32_t precision, char* err, int32_t cap);

/* seed_particles<T> (scene.hpp:204-230) over the given bodies; returns the
 * particle count, writes up to cap particles (precision layout). */
int64_t ckref_seed(const ckg_config* cfg, const ckref_body* bodies, int32_t nbodies,
                   void* out, int64_t cap);

/* Simulation<T> built from cfg (+extra), then restore()d to `particles`
 * (simulation.hpp:88-101, :120-129). */
void* ckref_sim_create(const ckg_config* cfg, const ckref_extra* extra, const void* particles,
                       uint64_t n, char* err, int32_t cap);
void ckref_sim_destroy(void* sim);
/* Simulation<T>::step; returns 0 or the exit-code class (2/3/4) with the message. */
int32_t ckref_sim_step(void* sim, double dt, char* err, int32_t cap);
double ckref_sim_cfl_dt(void* sim, double remaining);
uint64_t ckref_sim_count(void* sim);
int32_t ckref_sim_particles(void* sim, void* out, uint64_t n);
/* PhaseTimers seconds: sort, activate, clear, p2g, grid, g2p. */
void ckref_sim_timers(void* sim, double* out6);
uint64_t ckref_sim_active_blocks(void* sim);
/* Blocks in the reference's own (first-touch) order. nodes: nb*128*4. */
int32_t ckref_sim_grid(void* sim, int32_t* coords, double* nodes, uint64_t nb);
/* The reference's write_checkpoint / write_snapshot_{binary,text} (io.hpp:344-430)
 * on the current state; 0 ok, 4 io error, 5 shim built without io.hpp. */
int32_t ckref_sim_write_checkpoint(void* sim, const char* path);
int32_t ckref_sim_write_snapshot(void* sim, const char* path, int32_t frame, int32_t binary);
void ckref_sim_diagnostics(void* sim, ckg_diagnostics* out);
double ckref_sim_mass_epsilon(void* sim);

/* Serial P2G of scatter_all (simulation.hpp:279-337, deterministic branch)
 * on a sorted copy of `particles`: sort_particles -> activate -> clear ->
 * scatter.  Returns the active block count; fills up to nb blocks. */
int64_t ckref_p2g(const ckg_config* cfg, const void* particles, uint64_t n, double dt,
                  int32_t* coords, double* nodes, uint64_t nb, char* err, int32_t cap);

/* Reference sort_particles (simulation.hpp:248-274): keys[i], order[i] for
 * sorted position i (order = index into the input array). */
int32_t ckref_sort(const ckg_config* cfg, const void* particles, uint64_t n, uint32_t* keys,
                   uint32_t* order);

/* Kernel-level known answers (kernel.hpp:77-137). */
double ckref_ck_weight_1d(double u);
double ckref_ck_grad_1d(double u);
void ckref_axis_pair(double x, int32_t k, double dx, int32_t* base, double* f_w0_w1_g0_g1);

/* Math oracles (math.hpp): F row-major 9 doubles. */
void ckref_polar_rotation(const double* F, double* R);
void ckref_svd3(const double* F, double* U, double* sigma, double* V);
int32_t ckref_return_map_dp(const double* F, double alpha, double mu, double lambda, double* out);
void ckref_force_matrix(const ckg_particle_f64* p, const ckg_material* m, double* A, char* err,
                        int32_t cap);

#ifdef __cplusplus
}
#endif

#endif
