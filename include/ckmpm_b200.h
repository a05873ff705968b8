/*
 * ckmpm_b200.h — C-ABI of the B200-native CK-MPM per-substep transfer path.
 *
 * The reference (CK-MPM, arXiv 2412.10399, shipped as the header-only C++
 * engine under proj/include/ckmpm/) has no plugin/FFI seam: callers drive
 * `ckmpm::Simulation<T>` directly (proj/include/ckmpm/simulation.hpp:85-219).
 * This header is the seam a maintainer binds instead of the CPU engine's
 * `Simulation<T>::step` (simulation.hpp:150-188).  Every entry point below
 * names the reference interface it replaces.  Plain pointers and sizes only;
 * no torch or C++ types cross this boundary.
 *
 * Status convention (reference exception taxonomy, proj/include/ckmpm/
 * errors.hpp:9-32, exit codes of proj/tools/ckmpm_main.cpp:218-230):
 *   0 ok, 2 ConfigError, 3 NumericalError (sub-code in ckg_step_out), 4 IoError,
 *   5 device/runtime failure (no reference equivalent; never silently ignored).
 */
#ifndef CKMPM_B200_H_
#define CKMPM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKG_ABI_VERSION 2

#define CKG_OK 0
#define CKG_ERR_CONFIG 2
#define CKG_ERR_NUMERICAL 3
#define CKG_ERR_IO 4
#define CKG_ERR_DEVICE 5

/* Numerical sub-codes; each maps to one throw site of the reference. */
#define CKG_NUM_NONE 0
#define CKG_NUM_OUT_OF_DOMAIN 1      /* grid.hpp:122-126 OutOfDomainError "particle N violates the 2-cell domain inset on axis A" */
#define CKG_NUM_FC_STRESS_INVERTED 2 /* transfer.hpp:192-193 InvertedElementError "fixed corotated stress: det F <= 0" */
#define CKG_NUM_DP_STRESS_INVERTED 3 /* transfer.hpp:202-203 InvertedElementError "granular stress: det F <= 0" */
#define CKG_NUM_FLUID_STATE_J 4      /* material.hpp:134 NumericalError "fluid state: J must be > 0" */
#define CKG_NUM_NEAR_SINGULAR_D 5    /* transfer.hpp:226-227 NumericalError "near-singular APIC D matrix" */
#define CKG_NUM_SINGULAR_MLS 6       /* simulation.hpp:305-306 NumericalError "singular MLS moment matrix" */
#define CKG_NUM_RETURN_MAP_INVERTED 7/* material.hpp:159-160 InvertedElementError "plastic return map: det F <= 0" */
#define CKG_NUM_F_INVERTED 8         /* transfer.hpp:622-623 InvertedElementError "deformation gradient inverted" */
#define CKG_NUM_FLUID_J 9            /* transfer.hpp:616 NumericalError "fluid compression drove J <= 0" */
#define CKG_NUM_NONFINITE 10         /* simulation.hpp:384-387 NumericalError "non-finite particle state after step N" */
#define CKG_NUM_INACTIVE_BLOCK 11    /* grid.hpp:166-169 NumericalError "access to inactive grid block ..." (defensive) */
#define CKG_NUM_SUBSTEP_LIMIT 12     /* simulation.hpp:205-207 NumericalError "substep limit exceeded within one frame at t = T" */

#define CKG_MAX_MATERIALS 16
#define CKG_MAX_BOUNDARIES 32

/* MaterialModel (material.hpp:12) — same ordinal values. */
#define CKG_MODEL_FIXED_COROTATED 0
#define CKG_MODEL_J_FLUID 1
#define CKG_MODEL_DRUCKER_PRAGER 2

/* TransferScheme (transfer.hpp:16) — same ordinal values. */
#define CKG_SCHEME_PIC 0
#define CKG_SCHEME_APIC 1
#define CKG_SCHEME_MLS 2

/* BcKind (grid.hpp:20) — same ordinal values. */
#define CKG_BC_STICKY 0
#define CKG_BC_SLIP 1
#define CKG_BC_SEPARATE 2

/* Phases of Simulation::step (simulation.hpp:150-187), also the stop points
 * of ckg_step_phases. */
/* ckg_config.flags */
#define CKG_FLAG_QUADRATIC 1  /* KernelKind::quadratic (transfer.hpp:17): the 27-node B-spline baseline on one grid */
#define CKG_FLAG_FUSED 2      /* run each substep's G2P fused with the next substep's P2G (one kernel, DESIGN.md
                                 §4e; compact kernel, PIC/APIC, one GPU; ignored otherwise).  CKMPM_FUSED=1 in
                                 the environment has the same effect.  Off by default: on the B200 it is slower
                                 than the separate P2G / G2P kernels. */

#define CKG_PHASE_SORT 1
#define CKG_PHASE_ACTIVATE 2
#define CKG_PHASE_CLEAR 3
#define CKG_PHASE_P2G 4
#define CKG_PHASE_GRID 5
#define CKG_PHASE_G2P 6

/* Material<T> after finalize_material (material.hpp:34-50, :61-88).  The host
 * runs the reference's finalize; derived fields (mu, lambda, dp_alpha) are
 * passed in, never recomputed on the device. */
typedef struct ckg_material {
  int32_t model;
  int32_t _pad;
  double density, E, nu, mu, lambda;
  double bulk, gamma, viscosity;
  double friction_angle_deg, dp_alpha;
} ckg_material;

/* BoundaryCondition<T> (grid.hpp:26-56). */
typedef struct ckg_boundary {
  int32_t kind;
  int32_t _pad;
  double lo[3], hi[3], normal[3], velocity[3], omega[3], center[3];
} ckg_boundary;

/* Flattened SimConfig<T> (scene.hpp:159-182), the fields the step consumes.
 * precision: 8 = Simulation<double>, 4 = Simulation<float>.  All reals are
 * carried as double; in float mode they must be the exact widening of the
 * host's float values (dx and inv_dx included: dx = extent/T(res) and
 * inv_dx = T(1)/dx as the reference computes them in T, simulation.hpp:250,
 * grid.hpp:117, scene.hpp:181). */
typedef struct ckg_config {
  int32_t abi_version;   /* CKG_ABI_VERSION */
  int32_t precision;     /* 8 or 4 */
  int32_t resolution;    /* cubic cell resolution */
  int32_t scheme;        /* CKG_SCHEME_* */
  double extent, dx, inv_dx;
  double gravity[3];
  double mass_eps;       /* Simulation::compute_mass_epsilon (simulation.hpp:227-232) */
  int32_t clamp_singular;
  int32_t deterministic; /* the reference's serial-scatter switch (simulation.hpp:326-327): P2G node sums are
                            formed in a fixed order (per-block tiles summed by key-block offset, out-of-tile
                            records in particle order), so single-domain runs are bitwise reproducible on
                            the same GPU (not bitwise equal to the CPU engine); x-slab ranks ignore it */
  double clamp_floor;
  int32_t n_materials;
  int32_t n_boundaries;
  ckg_material materials[CKG_MAX_MATERIALS];
  ckg_boundary boundaries[CKG_MAX_BOUNDARIES];
  int32_t device;        /* CUDA ordinal */
  int32_t flags;         /* CKG_FLAG_*; 0 = compact kernel on the dual grids */
} ckg_config;

/* Particle<T> (transfer.hpp:19-28), byte-identical layout: 224 B (double),
 * 112 B (float).  Upload/download take arrays of these. */
typedef struct ckg_particle_f64 {
  double x[3], v[3], F[9], B[9];
  double J, mass, volume0;
  uint32_t material;
  uint32_t _pad;
} ckg_particle_f64;

typedef struct ckg_particle_f32 {
  float x[3], v[3], F[9], B[9];
  float J, mass, volume0;
  uint32_t material;
} ckg_particle_f32;

/* What Simulation::step/gather_all leave behind for cfl_dt and the caller
 * (simulation.hpp:380-395), plus TransferCounters (transfer.hpp:32-45) and
 * PhaseTimers (simulation.hpp:34-42) deltas for this step. */
typedef struct ckg_step_out {
  double vmax;                        /* sqrt(max |v|^2) over particles */
  double min_j[CKG_MAX_MATERIALS];    /* per-material min J over fluid particles, 1 if none */
  uint64_t p2g_node_visits, g2p_node_visits, p2g_transfers, g2p_transfers;
  double phase_ms[6];                 /* sort, activate, clear, p2g, grid, g2p (device time) */
  int32_t status;                     /* CKG_OK / CKG_ERR_* */
  int32_t error_code;                 /* CKG_NUM_* */
  int32_t error_axis;                 /* OutOfDomain axis */
  int32_t error_phase;                /* CKG_PHASE_* where the error was raised */
  uint64_t error_particle;            /* sorted particle index (OutOfDomainError::particle_index) */
  uint64_t active_blocks;             /* BlockSparseGrid::active_block_count after activate */
  uint64_t kernel_launches;           /* device kernels this call enqueued */
  uint64_t sort_changed;              /* particles whose block key changed since the last sort */
  int32_t sort_kind;                  /* 0 full radix, 1 identity, 2 incremental merge */
  int32_t slab_migration;             /* slab substeps: 1 boundary-plane compaction, 2 full relayout */
  uint64_t substeps_done;             /* substeps completed by this call (ckg_step_many stops at the first
                                         failing one; the state is the one after the last completed) */
} ckg_step_out;

/* advance_frame (simulation.hpp:193-211) on the device: the host passes the
 * reference driver's bookkeeping (time_, frame_index_, vmax_, min_j_ and the
 * config's cfl / max_dt / frame_dt / max_substeps_per_frame); the substeps,
 * cfl_dt (simulation.hpp:134-145) and the frame-boundary test run on the GPU as
 * one CUDA-graph launch (conditional WHILE node), with no host round trip per
 * substep.  Without a per-substep callback this replaces the reference loop;
 * with one, callers keep the host loop over ckg_step. */
typedef struct ckg_frame_in {
  double time;                        /* time_ at entry (T value) */
  double frame_dt;                    /* cfg.frame_dt */
  uint64_t frame_index;               /* frame_index_ (frame_end = frame_dt * (frame_index + 1)) */
  double cfl, max_dt;                 /* cfg.cfl, cfg.max_dt */
  uint64_t max_substeps;              /* cfg.max_substeps_per_frame */
  double vmax;                        /* vmax_ */
  double min_j[CKG_MAX_MATERIALS];    /* min_j_ */
} ckg_frame_in;

typedef struct ckg_frame_out {
  uint64_t substeps;                  /* substeps completed in this call */
  double time;                        /* time_ after the call (frame_end when the frame completed) */
  double last_dt;                     /* dt of the last completed substep */
  double vmax;                        /* vmax_ / min_j_ after the last completed substep */
  double min_j[CKG_MAX_MATERIALS];
  double device_ms;                   /* device time of the frame */
  int32_t status;                     /* CKG_OK / CKG_ERR_* (as ckg_step; the failing substep is not counted) */
  int32_t error_code;                 /* CKG_NUM_* (CKG_NUM_SUBSTEP_LIMIT after max_substeps + 1 substeps) */
  int32_t error_axis;
  int32_t error_phase;
  uint64_t error_particle;
  uint64_t active_blocks;
  uint64_t kernel_launches;           /* kernels executed (graph nodes x substeps) */
  int32_t graph;                      /* 1: device-driven graph; 0: host loop (slab mode, growing pool) */
  int32_t _pad;
  uint64_t sort_paths[3];             /* graph substeps by sort path: one-CTA crosser sort, padded radix, full radix */
} ckg_frame_out;

/* DiagnosticsRow<T> (simulation.hpp:44-53), computed on the device
 * (compute_diagnostics, simulation.hpp:55-69). */
typedef struct ckg_diagnostics {
  double momentum[3], angular[3], momentum_massfree[3];
  double kinetic_energy, vmax;
} ckg_diagnostics;

typedef struct ckg_ctx ckg_ctx;

/* ABI/build identification. */
int32_t ckg_abi_version(void);
const char* ckg_build_info(void);
const char* ckg_status_string(int32_t status);

/* Replaces Simulation<T>::Simulation(SimConfig) minus seeding
 * (simulation.hpp:88-101): validates, allocates device state on cfg->device.
 * The caller seeds with the reference's seed_particles (scene.hpp:204) and
 * passes the particles to ckg_upload. */
int32_t ckg_create(const ckg_config* cfg, ckg_ctx** out);
void ckg_destroy(ckg_ctx* ctx);

/* Replaces Simulation<T>::restore(particles, ...) / the seeded particles_
 * (simulation.hpp:120-129): host AoS -> device SoA.  Layout per precision. */
int32_t ckg_upload(ckg_ctx* ctx, const void* particles, uint64_t n);
/* Replaces Simulation<T>::particles() (simulation.hpp:106-107): device SoA ->
 * host AoS, in the device's current (sorted) order. */
int32_t ckg_download(ckg_ctx* ctx, void* particles, uint64_t n);
uint64_t ckg_particle_count(const ckg_ctx* ctx);
/* 1 when the context's substeps run the fused G2P2G kernel, else 0. */
int32_t ckg_fused(const ckg_ctx* ctx);

/* Replaces Simulation<T>::mass_eps_ (simulation.hpp:227-232; restore() sets it). */
int32_t ckg_set_mass_epsilon(ckg_ctx* ctx, double mass_eps);

/* Replaces Simulation<T>::step(dt) (simulation.hpp:150-188): one substep,
 * synchronous; on return `out` holds vmax/minJ/error for cfl_dt. */
int32_t ckg_step(ckg_ctx* ctx, double dt, ckg_step_out* out);
/* `count` substeps of fixed dt, as `count` ckg_step calls (untimed): stops at
 * the first failing substep, whose error `out` reports, leaving the state after
 * the last completed one (out->substeps_done), like the reference's state
 * after a throwing step() call in a loop.  A pool overflow grows the pool and
 * retries that substep.  Once the stored-order keys and the stress cache
 * exist (after a first substep) and the pool is dense, the substeps run as
 * one launch of the frame graph in a fixed-dt mode (no host round trip in
 * between; same results and the same stop-at-failure contract).  `out` may
 * be NULL. */
int32_t ckg_step_many(ckg_ctx* ctx, double dt, int32_t count, ckg_step_out* out);
/* Simulation::advance_frame() without a callback (simulation.hpp:193-211, :213-215). */
int32_t ckg_advance_frame(ckg_ctx* ctx, const ckg_frame_in* in, ckg_frame_out* out);

/* Checkpoint / snapshot bodies packed on the device from the current state,
 * in the exact byte layout of the reference's files (io.hpp:344-430), so a
 * writer only prepends the header:
 *   CKG_RECORDS_CHECKPOINT: CKCHKPT1 particle records (write_checkpoint,
 *     io.hpp:392-430): 27 T fields (x, v, F, B row-major, J, mass, volume0) + u32 material;
 *   CKG_RECORDS_SNAPSHOT: CKSNAP1 particle records (write_snapshot_binary,
 *     io.hpp:370-390): x, v, (J if fluid else det F) as 7 doubles + u32 material.
 * Particles are in the device's current (sorted) order, as the reference's
 * particles() after the same substeps.  async != 0 returns once the pack is
 * enqueued; the device-to-host copy runs on its own stream and later substeps
 * overlap it; ckg_records_wait() blocks until `host` is filled (use pinned
 * memory for a truly asynchronous copy). */
#define CKG_RECORDS_CHECKPOINT 0
#define CKG_RECORDS_SNAPSHOT 1
uint64_t ckg_record_bytes(const ckg_ctx* ctx, int32_t kind);
int32_t ckg_pack_records(ckg_ctx* ctx, int32_t kind, void* host, uint64_t bytes, int32_t async);
int32_t ckg_records_wait(ckg_ctx* ctx);

/* Runs step(dt) only up to and including `stop_after` (CKG_PHASE_*); particle
 * state is not advanced unless stop_after == CKG_PHASE_G2P.  Test/parity hook
 * (the reference exposes the same cut points through full_step's pieces,
 * transfer.hpp:634-669). */
int32_t ckg_step_phases(ckg_ctx* ctx, double dt, int32_t stop_after, ckg_step_out* out);

/* Binning parity hooks (simulation.hpp:248-274, kernel.hpp:114-120).  Both
 * work on the current device state without changing it.
 * ckg_debug_sort: keys[i] = block key of sorted position i, order[i] = index
 * (in current order) of the particle placed at sorted position i.
 * ckg_debug_bases: bases[(p*2+g)*3+a] = axis_pair(x_p[a], k_g, dx).base for
 * the particle at current position p (g = 0: k = -1, g = 1: k = +1). */
int32_t ckg_debug_sort(ckg_ctx* ctx, uint32_t* keys, uint32_t* order, uint64_t n);
int32_t ckg_debug_bases(ckg_ctx* ctx, int32_t* bases, uint64_t n);

/* Grid facade (BlockSparseGrid<T>, grid.hpp:75-281) over the device grid as
 * left by the last step / ckg_step_phases. */
uint64_t ckg_grid_active_block_count(ckg_ctx* ctx);     /* active_block_count (grid.hpp:153) */
/* coords: 3*nb int32 block coordinates; nodes: nb * 128 * 4 doubles in the
 * reference's Block::nodes order ((g<<6)|(i&3)<<4|(j&3)<<2|(k&3), each
 * {mass, p.x, p.y, p.z}; grid.hpp:81-84, :172-175).  Blocks are listed in
 * ascending directory order (the reference lists them in first-touch order;
 * compare as sets keyed by coordinate).  nodes may be NULL. */
int32_t ckg_grid_download(ckg_ctx* ctx, int32_t* coords, double* nodes, uint64_t nb);
/* total_mass / total_momentum per grid slot (grid.hpp:199-213). */
int32_t ckg_grid_totals(ckg_ctx* ctx, double mass[2], double momentum[6]);

/* compute_diagnostics on the device (simulation.hpp:55-69). */
int32_t ckg_diagnostics_compute(ckg_ctx* ctx, ckg_diagnostics* out);

/* ---- x-slab decomposition (net-new, the reference has none).
 * One context per GPU/rank owning block planes bx in [bx_lo, bx_hi); the
 * substep is split into stages and the host moves the exchange buffers
 * (device pointers) between them with NCCL (paper_2412_10399_b200/slab.py):
 *   ckg_slab_bin      key/sort of own particles; footprint flags (D^3 u32) -> core_out
 *   (host: the flags of the planes shared with each neighbour, MAX-merged)
 *   ckg_slab_p2g      activation from the merged flags, clear, P2G;
 *                     block counts of planes {bx_lo-1, bx_lo, bx_hi-1, bx_hi}
 *   ckg_slab_p2g_part the same in two parts: 1 = activation, clear and the
 *                     P2G of the boundary planes bx_lo, bx_hi-1 (the only
 *                     ones whose tiles reach the ghost planes; counts as
 *                     above), 2 = the interior planes' P2G, enqueued while
 *                     part 1's halo is in flight (part 0 = ckg_slab_p2g)
 *   ckg_slab_halo     (stream-ordered on ckg_stream, no host synchronisation)
 *                     op 0 pack a plane, 1 add into it, 2 overwrite it
 *                     (block = 2 grids x 4 values x 64 nodes of T); op 5 / 6
 *                     pack / overwrite the velocities only (2 x 3 x 64 of T
 *                     per block: the broadcast after the grid update);
 *                     deterministic mode: op 3 pack the plane's P2G tiles,
 *                     4 overwrite them (ckg_slab_tile_words() T per block):
 *                     the boundary planes' tiles replace the ghost-node
 *                     reduce-add, so the owner sums every node in the
 *                     single-domain order (bitwise equal to one domain)
 *   ckg_slab_grid     (deterministic mode: fixed-order tile sums, then) grid
 *                     update of own planes
 *   ckg_slab_g2p      G2P; counts of particles leaving left / right
 *   ckg_slab_pack     survivors compacted after nl_in incoming; migrant records
 *                     (ckg_slab_record_words() T words each) into left/right
 *   ckg_slab_finish   incoming records appended [left][survivors][right]
 * Must be called before ckg_upload. */
int32_t ckg_slab_set(ckg_ctx* ctx, int32_t rank, int32_t world, int32_t bx_lo, int32_t bx_hi);
/* Rebalancing: particles of the current state per sort-key plane bx
 * (counts[D], D = resolution/4 + 2), and new slab bounds that take effect at
 * the next substep's migration (ckg_slab_g2p classifies against them, the
 * planes that change hands travel with the migrants, ckg_slab_finish commits
 * them).  Every rank must apply one consistent partition, in which each
 * rank's new slab only overlaps its neighbours' old ones. */
int32_t ckg_slab_plane_counts(ckg_ctx* ctx, uint64_t* counts);
int32_t ckg_slab_rebound(ckg_ctx* ctx, int32_t bx_lo, int32_t bx_hi);
int32_t ckg_slab_bin(ckg_ctx* ctx, double dt, void* core_out);
int32_t ckg_slab_p2g(ckg_ctx* ctx, const void* core_in, uint64_t plane_blocks[4]);
int32_t ckg_slab_p2g_part(ckg_ctx* ctx, const void* core_in, uint64_t plane_blocks[4], int32_t part);
int32_t ckg_slab_halo(ckg_ctx* ctx, int32_t op, int32_t plane, void* buf);
int32_t ckg_slab_grid(ckg_ctx* ctx);
int32_t ckg_slab_g2p(ckg_ctx* ctx, uint64_t counts[2]);
int32_t ckg_slab_pack(ckg_ctx* ctx, uint64_t nl_in, void* left, void* right);
int32_t ckg_slab_finish(ckg_ctx* ctx, const void* left, uint64_t nl, const void* right, uint64_t nr,
                        ckg_step_out* out);
int32_t ckg_slab_record_words(void);
/* The context's CUDA stream (cudaStream_t): a host driving the slab exchanges
 * with NCCL enqueues them on it, so the library's kernels and the transfers
 * are ordered on the device with no host synchronisation in between. */
void* ckg_stream(ckg_ctx* ctx);
/* Words (T) per block of a deterministic-mode P2G tile message (ckg_slab_halo ops 3/4). */
int32_t ckg_slab_tile_words(void);

/* Device-side timing on the context's stream (the stream every kernel of
 * this context is launched on): record marker `slot` (0..15); elapsed ms
 * between two recorded markers (synchronises on `b`). */
int32_t ckg_timer_mark(ckg_ctx* ctx, int32_t slot);
int32_t ckg_timer_elapsed(ckg_ctx* ctx, int32_t a, int32_t b, double* ms);

/* Formats the last error exactly as the reference's exception message. */
int32_t ckg_last_error_message(ckg_ctx* ctx, char* buf, uint64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* CKMPM_B200_H_ */
