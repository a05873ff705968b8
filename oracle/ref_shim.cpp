// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Compiles the UNMODIFIED reference CK-MPM engine headers from
// /root/reference/proj/include (never copied into this repo) with the
// reference's own Release flags (proj/CMakeLists.txt:8-23: -O3 -DNDEBUG
// -fno-math-errno, no -march) and exposes them through the extern "C"
// surface declared in oracle/ckref.h.  Built by oracle/Makefile into
// oracle/_ref/libckref.so.
//
// Private members of ckmpm::Simulation (sort_particles, scatter_all, keys_)
// are reached by compiling the reference headers with `private` re-spelled
// as `public`: this only changes access checking, not code generation, so
// the arithmetic exercised here is byte-for-byte the reference's.

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <numbers>
#include <optional>
#include <ostream>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#define private public
#include "ckmpm/errors.hpp"
#include "ckmpm/grid.hpp"
#include "ckmpm/kernel.hpp"
#include "ckmpm/material.hpp"
#include "ckmpm/math.hpp"
#include "ckmpm/parallel.hpp"
#include "ckmpm/scene.hpp"
#include "ckmpm/simulation.hpp"
#include "ckmpm/transfer.hpp"
#undef private
#if __has_include(<json.hpp>)
#include "ckmpm/io.hpp"  // writers only (public API); needs nlohmann/json on the include path
#define CKREF_HAVE_IO 1
#endif

#include "ckref.h"

using namespace ckmpm;

namespace {

void put_err(char* err, int32_t cap, const std::string& s) {
  if (!err || cap <= 0) return;
  std::size_t k = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
  std::memcpy(err, s.data(), k);
  err[k] = '\0';
}

int32_t classify(const std::exception& e) {
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const NumericalError*>(&e)) return 3;
  if (dynamic_cast<const IoError*>(&e)) return 4;
  return 1;
}

template <typename T>
Vec3<T> v3(const double* a) {
  return {T(a[0]), T(a[1]), T(a[2])};
}

template <typename T>
Material<T> to_material(const ckg_material& m) {
  Material<T> r;
  r.model = static_cast<MaterialModel>(m.model);
  r.density = T(m.density);
  r.E = T(m.E);
  r.nu = T(m.nu);
  r.mu = T(m.mu);
  r.lambda = T(m.lambda);
  r.bulk = T(m.bulk);
  r.gamma = T(m.gamma);
  r.viscosity = T(m.viscosity);
  r.friction_angle_deg = T(m.friction_angle_deg);
  r.dp_alpha = T(m.dp_alpha);
  return r;
}

template <typename T>
BoundaryCondition<T> to_bc(const ckg_boundary& b) {
  BoundaryCondition<T> r;
  r.kind = static_cast<BcKind>(b.kind);
  r.lo = v3<T>(b.lo);
  r.hi = v3<T>(b.hi);
  r.normal = v3<T>(b.normal);
  r.velocity = v3<T>(b.velocity);
  r.omega = v3<T>(b.omega);
  r.center = v3<T>(b.center);
  return r;
}

template <typename T>
BodySpec<T> to_body(const ckref_body& b) {
  BodySpec<T> r;
  r.shape.kind = static_cast<ShapeKind>(b.kind);
  r.shape.center = v3<T>(b.center);
  r.shape.radius = T(b.radius);
  r.shape.inner_radius = T(b.inner_radius);
  r.shape.half_length = T(b.half_length);
  r.shape.axis = b.axis;
  r.shape.lo = v3<T>(b.lo);
  r.shape.hi = v3<T>(b.hi);
  r.material = b.material;
  r.ppc = b.ppc;
  r.seed = b.seed;
  r.velocity = v3<T>(b.velocity);
  r.shear_slope = T(b.shear_slope);
  r.omega = v3<T>(b.omega);
  return r;
}

// Resizes the reference's process-wide pool ahead of the Simulation ctor
// (which resizes it only when the count differs, simulation.hpp:94-99).
// Workaround for a reference-side race: ThreadPool::set_thread_count
// (parallel.hpp:30-37) starts new workers with seen = 0 while generation_
// keeps its old value, so after any earlier parallel loop each new worker
// wakes at once, calls the cleared job_ (std::bad_function_call, stored in
// worker_ex_) and decrements pending_; the next for_range then rethrows it.
// Tests that alternate thread counts in one process hit it.  Here the
// spurious wake-ups are let to finish, then one no-op loop resets pending_
// and drains the stored exception.
inline void prepare_pool(int threads) {
  int want = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  if (want < 1) want = 1;
  ThreadPool& pool = ThreadPool::instance();
  if (pool.thread_count() == want) return;
  pool.set_thread_count(want);
  if (want == 1) return;
  std::this_thread::sleep_for(std::chrono::milliseconds(50));
  try {
    pool.for_range(std::size_t(want), [](std::size_t, std::size_t, int) {});
  } catch (const std::bad_function_call&) {
  }
}

// Materials are taken as given (already finalized by the caller); the
// config-level validation of the reference still runs in the Simulation ctor.
template <typename T>
SimConfig<T> to_config(const ckg_config& c, const ckref_extra* ex) {
  SimConfig<T> cfg;
  cfg.resolution = c.resolution;
  cfg.extent = T(c.extent);
  cfg.kernel = (c.flags & CKG_FLAG_QUADRATIC) ? KernelKind::quadratic : KernelKind::compact;
  cfg.scheme = static_cast<TransferScheme>(c.scheme);
  cfg.gravity = v3<T>(c.gravity);
  cfg.deterministic = c.deterministic != 0;
  cfg.clamp_singular = c.clamp_singular != 0;
  cfg.clamp_floor = T(c.clamp_floor);
  if (ex) {
    cfg.cfl = T(ex->cfl);
    cfg.frame_dt = T(ex->frame_dt);
    cfg.max_dt = T(ex->max_dt);
    cfg.threads = ex->threads;
  }
  for (int i = 0; i < c.n_materials; ++i) cfg.materials.push_back(to_material<T>(c.materials[i]));
  for (int i = 0; i < c.n_boundaries; ++i) cfg.boundaries.push_back(to_bc<T>(c.boundaries[i]));
  prepare_pool(cfg.threads);
  return cfg;
}

template <typename T>
struct PLayout;
template <>
struct PLayout<double> {
  using type = ckg_particle_f64;
};
template <>
struct PLayout<float> {
  using type = ckg_particle_f32;
};

static_assert(sizeof(Particle<double>) == sizeof(ckg_particle_f64));
static_assert(sizeof(Particle<float>) == sizeof(ckg_particle_f32));
static_assert(offsetof(Particle<double>, material) == offsetof(ckg_particle_f64, material));
static_assert(offsetof(Particle<float>, material) == offsetof(ckg_particle_f32, material));

template <typename T>
std::vector<Particle<T>> from_raw(const void* raw, uint64_t n) {
  std::vector<Particle<T>> ps(n);
  if (n) std::memcpy(ps.data(), raw, n * sizeof(Particle<T>));
  return ps;
}

struct SimBase {
  int precision;
  virtual ~SimBase() = default;
};

template <typename T>
struct SimBox : SimBase {
  std::optional<Simulation<T>> sim;
};

// Simulation ctor needs at least one body; it is seeded and then replaced by
// restore().  A one-cell box inside the inset keeps that cheap.
template <typename T>
SimConfig<T> with_dummy_body(SimConfig<T> cfg) {
  BodySpec<T> b;
  b.shape.kind = ShapeKind::box;
  T dx = cfg.dx();
  b.shape.lo = {T(4) * dx, T(4) * dx, T(4) * dx};
  b.shape.hi = {T(5) * dx, T(5) * dx, T(5) * dx};
  b.material = 0;
  b.ppc = 8;
  cfg.bodies = {b};
  return cfg;
}

template <typename T>
SimBox<T>* as(void* s) {
  return static_cast<SimBox<T>*>(s);
}

template <typename T>
void grid_out(const BlockSparseGrid<T>& g, int32_t* coords, double* nodes, uint64_t nb) {
  auto blocks = g.blocks();
  uint64_t k = std::min<uint64_t>(nb, blocks.size());
  for (uint64_t b = 0; b < k; ++b) {
    if (coords) {
      coords[3 * b + 0] = blocks[b].coord.x;
      coords[3 * b + 1] = blocks[b].coord.y;
      coords[3 * b + 2] = blocks[b].coord.z;
    }
    if (nodes)
      for (int n = 0; n < 128; ++n) {
        const auto& nd = blocks[b].nodes[n];
        double* o = nodes + (b * 128 + n) * 4;
        o[0] = double(nd.mass);
        o[1] = double(nd.p.x);
        o[2] = double(nd.p.y);
        o[3] = double(nd.p.z);
      }
  }
}

template <typename T>
int64_t p2g_impl(const ckg_config* cfg, const void* particles, uint64_t n, double dt,
                 int32_t* coords, double* nodes, uint64_t nb, char* err, int32_t cap) {
  ckref_extra ex{0.5, 1.0 / 60.0, 0.0, 1, 0};
  SimConfig<T> c = with_dummy_body(to_config<T>(*cfg, &ex));
  c.deterministic = true;
  Simulation<T> sim(c);
  sim.restore(from_raw<T>(particles, n), T(0), 0, 0, T(cfg->mass_eps));
  try {
    sim.sort_particles();
    sim.positions_.resize(n);
    for (std::size_t i = 0; i < n; ++i) sim.positions_[i] = sim.particles_[i].x;
    sim.grid_->activate(sim.positions_);
    sim.grid_->clear();
    sim.scatter_all(T(dt));
  } catch (const std::exception& e) {
    put_err(err, cap, e.what());
    return -classify(e);
  }
  grid_out(*sim.grid_, coords, nodes, nb);
  return static_cast<int64_t>(sim.grid_->active_block_count());
}

}  // namespace

extern "C" {

int32_t ckref_finalize_material(ckg_material* m, int32_t precision, char* err, int32_t cap) {
  try {
    if (precision == 4) {
      Material<float> r = to_material<float>(*m);
      finalize_material(r);
      m->mu = r.mu;
      m->lambda = r.lambda;
      m->dp_alpha = r.dp_alpha;
    } else {
      Material<double> r = to_material<double>(*m);
      finalize_material(r);
      m->mu = r.mu;
      m->lambda = r.lambda;
      m->dp_alpha = r.dp_alpha;
    }
  } catch (const std::exception& e) {
    put_err(err, cap, e.what());
    return classify(e);
  }
  return 0;
}

int64_t ckref_seed(const ckg_config* cfg, const ckref_body* bodies, int32_t nbodies, void* out,
                   int64_t cap) {
  auto run = [&](auto tag) -> int64_t {
    using T = decltype(tag);
    SimConfig<T> c = to_config<T>(*cfg, nullptr);
    for (int i = 0; i < nbodies; ++i) c.bodies.push_back(to_body<T>(bodies[i]));
    std::vector<Particle<T>> ps = seed_particles(c);
    int64_t k = std::min<int64_t>(cap, static_cast<int64_t>(ps.size()));
    if (out && k > 0) std::memcpy(out, ps.data(), static_cast<std::size_t>(k) * sizeof(Particle<T>));
    return static_cast<int64_t>(ps.size());
  };
  try {
    return cfg->precision == 4 ? run(float{}) : run(double{});
  } catch (const std::exception&) {
    return -1;
  }
}

void* ckref_sim_create(const ckg_config* cfg, const ckref_extra* extra, const void* particles,
                       uint64_t n, char* err, int32_t cap) {
  try {
    if (cfg->precision == 4) {
      auto* box = new SimBox<float>();
      box->precision = 4;
      box->sim.emplace(with_dummy_body(to_config<float>(*cfg, extra)));
      box->sim->restore(from_raw<float>(particles, n), 0.0f, 0, 0, float(cfg->mass_eps));
      return box;
    }
    auto* box = new SimBox<double>();
    box->precision = 8;
    box->sim.emplace(with_dummy_body(to_config<double>(*cfg, extra)));
    box->sim->restore(from_raw<double>(particles, n), 0.0, 0, 0, cfg->mass_eps);
    return box;
  } catch (const std::exception& e) {
    put_err(err, cap, e.what());
    return nullptr;
  }
}

void ckref_sim_destroy(void* s) { delete static_cast<SimBase*>(s); }

#define CKREF_DISPATCH(s, expr_f, expr_d) \
  (static_cast<SimBase*>(s)->precision == 4 ? (expr_f) : (expr_d))

int32_t ckref_sim_step(void* s, double dt, char* err, int32_t cap) {
  try {
    if (static_cast<SimBase*>(s)->precision == 4)
      as<float>(s)->sim->step(float(dt));
    else
      as<double>(s)->sim->step(dt);
  } catch (const std::exception& e) {
    put_err(err, cap, e.what());
    return classify(e);
  }
  return 0;
}

double ckref_sim_cfl_dt(void* s, double remaining) {
  return CKREF_DISPATCH(s, double(as<float>(s)->sim->cfl_dt(float(remaining))),
                        as<double>(s)->sim->cfl_dt(remaining));
}

uint64_t ckref_sim_count(void* s) {
  return CKREF_DISPATCH(s, as<float>(s)->sim->particles_.size(),
                        as<double>(s)->sim->particles_.size());
}

int32_t ckref_sim_particles(void* s, void* out, uint64_t n) {
  if (static_cast<SimBase*>(s)->precision == 4) {
    auto& ps = as<float>(s)->sim->particles_;
    if (n != ps.size()) return 2;
    std::memcpy(out, ps.data(), n * sizeof(Particle<float>));
  } else {
    auto& ps = as<double>(s)->sim->particles_;
    if (n != ps.size()) return 2;
    std::memcpy(out, ps.data(), n * sizeof(Particle<double>));
  }
  return 0;
}

void ckref_sim_timers(void* s, double* o) {
  const PhaseTimers& t = CKREF_DISPATCH(s, as<float>(s)->sim->timers(), as<double>(s)->sim->timers());
  o[0] = t.sort_s;
  o[1] = t.activate_s;
  o[2] = t.clear_s;
  o[3] = t.p2g_s;
  o[4] = t.grid_s;
  o[5] = t.g2p_s;
}

uint64_t ckref_sim_active_blocks(void* s) {
  return CKREF_DISPATCH(s, as<float>(s)->sim->grid().active_block_count(),
                        as<double>(s)->sim->grid().active_block_count());
}

int32_t ckref_sim_grid(void* s, int32_t* coords, double* nodes, uint64_t nb) {
  if (static_cast<SimBase*>(s)->precision == 4)
    grid_out(as<float>(s)->sim->grid(), coords, nodes, nb);
  else
    grid_out(as<double>(s)->sim->grid(), coords, nodes, nb);
  return 0;
}

void ckref_sim_diagnostics(void* s, ckg_diagnostics* out) {
  auto fill = [&](auto row) {
    for (int a = 0; a < 3; ++a) {
      out->momentum[a] = double(row.momentum[a]);
      out->angular[a] = double(row.angular[a]);
      out->momentum_massfree[a] = double(row.momentum_massfree[a]);
    }
    out->kinetic_energy = double(row.kinetic_energy);
    out->vmax = double(row.vmax);
  };
  if (static_cast<SimBase*>(s)->precision == 4)
    fill(as<float>(s)->sim->diagnostics());
  else
    fill(as<double>(s)->sim->diagnostics());
}

double ckref_sim_mass_epsilon(void* s) {
  return CKREF_DISPATCH(s, double(as<float>(s)->sim->mass_epsilon()),
                        as<double>(s)->sim->mass_epsilon());
}

int64_t ckref_p2g(const ckg_config* cfg, const void* particles, uint64_t n, double dt,
                  int32_t* coords, double* nodes, uint64_t nb, char* err, int32_t cap) {
  try {
    if (cfg->precision == 4)
      return p2g_impl<float>(cfg, particles, n, dt, coords, nodes, nb, err, cap);
    return p2g_impl<double>(cfg, particles, n, dt, coords, nodes, nb, err, cap);
  } catch (const std::exception& e) {
    put_err(err, cap, e.what());
    return -classify(e);
  }
}

// Stable-sort permutation and keys as the reference computes them: the
// particle's position in the pre-sort array is smuggled through volume0
// (sort_particles reads only x, simulation.hpp:248-274; restore's
// refresh_velocity_stats reads v, J and indexes the material table, so the
// material tag must stay a valid index).  Exact for n < 2^24 in float.
int32_t ckref_sort(const ckg_config* cfg, const void* particles, uint64_t n, uint32_t* keys,
                   uint32_t* order) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    ckref_extra ex{0.5, 1.0 / 60.0, 0.0, 1, 0};
    SimConfig<T> c = with_dummy_body(to_config<T>(*cfg, &ex));
    Simulation<T> sim(c);
    std::vector<Particle<T>> ps = from_raw<T>(particles, n);
    for (uint64_t i = 0; i < n; ++i) {
      ps[i].material = 0;
      ps[i].volume0 = static_cast<T>(i);
    }
    sim.restore(std::move(ps), T(0), 0, 0, T(cfg->mass_eps));
    sim.sort_particles();
    for (uint64_t i = 0; i < n; ++i) {
      uint32_t src = static_cast<uint32_t>(sim.particles_[i].volume0);
      order[i] = src;
      keys[i] = static_cast<uint32_t>(sim.keys_[src]);
    }
  };
  try {
    if (cfg->precision == 4)
      run(float{});
    else
      run(double{});
  } catch (const std::exception&) {
    return 3;
  }
  return 0;
}

double ckref_ck_weight_1d(double u) { return ck_weight_1d(u); }
double ckref_ck_grad_1d(double u) { return ck_grad_1d(u); }

void ckref_axis_pair(double x, int32_t k, double dx, int32_t* base, double* o) {
  AxisPair<double> p = axis_pair(x, k, dx);
  *base = p.base;
  o[0] = p.f;
  o[1] = p.w0;
  o[2] = p.w1;
  o[3] = p.g0;
  o[4] = p.g1;
}

static Mat3<double> m3(const double* a) {
  Mat3<double> m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = a[3 * i + j];
  return m;
}
static void m3out(const Mat3<double>& m, double* a) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[3 * i + j] = m[i][j];
}

void ckref_polar_rotation(const double* F, double* R) { m3out(polar_rotation(m3(F)), R); }

void ckref_svd3(const double* F, double* U, double* sigma, double* V) {
  Svd3<double> s = svd3(m3(F));
  m3out(s.U, U);
  m3out(s.V, V);
  sigma[0] = s.sigma[0];
  sigma[1] = s.sigma[1];
  sigma[2] = s.sigma[2];
}

int32_t ckref_return_map_dp(const double* F, double alpha, double mu, double lambda, double* out) {
  try {
    m3out(return_map_drucker_prager(m3(F), alpha, mu, lambda), out);
  } catch (const std::exception& e) {
    return classify(e);
  }
  return 0;
}

void ckref_force_matrix(const ckg_particle_f64* p, const ckg_material* m, double* A, char* err,
                        int32_t cap) {
  Particle<double> pp;
  std::memcpy(&pp, p, sizeof(pp));
  try {
    m3out(force_matrix(pp, to_material<double>(*m)), A);
    put_err(err, cap, "");
  } catch (const std::exception& e) {
    put_err(err, cap, e.what());
  }
}

}  // extern "C"

// The reference's own checkpoint / snapshot writers (io.hpp:344-430), for the
// byte-exact comparison of the device-packed files.  5 = built without io.hpp.
extern "C" int32_t ckref_sim_write_checkpoint(void* s, const char* path) {
#ifdef CKREF_HAVE_IO
  try {
    if (static_cast<SimBase*>(s)->precision == 4)
      write_checkpoint(path, *as<float>(s)->sim);
    else
      write_checkpoint(path, *as<double>(s)->sim);
  } catch (const std::exception&) {
    return 4;
  }
  return 0;
#else
  (void)s;
  (void)path;
  return 5;
#endif
}

extern "C" int32_t ckref_sim_write_snapshot(void* s, const char* path, int32_t frame, int32_t binary) {
#ifdef CKREF_HAVE_IO
  auto run = [&](auto& sim) {
    using T = std::decay_t<decltype(sim.time())>;
    std::span<const Particle<T>> ps = sim.particles();
    std::span<const Material<T>> mats(sim.config().materials);
    if (binary)
      write_snapshot_binary<T>(path, ps, mats, frame, sim.time(), sim.config().dx());
    else
      write_snapshot_text<T>(path, ps, mats, frame, sim.time(), sim.config().dx());
  };
  try {
    if (static_cast<SimBase*>(s)->precision == 4)
      run(*as<float>(s)->sim);
    else
      run(*as<double>(s)->sim);
  } catch (const std::exception&) {
    return 4;
  }
  return 0;
#else
  (void)s;
  (void)path;
  (void)frame;
  (void)binary;
  return 5;
#endif
}
