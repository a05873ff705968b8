// ckmpm_b200/simulation.hpp — C++ drop-in for ckmpm::Simulation<T> backed by
// the B200 C ABI (include/ckmpm_b200.h, libckmpm_b200.so).
//
// Replace
//     ckmpm::Simulation<double> sim(cfg);
// with
//     ckmpm::b200::Simulation<double> sim(cfg);
// and keep the rest of the caller: the public surface mirrors the reference
// (proj/include/ckmpm/simulation.hpp:85-219) and the reference's own types
// (SimConfig, Particle, Material, BoundaryCondition, PhaseTimers,
// TransferCounters, DiagnosticsRow, the exception taxonomy) are used as-is.
// The reference headers must be on the include path (the caller already has
// them); seeding, config validation and diagnostics reuse the reference's
// functions, only the substep runs on the GPU.
//
// Host/device ownership: the device state is authoritative; the
// host vector returned by particles() is refreshed lazily.  The non-const
// particles() accessor hands out a writable vector and marks it
// authoritative, so the next step() re-uploads it (the reference's tests write
// through it, tests/test_sim.cpp:415).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ckmpm/errors.hpp"
#include "ckmpm/scene.hpp"
#include "ckmpm/simulation.hpp"
#include "ckmpm/transfer.hpp"
#include "../ckmpm_b200.h"

namespace ckmpm {
namespace b200 {

template <typename T>
struct ParticleLayout;
template <>
struct ParticleLayout<double> {
  using type = ckg_particle_f64;
  static constexpr int precision = 8;
};
template <>
struct ParticleLayout<float> {
  using type = ckg_particle_f32;
  static constexpr int precision = 4;
};

static_assert(sizeof(Particle<double>) == sizeof(ckg_particle_f64), "Particle<double> ABI layout");
static_assert(sizeof(Particle<float>) == sizeof(ckg_particle_f32), "Particle<float> ABI layout");

// Read side of BlockSparseGrid<T> (grid.hpp:75-281) over the device grid.
class GridFacade {
 public:
  explicit GridFacade(ckg_ctx* ctx) : ctx_(ctx) {}
  std::size_t active_block_count() const { return std::size_t(ckg_grid_active_block_count(ctx_)); }
  double total_mass(int slot) const {
    double m[2], p[6];
    check(ckg_grid_totals(ctx_, m, p));
    return m[slot];
  }
  Vec3<double> total_momentum(int slot) const {
    double m[2], p[6];
    check(ckg_grid_totals(ctx_, m, p));
    return {p[slot * 3], p[slot * 3 + 1], p[slot * 3 + 2]};
  }

 private:
  static void check(int32_t rc) {
    if (rc != CKG_OK) throw NumericalError("b200 grid facade: device error");
  }
  ckg_ctx* ctx_;
};

template <typename T>
class Simulation {
 public:
  explicit Simulation(SimConfig<T> cfg, int device = 0) : cfg_(std::move(cfg)) {
    validate_config(cfg_);  // scene.hpp:184-200
    host_ = seed_particles(cfg_);  // scene.hpp:204-230
    mass_eps_ = compute_mass_epsilon(host_);
    min_j_.assign(cfg_.materials.size(), T(1));
    ckg_config c = to_abi(device);
    int32_t rc = ckg_create(&c, &ctx_);
    if (rc != CKG_OK) throw ConfigError("ckg_create failed (" + std::to_string(rc) + ")");
    upload();
    refresh_velocity_stats();
  }
  ~Simulation() {
    if (ctx_) ckg_destroy(ctx_);
  }
  Simulation(const Simulation&) = delete;
  Simulation& operator=(const Simulation&) = delete;

  const SimConfig<T>& config() const { return cfg_; }
  GridFacade grid() const { return GridFacade(ctx_); }

  // Non-const access: the caller may write; the next step re-uploads.
  std::vector<Particle<T>>& particles() {
    sync_host();
    host_dirty_ = true;
    return host_;
  }
  std::span<const Particle<T>> particles() const {
    const_cast<Simulation*>(this)->sync_host();
    return host_;
  }
  T time() const { return time_; }
  std::uint64_t step_count() const { return step_count_; }
  int frame_index() const { return frame_index_; }
  T mass_epsilon() const { return mass_eps_; }
  const TransferCounters& counters() const { return counters_; }
  void reset_counters() { counters_ = {}; }
  const PhaseTimers& timers() const { return timers_; }
  void reset_timers() { timers_ = {}; }

  // simulation.hpp:120-129
  void restore(std::vector<Particle<T>> particles, T time, std::uint64_t step, int frame, T mass_eps) {
    host_ = std::move(particles);
    time_ = time;
    step_count_ = step;
    frame_index_ = frame;
    mass_eps_ = mass_eps;
    ckg_set_mass_epsilon(ctx_, double(mass_eps_));
    min_j_.assign(cfg_.materials.size(), T(1));
    upload();
    refresh_velocity_stats();
  }

  // simulation.hpp:134-145
  T cfl_dt(T remaining) const {
    T cmax = 0;
    for (std::size_t mi = 0; mi < cfg_.materials.size(); ++mi) {
      const Material<T>& m = cfg_.materials[mi];
      T c = m.is_fluid() ? sound_speed_fluid(m, min_j_[mi]) : sound_speed_solid(m);
      cmax = std::max(cmax, c);
    }
    T denom = std::max(vmax_, cmax);
    T dt = denom > T(0) ? cfg_.cfl * cfg_.dx() / denom : remaining;
    if (cfg_.max_dt > T(0)) dt = std::min(dt, cfg_.max_dt);
    return std::min(dt, remaining);
  }

  // simulation.hpp:150-188, on the device.
  void step(T dt) {
    if (host_dirty_) upload();
    ckg_step_out out{};
    int32_t rc = ckg_step(ctx_, double(dt), &out);
    if (rc != CKG_OK) throw_for(rc, out);
    absorb(out);
    time_ += dt;
    ++step_count_;
    host_valid_ = false;
  }

  // simulation.hpp:193-211
  template <typename Cb>
  void advance_frame(Cb&& cb) {
    T frame_end = cfg_.frame_dt * T(frame_index_ + 1);
    std::uint64_t steps_this_frame = 0;
    for (;;) {
      T rem = frame_end - time_;
      if (rem <= cfg_.frame_dt * T(1e-9)) {
        time_ = frame_end;
        break;
      }
      T dt = cfl_dt(rem);
      step(dt);
      cb(*this, dt);
      if (++steps_this_frame > cfg_.max_substeps_per_frame)
        throw NumericalError("substep limit exceeded within one frame at t = " +
                             std::to_string(static_cast<double>(time_)));
    }
    ++frame_index_;
  }
  // Without a per-substep callback the whole frame runs on the device
  // (ckg_advance_frame: one CUDA-graph launch, cfl_dt and the frame-boundary
  // test evaluated on the GPU, no host round trip per substep).
  void advance_frame() {
    if (host_dirty_) upload();
    ckg_frame_in in{};
    in.time = double(time_);
    in.frame_dt = double(cfg_.frame_dt);
    in.frame_index = std::uint64_t(frame_index_);
    in.cfl = double(cfg_.cfl);
    in.max_dt = double(cfg_.max_dt);
    in.max_substeps = std::uint64_t(cfg_.max_substeps_per_frame);
    in.vmax = double(vmax_);
    for (int m = 0; m < CKG_MAX_MATERIALS; ++m)
      in.min_j[m] = m < int(min_j_.size()) ? double(min_j_[m]) : 1.0;
    ckg_frame_out out{};
    const int32_t rc = ckg_advance_frame(ctx_, &in, &out);
    // completed substeps are kept also when a later one failed (as the
    // reference, whose state advances substep by substep)
    time_ = T(out.time);
    step_count_ += out.substeps;
    vmax_ = T(out.vmax);
    for (std::size_t m = 0; m < min_j_.size(); ++m) min_j_[m] = T(out.min_j[m]);
    timers_.substeps += out.substeps;
    // node visits per particle (transfer.hpp:32-45): compact 2 x 8 (MLS
    // scatters twice), quadratic baseline 27
    const bool quad = cfg_.kernel == KernelKind::quadratic;
    const std::uint64_t per = quad ? 27 : cfg_.scheme == TransferScheme::mls ? 32 : 16;
    counters_.p2g_node_visits += per * host_.size() * out.substeps;
    counters_.g2p_node_visits += (quad ? 27 : 16) * host_.size() * out.substeps;
    counters_.p2g_transfers += host_.size() * out.substeps;
    counters_.g2p_transfers += host_.size() * out.substeps;
    if (out.substeps) host_valid_ = false;
    if (rc != CKG_OK) {
      ckg_step_out so{};
      so.error_code = out.error_code;
      so.error_particle = out.error_particle;
      throw_for(rc, so);
    }
    ++frame_index_;
  }

  // Device-packed checkpoint / snapshot bodies (ckg_pack_records): the file
  // body of the reference's CKCHKPT1 / CKSNAP1 writers, one record per
  // particle in the current order (include/ckmpm_b200/io.hpp writes the files).
  std::size_t record_bytes(int kind) const { return std::size_t(ckg_record_bytes(ctx_, kind)); }
  void pack_records(int kind, void* buf, std::size_t bytes, bool async = false) const {
    if (host_dirty_) const_cast<Simulation*>(this)->upload();
    const int32_t rc = ckg_pack_records(ctx_, kind, buf, bytes, async ? 1 : 0);
    if (rc != CKG_OK) const_cast<Simulation*>(this)->throw_for(rc, ckg_step_out{});
  }
  void records_wait() const { ckg_records_wait(ctx_); }
  std::size_t particle_count() const { return host_.size(); }

  // B200 extension: the same row reduced on the device (no particle download;
  // summation order differs from the serial host loop at round-off).
  DiagnosticsRow<T> device_diagnostics() const {
    ckg_diagnostics d{};
    if (host_dirty_) const_cast<Simulation*>(this)->upload();
    if (ckg_diagnostics_compute(ctx_, &d) != CKG_OK) throw NumericalError("ckg_diagnostics_compute failed");
    DiagnosticsRow<T> r;
    r.step = step_count_;
    r.time = time_;
    for (int a = 0; a < 3; ++a) {
      r.momentum[a] = T(d.momentum[a]);
      r.angular[a] = T(d.angular[a]);
      r.momentum_massfree[a] = T(d.momentum_massfree[a]);
    }
    r.kinetic_energy = T(d.kinetic_energy);
    r.vmax = T(d.vmax);
    return r;
  }

  // simulation.hpp:213-215 — the reference's own reduction on the synced host copy.
  DiagnosticsRow<T> diagnostics() const {
    const_cast<Simulation*>(this)->sync_host();
    return compute_diagnostics<T>(host_, step_count_, time_);
  }

 private:
  using Raw = typename ParticleLayout<T>::type;

  static T compute_mass_epsilon(const std::vector<Particle<T>>& ps) {  // simulation.hpp:227-232
    std::vector<T> masses(ps.size());
    for (std::size_t i = 0; i < ps.size(); ++i) masses[i] = ps[i].mass;
    std::nth_element(masses.begin(), masses.begin() + masses.size() / 2, masses.end());
    return T(1e-12) * masses[masses.size() / 2];
  }

  ckg_config to_abi(int device) const {
    ckg_config c{};
    c.abi_version = CKG_ABI_VERSION;
    c.precision = ParticleLayout<T>::precision;
    c.resolution = cfg_.resolution;
    c.scheme = static_cast<int32_t>(cfg_.scheme);
    c.extent = double(cfg_.extent);
    const T dx = cfg_.dx();
    c.dx = double(dx);
    c.inv_dx = double(T(1) / dx);
    for (int a = 0; a < 3; ++a) c.gravity[a] = double(cfg_.gravity[a]);
    c.mass_eps = double(mass_eps_);
    c.clamp_singular = cfg_.clamp_singular ? 1 : 0;
    c.deterministic = cfg_.deterministic ? 1 : 0;
    c.clamp_floor = double(cfg_.clamp_floor);
    if (cfg_.materials.size() > CKG_MAX_MATERIALS) throw ConfigError("materials: too many for the device table");
    if (cfg_.boundaries.size() > CKG_MAX_BOUNDARIES) throw ConfigError("boundaries: too many");
    c.n_materials = int32_t(cfg_.materials.size());
    for (std::size_t i = 0; i < cfg_.materials.size(); ++i) {
      const Material<T>& m = cfg_.materials[i];
      ckg_material& d = c.materials[i];
      d.model = static_cast<int32_t>(m.model);
      d.density = double(m.density);
      d.E = double(m.E);
      d.nu = double(m.nu);
      d.mu = double(m.mu);
      d.lambda = double(m.lambda);
      d.bulk = double(m.bulk);
      d.gamma = double(m.gamma);
      d.viscosity = double(m.viscosity);
      d.friction_angle_deg = double(m.friction_angle_deg);
      d.dp_alpha = double(m.dp_alpha);
    }
    c.n_boundaries = int32_t(cfg_.boundaries.size());
    for (std::size_t i = 0; i < cfg_.boundaries.size(); ++i) {
      const BoundaryCondition<T>& b = cfg_.boundaries[i];
      ckg_boundary& d = c.boundaries[i];
      d.kind = static_cast<int32_t>(b.kind);
      for (int a = 0; a < 3; ++a) {
        d.lo[a] = double(b.lo[a]);
        d.hi[a] = double(b.hi[a]);
        d.normal[a] = double(b.normal[a]);
        d.velocity[a] = double(b.velocity[a]);
        d.omega[a] = double(b.omega[a]);
        d.center[a] = double(b.center[a]);
      }
    }
    c.flags = cfg_.kernel == KernelKind::quadratic ? CKG_FLAG_QUADRATIC : 0;
    c.device = device;
    return c;
  }

  void upload() {
    int32_t rc = ckg_upload(ctx_, host_.data(), host_.size());
    if (rc != CKG_OK) throw NumericalError("ckg_upload failed (" + std::to_string(rc) + ")");
    host_dirty_ = false;
    host_valid_ = true;
  }

  void sync_host() {
    if (host_valid_ || host_dirty_) return;
    int32_t rc = ckg_download(ctx_, host_.data(), host_.size());
    if (rc != CKG_OK) throw NumericalError("ckg_download failed (" + std::to_string(rc) + ")");
    host_valid_ = true;
  }

  void refresh_velocity_stats() {  // simulation.hpp:234-243
    T vm = 0;
    for (const Particle<T>& p : host_) vm = std::max(vm, norm(p.v));
    vmax_ = vm;
    for (const Particle<T>& p : host_) {
      const Material<T>& m = cfg_.materials[p.material];
      if (m.is_fluid()) min_j_[p.material] = std::min(min_j_[p.material], p.J);
    }
  }

  void absorb(const ckg_step_out& out) {
    vmax_ = T(out.vmax);
    for (std::size_t m = 0; m < min_j_.size(); ++m) min_j_[m] = T(out.min_j[m]);
    timers_.sort_s += out.phase_ms[0] * 1e-3;
    timers_.activate_s += out.phase_ms[1] * 1e-3;
    timers_.clear_s += out.phase_ms[2] * 1e-3;
    timers_.p2g_s += out.phase_ms[3] * 1e-3;
    timers_.grid_s += out.phase_ms[4] * 1e-3;
    timers_.g2p_s += out.phase_ms[5] * 1e-3;
    timers_.substeps += 1;
    counters_.p2g_node_visits += out.p2g_node_visits;
    counters_.g2p_node_visits += out.g2p_node_visits;
    counters_.p2g_transfers += out.p2g_transfers;
    counters_.g2p_transfers += out.g2p_transfers;
  }

  [[noreturn]] void throw_for(int32_t rc, const ckg_step_out& out) {
    char buf[512];
    ckg_last_error_message(ctx_, buf, sizeof buf);
    const std::string msg(buf);
    if (rc == CKG_ERR_CONFIG) throw ConfigError(msg);
    if (rc == CKG_ERR_NUMERICAL) {
      switch (out.error_code) {
        case CKG_NUM_OUT_OF_DOMAIN:
          throw OutOfDomainError(std::size_t(out.error_particle), msg);
        case CKG_NUM_FC_STRESS_INVERTED:
        case CKG_NUM_DP_STRESS_INVERTED:
        case CKG_NUM_RETURN_MAP_INVERTED:
        case CKG_NUM_F_INVERTED:
          throw InvertedElementError(msg);
        default:
          throw NumericalError(msg);
      }
    }
    if (rc == CKG_ERR_IO) throw IoError(msg);
    throw std::runtime_error("B200 device error: " + msg);
  }

  SimConfig<T> cfg_;
  ckg_ctx* ctx_ = nullptr;
  std::vector<Particle<T>> host_;
  bool host_valid_ = true;
  bool host_dirty_ = false;
  std::vector<T> min_j_;
  T time_ = 0;
  std::uint64_t step_count_ = 0;
  int frame_index_ = 0;
  T mass_eps_ = 0;
  T vmax_ = 0;
  TransferCounters counters_;
  PhaseTimers timers_;
};

}  // namespace b200
}  // namespace ckmpm
