// dropin_test.cpp — the C++ drop-in (include/ckmpm_b200/simulation.hpp) used
// exactly like the reference's ckmpm::Simulation<T>, next to the reference
// engine itself (compiled from /root/reference/proj/include, unmodified).
// Built by `make dropin` in the build container; the binary travels to the
// GPU box and is run by tests/test_gpu_dropin.py.
//
//   dropin_test parity    reference vs B200, same scene, 30 substeps
//   dropin_test errors    reference exception types/messages through the drop-in
//   dropin_test rod       acceptance criterion 4 (tests/acceptance_main.cpp:244-270)
//   dropin_test spheres   acceptance criterion 3 at 128^3, PIC (tests/acceptance_main.cpp:214-238)
//   dropin_test stress    acceptance criterion 10 (tests/acceptance_main.cpp:530-562)
//   dropin_test io        CKCHKPT1 / CKSNAP1 files vs the reference's writers, restart
//   dropin_test jelly [dir [frames]]  acceptance criteria 8 + 9a (compact vs quadratic, jelly cube)
//   dropin_test contact [dir]  acceptance criterion 9b (contact gap, ball through a tube)
//
// Each prints one JSON line and exits 0 on PASS, 1 on FAIL.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ckmpm/grid.hpp"
#include "ckmpm/material.hpp"
#include "ckmpm/scene.hpp"
#include "ckmpm/simulation.hpp"
#include "ckmpm_b200/simulation.hpp"
#if __has_include(<json.hpp>)
#include "ckmpm/io.hpp"
#define DROPIN_HAVE_REF_IO 1
#endif
#include "ckmpm_b200/io.hpp"
#include <fstream>
#include <iterator>

using namespace ckmpm;
using Vec3d = Vec3<double>;
using P = Particle<double>;

namespace {

Material<double> fc(double rho, double E, double nu) {
  Material<double> m;
  m.model = MaterialModel::fixed_corotated;
  m.density = rho;
  m.E = E;
  m.nu = nu;
  finalize_material(m);
  return m;
}

BodySpec<double> box(Vec3d lo, Vec3d hi, Vec3d v = {}) {
  BodySpec<double> b;
  b.shape.kind = ShapeKind::box;
  b.shape.lo = lo;
  b.shape.hi = hi;
  b.velocity = v;
  return b;
}

BodySpec<double> sphere(Vec3d c, double r, Vec3d v = {}) {
  BodySpec<double> b;
  b.shape.kind = ShapeKind::sphere;
  b.shape.center = c;
  b.shape.radius = r;
  b.velocity = v;
  return b;
}

// The reference scene files, restated programmatically (io.hpp is not built).
SimConfig<double> rod_config() {  // configs/rotating_rod.json
  SimConfig<double> c;
  c.resolution = 128;
  c.scheme = TransferScheme::apic;
  c.frame_dt = 0.016666666666666666;
  c.frames = 300;
  c.materials = {fc(1000.0, 1e6, 0.4)};
  BodySpec<double> b;
  b.shape.kind = ShapeKind::cylinder;
  b.shape.center = {0.5, 0.5, 0.5};
  b.shape.radius = 0.01953125;
  b.shape.half_length = 0.078125;
  b.shape.axis = 1;
  b.shear_slope = 12.8;
  c.bodies = {b};
  return c;
}

SimConfig<double> spheres_config() {  // configs/two_spheres.json
  SimConfig<double> c;
  c.resolution = 128;
  c.scheme = TransferScheme::pic;
  c.frame_dt = 0.016666666666666666;
  c.frames = 300;
  c.materials = {fc(1000.0, 1e6, 0.4)};
  c.bodies = {sphere({0.125, 0.125, 0.125}, 0.078125, {0.05, 0.05, 0.05}),
              sphere({0.5, 0.5, 0.5}, 0.078125, {-0.05, -0.05, -0.05})};
  return c;
}

SimConfig<double> sand_config() {  // configs/sand_armadillos_reduced.json
  SimConfig<double> c;
  c.resolution = 64;
  c.scheme = TransferScheme::apic;
  c.gravity = {0, -2.0, 0};
  c.frame_dt = 0.016666666666666666;
  c.frames = 40;
  Material<double> m;
  m.model = MaterialModel::drucker_prager;
  m.density = 1400.0;
  m.E = 1e4;
  m.nu = 0.4;
  m.friction_angle_deg = 30.0;
  finalize_material(m);
  c.materials = {m};
  c.bodies = {sphere({0.5, 0.35, 0.3}, 0.09375, {0, 0, 0.5}), sphere({0.5, 0.35, 0.7}, 0.09375, {0, 0, -0.5})};
  BoundaryCondition<double> bc;
  bc.kind = BcKind::separate;
  bc.lo = {0, 0, 0};
  bc.hi = {1, 0.0625, 1};
  bc.normal = {0, 1, 0};
  c.boundaries = {bc};
  return c;
}

SimConfig<double> dam_config() {  // configs/dam_break_reduced.json
  SimConfig<double> c;
  c.resolution = 64;
  c.scheme = TransferScheme::apic;
  c.gravity = {0, -2.0, 0};
  c.frame_dt = 0.016666666666666666;
  c.frames = 30;
  Material<double> m;
  m.model = MaterialModel::j_fluid;
  m.density = 1000.0;
  m.bulk = 10.0;
  m.gamma = 7.15;
  m.viscosity = 0.1;
  finalize_material(m);
  c.materials = {m};
  c.bodies = {box({0.0625, 0.0625, 0.0625}, {0.21875, 0.375, 0.28125})};
  auto slip = [](Vec3d lo, Vec3d hi, Vec3d n) {
    BoundaryCondition<double> bc;
    bc.kind = BcKind::slip;
    bc.lo = lo;
    bc.hi = hi;
    bc.normal = n;
    return bc;
  };
  c.boundaries = {slip({0, 0, 0}, {1, 0.0625, 1}, {0, 1, 0}), slip({0, 0, 0}, {0.0625, 1, 1}, {1, 0, 0}),
                  slip({0.9375, 0, 0}, {1, 1, 1}, {1, 0, 0}), slip({0, 0, 0}, {1, 1, 0.0625}, {0, 0, 1}),
                  slip({0, 0, 0.9375}, {1, 1, 1}, {0, 0, 1})};
  return c;
}

Vec3d angular_about(std::span<const P> ps, const Vec3d& c) {  // acceptance_main.cpp:114-118
  Vec3d L{};
  for (const P& p : ps) L = L + (cross(p.x - c, p.v) + axial(p.B)) * p.mass;
  return L;
}

Vec3d mass_free_momentum(std::span<const P> ps) {
  Vec3d s{};
  for (const P& p : ps) s = s + p.v;
  return s;
}

int parity() {
  SimConfig<double> cfg;
  cfg.resolution = 32;
  cfg.scheme = TransferScheme::apic;
  cfg.gravity = {0, -9.8, 0};
  cfg.deterministic = true;
  cfg.threads = 1;
  cfg.materials = {fc(1000.0, 1e5, 0.4)};
  cfg.bodies = {box({0.375, 0.3125, 0.375}, {0.53125, 0.46875, 0.53125}, {0.3, 0.0, -0.2})};
  BoundaryCondition<double> bc;
  bc.lo = {0, 0, 0};
  bc.hi = {1, 0.25, 1};
  cfg.boundaries = {bc};
  Simulation<double> ref(cfg);
  b200::Simulation<double> gpu(cfg);
  double worst = 0.0;
  bool order_ok = true;
  for (int s = 0; s < 30; ++s) {
    double dt = ref.cfl_dt(1.0);
    double dtg = gpu.cfl_dt(1.0);
    worst = std::max(worst, std::abs(dt - dtg) / dt);
    ref.step(dt);
    gpu.step(dt);
  }
  auto a = ref.particles();
  auto b = gpu.particles();
  double xs = 0, vs = 0, fs = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    if (a[i].volume0 != b[i].volume0 || a[i].mass != b[i].mass) order_ok = false;
    for (int k = 0; k < 3; ++k) {
      xs = std::max(xs, std::abs(a[i].x[k] - b[i].x[k]));
      vs = std::max(vs, std::abs(a[i].v[k] - b[i].v[k]));
      for (int l = 0; l < 3; ++l) fs = std::max(fs, std::abs(a[i].F[k][l] - b[i].F[k][l]));
    }
  }
  DiagnosticsRow<double> da = ref.diagnostics(), db = gpu.diagnostics();
  double pdev = 0;
  for (int k = 0; k < 3; ++k) pdev = std::max(pdev, std::abs(da.momentum[k] - db.momentum[k]));
  bool pass = order_ok && worst < 1e-9 && xs < 1e-12 && vs < 1e-10 && fs < 1e-10 && pdev < 1e-12 &&
              gpu.timers().substeps == 30 && gpu.counters().p2g_node_visits == 30ull * 16 * a.size();
  std::printf(
      "{\"test\":\"parity\",\"pass\":%s,\"particles\":%zu,\"dt_rel\":%.3e,\"x_abs\":%.3e,\"v_abs\":%.3e,"
      "\"F_abs\":%.3e,\"momentum_abs\":%.3e,\"order_ok\":%s}\n",
      pass ? "true" : "false", a.size(), worst, xs, vs, fs, pdev, order_ok ? "true" : "false");
  return pass ? 0 : 1;
}

int errors() {
  SimConfig<double> cfg;
  cfg.resolution = 16;
  cfg.materials = {fc(1000.0, 1e5, 0.3)};
  cfg.bodies = {box({0.4, 0.4, 0.4}, {0.6, 0.6, 0.6})};
  bool ok = true;
  std::string got_ref, got_gpu;
  // out of domain: the reference error type, particle index and message
  {
    Simulation<double> ref(cfg);
    b200::Simulation<double> gpu(cfg);
    ref.particles()[7].x.x = 1.5 / 16;
    gpu.particles()[7].x.x = 1.5 / 16;
    std::size_t ir = 0, ig = 1;
    try { ref.step(1e-4); } catch (const OutOfDomainError& e) { got_ref = e.what(); ir = e.particle_index; }
    try { gpu.step(1e-4); } catch (const OutOfDomainError& e) { got_gpu = e.what(); ig = e.particle_index; }
    ok = ok && !got_ref.empty() && got_ref == got_gpu && ir == ig;
  }
  // inverted element
  {
    Simulation<double> ref(cfg);
    b200::Simulation<double> gpu(cfg);
    ref.particles()[3].F = Mat3<double>::diag(1, 1, -1);
    gpu.particles()[3].F = Mat3<double>::diag(1, 1, -1);
    std::string a, b;
    try { ref.step(1e-4); } catch (const InvertedElementError& e) { a = e.what(); }
    try { gpu.step(1e-4); } catch (const InvertedElementError& e) { b = e.what(); }
    ok = ok && !a.empty() && a == b;
  }
  std::printf("{\"test\":\"errors\",\"pass\":%s,\"message\":\"%s\"}\n", ok ? "true" : "false", got_gpu.c_str());
  return ok ? 0 : 1;
}

int rod() {
  SimConfig<double> cfg = rod_config();
  b200::Simulation<double> sim(cfg);
  const Vec3d center{0.5, 0.5, 0.5};
  Vec3d L0 = angular_about(sim.particles(), center);
  double lz0 = std::abs(L0.z);
  const double pinned = 4.9639e-3;
  bool pin_ok = std::abs(lz0 - pinned) <= 0.01 * pinned;
  double max_z = 0, max_xy = 0;
  for (int f = 0; f < cfg.frames; ++f) {
    sim.advance_frame([&](b200::Simulation<double>& s, double) {
      Vec3d L = angular_about(s.particles(), center);
      max_z = std::max(max_z, std::abs(L.z - L0.z));
      max_xy = std::max({max_xy, std::abs(L.x - L0.x), std::abs(L.y - L0.y)});
    });
  }
  // the reference's gate is z <= 1e-2, xy <= 1e-4; its own FP64 run measures
  // 3.72e-11 / 5.20e-11, so the device is held to 1e-9
  bool pass = pin_ok && max_z / lz0 <= 1e-9 && max_xy / lz0 <= 1e-9;
  std::printf(
      "{\"test\":\"rod\",\"pass\":%s,\"lz0\":%.6e,\"z_drift_rate\":%.3e,\"xy_leakage\":%.3e,\"substeps\":%llu,"
      "\"gate\":\"criterion 4 (pin 4.9639e-3 +-1%%, z<=1e-2, xy<=1e-4) tightened to the reference's measured level: "
      "z, xy <= 1e-9 (reference 3.72e-11 / 5.20e-11)\"}\n",
      pass ? "true" : "false", lz0, max_z / lz0, max_xy / lz0, (unsigned long long)sim.step_count());
  return pass ? 0 : 1;
}

int spheres() {
  SimConfig<double> cfg = spheres_config();
  b200::Simulation<double> sim(cfg);
  Vec3d sv0 = mass_free_momentum(sim.particles());
  const double norm = 2905.69;  // acceptance_main.cpp:216
  double max_err = 0;
  // every substep, like the reference gate; the sum is reduced on the device
  for (int f = 0; f < cfg.frames; ++f) {
    sim.advance_frame([&](b200::Simulation<double>& s, double) {
      Vec3d sv = s.device_diagnostics().momentum_massfree;
      max_err = std::max(max_err, norm_inf(sv - sv0) / norm);
    });
  }
  // reference gate 1e-4 (acceptance_main.cpp:231-238); held to 1e-9 here
  bool pass = max_err <= 1e-9;
  std::printf("{\"test\":\"spheres\",\"pass\":%s,\"drift_rate\":%.3e,\"substeps\":%llu,\"gate\":1e-9}\n",
              pass ? "true" : "false", max_err, (unsigned long long)sim.step_count());
  return pass ? 0 : 1;
}

int stress() {
  double devs[2] = {0, 0};
  bool finite = true;
  SimConfig<double> cfgs[2] = {dam_config(), sand_config()};
  for (int k = 0; k < 2; ++k) {
    b200::Simulation<double> sim(cfgs[k]);
    double total = 0;
    for (const P& p : sim.particles()) total += p.mass;
    for (int f = 0; f < cfgs[k].frames; ++f)
      sim.advance_frame([&](b200::Simulation<double>& s, double) {
        for (int slot = 0; slot < 2; ++slot)
          devs[k] = std::max(devs[k], std::abs(s.grid().total_mass(slot) - total) / total);
      });
    for (const P& p : sim.particles())
      for (int a = 0; a < 3; ++a) finite = finite && std::isfinite(p.x[a]) && std::isfinite(p.v[a]);
  }
  bool pass = finite && devs[0] <= 1e-8 && devs[1] <= 1e-8;
  std::printf("{\"test\":\"stress\",\"pass\":%s,\"dam_mass_dev\":%.3e,\"sand_mass_dev\":%.3e,\"finite\":%s}\n",
              pass ? "true" : "false", devs[0], devs[1], finite ? "true" : "false");
  return pass ? 0 : 1;
}

std::string slurp(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  return std::string(std::istreambuf_iterator<char>(is), std::istreambuf_iterator<char>());
}

// Checkpoint / snapshot files of the drop-in against the reference's own
// writers (io.hpp:344-430) on the same state, and a restart through
// read_checkpoint that continues exactly like the uninterrupted run.
int io() {
  SimConfig<double> cfg = sand_config();
  const std::string dir = "/tmp/ckmpm_b200_io_";
  ckmpm::b200::Simulation<double> gpu(cfg);
  bool same0 = true, snap_bin = true, snap_txt = true;
#ifdef DROPIN_HAVE_REF_IO
  Simulation<double> ref(cfg);
  ckmpm::write_checkpoint(dir + "ref.ckpt", ref);
  ckmpm::b200::write_checkpoint(dir + "gpu.ckpt", gpu);
  same0 = slurp(dir + "ref.ckpt") == slurp(dir + "gpu.ckpt");
  ckmpm::write_snapshot_binary<double>(dir + "ref.snap", ref.particles(), cfg.materials, 0, ref.time(), cfg.dx());
  ckmpm::b200::write_snapshot_binary(dir + "gpu.snap", gpu, 0);
  snap_bin = slurp(dir + "ref.snap") == slurp(dir + "gpu.snap");
  ckmpm::write_snapshot_text<double>(dir + "ref.txt", ref.particles(), cfg.materials, 0, ref.time(), cfg.dx());
  ckmpm::b200::write_snapshot_text(dir + "gpu.txt", gpu, 0);
  snap_txt = slurp(dir + "ref.txt") == slurp(dir + "gpu.txt");
#endif
  for (int k = 0; k < 10; ++k) gpu.step(gpu.cfl_dt(1.0));
  ckmpm::b200::write_checkpoint(dir + "gpu10.ckpt", gpu);
  ckmpm::b200::Simulation<double> restart(cfg);
  ckmpm::b200::read_checkpoint(dir + "gpu10.ckpt", restart);
  ckmpm::b200::write_checkpoint(dir + "restart10.ckpt", restart);
  const bool roundtrip = slurp(dir + "gpu10.ckpt") == slurp(dir + "restart10.ckpt");
  double dev0 = 0;
  {
    auto a0 = gpu.particles();
    auto b0 = restart.particles();
    for (std::size_t i = 0; i < a0.size(); ++i)
      for (int c = 0; c < 3; ++c) dev0 = std::max(dev0, std::fabs(a0[i].x[c] - b0[i].x[c]));
  }
  double dev = 0;
  for (int k = 0; k < 10; ++k) {
    const double dt = gpu.cfl_dt(1.0);
    if (dt != restart.cfl_dt(1.0)) dev = 1.0;
    gpu.step(dt);
    restart.step(dt);
  }
  auto a = gpu.particles();
  auto b = restart.particles();
  for (std::size_t i = 0; i < a.size(); ++i)
    for (int c = 0; c < 3; ++c) dev = std::max(dev, std::fabs(a[i].x[c] - b[i].x[c]));
  std::vector<double> xa, xb;
  for (std::size_t i = 0; i < a.size(); ++i) {
    xa.push_back(a[i].x[0]);
    xb.push_back(b[i].x[0]);
  }
  std::sort(xa.begin(), xa.end());
  std::sort(xb.begin(), xb.end());
  double dsort = 0;
  for (std::size_t i = 0; i < xa.size(); ++i) dsort = std::max(dsort, std::fabs(xa[i] - xb[i]));
  // after restore the state is identical by index (dev0 = 0); 10 substeps later
  // the P2G flush atomics' summation order may differ (as the reference's
  // atomic mode), and an ulp at a block face can swap two particles' sorted
  // positions, so the continued runs are compared as coordinate multisets
  const bool pass = same0 && snap_bin && snap_txt && roundtrip && dev0 == 0.0 && dsort <= 1e-12 &&
                    restart.step_count() == gpu.step_count() && restart.time() == gpu.time();
  std::fprintf(stderr, "io: dev0 %.3e dev %.3e sorted-x dev %.3e\n", dev0, dev, dsort);
  std::printf("{\"test\":\"io\",\"pass\":%s,\"checkpoint_bytes_equal\":%s,\"snapshot_binary_equal\":%s,"
              "\"snapshot_text_equal\":%s,\"restart_roundtrip\":%s,\"restart_dev0\":%.3e,\"restart_sorted_dx\":%.3e,"
              "\"particles\":%zu}\n",
              pass ? "true" : "false", same0 ? "true" : "false", snap_bin ? "true" : "false",
              snap_txt ? "true" : "false", roundtrip ? "true" : "false", dev0, dsort, a.size());
  return pass ? 0 : 1;
}

#ifdef DROPIN_HAVE_REF_IO
// Acceptance criteria 8 + 9a (tests/acceptance_main.cpp:419-471, :499-528):
// the jelly cube dropped on an identical substep schedule with the compact
// kernel, then the quadratic B-spline baseline replaying the compact run's
// dts.  The reference engine's own run of this scene inverts an element
// mid-run (profiles/r02_reference_acceptance_8_9.log), so the full 120-frame
// gates cannot be evaluated; the drop-in runs the first `frames` frames (the
// part the reference completes) next to the reference engine on the same
// schedule, and reports the transfer-phase speed-up (criterion 8, soft gate
// 1.2x) and both kernels' KE trajectories against the reference's.
int jelly(const std::string& dir, int frames) {
  SimConfig<double> cfg = load_config<double>(dir + "/jelly_cube.json");
  cfg.threads = 0;
  frames = std::min(frames, cfg.frames);
  b200::Simulation<double> compact(cfg);
  Simulation<double> ref_c(cfg);
  std::vector<double> dts;
  std::vector<std::size_t> ends;
  double ke_dev_c = 0, ke_max = 0;
  for (int f = 0; f < frames; ++f) {
    compact.advance_frame([&](b200::Simulation<double>&, double dt) { dts.push_back(dt); });
    ends.push_back(dts.size());
  }
  {
    std::size_t idx = 0;
    b200::Simulation<double> rerun(cfg);  // ke per frame on both engines, same schedule
    for (int f = 0; f < frames; ++f) {
      while (idx < ends[static_cast<std::size_t>(f)]) {
        ref_c.step(dts[idx]);
        rerun.step(dts[idx]);
        ++idx;
      }
      const double a = rerun.device_diagnostics().kinetic_energy, b = ref_c.diagnostics().kinetic_energy;
      ke_dev_c = std::max(ke_dev_c, std::abs(a - b));
      ke_max = std::max(ke_max, std::abs(b));
    }
  }
  SimConfig<double> qcfg = cfg;
  qcfg.kernel = KernelKind::quadratic;
  b200::Simulation<double> quad(qcfg);
  Simulation<double> ref_q(qcfg);
  double ke_dev_q = 0;
  std::size_t idx = 0;
  for (int f = 0; f < frames; ++f) {
    while (idx < ends[static_cast<std::size_t>(f)]) {
      quad.step(dts[idx]);
      ref_q.step(dts[idx]);
      ++idx;
    }
    ke_dev_q = std::max(ke_dev_q,
                        std::abs(quad.device_diagnostics().kinetic_energy - ref_q.diagnostics().kinetic_energy));
  }
  const double ct = compact.timers().transfer_total(), qt = quad.timers().transfer_total();
  const double speedup = ct > 0 ? qt / ct : 0.0;
  const double rc = ref_c.timers().transfer_total(), rq = ref_q.timers().transfer_total();
  const bool ok = ke_dev_c <= 1e-9 * ke_max && ke_dev_q <= 1e-9 * ke_max;
  std::printf("{\"test\":\"jelly\",\"pass\":%s,\"frames\":%d,\"substeps\":%zu,\"speedup\":%.3f,"
              "\"speedup_soft_gate_1_2\":%s,\"compact_transfer_s\":%.4f,\"quadratic_transfer_s\":%.4f,"
              "\"reference_speedup\":%.3f,\"ke_rel_dev_compact\":%.3e,\"ke_rel_dev_quadratic\":%.3e}\n",
              ok ? "true" : "false", frames, dts.size(), speedup, speedup >= 1.2 ? "true" : "false", ct, qt,
              rc > 0 ? rq / rc : 0.0, ke_max > 0 ? ke_dev_c / ke_max : 0.0, ke_max > 0 ? ke_dev_q / ke_max : 0.0);
  return ok ? 0 : 1;
}

// Acceptance criterion 9b (tests/acceptance_main.cpp:473-497): a ball falls
// through a tube whose bore clears it by 1.5 cells; the compact kernel lets
// it pass the tube midpoint, the quadratic baseline couples it to the wall.
double contact_ball_y(const std::string& dir, KernelKind kernel) {
  SimConfig<double> cfg = load_config<double>(dir + "/contact_cylinder.json");
  cfg.kernel = kernel;
  b200::Simulation<double> sim(cfg);
  for (int f = 0; f < cfg.frames; ++f) sim.advance_frame();
  Vec3d sum{};
  std::size_t count = 0;
  for (const P& p : sim.particles())
    if (p.material == 1u) {
      sum = sum + p.x;
      ++count;
    }
  if (count == 0) throw NumericalError("contact scene lost every ball particle");
  return sum.y / static_cast<double>(count);
}

// The same with the reference engine (no GPU needed): its own criterion-9b values.
double contact_ball_y_ref(const std::string& dir, KernelKind kernel) {
  SimConfig<double> cfg = load_config<double>(dir + "/contact_cylinder.json");
  cfg.kernel = kernel;
  cfg.threads = 0;
  Simulation<double> sim(cfg);
  for (int f = 0; f < cfg.frames; ++f) sim.advance_frame();
  Vec3d sum{};
  std::size_t count = 0;
  for (const P& p : sim.particles())
    if (p.material == 1u) {
      sum = sum + p.x;
      ++count;
    }
  return count ? sum.y / static_cast<double>(count) : 0.0;
}

int contact_ref(const std::string& dir) {
  const double yc = contact_ball_y_ref(dir, KernelKind::compact), yq = contact_ball_y_ref(dir, KernelKind::quadratic);
  const bool ok = yc < 0.5 && yq > 0.5;
  std::printf("{\"test\":\"contact_ref\",\"pass\":%s,\"ball_y_compact\":%.5f,\"ball_y_quadratic\":%.5f}\n",
              ok ? "true" : "false", yc, yq);
  return ok ? 0 : 1;
}

int contact(const std::string& dir) {
  const double yc = contact_ball_y(dir, KernelKind::compact), yq = contact_ball_y(dir, KernelKind::quadratic);
  const bool ok = yc < 0.5 && yq > 0.5;
  std::printf("{\"test\":\"contact\",\"pass\":%s,\"ball_y_compact\":%.5f,\"ball_y_quadratic\":%.5f}\n",
              ok ? "true" : "false", yc, yq);
  return ok ? 0 : 1;
}
#endif

}  // namespace

int main(int argc, char** argv) {
  std::string what = argc > 1 ? argv[1] : "parity";
  try {
    if (what == "parity") return parity();
    if (what == "errors") return errors();
    if (what == "rod") return rod();
    if (what == "spheres") return spheres();
    if (what == "stress") return stress();
    if (what == "io") return io();
#ifdef DROPIN_HAVE_REF_IO
    const std::string dir = argc > 2 ? argv[2] : "tests/golden/configs";
    if (what == "jelly") return jelly(dir, argc > 3 ? std::atoi(argv[3]) : 12);
    if (what == "contact") return contact(dir);
    if (what == "contact_ref") return contact_ref(dir);
#endif
  } catch (const std::exception& e) {
    std::printf("{\"test\":\"%s\",\"pass\":false,\"exception\":\"%s\"}\n", what.c_str(), e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown test %s\n", what.c_str());
  return 2;
}
