// ckmpm_b200/io.hpp — the reference's checkpoint / snapshot files
// (proj/include/ckmpm/io.hpp:344-477) for the B200 drop-in Simulation.
//
// The reference writers take `const ckmpm::Simulation<T>&` and walk the host
// AoS; here the file body is packed on the device from the SoA state
// (ckg_pack_records, csrc/ckg_io.cuh) in the exact byte layout, and the host
// prepends the same header: the files are byte-identical to what the
// reference writes for the same state, and read_checkpoint restores exactly.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "ckmpm/errors.hpp"
#include "simulation.hpp"

namespace ckmpm::b200 {

namespace detail {
inline void g17(std::string& out, double v) {  // io.hpp:334-338
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  out += buf;
}
}  // namespace detail

// write_checkpoint (io.hpp:392-430): CKCHKPT1.
template <typename T>
inline void write_checkpoint(const std::string& path, const Simulation<T>& sim) {
  std::vector<char> body(sim.particle_count() * sim.record_bytes(CKG_RECORDS_CHECKPOINT));
  sim.pack_records(CKG_RECORDS_CHECKPOINT, body.data(), body.size());
  std::ofstream os(path, std::ios::binary);
  if (!os) throw IoError("cannot open checkpoint file for writing: " + path);
  const char magic[8] = {'C', 'K', 'C', 'H', 'K', 'P', 'T', '1'};
  os.write(magic, 8);
  std::uint32_t scalar = sizeof(T);
  std::uint64_t step = sim.step_count();
  std::int32_t frame = sim.frame_index();
  T time = sim.time(), eps = sim.mass_epsilon();
  std::uint64_t count = sim.particle_count();
  os.write(reinterpret_cast<const char*>(&scalar), 4);
  os.write(reinterpret_cast<const char*>(&step), 8);
  os.write(reinterpret_cast<const char*>(&frame), 4);
  os.write(reinterpret_cast<const char*>(&time), sizeof(T));
  os.write(reinterpret_cast<const char*>(&eps), sizeof(T));
  os.write(reinterpret_cast<const char*>(&count), 8);
  os.write(body.data(), std::streamsize(body.size()));
  if (!os) throw IoError("checkpoint write failed: " + path);
}

// read_checkpoint (io.hpp:432-477): the same checks and messages, then restore().
template <typename T>
inline void read_checkpoint(const std::string& path, Simulation<T>& sim) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw IoError("cannot open checkpoint file: " + path);
  char magic[8];
  is.read(magic, 8);
  const char want[8] = {'C', 'K', 'C', 'H', 'K', 'P', 'T', '1'};
  if (!is || std::memcmp(magic, want, 8) != 0) throw IoError("not a checkpoint file: " + path);
  std::uint32_t scalar = 0;
  is.read(reinterpret_cast<char*>(&scalar), 4);
  if (scalar != sizeof(T)) throw IoError("checkpoint scalar width mismatch in " + path);
  std::uint64_t step = 0, count = 0;
  std::int32_t frame = 0;
  T time = 0, eps = 0;
  is.read(reinterpret_cast<char*>(&step), 8);
  is.read(reinterpret_cast<char*>(&frame), 4);
  is.read(reinterpret_cast<char*>(&time), sizeof(T));
  is.read(reinterpret_cast<char*>(&eps), sizeof(T));
  is.read(reinterpret_cast<char*>(&count), 8);
  if (!is) throw IoError("truncated checkpoint header: " + path);
  std::vector<Particle<T>> particles(count);
  for (Particle<T>& p : particles) {
    T fields[27];
    std::uint32_t mid = 0;
    is.read(reinterpret_cast<char*>(fields), sizeof fields);
    is.read(reinterpret_cast<char*>(&mid), 4);
    if (!is) throw IoError("truncated checkpoint particle data: " + path);
    int k = 0;
    for (int a = 0; a < 3; ++a) p.x[a] = fields[k++];
    for (int a = 0; a < 3; ++a) p.v[a] = fields[k++];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) p.F[r][c] = fields[k++];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) p.B[r][c] = fields[k++];
    p.J = fields[k++];
    p.mass = fields[k++];
    p.volume0 = fields[k++];
    p.material = mid;
  }
  sim.restore(std::move(particles), time, step, int(frame), eps);
}

// write_snapshot_binary (io.hpp:370-390): CKSNAP1.
template <typename T>
inline void write_snapshot_binary(const std::string& path, const Simulation<T>& sim, int frame) {
  std::vector<char> body(sim.particle_count() * sim.record_bytes(CKG_RECORDS_SNAPSHOT));
  sim.pack_records(CKG_RECORDS_SNAPSHOT, body.data(), body.size());
  std::ofstream os(path, std::ios::binary);
  if (!os) throw IoError("cannot open snapshot file for writing: " + path);
  const char magic[8] = {'C', 'K', 'S', 'N', 'A', 'P', '1', '\0'};
  std::int64_t fr = frame, count = std::int64_t(sim.particle_count());
  double t = static_cast<double>(sim.time()), d = static_cast<double>(sim.config().dx());
  os.write(magic, 8);
  os.write(reinterpret_cast<const char*>(&fr), 8);
  os.write(reinterpret_cast<const char*>(&t), 8);
  os.write(reinterpret_cast<const char*>(&count), 8);
  os.write(reinterpret_cast<const char*>(&d), 8);
  os.write(body.data(), std::streamsize(body.size()));
  if (!os) throw IoError("snapshot write failed: " + path);
}

// write_snapshot_text (io.hpp:344-368), formatted from the device-packed records.
template <typename T>
inline void write_snapshot_text(const std::string& path, const Simulation<T>& sim, int frame) {
  const std::size_t n = sim.particle_count(), rb = sim.record_bytes(CKG_RECORDS_SNAPSHOT);
  std::vector<char> body(n * rb);
  sim.pack_records(CKG_RECORDS_SNAPSHOT, body.data(), body.size());
  std::ofstream os(path);
  if (!os) throw IoError("cannot open snapshot file for writing: " + path);
  std::string line;
  line += "# ckmpm-snapshot-v1\n";
  line += "frame " + std::to_string(frame) + "\n";
  line += "time ";
  detail::g17(line, static_cast<double>(sim.time()));
  line += "\ncount " + std::to_string(n) + "\n";
  line += "dx ";
  detail::g17(line, static_cast<double>(sim.config().dx()));
  line += "\n# x y z vx vy vz J_or_detF material_id\n";
  os << line;
  for (std::size_t i = 0; i < n; ++i) {
    double cols[7];
    std::uint32_t mid;
    std::memcpy(cols, body.data() + i * rb, sizeof cols);
    std::memcpy(&mid, body.data() + i * rb + sizeof cols, 4);
    line.clear();
    for (double c : cols) {
      detail::g17(line, c);
      line += ' ';
    }
    line += std::to_string(mid);
    line += '\n';
    os << line;
  }
  if (!os) throw IoError("snapshot write failed: " + path);
}

}  // namespace ckmpm::b200
