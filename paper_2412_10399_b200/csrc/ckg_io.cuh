// ckg_io.cuh — checkpoint / snapshot records packed on the device (SURVEY §8f
// rank 3).  The reference writes its files particle by particle from the host
// AoS (proj/include/ckmpm/io.hpp:344-430); here one kernel packs the records
// of the device SoA into the exact byte layout of the file body, so the host
// only prepends the header and writes the buffer (bit-identical files):
//   CKCHKPT1 (write_checkpoint, io.hpp:392-430): per particle 27 T fields
//     (x, v, F row-major, B row-major, J, mass, volume0) + u32 material;
//   CKSNAP1  (write_snapshot_binary, io.hpp:370-390): per particle 7 doubles
//     (x, v, J for fluids else det F) + u32 material.
#pragma once

#include <cstdint>

#include "ckg_kernels.cuh"

namespace ckg {

// det (math.hpp:130-134) with the reference's rounding (no FMA contraction).
template <typename T>
__device__ __forceinline__ T det_rn(const T (&F)[9]) {
  const T a = sub_rn(mul_rn(F[4], F[8]), mul_rn(F[5], F[7]));
  const T b = sub_rn(mul_rn(F[3], F[8]), mul_rn(F[5], F[6]));
  const T c = sub_rn(mul_rn(F[3], F[7]), mul_rn(F[4], F[6]));
  return add_rn(sub_rn(mul_rn(F[0], a), mul_rn(F[1], b)), mul_rn(F[2], c));
}

template <typename T>
__device__ __forceinline__ void put_words(uint32_t* w, T v) {
  uint32_t u[sizeof(T) / 4];
  memcpy(u, &v, sizeof(T));
#pragma unroll
  for (int k = 0; k < int(sizeof(T) / 4); ++k) w[k] = u[k];
}

template <typename T>
__host__ __device__ constexpr uint32_t checkpoint_words() {
  return uint32_t((kNumFields * sizeof(T) + 4) / 4);
}
constexpr uint32_t kSnapshotWords = 15;  // 7 doubles + u32

// kind 0: CKCHKPT1 records; kind 1: CKSNAP1 records.  fluid_mask bit m: material
// m is a J-fluid (Material::is_fluid, material.hpp:49).
template <typename T>
__global__ void pack_records_kernel(PState<T> s, int kind, uint32_t fluid_mask, uint32_t* __restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= s.n) return;
  const uint32_t mat = s.mat[i];
  if (kind == 0) {
    uint32_t* r = out + i * checkpoint_words<T>();
#pragma unroll 3
    for (int k = 0; k < kNumFields; ++k) put_words(r + k * (sizeof(T) / 4), s.f[uint64_t(k) * s.stride + i]);
    r[checkpoint_words<T>() - 1] = mat;
    return;
  }
  uint32_t* r = out + i * kSnapshotWords;
#pragma unroll
  for (int k = 0; k < 6; ++k) put_words(r + 2 * k, double(s.f[uint64_t(kX + k) * s.stride + i]));
  T vol;
  if (mat < 32 && ((fluid_mask >> mat) & 1u)) {
    vol = s.f[uint64_t(kJ) * s.stride + i];
  } else {
    T F[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) F[k] = s.f[uint64_t(kF + k) * s.stride + i];
    vol = det_rn(F);
  }
  put_words(r + 12, double(vol));
  r[14] = mat;
}

}  // namespace ckg
