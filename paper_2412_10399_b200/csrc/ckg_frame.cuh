// ckg_frame.cuh — device-side frame driver.
//
// advance_frame (proj/include/ckmpm/simulation.hpp:193-211) as one CUDA graph
// launch: a conditional WHILE node runs substeps until the frame boundary, the
// step size cfl_dt(remaining) (:134-145) is computed on the device from the
// previous substep's gather_all reductions (:380-395), and the sort path
// (incremental merge vs full radix) is chosen by a device-set IF node, so no
// substep needs a host round trip.  Everything is evaluated in T with the
// reference's operation order and no FMA contraction, so the dt sequence is the
// host's bit for bit (std::pow of the fluid sound speed aside: CUDA's pow is
// within 2 ulp of the host's).
#pragma once

#include <cstdint>

#include "ckg_kernels.cuh"

namespace ckg {

// Frame state, device-resident for the duration of one advance_frame.
struct FrameState {
  double time, frame_end, frame_dt;  // T values
  double cfl, max_dt;
  double vmax;                      // vmax_ (T)
  double min_j[kMaxMaterials];      // min_j_ (T)
  double dt;                        // dt of the substep in flight / last completed
  unsigned int substeps, max_substeps;
  unsigned int status;              // 0 running, 1 frame done, 2 device error latched, 3 substep limit
  unsigned int parity;              // state buffer holding the current particles
  unsigned int sort_paths[3];       // substeps per sort path: one-CTA, padded radix, full radix
  // fixed-dt mode (ckg_step_many through the graph): every substep at
  // fixed_dt, until `target` substeps are done (no CFL, no frame boundary)
  double fixed_dt;
  unsigned int target;
};

template <typename T>
__device__ __forceinline__ T tmax(T a, T b) {  // std::max(a, b)
  return (a < b) ? b : a;
}
template <typename T>
__device__ __forceinline__ T tmin(T a, T b) {  // std::min(a, b)
  return (b < a) ? b : a;
}

__device__ __forceinline__ double sqrt_rn(double x) { return __dsqrt_rn(x); }
__device__ __forceinline__ float sqrt_rn(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double pow_t(double a, double b) { return pow(a, b); }
__device__ __forceinline__ float pow_t(float a, float b) { return powf(a, b); }

// cfl_dt(remaining) (simulation.hpp:134-145) with sound_speed_solid/_fluid (:73-81).
template <typename T>
__device__ T device_cfl_dt(const FrameState& fs, const StepConst<T>& c, T remaining) {
  T cmax = T(0);
  for (int mi = 0; mi < c.n_materials && mi < kMaxMaterials; ++mi) {
    const MatParam<T>& m = c.mats[mi];
    T s;
    if (m.model == kModelFluid) {
      const T pj = pow_t(T(fs.min_j[mi]), sub_rn(T(1), m.gamma));
      s = sqrt_rn(div_rn(mul_rn(mul_rn(m.bulk, m.gamma), pj), m.density));
    } else {
      s = sqrt_rn(div_rn(add_rn(m.lambda, mul_rn(T(2), m.mu)), m.density));
    }
    cmax = tmax(cmax, s);
  }
  const T denom = tmax(T(fs.vmax), cmax);
  T dt = denom > T(0) ? div_rn(mul_rn(T(fs.cfl), c.dx), denom) : remaining;
  if (T(fs.max_dt) > T(0)) dt = tmin(dt, T(fs.max_dt));
  return tmin(dt, remaining);
}

// Start of a substep: dt = cfl_dt(frame_end - time).
template <typename T>
__global__ void frame_ctl_kernel(FrameState* fs, StepConst<T> c, T* dtp) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const T rem = sub_rn(T(fs->frame_end), T(fs->time));
  const T dt = fs->fixed_dt > 0.0 ? T(fs->fixed_dt) : device_cfl_dt(*fs, c, rem);
  *dtp = dt;
  fs->dt = double(dt);
}

// End of a substep: latch errors, fold gather_all's reductions into vmax_ /
// min_j_, advance time, apply the substep limit and the frame-boundary test
// (simulation.hpp:197-208), and set the loop conditions.
template <typename T>
__global__ void frame_end_kernel(FrameState* fs, const DevStatus* st, cudaGraphConditionalHandle h_loop,
                                 cudaGraphConditionalHandle h_next, int n_materials) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned int cont = 0;
  if (st->err != ~0ull || st->nonfinite || st->overflow) {
    fs->status = 2;
  } else {
    double vm2;
    unsigned long long vb = st->vmax2;
    memcpy(&vm2, &vb, sizeof vm2);
    fs->vmax = double(sqrt_rn(T(vm2)));
    for (int m = 0; m < n_materials && m < kMaxMaterials; ++m) {
      double j;
      unsigned long long b = st->minj[m];
      memcpy(&j, &b, sizeof j);
      fs->min_j[m] = isfinite(j) ? j : 1.0;
    }
    fs->time = double(add_rn(T(fs->time), T(fs->dt)));
    fs->substeps += 1;
    fs->parity ^= 1u;
    if (fs->fixed_dt > 0.0) {
      if (fs->substeps >= fs->target) fs->status = 1;
      else cont = 1;
    } else if (fs->substeps > fs->max_substeps) {
      fs->status = 3;
    } else {
      const T rem = sub_rn(T(fs->frame_end), T(fs->time));
      if (rem <= mul_rn(T(fs->frame_dt), T(1e-9))) {
        fs->time = fs->frame_end;
        fs->status = 1;
      } else {
        cont = 1;
      }
    }
  }
  cudaGraphSetConditional(h_loop, cont);
  cudaGraphSetConditional(h_next, cont);
}

// Sort path of a graph substep, from the crosser count of the warp-count
// scan: up to kSmallSort crossers are ordered by one CTA; up to `bound` (the
// host path's merge threshold n/8) they are padded to `bound` entries and
// radix sorted at that fixed size; more take the full radix sort.
constexpr uint32_t kSmallSort = 8192;

__global__ void sort_decide_kernel(const uint32_t* __restrict__ woff, const uint32_t* __restrict__ wcnt,
                                   uint64_t nw, uint32_t bound, uint32_t* __restrict__ nc_out, FrameState* fs,
                                   cudaGraphConditionalHandle h_small, cudaGraphConditionalHandle h_mid,
                                   cudaGraphConditionalHandle h_full) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint32_t nc = nw ? woff[nw - 1] + wcnt[nw - 1] : 0u;
  *nc_out = nc;
  const unsigned small = nc <= kSmallSort, mid = !small && nc <= bound;
  fs->sort_paths[small ? 0 : (mid ? 1 : 2)] += 1;
  cudaGraphSetConditional(h_small, small);
  cudaGraphSetConditional(h_mid, mid);
  cudaGraphSetConditional(h_full, !small && !mid);
}

// Entries [nc, bound) of the crosser list get the largest key of the sorted
// bit range (a real key equal to it stays ahead: the sort is stable and the
// padding indices are larger), so a fixed-size sort leaves the nc real
// entries first, in order.
__global__ void pad_crossers_kernel(uint32_t* __restrict__ ck, uint32_t* __restrict__ ci,
                                    const uint32_t* __restrict__ ncp, uint32_t bound, uint32_t pad_key) {
  const uint32_t nc = *ncp;
  for (uint32_t i = nc + blockIdx.x * blockDim.x + threadIdx.x; i < bound; i += gridDim.x * blockDim.x) {
    ck[i] = pad_key;
    ci[i] = 0xffffffffu;
  }
}

// Stable sort of the compacted crossers (keys ck, indices ci in increasing
// index order) by key: a bitonic sort of (key << 32 | index) in shared memory,
// a total order, hence stable.  One CTA, nc <= kSmallSort (device count).
__global__ void __launch_bounds__(1024) small_sort_kernel(const uint32_t* __restrict__ ck,
                                                          const uint32_t* __restrict__ ci,
                                                          const uint32_t* __restrict__ ncp,
                                                          uint32_t* __restrict__ sck, uint32_t* __restrict__ sci) {
  extern __shared__ unsigned long long sv[];
  const uint32_t nc = *ncp;
  uint32_t m = 1;
  while (m < nc) m <<= 1;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x)
    sv[i] = i < nc ? ((static_cast<unsigned long long>(ck[i]) << 32) | ci[i]) : ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= m; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const unsigned long long a = sv[i], b = sv[l];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            sv[i] = b;
            sv[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
    sck[i] = static_cast<uint32_t>(sv[i] >> 32);
    sci[i] = static_cast<uint32_t>(sv[i] & 0xffffffffu);
  }
}

}  // namespace ckg
