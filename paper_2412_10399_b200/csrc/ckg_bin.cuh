// ckg_bin.cuh — binning, activation and segment kernels (sm_100a).
//
//  K1  key_footprint_kernel: block key (simulation.hpp:255-266, bit-exact),
//      the particle's stencil-footprint blocks ("core" flags) and the 2-cell
//      inset check (grid.hpp:121-126), one pass over x in current order.
//  K2  stable LSD radix sort (ckg_scan.cuh) -> perm, sorted keys.
//  K3  inset_fixup_kernel: only when K1 saw a violation, the lowest SORTED
//      index and its first failing axis (the reference throws from activate,
//      which walks the sorted array).
//  K4  dilate_kernel: active = core (+) {0,1}^3 — the reference's one-block
//      positive halo (grid.hpp:137-139) as a Minkowski sum over the directory.
//  K5  scan + compact_kernel: directory slots in ascending directory order.
//  K6  segments_kernel: [begin, end) of every block key in sorted order.
#pragma once

#include "ckg_kernels.cuh"

namespace ckg {

// Footprint of one axis relative to the key block: lo block = floor(s-1/4)>>2
// (the +1 grid's lower node), hi block = (floor(s+1/4)+1)>>2 (the -1 grid's
// upper node), with s = x*inv_dx exactly as activate computes it
// (grid.hpp:121-137).  The key cell floor(s + 1/4) is the same rounded sum,
// so lo, hi are within one block of the key block.
// Quadratic baseline (grid.hpp:133-136): nodes floor(s - 1/2) .. +2.
template <typename T>
__device__ __forceinline__ void axis_footprint(T x, T inv_dx, int quad, int& lo, int& hi) {
  const T s = mul_rn(x, inv_dx);
  if (quad) {
    const int base = static_cast<int>(dfloor(sub_rn(s, T(0.5))));
    lo = base >> 2;
    hi = (base + 2) >> 2;
    return;
  }
  lo = static_cast<int>(dfloor(sub_rn(s, T(0.25)))) >> 2;
  hi = (static_cast<int>(dfloor(add_rn(s, T(0.25)))) + 1) >> 2;
}

template <typename T>
__device__ __forceinline__ bool inset_ok(T x, T inv_dx, int res) {
  const T s = mul_rn(x, inv_dx);
  return s >= T(2) && s <= T(res - 2);
}

// Marks the footprint box of key block kb with extension bits ext (bit 2a:
// one block lower on axis a, bit 2a+1: one block higher).
__device__ __forceinline__ void mark_footprint_box(uint32_t* __restrict__ core, const int (&kb)[3], uint32_t ext,
                                                   int D) {
  // inset particles (s in [2, res-2]) have footprint cells in [1, res-1], so
  // every box block lies inside the (res/4 + 2)^3 directory: no bounds checks
  // Per axis the box is 1 or 2 blocks: the low extension needs s < 4 kb + 1/4
  // and the high one s >= 4 kb + 11/4, never both.  So 2 x 2 x 2 predicated
  // stores cover every box (no data-dependent loop).
  const bool ex = (ext & 3u) != 0u, ey = ((ext >> 2) & 3u) != 0u, ez = ((ext >> 4) & 3u) != 0u;
  const int64_t DD = int64_t(D) * D;
  uint32_t* c0 = core + (int64_t(kb[0] - int(ext & 1u)) * D + (kb[1] - int((ext >> 2) & 1u))) * D +
                 (kb[2] - int((ext >> 4) & 1u));
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int k = 0; k < 2; ++k)
        if ((a == 0 || ex) && (b == 0 || ey) && (k == 0 || ez)) c0[a * DD + b * D + k] = 1u;
}

// One particle of the key pass (all 32 lanes of the warp call it for 32
// consecutive particles; x and the stored key are loaded by the caller).
template <typename T>
__device__ __forceinline__ void key_footprint_one(uint64_t i, bool live, const T (&x)[3], uint32_t kov, uint64_t n,
                                                  T inv_dx, int res, int D, int quad, uint32_t* __restrict__ keys,
                                                  uint32_t* __restrict__ core, const uint32_t* __restrict__ ko,
                                                  uint32_t* __restrict__ cbits, uint32_t* __restrict__ wcnt,
                                                  uint8_t* __restrict__ cls, DevStatus* st) {
  bool ok = live, changed = false;
  uint32_t key = 0xffffffffu, ext = 0;
  int kb[3] = {0, 0, 0};
  if (live) {
#pragma unroll
    for (int a = 0; a < 3; ++a) kb[a] = key_axis(x[a], inv_dx, D);
    key = (uint32_t(kb[0]) * uint32_t(D) + uint32_t(kb[1])) * uint32_t(D) + uint32_t(kb[2]);
    keys[i] = key;
    if (cls) {
      // P2G sub-octant class (frac(x/dx - 1/4) >= 1/2 per axis), read by
      // xfer_prep_kernel through the sort permutation
      uint32_t q = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const T sa = sub_rn(mul_rn(x[a], inv_dx), T(0.25));
        q |= ((sa - dfloor(sa)) >= T(0.5) ? 1u : 0u) << a;
      }
      cls[i] = uint8_t(q);
    }
    if (ko) changed = key != kov;
    // footprint blocks relative to the key block: lo in {kb-1, kb}, hi in {kb, kb+1}
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      ok = ok && inset_ok(x[a], inv_dx, res);
      int lo, hi;
      axis_footprint(x[a], inv_dx, quad, lo, hi);
      ok = ok && lo >= kb[a] - 1 && hi <= kb[a] + 1;
      ext |= (lo < kb[a] ? 1u : 0u) << (2 * a);
      ext |= (hi > kb[a] ? 1u : 0u) << (2 * a + 1);
    }
    if (!ok) atomicOr(&st->inset_fail, 1u);
  }
  if (ko) {
    // one word of changed flags and its count per warp (ckg_isort.cuh ranks
    // from these instead of a per-particle scan)
    const uint32_t cb = __ballot_sync(0xffffffffu, changed);
    if ((threadIdx.x & 31) == 0 && i < n) {
      cbits[i >> 5] = cb;
      wcnt[i >> 5] = uint32_t(__popc(cb));
      if (cb) atomicAdd(&st->nchanged, uint32_t(__popc(cb)));
    }
  }
  // Lanes with the same footprint box (same key block and extent bits) mark
  // it once.  (A bounding box over different boxes would over-activate.)
  const uint64_t gbox = ok ? ((uint64_t(key) << 8) | ext) : (~0ull - (threadIdx.x & 31));
  const uint32_t peers = __match_any_sync(0xffffffffu, gbox);
  if (!ok || (__ffs(peers) - 1) != int(threadIdx.x & 31)) return;
  mark_footprint_box(core, kb, ext, D);
}

// The compact-kernel key pass with one rounded-to-floor conversion per
// grid offset and axis: with s = x * inv_dx (T-rounded, as the reference),
//   ip = floor(s + 1/4)      -> key block ip >> 2 (simulation.hpp:255-266) and
//                               the -1 grid's upper node ip + 1 (hi block)
//   i2 = floor(2 (s - 1/4))  -> floor(s - 1/4) = i2 >> 1 (lo block i2 >> 3) and
//                               the class bit frac(s - 1/4) >= 1/2 = i2 & 1
// (2x is exact).  For inset particles (2 <= s <= res - 2) the key block needs
// no clamp and lo / hi lie within one block of it, so the only failure is the
// inset itself (grid.hpp:121-126).
__device__ __forceinline__ int floor_int(double v) { return __double2int_rd(v); }
__device__ __forceinline__ int floor_int(float v) { return __float2int_rd(v); }

template <typename T>
__device__ __forceinline__ void key_footprint_compact(uint64_t i, bool live, const T (&x)[3], uint32_t kov,
                                                      uint64_t n, T inv_dx, int res, int D,
                                                      uint32_t* __restrict__ keys, uint32_t* __restrict__ core,
                                                      const uint32_t* __restrict__ ko,
                                                      uint32_t* __restrict__ cbits, uint32_t* __restrict__ wcnt,
                                                      uint8_t* __restrict__ cls, DevStatus* st) {
  bool ok = live, changed = false;
  uint32_t key = 0xffffffffu, ext = 0, q = 0;
  int kb[3] = {0, 0, 0};
  if (live) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T s = mul_rn(x[a], inv_dx);
      const int ip = floor_int(add_rn(s, T(0.25)));
      const int i2 = floor_int(T(2) * sub_rn(s, T(0.25)));
      const int b = ip >> 2;
      kb[a] = b < 0 ? 0 : (b > D - 1 ? D - 1 : b);
      q |= uint32_t(i2 & 1) << a;
      ok = ok && s >= T(2) && s <= T(res - 2);
      ext |= ((i2 >> 3) < kb[a] ? 1u : 0u) << (2 * a);
      ext |= (((ip + 1) >> 2) > kb[a] ? 1u : 0u) << (2 * a + 1);
    }
    key = (uint32_t(kb[0]) * uint32_t(D) + uint32_t(kb[1])) * uint32_t(D) + uint32_t(kb[2]);
    keys[i] = key;
    if (cls) cls[i] = uint8_t(q);
    if (ko) changed = key != kov;
    if (!ok) atomicOr(&st->inset_fail, 1u);
  }
  if (ko) {
    const uint32_t cb = __ballot_sync(0xffffffffu, changed);
    if ((threadIdx.x & 31) == 0 && i < n) {
      cbits[i >> 5] = cb;
      wcnt[i >> 5] = uint32_t(__popc(cb));
      if (cb) atomicAdd(&st->nchanged, uint32_t(__popc(cb)));
    }
  }
  const uint64_t gbox = ok ? ((uint64_t(key) << 8) | ext) : (~0ull - (threadIdx.x & 31));
  const uint32_t peers = __match_any_sync(0xffffffffu, gbox);
  if (!ok || (__ffs(peers) - 1) != int(threadIdx.x & 31)) return;
  mark_footprint_box(core, kb, ext, D);
}

// K1 key pass: block key (simulation.hpp:255-266), footprint boxes + inset
// (grid.hpp:121-137), changed words, P2G class byte.  Each warp covers
// kKeyPer x 32 consecutive particles with all their position / stored-key
// loads issued up front (memory-level parallelism: the pass is latency-bound
// at one particle per thread).
#ifndef CKG_KEY_PER
#define CKG_KEY_PER 2
#endif
constexpr int kKeyPer = CKG_KEY_PER;
template <typename T, int QUAD>
__global__ void __launch_bounds__(256) key_footprint_kernel(PState<T> cur, T inv_dx, int res, int D, int quad,
                                                            uint32_t* __restrict__ keys,
                                                            uint32_t* __restrict__ core,
                                                            const uint32_t* __restrict__ ko,
                                                            uint32_t* __restrict__ cbits,
                                                            uint32_t* __restrict__ wcnt,
                                                            uint8_t* __restrict__ cls, DevStatus* st) {
  const uint64_t gt = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t base = (gt >> 5) * (32 * kKeyPer) + (gt & 31);
  T x[kKeyPer][3];
  uint32_t kov[kKeyPer];
#pragma unroll
  for (int r = 0; r < kKeyPer; ++r) {
    const uint64_t i = base + 32 * r;
    const bool live = i < cur.n;
#pragma unroll
    for (int a = 0; a < 3; ++a) x[r][a] = live ? __ldg(cur.f + uint64_t(kX + a) * cur.stride + i) : T(0);
    kov[r] = (live && ko) ? __ldg(ko + i) : 0u;
  }
#pragma unroll
  for (int r = 0; r < kKeyPer; ++r) {
    const uint64_t i = base + 32 * r;
    if (QUAD)
      key_footprint_one<T>(i, i < cur.n, x[r], kov[r], cur.n, inv_dx, res, D, quad, keys, core, ko, cbits, wcnt,
                           cls, st);
    else
      key_footprint_compact<T>(i, i < cur.n, x[r], kov[r], cur.n, inv_dx, res, D, keys, core, ko, cbits, wcnt, cls,
                               st);
  }
}

// Lowest sorted index violating the inset (only runs its loop on failure).
template <typename T>
__global__ void inset_fixup_kernel(PState<T> cur, const uint32_t* __restrict__ perm, T inv_dx, int res,
                                   DevStatus* st, int step) {
  if (*reinterpret_cast<volatile unsigned int*>(&st->inset_fail) == 0u) return;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < cur.n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t src = perm[i];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (!inset_ok(cur.f[uint64_t(kX + a) * cur.stride + src], inv_dx, res)) {
        record_error(st, step, kPhaseActivate, i, a, kErrOutOfDomain);
        break;
      }
    }
  }
}

// active(B) = OR_{delta in {0,1}^3} core(B - delta).
__global__ void __launch_bounds__(256) dilate_kernel(const uint32_t* __restrict__ core,
                                                     uint32_t* __restrict__ act, int D) {
  // 32-bit index arithmetic (the directory has (res/4 + 2)^3 < 2^32 entries;
  // 64-bit div/mod was most of this kernel's instructions)
  const uint32_t ud = uint32_t(D), nd = ud * ud * ud;
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nd) return;
  const uint32_t row = d / ud, bz = d - row * ud;
  const uint32_t bx = row / ud, by = row - bx * ud;
  const uint32_t sx = ud * ud;
  uint32_t a = __ldg(core + d);
  if (bz > 0) a |= __ldg(core + d - 1);
  if (by > 0) {
    a |= __ldg(core + d - ud);
    if (bz > 0) a |= __ldg(core + d - ud - 1);
  }
  if (bx > 0) {
    a |= __ldg(core + d - sx);
    if (bz > 0) a |= __ldg(core + d - sx - 1);
    if (by > 0) {
      a |= __ldg(core + d - sx - ud);
      if (bz > 0) a |= __ldg(core + d - sx - ud - 1);
    }
  }
  act[d] = a ? 1u : 0u;
}

// Directory from the exclusive scan of act (computed in place in dir):
// dir[d] = slot or -1; active[slot] = d in ascending order.  Resets the
// per-step scratch (core, act, segment bounds) for the next substep.
__global__ void __launch_bounds__(256) compact_kernel(uint32_t* __restrict__ core, uint32_t* __restrict__ act,
                                                      int32_t* __restrict__ dir, uint32_t* __restrict__ active,
                                                      uint32_t* __restrict__ seg_begin,
                                                      uint32_t* __restrict__ seg_end, uint64_t nd, uint32_t cap,
                                                      DevStatus* st) {
  const uint64_t d = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d >= nd) return;
  const uint32_t f = act[d];
  const uint32_t s = static_cast<uint32_t>(dir[d]);
  if (f) {
    if (s < cap)
      active[s] = static_cast<uint32_t>(d);
    else
      st->overflow = 1u;
    act[d] = 0u;
  } else {
    dir[d] = -1;
  }
  core[d] = 0u;
  if (seg_begin) {  // (null: the caller resets the segment table itself)
    seg_begin[d] = 0u;
    seg_end[d] = 0u;
  }
  if (d == nd - 1) {
    st->n_active = s + f;
    st->item_lo = st->grid_lo = st->clear_lo = 0u;
    st->item_hi = st->grid_hi = st->clear_hi = s + f;
  }
}

// [begin, end) of each block key's run in the sorted order.
__global__ void __launch_bounds__(256) segments_kernel(const uint32_t* __restrict__ skeys, uint64_t n,
                                                       uint32_t* __restrict__ seg_begin,
                                                       uint32_t* __restrict__ seg_end) {
  // four sorted keys per thread (16-byte loads); neighbours across threads
  // by shuffles, across warps from memory
  const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t i0 = q * 4;
  const int lane = threadIdx.x & 31;
  uint32_t k[4];
  if (i0 + 3 < n) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(skeys) + q);
    k[0] = v.x, k[1] = v.y, k[2] = v.z, k[3] = v.w;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) k[e] = i0 + e < n ? skeys[i0 + e] : 0xffffffffu;
  }
  uint32_t prev = __shfl_up_sync(0xffffffffu, k[3], 1);
  uint32_t next = __shfl_down_sync(0xffffffffu, k[0], 1);
  if (lane == 0) prev = i0 > 0 && i0 - 1 < n ? skeys[i0 - 1] : 0xffffffffu;
  if (lane == 31) next = i0 + 4 < n ? skeys[i0 + 4] : 0xffffffffu;
  if (i0 >= n) return;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint64_t i = i0 + e;
    if (i >= n) break;
    const uint32_t kp = e == 0 ? prev : k[e - 1];
    const uint32_t kn = (e == 3 || i + 1 >= n) ? (i + 1 < n ? next : 0xffffffffu) : k[e + 1];
    if (i == 0 || kp != k[e]) seg_begin[k[e]] = uint32_t(i);
    if (i == n - 1 || kn != k[e]) seg_end[k[e]] = uint32_t(i + 1);
  }
}

}  // namespace ckg
