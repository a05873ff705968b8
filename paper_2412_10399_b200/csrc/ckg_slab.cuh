// ckg_slab.cuh — x-slab decomposition kernels.
//
// Each rank owns block planes bx in [bx_lo, bx_hi) and the particles whose
// sort key lies there.  The block directory is global and identical on every
// rank (the footprint flags are MAX-all-reduced before activation), and the
// active list is in directory order, so every block plane bx occupies the
// contiguous slot range [plane_start[bx], plane_start[bx+1]) on all ranks:
// halo exchanges are contiguous slices of the block pool, no coordinate
// matching.  Per substep:
//   P2G writes ghost planes bx_lo-1 and bx_hi  -> sent to the owners, added
//   grid update on owned planes                -> boundary planes sent back
//   G2P on owned particles                     -> migrants (new key outside
//   [bx_lo, bx_hi)) packed in order and sent; the receiver builds
//   [left migrants][survivors][right migrants], which the next substep's
//   stable sort turns into the global stable order restricted to the slab.
#pragma once

#include <cstdint>

#include "ckg_kernels.cuh"
#include "ckg_transfer.cuh"

namespace ckg {

// plane_start[bx] = first slot of block plane bx: the exclusive scan of the
// active flags at directory index (bx, 0, 0) (read before compaction).
__global__ void plane_start_kernel(const uint32_t* __restrict__ scan_of_act, const uint32_t* __restrict__ act,
                                   int D, uint32_t* __restrict__ plane_start) {
  const int bx = blockIdx.x * blockDim.x + threadIdx.x;
  if (bx > D) return;
  if (bx == D) {
    const uint64_t last = uint64_t(D) * D * D - 1;
    plane_start[D] = scan_of_act[last] + act[last];
    return;
  }
  plane_start[bx] = scan_of_act[uint64_t(bx) * D * D];
}

// Work ranges of this rank after compaction: transfer items (own planes),
// grid update (own planes), clear (own planes and both ghost planes).
__global__ void slab_ranges_kernel(const uint32_t* __restrict__ plane_start, int D, int bx_lo, int bx_hi,
                                   DevStatus* st) {
  const int g0 = bx_lo > 0 ? bx_lo - 1 : 0, g1 = bx_hi < D ? bx_hi + 1 : D;
  st->item_lo = plane_start[bx_lo];
  st->item_hi = plane_start[bx_hi];
  st->grid_lo = plane_start[bx_lo];
  st->grid_hi = plane_start[bx_hi];
  st->clear_lo = plane_start[g0];
  st->clear_hi = plane_start[g1];
}

// Transfer item range [plane_start[a], plane_start[b]) for the next P2G
// launch (its work counter restarted): the x-slab P2G runs the two boundary
// planes first, so their halo leaves while the interior planes scatter.
__global__ void slab_item_range_kernel(const uint32_t* __restrict__ plane_start, int a, int b, DevStatus* st) {
  st->item_lo = plane_start[a];
  st->item_hi = plane_start[b];
  st->work[0] = 0u;
}

// op 0: dst[...] = pool plane; op 1: pool plane += src; op 2: pool plane = src;
// op 5 / 6: the same as 0 / 2 for the nodal velocities only (the broadcast
// after the grid update: 3 of each block's 4 values per grid, 384 of 512
// words).
template <typename T>
__global__ void halo_kernel(T* __restrict__ pool, const uint32_t* __restrict__ plane_start, int bx, int op,
                            T* __restrict__ buf) {
  const uint64_t s0 = plane_start[bx], s1 = plane_start[bx + 1];
  const bool vel = op >= 5;
  const uint64_t per = vel ? 384 : kBlockVals;
  const uint64_t total = (s1 - s0) * per;
  T* p = pool + s0 * kBlockVals;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total; k += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t w = k;
    if (vel) {  // block b, word r of its 384: grid r / 192, value 1 + (r % 192) / 64, node r % 64
      const uint64_t b = k / 384, r = k % 384;
      w = b * kBlockVals + (r / 192) * 256 + 64 + (r % 192);
    }
    if (op == 0 || op == 5)
      buf[k] = p[w];
    else if (op == 1)
      p[w] += buf[k];
    else
      p[w] = buf[k];
  }
}

// Deterministic mode: a plane's per-block P2G tiles (kDetVals words per slot)
// op 3: dst[...] = tiles of the plane; op 4: tiles of the plane = src.
template <typename T>
__global__ void tile_halo_kernel(T* __restrict__ dtile, uint32_t dcap, const uint32_t* __restrict__ plane_start,
                                 int bx, int op, T* __restrict__ buf, unsigned int* overflow) {
  const uint64_t s0 = plane_start[bx], s1 = plane_start[bx + 1];
  if (s1 > dcap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(overflow, 2u);
    return;
  }
  const uint64_t total = (s1 - s0) * uint64_t(kDetVals);
  T* p = dtile + s0 * uint64_t(kDetVals);
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total; k += uint64_t(gridDim.x) * blockDim.x) {
    if (op == 3)
      buf[k] = p[k];
    else
      p[k] = buf[k];
  }
}

// Particles per sort-key plane bx (rebalancing input).
template <typename T>
__global__ void plane_count_kernel(PState<T> p, T inv_dx, int D, unsigned long long* __restrict__ counts) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < p.n; i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(counts + key_axis(p.f[uint64_t(kX) * p.stride + i], inv_dx, D), 1ull);
}

// Migration class of each particle of the new state: 0 stays, 1 left, 2 right.
template <typename T>
__global__ void classify_kernel(PState<T> st_new, T inv_dx, int D, int bx_lo, int bx_hi,
                                uint32_t* __restrict__ stay, uint32_t* __restrict__ left,
                                uint32_t* __restrict__ right) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= st_new.n) return;
  const int bx = key_axis(st_new.f[uint64_t(kX) * st_new.stride + i], inv_dx, D);
  const uint32_t l = bx < bx_lo, r = bx >= bx_hi;
  left[i] = l;
  right[i] = r;
  stay[i] = (l | r) ? 0u : 1u;
}

// Migrant record: 27 state fields, material (bit pattern in a T word), the 6
// stress-cache values and the particle's previous sorted key (a T word).
constexpr int kMigrantWords = kNumFields + 1 + 6 + 1;

template <typename T>
__device__ __forceinline__ T word_of(uint32_t v) {
  T w = T(0);
  *reinterpret_cast<uint32_t*>(&w) = v;
  return w;
}
template <typename T>
__device__ __forceinline__ uint32_t word_to_u32(T w) {
  return *reinterpret_cast<const uint32_t*>(&w);
}

// Survivors -> dst (at pos_stay + offset, with their old keys), migrants of
// the chosen sides -> records at their scanned positions.
template <typename T>
__global__ void migrate_out_kernel(PState<T> src, const uint32_t* __restrict__ src_oldkey,
                                   const uint32_t* __restrict__ stay, const uint32_t* __restrict__ pos_stay,
                                   const uint32_t* __restrict__ left, const uint32_t* __restrict__ pos_left,
                                   const uint32_t* __restrict__ right, const uint32_t* __restrict__ pos_right,
                                   PState<T> dst, uint32_t* __restrict__ dst_oldkey, uint64_t offset,
                                   T* __restrict__ rec_left, T* __restrict__ rec_right) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= src.n) return;
  if (stay[i]) {
    const uint64_t j = pos_stay[i] + offset;
#pragma unroll 4
    for (int k = 0; k < kNumFields; ++k) dst.f[uint64_t(k) * dst.stride + j] = src.f[uint64_t(k) * src.stride + i];
#pragma unroll
    for (int k = 0; k < 6; ++k) dst.tau[uint64_t(k) * dst.stride + j] = src.tau[uint64_t(k) * src.stride + i];
    dst.mat[j] = src.mat[i];
    dst_oldkey[j] = src_oldkey[i];
    return;
  }
  T* rec = left[i] ? rec_left + uint64_t(pos_left[i]) * kMigrantWords
                   : rec_right + uint64_t(pos_right[i]) * kMigrantWords;
  (void)right;
#pragma unroll 4
  for (int k = 0; k < kNumFields; ++k) rec[k] = src.f[uint64_t(k) * src.stride + i];
  rec[kNumFields] = word_of<T>(src.mat[i]);
#pragma unroll
  for (int k = 0; k < 6; ++k) rec[kNumFields + 1 + k] = src.tau[uint64_t(k) * src.stride + i];
  rec[kNumFields + 7] = word_of<T>(src_oldkey[i]);
}

// Received records -> dst positions [offset, offset + count).
template <typename T>
__global__ void migrate_in_kernel(const T* __restrict__ rec, uint64_t count, PState<T> dst,
                                  uint32_t* __restrict__ dst_oldkey, uint64_t offset) {
  const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= count) return;
  const T* p = rec + r * kMigrantWords;
  const uint64_t j = offset + r;
#pragma unroll 4
  for (int k = 0; k < kNumFields; ++k) dst.f[uint64_t(k) * dst.stride + j] = p[k];
  dst.mat[j] = word_to_u32(p[kNumFields]);
#pragma unroll
  for (int k = 0; k < 6; ++k) dst.tau[uint64_t(k) * dst.stride + j] = p[kNumFields + 1 + k];
  dst_oldkey[j] = word_to_u32(p[kNumFields + 7]);
}

// ---- windowed migration (region path) -----------------------------------
// In a slab the state lives in a window [wb, wb + n) of each buffer.  Block
// crossers can only come from the first and last owned block plane (a
// substep moves a particle less than a cell), i.e. from the sorted prefix
// [0, PL) and suffix [PR, n).  Only those regions are compacted; the middle
// stays in place and the window start moves by (out_left - in_left).

// PL = first sorted position with key >= key_a, PR = first with key >= key_b.
__global__ void slab_regions_kernel(const uint32_t* __restrict__ skeys, uint64_t n, uint32_t key_a,
                                    uint32_t key_b, unsigned long long* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint32_t kk[2] = {key_a, key_b};
  for (int q = 0; q < 2; ++q) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (skeys[mid] < kk[q]) lo = mid + 1; else hi = mid;
    }
    out[q] = lo;
  }
}

// Migrants found in the middle region: the region path does not apply.
__global__ void count_far_kernel(const uint32_t* __restrict__ left, const uint32_t* __restrict__ right,
                                 uint64_t i0, uint64_t i1, unsigned long long* __restrict__ far) {
  unsigned int c = 0;
  for (uint64_t i = i0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < i1;
       i += uint64_t(gridDim.x) * blockDim.x)
    c += left[i] | right[i];
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(far, (unsigned long long)c);
}

template <typename T>
__device__ __forceinline__ void copy_particle(const PState<T>& a, uint64_t i, const PState<T>& b, uint64_t j) {
#pragma unroll 3
  for (int k = 0; k < kNumFields; ++k) b.f[uint64_t(k) * b.stride + j] = a.f[uint64_t(k) * a.stride + i];
#pragma unroll
  for (int k = 0; k < 6; ++k) b.tau[uint64_t(k) * b.stride + j] = a.tau[uint64_t(k) * a.stride + i];
  b.mat[j] = a.mat[i];
}

// Region [i0, i1): migrants -> records (scanned positions pos_*[i - i0] local
// to the region), survivors -> tmp at the same index.
template <typename T>
__global__ void region_out_kernel(PState<T> src, const uint32_t* __restrict__ oldkey, uint64_t i0, uint64_t i1,
                                  const uint32_t* __restrict__ fl_left, const uint32_t* __restrict__ pos_left,
                                  const uint32_t* __restrict__ fl_right, const uint32_t* __restrict__ pos_right,
                                  T* __restrict__ rec_left, T* __restrict__ rec_right, PState<T> tmp) {
  const uint64_t i = i0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= i1) return;
  const uint64_t r = i - i0;
  if (fl_left[i] | fl_right[i]) {
    T* rec = fl_left[i] ? rec_left + uint64_t(pos_left[r]) * kMigrantWords
                        : rec_right + uint64_t(pos_right[r]) * kMigrantWords;
#pragma unroll 4
    for (int k = 0; k < kNumFields; ++k) rec[k] = src.f[uint64_t(k) * src.stride + i];
    rec[kNumFields] = word_of<T>(src.mat[i]);
#pragma unroll
    for (int k = 0; k < 6; ++k) rec[kNumFields + 1 + k] = src.tau[uint64_t(k) * src.stride + i];
    rec[kNumFields + 7] = word_of<T>(oldkey[i]);
    return;
  }
  copy_particle(src, i, tmp, i);
}

// Region survivors back from tmp to dst at dst_base + (local scan of stay).
template <typename T>
__global__ void region_in_kernel(PState<T> tmp, uint64_t i0, uint64_t i1, const uint32_t* __restrict__ fl_stay,
                                 const uint32_t* __restrict__ pos_stay, PState<T> dst, int64_t dst_base) {
  const uint64_t i = i0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= i1 || !fl_stay[i]) return;
  copy_particle(tmp, i, dst, uint64_t(dst_base + int64_t(pos_stay[i - i0])));
}

// Next substep's stored-order keys (relative to the new window): middle
// [PL, PR) shifted by `shift` = in_left - out_left, region survivors at their
// compacted positions; incoming migrants are filled by migrate_in_kernel.
__global__ void region_keys_kernel(const uint32_t* __restrict__ skeys, uint64_t n, uint64_t PL, uint64_t PR,
                                   int64_t shift, const uint32_t* __restrict__ fl_stay,
                                   const uint32_t* __restrict__ pos_stay_l, const uint32_t* __restrict__ pos_stay_r,
                                   uint64_t in_left, uint64_t stay_l, uint32_t* __restrict__ ko_new) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i >= PL && i < PR) {
    ko_new[uint64_t(int64_t(i) + shift)] = skeys[i];
  } else if (fl_stay[i]) {
    const uint64_t j = i < PL ? in_left + pos_stay_l[i] : in_left + stay_l + (PR - PL) + pos_stay_r[i - PR];
    ko_new[j] = skeys[i];
  }
}

}  // namespace ckg
