// ckg_scan.cuh — device-wide exclusive scan and stable LSD radix sort of
// (block key, particle index) pairs, hand-written for sm_100a.
//
// Replaces the reference's serial stable counting sort
// (proj/include/ckmpm/simulation.hpp:248-274).  Stability is what makes the
// sorted order bit-identical to the reference: within a digit bucket, items
// keep their input order (warp rounds in index order, lanes in index order,
// warps and tiles prefix-summed in index order).
#pragma once

#include <cstdint>

namespace ckg {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive block-wide scan of one value per thread; returns the exclusive
// prefix, writes the block total to *total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kScanThreads / 32) warp_sums[lane] = s;  // inclusive
  }
  __syncthreads();
  uint32_t warp_prefix = wid ? warp_sums[wid - 1] : 0;
  *total = warp_sums[kScanThreads / 32 - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

// Phase 1: per-tile sums.
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in,
                                                                  uint64_t n,
                                                                  uint32_t* __restrict__ partials) {
  uint64_t base = uint64_t(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += in[base + k];
  uint32_t total;
  block_exclusive_scan(s, &total);
  if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

// Phase 2: single-CTA exclusive scan of the partials (any count, chunked).
__global__ void __launch_bounds__(kScanThreads) scan_partials_kernel(uint32_t* partials, uint64_t np) {
  uint32_t carry = 0;
  for (uint64_t start = 0; start < np; start += kScanTile) {
    uint64_t base = start + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      v[k] = base + k < np ? partials[base + k] : 0;
      s += v[k];
    }
    uint32_t total;
    uint32_t pre = block_exclusive_scan(s, &total) + carry;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      if (base + k < np) partials[base + k] = pre;
      pre += v[k];
    }
    carry += total;
  }
}

// Phase 3: per-tile exclusive scan plus the tile's offset.
__global__ void __launch_bounds__(kScanThreads) scan_downsweep_kernel(const uint32_t* __restrict__ in,
                                                                     uint64_t n,
                                                                     const uint32_t* __restrict__ partials,
                                                                     uint32_t* __restrict__ out) {
  uint64_t base = uint64_t(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  uint32_t total;
  uint32_t pre = block_exclusive_scan(s, &total) + partials[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = pre;
    pre += v[k];
  }
}

inline uint64_t scan_tiles(uint64_t n) { return (n + kScanTile - 1) / kScanTile; }

// Exclusive scan in -> out (may alias).  partials needs scan_tiles(n) words.
inline void exclusive_scan(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* partials,
                           cudaStream_t st) {
  uint64_t nt = scan_tiles(n);
  if (nt == 0) return;
  scan_reduce_kernel<<<unsigned(nt), kScanThreads, 0, st>>>(in, n, partials);
  scan_partials_kernel<<<1, kScanThreads, 0, st>>>(partials, nt);
  scan_downsweep_kernel<<<unsigned(nt), kScanThreads, 0, st>>>(in, n, partials, out);
}

// ---------------------------------------------------------------- radix sort

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048 keys

__global__ void __launch_bounds__(kSortThreads) radix_upsweep_kernel(const uint32_t* __restrict__ keys,
                                                                    uint64_t n, int shift,
                                                                    uint32_t* __restrict__ hist,
                                                                    uint32_t ntiles) {
  __shared__ uint32_t cnt[kRadix];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  uint64_t base = uint64_t(blockIdx.x) * kSortTile;
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    uint64_t i = base + uint64_t(k) * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  hist[uint64_t(threadIdx.x) * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

// Stable scatter of one digit pass.  vals_in == nullptr means identity values.
__global__ void __launch_bounds__(kSortThreads) radix_downsweep_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint64_t n, int shift,
    const uint32_t* __restrict__ offsets, uint32_t ntiles, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out) {
  __shared__ uint32_t wcnt[kSortWarps][kRadix];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kSortWarps; ++k) wcnt[k][threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = uint64_t(blockIdx.x) * kSortTile + uint64_t(w) * (32 * kSortItems);
  uint32_t key[kSortItems], val[kSortItems], local[kSortItems];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    uint64_t i = base + uint64_t(r) * 32 + lane;
    bool valid = i < n;
    key[r] = valid ? keys_in[i] : 0u;
    val[r] = valid ? (vals_in ? vals_in[i] : uint32_t(i)) : 0u;
    uint32_t d = valid ? ((key[r] >> shift) & (kRadix - 1)) : (uint32_t(kRadix) + lane);
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t rank = __popc(peers & lt);
    uint32_t before = valid ? wcnt[w][d & (kRadix - 1)] : 0u;
    __syncwarp();
    if (valid && rank == 0) wcnt[w][d] = before + __popc(peers);
    __syncwarp();
    local[r] = before + rank;
  }
  __syncthreads();
  {
    const int d = threadIdx.x;  // one thread per digit
    uint32_t run = offsets[uint64_t(d) * ntiles + blockIdx.x];
#pragma unroll
    for (int k = 0; k < kSortWarps; ++k) {
      uint32_t c = wcnt[k][d];
      wcnt[k][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    uint64_t i = base + uint64_t(r) * 32 + lane;
    if (i < n) {
      uint32_t d = (key[r] >> shift) & (kRadix - 1);
      uint32_t pos = wcnt[w][d] + local[r];
      keys_out[pos] = key[r];
      vals_out[pos] = val[r];
    }
  }
}

struct RadixScratch {
  uint32_t* keys_alt = nullptr;
  uint32_t* vals_alt = nullptr;
  uint32_t* hist = nullptr;      // kRadix * ntiles
  uint32_t* partials = nullptr;  // scan_tiles(kRadix * ntiles)
};

inline uint32_t sort_tiles(uint64_t n) { return uint32_t((n + kSortTile - 1) / kSortTile); }

// Stable sort of keys[0..n) (only the low `bits` bits are significant).
// On return *keys_res / *vals_res point at the sorted keys and the permutation
// (either the caller's buffers or the scratch ones).
// vals_init == nullptr: the values are the input indices (a permutation).
inline void radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint64_t n, int bits, RadixScratch& s,
                             cudaStream_t st, uint32_t** keys_res, uint32_t** vals_res,
                             uint32_t* vals_init = nullptr) {
  uint32_t ntiles = sort_tiles(n);
  uint32_t *kin = keys, *vin = vals_init, *kout = s.keys_alt, *vout = s.vals_alt;
  int passes = (bits + kRadixBits - 1) / kRadixBits;
  if (passes < 1) passes = 1;
  for (int p = 0; p < passes; ++p) {
    int shift = p * kRadixBits;
    radix_upsweep_kernel<<<ntiles, kSortThreads, 0, st>>>(kin, n, shift, s.hist, ntiles);
    exclusive_scan(s.hist, s.hist, uint64_t(kRadix) * ntiles, s.partials, st);
    radix_downsweep_kernel<<<ntiles, kSortThreads, 0, st>>>(kin, vin, n, shift, s.hist, ntiles, kout,
                                                            vout);
    // ping-pong: the next pass reads what this one wrote
    uint32_t* nk = (kout == s.keys_alt) ? keys : s.keys_alt;
    uint32_t* nv = (vout == s.vals_alt) ? vals : s.vals_alt;
    kin = kout;
    vin = vout;
    kout = nk;
    vout = nv;
  }
  *keys_res = kin;
  *vals_res = vin;
}

}  // namespace ckg
