// ckg_isort.cuh — incremental stable sort by block key (sm_100a).
//
// The reference re-sorts the whole particle array every substep with a stable
// counting sort (proj/include/ckmpm/simulation.hpp:248-274).  Here the state
// is stored in the last sorted order, so the previous sorted keys `ko` are
// non-decreasing and only particles that crossed a block boundary ("changed",
// key != ko) can be out of place.  The stable sort of the new keys is then the
// stable merge, by (key, index), of
//   U = unchanged particles (already sorted, keys == ko), and
//   C = changed particles, stably sorted by key (radix sort of |C| entries).
// Output position of u in U: (#U before u) + #{c in C : (k_c, i_c) < (k_u, i_u)}
// Output position of c in C: rank_C(c) + #{u in U : (k_u, i_u) < (k_c, i_c)},
// the latter from a binary search of ko.  The result is bit-identical to a
// full stable sort; |C| = 0 gives the identity permutation.
#pragma once

#include <cstdint>

namespace ckg {

// Changed flags are one ballot word per warp of 32 stored positions (cbits,
// from key_footprint_kernel) with woff = exclusive scan of their popcounts, so
// the number of changed positions before P is
//   woff[P >> 5] + popc(cbits[P >> 5] & lanemask(P & 31)).
__device__ __forceinline__ uint32_t changed_before(const uint32_t* __restrict__ cbits,
                                                   const uint32_t* __restrict__ woff, uint64_t p) {
  const uint32_t b = __ldg(cbits + (p >> 5));
  return __ldg(woff + (p >> 5)) + uint32_t(__popc(b & ((1u << (p & 31)) - 1u)));
}

// |C| entries in index order (compacted changed list): one thread per warp
// word of changed flags, work proportional to the crossers.
__global__ void __launch_bounds__(256) compact_changed_kernel(const uint32_t* __restrict__ keys,
                                                              const uint32_t* __restrict__ cbits,
                                                              const uint32_t* __restrict__ woff, uint64_t n,
                                                              uint32_t* __restrict__ ck, uint32_t* __restrict__ ci) {
  const uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= (n + 31) / 32) return;
  uint32_t b = __ldg(cbits + w);
  uint32_t pos = __ldg(woff + w);
  while (b) {
    const uint64_t i = w * 32 + uint64_t(__ffs(b) - 1);
    ck[pos] = keys[i];
    ci[pos] = uint32_t(i);
    ++pos;
    b &= b - 1u;
  }
}

__global__ void __launch_bounds__(256) iota_kernel(uint32_t* __restrict__ p, uint64_t n) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = uint32_t(i);
}

// Unchanged particles: count changed entries ordered before (k, i).  The
// unchanged entries of a 256-position tile are in increasing (k, i) order, so
// merge_bounds_kernel binary searches once per tile for (key of its first
// unchanged entry, tile start) -- one thread per tile, all tiles in a single
// wave -- and merge_unchanged_kernel walks forward from that bound (usually
// zero or one step: only changed entries whose (key, index) falls inside the
// tile), with a binary search when the walk is long.
__device__ __forceinline__ bool changed_entry_before(const uint32_t* __restrict__ ck,
                                                     const uint32_t* __restrict__ ci, uint32_t j, uint32_t k,
                                                     uint64_t idx) {
  const uint32_t kj = __ldg(ck + j);
  return kj < k || (kj == k && uint64_t(__ldg(ci + j)) < idx);
}
__device__ __forceinline__ uint32_t changed_lower(const uint32_t* __restrict__ ck, const uint32_t* __restrict__ ci,
                                                  uint32_t lo, uint32_t hi, uint32_t k, uint64_t idx) {
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (changed_entry_before(ck, ci, mid, k, idx)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

constexpr int kMergeTile = 256;

__global__ void __launch_bounds__(256) merge_bounds_kernel(const uint32_t* __restrict__ keys,
                                                           const uint32_t* __restrict__ cbits, uint64_t n,
                                                           const uint32_t* __restrict__ ck,
                                                           const uint32_t* __restrict__ ci, uint32_t nc,
                                                           const uint32_t* __restrict__ ncp,
                                                           uint32_t* __restrict__ tile_lo) {
  if (ncp) nc = *ncp;  // device count (graph substeps)
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t base = t * kMergeTile;
  if (base >= n) return;
  uint64_t first = n;
  for (int w = 0; w < kMergeTile / 32 && base + 32 * w < n; ++w) {
    const uint32_t un = ~__ldg(cbits + (base >> 5) + w);
    if (un) {
      first = base + 32 * w + (__ffs(un) - 1);
      break;
    }
  }
  tile_lo[t] = first < n ? changed_lower(ck, ci, 0, nc, keys[first], base) : 0u;
}

// Four consecutive stored positions per thread (one 16-byte key load; the
// walk over the changed list continues from the previous position's bound,
// since a thread's unchanged entries are in increasing (key, index) order).
#ifndef CKG_MERGE_PER
#define CKG_MERGE_PER 2  // positions per thread (10M bench: 4 -> 2 saves ~13 us: the stores coalesce better)
#endif
constexpr int kMergePer = CKG_MERGE_PER;
__global__ void __launch_bounds__(256) merge_unchanged_kernel(const uint32_t* __restrict__ keys,
                                                              const uint32_t* __restrict__ cbits,
                                                              const uint32_t* __restrict__ woff, uint64_t n,
                                                              const uint32_t* __restrict__ ck,
                                                              const uint32_t* __restrict__ ci, uint32_t nc,
                                                              const uint32_t* __restrict__ ncp,
                                                              const uint32_t* __restrict__ tile_lo,
                                                              uint32_t* __restrict__ perm,
                                                              uint32_t* __restrict__ skeys) {
  const uint64_t i0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * kMergePer;
  if (i0 >= n) return;
  if (ncp) nc = *ncp;
  const uint32_t b = __ldg(cbits + (i0 >> 5));
  const uint32_t wo = __ldg(woff + (i0 >> 5));
  uint32_t k[kMergePer];
  bool vec = false;
  if constexpr (kMergePer == 4) {
    if (i0 + kMergePer <= n) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(keys) + (i0 / kMergePer));
      k[0] = v.x, k[1] = v.y, k[2] = v.z, k[3] = v.w;
      vec = true;
    }
  }
  if (!vec) {
#pragma unroll
    for (int e = 0; e < kMergePer; ++e) k[e] = i0 + e < n ? keys[i0 + e] : 0u;
  }
  uint32_t lo = __ldg(tile_lo + (i0 / kMergeTile));
  const int sh = int(i0 & 31);
#pragma unroll
  for (int e = 0; e < kMergePer; ++e) {
    const uint64_t i = i0 + e;
    if (i >= n || ((b >> (sh + e)) & 1u)) continue;
    int steps = 0;
    while (lo < nc && steps < 8 && changed_entry_before(ck, ci, lo, k[e], i)) {
      ++lo;
      ++steps;
    }
    if (steps == 8) lo = changed_lower(ck, ci, lo, nc, k[e], i);
    const uint64_t pos = (i - (wo + uint32_t(__popc(b & ((1u << (sh + e)) - 1u))))) + lo;
    perm[pos] = uint32_t(i);
    skeys[pos] = k[e];
  }
}

// Changed particles: count unchanged entries ordered before (k, j) using the
// sorted old keys ko (unchanged entries carry key == ko).
// When the previous substep's segment table is still intact (seg_begin/end
// hold the runs of ko), a non-empty run gives lower/upper_bound(ko, k)
// directly; otherwise binary search.
__global__ void __launch_bounds__(256) merge_changed_kernel(const uint32_t* __restrict__ ko,
                                                            const uint32_t* __restrict__ cbits,
                                                            const uint32_t* __restrict__ woff, uint64_t n,
                                                            const uint32_t* __restrict__ ck,
                                                            const uint32_t* __restrict__ ci, uint32_t nc,
                                                            const uint32_t* __restrict__ ncp,
                                                            const uint32_t* __restrict__ old_begin,
                                                            const uint32_t* __restrict__ old_end,
                                                            uint32_t* __restrict__ perm,
                                                            uint32_t* __restrict__ skeys) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (ncp) nc = *ncp;
  if (r >= nc) return;
  const uint32_t k = ck[r], j = ci[r];
  uint64_t lb, ub;
  const uint32_t ob = old_begin ? __ldg(old_begin + k) : 0u, oe = old_begin ? __ldg(old_end + k) : 0u;
  if (oe > ob) {
    lb = ob;
    ub = oe;
  } else {
    uint64_t lo = 0, hi = n;  // lower_bound(ko, k)
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (__ldg(ko + mid) < k) lo = mid + 1; else hi = mid;
    }
    lb = lo;
    if (!old_begin) {  // no segment table: upper_bound(ko, k) as well
      hi = n;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (__ldg(ko + mid) <= k) lo = mid + 1; else hi = mid;
      }
    }
    ub = lo;  // (with a segment table an empty run means lower == upper bound)
  }
  // positions [0, P) hold exactly the entries with (ko, idx) < (k, j)
  const uint64_t P = j < lb ? lb : (j > ub ? ub : j);
  const uint64_t cb = P < n ? changed_before(cbits, woff, P) : uint64_t(nc);
  const uint64_t pos = r + (P - cb);
  perm[pos] = j;
  skeys[pos] = k;
}

}  // namespace ckg
