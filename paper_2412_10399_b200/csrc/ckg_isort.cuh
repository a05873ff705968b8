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

__global__ void __launch_bounds__(256) changed_kernel(const uint32_t* __restrict__ keys,
                                                      const uint32_t* __restrict__ ko, uint64_t n,
                                                      uint32_t* __restrict__ chg) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) chg[i] = keys[i] != ko[i] ? 1u : 0u;
}

// After the exclusive scan: |C| and the compacted changed list (index order).
__global__ void __launch_bounds__(256) compact_changed_kernel(const uint32_t* __restrict__ keys,
                                                              const uint32_t* __restrict__ chg,
                                                              const uint32_t* __restrict__ cpre, uint64_t n,
                                                              uint32_t* __restrict__ ck, uint32_t* __restrict__ ci,
                                                              uint32_t* __restrict__ count) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (chg[i]) {
    ck[cpre[i]] = keys[i];
    ci[cpre[i]] = uint32_t(i);
  }
  if (i == n - 1) *count = cpre[i] + chg[i];
}

__global__ void __launch_bounds__(256) iota_kernel(uint32_t* __restrict__ p, uint64_t n) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = uint32_t(i);
}

// Unchanged particles: count changed entries ordered before (k, i).
__global__ void __launch_bounds__(256) merge_unchanged_kernel(const uint32_t* __restrict__ keys,
                                                              const uint32_t* __restrict__ chg,
                                                              const uint32_t* __restrict__ cpre, uint64_t n,
                                                              const uint32_t* __restrict__ ck,
                                                              const uint32_t* __restrict__ ci, uint32_t nc,
                                                              uint32_t* __restrict__ perm,
                                                              uint32_t* __restrict__ skeys) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || chg[i]) return;
  const uint32_t k = keys[i];
  uint32_t lo = 0, hi = nc;  // first c with (ck, ci) >= (k, i)
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint32_t km = __ldg(ck + mid);
    if (km < k || (km == k && __ldg(ci + mid) < uint32_t(i)))
      lo = mid + 1;
    else
      hi = mid;
  }
  const uint64_t pos = (i - cpre[i]) + lo;
  perm[pos] = uint32_t(i);
  skeys[pos] = k;
}

// Changed particles: count unchanged entries ordered before (k, j) using the
// sorted old keys ko (unchanged entries carry key == ko).
__global__ void __launch_bounds__(256) merge_changed_kernel(const uint32_t* __restrict__ ko,
                                                            const uint32_t* __restrict__ cpre, uint64_t n,
                                                            const uint32_t* __restrict__ ck,
                                                            const uint32_t* __restrict__ ci, uint32_t nc,
                                                            uint32_t* __restrict__ perm,
                                                            uint32_t* __restrict__ skeys) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nc) return;
  const uint32_t k = ck[r], j = ci[r];
  uint64_t lo = 0, hi = n;  // lower_bound(ko, k)
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(ko + mid) < k) lo = mid + 1; else hi = mid;
  }
  const uint64_t lb = lo;
  hi = n;  // upper_bound(ko, k)
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(ko + mid) <= k) lo = mid + 1; else hi = mid;
  }
  const uint64_t ub = lo;
  // positions [0, P) hold exactly the entries with (ko, idx) < (k, j)
  const uint64_t P = j < lb ? lb : (j > ub ? ub : j);
  const uint64_t changed_before = P < n ? cpre[P] : uint64_t(nc);
  const uint64_t pos = r + (P - changed_before);
  perm[pos] = j;
  skeys[pos] = k;
}

}  // namespace ckg
