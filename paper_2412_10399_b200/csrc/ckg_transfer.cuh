// ckg_transfer.cuh — block-tiled P2G, grid update and G2P kernels (sm_100a).
//
// Both transfer kernels are persistent: each CTA pulls the next active block
// (directory order) from a device work counter and processes that block's
// particle segment [seg_begin, seg_end) of the sorted order.
//
// Tile geometry: a particle whose sort key is block b has
// stencil bases inside [4b-1, 4b+4] on the +1 grid and [4b, 4b+4] on the -1
// grid (per axis, nodes up to +1 further), so a 6^3-node tile per grid with
// origin 4b (grid 0, k=-1) / 4b-1 (grid 1, k=+1) holds the whole footprint.
// The rare particles outside it (multiply/divide rounding disagreement at
// non-power-of-two dx) take a direct global path.
//
// P2G (scatter_one, transfer.hpp:235-283): each warp accumulates into a
// private FP64 tile in shared memory (no shared-memory FP64 atomics — on
// sm_100a those are CAS loops), lanes that hit the same base cell are
// serialised by match_any rank layers, and the CTA flushes the summed tile
// once per block with coalesced global REDs (native REDG.ADD.F64).
//
// G2P (gather_one + update_particle_state, transfer.hpp:465-627): the CTA
// stages the block's 2 x 6^3 nodal velocities in shared memory and every
// particle gathers its 16 nodes with a sum-factorised (separable) contraction.
#pragma once

#include <type_traits>

#include "ckg_kernels.cuh"
#include "ckg_scan.cuh"

namespace ckg {

constexpr int kTileN = 6;
constexpr int kTileNodes = kTileN * kTileN * kTileN;  // 216
constexpr int kTileVals = 2 * 4 * kTileNodes;         // 1728 (m, px, py, pz on both grids)
constexpr int kVelVals = 2 * 3 * kTileNodes;          // 1296
constexpr int kQG = 7, kQGNodes = kQG * kQG * kQG;   // quadratic G2P tile (3 x 343 <= kVelVals)
constexpr int kXferThreads = 256;
constexpr int kXferWarps = kXferThreads / 32;
// G2P CTA shape: small CTAs keep more of them resident per SM when one
// stalls at its tile-staging barrier (measured on the 10M bench: 128 x 4 and
// 64 x 8 beat 256 x 2 by 9%).
#ifndef CKG_G2P_THREADS
#define CKG_G2P_THREADS 128
#endif
#ifndef CKG_G2P_MINB
#define CKG_G2P_MINB 3
#endif
#ifndef CKG_G2P_DUAL_SINCOS
#define CKG_G2P_DUAL_SINCOS 1  // G2P: one sincos per axis for both grids
#endif
// +1 grid axes in P2G: 0 re-evaluated with a second sincos per axis, 1 rebuilt
// from the dual evaluation's scaled sine and gradient factor kept in registers
// (10M bench, P2G: FP32 0.709 -> 0.699 ms; FP64 at 4 CTAs/SM (128 registers)
// 1.511 -> 1.525 ms from the extra spills, at 3 CTAs/SM (168 registers)
// 1.299 -> 1.202 ms).
#ifndef CKG_P2G_CARRY_F64
#define CKG_P2G_CARRY_F64 1
#endif
#ifndef CKG_P2G_CARRY_F32
#define CKG_P2G_CARRY_F32 1
#endif
#ifndef CKG_G2P_MINB_F32
#define CKG_G2P_MINB_F32 4
#endif
constexpr int kG2PThreads = CKG_G2P_THREADS;
#ifndef CKG_G2P_PREFETCH
#define CKG_G2P_PREFETCH 1  // G2P: next item's velocity tile fetched with cp.async during this item
#endif
// G2P dynamic shared memory: [+1 grid sin/cos stash (6 x threads)][2 velocity tiles]
template <typename T>
constexpr size_t g2p_dyn_smem() {
  return (CKG_G2P_DUAL_SINCOS ? size_t(6) * kG2PThreads * sizeof(T) : 0) +
         (CKG_G2P_PREFETCH ? size_t(2) * kVelVals * sizeof(T) : 0);
}
constexpr int kG2PWarps = kG2PThreads / 32;
constexpr int kP2GChunk = 512;  // particles binned per pass (segment of a full lattice block)

// P2G class tiles: warp w scatters sub-octant class w only, whose bases lie in
// a 4-wide range per axis on both grids (slot 0 origin 4b, slot 1 origin
// 4b - c_a with c_a = bit a of w), so each warp-private tile is 5^3 nodes per
// grid instead of the 6^3 block halo.  8 warps x 2 x 4 x 125 FP64 = 64 KB per
// CTA, which leaves L1 room for the particle gathers and register spills.
constexpr int kPT = 5;
constexpr int kPTNodes = kPT * kPT * kPT;  // 125
// Tile layout [grid][value][node] (value stride = the grid tile's node
// count).  The +1 grid tile is either the 6^3 block halo from 4b - 1, common
// to all warps (CKG_P2G_T1FULL = 1: uniform flush), or warp w's 5^3 class
// window from 4b - c_w (0: 20 KB less shared memory per CTA).
#ifndef CKG_P2G_T1FULL
#define CKG_P2G_T1FULL 1
#endif
constexpr int kT1 = CKG_P2G_T1FULL ? kTileN : kPT;
constexpr int kT1Nodes = kT1 * kT1 * kT1;
constexpr int kWarpVals = 4 * kPTNodes + 4 * kT1Nodes;
// Warp-tile slot layout.  A class round's 32 lanes cover two lx planes of a
// 4 x 4 (ly, lz) window, which the node offsets shift over the plane; the
// dense index (lx E + ly) E + lz puts such windows on repeated banks.  FP32
// (CKG_P2G_SWZ_F32): rows of 8 slots with lz XOR-swizzled by bit 1 of ly and
// planes of 48 slots (16 mod 32 banks), so every window is conflict-free;
// 1.5x the shared memory.  Correct (GPU parity suite green) but slower: the
// 10M bench's FP32 P2G goes 0.695 -> 1.004 ms (L1 lost to the larger tiles,
// 80 -> 140 B spills), so it is off; FP64 could not fit it at all.
#ifndef CKG_P2G_SWZ_F32
#define CKG_P2G_SWZ_F32 0
#endif
// Deterministic-mode buffers (det_gather_kernel): per active block its summed
// P2G tile in the flush layout (-1 grid 4 x 5^3, then +1 grid 4 x 6^3), and
// the out-of-tile particle contributions.
constexpr int kDetVals = 4 * kPTNodes + 4 * kTileNodes;  // 1364
template <typename T>
struct DetSpill {
  uint32_t idx;  // sorted particle index
  int g;         // grid
  int base[3];   // stencil base
  T v[8][4];     // m, px, py, pz of the 8 nodes
};
template <typename T>
struct DetBuf {
  T* tile;  // null: REDG mode
  uint32_t cap;
  DetSpill<T>* spill;
  uint32_t spill_cap;
};

// FP64 (CKG_P2G_ROT64): a class round's half-warp (16 lanes, one 64-bit
// wavefront) covers a 4 x 4 (ly, lz) window at one lx, shifted over the
// plane by the node offsets.  With ly as the slowest axis and a row stride
// R = 4 (mod 16) -- slot = ly R + lx E + lz, the lx rows of one ly packed
// side by side -- the window's 16 slots are 4 ly-apart runs of 4, distinct
// mod 16, i.e. conflict-free at every offset.  +1 grid (6^3): R = 36, the
// dense size; -1 grid (5^3): R = 28 (25 used), 140 slots instead of 125.
// Measured (10M bench, ncu): shared-memory bank conflicts 86.1M -> 51.6M,
// L1 data-pipe wavefronts 331M -> 295M (77 -> 69 % of peak), spills 260 ->
// 208 B; P2G time unchanged (1.487 vs 1.492 ms): the kernel is bound by its
// per-round dependency chains at 16 warps/SM, not by the L1 data path.
#ifndef CKG_P2G_ROT64
#define CKG_P2G_ROT64 1
#endif
template <typename T>
struct P2GTile {
  static constexpr bool kSwz = sizeof(T) == 4 && CKG_P2G_SWZ_F32 && CKG_P2G_T1FULL;
  static constexpr bool kRot = sizeof(T) == 8 && CKG_P2G_ROT64 && CKG_P2G_T1FULL;
  static constexpr int R0 = kSwz ? 8 : kPT, P0 = kSwz ? 48 : kPT * kPT;  // -1 grid row / plane stride
  static constexpr int R1 = kSwz ? 8 : kT1, P1 = kSwz ? 48 : kT1 * kT1;  // +1 grid
  static constexpr int kRotR0 = 28, kRotR1 = 36;                         // kRot: ly strides
  static constexpr int N0 = kRot ? kPT * kRotR0 : kPT * P0;              // slots per value
  static constexpr int N1 = kRot ? kT1 * kRotR1 : kT1 * P1;
  static constexpr int kVals = 4 * N0 + 4 * N1;
  __device__ static __forceinline__ int col(int ly, int lz) { return kSwz ? (lz ^ ((ly & 2) << 1)) : lz; }
  __device__ static __forceinline__ int slot(int g, int lx, int ly, int lz) {
    if constexpr (kRot) return g ? ly * kRotR1 + lx * kT1 + lz : ly * kRotR0 + lx * kPT + lz;
    if constexpr (!kSwz) return g ? (lx * kT1 + ly) * kT1 + lz : (lx * kPT + ly) * kPT + lz;
    return g ? lx * P1 + ly * R1 + col(ly, lz) : lx * P0 + ly * R0 + col(ly, lz);
  }
  // slot steps of a unit node offset in x / y (unswizzled layouts)
  __host__ __device__ static constexpr int sx(int g) { return kRot ? (g ? kT1 : kPT) : (g ? kT1 * kT1 : kPT * kPT); }
  __host__ __device__ static constexpr int sy(int g) { return kRot ? (g ? kRotR1 : kRotR0) : (g ? kT1 : kPT); }
  // node of a flush slot; false for a padding slot
  __device__ static __forceinline__ bool node(int g, int sl, int& i, int& j, int& k) {
    const int E = g ? kT1 : kPT;
    if constexpr (kRot) {
      const int R = g ? kRotR1 : kRotR0;
      j = sl / R;
      const int r = sl % R;
      i = r / E;
      k = r % E;
      return i < E;
    } else if constexpr (kSwz) {
      const int P = g ? P1 : P0, R = g ? R1 : R0;
      i = sl / P;
      j = (sl % P) / R;
      k = col(j, sl % R);
      return j < E && k < E;
    } else {
      i = sl / (E * E);
      j = (sl / E) % E;
      k = sl % E;
      return true;
    }
  }
};
template <typename T>
__device__ __forceinline__ void tile_add4(T* p, const T (&o)[4], int vs) {
  // all four loads issued before the first add
  const T a0 = p[0], a1 = p[vs], a2 = p[2 * vs], a3 = p[3 * vs];
  p[0] = a0 + o[0];
  p[vs] = a1 + o[1];
  p[2 * vs] = a2 + o[2];
  p[3 * vs] = a3 + o[3];
}
// Compact-kernel P2G CTA: kP2GWarps warps, each scattering CKG_P2G_CPW of
// the 8 sub-octant classes in turn into its own tile (any class fits the
// common tile layout when the +1 grid tile is the full halo).
#ifndef CKG_P2G_CPW
#define CKG_P2G_CPW 2
#endif
static_assert(CKG_P2G_CPW == 1 || CKG_P2G_T1FULL, "several classes per warp need the full +1 grid tile");
constexpr int kP2GWarps = 8 / CKG_P2G_CPW;
constexpr int kP2GThreads = 32 * kP2GWarps;
// Resident P2G CTAs (4 warps each) per SM the register budget is compiled
// for.  10M bench: FP64 3 CTAs = 168 registers, 24 B of spills: 1.20 ms
// (4 CTAs = 128 registers, 260 B of spills: 1.49 ms; 2 CTAs: 1.42 ms);
// FP32 5 CTAs = 96 registers: 0.661 ms (6: 0.692, 4: 0.721).  The spills
// were the cost: at 4 CTAs the 106 KB per SM of spilled state does not fit
// the L1 left beside the tiles, so every reload went to L2.
#ifndef CKG_P2G_MINCTAS_F64
#define CKG_P2G_MINCTAS_F64 3
#endif
#ifndef CKG_P2G_MINCTAS_F32
#define CKG_P2G_MINCTAS_F32 5
#endif
template <typename T>
constexpr int p2g_min_ctas() {
  return sizeof(T) == 4 ? CKG_P2G_MINCTAS_F32 : CKG_P2G_MINCTAS_F64;
}
template <typename T>
constexpr size_t p2g_smem_bytes() {
  return size_t(kP2GWarps) * P2GTile<T>::kVals * sizeof(T);
}

__device__ __forceinline__ void decode_key(uint32_t key, int D, int& bx, int& by, int& bz) {
  bz = int(key % uint32_t(D));
  by = int((key / uint32_t(D)) % uint32_t(D));
  bx = int(key / (uint32_t(D) * uint32_t(D)));
}

// Global pool offset of node (gi, gj, gk) on grid g through the block's 3^3
// neighbour slots (nbr[(ox*3+oy)*3+oz], o = node block - key block + 1).
__device__ __forceinline__ int64_t nbr_offset(const int32_t* nbr, int g, int gi, int gj, int gk, int bx, int by,
                                              int bz) {
  const int ox = (gi >> 2) - bx + 1, oy = (gj >> 2) - by + 1, oz = (gk >> 2) - bz + 1;
  if (ox < 0 || oy < 0 || oz < 0 || ox > 2 || oy > 2 || oz > 2) return -1;
  const int32_t slot = nbr[(ox * 3 + oy) * 3 + oz];
  if (slot < 0) return -1;
  return int64_t(slot) * kBlockVals + g * 256 + (((gi & 3) << 4) | ((gj & 3) << 2) | (gk & 3));
}

// ---- cp.async (global -> shared, L1-allocating); a false predicate
// zero-fills the destination
__device__ __forceinline__ void cp_async4(void* sm, const void* gm, bool pred) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gm), "r"(pred ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async8(void* sm, const void* gm, bool pred) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gm), "r"(pred ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_t(double* sm, const double* gm, bool pred) { cp_async8(sm, gm, pred); }
__device__ __forceinline__ void cp_async_t(float* sm, const float* gm, bool pred) { cp_async4(sm, gm, pred); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ---- per-item records (one per active block, built once per substep by
// xfer_prep_kernel and read by both transfer kernels with a single 160-byte
// load instead of the active -> segment -> directory lookup chain)
constexpr int kRecWords = 40;
constexpr int kRecKey = 0, kRecS0 = 1, kRecS1 = 2, kRecNbr = 4, kRecCls = 32;

// Sub-octant class of a particle (frac(x/dx - 1/4) >= 1/2 per axis): particles
// of one class have distinct -1 and +1 grid bases as soon as their +1 cells
// differ, so a warp scattering one class sees (for lattice-like layouts) a
// single rank layer per grid.
template <typename T>
__device__ __forceinline__ uint32_t subocta_class(const PState<T>& p, uint32_t src, const StepConst<T>& c) {
  uint32_t q = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const T sa = sub_rn(over_dx(__ldg(p.f + uint64_t(kX + a) * p.stride + src), c.dx, c.inv_dx, c.pow2), T(0.25));
    q |= ((sa - dfloor(sa)) >= T(0.5) ? 1u : 0u) << a;
  }
  return q;
}

// Transfer preparation (after activation + segments), one warp per active
// item: its record {key, s0, s1, 27 neighbour slots, class counts of chunk 0},
// and for the compact kernel's P2G the class order of every 512-particle
// chunk of its segment: cord[cb + j] = state index of the j-th particle of
// the chunk in (class, sorted position) order — stable and deterministic
// (ballot ranks, no atomics).  Class counts of chunks past the first go to
// ccnt[cb >> 9] (chunk starts past a segment's first are >= 513 apart, so the
// index is unique).  Warps are independent (no CTA barriers) and each issues
// its chunk's loads four 32-particle groups at a time, so the item's short
// dependency chain (active -> segment -> perm -> x) is hidden by the other
// warps in flight.
constexpr int kPrepWarps = 8;
template <typename T>
__global__ void __launch_bounds__(kPrepWarps * 32, 4) xfer_prep_kernel(
    PState<T> cur, const uint32_t* __restrict__ perm, StepConst<T> c, const int32_t* __restrict__ dir,
    const uint32_t* __restrict__ active, const uint32_t* __restrict__ seg_begin,
    const uint32_t* __restrict__ seg_end, uint32_t cap, const DevStatus* st, uint32_t* __restrict__ rec,
    uint32_t* __restrict__ cord, uint4* __restrict__ ccnt, const uint8_t* __restrict__ cls) {
  constexpr int kG = kP2GChunk / 32;  // 32-particle groups per chunk
  const int lane = threadIdx.x & 31;
  const uint32_t na = min(st->item_hi, cap), lo = st->item_lo;
  const uint32_t lt = lanemask_lt();
  const int D = c.D;
  const uint32_t nwarps = gridDim.x * kPrepWarps;
  __shared__ uint32_t wcnt[kPrepWarps][8];
  const int wib = threadIdx.x >> 5;
  for (uint32_t item = lo + blockIdx.x * kPrepWarps + (threadIdx.x >> 5); item < na; item += nwarps) {
    const uint32_t key = __ldg(active + item);
    const uint32_t s0 = __ldg(seg_begin + key), s1 = __ldg(seg_end + key);
    uint32_t* r = rec + uint64_t(item) * kRecWords;
    {
      int bx, by, bz;
      decode_key(key, D, bx, by, bz);
      uint32_t w = 0;
      if (lane == kRecKey) w = key;
      else if (lane == kRecS0) w = s0;
      else if (lane == kRecS1) w = s1;
      else if (lane >= kRecNbr && lane < kRecNbr + 27) {
        const int t = lane - kRecNbr;
        w = uint32_t(pool_slot(dir, D, bx - 1 + t / 9, by - 1 + (t / 3) % 3, bz - 1 + t % 3, c.dense));
      }
      r[lane] = w;
    }
    if (!cls || s1 <= s0) {
      if (lane < kRecWords - kRecCls) r[kRecCls + lane] = 0u;
      continue;
    }
    for (uint32_t cb = s0; cb < s1; cb += kP2GChunk) {
      const uint32_t len = min(uint32_t(kP2GChunk), s1 - cb);
      uint32_t src[kG];
      uint32_t qp[2] = {0u, 0u};  // 4-bit class per group (8 = none)
      if (lane < 8) wcnt[wib][lane] = 0u;
      __syncwarp();
      // pass 1: classes (from the key pass), four groups' loads in flight at
      // a time; per-class totals accumulated by each class's leader lane
#pragma unroll
      for (int g0 = 0; g0 < kG; g0 += 4) {
        uint32_t qs[4];
#pragma unroll
        for (int g = g0; g < g0 + 4; ++g) {
          const uint32_t j = uint32_t(g) * 32 + lane;
          src[g] = j < len ? __ldg(perm + cb + j) : 0u;
        }
#pragma unroll
        for (int g = g0; g < g0 + 4; ++g) {
          const uint32_t j = uint32_t(g) * 32 + lane;
          qs[g - g0] = j < len ? uint32_t(__ldg(cls + src[g])) : 8u;
        }
#pragma unroll
        for (int g = g0; g < g0 + 4; ++g) {
          const uint32_t q = qs[g - g0];
          qp[g >> 3] |= q << (4 * (g & 7));
          const uint32_t peers = __match_any_sync(0xffffffffu, q);
          if (q < 8u && (peers & lt) == 0u) wcnt[wib][q] += __popc(peers);
          __syncwarp();
        }
      }
      const uint32_t tot = lane < 8 ? wcnt[wib][lane] : 0u;
      // class bases: exclusive scan of the 8 totals (lanes 0..7)
      uint32_t base = tot;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, base, o);
        if (lane >= o) base += u;
      }
      base -= tot;
      __syncwarp();
      if (lane < 8) wcnt[wib][lane] = base;  // next position of class lane
      __syncwarp();
      // pass 2: positions (class base + earlier groups of the class + rank)
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const uint32_t q = (qp[g >> 3] >> (4 * (g & 7))) & 0xfu;
        const uint32_t peers = __match_any_sync(0xffffffffu, q);
        if (q < 8u) {
          cord[cb + wcnt[wib][q] + __popc(peers & lt)] = src[g];
        }
        __syncwarp();
        if (q < 8u && (peers & lt) == 0u) wcnt[wib][q] += __popc(peers);
        __syncwarp();
      }
      // chunk class counts (u16 pairs)
      uint32_t pair = tot | (__shfl_down_sync(0xffffffffu, tot, 1) << 16);
      if (lane < 8 && !(lane & 1)) {
        if (cb == s0) r[kRecCls + (lane >> 1)] = pair;
        else reinterpret_cast<uint32_t*>(ccnt + (cb >> 9))[lane >> 1] = pair;
      }
      if (cb == s0 && lane >= 4 && lane < kRecWords - kRecCls) r[kRecCls + lane] = 0u;
    }
  }
}

// One grid's 8-node scatter of one particle (scatter_one, transfer.hpp:
// 235-283) in separable form: with w = wx_s wy_t wz_u, grad w = (gx_s wy_t
// wz_u, wx_s gy_t wz_u, wx_s wy_t gz_u) (g1 = -g0 per axis) and the node
// momentum base b = u0 + dx (s, t, u) . Q_a, the contribution
// w b - A grad w regroups exactly into
//   mass(s,t,u)  = (m wx_s) (wy_t wz_u)
//   mom_a(s,t,u) = X_a(s) (wy_t wz_u) + wx_s (Y_a(t) wz_u + wy_t Z_a(u)),
//   X_a(s) = wx_s (u0_a + s dx Q_a0) - A_a0 gx_s,  Y_a(t) = t dx Q_a1 wy_t - A_a1 gy_t,
//   Z_a(u) = u dx Q_a2 wz_u - A_a2 gz_u
// (~130 FP64 operations per grid instead of ~200; same sum up to the
// rounding of the regrouping).  Node offsets are visited in the order
// (t, u) outer, s inner so each Y/Z pair is formed once.  Used for FP32
// (0.668 -> 0.661 ms); FP64 at 168 registers keeps the direct form (1.219
// -> 1.202 ms: fewer live values across the node loop, 44 -> 24 B spills).
#ifndef CKG_P2G_SEPARABLE_F64
#define CKG_P2G_SEPARABLE_F64 0
#endif
#ifndef CKG_P2G_SEPARABLE_F32
#define CKG_P2G_SEPARABLE_F32 1
#endif
// P2G: the two grids' scatters as a rolled loop (half the code: instruction
// cache) instead of unrolled
#ifndef CKG_P2G_ROLL_GRIDS
#define CKG_P2G_ROLL_GRIDS 0
#endif
template <typename T, int SCHEME, bool SWZ>
__device__ __forceinline__ void scatter_separable(const Axis<T> (&ax)[3], T m, const T (&u0)[3], const M3<T>& Q,
                                                  const M3<T>& Ap, T dx, T* tb, T* p0, int g, int lx, int ly,
                                                  int lz, int E, int VS, uint32_t tmask) {
  const T wx0 = ax[0].w0, wx1 = ax[0].w1, wy0 = ax[1].w0, wy1 = ax[1].w1, wz0 = ax[2].w0, wz1 = ax[2].w1;
  const T gx = ax[0].g0, gy = ax[1].g0, gz = ax[2].g0;
  T X0[3], X1[3], Y0[3], Y1[3], Z0[3], Z1[3];
  // MLS: the force is already folded into u0 / Q (no gradient term)
  constexpr bool kGrad = SCHEME != kSchemeMls;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const T u = u0[a];
    if constexpr (!kGrad) {
      X0[a] = wx0 * u;
      X1[a] = wx1 * fma(Q.a[a][0], dx, u);
      Y0[a] = Z0[a] = T(0);
      Y1[a] = (Q.a[a][1] * dx) * wy1;
      Z1[a] = (Q.a[a][2] * dx) * wz1;
      continue;
    }
    X0[a] = wx0 * u - Ap.a[a][0] * gx;
    Y0[a] = -(Ap.a[a][1] * gy);
    Z0[a] = -(Ap.a[a][2] * gz);
    if constexpr (SCHEME != kSchemePic) {
      X1[a] = wx1 * fma(Q.a[a][0], dx, u) + Ap.a[a][0] * gx;
      Y1[a] = (Q.a[a][1] * dx) * wy1 + Ap.a[a][1] * gy;
      Z1[a] = (Q.a[a][2] * dx) * wz1 + Ap.a[a][2] * gz;
    } else {
      X1[a] = wx1 * u + Ap.a[a][0] * gx;
      Y1[a] = Ap.a[a][1] * gy;
      Z1[a] = Ap.a[a][2] * gz;
    }
  }
  const T mw0 = m * wx0, mw1 = m * wx1;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const T wyt = t ? wy1 : wy0, wzu = u ? wz1 : wz0;
      const T wyz = wyt * wzu;
      T YZ[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) YZ[a] = (t ? Y1[a] : Y0[a]) * wzu + wyt * (u ? Z1[a] : Z0[a]);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        T o[4];
        o[0] = (s ? mw1 : mw0) * wyz;
#pragma unroll
        for (int a = 0; a < 3; ++a) o[1 + a] = (s ? X1[a] : X0[a]) * wyz + (s ? wx1 : wx0) * YZ[a];
        if constexpr (SWZ)
          tile_add4(tb + P2GTile<T>::slot(g, lx + s, ly + t, lz + u), o, VS);
        else
          tile_add4(p0 + s * P2GTile<T>::sx(g) + t * P2GTile<T>::sy(g) + u, o, VS);
        // node (s,t,u) of one lane can be another offset's node of its
        // neighbour: order the read-modify-writes across lanes
        __syncwarp(tmask);
      }
    }
}

// DET: deterministic mode (per-block tiles stored for det_gather_kernel);
// a separate instance so the default kernel carries none of its code.
template <typename T, int SCHEME, bool DET = false>
__global__ void __launch_bounds__(kP2GThreads, p2g_min_ctas<T>())
    p2g_tile_kernel(PState<T> cur, const uint32_t* __restrict__ perm, StepConst<T> c,
                    const int32_t* __restrict__ dir, const uint32_t* __restrict__ rec,
                    const uint32_t* __restrict__ cord, const uint4* __restrict__ ccnt,
                    T* __restrict__ pool, uint32_t cap, DevStatus* st, int step, DetBuf<T> det) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tiles = reinterpret_cast<T*>(smem_raw);
  // Items are claimed two ahead: while item k is processed, warp 0's claim of
  // item k+2 is in flight (its atomic issued at the start of item k, its
  // record fetched with cp.async during item k's flush), and item k+1's
  // record is already in shared memory -- no claim latency between items.
  __shared__ uint32_t s_recb[3][kRecWords];
  __shared__ uint32_t s_itemb[3];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  using L = P2GTile<T>;
  T* wt = tiles + warp * L::kVals;
  for (int e = tid; e < kP2GWarps * L::kVals; e += kP2GThreads) tiles[e] = T(0);
  const uint32_t na = min(st->item_hi, cap), item0 = st->item_lo;
  const uint32_t lt = lanemask_lt();
  const int D = c.D;
  const T dx = c.dx, dt = step_dt(c);
  // warp 0: publish a claimed item and fetch its record (async)
  auto stage = [&](int b, uint32_t it) {
    if (lane == 0) s_itemb[b] = it;
    if (it < na) {
      const uint32_t* r = rec + uint64_t(it) * kRecWords;
      cp_async4(&s_recb[b][lane], r + lane, true);
      if (lane < kRecWords - 32) cp_async4(&s_recb[b][32 + lane], r + 32 + lane, true);
    }
    cp_async_commit();
  };
  if (warp == 0) {
    uint32_t a = 0, b = 0;
    if (lane == 0) {
      a = item0 + atomicAdd(&st->work[0], 1u);
      b = item0 + atomicAdd(&st->work[0], 1u);
    }
    stage(0, __shfl_sync(0xffffffffu, a, 0));
    stage(1, __shfl_sync(0xffffffffu, b, 0));
  }
  for (int k = 0;; ++k) {
    const int buf = k % 3;
    if (warp == 0) asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // record k (and k+1 unless newest)
    __syncthreads();
    const uint32_t item = s_itemb[buf];
    if (item >= na) break;
    uint32_t pend = 0;  // claim of item k+2
    if (tid == 0) pend = item0 + atomicAdd(&st->work[0], 1u);
    const uint32_t* s_rec = s_recb[buf];
    const int32_t* nbr = reinterpret_cast<const int32_t*>(s_rec + kRecNbr);
    const uint32_t key = s_rec[kRecKey];
    const uint32_t s0 = s_rec[kRecS0], s1 = s_rec[kRecS1];
    if (s1 <= s0) {
      // deterministic mode: an empty block (activation halo) contributes a
      // zero tile (its slot may hold a stale one from an earlier substep)
      if (DET && item < det.cap)
        for (int e = tid; e < kDetVals; e += kP2GThreads) det.tile[uint64_t(item) * kDetVals + e] = T(0);
      if (warp == 0) stage((k + 2) % 3, __shfl_sync(0xffffffffu, pend, 0));
      continue;
    }
    int bx, by, bz;
    decode_key(key, D, bx, by, bz);
    for (uint32_t cb = s0; cb < s1; cb += kP2GChunk) {
#pragma unroll 1
    for (int ci = 0; ci < CKG_P2G_CPW; ++ci) {
      const int cl = warp + ci * kP2GWarps;  // this pass's sub-octant class
      const int cx = cl & 1, cy = (cl >> 1) & 1, cz = (cl >> 2) & 1;  // class bits
      // this warp's class list of the chunk (xfer_prep_kernel)
      uint32_t my_cnt = 0, my_off = 0;
      {
        uint4 v;
        if (cb == s0) v = make_uint4(s_rec[kRecCls], s_rec[kRecCls + 1], s_rec[kRecCls + 2], s_rec[kRecCls + 3]);
        else v = __ldg(ccnt + (cb >> 9));
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t cq = (w4[q >> 1] >> (16 * (q & 1))) & 0xffffu;
          if (q < cl) my_off += cq;
          if (q == cl) my_cnt = cq;
        }
      }
      for (uint32_t rb = 0; rb < my_cnt; rb += 32) {
      const bool in_round = rb + lane < my_cnt;
      const uint32_t src = in_round ? __ldg(cord + cb + my_off + rb + lane) : 0u;
      // sorted index of this particle, for error reports only (rare path)
      auto sorted_index = [&]() -> uint32_t {
        for (uint32_t k = cb; k < min(cb + uint32_t(kP2GChunk), s1); ++k)
          if (__ldg(perm + k) == src) return k;
        return cb;
      };
      bool valid = in_round;
      // ---- per-particle state (scatter_all, simulation.hpp:289-324)
      T x = 0, y = 0, z = 0, m = 0;
      T mv[3] = {0, 0, 0};
      M3<T> Ap, Q, Bp;  // Ap = dt * V0 * tau, Q = m * C
      T Minv[4][4];
      Dual<T> ds;
      constexpr bool kCarry = (sizeof(T) == 4 ? CKG_P2G_CARRY_F32 : CKG_P2G_CARRY_F64) != 0;
      T c_sn[3] = {0, 0, 0}, c_g0[3] = {0, 0, 0};  // kCarry: +1 grid scaled sines, gradient factors
      if (valid) {
        // every field load is issued before the first use
        const uint64_t n = cur.stride;  // field stride (buffer capacity)
        T v3[3], t6[6];
        x = __ldg(cur.f + kX * n + src);
        y = __ldg(cur.f + (kX + 1) * n + src);
        z = __ldg(cur.f + (kX + 2) * n + src);
        m = __ldg(cur.f + kMass * n + src);
#pragma unroll
        for (int k = 0; k < 3; ++k) v3[k] = __ldg(cur.f + (kV + k) * n + src);
#pragma unroll
        for (int k = 0; k < 6; ++k) t6[k] = __ldg(cur.tau + uint64_t(k) * n + src);
        if (SCHEME != kSchemePic) Bp = load_m3(cur, kB, src);
#pragma unroll
        for (int k = 0; k < 3; ++k) mv[k] = m * v3[k];
        // dt * V0 * tau from the stress cache written by the previous G2P
        // (or the initial stress pass): P2G runs no constitutive model.
#pragma unroll
        for (int k = 0; k < 6; ++k) t6[k] = dt * t6[k];
        Ap.a[0][0] = t6[0];
        Ap.a[0][1] = Ap.a[1][0] = t6[1];
        Ap.a[0][2] = Ap.a[2][0] = t6[2];
        Ap.a[1][1] = t6[3];
        Ap.a[1][2] = Ap.a[2][1] = t6[4];
        Ap.a[2][2] = t6[5];
        if constexpr (kCarry) {
          ds = dual_stencil_sn(x, y, z, dx, c.inv_dx, c.pow2, c_sn);
#pragma unroll
          for (int k = 0; k < 3; ++k) c_g0[k] = ds.ax[1][k].g0;
        } else {
          ds = dual_stencil(x, y, z, dx, c.inv_dx, c.pow2);
        }
        if (SCHEME != kSchemePic) {
          M3<T> Di;
          if (!apic_d_inverse(apic_D(ds, dx), Di)) {
            record_error(st, step, kPhaseP2G, sorted_index(), 0, kErrNearSingularD);
            valid = false;
          }
          Q = scale(m, mul(Bp, Di));  // m * B D^-1
        }
        if (SCHEME == kSchemeMls) {
          T Mm[4][4];
          mls_moment(ds, dx, Mm);
          if (!gauss_inverse4(Mm, Minv)) {
            record_error(st, step, kPhaseP2G, sorted_index(), 0, kErrSingularMls);
            valid = false;
          }
          // scatter_force_mls_one (transfer.hpp:335-369) adds -A' w (M^-1
          // P(xi))_{1..3} per node, P(xi) = (1, xi): with K = A' M^-1_{1..3,:}
          // (3 x 4) that is -w (K_0 + K_{1..3} xi), an affine function of the
          // node offset like the APIC term w (m v + Q xi).  Folded into the
          // latter (Q <- Q - K_{1..3}, m v <- m v - K_0) the MLS node
          // contribution is the APIC one without a gradient term.
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            T k4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              k4[k] = Ap.a[a][0] * Minv[1][k] + Ap.a[a][1] * Minv[2][k] + Ap.a[a][2] * Minv[3][k];
            mv[a] -= k4[0];
#pragma unroll
            for (int j = 0; j < 3; ++j) Q.a[a][j] -= k4[1 + j];
          }
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) Ap.a[a][b] = T(0);
        }
      }
      // ---- scatter, grid by grid.  Only one grid's stencil is live during
      // its scatter: the +1 grid's axes are re-evaluated (axis_pair with
      // k = +1/4 is bit-identical to the dual evaluation) instead of being
      // carried through the -1 grid's scatter, which frees the registers
      // that let each node's four read-modify-writes overlap.
#if CKG_P2G_ROLL_GRIDS
#pragma unroll 1
#else
#pragma unroll
#endif
      for (int g = 0; g < 2; ++g) {
        Axis<T> ax[3];
        if (g == 0) {
          ax[0] = ds.ax[0][0];
          ax[1] = ds.ax[0][1];
          ax[2] = ds.ax[0][2];
        } else {
          if constexpr (kCarry) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
              ax[k] = axis_plus_carried(k == 0 ? x : k == 1 ? y : z, dx, c.inv_dx, c.pow2, c_sn[k], c_g0[k]);
          } else {
            ax[0] = axis_pair(x, dx, c.inv_dx, c.pow2, T(0.25));
            ax[1] = axis_pair(y, dx, c.inv_dx, c.pow2, T(0.25));
            ax[2] = axis_pair(z, dx, c.inv_dx, c.pow2, T(0.25));
          }
        }
        // tile edge and origin shift of this grid (see kT1)
        const int E = g ? kT1 : kPT, VS = g ? L::N1 : L::N0;
        const int shx = g ? (CKG_P2G_T1FULL ? 1 : cx) : 0, shy = g ? (CKG_P2G_T1FULL ? 1 : cy) : 0,
                  shz = g ? (CKG_P2G_T1FULL ? 1 : cz) : 0;
        const int lx = ax[0].base - (4 * bx - shx), ly = ax[1].base - (4 * by - shy), lz = ax[2].base - (4 * bz - shz);
        const bool in_tile =
            valid && lx >= 0 && ly >= 0 && lz >= 0 && lx <= E - 2 && ly <= E - 2 && lz <= E - 2;
        const uint32_t cell = in_tile ? uint32_t((lx * E + ly) * E + lz) : (1024u + lane);
        const uint32_t peers = __match_any_sync(0xffffffffu, cell);
        const uint32_t rank = __popc(peers & lt);
        const uint32_t maxrank = __reduce_max_sync(0xffffffffu, rank);
        const uint32_t tmask = __ballot_sync(0xffffffffu, in_tile);
        // node momentum base b_stu = m v + Q xi_stu = u0 + dx (s Qx + t Qy + u Qz)
        T u0[3] = {mv[0], mv[1], mv[2]};
        if (SCHEME != kSchemePic) {
#pragma unroll
          for (int a = 0; a < 3; ++a)
            u0[a] += Q.a[a][0] * ax[0].xi0 + Q.a[a][1] * ax[1].xi0 + Q.a[a][2] * ax[2].xi0;
        }
        // Node contribution (m w, w b - A' grad w) or, for MLS, the force
        // through grad Phi = w M^-1 P(xi) (transfer.hpp:335-369).
        // (selects, not arrays indexed by s/t/u: the rolled paths below
        // would otherwise put the axis weights in local memory)
        auto contrib = [&](int s, int t, int u, T (&o)[4]) {
          const T wxs = s ? ax[0].w1 : ax[0].w0, wyt = t ? ax[1].w1 : ax[1].w0, wzu = u ? ax[2].w1 : ax[2].w0;
          const T wyz = wyt * wzu;
          const T w = wxs * wyz;
          T gw0 = T(0), gw1 = T(0), gw2 = T(0);
          if (SCHEME != kSchemeMls) {  // MLS: force folded into u0 / Q above
            const T gxs = s ? -ax[0].g0 : ax[0].g0, gyt = t ? -ax[1].g0 : ax[1].g0, gzu = u ? -ax[2].g0 : ax[2].g0;
            gw0 = gxs * wyz;
            gw1 = wxs * (gyt * wzu);
            gw2 = wxs * (wyt * gzu);
          }
          o[0] = w * m;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            T b = u0[a];
            if (SCHEME != kSchemePic) {
              // + Q (s, t, u) dx, fused (no dx-scaled copy of Q kept live)
              if (s) b = fma(Q.a[a][0], dx, b);
              if (t) b = fma(Q.a[a][1], dx, b);
              if (u) b = fma(Q.a[a][2], dx, b);
            }
            o[1 + a] = SCHEME == kSchemeMls ? w * b
                                             : w * b - (Ap.a[a][0] * gw0 + Ap.a[a][1] * gw1 + Ap.a[a][2] * gw2);
          }
        };
        T* tb = wt + g * 4 * L::N0;  // this grid's tile
        T* p0 = tb + (L::kSwz ? 0 : L::slot(g, lx, ly, lz));  // unswizzled layouts
        if (maxrank == 0) {
          // fast path: every lane owns a distinct base cell in this warp, so
          // at a fixed node offset all lanes write distinct nodes
          if (in_tile) {
            if constexpr ((sizeof(T) == 8 ? CKG_P2G_SEPARABLE_F64 : CKG_P2G_SEPARABLE_F32) != 0) {
              scatter_separable<T, SCHEME, L::kSwz>(ax, m, u0, Q, Ap, dx, tb, p0, g, lx, ly, lz, E, VS, tmask);
            } else {
#pragma unroll
            for (int s = 0; s < 2; ++s)
#pragma unroll
              for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  T o[4];
                  contrib(s, t, u, o);
                  if constexpr (L::kSwz)
                    tile_add4(tb + L::slot(g, lx + s, ly + t, lz + u), o, VS);
                  else
                    tile_add4(p0 + s * L::sx(g) + t * L::sy(g) + u, o, VS);
                  // node (s,t,u) of one lane can be node (0,0,0) of its
                  // neighbour: order the read-modify-writes across lanes
                  __syncwarp(tmask);
                }
            }
          }
        } else {
          // shared base cells: serialise by rank layers (rolled loop)
#pragma unroll 1
          for (int nid = 0; nid < 8; ++nid) {
            const int s = nid >> 2, t = (nid >> 1) & 1, u = nid & 1;
            T o[4];
            contrib(s, t, u, o);
            T* p = L::kSwz ? tb + L::slot(g, lx + s, ly + t, lz + u) : p0 + s * L::sx(g) + t * L::sy(g) + u;
            for (uint32_t layer = 0; layer <= maxrank; ++layer) {
              if (in_tile && rank == layer) tile_add4(p, o, VS);
              __syncwarp();
            }
          }
        }
        if (DET && valid && !in_tile) {
          // deterministic mode: the contribution is recorded and applied in
          // sorted-particle order after the tile gather (det_spill_kernel)
          const uint32_t k = atomicAdd(&st->spill_n, 1u);
          if (k >= det.spill_cap) {
            atomicOr(&st->overflow, 4u);
          } else {
            DetSpill<T>& e = det.spill[k];
            e.idx = sorted_index();
            e.g = g;
            e.base[0] = ax[0].base;
            e.base[1] = ax[1].base;
            e.base[2] = ax[2].base;
#pragma unroll 1
            for (int nid = 0; nid < 8; ++nid) {
              T o[4];
              contrib(nid >> 2, (nid >> 1) & 1, nid & 1, o);
#pragma unroll
              for (int q = 0; q < 4; ++q) e.v[nid][q] = o[q];
            }
          }
        } else if (valid && !in_tile) {
          // footprint outside the block tile: direct REDs through the directory
#pragma unroll 1
          for (int nid = 0; nid < 8; ++nid) {
            const int s = nid >> 2, t = (nid >> 1) & 1, u = nid & 1;
            T o[4];
            contrib(s, t, u, o);
            const int gi = ax[0].base + s, gj = ax[1].base + t, gk = ax[2].base + u;
            const int32_t slot = pool_slot(dir, D, gi >> 2, gj >> 2, gk >> 2, c.dense);
            if (slot < 0 || uint32_t(slot) >= cap) {
              record_error(st, step, kPhaseP2G, sorted_index(), 0, kErrInactive);
            } else {
              T* nd = pool + node_off(slot, g, gi, gj, gk);
              atomicAdd(nd, o[0]);
              atomicAdd(nd + 64, o[1]);
              atomicAdd(nd + 128, o[2]);
              atomicAdd(nd + 192, o[3]);
            }
          }
        }
      }
      }  // rounds of this warp's class list
    }  // classes of this warp
    }
    __syncthreads();
    if (warp == 0) stage((k + 2) % 3, __shfl_sync(0xffffffffu, pend, 0));
    // ---- flush: sum the warp tiles, one REDG per non-zero node value.
    // Slot 0: all class tiles share origin 4b (5^3).  Slot 1: the 6^3 halo
    // from 4b - 1 (T1FULL: every warp's tile is that halo; else warp w's
    // 5^3 window covers offsets [1 - c, 5 - c] per axis).
    constexpr int F1 = CKG_P2G_T1FULL ? L::N1 : kTileNodes;  // +1 grid flush slots per value
    for (int e = tid; e < 4 * L::N0 + 4 * F1; e += kP2GThreads) {
      T sum = T(0);
      int g, v, i, j, k;
      if (e < 4 * L::N0) {
        g = 0;
        v = e / L::N0;
        if (!L::node(0, e % L::N0, i, j, k)) continue;  // padding slot
#pragma unroll
        for (int w = 0; w < kP2GWarps; ++w) {
          T* q = tiles + w * L::kVals + e;
          sum += *q;
          *q = T(0);
        }
      } else {
        g = 1;
        const int e1 = e - 4 * L::N0;
        v = e1 / F1;
        if (CKG_P2G_T1FULL ? !L::node(1, e1 % F1, i, j, k) : false) continue;  // padding slot
        if (!CKG_P2G_T1FULL) {
          const int sl = e1 % F1;
          i = sl / (kTileN * kTileN);
          j = (sl / kTileN) % kTileN;
          k = sl % kTileN;
        }
#pragma unroll
        for (int w = 0; w < kP2GWarps; ++w) {
          if (CKG_P2G_T1FULL) {
            T* q = tiles + w * L::kVals + e;
            sum += *q;
            *q = T(0);
          } else {
            const int li = i - 1 + (w & 1), lj = j - 1 + ((w >> 1) & 1), lk = k - 1 + ((w >> 2) & 1);
            if (li >= 0 && lj >= 0 && lk >= 0 && li < kPT && lj < kPT && lk < kPT) {
              T* q = tiles + w * L::kVals + 4 * kPTNodes + v * kT1Nodes + (li * kPT + lj) * kPT + lk;
              sum += *q;
              *q = T(0);
            }
          }
        }
      }
      if constexpr (DET) {
        // deterministic mode: the block's summed tile is stored as is; the
        // nodes are summed over the neighbouring tiles in a fixed order by
        // det_gather_kernel
        // (det_gather_kernel's dense layout: -1 grid 4 x 5^3, then +1 grid 4 x 6^3)
        const int de = g == 0 ? v * kPTNodes + (i * kPT + j) * kPT + k
                              : 4 * kPTNodes + v * kTileNodes + (i * kTileN + j) * kTileN + k;
        if (item < det.cap) det.tile[uint64_t(item) * kDetVals + de] = sum;
        else if (e == 0) atomicOr(&st->overflow, 2u);
      } else if (sum != T(0)) {
        const int gi = 4 * bx - g + i, gj = 4 * by - g + j, gk = 4 * bz - g + k;
        const int64_t off = nbr_offset(nbr, g, gi, gj, gk, bx, by, bz);
        if (off < 0 || uint64_t(off) >= uint64_t(cap) * kBlockVals)
          record_error(st, step, kPhaseP2G, s0, 0, kErrInactive);
        else
          atomicAdd(pool + off + v * 64, sum);
      }
    }
  }
}

// Deterministic mode (cfg.deterministic; the reference switches to its serial
// scatter, simulation.hpp:326-327): every node of every active block is the
// sum of the covering blocks' P2G tiles in a fixed order -- key block
// offsets ascending in x, then y, then z -- instead of REDG arrival order.
// A node at local index l of its block on the -1 grid (tile 5^3 from 4b) is
// covered by the tiles of b = B (slot l) and, for l = 0, b = B - 1 (slot 4);
// on the +1 grid (tile 6^3 from 4b - 1) by b = B - 1 (l = 0, slot 5), b = B
// (slot l + 1) and b = B + 1 (l = 3, slot 0).  Bitwise run-to-run
// reproducible on the same GPU (not bitwise equal to the CPU engine).
template <typename T>
__global__ void det_gather_kernel(T* __restrict__ pool, const uint32_t* __restrict__ active,
                                  const int32_t* __restrict__ dir, const T* __restrict__ dtile, uint32_t dcap,
                                  const DevStatus* st, uint32_t cap, int D) {
  const uint32_t na = min(min(st->grid_hi, cap), dcap);
  const uint32_t n0 = st->grid_lo;
  const uint64_t total = na > n0 ? uint64_t(na - n0) * 128 : 0;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t slot = n0 + uint32_t(k >> 7);
    const int g = int(k >> 6) & 1, l = int(k & 63);
    const int li = (l >> 4) & 3, lj = (l >> 2) & 3, lk = l & 3;
    int Bx, By, Bz;
    decode_key(__ldg(active + slot), D, Bx, By, Bz);
    const int L[3] = {li, lj, lk};
    // covering key blocks per axis (ascending) and the node's slot in their tile
    int ob[3][3], os[3][3], no[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int m = 0;
      if (g == 0) {
        if (L[a] == 0) { ob[a][m] = -1; os[a][m] = 4; ++m; }
        ob[a][m] = 0; os[a][m] = L[a]; ++m;
      } else {
        if (L[a] == 0) { ob[a][m] = -1; os[a][m] = 5; ++m; }
        ob[a][m] = 0; os[a][m] = L[a] + 1; ++m;
        if (L[a] == 3) { ob[a][m] = 1; os[a][m] = 0; ++m; }
      }
      no[a] = m;
    }
    T sum[4] = {T(0), T(0), T(0), T(0)};
    for (int ix = 0; ix < no[0]; ++ix)
      for (int iy = 0; iy < no[1]; ++iy)
        for (int iz = 0; iz < no[2]; ++iz) {
          const int32_t nb = dir_lookup(dir, D, Bx + ob[0][ix], By + ob[1][iy], Bz + ob[2][iz]);
          if (nb < 0 || uint32_t(nb) >= dcap) continue;
          const T* t = dtile + uint64_t(nb) * kDetVals;
          int e;
          if (g == 0) e = (os[0][ix] * kPT + os[1][iy]) * kPT + os[2][iz];
          else e = 4 * kPTNodes + (os[0][ix] * kTileN + os[1][iy]) * kTileN + os[2][iz];
          const int vs = g == 0 ? kPTNodes : kTileNodes;
#pragma unroll
          for (int v = 0; v < 4; ++v) sum[v] += __ldg(t + e + v * vs);
        }
    T* base = pool + uint64_t(slot) * kBlockVals + g * 256 + l;
#pragma unroll
    for (int v = 0; v < 4; ++v) base[v * 64] = sum[v];
  }
}

// Deterministic mode: the rare out-of-tile contributions (multiply/divide
// rounding disagreement at a non-power-of-two dx), applied after the gather
// in sorted-particle order by one CTA (bitonic sort of the records, then a
// serial pass).
constexpr int kDetSpillMax = 4096;
template <typename T>
__global__ void __launch_bounds__(1024) det_spill_kernel(T* __restrict__ pool, const int32_t* __restrict__ dir,
                                                         const DetSpill<T>* __restrict__ spill, DevStatus* st,
                                                         uint32_t cap, int D, int slab) {
  __shared__ unsigned long long key[kDetSpillMax];
  const uint32_t n = min(st->spill_n, uint32_t(kDetSpillMax));
  if (n == 0) return;
  if (slab) {  // x-slab ranks exchange tiles only: no out-of-tile records
    if (threadIdx.x == 0) atomicOr(&st->overflow, 8u);
    return;
  }
  uint32_t m = 1;
  while (m < n) m <<= 1;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x)
    key[i] = i < n ? (static_cast<unsigned long long>(spill[i].idx) << 32) | (uint64_t(spill[i].g) << 31) | i
                   : ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= m; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint32_t p = i ^ j;
        if (p > i) {
          const bool up = (i & k) == 0;
          const unsigned long long a = key[i], b = key[p];
          if ((a > b) == up) {
            key[i] = b;
            key[p] = a;
          }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x != 0) return;
  for (uint32_t r = 0; r < n; ++r) {
    const DetSpill<T>& e = spill[key[r] & 0x7fffffffu];
    for (int nid = 0; nid < 8; ++nid) {
      const int gi = e.base[0] + (nid >> 2), gj = e.base[1] + ((nid >> 1) & 1), gk = e.base[2] + (nid & 1);
      const int32_t slot = dir_lookup(dir, D, gi >> 2, gj >> 2, gk >> 2);
      if (slot < 0 || uint32_t(slot) >= cap) {
        record_error(st, 0, kPhaseP2G, e.idx, 0, kErrInactive);
        continue;
      }
      T* nd = pool + node_off(slot, e.g, gi, gj, gk);
#pragma unroll
      for (int q = 0; q < 4; ++q) nd[q * 64] += e.v[nid][q];
    }
  }
}

// Grid update on both grids (grid_update_block, transfer.hpp:419-440;
// BoundaryCondition::contains/apply, grid.hpp:34-55).
template <typename T>
__global__ void grid_update_kernel(T* __restrict__ pool, const uint32_t* __restrict__ active,
                                   const DevStatus* st, uint32_t cap, StepConst<T> c,
                                   const BcParam<T>* __restrict__ bcs) {
  const uint32_t g0 = st->grid_lo;
  uint32_t g1 = st->grid_hi;
  if (g1 > cap) g1 = cap;
  // both grids (compact kernel) or slot 0 only (quadratic baseline)
  const int sh = c.quad ? 6 : 7;
  const uint64_t total = g1 > g0 ? uint64_t(g1 - g0) << sh : 0;
  const int D = c.D;
  const T dt = step_dt(c);
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t j = g0 + uint32_t(k >> sh);  // active-list position
    const uint32_t slot = c.dense ? __ldg(active + j) : j;
    const int g = int(k >> 6) & (c.quad ? 0 : 1);
    const int l = int(k & 63);
    T* base = pool + uint64_t(slot) * kBlockVals + g * 256 + l;
    const T mass = base[0];
    if (mass > c.mass_eps) {
      const T inv = T(1) / mass;
      T v[3] = {base[64] * inv + c.gravity[0] * dt, base[128] * inv + c.gravity[1] * dt,
                base[192] * inv + c.gravity[2] * dt};
      if (c.n_boundaries > 0) {
        int bx, by, bz;
        decode_key(__ldg(active + j), D, bx, by, bz);
        const T off = (c.quad ? T(0) : (g == 0 ? T(-0.25) : T(0.25))) * c.dx;  // grid.hpp:194-197, tag 0 / -1 / +1
        const T xp[3] = {T(bx * 4 + ((l >> 4) & 3)) * c.dx + off, T(by * 4 + ((l >> 2) & 3)) * c.dx + off,
                         T(bz * 4 + (l & 3)) * c.dx + off};
        for (int b = 0; b < c.n_boundaries; ++b) {
          const BcParam<T>& bc = bcs[b];
          if (!(xp[0] >= bc.lo[0] && xp[0] <= bc.hi[0] && xp[1] >= bc.lo[1] && xp[1] <= bc.hi[1] &&
                xp[2] >= bc.lo[2] && xp[2] <= bc.hi[2]))
            continue;
          if (bc.kind == 0) {  // sticky: v0 + omega x (x - c)
            const T r0 = xp[0] - bc.center[0], r1 = xp[1] - bc.center[1], r2 = xp[2] - bc.center[2];
            v[0] = bc.velocity[0] + (bc.omega[1] * r2 - bc.omega[2] * r1);
            v[1] = bc.velocity[1] + (bc.omega[2] * r0 - bc.omega[0] * r2);
            v[2] = bc.velocity[2] + (bc.omega[0] * r1 - bc.omega[1] * r0);
          } else {
            const T vn = v[0] * bc.normal[0] + v[1] * bc.normal[1] + v[2] * bc.normal[2];
            if (bc.kind == 1 || vn < T(0)) {
              v[0] -= bc.normal[0] * vn;
              v[1] -= bc.normal[1] * vn;
              v[2] -= bc.normal[2] * vn;
            }
          }
        }
      }
      base[64] = v[0];
      base[128] = v[1];
      base[192] = v[2];
    } else {
      base[0] = T(0);
      base[64] = T(0);
      base[128] = T(0);
      base[192] = T(0);
    }
  }
}

template <typename T>
__device__ __forceinline__ unsigned long long as_ordered_bits(T v) {
  return static_cast<unsigned long long>(__double_as_longlong(static_cast<double>(v)));
}

// One grid's contribution to gather_one (transfer.hpp:465-510), separable
// (sum-factorised over z, then y, then x).  V(s,t,u,c) yields the nodal
// velocity component c of stencil node (s,t,u).
template <typename T, typename VelFn>
__device__ __forceinline__ void gather_grid(const Axis<T>* ax, T dx, VelFn V, T (&v)[3], M3<T>& Bm, M3<T>& G) {
  const T wx0 = ax[0].w0, wx1 = ax[0].w1, wy0 = ax[1].w0, wy1 = ax[1].w1, wz0 = ax[2].w0, wz1 = ax[2].w1;
  const T gx0 = ax[0].g0, gy0 = ax[1].g0, gz0 = ax[2].g0;
  const T xx0 = ax[0].xi0, xx1 = ax[0].xi0 + dx, xy0 = ax[1].xi0, xy1 = ax[1].xi0 + dx;
  const T xz0 = ax[2].xi0, xz1 = ax[2].xi0 + dx;
#pragma unroll
  for (int cc = 0; cc < 3; ++cc) {
    T Y[2], Yg[2], Yz[2], Yx[2], Yzx[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      T Z[2], Zg[2], Zx[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const T a0 = V(s, t, 0, cc), a1 = V(s, t, 1, cc);
        Z[t] = wz0 * a0 + wz1 * a1;
        Zg[t] = gz0 * (a0 - a1);
        Zx[t] = wz0 * xz0 * a0 + wz1 * xz1 * a1;
      }
      Y[s] = wy0 * Z[0] + wy1 * Z[1];
      Yg[s] = gy0 * (Z[0] - Z[1]);
      Yz[s] = wy0 * Zg[0] + wy1 * Zg[1];
      Yx[s] = wy0 * xy0 * Z[0] + wy1 * xy1 * Z[1];
      Yzx[s] = wy0 * Zx[0] + wy1 * Zx[1];
    }
    v[cc] += T(0.5) * (wx0 * Y[0] + wx1 * Y[1]);
    G.a[cc][0] += T(0.5) * (gx0 * (Y[0] - Y[1]));
    G.a[cc][1] += T(0.5) * (wx0 * Yg[0] + wx1 * Yg[1]);
    G.a[cc][2] += T(0.5) * (wx0 * Yz[0] + wx1 * Yz[1]);
    Bm.a[cc][0] += T(0.5) * (wx0 * xx0 * Y[0] + wx1 * xx1 * Y[1]);
    Bm.a[cc][1] += T(0.5) * (wx0 * Yx[0] + wx1 * Yx[1]);
    Bm.a[cc][2] += T(0.5) * (wx0 * Yzx[0] + wx1 * Yzx[1]);
  }
}

// One velocity component cc of one grid's gather_one contribution
// (transfer.hpp:465-510), separable: o = {v, grad v row (3), B row (3)}, each
// already scaled by the dual-grid average's 1/2 (same operations and order as
// gather_grid).
template <typename T, typename VelFn>
__device__ __forceinline__ void gather_grid_cc(const Axis<T>* ax, T dx, VelFn V, int cc, T (&o)[7]) {
  const T wx0 = ax[0].w0, wx1 = ax[0].w1, wy0 = ax[1].w0, wy1 = ax[1].w1, wz0 = ax[2].w0, wz1 = ax[2].w1;
  const T gx0 = ax[0].g0, gy0 = ax[1].g0, gz0 = ax[2].g0;
  const T xx0 = ax[0].xi0, xx1 = ax[0].xi0 + dx, xy0 = ax[1].xi0, xy1 = ax[1].xi0 + dx;
  const T xz0 = ax[2].xi0, xz1 = ax[2].xi0 + dx;
  T Y[2], Yg[2], Yz[2], Yx[2], Yzx[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    T Z[2], Zg[2], Zx[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const T a0 = V(s, t, 0, cc), a1 = V(s, t, 1, cc);
      Z[t] = wz0 * a0 + wz1 * a1;
      Zg[t] = gz0 * (a0 - a1);
      Zx[t] = wz0 * xz0 * a0 + wz1 * xz1 * a1;
    }
    Y[s] = wy0 * Z[0] + wy1 * Z[1];
    Yg[s] = gy0 * (Z[0] - Z[1]);
    Yz[s] = wy0 * Zg[0] + wy1 * Zg[1];
    Yx[s] = wy0 * xy0 * Z[0] + wy1 * xy1 * Z[1];
    Yzx[s] = wy0 * Zx[0] + wy1 * Zx[1];
  }
  o[0] = T(0.5) * (wx0 * Y[0] + wx1 * Y[1]);
  o[1] = T(0.5) * (gx0 * (Y[0] - Y[1]));
  o[2] = T(0.5) * (wx0 * Yg[0] + wx1 * Yg[1]);
  o[3] = T(0.5) * (wx0 * Yz[0] + wx1 * Yz[1]);
  o[4] = T(0.5) * (wx0 * xx0 * Y[0] + wx1 * xx1 * Y[1]);
  o[5] = T(0.5) * (wx0 * Yx[0] + wx1 * Yx[1]);
  o[6] = T(0.5) * (wx0 * Yzx[0] + wx1 * Yzx[1]);
}

// gather_one over the 27-node quadratic stencil (transfer.hpp:512-543),
// sum-factorised; V(s,t,u,c) yields nodal velocity component c.
template <typename T, typename VelFn>
__device__ __forceinline__ void gather_quad(const QAxis<T> (&q)[3], T dx, VelFn V, T (&v)[3], M3<T>& Bm,
                                            M3<T>& G) {
#pragma unroll
  for (int cc = 0; cc < 3; ++cc) {
    T Y[3], Yg[3], Yz[3], Yx[3], Yzx[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      T Z[3], Zg[3], Zx[3];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const T a0 = V(s, t, 0, cc), a1 = V(s, t, 1, cc), a2 = V(s, t, 2, cc);
        Z[t] = q[2].w[0] * a0 + q[2].w[1] * a1 + q[2].w[2] * a2;
        Zg[t] = q[2].g[0] * a0 + q[2].g[1] * a1 + q[2].g[2] * a2;
        Zx[t] = q[2].w[0] * q[2].xi0 * a0 + q[2].w[1] * (q[2].xi0 + dx) * a1 +
                q[2].w[2] * (q[2].xi0 + T(2) * dx) * a2;
      }
      Y[s] = q[1].w[0] * Z[0] + q[1].w[1] * Z[1] + q[1].w[2] * Z[2];
      Yg[s] = q[1].g[0] * Z[0] + q[1].g[1] * Z[1] + q[1].g[2] * Z[2];
      Yz[s] = q[1].w[0] * Zg[0] + q[1].w[1] * Zg[1] + q[1].w[2] * Zg[2];
      Yx[s] = q[1].w[0] * q[1].xi0 * Z[0] + q[1].w[1] * (q[1].xi0 + dx) * Z[1] +
              q[1].w[2] * (q[1].xi0 + T(2) * dx) * Z[2];
      Yzx[s] = q[1].w[0] * Zx[0] + q[1].w[1] * Zx[1] + q[1].w[2] * Zx[2];
    }
    v[cc] = q[0].w[0] * Y[0] + q[0].w[1] * Y[1] + q[0].w[2] * Y[2];
    G.a[cc][0] = q[0].g[0] * Y[0] + q[0].g[1] * Y[1] + q[0].g[2] * Y[2];
    G.a[cc][1] = q[0].w[0] * Yg[0] + q[0].w[1] * Yg[1] + q[0].w[2] * Yg[2];
    G.a[cc][2] = q[0].w[0] * Yz[0] + q[0].w[1] * Yz[1] + q[0].w[2] * Yz[2];
    Bm.a[cc][0] = q[0].w[0] * q[0].xi0 * Y[0] + q[0].w[1] * (q[0].xi0 + dx) * Y[1] +
                  q[0].w[2] * (q[0].xi0 + T(2) * dx) * Y[2];
    Bm.a[cc][1] = q[0].w[0] * Yx[0] + q[0].w[1] * Yx[1] + q[0].w[2] * Yx[2];
    Bm.a[cc][2] = q[0].w[0] * Yzx[0] + q[0].w[1] * Yzx[1] + q[0].w[2] * Yzx[2];
  }
}

// KQ = 0: compact kernel on the dual grids; 1: quadratic B-spline baseline
// on grid slot 0 (the particle update below is shared).
// MM: the material models (and SV clamp) the kernel instance handles
// (kMFC | kMFluid | kMDP | kMClamp); the host picks the narrowest instance
// covering the scene, so an elastic-only scene carries no return-map or SVD
// code (and none of its register pressure).
constexpr int kMFC = 1, kMFluid = 2, kMDP = 4, kMClamp = 8, kMAll = 15;
template <typename T, int SCHEME, int KQ = 0, int MM = kMAll>
__global__ void __launch_bounds__(kG2PThreads, sizeof(T) == 4 ? CKG_G2P_MINB_F32 : CKG_G2P_MINB)
    g2p_tile_kernel(PState<T> cur, PState<T> nxt, const uint32_t* __restrict__ perm, StepConst<T> c,
                    const int32_t* __restrict__ dir, const uint32_t* __restrict__ rec,
                    const T* __restrict__ pool, uint32_t cap, DevStatus* st, int step) {
#if !CKG_G2P_PREFETCH
  __shared__ T vt[kVelVals];
#endif
  // per-thread gather results {v, grad v row, B row} x 3 components: the
  // -1 grid's partials, then (after the +1 grid) the final values, so no
  // accumulator is held in registers across the two grids' gathers
  __shared__ T gst[21][kG2PThreads];
  // per-thread prefetch (cp.async, issued before the gather) of the state the
  // particle update reads after it: F (9), J, mass, V0
  __shared__ T pst[12][kG2PThreads];
  // (dynamic) per-thread +1 grid sin/cos (unscaled) of the three axes, see
  // the gather (CKG_G2P_DUAL_SINCOS)
  extern __shared__ __align__(16) unsigned char g2p_dyn[];
#if CKG_G2P_PREFETCH
  // (dynamic, after the stash) two velocity tiles: the next item's is
  // fetched with cp.async while this item's particles are processed
  T* vtb = reinterpret_cast<T*>(g2p_dyn) + (CKG_G2P_DUAL_SINCOS ? 6 * kG2PThreads : 0);
  __shared__ uint32_t s_recb[2][kRecNbr + 27];
  __shared__ uint32_t s_itemb[2];
#else
  __shared__ uint32_t s_rec[kRecNbr + 27];
  __shared__ uint32_t s_item;
#endif
  __shared__ T wmax[kG2PWarps];
  // material table in shared memory: indexing the by-value kernel parameter
  // with the particle's material would copy the whole table to local memory
  __shared__ MatParam<T> s_mats[kMaxMaterials];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int m = 0; m < kMaxMaterials; ++m)
    if (tid == m) s_mats[m] = c.mats[m];
  const uint32_t na = min(st->item_hi, cap), item0 = st->item_lo;
  const int D = c.D;
  const T dx = c.dx, dt = step_dt(c);
  T vmax2 = T(0);
  // nodal velocity e of an item's tile (KQ = 0: both grids' 6^3; KQ = 1: the
  // quadratic baseline's 7^3 slot-0 nodes from 4b - 1): pool offset or -1
  auto tile_src = [&](const int32_t* nb, int bx, int by, int bz, int e) -> int64_t {
    if (KQ) {
      if (e >= 3 * kQGNodes) return -1;
      const int cc = e / kQGNodes, node = e % kQGNodes;
      const int gi = 4 * bx - 1 + node / (kQG * kQG), gj = 4 * by - 1 + (node / kQG) % kQG,
                gk = 4 * bz - 1 + node % kQG;
      const int64_t off = nbr_offset(nb, 0, gi, gj, gk, bx, by, bz);
      return (off >= 0 && uint64_t(off) < uint64_t(cap) * kBlockVals) ? off + (1 + cc) * 64 : -1;
    }
    if (e >= kVelVals) return -1;
    const int g = e / (3 * kTileNodes);
    const int cc = (e / kTileNodes) % 3;
    const int node = e % kTileNodes;
    const int gi = 4 * bx - g + node / (kTileN * kTileN);
    const int gj = 4 * by - g + (node / kTileN) % kTileN;
    const int gk = 4 * bz - g + node % kTileN;
    const int64_t off = nbr_offset(nb, g, gi, gj, gk, bx, by, bz);
    return (off >= 0 && uint64_t(off) < uint64_t(cap) * kBlockVals) ? off + (1 + cc) * 64 : -1;
  };
#if CKG_G2P_PREFETCH
  // claim an item (warp 0) and fetch its record into s_recb[b]
  auto claim = [&](int b) {
    if (warp == 0) {
      uint32_t it = 0;
      if (lane == 0) it = item0 + atomicAdd(&st->work[1], 1u);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (lane == 0) s_itemb[b] = it;
      if (it < na) {
        const uint32_t* r = rec + uint64_t(it) * kRecWords;
        if (lane < kRecNbr + 27) s_recb[b][lane] = __ldg(r + lane);
      }
    }
  };
  // all threads: cp.async of item s_itemb[b]'s velocity tile into buffer b
  auto stage_async = [&](int b) {
    const uint32_t it = s_itemb[b];
    if (it < na && s_recb[b][kRecS1] > s_recb[b][kRecS0]) {
      int bx, by, bz;
      decode_key(s_recb[b][kRecKey], D, bx, by, bz);
      const int32_t* nb = reinterpret_cast<const int32_t*>(s_recb[b] + kRecNbr);
      T* dst = vtb + b * kVelVals;
      for (int e = tid; e < kVelVals; e += kG2PThreads) {
        const int64_t off = tile_src(nb, bx, by, bz, e);
        cp_async_t(dst + e, pool + (off >= 0 ? off : 0), off >= 0);
      }
    }
    cp_async_commit();
  };
  claim(0);
  __syncthreads();
  stage_async(0);
  for (int k = 0;; ++k) {
    const int buf = k & 1;
    __syncthreads();  // everyone is done with buffer buf ^ 1 (item k - 1)
    claim(buf ^ 1);
    cp_async_wait_all();  // item k's tile (issued one item ago)
    __syncthreads();
    const uint32_t item = s_itemb[buf];
    if (item >= na) break;
    stage_async(buf ^ 1);  // item k + 1's tile, behind this item's work
    const uint32_t* s_rec = s_recb[buf];
    const int32_t* nbr = reinterpret_cast<const int32_t*>(s_rec + kRecNbr);
    const T* vt = vtb + buf * kVelVals;
    const uint32_t key = s_rec[kRecKey];
    const uint32_t s0 = s_rec[kRecS0], s1 = s_rec[kRecS1];
    if (s1 <= s0) continue;
    int bx, by, bz;
    decode_key(key, D, bx, by, bz);
#else
  const int32_t* nbr = reinterpret_cast<const int32_t*>(s_rec + kRecNbr);
  for (;;) {
    __syncthreads();
    if (warp == 0) {
      uint32_t it = 0;
      if (lane == 0) it = item0 + atomicAdd(&st->work[1], 1u);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (lane == 0) s_item = it;
      if (it < na) {
        const uint32_t* r = rec + uint64_t(it) * kRecWords;
        if (lane < kRecNbr + 27) s_rec[lane] = __ldg(r + lane);
      }
    }
    __syncthreads();
    const uint32_t item = s_item;
    if (item >= na) break;
    const uint32_t key = s_rec[kRecKey];
    const uint32_t s0 = s_rec[kRecS0], s1 = s_rec[kRecS1];
    if (s1 <= s0) continue;
    int bx, by, bz;
    decode_key(key, D, bx, by, bz);
    // stage nodal velocities of both grids' 6^3 tiles: all of a thread's
    // loads are issued before the first shared store
    {
      constexpr int kPer = (kVelVals + kG2PThreads - 1) / kG2PThreads;
      T val[kPer];
#pragma unroll
      for (int r = 0; r < kPer; ++r) {
        const int e = tid + r * kG2PThreads;
        const int64_t off = tile_src(nbr, bx, by, bz, e);
        val[r] = off >= 0 ? __ldg(pool + off) : T(0);
      }
#pragma unroll
      for (int r = 0; r < kPer; ++r) {
        const int e = tid + r * kG2PThreads;
        if (e < kVelVals) vt[e] = val[r];
      }
    }
    __syncthreads();
#endif
    // software pipeline over this thread's particles of the block: the next
    // particle's index is loaded when one starts, its position during the
    // gather (the perm -> position chain is off the critical path)
    uint32_t src_nx = s0 + tid < s1 ? __ldg(perm + s0 + tid) : 0u;
    T xn = T(0), yn = T(0), zn = T(0);
    bool have_x = false;
    for (uint32_t cb = s0; cb < s1; cb += kG2PThreads) {
      const uint32_t i = cb + tid;
      const bool live = i < s1;
      bool fluid = false;
      T Jout = T(1);
      uint32_t mi = 0;
      if (live) {
        const uint32_t src = src_nx;
        const bool has_next = i + kG2PThreads < s1;
        if (has_next) src_nx = __ldg(perm + i + kG2PThreads);
        const uint64_t n = cur.stride;  // field stride (buffer capacity)
        T* ps = &pst[0][tid];  // ps[k * kG2PThreads]
#pragma unroll
        for (int k = 0; k < 9; ++k) cp_async_t(ps + k * kG2PThreads, cur.f + (kF + k) * n + src, true);
        cp_async_t(ps + 9 * kG2PThreads, cur.f + kJ * n + src, true);
        cp_async_t(ps + 10 * kG2PThreads, cur.f + kMass * n + src, true);
        cp_async_t(ps + 11 * kG2PThreads, cur.f + kVol * n + src, true);
        cp_async_commit();
        T x, y, z;
        if (have_x) {
          x = xn;
          y = yn;
          z = zn;
        } else {
          x = __ldg(cur.f + kX * n + src);
          y = __ldg(cur.f + (kX + 1) * n + src);
          z = __ldg(cur.f + (kX + 2) * n + src);
        }
        mi = __ldg(cur.mat + src);
        T* gs = &gst[0][tid];  // gs[k * kG2PThreads]
#if CKG_G2P_DUAL_SINCOS
        T* sc6 = reinterpret_cast<T*>(g2p_dyn) + tid;  // sc6[k * kG2PThreads], k < 6
#endif
        if (KQ) {
          // quadratic baseline: 27 nodes of grid slot 0 (transfer.hpp:512-543)
          T v[3];
          M3<T> Bn, G;
          const QAxis<T> q[3] = {quad_axis(x, dx, c.inv_dx, c.pow2), quad_axis(y, dx, c.inv_dx, c.pow2),
                                 quad_axis(z, dx, c.inv_dx, c.pow2)};
          const int lx = q[0].base - (4 * bx - 1), ly = q[1].base - (4 * by - 1), lz = q[2].base - (4 * bz - 1);
          if (lx >= 0 && ly >= 0 && lz >= 0 && lx <= kQG - 3 && ly <= kQG - 3 && lz <= kQG - 3) {
            const T* vg = vt + (lx * kQG + ly) * kQG + lz;
            gather_quad<T>(
                q, dx, [&](int s, int t, int u, int cc) { return vg[cc * kQGNodes + (s * kQG + t) * kQG + u]; }, v,
                Bn, G);
          } else {
            gather_quad<T>(
                q, dx,
                [&](int s, int t, int u, int cc) {
                  const int gi = q[0].base + s, gj = q[1].base + t, gk = q[2].base + u;
                  const int32_t slot = pool_slot(dir, D, gi >> 2, gj >> 2, gk >> 2, c.dense);
                  if (slot < 0 || uint32_t(slot) >= cap) {
                    record_error(st, step, kPhaseG2P, i, 0, kErrInactive);
                    return T(0);
                  }
                  return __ldg(pool + node_off(slot, 0, gi, gj, gk) + (1 + cc) * 64);
                },
                v, Bn, G);
          }
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) {
            gs[(cc * 7) * kG2PThreads] = v[cc];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              gs[(cc * 7 + 1 + k) * kG2PThreads] = G.a[cc][k];
              gs[(cc * 7 + 4 + k) * kG2PThreads] = Bn.a[cc][k];
            }
          }
        }
#pragma unroll
        for (int g = 0; g < (KQ ? 0 : 2); ++g) {
          const T kq = g == 0 ? T(-0.25) : T(0.25);
#if CKG_G2P_DUAL_SINCOS
          // one sincos per axis for both grids: the -1 and +1 grid fractions
          // differ by exactly 1/2 (sin/cos flip sign; axis_pair_dual), the
          // +1 grid's values wait in the thread's shared-memory stash
          Axis<T> ax[3];
          {
            const T p3[3] = {x, y, z};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              if (g == 0) {
                T snp, csp;
                ax[a] = axis_pair_lo(p3[a], dx, c.inv_dx, c.pow2, &snp, &csp);
                sc6[(2 * a) * kG2PThreads] = snp;
                sc6[(2 * a + 1) * kG2PThreads] = csp;
              } else {
                ax[a] = axis_with(p3[a], dx, c.inv_dx, c.pow2, T(0.25), sc6[(2 * a) * kG2PThreads],
                                  sc6[(2 * a + 1) * kG2PThreads]);
              }
            }
          }
#else
          const Axis<T> ax[3] = {axis_pair(x, dx, c.inv_dx, c.pow2, kq), axis_pair(y, dx, c.inv_dx, c.pow2, kq),
                                 axis_pair(z, dx, c.inv_dx, c.pow2, kq)};
#endif
          const int lx = ax[0].base - (4 * bx - g), ly = ax[1].base - (4 * by - g), lz = ax[2].base - (4 * bz - g);
          const bool in_tile =
              lx >= 0 && ly >= 0 && lz >= 0 && lx <= kTileN - 2 && ly <= kTileN - 2 && lz <= kTileN - 2;
          // component by component: -1 grid to the stash, +1 grid added
          auto emit = [&](int cc, const T (&o)[7]) {
#pragma unroll
            for (int k = 0; k < 7; ++k) {
              T* p = gs + (cc * 7 + k) * kG2PThreads;
              *p = g == 0 ? o[k] : *p + o[k];
            }
          };
          if (in_tile) {
            const T* vg = vt + g * 3 * kTileNodes + (lx * kTileN + ly) * kTileN + lz;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
              T o[7];
              gather_grid_cc<T>(
                  ax, dx,
                  [&](int s, int t, int u, int c2) { return vg[c2 * kTileNodes + (s * kTileN + t) * kTileN + u]; },
                  cc, o);
              emit(cc, o);
            }
          } else {
            // rare: footprint outside the block tile -> stage the 8 nodes via
            // the directory into the same registers layout
            T V[2][2][2][3];
#pragma unroll 1
            for (int nid = 0; nid < 8; ++nid) {
              const int s = nid >> 2, t = (nid >> 1) & 1, u = nid & 1;
              const int gi = ax[0].base + s, gj = ax[1].base + t, gk = ax[2].base + u;
              const int32_t slot = pool_slot(dir, D, gi >> 2, gj >> 2, gk >> 2, c.dense);
              T a0 = T(0), a1 = T(0), a2 = T(0);
              if (slot < 0 || uint32_t(slot) >= cap) {
                record_error(st, step, kPhaseG2P, i, 0, kErrInactive);
              } else {
                const T* nd = pool + node_off(slot, g, gi, gj, gk);
                a0 = __ldg(nd + 64);
                a1 = __ldg(nd + 128);
                a2 = __ldg(nd + 192);
              }
#pragma unroll
              for (int ss = 0; ss < 2; ++ss)
#pragma unroll
                for (int tt = 0; tt < 2; ++tt)
#pragma unroll
                  for (int uu = 0; uu < 2; ++uu)
                    if (ss == s && tt == t && uu == u) {
                      V[ss][tt][uu][0] = a0;
                      V[ss][tt][uu][1] = a1;
                      V[ss][tt][uu][2] = a2;
                    }
            }
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
              T o[7];
              gather_grid_cc<T>(ax, dx, [&](int s, int t, int u, int c2) { return V[s][t][u][c2]; }, cc, o);
              emit(cc, o);
            }
          }
        }
        have_x = has_next;
        if (has_next) {
          xn = __ldg(cur.f + kX * n + src_nx);
          yn = __ldg(cur.f + (kX + 1) * n + src_nx);
          zn = __ldg(cur.f + (kX + 2) * n + src_nx);
        }
        cp_async_wait_all();
        const T mass = ps[10 * kG2PThreads], vol0 = ps[11 * kG2PThreads];
        T v[3];
        M3<T> Bn, G;
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          v[cc] = gs[(cc * 7) * kG2PThreads];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            G.a[cc][k] = gs[(cc * 7 + 1 + k) * kG2PThreads];
            Bn.a[cc][k] = gs[(cc * 7 + 4 + k) * kG2PThreads];
          }
        }
        // update_particle_state (transfer.hpp:594-627).  Outputs are stored
        // as soon as they are final so the stress evaluation at the end runs
        // with only F live (register pressure).
        const MatParam<T>& mp = s_mats[mi < kMaxMaterials ? mi : 0];
        M3<T> L = G;
        if (SCHEME == kSchemeMls) {
          const Dual<T> ds = dual_stencil(x, y, z, dx, c.inv_dx, c.pow2);
          M3<T> Di;
          if (!apic_d_inverse(apic_D(ds, dx), Di)) record_error(st, step, kPhaseG2P, i, 0, kErrNearSingularD);
          L = mul(Bn, Di);
        }
        {
          M3<T> Bout = SCHEME == kSchemePic ? load_m3(cur, kB, src) : Bn;
          if ((MM & kMFluid) && mp.model == kModelFluid && mp.viscosity > T(0) && SCHEME != kSchemePic) {
            const T f = dexp(-mp.viscosity * dt / (mp.density * dx * dx));
            const T tb = trace(Bout) / T(3);
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int b = 0; b < 3; ++b)
                Bout.a[a][b] = (a == b ? tb : T(0)) + (Bout.a[a][b] - (a == b ? tb : T(0))) * f;
          }
          store_m3(nxt, kB, i, Bout);
        }
        x += v[0] * dt;
        y += v[1] * dt;
        z += v[2] * dt;
        nxt.f[kX * n + i] = x;
        nxt.f[(kX + 1) * n + i] = y;
        nxt.f[(kX + 2) * n + i] = z;
        nxt.f[kV * n + i] = v[0];
        nxt.f[(kV + 1) * n + i] = v[1];
        nxt.f[(kV + 2) * n + i] = v[2];
        nxt.f[kMass * n + i] = mass;
        nxt.f[kVol * n + i] = vol0;
        nxt.mat[i] = mi;
        {
          const T s2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
          if (!dfinite(s2) || !dfinite(x * x + y * y + z * z)) atomicOr(&st->nonfinite, 1u);
          if (s2 > vmax2) vmax2 = s2;  // NaN never wins (std::max(vm, s2) semantics)
        }
        T J = ps[9 * kG2PThreads];
        M3<T> Fout;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c2 = 0; c2 < 3; ++c2) Fout.a[r][c2] = ps[(3 * r + c2) * kG2PThreads];
        T t6[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};  // V0 tau of the new state
        if ((MM & kMFluid) && mp.model == kModelFluid) {
          fluid = true;
          store_m3(nxt, kF, i, Fout);  // fluids carry F unchanged (transfer.hpp:609-617)
          J *= T(1) + dt * trace(L);
          if (!(J > T(0))) {
            record_error(st, step, kPhaseG2P, i, 0, kErrFluidJ);
          } else {
            stress_tau6(Fout, J, vol0, mp, t6);
          }
        } else {
          M3<T> Ld;
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) Ld.a[a][b] = (a == b ? T(1) : T(0)) + L.a[a][b] * dt;
          M3<T> Fn = mul(Ld, Fout);
          if ((MM & kMClamp) && c.clamp_singular) clamp_singular_values(Fn, c.clamp_floor);
          if ((MM & kMDP) && mp.model == kModelDP) {
            const int e = return_map_dp(Fn, mp.dp_alpha, mp.mu, mp.lambda, t6);
            if (e) record_error(st, step, kPhaseG2P, i, 0, e);
#pragma unroll
            for (int k = 0; k < 6; ++k) t6[k] *= vol0;
          } else if (!(det(Fn) > T(0))) {
            record_error(st, step, kPhaseG2P, i, 0, kErrFInverted);
          }
          store_m3(nxt, kF, i, Fn);
          if ((MM & kMFC) && mp.model == kModelFC && det(Fn) > T(0)) stress_tau6(Fn, J, vol0, mp, t6);
        }
        nxt.f[kJ * n + i] = J;
#pragma unroll
        for (int k = 0; k < 6; ++k) nxt.tau[uint64_t(k) * n + i] = t6[k];
        Jout = J;

      }
      // per-material min J over fluid particles (gather_all, simulation.hpp:371-372)
      uint32_t todo = __ballot_sync(0xffffffffu, live && fluid);
      while (todo) {
        const int leader = __ffs(todo) - 1;
        const uint32_t lead_mat = __shfl_sync(0xffffffffu, mi, leader);
        const bool mine = live && fluid && mi == lead_mat;
        T jv = mine ? Jout : T(INFINITY);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const T other = __shfl_xor_sync(0xffffffffu, jv, o);
          jv = (other < jv) ? other : jv;
        }
        if (lane == leader && lead_mat < kMaxMaterials && jv > T(0))
          atomicMin(&st->minj[lead_mat], as_ordered_bits(jv));
        todo &= ~__ballot_sync(0xffffffffu, mine);
      }
    }
  }
  // vmax^2: warp, CTA, then one atomic per CTA
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T other = __shfl_xor_sync(0xffffffffu, vmax2, o);
    vmax2 = (vmax2 < other) ? other : vmax2;
  }
  if (lane == 0) wmax[warp] = vmax2;
  __syncthreads();
  if (tid == 0) {
    T b = T(0);
    for (int w = 0; w < kG2PWarps; ++w) b = (b < wmax[w]) ? wmax[w] : b;
    if (b > T(0)) atomicMax(&st->vmax2, as_ordered_bits(b));
  }
}

// Initial stress cache for a freshly uploaded state (force_matrix of every
// particle, transfer.hpp:183-216), walked in the substep's sorted order
// (perm: sorted position -> stored index) so that a constitutive error is
// reported, like the P2G's own errors, at the first failing particle of the
// reference's scatter order (sorted index, atomicMin).
template <typename T>
__global__ void __launch_bounds__(256) stress_kernel(PState<T> cur, const uint32_t* __restrict__ perm, StepConst<T> c,
                                                     DevStatus* st, int step) {
  const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= cur.n) return;
  const uint32_t i = perm ? perm[j] : uint32_t(j);
  const uint32_t mi = cur.mat[i];
  T t6[6];
  const int e = stress_tau6(load_m3(cur, kF, i), cur.f[kJ * cur.stride + i], cur.f[kVol * cur.stride + i],
                            c.mats[mi < kMaxMaterials ? mi : 0], t6);
  if (e) record_error(st, step, kPhaseP2G, j, 0, e);
#pragma unroll
  for (int k = 0; k < 6; ++k) cur.tau[uint64_t(k) * cur.stride + i] = e ? T(0) : t6[k];
}

// K4: clear the active part of the pool (grid.hpp:148-151).
template <typename T>
__global__ void clear_kernel(T* __restrict__ pool, const DevStatus* st, uint32_t cap) {
  const uint32_t c0 = st->clear_lo;
  uint32_t c1 = st->clear_hi;
  if (c1 > cap) c1 = cap;
  const uint64_t total = c1 > c0 ? uint64_t(c1 - c0) * kBlockVals / 2 : 0;  // in 2-element words
  using W = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  W* p = reinterpret_cast<W*>(pool + uint64_t(c0) * kBlockVals);
  W zero;
  zero.x = T(0);
  zero.y = T(0);
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total; k += uint64_t(gridDim.x) * blockDim.x)
    p[k] = zero;
}

// Status reset before a substep.
__global__ void status_reset_kernel(DevStatus* st, int reset_err, int reset_perr = 0) {
  if (threadIdx.x == 0) {
    if (reset_err) st->err = ~0ull;
    if (reset_perr) st->perr = ~0ull;
    st->vmax2 = 0ull;
    st->nonfinite = 0u;
    st->spill_n = 0u;
    st->n_active_prev = st->n_active;
    st->n_active = 0u;
    st->overflow = 0u;
    st->inset_fail = 0u;
    st->nchanged = 0u;
  }
  if (threadIdx.x < 4) st->work[threadIdx.x] = 0u;
  if (threadIdx.x < kMaxMaterials) st->minj[threadIdx.x] = 0x7ff0000000000000ull;  // +inf
}

// AoS <-> SoA transposes for the C-ABI (Particle<T> layout, transfer.hpp:19-28).
// Particle<T> AoS <-> SoA, tiled through shared memory: 64 particles per
// tile, the AoS side read/written as one contiguous run, the SoA side as one
// 64-particle run per field (both coalesced; odd row pitch: no bank conflicts).
constexpr int kXpTile = 64;
constexpr int kXpPitch = kNumFields + 2;  // 27 fields + material word, +1 pad (odd)

template <typename T>
__device__ __forceinline__ T mat_word(uint32_t m) {
  T w = T(0);
  memcpy(&w, &m, sizeof(uint32_t));
  return w;
}
template <typename T>
__device__ __forceinline__ uint32_t word_mat(T w) {
  uint32_t m;
  memcpy(&m, &w, sizeof(uint32_t));
  return m;
}

template <typename T>
__global__ void __launch_bounds__(256) aos_to_soa_kernel(const T* __restrict__ aos, PState<T> p) {
  constexpr int W = kNumFields + 1;
  __shared__ T tile[kXpTile * kXpPitch];
  for (uint64_t b = uint64_t(blockIdx.x) * kXpTile; b < p.n; b += uint64_t(gridDim.x) * kXpTile) {
    const int cnt = int(min(uint64_t(kXpTile), p.n - b));
    for (int e = threadIdx.x; e < cnt * W; e += blockDim.x) tile[(e / W) * kXpPitch + e % W] = aos[b * W + e];
    __syncthreads();
    for (int e = threadIdx.x; e < W * kXpTile; e += blockDim.x) {
      const int f = e / kXpTile, j = e % kXpTile;
      if (j < cnt) {
        const T v = tile[j * kXpPitch + f];
        if (f < kNumFields)
          p.f[uint64_t(f) * p.stride + b + j] = v;
        else
          p.mat[b + j] = word_mat(v);
      }
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(256) soa_to_aos_kernel(PState<T> p, T* __restrict__ aos) {
  constexpr int W = kNumFields + 1;
  __shared__ T tile[kXpTile * kXpPitch];
  for (uint64_t b = uint64_t(blockIdx.x) * kXpTile; b < p.n; b += uint64_t(gridDim.x) * kXpTile) {
    const int cnt = int(min(uint64_t(kXpTile), p.n - b));
    for (int e = threadIdx.x; e < W * kXpTile; e += blockDim.x) {
      const int f = e / kXpTile, j = e % kXpTile;
      if (j < cnt)
        tile[j * kXpPitch + f] = f < kNumFields ? p.f[uint64_t(f) * p.stride + b + j] : mat_word<T>(p.mat[b + j]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * W; e += blockDim.x) aos[b * W + e] = tile[(e / W) * kXpPitch + e % W];
    __syncthreads();
  }
}

// Per-particle dual-stencil bases (binning parity hook).
template <typename T>
__global__ void bases_kernel(PState<T> p, T dx, T inv_dx, int pow2, int32_t* __restrict__ out) {
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const T kq = g == 0 ? T(-0.25) : T(0.25);
#pragma unroll
    for (int a = 0; a < 3; ++a)
      out[(i * 2 + g) * 3 + a] = axis_base(p.f[uint64_t(kX + a) * p.stride + i], dx, inv_dx, pow2, kq);
  }
}

// Grid pool -> reference Block::nodes order for the grid facade.
template <typename T>
__global__ void grid_export_kernel(const T* __restrict__ pool, const uint32_t* __restrict__ active,
                                   uint64_t nb, int D, int32_t* __restrict__ coords,
                                   double* __restrict__ nodes, int dense) {
  const uint64_t total = nb * 128;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = k >> 7;
    const int nn = int(k & 127);
    const int g = nn >> 6, l = nn & 63;
    const T* base = pool + (dense ? uint64_t(active[b]) : b) * kBlockVals + g * 256 + l;
    if (nodes) {
      double* o = nodes + k * 4;
      o[0] = double(base[0]);
      o[1] = double(base[64]);
      o[2] = double(base[128]);
      o[3] = double(base[192]);
    }
    if (coords && nn == 0) {
      int bx, by, bz;
      decode_key(active[b], D, bx, by, bz);
      coords[b * 3 + 0] = bx;
      coords[b * 3 + 1] = by;
      coords[b * 3 + 2] = bz;
    }
  }
}

// compute_diagnostics on the device (simulation.hpp:55-69).
template <typename T>
__global__ void diagnostics_kernel(PState<T> p, double* __restrict__ acc /* 10 sums */,
                                   unsigned long long* __restrict__ vmax_bits) {
  double s[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  double vm = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < p.n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double m = double(p.f[kMass * p.stride + i]);
    const double x[3] = {double(p.f[kX * p.stride + i]), double(p.f[(kX + 1) * p.stride + i]), double(p.f[(kX + 2) * p.stride + i])};
    const double v[3] = {double(p.f[kV * p.stride + i]), double(p.f[(kV + 1) * p.stride + i]), double(p.f[(kV + 2) * p.stride + i])};
    s[0] += v[0] * m;
    s[1] += v[1] * m;
    s[2] += v[2] * m;
    s[3] += (x[1] * v[2] - x[2] * v[1]) * m;
    s[4] += (x[2] * v[0] - x[0] * v[2]) * m;
    s[5] += (x[0] * v[1] - x[1] * v[0]) * m;
    s[6] += v[0];
    s[7] += v[1];
    s[8] += v[2];
    const double n2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    s[9] += 0.5 * m * n2;
    vm = vm < n2 ? n2 : vm;
  }
#pragma unroll
  for (int k = 0; k < 10; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s[k] += __shfl_xor_sync(0xffffffffu, s[k], o);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double other = __shfl_xor_sync(0xffffffffu, vm, o);
    vm = vm < other ? other : vm;
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 10; ++k) atomicAdd(acc + k, s[k]);
    atomicMax(vmax_bits, static_cast<unsigned long long>(__double_as_longlong(vm)));
  }
}

}  // namespace ckg
