// ckg_g2p2g.cuh — fused G2P2G for sm_100a (the paper's
// GPU design): one persistent kernel runs, per active
// block of substep n, the gather and particle update of substep n
// (gather_one + update_particle_state, transfer.hpp:465-627) AND the scatter
// of substep n+1 (scatter_one, transfer.hpp:235-283) of the particles it has
// just updated, so the scatter's particle state never leaves the SM:
//
//   phase A  one particle per thread, sorted order: stage-free gather from
//            the block's 2 x 6^3 velocity tile (grid n), F/x/v/B/J update,
//            Kirchhoff stress of the new F; the new state is written to the
//            next state buffer (coalesced, sorted order) and the scatter
//            inputs {x, m, v, V0 tau, B} to a per-thread shared-memory record;
//   phase B  the chunk's records re-ordered by sub-octant class of the new
//            position (deterministic ballot ranks); warp w scatters classes
//            2w and 2w+1 into its private FP64 tile of grid n+1 (same-cell
//            pairs of the two classes only meet on the +1 grid: two rank
//            layers), footprints outside the block's tile go straight to
//            global REDs;
//   flush    the four warp tiles are summed and reduced into grid n+1 once
//            per block with REDG.ADD.F64.
//
// Grid n+1's active set is not known while grid n is being read (the sort
// and activation of substep n+1 need the new positions), so both grids are
// DENSE block pools indexed by the block key (slot = (bx D + by) D + bz);
// the host clears grid n's blocks after the kernel (active set n) so each
// pool is zero outside the active set it next receives.
//
// dt of substep n+1 enters the scatter (the -dt A grad w force term): the
// host passes the substep's own dt as the speculation and re-runs the plain
// P2G (ckg_transfer.cuh) whenever the next ckg_step is called with another
// dt.
#pragma once

#include "ckg_transfer.cuh"

namespace ckg {

#ifndef CKG_FA_INL
#define CKG_FA_INL __device__ __forceinline__
#endif
#ifndef CKG_FB_INL
#define CKG_FB_INL __device__ __noinline__
#endif
constexpr int kFThreads = 128;
constexpr int kFWarps = kFThreads / 32;
#ifndef CKG_FUSED_MINB
#define CKG_FUSED_MINB 3
#endif
#ifndef CKG_FUSED_MINB_F32
#define CKG_FUSED_MINB_F32 4
#endif
// scatter record fields (per particle, in phase-B order of need)
constexpr int kRX = 0, kRM = 3, kRV = 4, kRT = 7, kRB = 13, kRecMax = 22;
template <int SCHEME>
__host__ __device__ constexpr int frec_fields() {
  return SCHEME == kSchemePic ? kRB : kRecMax;
}
// warp tile of grid n+1: -1 grid 5^3 nodes from (4b, 4b, 4b); +1 grid
// 6 x 5 x 5 from (4b - 1, 4b - cy, 4b - cz) for the warp's class pair (the
// y/z class bits cy = w & 1, cz = w >> 1 are fixed per warp, x is free).
// Both use row stride 5 and plane stride 25.
constexpr int kFT0 = 125, kFT1 = 150;
constexpr int kFWarpVals = 4 * kFT0 + 4 * kFT1;  // 1100
template <typename T, int SCHEME>
constexpr size_t g2p2g_smem_bytes() {
  return (size_t(kFWarps) * kFWarpVals + size_t(frec_fields<SCHEME>() < 21 ? 21 : frec_fields<SCHEME>()) *
                                             kFThreads) * sizeof(T);
}

// Stash / record column of thread t: t ^ ((t >> 3) & 7).  A warp's own
// columns (stash and record writes) stay conflict-free, and so do the phase-B
// reads, whose lanes take one class of a lattice chunk -- threads 8j + o,
// stride 8 (8-way conflicts unswizzled).
__device__ __forceinline__ int fcol(int t) { return t ^ ((t >> 3) & 7); }

// Node (gi, gj, gk) of grid g in a dense block pool; -1 outside the directory box.
__device__ __forceinline__ int64_t dense_node(int D, int g, int gi, int gj, int gk) {
  if (gi < 0 || gj < 0 || gk < 0) return -1;
  const int bi = gi >> 2, bj = gj >> 2, bk = gk >> 2;
  if (bi >= D || bj >= D || bk >= D) return -1;
  return int64_t((bi * D + bj) * D + bk) * kBlockVals + g * 256 + (((gi & 3) << 4) | ((gj & 3) << 2) | (gk & 3));
}

// Phase A of the fused kernel for one particle (sorted position i): gather
// from the block's velocity tile vt (grid n), update_particle_state
// (transfer.hpp:594-627), new state to nxt[i], scatter record to the
// thread's stash column gs[k * kFThreads].  Out of line (see
// fused_scatter_round).
template <typename T>
struct FusedA {
  uint32_t q, mi;
  T J, vmax2;
  bool fluid;
};
template <typename T, int SCHEME, int MM>
CKG_FA_INL FusedA<T> fused_gather_update(PState<T> cur, PState<T> nxt, const uint32_t* __restrict__ perm,
                                                      uint32_t i, T* gs, const T* vt, const MatParam<T>* s_mats,
                                                      T dx, T inv_dx, int pow2, int D, T dt, int clamp_singular,
                                                      T clamp_floor, int bx, int by, int bz, T vmax2,
                                                      const T* __restrict__ pool_in, DevStatus* st, int step) {
  FusedA<T> r;
  r.q = 8u;
  r.mi = 0;
  r.J = T(1);
  r.vmax2 = vmax2;
  r.fluid = false;

  const uint32_t src = __ldg(perm + i);
  const uint64_t n = cur.stride;
  T x = __ldg(cur.f + kX * n + src);
  T y = __ldg(cur.f + (kX + 1) * n + src);
  T z = __ldg(cur.f + (kX + 2) * n + src);
  const uint32_t mi = __ldg(cur.mat + src);
  r.mi = mi;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const T kq = g == 0 ? T(-0.25) : T(0.25);
    const Axis<T> ax[3] = {axis_pair(x, dx, inv_dx, pow2, kq), axis_pair(y, dx, inv_dx, pow2, kq),
                           axis_pair(z, dx, inv_dx, pow2, kq)};
    const int lx = ax[0].base - (4 * bx - g), ly = ax[1].base - (4 * by - g), lz = ax[2].base - (4 * bz - g);
    const bool in_tile =
        lx >= 0 && ly >= 0 && lz >= 0 && lx <= kTileN - 2 && ly <= kTileN - 2 && lz <= kTileN - 2;
    auto emit = [&](int cc, const T (&o)[7]) {
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        T* p = gs + (cc * 7 + k) * kFThreads;
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
      // rare: footprint outside the block tile -> the 8 nodes from the pool
      T V[2][2][2][3];
#pragma unroll 1
      for (int nid = 0; nid < 8; ++nid) {
        const int s = nid >> 2, t = (nid >> 1) & 1, u = nid & 1;
        const int64_t off = dense_node(D, g, ax[0].base + s, ax[1].base + t, ax[2].base + u);
        T a0 = T(0), a1 = T(0), a2 = T(0);
        if (off >= 0) {
          a0 = __ldg(pool_in + off + 64);
          a1 = __ldg(pool_in + off + 128);
          a2 = __ldg(pool_in + off + 192);
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
  const T mass = __ldg(cur.f + kMass * n + src), vol0 = __ldg(cur.f + kVol * n + src);
  T v[3];
  M3<T> Bn, G;
#pragma unroll
  for (int cc = 0; cc < 3; ++cc) {
    v[cc] = gs[(cc * 7) * kFThreads];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      G.a[cc][k] = gs[(cc * 7 + 1 + k) * kFThreads];
      Bn.a[cc][k] = gs[(cc * 7 + 4 + k) * kFThreads];
    }
  }
  // update_particle_state (transfer.hpp:594-627); the stash column is
  // now free and becomes this particle's scatter record
  const MatParam<T>& mp = s_mats[mi < kMaxMaterials ? mi : 0];
  const M3<T> L = G;
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
    if (SCHEME != kSchemePic) {
#pragma unroll
      for (int k = 0; k < 9; ++k) gs[(kRB + k) * kFThreads] = Bout.a[k / 3][k % 3];
    }
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
  gs[(kRX + 0) * kFThreads] = x;
  gs[(kRX + 1) * kFThreads] = y;
  gs[(kRX + 2) * kFThreads] = z;
  gs[kRM * kFThreads] = mass;
  gs[(kRV + 0) * kFThreads] = v[0];
  gs[(kRV + 1) * kFThreads] = v[1];
  gs[(kRV + 2) * kFThreads] = v[2];
  {
    const T s2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    if (!dfinite(s2) || !dfinite(x * x + y * y + z * z)) atomicOr(&st->nonfinite, 1u);
    if (s2 > r.vmax2) r.vmax2 = s2;
  }
  // class of the new position (frac(x/dx - 1/4) >= 1/2 per axis)
  {
    const T p3[3] = {x, y, z};
    uint32_t qq = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const T sa = sub_rn(over_dx(p3[a], dx, inv_dx, pow2), T(0.25));
      qq |= ((sa - dfloor(sa)) >= T(0.5) ? 1u : 0u) << a;
    }
    r.q = qq;
  }
  T J = __ldg(cur.f + kJ * n + src);
  const M3<T> Fin = load_m3(cur, kF, src);
  T t6[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
  if ((MM & kMFluid) && mp.model == kModelFluid) {
    r.fluid = true;
    store_m3(nxt, kF, i, Fin);  // fluids carry F unchanged (transfer.hpp:609-617)
    J *= T(1) + dt * trace(L);
    if (!(J > T(0))) {
      record_error(st, step, kPhaseG2P, i, 0, kErrFluidJ);
    } else {
      stress_tau6(Fin, J, vol0, mp, t6);
    }
  } else {
    M3<T> Ld;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) Ld.a[a][b] = (a == b ? T(1) : T(0)) + L.a[a][b] * dt;
    M3<T> Fn = mul(Ld, Fin);
    if ((MM & kMClamp) && clamp_singular) clamp_singular_values(Fn, clamp_floor);
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
  for (int k = 0; k < 6; ++k) gs[(kRT + k) * kFThreads] = t6[k];
  r.J = J;
  return r;
}

// One 32-lane round of the fused kernel's scatter (scatter_one,
// transfer.hpp:235-283) from the lane's shared-memory record r[k * kFThreads]
// into the warp's tile of grid n+1 (or, outside it, the pool).  Out of line:
// the gather/update phase and this one get separate register allocations
// (inlined into one loop body they spilled 700 B).
template <typename T, int SCHEME>
CKG_FB_INL void fused_scatter_round(const T* r, bool valid, uint32_t err_index, T dx, T inv_dx,
                                                 int pow2, int D, T dt_next, int bx, int by, int bz, int cy, int cz,
                                                 T* wt, T* __restrict__ pool_out, DevStatus* st) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
    T x = 0, y = 0, z = 0, m = 0;
    T mv[3] = {0, 0, 0};
    M3<T> Ap, Q;
    Dual<T> ds;
    if (valid) {
      x = r[(kRX + 0) * kFThreads];
      y = r[(kRX + 1) * kFThreads];
      z = r[(kRX + 2) * kFThreads];
      m = r[kRM * kFThreads];
      T t6[6];
#pragma unroll
      for (int k = 0; k < 3; ++k) mv[k] = m * r[(kRV + k) * kFThreads];
#pragma unroll
      for (int k = 0; k < 6; ++k) t6[k] = dt_next * r[(kRT + k) * kFThreads];
      Ap.a[0][0] = t6[0];
      Ap.a[0][1] = Ap.a[1][0] = t6[1];
      Ap.a[0][2] = Ap.a[2][0] = t6[2];
      Ap.a[1][1] = t6[3];
      Ap.a[1][2] = Ap.a[2][1] = t6[4];
      Ap.a[2][2] = t6[5];
      ds = dual_stencil(x, y, z, dx, inv_dx, pow2);
      if (SCHEME != kSchemePic) {
        M3<T> Bp, Di;
#pragma unroll
        for (int k = 0; k < 9; ++k) Bp.a[k / 3][k % 3] = r[(kRB + k) * kFThreads];
        if (!apic_d_inverse(apic_D(ds, dx), Di)) {
          // substep n+1's P2G error, latched for that substep (the
          // particle's sorted index of substep n)
          record_error_at(&st->perr, 0, kPhaseP2G, err_index, 0, kErrNearSingularD);
          valid = false;
        }
        Q = scale(m, mul(Bp, Di));  // m * B D^-1
      }
    }
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      Axis<T> ax[3];
      if (g == 0) {
        ax[0] = ds.ax[0][0];
        ax[1] = ds.ax[0][1];
        ax[2] = ds.ax[0][2];
      } else {
        ax[0] = axis_pair(x, dx, inv_dx, pow2, T(0.25));
        ax[1] = axis_pair(y, dx, inv_dx, pow2, T(0.25));
        ax[2] = axis_pair(z, dx, inv_dx, pow2, T(0.25));
      }
      // this warp's tile of grid g (origins: see kFT0 / kFT1)
      const int lx = ax[0].base - (4 * bx - g), ly = ax[1].base - (4 * by - (g ? cy : 0)),
                lz = ax[2].base - (4 * bz - (g ? cz : 0));
      const bool in_tile = valid && lx >= 0 && ly >= 0 && lz >= 0 && lx <= (g ? 4 : 3) && ly <= 3 && lz <= 3;
      const int VS = g ? kFT1 : kFT0;
      const uint32_t cell = in_tile ? uint32_t((lx * 5 + ly) * 5 + lz) : (1024u + lane);
      const uint32_t cpeers = __match_any_sync(0xffffffffu, cell);
      const uint32_t rank = __popc(cpeers & lt);
      const uint32_t maxrank = __reduce_max_sync(0xffffffffu, rank);
      const uint32_t tmask = __ballot_sync(0xffffffffu, in_tile);
      T u0[3] = {mv[0], mv[1], mv[2]};
      if (SCHEME != kSchemePic) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
          u0[a] += Q.a[a][0] * ax[0].xi0 + Q.a[a][1] * ax[1].xi0 + Q.a[a][2] * ax[2].xi0;
      }
      auto contrib = [&](int s, int t, int u, T (&o)[4]) {
        const T wxs = s ? ax[0].w1 : ax[0].w0, wyt = t ? ax[1].w1 : ax[1].w0, wzu = u ? ax[2].w1 : ax[2].w0;
        const T wyz = wyt * wzu;
        const T w = wxs * wyz;
        const T gxs = s ? -ax[0].g0 : ax[0].g0, gyt = t ? -ax[1].g0 : ax[1].g0, gzu = u ? -ax[2].g0 : ax[2].g0;
        const T gw0 = gxs * wyz, gw1 = wxs * (gyt * wzu), gw2 = wxs * (wyt * gzu);
        o[0] = w * m;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          T b = u0[a];
          if (SCHEME != kSchemePic) {
            if (s) b = fma(Q.a[a][0], dx, b);
            if (t) b = fma(Q.a[a][1], dx, b);
            if (u) b = fma(Q.a[a][2], dx, b);
          }
          o[1 + a] = w * b - (Ap.a[a][0] * gw0 + Ap.a[a][1] * gw1 + Ap.a[a][2] * gw2);
        }
      };
      T* p0 = wt + g * 4 * kFT0 + (lx * 5 + ly) * 5 + lz;
      if (maxrank == 0) {
        if (in_tile) {
#pragma unroll
          for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                T o[4];
                contrib(s, t, u, o);
                tile_add4(p0 + (s * 5 + t) * 5 + u, o, VS);
                __syncwarp(tmask);
              }
        }
      } else if (maxrank == 1) {
        // two rank layers (a lattice chunk's same-cell class pair on
        // the +1 grid), unrolled
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              T o[4];
              contrib(s, t, u, o);
              T* p = p0 + (s * 5 + t) * 5 + u;
              if (in_tile && rank == 0) tile_add4(p, o, VS);
              __syncwarp();
              if (in_tile && rank == 1) tile_add4(p, o, VS);
              __syncwarp();
            }
      } else {
#pragma unroll 1
        for (int nid = 0; nid < 8; ++nid) {
          const int s = nid >> 2, t = (nid >> 1) & 1, u = nid & 1;
          T o[4];
          contrib(s, t, u, o);
          T* p = p0 + (s * 5 + t) * 5 + u;
          for (uint32_t layer = 0; layer <= maxrank; ++layer) {
            if (in_tile && rank == layer) tile_add4(p, o, VS);
            __syncwarp();
          }
        }
      }
      if (valid && !in_tile) {
        // footprint outside this warp's tile: direct REDs into grid n+1
#pragma unroll 1
        for (int nid = 0; nid < 8; ++nid) {
          const int s = nid >> 2, t = (nid >> 1) & 1, u = nid & 1;
          T o[4];
          contrib(s, t, u, o);
          const int64_t off = dense_node(D, g, ax[0].base + s, ax[1].base + t, ax[2].base + u);
          if (off >= 0) {
            T* nd = pool_out + off;
            atomicAdd(nd, o[0]);
            atomicAdd(nd + 64, o[1]);
            atomicAdd(nd + 128, o[2]);
            atomicAdd(nd + 192, o[3]);
          }
        }
      }
    }
}

template <typename T, int SCHEME, int MM>
__global__ void __launch_bounds__(kFThreads, sizeof(T) == 4 ? CKG_FUSED_MINB_F32 : CKG_FUSED_MINB)
    g2p2g_kernel(PState<T> cur, PState<T> nxt, const uint32_t* __restrict__ perm, StepConst<T> c,
                 const uint32_t* __restrict__ rec, uint32_t cap, const T* __restrict__ pool_in,
                 T* __restrict__ pool_out, T dt_next, DevStatus* st, int step) {
  static_assert(SCHEME != kSchemeMls, "MLS runs the unfused transfers");
  extern __shared__ __align__(16) unsigned char fsm[];
  T* tiles = reinterpret_cast<T*>(fsm);
  T* gst = tiles + kFWarps * kFWarpVals;  // [RS][kFThreads]: gather stash, then the scatter record
  __shared__ T vt[kVelVals];
  __shared__ uint32_t s_item, s_key, s_s0, s_s1;
  __shared__ uint32_t s_wcnt[kFWarps][8];
  __shared__ uint32_t s_base[kFWarps][8];
  __shared__ uint32_t s_cstart[9];
  __shared__ uint8_t s_slot[kFThreads];
  __shared__ T wmax[kFWarps];
  __shared__ MatParam<T> s_mats[kMaxMaterials];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int m = 0; m < kMaxMaterials; ++m)
    if (tid == m) s_mats[m] = c.mats[m];
  for (int e = tid; e < kFWarps * kFWarpVals; e += kFThreads) tiles[e] = T(0);
  if (tid < 32) s_wcnt[tid >> 3][tid & 7] = 0u;
  const uint32_t na = min(st->item_hi, cap), item0 = st->item_lo;
  const int D = c.D;
  const T dx = c.dx, dt = step_dt(c);
  const int cy = warp & 1, cz = warp >> 1;  // this warp's fixed class bits (y, z)
  T* wt = tiles + warp * kFWarpVals;
  T vmax2 = T(0);
  for (;;) {
    __syncthreads();
    if (warp == 0) {
      uint32_t it = 0;
      if (lane == 0) it = item0 + atomicAdd(&st->work[1], 1u);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (lane == 0) {
        s_item = it;
        if (it < na) {
          const uint32_t* r = rec + uint64_t(it) * kRecWords;
          s_key = __ldg(r + kRecKey);
          s_s0 = __ldg(r + kRecS0);
          s_s1 = __ldg(r + kRecS1);
        }
      }
    }
    __syncthreads();
    if (s_item >= na) break;
    const uint32_t key = s_key, s0 = s_s0, s1 = s_s1;
    if (s1 <= s0) continue;
    int bx, by, bz;
    decode_key(key, D, bx, by, bz);
    // ---- grid n velocities of both grids' 6^3 tiles (dense pool)
    {
      constexpr int kPer = (kVelVals + kFThreads - 1) / kFThreads;
      T val[kPer];
#pragma unroll
      for (int r = 0; r < kPer; ++r) {
        const int e = tid + r * kFThreads;
        val[r] = T(0);
        if (e < kVelVals) {
          const int g = e / (3 * kTileNodes);
          const int cc = (e / kTileNodes) % 3;
          const int node = e % kTileNodes;
          const int64_t off = dense_node(D, g, 4 * bx - g + node / (kTileN * kTileN),
                                         4 * by - g + (node / kTileN) % kTileN, 4 * bz - g + node % kTileN);
          if (off >= 0) val[r] = __ldg(pool_in + off + (1 + cc) * 64);
        }
      }
#pragma unroll
      for (int r = 0; r < kPer; ++r) {
        const int e = tid + r * kFThreads;
        if (e < kVelVals) vt[e] = val[r];
      }
    }
    __syncthreads();
    for (uint32_t cb = s0; cb < s1; cb += kFThreads) {
      // =============================== phase A: gather + update (substep n)
      const uint32_t i = cb + tid;
      const bool live = i < s1;
      bool fluid = false;
      T Jout = T(1);
      uint32_t mi = 0;
      uint32_t q = 8u;  // sub-octant class of the new position (8: none)
      T* gs = gst + fcol(tid);  // gs[k * kFThreads]
      if (live) {
        const FusedA<T> fa = fused_gather_update<T, SCHEME, MM>(cur, nxt, perm, i, gs, vt, s_mats, dx, c.inv_dx, c.pow2,
                                                                D, dt, c.clamp_singular, c.clamp_floor, bx, by, bz,
                                                                vmax2, pool_in, st, step);
        q = fa.q;
        mi = fa.mi;
        Jout = fa.J;
        fluid = fa.fluid;
        vmax2 = fa.vmax2;
      }
      // per-material min J over fluid particles (gather_all, simulation.hpp:371-372)
      if (MM & kMFluid) {
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
      // =============================== class order of the chunk (stable, no atomics)
      const uint32_t peers = __match_any_sync(0xffffffffu, q);
      const uint32_t qrank = __popc(peers & lt);
      if (q < 8u && qrank == 0) s_wcnt[warp][q] = __popc(peers);
      __syncthreads();
      if (tid == 0) {
        uint32_t run = 0;
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
          s_cstart[qq] = run;
#pragma unroll
          for (int w = 0; w < kFWarps; ++w) {
            s_base[w][qq] = run;
            run += s_wcnt[w][qq];
          }
        }
        s_cstart[8] = run;
      }
      __syncthreads();
      if (q < 8u) s_slot[s_base[warp][q] + qrank] = uint8_t(tid);
      if (tid < 32) s_wcnt[tid >> 3][tid & 7] = 0u;
      __syncthreads();
      // =============================== phase B: scatter (substep n+1)
#ifndef CKG_FUSED_NO_SCATTER  // (defined: phase A alone, a timing experiment)
      {
        const uint32_t lo = s_cstart[2 * warp], hi = s_cstart[2 * warp + 2];
        for (uint32_t rb = lo; rb < hi; rb += 32) {
          const bool in_round = rb + lane < hi;
          const int sl = in_round ? int(s_slot[rb + lane]) : 0;
          fused_scatter_round<T, SCHEME>(gst + fcol(sl), in_round, cb + sl, dx, c.inv_dx, c.pow2, D, dt_next, bx, by, bz,
                                         cy, cz, wt, pool_out, st);
        }
      }
#endif
      __syncthreads();  // records and the slot table are reused by the next chunk
    }
    // =============================== flush the warp tiles into grid n+1
    for (int e = tid; e < 4 * kFT0 + 4 * kTileNodes; e += kFThreads) {
      T sum = T(0);
      int g, v, ii, jj, kk;
      if (e < 4 * kFT0) {
        g = 0;
        v = e / kFT0;
        const int sl = e % kFT0;
        ii = sl / 25;
        jj = (sl / 5) % 5;
        kk = sl % 5;
#pragma unroll
        for (int w = 0; w < kFWarps; ++w) {
          T* p = tiles + w * kFWarpVals + e;
          sum += *p;
          *p = T(0);
        }
      } else {
        g = 1;
        const int e1 = e - 4 * kFT0;
        v = e1 / kTileNodes;
        const int sl = e1 % kTileNodes;
        ii = sl / (kTileN * kTileN);
        jj = (sl / kTileN) % kTileN;
        kk = sl % kTileN;
        // node (ii, jj, kk) of the 6^3 halo from 4b - 1; warp w's window
        // holds it at (ii, jj - 1 + cy_w, kk - 1 + cz_w)
#pragma unroll
        for (int w = 0; w < kFWarps; ++w) {
          const int lj = jj - 1 + (w & 1), lk = kk - 1 + (w >> 1);
          if (lj >= 0 && lj < 5 && lk >= 0 && lk < 5) {
            T* p = tiles + w * kFWarpVals + 4 * kFT0 + v * kFT1 + (ii * 5 + lj) * 5 + lk;
            sum += *p;
            *p = T(0);
          }
        }
      }
      if (sum != T(0)) {
        const int64_t off = dense_node(D, g, 4 * bx - g + ii, 4 * by - g + jj, 4 * bz - g + kk);
        if (off >= 0) atomicAdd(pool_out + off + v * 64, sum);
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
    for (int w = 0; w < kFWarps; ++w) b = (b < wmax[w]) ? wmax[w] : b;
    if (b > T(0)) atomicMax(&st->vmax2, as_ordered_bits(b));
  }
}

// Clear the blocks of an active list in a dense pool (grid.hpp:148-151 for
// the blocks a substep used; every write of that substep stayed inside them).
template <typename T>
__global__ void clear_list_kernel(T* __restrict__ pool, const uint32_t* __restrict__ list,
                                  const unsigned int* count, uint32_t cap) {
  const uint32_t nb = min(*count, cap);
  using W = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  W zero;
  zero.x = T(0);
  zero.y = T(0);
  constexpr int kW = kBlockVals / 2;  // 2-element words per block
  const uint64_t total = uint64_t(nb) * kW;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t slot = __ldg(list + (k / kW));
    reinterpret_cast<W*>(pool + uint64_t(slot) * kBlockVals)[k % kW] = zero;
  }
}

// A scatter error the fused kernel found for the next substep becomes that
// substep's error once its activation ran (an OutOfDomainError of the
// activation, phase 2, wins over the P2G's, phase 4, as in the reference's
// phase order).
__global__ void promote_pending_error_kernel(DevStatus* st) {
  if (threadIdx.x == 0 && st->perr != ~0ull) {
    atomicMin(&st->err, st->perr);
    st->perr = ~0ull;
  }
}

}  // namespace ckg
