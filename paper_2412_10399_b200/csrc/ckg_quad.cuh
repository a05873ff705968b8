// ckg_quad.cuh — quadratic B-spline baseline P2G on the unstaggered grid
// (kernel.hpp:208-241, transfer.hpp:285-320 scatter_one,
// simulation.hpp:311-321).  Same persistent block-tile design as the compact
// kernel's p2g_tile_kernel: a block's particle segment is binned by sub-cell
// class (frac(x/dx - 1/2) >= 1/2 per axis), warp w scatters class w into a
// private FP64 tile of the 7^3 nodes a block's quadratic stencils can reach
// (origin 4b - 1), node offsets ordered by __syncwarp, and the CTA flushes the
// summed tiles with one REDG per non-zero node value into grid slot 0.
#pragma once

#include "ckg_transfer.cuh"

namespace ckg {

constexpr int kQT = 7;                      // tile nodes per axis
constexpr int kQTNodes = kQT * kQT * kQT;   // 343
constexpr int kQTVals = 4 * kQTNodes;       // m, px, py, pz
// CTA shape: kQWarps warps, each scattering CKG_QUAD_CPW of the 8 classes in
// turn into its own full 7^3 tile; CKG_QUAD_MINCTAS CTAs per SM.  10M bench
// (FP64): 8 warps x 2 CTAs (128 registers, 274 B of spills) 2.60 ms; 8 x 1
// 3.19 ms; 4 warps x 3 CTAs (168 registers) -- see DESIGN §4c.
#ifndef CKG_QUAD_CPW
#define CKG_QUAD_CPW 2
#endif
#ifndef CKG_QUAD_MINCTAS
#define CKG_QUAD_MINCTAS 3
#endif
#ifndef CKG_QUAD_MINCTAS_F32
#define CKG_QUAD_MINCTAS_F32 5
#endif
template <typename T>
constexpr int quad_min_ctas() {
  return sizeof(T) == 4 ? CKG_QUAD_MINCTAS_F32 : CKG_QUAD_MINCTAS;
}
constexpr int kQWarps = 8 / CKG_QUAD_CPW;
constexpr int kQThreads = 32 * kQWarps;
template <typename T>
constexpr size_t p2g_quad_smem_bytes() {
  return size_t(kQWarps) * kQTVals * sizeof(T);
}

template <typename T, int SCHEME>
__global__ void __launch_bounds__(kQThreads, quad_min_ctas<T>())
    p2g_quad_kernel(PState<T> cur, const uint32_t* __restrict__ perm, StepConst<T> c,
                    const int32_t* __restrict__ dir, const uint32_t* __restrict__ active,
                    const uint32_t* __restrict__ seg_begin, const uint32_t* __restrict__ seg_end,
                    T* __restrict__ pool, uint32_t cap, DevStatus* st, int step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tiles = reinterpret_cast<T*>(smem_raw);
  __shared__ int32_t nbr[27];
  __shared__ uint32_t s_item;
  __shared__ uint32_t cls_cnt[8], cls_off[8];
  __shared__ uint32_t cls_list[kP2GChunk];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* wt = tiles + warp * kQTVals;
  for (int e = tid; e < kQWarps * kQTVals; e += kQThreads) tiles[e] = T(0);
  const uint32_t na = min(st->item_hi, cap), item0 = st->item_lo;
  const uint32_t lt = lanemask_lt();
  const int D = c.D;
  const T dx = c.dx, dt = step_dt(c);
  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = item0 + atomicAdd(&st->work[0], 1u);
    __syncthreads();
    const uint32_t item = s_item;
    if (item >= na) break;
    const uint32_t key = active[item];
    const uint32_t s0 = seg_begin[key], s1 = seg_end[key];
    if (s1 <= s0) continue;
    int bx, by, bz;
    decode_key(key, D, bx, by, bz);
    if (tid < 27) nbr[tid] = dir_lookup(dir, D, bx - 1 + tid / 9, by - 1 + (tid / 3) % 3, bz - 1 + tid % 3);
    __syncthreads();
    for (uint32_t cb = s0; cb < s1; cb += kP2GChunk) {
      // ---- bin by class: particles of one class and different cells have
      // different bases (lattice layouts: one rank layer)
      const uint32_t len = min(uint32_t(kP2GChunk), s1 - cb);
      if (tid < 8) cls_cnt[tid] = 0;
      __syncthreads();
      uint32_t myq[kP2GChunk / kQThreads], myslot[kP2GChunk / kQThreads], mysrc[kP2GChunk / kQThreads];
#pragma unroll
      for (int r = 0; r < kP2GChunk / kQThreads; ++r) {
        const uint32_t j = tid + r * kQThreads;
        if (j < len) {
          const uint32_t src = __ldg(perm + cb + j);
          mysrc[r] = src;
          uint32_t q = 0;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const T sa =
                sub_rn(over_dx(__ldg(cur.f + uint64_t(kX + a) * cur.stride + src), dx, c.inv_dx, c.pow2), T(0.5));
            q |= ((sa - dfloor(sa)) >= T(0.5) ? 1u : 0u) << a;
          }
          myq[r] = q;
          myslot[r] = atomicAdd(&cls_cnt[q], 1u);
        }
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t run = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          cls_off[q] = run;
          run += cls_cnt[q];
        }
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kP2GChunk / kQThreads; ++r) {
        const uint32_t j = tid + r * kQThreads;
        if (j < len) cls_list[cls_off[myq[r]] + myslot[r]] = mysrc[r];
      }
      __syncthreads();
#pragma unroll 1
      for (int ci = 0; ci < CKG_QUAD_CPW; ++ci) {
      const int cl = warp + ci * kQWarps;  // this pass's class
      const uint32_t my_cnt = cls_cnt[cl], my_off = cls_off[cl];
      for (uint32_t rb = 0; rb < my_cnt; rb += 32) {
        const bool in_round = rb + lane < my_cnt;
        const uint32_t src = in_round ? cls_list[my_off + rb + lane] : 0u;
        auto sorted_index = [&]() -> uint32_t {
          for (uint32_t k = cb; k < min(cb + uint32_t(kP2GChunk), s1); ++k)
            if (__ldg(perm + k) == src) return k;
          return cb;
        };
        bool valid = in_round;
        T m = 0;
        T u0[3] = {0, 0, 0};
        M3<T> Ap, Q;
        QAxis<T> q[3];
        if (valid) {
          const uint64_t n = cur.stride;
          const T x = __ldg(cur.f + kX * n + src), y = __ldg(cur.f + (kX + 1) * n + src),
                  z = __ldg(cur.f + (kX + 2) * n + src);
          m = __ldg(cur.f + kMass * n + src);
          T v3[3], t6[6];
#pragma unroll
          for (int k = 0; k < 3; ++k) v3[k] = __ldg(cur.f + (kV + k) * n + src);
#pragma unroll
          for (int k = 0; k < 6; ++k) t6[k] = dt * __ldg(cur.tau + uint64_t(k) * n + src);
          Ap.a[0][0] = t6[0];
          Ap.a[0][1] = Ap.a[1][0] = t6[1];
          Ap.a[0][2] = Ap.a[2][0] = t6[2];
          Ap.a[1][1] = t6[3];
          Ap.a[1][2] = Ap.a[2][1] = t6[4];
          Ap.a[2][2] = t6[5];
          q[0] = quad_axis(x, dx, c.inv_dx, c.pow2);
          q[1] = quad_axis(y, dx, c.inv_dx, c.pow2);
          q[2] = quad_axis(z, dx, c.inv_dx, c.pow2);
#pragma unroll
          for (int a = 0; a < 3; ++a) u0[a] = m * v3[a];
          if (SCHEME != kSchemePic) {
            M3<T> Di;
            if (!apic_d_inverse(apic_D_quad(q, dx), Di)) {
              record_error(st, step, kPhaseP2G, sorted_index(), 0, kErrNearSingularD);
              valid = false;
            }
            Q = scale(m, mul(load_m3(cur, kB, src), Di));  // m * B D^-1
#pragma unroll
            for (int a = 0; a < 3; ++a)
              u0[a] += Q.a[a][0] * q[0].xi0 + Q.a[a][1] * q[1].xi0 + Q.a[a][2] * q[2].xi0;
          }
        } else {
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            q[a].base = 0;
            q[a].xi0 = T(0);
#pragma unroll
            for (int k = 0; k < 3; ++k) q[a].w[k] = q[a].g[k] = T(0);
          }
        }
        const int lx = q[0].base - (4 * bx - 1), ly = q[1].base - (4 * by - 1), lz = q[2].base - (4 * bz - 1);
        const bool in_tile =
            valid && lx >= 0 && ly >= 0 && lz >= 0 && lx <= kQT - 3 && ly <= kQT - 3 && lz <= kQT - 3;
        const uint32_t cell = in_tile ? uint32_t((lx * kQT + ly) * kQT + lz) : (1024u + lane);
        const uint32_t peers = __match_any_sync(0xffffffffu, cell);
        const uint32_t rank = __popc(peers & lt);
        const uint32_t maxrank = __reduce_max_sync(0xffffffffu, rank);
        // node (s,t,u): (m w, w (m v + Q xi) - A' grad w) (transfer.hpp:292-316)
        // (selects, not indexing: the rolled paths must not put q in local memory)
        auto pick = [](const T (&a)[3], int i) { return i == 0 ? a[0] : (i == 1 ? a[1] : a[2]); };
        auto contrib = [&](int s, int t, int u, T (&o)[4]) {
          const T wy = pick(q[1].w, t), wz = pick(q[2].w, u), wx = pick(q[0].w, s);
          const T wyz = wy * wz;
          const T w = wx * wyz;
          const T gw0 = pick(q[0].g, s) * wyz, gw1 = wx * (pick(q[1].g, t) * wz), gw2 = wx * (wy * pick(q[2].g, u));
          o[0] = w * m;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            T b = u0[a];
            if (SCHEME != kSchemePic) {
              if (s) b = fma(Q.a[a][0], T(s) * dx, b);
              if (t) b = fma(Q.a[a][1], T(t) * dx, b);
              if (u) b = fma(Q.a[a][2], T(u) * dx, b);
            }
            o[1 + a] = w * b - (Ap.a[a][0] * gw0 + Ap.a[a][1] * gw1 + Ap.a[a][2] * gw2);
          }
        };
        T* p0 = wt + (lx * kQT + ly) * kQT + lz;
        if (maxrank == 0) {
#pragma unroll
          for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
              for (int u = 0; u < 3; ++u) {
                T o[4];
                contrib(s, t, u, o);
                T* p = p0 + (s * kQT + t) * kQT + u;
                if (in_tile) {
                  p[0] += o[0];
                  p[kQTNodes] += o[1];
                  p[2 * kQTNodes] += o[2];
                  p[3 * kQTNodes] += o[3];
                }
                __syncwarp();  // a lane's node can be a neighbour's node at another offset
              }
        } else {
#pragma unroll 1
          for (int nid = 0; nid < 27; ++nid) {
            const int s = nid / 9, t = (nid / 3) % 3, u = nid % 3;
            T o[4];
            contrib(s, t, u, o);
            T* p = p0 + (s * kQT + t) * kQT + u;
            for (uint32_t layer = 0; layer <= maxrank; ++layer) {
              if (in_tile && rank == layer) {
                p[0] += o[0];
                p[kQTNodes] += o[1];
                p[2 * kQTNodes] += o[2];
                p[3 * kQTNodes] += o[3];
              }
              __syncwarp();
            }
          }
        }
        if (valid && !in_tile) {
#pragma unroll 1
          for (int nid = 0; nid < 27; ++nid) {
            const int s = nid / 9, t = (nid / 3) % 3, u = nid % 3;
            T o[4];
            contrib(s, t, u, o);
            const int gi = q[0].base + s, gj = q[1].base + t, gk = q[2].base + u;
            const int32_t slot = dir_lookup(dir, D, gi >> 2, gj >> 2, gk >> 2);
            if (slot < 0 || uint32_t(slot) >= cap) {
              record_error(st, step, kPhaseP2G, sorted_index(), 0, kErrInactive);
            } else {
              T* nd = pool + node_off(slot, 0, gi, gj, gk);
              atomicAdd(nd, o[0]);
              atomicAdd(nd + 64, o[1]);
              atomicAdd(nd + 128, o[2]);
              atomicAdd(nd + 192, o[3]);
            }
          }
        }
      }
      }  // classes of this warp
      __syncthreads();
    }
    __syncthreads();
    // ---- flush: sum the warp tiles (common origin 4b - 1), one REDG per value
    for (int e = tid; e < kQTVals; e += kQThreads) {
      T sum = T(0);
#pragma unroll
      for (int w = 0; w < kQWarps; ++w) {
        T* qv = tiles + w * kQTVals + e;
        sum += *qv;
        *qv = T(0);
      }
      if (sum != T(0)) {
        const int v = e / kQTNodes, node = e % kQTNodes;
        const int gi = 4 * bx - 1 + node / (kQT * kQT), gj = 4 * by - 1 + (node / kQT) % kQT,
                  gk = 4 * bz - 1 + node % kQT;
        const int64_t off = nbr_offset(nbr, 0, gi, gj, gk, bx, by, bz);
        if (off < 0 || uint64_t(off) >= uint64_t(cap) * kBlockVals)
          record_error(st, step, kPhaseP2G, s0, 0, kErrInactive);
        else
          atomicAdd(pool + off + v * 64, sum);
      }
    }
  }
}

}  // namespace ckg
