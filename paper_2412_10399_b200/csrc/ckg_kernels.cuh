// ckg_kernels.cuh — the per-substep CK-MPM transfer kernels for sm_100a.
//
// Pipeline (reference order, proj/include/ckmpm/simulation.hpp:147-188 and
// SPEC.md:407): key -> stable radix sort -> activate -> compact -> clear ->
// P2G -> grid update -> G2P (+ state update, advection, reductions).
//
// Device layout:
//  * particles: SoA, 27 scalar fields of T (x3 v3 F9 B9 J mass volume0),
//    field k of particle i at f[k*n + i], plus a u32 material array.  Two
//    copies (cur/next): G2P reads cur through the sort permutation and writes
//    next in sorted order, so the reference's full-AoS permute
//    (simulation.hpp:268-273) costs no extra pass.
//  * grid: dense int32 block directory over (res/4+2)^3 (grid.hpp:91-94) and a
//    pool of active blocks, each 2 grids x 4 values x 64 nodes of T
//    (block-local SoA: [g][m,px,py,pz][(i&3)<<4|(j&3)<<2|(k&3)]).
#pragma once

#include <cstdint>

#include "ckg_math.cuh"

namespace ckg {

// ------------------------------------------------------------ parameters

enum Field : int { kX = 0, kV = 3, kF = 6, kB = 15, kJ = 24, kMass = 25, kVol = 26, kNumFields = 27 };

template <typename T>
struct PState {
  T* f;           // kNumFields * n
  uint32_t* mat;  // n
  uint64_t n;
  __device__ __forceinline__ T& at(int k, uint64_t i) const { return f[uint64_t(k) * n + i]; }
};

template <typename T>
struct MatParam {
  int model;
  T mu, lambda, dp_alpha, bulk, gamma, viscosity, density;
};

constexpr int kMaxMaterials = 16;
constexpr int kMaxBoundaries = 32;

template <typename T>
struct StepConst {
  T dx, inv_dx, dt, mass_eps, clamp_floor;
  T gravity[3];
  int res, D, scheme, n_materials, clamp_singular, n_boundaries;
  MatParam<T> mats[kMaxMaterials];
};

template <typename T>
struct BcParam {
  int kind;
  T lo[3], hi[3], normal[3], velocity[3], omega[3], center[3];
};

constexpr int kSchemePic = 0, kSchemeApic = 1, kSchemeMls = 2;
constexpr int kModelFC = 0, kModelFluid = 1, kModelDP = 2;

// Device status record, one per context, reset before every substep.
struct DevStatus {
  unsigned long long err;       // packed, min wins; ~0 = none
  unsigned long long vmax2;     // bits of max |v|^2 as double (non-negative => integer order)
  unsigned long long minj[kMaxMaterials];  // bits of min J as double (J > 0)
  unsigned int nonfinite;
  unsigned int n_active;
  unsigned int overflow;
  unsigned int pad;
};

// err = step<<56 | phase<<52 | particle<<12 | axis<<8 | code
__device__ __forceinline__ void record_error(DevStatus* st, int step, int phase, uint64_t particle,
                                             int axis, int code) {
  unsigned long long p = (static_cast<unsigned long long>(step & 0xff) << 56) |
                         (static_cast<unsigned long long>(phase & 0xf) << 52) |
                         ((particle & 0xffffffffffull) << 12) |
                         (static_cast<unsigned long long>(axis & 0xf) << 8) |
                         static_cast<unsigned long long>(code & 0xff);
  atomicMin(&st->err, p);
}

// Error codes (mirror include/ckmpm_b200.h CKG_NUM_*).
constexpr int kErrOutOfDomain = 1, kErrFcStress = 2, kErrDpStress = 3, kErrFluidState = 4,
              kErrNearSingularD = 5, kErrSingularMls = 6, kErrReturnMap = 7, kErrFInverted = 8,
              kErrFluidJ = 9, kErrInactive = 11;
constexpr int kPhaseActivate = 2, kPhaseP2G = 4, kPhaseG2P = 6;

// ------------------------------------------------- bit-exact binning math

// nvcc contracts a*b+c into DFMA by default; the reference build (x86-64
// baseline) never does.  Binning must be bit-exact, so these expressions use
// round-to-nearest intrinsics that are never fused.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }

// Sort key axis term: clamp(int(floor(c*inv_dx + 0.25)) >> 2, 0, D-1)
// (simulation.hpp:256-261).
template <typename T>
__device__ __forceinline__ int key_axis(T c, T inv_dx, int D) {
  int b = static_cast<int>(dfloor(add_rn(mul_rn(c, inv_dx), T(0.25)))) >> 2;
  return b < 0 ? 0 : (b > D - 1 ? D - 1 : b);
}

template <typename T>
__device__ __forceinline__ uint32_t block_key(T x, T y, T z, T inv_dx, int D) {
  return (uint32_t(key_axis(x, inv_dx, D)) * uint32_t(D) + uint32_t(key_axis(y, inv_dx, D))) *
             uint32_t(D) +
         uint32_t(key_axis(z, inv_dx, D));
}

// One axis of one grid's stencil (kernel.hpp:114-137 + transfer.hpp:65-68):
// base = floor(x/dx - k/4) (division form, bit-exact), w0/w1/g0 (g1 = -g0),
// xi0 = (base + k/4) dx - x (xi1 = xi0 + dx).
template <typename T>
struct Axis {
  int base;
  T w0, w1, g0, xi0;
};

template <typename T>
struct TwoPi;
template <>
struct TwoPi<double> {
  static constexpr double v = 2.0 * 3.14159265358979323846;
  static constexpr double inv = 1.0 / (2.0 * 3.14159265358979323846);
};
template <>
struct TwoPi<float> {
  static constexpr float v = 2.0f * 3.14159265358979323846f;
  static constexpr float inv = 1.0f / (2.0f * 3.14159265358979323846f);
};

template <typename T>
__device__ __forceinline__ int axis_base(T x, T dx, T kq) {
  return static_cast<int>(dfloor(sub_rn(div_rn(x, dx), kq)));
}

template <typename T>
__device__ __forceinline__ Axis<T> axis_pair(T x, T dx, T kq) {
  T s = sub_rn(div_rn(x, dx), kq);
  T fb = dfloor(s);
  Axis<T> a;
  a.base = static_cast<int>(fb);
  T f = sub_rn(s, fb);
  T sn, cs;
  dsincos(mul_rn(TwoPi<T>::v, f), &sn, &cs);
  sn = sn * TwoPi<T>::inv;
  a.w0 = T(1) - f + sn;
  a.w1 = f - sn;
  a.g0 = (cs - T(1)) / dx;
  a.xi0 = (T(a.base) + kq) * dx - x;
  return a;
}

// ------------------------------------------------------------ grid access

__device__ __forceinline__ int32_t dir_lookup(const int32_t* __restrict__ dir, int D, int bi, int bj,
                                              int bk) {
  if (bi < 0 || bj < 0 || bk < 0 || bi >= D || bj >= D || bk >= D) return -1;
  return __ldg(dir + (int64_t(bi) * D + bj) * D + bk);
}

constexpr int kBlockVals = 512;  // 2 grids * 4 values * 64 nodes

__device__ __forceinline__ uint64_t node_off(int32_t slot, int g, int i, int j, int k) {
  return uint64_t(slot) * kBlockVals + uint64_t(g) * 256 + uint64_t(((i & 3) << 4) | ((j & 3) << 2) | (k & 3));
}

// ------------------------------------------------------------ materials

// force_matrix: V0 * Kirchhoff stress (transfer.hpp:183-216).  Returns an
// error code (0 = ok).
template <typename T>
__device__ __forceinline__ int force_matrix(const M3<T>& F, T J, T vol0, const MatParam<T>& m,
                                            M3<T>& A) {
  if (m.model == kModelFC) {
    T dJ = det(F);
    if (!(dJ > T(0))) return kErrFcStress;
    M3<T> R = polar_rotation(F);
    M3<T> FmR;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) FmR.a[i][j] = F.a[i][j] - R.a[i][j];
    M3<T> P = mul_bt(FmR, F);  // (F - R) F^T
    T s2mu = T(2) * m.mu;
    T diag = m.lambda * dJ * (dJ - T(1));
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) A.a[i][j] = vol0 * (P.a[i][j] * s2mu + (i == j ? diag : T(0)));
    return 0;
  }
  if (m.model == kModelDP) {
    M3<T> U, V;
    V3<T> sg;
    svd3(F, U, sg, V);
    if (!(sg.z > T(0))) return kErrDpStress;
    T e0 = dlog(sg.x), e1 = dlog(sg.y), e2 = dlog(sg.z);
    T tr = e0 + e1 + e2;
    T s2mu = T(2) * m.mu;
    T t0 = s2mu * e0 + m.lambda * tr, t1 = s2mu * e1 + m.lambda * tr, t2 = s2mu * e2 + m.lambda * tr;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        A.a[i][j] = vol0 * (U.a[i][0] * t0 * U.a[j][0] + U.a[i][1] * t1 * U.a[j][1] +
                            U.a[i][2] * t2 * U.a[j][2]);
    return 0;
  }
  // j_fluid: -J p(J) I with p = B (J^-gamma - 1) (material.hpp:132-143)
  if (!(J > T(0))) return kErrFluidState;
  T pr = m.bulk * (dpow(J, -m.gamma) - T(1));
  T sd = vol0 * (-J * pr);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) A.a[i][j] = i == j ? sd : T(0);
  return 0;
}

// return_map_drucker_prager (material.hpp:157-175).
template <typename T>
__device__ __forceinline__ int return_map_dp(M3<T>& F, T alpha, T mu, T lambda) {
  if (!(det(F) > T(0))) return kErrReturnMap;
  M3<T> U, V;
  V3<T> sg;
  svd3(F, U, sg, V);
  T e0 = dlog(sg.x), e1 = dlog(sg.y), e2 = dlog(sg.z);
  T tr = e0 + e1 + e2;
  if (tr > T(0)) {
    e0 = e1 = e2 = T(0);
  } else {
    T t3 = tr / T(3);
    T d0 = e0 - t3, d1 = e1 - t3, d2 = e2 - t3;
    T dn = dsqrt(d0 * d0 + d1 * d1 + d2 * d2);
    T dgamma = dn + alpha * (T(3) * lambda + T(2) * mu) / (T(2) * mu) * tr;
    if (dgamma <= T(0)) return 0;
    T f = dgamma / dn;
    e0 -= d0 * f;
    e1 -= d1 * f;
    e2 -= d2 * f;
  }
  T s0 = dexp(e0), s1 = dexp(e1), s2 = dexp(e2);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      F.a[i][j] = U.a[i][0] * s0 * V.a[j][0] + U.a[i][1] * s1 * V.a[j][1] + U.a[i][2] * s2 * V.a[j][2];
  return 0;
}

// clamp_singular_values (material.hpp:179-191).
template <typename T>
__device__ __forceinline__ void clamp_singular_values(M3<T>& F, T floor_value) {
  M3<T> U, V;
  V3<T> sg;
  svd3(F, U, sg, V);
  bool touched = false;
  if (sg.x < floor_value) { sg.x = floor_value; touched = true; }
  if (sg.y < floor_value) { sg.y = floor_value; touched = true; }
  if (sg.z < floor_value) { sg.z = floor_value; touched = true; }
  if (!touched) return;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      F.a[i][j] = U.a[i][0] * sg.x * V.a[j][0] + U.a[i][1] * sg.y * V.a[j][1] + U.a[i][2] * sg.z * V.a[j][2];
}

// ------------------------------------------------------------ stencils

template <typename T>
struct Dual {
  Axis<T> ax[2][3];
};

template <typename T>
__device__ __forceinline__ Dual<T> dual_stencil(T x, T y, T z, T dx) {
  Dual<T> d;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const T kq = g == 0 ? T(-0.25) : T(0.25);  // T(k) * T(0.25), k = -1 / +1
    d.ax[g][0] = axis_pair(x, dx, kq);
    d.ax[g][1] = axis_pair(y, dx, kq);
    d.ax[g][2] = axis_pair(z, dx, kq);
  }
  return d;
}

// compute_apic_D (transfer.hpp:77-100).
template <typename T>
__device__ __forceinline__ M3<T> apic_D(const Dual<T>& ds, T dx) {
  M3<T> D;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) D.a[i][j] = T(0);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const Axis<T>* ax = ds.ax[g];
    const T wx[2] = {ax[0].w0, ax[0].w1}, wy[2] = {ax[1].w0, ax[1].w1}, wz[2] = {ax[2].w0, ax[2].w1};
    const T xx[2] = {ax[0].xi0, ax[0].xi0 + dx}, xy[2] = {ax[1].xi0, ax[1].xi0 + dx},
            xz[2] = {ax[2].xi0, ax[2].xi0 + dx};
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          T w = T(0.5) * wx[s] * wy[t] * wz[u];
          T xi[3] = {xx[s], xy[t], xz[u]};
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) D.a[a][b] += w * xi[a] * xi[b];
        }
  }
  return D;
}

// apic_d_inverse guard (transfer.hpp:222-229).
template <typename T>
__device__ __forceinline__ bool apic_d_inverse(const M3<T>& D, M3<T>& Di) {
  T sc = (D.a[0][0] + D.a[1][1] + D.a[2][2]) / T(3);
  T d = det(D);
  if (!(d > sc * sc * sc * T(1e-12))) return false;
  Di = scale(T(1) / d, adjugate(D));
  return true;
}

// mls_moment (transfer.hpp:127-150).
template <typename T>
__device__ __forceinline__ void mls_moment(const Dual<T>& ds, T dx, T (&Mm)[4][4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Mm[i][j] = T(0);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const Axis<T>* ax = ds.ax[g];
    const T wx[2] = {ax[0].w0, ax[0].w1}, wy[2] = {ax[1].w0, ax[1].w1}, wz[2] = {ax[2].w0, ax[2].w1};
    const T xx[2] = {ax[0].xi0, ax[0].xi0 + dx}, xy[2] = {ax[1].xi0, ax[1].xi0 + dx},
            xz[2] = {ax[2].xi0, ax[2].xi0 + dx};
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          T w = T(0.5) * wx[s] * wy[t] * wz[u];
          T P[4] = {T(1), xx[s], xy[t], xz[u]};
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) Mm[a][b] += w * P[a] * P[b];
        }
  }
}

template <typename T>
__device__ __forceinline__ M3<T> load_m3(const PState<T>& p, int k, uint64_t i) {
  M3<T> m;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) m.a[r][c] = __ldg(p.f + uint64_t(k + 3 * r + c) * p.n + i);
  return m;
}

template <typename T>
__device__ __forceinline__ void store_m3(const PState<T>& p, int k, uint64_t i, const M3<T>& m) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) p.f[uint64_t(k + 3 * r + c) * p.n + i] = m.a[r][c];
}

// ================================================================ kernels

// K1: block key per particle in current order (simulation.hpp:255-266).
template <typename T>
__global__ void key_kernel(PState<T> cur, T inv_dx, int D, uint32_t* __restrict__ keys) {
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= cur.n) return;
  keys[i] = block_key(__ldg(cur.f + kX * cur.n + i), __ldg(cur.f + (kX + 1) * cur.n + i),
                      __ldg(cur.f + (kX + 2) * cur.n + i), inv_dx, D);
}

// K3: activation over sorted particles (grid.hpp:114-145): 2-cell inset check
// (OutOfDomainError with the lowest sorted index and its first failing axis),
// footprint blocks plus one positive halo block per axis.  The footprint's
// lower/upper block offsets relative to the key block are OR-reduced across
// same-key lanes of a warp so each warp marks each distinct box once.
template <typename T>
__global__ void activate_kernel(PState<T> cur, const uint32_t* __restrict__ perm, T inv_dx, int res,
                                int D, uint32_t* __restrict__ flags, DevStatus* st, int step) {
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool valid = i < cur.n;
  int lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
  if (valid) {
    uint32_t src = perm[i];
    bool bad = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      T s = mul_rn(__ldg(cur.f + (kX + a) * cur.n + src), inv_dx);
      if (!bad && !(s >= T(2) && s <= T(res - 2))) {
        record_error(st, step, kPhaseActivate, i, a, kErrOutOfDomain);
        bad = true;
      }
      int base_plus = static_cast<int>(dfloor(sub_rn(s, T(0.25))));
      int base_minus = static_cast<int>(dfloor(add_rn(s, T(0.25))));
      lo[a] = base_plus >> 2;
      hi[a] = ((base_minus + 1) >> 2) + 1;
    }
    if (bad) {
      valid = false;
      hi[0] = -1;
    }
  }
  // Warp dedupe: lanes with identical boxes mark once.
  uint64_t boxkey = valid ? ((uint64_t(uint32_t(lo[0]) & 0xfff) << 48) | (uint64_t(uint32_t(lo[1]) & 0xfff) << 36) |
                             (uint64_t(uint32_t(lo[2]) & 0xfff) << 24) | (uint64_t(uint32_t(hi[0]) & 0xff) << 16) |
                             (uint64_t(uint32_t(hi[1]) & 0xff) << 8) | uint64_t(uint32_t(hi[2]) & 0xff))
                          : ~0ull;
  uint32_t peers = __match_any_sync(0xffffffffu, boxkey);
  bool leader = (__ffs(peers) - 1) == int(threadIdx.x & 31);
  if (!valid || !leader) return;
  for (int bi = lo[0]; bi <= hi[0]; ++bi)
    for (int bj = lo[1]; bj <= hi[1]; ++bj)
      for (int bk = lo[2]; bk <= hi[2]; ++bk)
        if (bi >= 0 && bj >= 0 && bk >= 0 && bi < D && bj < D && bk < D)
          flags[(int64_t(bi) * D + bj) * D + bk] = 1u;
}

// K3b: directory from the exclusive scan of flags (in place in dir), active
// list in ascending directory order, flags reset for the next substep.
__global__ void compact_kernel(uint32_t* __restrict__ flags, int32_t* __restrict__ dir,
                               uint32_t* __restrict__ active, uint64_t nd, uint32_t cap,
                               DevStatus* st) {
  uint64_t d = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d >= nd) return;
  uint32_t f = flags[d];
  uint32_t s = static_cast<uint32_t>(dir[d]);
  if (f) {
    if (s < cap) {
      active[s] = static_cast<uint32_t>(d);
    } else {
      st->overflow = 1u;
    }
    flags[d] = 0u;
  } else {
    dir[d] = -1;
  }
  if (d == nd - 1) st->n_active = s + f;
}

// K4: clear the active part of the pool (grid.hpp:148-151).
template <typename T>
__global__ void clear_kernel(T* __restrict__ pool, const DevStatus* st, uint32_t cap) {
  uint32_t na = st->n_active;
  if (na > cap) na = cap;
  uint64_t total = uint64_t(na) * kBlockVals;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x)
    pool[k] = T(0);
}

__device__ __forceinline__ void red_add(double* a, double v) { atomicAdd(a, v); }
__device__ __forceinline__ void red_add(float* a, float v) { atomicAdd(a, v); }

// K5: P2G (scatter_all, simulation.hpp:279-337; scatter_one, transfer.hpp:235-283;
// MLS force scatter, transfer.hpp:335-369).  One thread per sorted particle,
// 16 nodes x 4 values into the block pool.
template <typename T, int SCHEME>
__global__ void __launch_bounds__(128) p2g_kernel(PState<T> cur, const uint32_t* __restrict__ perm,
                                                  StepConst<T> c, const int32_t* __restrict__ dir,
                                                  T* __restrict__ pool, uint32_t cap, DevStatus* st,
                                                  int step) {
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= cur.n) return;
  const uint32_t src = __ldg(perm + i);
  const uint64_t n = cur.n;
  const T x = __ldg(cur.f + kX * n + src), y = __ldg(cur.f + (kX + 1) * n + src),
          z = __ldg(cur.f + (kX + 2) * n + src);
  const T vx = __ldg(cur.f + kV * n + src), vy = __ldg(cur.f + (kV + 1) * n + src),
          vz = __ldg(cur.f + (kV + 2) * n + src);
  const T m = __ldg(cur.f + kMass * n + src);
  const T vol0 = __ldg(cur.f + kVol * n + src);
  const T J = __ldg(cur.f + kJ * n + src);
  const uint32_t mi = __ldg(cur.mat + src);
  const M3<T> F = load_m3(cur, kF, src);
  M3<T> A;
  int e = force_matrix(F, J, vol0, c.mats[mi < kMaxMaterials ? mi : 0], A);
  if (e) {
    record_error(st, step, kPhaseP2G, i, 0, e);
    return;
  }
  const T dx = c.dx, dt = c.dt;
  const Dual<T> ds = dual_stencil(x, y, z, dx);
  M3<T> Cm;
  if (SCHEME != kSchemePic) {
    M3<T> Dm = apic_D(ds, dx), Di;
    if (!apic_d_inverse(Dm, Di)) {
      record_error(st, step, kPhaseP2G, i, 0, kErrNearSingularD);
      return;
    }
    Cm = mul(load_m3(cur, kB, src), Di);
  }
  T Minv[4][4];
  if (SCHEME == kSchemeMls) {
    T Mm[4][4];
    mls_moment(ds, dx, Mm);
    if (!gauss_inverse4(Mm, Minv)) {
      record_error(st, step, kPhaseP2G, i, 0, kErrSingularMls);
      return;
    }
  }
  const int D = c.D;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const Axis<T>* ax = ds.ax[g];
    const T wx[2] = {ax[0].w0, ax[0].w1}, wy[2] = {ax[1].w0, ax[1].w1}, wz[2] = {ax[2].w0, ax[2].w1};
    const T gx[2] = {ax[0].g0, -ax[0].g0}, gy[2] = {ax[1].g0, -ax[1].g0}, gz[2] = {ax[2].g0, -ax[2].g0};
    const T xx[2] = {ax[0].xi0, ax[0].xi0 + dx}, xy[2] = {ax[1].xi0, ax[1].xi0 + dx},
            xz[2] = {ax[2].xi0, ax[2].xi0 + dx};
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int ni = ax[0].base + s, nj = ax[1].base + t, nk = ax[2].base + u;
          const int32_t slot = dir_lookup(dir, D, ni >> 2, nj >> 2, nk >> 2);
          if (slot < 0 || uint32_t(slot) >= cap) {
            record_error(st, step, kPhaseP2G, i, 0, kErrInactive);
            continue;
          }
          const T w = wx[s] * wy[t] * wz[u];
          const T wm = w * m;
          T mx = vx * wm, my = vy * wm, mz = vz * wm;
          if (SCHEME != kSchemePic) {
            const V3<T> cx = mul(Cm, V3<T>{xx[s], xy[t], xz[u]});
            mx += cx.x * wm;
            my += cx.y * wm;
            mz += cx.z * wm;
          }
          if (SCHEME != kSchemeMls) {
            const V3<T> gw = {gx[s] * wy[t] * wz[u], wx[s] * gy[t] * wz[u], wx[s] * wy[t] * gz[u]};
            const V3<T> ag = mul(A, gw);
            mx -= ag.x * dt;
            my -= ag.y * dt;
            mz -= ag.z * dt;
          } else {
            T q[4];
            const T P[4] = {T(1), xx[s], xy[t], xz[u]};
#pragma unroll
            for (int a = 0; a < 4; ++a)
              q[a] = Minv[a][0] * P[0] + Minv[a][1] * P[1] + Minv[a][2] * P[2] + Minv[a][3] * P[3];
            const V3<T> ag = mul(A, V3<T>{w * q[1], w * q[2], w * q[3]});
            mx -= ag.x * dt;
            my -= ag.y * dt;
            mz -= ag.z * dt;
          }
          T* nd = pool + node_off(slot, g, ni, nj, nk);
          red_add(nd, wm);
          red_add(nd + 64, mx);
          red_add(nd + 128, my);
          red_add(nd + 192, mz);
        }
  }
}

// K6: grid update on both grids (grid_update_block, transfer.hpp:419-440;
// BoundaryCondition::contains/apply, grid.hpp:34-55).
template <typename T>
__global__ void grid_update_kernel(T* __restrict__ pool, const uint32_t* __restrict__ active,
                                   const DevStatus* st, uint32_t cap, StepConst<T> c,
                                   const BcParam<T>* __restrict__ bcs) {
  uint32_t na = st->n_active;
  if (na > cap) na = cap;
  const uint64_t total = uint64_t(na) * 128;
  const int D = c.D;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t slot = uint32_t(k >> 7);
    const int g = int(k >> 6) & 1;
    const int l = int(k & 63);
    T* base = pool + uint64_t(slot) * kBlockVals + g * 256 + l;
    const T mass = base[0];
    if (mass > c.mass_eps) {
      const T inv = T(1) / mass;
      T v[3] = {base[64] * inv + c.gravity[0] * c.dt, base[128] * inv + c.gravity[1] * c.dt,
                base[192] * inv + c.gravity[2] * c.dt};
      if (c.n_boundaries > 0) {
        const uint32_t d = __ldg(active + slot);
        const int bz = int(d % uint32_t(D)), by = int((d / uint32_t(D)) % uint32_t(D)),
                  bx = int(d / (uint32_t(D) * uint32_t(D)));
        const T off = (g == 0 ? T(-0.25) : T(0.25)) * c.dx;
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

// K7: G2P gather + state update + advection + reductions
// (gather_all, simulation.hpp:339-396; gather_one, transfer.hpp:465-510;
// update_particle_state, transfer.hpp:594-627).  Reads cur at perm[i],
// writes nxt at i (sorted order).
template <typename T, int SCHEME>
__global__ void __launch_bounds__(128) g2p_kernel(PState<T> cur, PState<T> nxt,
                                                  const uint32_t* __restrict__ perm, StepConst<T> c,
                                                  const int32_t* __restrict__ dir,
                                                  const T* __restrict__ pool, uint32_t cap,
                                                  DevStatus* st, int step) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool live = i < cur.n;
  T s2 = T(0);
  bool fluid = false;
  T Jout = T(1);
  uint32_t mi = 0;
  bool bad = false;
  if (live) {
    const uint32_t src = __ldg(perm + i);
    const uint64_t n = cur.n;
    T x = __ldg(cur.f + kX * n + src), y = __ldg(cur.f + (kX + 1) * n + src),
      z = __ldg(cur.f + (kX + 2) * n + src);
    const T m = __ldg(cur.f + kMass * n + src);
    const T vol0 = __ldg(cur.f + kVol * n + src);
    T J = __ldg(cur.f + kJ * n + src);
    mi = __ldg(cur.mat + src);
    const MatParam<T>& mp = c.mats[mi < kMaxMaterials ? mi : 0];
    const T dx = c.dx, dt = c.dt;
    const Dual<T> ds = dual_stencil(x, y, z, dx);
    // gather: v = 1/2 sum w v~, B = 1/2 sum w v~ xi^T, gradv = 1/2 sum v~ gw^T
    T v[3] = {T(0), T(0), T(0)};
    M3<T> Bn, G;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        Bn.a[a][b] = T(0);
        G.a[a][b] = T(0);
      }
    const int D = c.D;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const Axis<T>* ax = ds.ax[g];
      const T wx[2] = {ax[0].w0, ax[0].w1}, wy[2] = {ax[1].w0, ax[1].w1}, wz[2] = {ax[2].w0, ax[2].w1};
      const T gx[2] = {ax[0].g0, -ax[0].g0}, gy[2] = {ax[1].g0, -ax[1].g0}, gz[2] = {ax[2].g0, -ax[2].g0};
      const T xx[2] = {ax[0].xi0, ax[0].xi0 + dx}, xy[2] = {ax[1].xi0, ax[1].xi0 + dx},
              xz[2] = {ax[2].xi0, ax[2].xi0 + dx};
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int ni = ax[0].base + s, nj = ax[1].base + t, nk = ax[2].base + u;
            const int32_t slot = dir_lookup(dir, D, ni >> 2, nj >> 2, nk >> 2);
            if (slot < 0 || uint32_t(slot) >= cap) {
              record_error(st, step, kPhaseG2P, i, 0, kErrInactive);
              continue;
            }
            const T* nd = pool + node_off(slot, g, ni, nj, nk);
            const T vn[3] = {__ldg(nd + 64), __ldg(nd + 128), __ldg(nd + 192)};
            const T hw = T(0.5) * (wx[s] * wy[t] * wz[u]);
            const T xi[3] = {xx[s], xy[t], xz[u]};
            const T gw[3] = {gx[s] * wy[t] * wz[u], wx[s] * gy[t] * wz[u], wx[s] * wy[t] * gz[u]};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              v[a] += vn[a] * hw;
#pragma unroll
              for (int b = 0; b < 3; ++b) {
                Bn.a[a][b] += hw * vn[a] * xi[b];
                G.a[a][b] += T(0.5) * vn[a] * gw[b];
              }
            }
          }
    }
    // update_particle_state
    M3<T> L = G;
    if (SCHEME == kSchemeMls) {
      M3<T> Dm = apic_D(ds, dx), Di;
      if (!apic_d_inverse(Dm, Di)) {
        record_error(st, step, kPhaseG2P, i, 0, kErrNearSingularD);
        bad = true;
      }
      L = mul(Bn, Di);
    }
    M3<T> Bout = SCHEME == kSchemePic ? load_m3(cur, kB, src) : Bn;
    M3<T> Fout = load_m3(cur, kF, src);
    if (mp.model == kModelFluid) {
      fluid = true;
      if (mp.viscosity > T(0) && SCHEME != kSchemePic) {
        const T f = dexp(-mp.viscosity * dt / (mp.density * dx * dx));
        const T tb = trace(Bout) / T(3);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) Bout.a[a][b] = (a == b ? tb : T(0)) + (Bout.a[a][b] - (a == b ? tb : T(0))) * f;
      }
      J *= T(1) + dt * trace(L);
      if (!(J > T(0))) {
        record_error(st, step, kPhaseG2P, i, 0, kErrFluidJ);
        bad = true;
      }
    } else {
      M3<T> Ld;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) Ld.a[a][b] = (a == b ? T(1) : T(0)) + L.a[a][b] * dt;
      M3<T> Fn = mul(Ld, Fout);
      if (c.clamp_singular) clamp_singular_values(Fn, c.clamp_floor);
      if (mp.model == kModelDP) {
        int e = return_map_dp(Fn, mp.dp_alpha, mp.mu, mp.lambda);
        if (e) {
          record_error(st, step, kPhaseG2P, i, 0, e);
          bad = true;
        }
      } else if (!(det(Fn) > T(0))) {
        record_error(st, step, kPhaseG2P, i, 0, kErrFInverted);
        bad = true;
      }
      Fout = Fn;
    }
    x += v[0] * dt;
    y += v[1] * dt;
    z += v[2] * dt;
    // write the new state in sorted order
    nxt.f[kX * n + i] = x;
    nxt.f[(kX + 1) * n + i] = y;
    nxt.f[(kX + 2) * n + i] = z;
    nxt.f[kV * n + i] = v[0];
    nxt.f[(kV + 1) * n + i] = v[1];
    nxt.f[(kV + 2) * n + i] = v[2];
    store_m3(nxt, kF, i, Fout);
    store_m3(nxt, kB, i, Bout);
    nxt.f[kJ * n + i] = J;
    nxt.f[kMass * n + i] = m;
    nxt.f[kVol * n + i] = vol0;
    nxt.mat[i] = mi;
    s2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    Jout = J;
    if (!dfinite(s2) || !dfinite(x * x + y * y + z * z)) atomicOr(&st->nonfinite, 1u);
    (void)bad;
  }
  // vmax^2 reduction (NaN never wins, like std::max(vm, s2)).
  T vm = (s2 > T(0)) ? s2 : T(0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T other = __shfl_xor_sync(0xffffffffu, vm, o);
    vm = (vm < other) ? other : vm;
  }
  __shared__ T wmax[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) wmax[wid] = vm;
  __syncthreads();
  if (wid == 0) {
    T b = lane < int(blockDim.x >> 5) ? wmax[lane] : T(0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      T other = __shfl_xor_sync(0xffffffffu, b, o);
      b = (b < other) ? other : b;
    }
    if (lane == 0 && b > T(0)) atomicMax(&st->vmax2, as_ordered_bits(b));
  }
  // per-material min J over fluid particles
  uint32_t todo = __ballot_sync(0xffffffffu, live && fluid);
  while (todo) {
    const uint32_t lead_mat = __shfl_sync(0xffffffffu, mi, __ffs(todo) - 1);
    const bool mine = live && fluid && mi == lead_mat;
    T jv = mine ? Jout : T(INFINITY);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      T other = __shfl_xor_sync(0xffffffffu, jv, o);
      jv = (other < jv) ? other : jv;
    }
    if (lane == __ffs(todo) - 1 && lead_mat < kMaxMaterials && jv > T(0))
      atomicMin(&st->minj[lead_mat], as_ordered_bits(jv));
    todo &= ~__ballot_sync(0xffffffffu, mine);
  }
}

// Status reset before a substep.
__global__ void status_reset_kernel(DevStatus* st, int reset_err) {
  if (threadIdx.x == 0) {
    if (reset_err) st->err = ~0ull;
    st->vmax2 = 0ull;
    st->nonfinite = 0u;
    st->n_active = 0u;
    st->overflow = 0u;
  }
  if (threadIdx.x < kMaxMaterials) st->minj[threadIdx.x] = 0x7ff0000000000000ull;  // +inf
}

// AoS <-> SoA transposes for the C-ABI (Particle<T> layout, transfer.hpp:19-28).
// One thread per (particle, field) word so both sides stay coalesced enough.
template <typename T>
__global__ void aos_to_soa_kernel(const T* __restrict__ aos, PState<T> p) {
  constexpr int W = kNumFields + 1;  // 27 fields + material word(s)
  const uint64_t total = p.n * W;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = k / W;
    const int f = int(k - i * W);
    if (f < kNumFields)
      p.f[uint64_t(f) * p.n + i] = aos[k];
    else
      p.mat[i] = *reinterpret_cast<const uint32_t*>(aos + k);
  }
}

template <typename T>
__global__ void soa_to_aos_kernel(PState<T> p, T* __restrict__ aos) {
  constexpr int W = kNumFields + 1;
  const uint64_t total = p.n * W;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = k / W;
    const int f = int(k - i * W);
    if (f < kNumFields) {
      aos[k] = p.f[uint64_t(f) * p.n + i];
    } else {
      T word = T(0);
      *reinterpret_cast<uint32_t*>(&word) = p.mat[i];
      aos[k] = word;
    }
  }
}

// Per-particle dual-stencil bases (binning parity hook).
template <typename T>
__global__ void bases_kernel(PState<T> p, T dx, int32_t* __restrict__ out) {
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const T kq = g == 0 ? T(-0.25) : T(0.25);
#pragma unroll
    for (int a = 0; a < 3; ++a) out[(i * 2 + g) * 3 + a] = axis_base(p.f[uint64_t(kX + a) * p.n + i], dx, kq);
  }
}

// Grid pool -> reference Block::nodes order for the grid facade.
template <typename T>
__global__ void grid_export_kernel(const T* __restrict__ pool, const uint32_t* __restrict__ active,
                                   uint64_t nb, int D, int32_t* __restrict__ coords,
                                   double* __restrict__ nodes) {
  const uint64_t total = nb * 128;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = k >> 7;
    const int nn = int(k & 127);
    const int g = nn >> 6, l = nn & 63;
    const T* base = pool + b * kBlockVals + g * 256 + l;
    if (nodes) {
      double* o = nodes + k * 4;
      o[0] = double(base[0]);
      o[1] = double(base[64]);
      o[2] = double(base[128]);
      o[3] = double(base[192]);
    }
    if (coords && nn == 0) {
      const uint32_t d = active[b];
      coords[b * 3 + 2] = int(d % uint32_t(D));
      coords[b * 3 + 1] = int((d / uint32_t(D)) % uint32_t(D));
      coords[b * 3 + 0] = int(d / (uint32_t(D) * uint32_t(D)));
    }
  }
}

// compute_diagnostics on the device (simulation.hpp:55-69): 11 sums/max.
template <typename T>
__global__ void diagnostics_kernel(PState<T> p, double* __restrict__ acc /* 10 sums */,
                                   unsigned long long* __restrict__ vmax_bits) {
  double s[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  double vm = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < p.n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double m = double(p.f[kMass * p.n + i]);
    const double x[3] = {double(p.f[kX * p.n + i]), double(p.f[(kX + 1) * p.n + i]), double(p.f[(kX + 2) * p.n + i])};
    const double v[3] = {double(p.f[kV * p.n + i]), double(p.f[(kV + 1) * p.n + i]), double(p.f[(kV + 2) * p.n + i])};
    s[0] += v[0] * m; s[1] += v[1] * m; s[2] += v[2] * m;
    s[3] += (x[1] * v[2] - x[2] * v[1]) * m;
    s[4] += (x[2] * v[0] - x[0] * v[2]) * m;
    s[5] += (x[0] * v[1] - x[1] * v[0]) * m;
    s[6] += v[0]; s[7] += v[1]; s[8] += v[2];
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
