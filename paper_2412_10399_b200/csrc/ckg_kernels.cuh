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
  T* tau;         // 6 fields: V0 * Kirchhoff stress of the current F (symmetric, xx xy xz yy yz zz)
  uint64_t n;       // live particles in this window
  uint64_t stride;  // distance between fields (buffer capacity); f/mat/tau may be offset into the buffer
  __device__ __forceinline__ T& at(int k, uint64_t i) const { return f[uint64_t(k) * stride + i]; }
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
  const T* dtp;  // device-resident dt (frame driver); null: use dt
  T gravity[3];
  int res, D, scheme, n_materials, clamp_singular, n_boundaries;
  int pow2;  // dx is a power of two: x/dx == x*inv_dx exactly (both are exact scalings)
  int quad;  // quadratic B-spline baseline (single grid, slot 0)
  int dense; // block pool indexed by the block key (fused G2P2G mode, ckg_g2p2g.cuh)
  MatParam<T> mats[kMaxMaterials];
};

template <typename T>
__device__ __forceinline__ T step_dt(const StepConst<T>& c) {
  return c.dtp ? *c.dtp : c.dt;
}

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
  unsigned int n_active_prev;   // n_active of the previous substep (set by the status reset)
  unsigned int overflow;
  unsigned int inset_fail;      // some particle violated the 2-cell inset (index fixed up after the sort)
  unsigned int nchanged;        // particles whose block key differs from the stored sorted key
  unsigned int work[4];         // persistent-kernel work counters (P2G, G2P)
  unsigned int item_lo, item_hi;    // active-list range the transfer kernels walk
  unsigned int grid_lo, grid_hi;    // slot range of the grid update
  unsigned int clear_lo, clear_hi;  // slot range cleared before P2G
  unsigned long long perr;      // packed error of the NEXT substep's scatter (fused G2P2G), ~0 = none
  unsigned int spill_n;         // deterministic mode: out-of-tile P2G records
};

// err = step<<56 | phase<<52 | particle<<12 | axis<<8 | code
__device__ __forceinline__ void record_error_at(unsigned long long* slot, int step, int phase, uint64_t particle,
                                                int axis, int code) {
  unsigned long long p = (static_cast<unsigned long long>(step & 0xff) << 56) |
                         (static_cast<unsigned long long>(phase & 0xf) << 52) |
                         ((particle & 0xffffffffffull) << 12) |
                         (static_cast<unsigned long long>(axis & 0xf) << 8) |
                         static_cast<unsigned long long>(code & 0xff);
  atomicMin(slot, p);
}
__device__ __forceinline__ void record_error(DevStatus* st, int step, int phase, uint64_t particle,
                                             int axis, int code) {
  record_error_at(&st->err, step, phase, particle, axis, code);
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

// x/dx exactly as the reference rounds it (kernel.hpp:116).  For a
// power-of-two dx (every benchmark scene: extent 1, res 2^k) the product with
// inv_dx is the same exact scaling, so the division is skipped.
template <typename T>
__device__ __forceinline__ T over_dx(T x, T dx, T inv_dx, int pow2) {
  return pow2 ? mul_rn(x, inv_dx) : div_rn(x, dx);
}

template <typename T>
__device__ __forceinline__ int axis_base(T x, T dx, T inv_dx, int pow2, T kq) {
  return static_cast<int>(dfloor(sub_rn(over_dx(x, dx, inv_dx, pow2), kq)));
}

// sin(2 pi f), cos(2 pi f) for f in [0,1): sincospi(2f) (2f is exact) instead
// of sin(fl(2 pi f)) — differs from the reference by the rounding of 2 pi f
// (<= 1 ulp of the argument); the paired scheme keeps w0 + w1 = 1 and
// g1 = -g0 exact regardless (kernel.hpp:103-105).
// sin/cos(2 pi f) for the stencil fraction f in [0, 1): exact reduction to
// t = f - round(f) - q/4 in [-1/8, 1/8] (Sterbenz), then the Taylor series of
// sin(2 pi t) (to t^15) and cos(2 pi t) (to t^16), whose truncation error at
// |2 pi t| <= pi/4 is below 1e-16 relative; ~1-2 ulp overall, branch-free, two
// independent FMA chains (the library sincospi costs ~70 instructions with its
// general range reduction).
// Polynomial coefficients in the constant bank: DFMA reads c[bank][off]
// operands directly, where literal FP64 constants cost two uniform-register
// moves (UMOV) per use in every unrolled evaluation.
#ifndef CKG_SINCOS_CBANK
#define CKG_SINCOS_CBANK 1
#endif
#if CKG_SINCOS_CBANK
__constant__ double kSinPoly[8] = {-0.7181223017785006, 3.819952584848282,  -15.09464257682299, 42.058693944897655,
                                   -76.70585975306139,  81.60524927607506,  -41.34170224039976, 6.283185307179586};
__constant__ double kCosPoly[9] = {0.28200596845579123, -1.714390711088672, 7.903536371318469,
                                   -26.4262567833744,   60.24464137187666,  -85.45681720669373,
                                   64.9393940226683,    -19.739208802178716, 1.0};
#endif
__device__ __forceinline__ void sincos_2pi(double f, double* s, double* c) {
  const double r = f - rint(f);
  const double qd = rint(4.0 * r);
  const double t = fma(qd, -0.25, r);
  const double t2 = t * t;
#if CKG_SINCOS_CBANK
  double ps = kSinPoly[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) ps = fma(ps, t2, kSinPoly[k]);
  double pc = kCosPoly[0];
#pragma unroll
  for (int k = 1; k < 9; ++k) pc = fma(pc, t2, kCosPoly[k]);
#else
  double ps = -0.7181223017785006;
  ps = fma(ps, t2, 3.819952584848282);
  ps = fma(ps, t2, -15.09464257682299);
  ps = fma(ps, t2, 42.058693944897655);
  ps = fma(ps, t2, -76.70585975306139);
  ps = fma(ps, t2, 81.60524927607506);
  ps = fma(ps, t2, -41.34170224039976);
  ps = fma(ps, t2, 6.283185307179586);
  double pc = 0.28200596845579123;
  pc = fma(pc, t2, -1.714390711088672);
  pc = fma(pc, t2, 7.903536371318469);
  pc = fma(pc, t2, -26.4262567833744);
  pc = fma(pc, t2, 60.24464137187666);
  pc = fma(pc, t2, -85.45681720669373);
  pc = fma(pc, t2, 64.9393940226683);
  pc = fma(pc, t2, -19.739208802178716);
  pc = fma(pc, t2, 1.0);
#endif
  const double sn = t * ps;
  const int q = int(qd) & 3;  // quadrant: angle = 2 pi t + q pi/2
  *s = (q == 0) ? sn : (q == 1) ? pc : (q == 2) ? -sn : -pc;
  *c = (q == 0) ? pc : (q == 1) ? -sn : (q == 2) ? -pc : sn;
}
__device__ __forceinline__ void sincos_2pi(float f, float* s, float* c) { sincospif(f + f, s, c); }

template <typename T>
__device__ __forceinline__ Axis<T> axis_pair(T x, T dx, T inv_dx, int pow2, T kq) {
  T s = sub_rn(over_dx(x, dx, inv_dx, pow2), kq);
  T fb = dfloor(s);
  Axis<T> a;
  a.base = static_cast<int>(fb);
  T f = s - fb;  // exact (Sterbenz)
  T sn, cs;
  sincos_2pi(f, &sn, &cs);
  sn = sn * TwoPi<T>::inv;
  a.w0 = T(1) - f + sn;
  a.w1 = f - sn;
  a.g0 = (cs - T(1)) * inv_dx;
  a.xi0 = (T(a.base) + kq) * dx - x;
  return a;
}

// One axis of one grid from a given sin/cos(2 pi f) (unscaled): the same
// operations as axis_pair after its sincos.
template <typename T>
__device__ __forceinline__ Axis<T> axis_with(T x, T dx, T inv_dx, int pow2, T kq, T sn, T cs) {
  const T s = sub_rn(over_dx(x, dx, inv_dx, pow2), kq);
  const T fb = dfloor(s);
  Axis<T> a;
  a.base = static_cast<int>(fb);
  const T f = s - fb;
  sn = sn * TwoPi<T>::inv;
  a.w0 = T(1) - f + sn;
  a.w1 = f - sn;
  a.g0 = (cs - T(1)) * inv_dx;
  a.xi0 = (T(a.base) + kq) * dx - x;
  return a;
}

// The -1 grid's axis (kq = -1/4) from the +1 grid's sincos when the two
// fractions differ by exactly 1/2 (sin/cos(2 pi (f + 1/2)) = -sin/cos(2 pi f),
// as axis_pair_dual); *snp / *csp return the +1 grid's (unscaled) values.
template <typename T>
__device__ __forceinline__ Axis<T> axis_pair_lo(T x, T dx, T inv_dx, int pow2, T* snp, T* csp) {
  const T xd = over_dx(x, dx, inv_dx, pow2);
  const T sm = sub_rn(xd, T(-0.25)), sp = sub_rn(xd, T(0.25));
  const T fbm = dfloor(sm), fbp = dfloor(sp);
  const T fm = sm - fbm, fp = sp - fbp;
  T sn, cs;
  sincos_2pi(fp, snp, csp);
  const T d = fm - fp;
  if (d == T(0.5) || d == T(-0.5)) {
    sn = -*snp;
    cs = -*csp;
  } else {
    sincos_2pi(fm, &sn, &cs);
  }
  Axis<T> a;
  a.base = static_cast<int>(fbm);
  sn = sn * TwoPi<T>::inv;
  a.w0 = T(1) - fm + sn;
  a.w1 = fm - sn;
  a.g0 = (cs - T(1)) * inv_dx;
  a.xi0 = (T(a.base) + T(-0.25)) * dx - x;
  return a;
}

// ------------------------------------------------------------ grid access

__device__ __forceinline__ int32_t dir_lookup(const int32_t* __restrict__ dir, int D, int bi, int bj,
                                              int bk) {
  if (bi < 0 || bj < 0 || bk < 0 || bi >= D || bj >= D || bk >= D) return -1;
  return __ldg(dir + (int64_t(bi) * D + bj) * D + bk);
}

constexpr int kBlockVals = 512;  // 2 grids * 4 values * 64 nodes

// Pool slot of block (bi, bj, bk): the directory's compact slot, or (dense
// pools, fused G2P2G mode) the block key itself for an active block.
__device__ __forceinline__ int32_t pool_slot(const int32_t* __restrict__ dir, int D, int bi, int bj, int bk,
                                             int dense) {
  const int32_t s = dir_lookup(dir, D, bi, bj, bk);
  return (dense && s >= 0) ? (bi * D + bj) * D + bk : s;
}

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
    M3<T> R = polar_rotation_fast(F);
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

// V0 * Kirchhoff stress as 6 symmetric components (force_matrix,
// transfer.hpp:183-216; tau is symmetric for all three models).
template <typename T>
__device__ __forceinline__ int stress_tau6(const M3<T>& F, T J, T vol0, const MatParam<T>& m, T (&t6)[6]) {
  M3<T> A;
  const int e = force_matrix(F, J, vol0, m, A);
  t6[0] = A.a[0][0];
  t6[1] = T(0.5) * (A.a[0][1] + A.a[1][0]);
  t6[2] = T(0.5) * (A.a[0][2] + A.a[2][0]);
  t6[3] = A.a[1][1];
  t6[4] = T(0.5) * (A.a[1][2] + A.a[2][1]);
  t6[5] = A.a[2][2];
  return e;
}

// return_map_drucker_prager (material.hpp:157-175).  Also returns the
// Kirchhoff stress of the projected F (what force_matrix would compute from
// it at the next P2G, transfer.hpp:197-208): the projected F has singular
// vectors U, V and singular values exp(eps), so tau = U diag(2 mu eps +
// lambda tr eps) U^T with no second SVD.
template <typename T>
__device__ __forceinline__ int return_map_dp(M3<T>& F, T alpha, T mu, T lambda, T (&tau6)[6]) {
  if (!(det(F) > T(0))) return kErrReturnMap;
  M3<T> U, V;
  V3<T> sg;
  svd3_inl(F, U, sg, V);
  T e0 = dlog(sg.x), e1 = dlog(sg.y), e2 = dlog(sg.z);
  T tr = e0 + e1 + e2;
  bool project = true;
  if (tr > T(0)) {
    e0 = e1 = e2 = T(0);
  } else {
    T t3 = tr / T(3);
    T d0 = e0 - t3, d1 = e1 - t3, d2 = e2 - t3;
    T dn = dsqrt(d0 * d0 + d1 * d1 + d2 * d2);
    T dgamma = dn + alpha * (T(3) * lambda + T(2) * mu) / (T(2) * mu) * tr;
    if (dgamma <= T(0)) {
      project = false;
    } else {
      T f = dgamma / dn;
      e0 -= d0 * f;
      e1 -= d1 * f;
      e2 -= d2 * f;
    }
  }
  if (project) {
    T s0 = dexp(e0), s1 = dexp(e1), s2 = dexp(e2);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        F.a[i][j] = U.a[i][0] * s0 * V.a[j][0] + U.a[i][1] * s1 * V.a[j][1] + U.a[i][2] * s2 * V.a[j][2];
  }
  const T te = e0 + e1 + e2;
  const T t0 = T(2) * mu * e0 + lambda * te, t1 = T(2) * mu * e1 + lambda * te, t2 = T(2) * mu * e2 + lambda * te;
  int k = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j)
      tau6[k++] = U.a[i][0] * t0 * U.a[j][0] + U.a[i][1] * t1 * U.a[j][1] + U.a[i][2] * t2 * U.a[j][2];
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

// Both grids' slices of one axis from a single sincos: the -1 and +1 grid
// fractions of the same coordinate differ by exactly 1/2 (mod 1) whenever
// x/dx +- 1/4 round exactly (always, away from powers of two), and
// sin/cos(2 pi (f + 1/2)) = -sin/cos(2 pi f).  Otherwise both are evaluated.
template <typename T>
__device__ __forceinline__ void axis_pair_dual(T x, T dx, T inv_dx, int pow2, Axis<T>& am, Axis<T>& ap,
                                               T* snp_out = nullptr) {
  const T xd = over_dx(x, dx, inv_dx, pow2);
  const T sm = sub_rn(xd, T(-0.25)), sp = sub_rn(xd, T(0.25));
  const T fbm = dfloor(sm), fbp = dfloor(sp);
  const T fm = sm - fbm, fp = sp - fbp;
  T snp, csp, snm, csm;
  sincos_2pi(fp, &snp, &csp);
  const T d = fm - fp;
  if (d == T(0.5) || d == T(-0.5)) {
    snm = -snp;
    csm = -csp;
  } else {
    sincos_2pi(fm, &snm, &csm);
  }
  snp *= TwoPi<T>::inv;
  snm *= TwoPi<T>::inv;
  if (snp_out) *snp_out = snp;
  am.base = static_cast<int>(fbm);
  am.w0 = T(1) - fm + snm;
  am.w1 = fm - snm;
  am.g0 = (csm - T(1)) * inv_dx;
  am.xi0 = (T(am.base) + T(-0.25)) * dx - x;
  ap.base = static_cast<int>(fbp);
  ap.w0 = T(1) - fp + snp;
  ap.w1 = fp - snp;
  ap.g0 = (csp - T(1)) * inv_dx;
  ap.xi0 = (T(ap.base) + T(0.25)) * dx - x;
}

template <typename T>
__device__ __forceinline__ Dual<T> dual_stencil(T x, T y, T z, T dx, T inv_dx, int pow2) {
  Dual<T> d;
  axis_pair_dual(x, dx, inv_dx, pow2, d.ax[0][0], d.ax[1][0]);
  axis_pair_dual(y, dx, inv_dx, pow2, d.ax[0][1], d.ax[1][1]);
  axis_pair_dual(z, dx, inv_dx, pow2, d.ax[0][2], d.ax[1][2]);
  return d;
}

// dual_stencil that also hands out the +1 grid's scaled sines, so a caller
// can rebuild that grid's axes later with axis_plus_carried (bit-identical to
// ax[1]) without a second sincos.
template <typename T>
__device__ __forceinline__ Dual<T> dual_stencil_sn(T x, T y, T z, T dx, T inv_dx, int pow2, T (&snp)[3]) {
  Dual<T> d;
  axis_pair_dual(x, dx, inv_dx, pow2, d.ax[0][0], d.ax[1][0], &snp[0]);
  axis_pair_dual(y, dx, inv_dx, pow2, d.ax[0][1], d.ax[1][1], &snp[1]);
  axis_pair_dual(z, dx, inv_dx, pow2, d.ax[0][2], d.ax[1][2], &snp[2]);
  return d;
}

// The +1 grid's axis from its carried scaled sine and gradient factor (the
// same operations as axis_pair_dual's ap: bit-identical).
template <typename T>
__device__ __forceinline__ Axis<T> axis_plus_carried(T x, T dx, T inv_dx, int pow2, T snp, T g0p) {
  const T sp = sub_rn(over_dx(x, dx, inv_dx, pow2), T(0.25));
  const T fbp = dfloor(sp);
  const T fp = sp - fbp;
  Axis<T> a;
  a.base = static_cast<int>(fbp);
  a.w0 = T(1) - fp + snp;
  a.w1 = fp - snp;
  a.g0 = g0p;
  a.xi0 = (T(a.base) + T(0.25)) * dx - x;
  return a;
}

// Quadratic B-spline baseline (kernel.hpp:208-241): 3 nodes per axis on the
// unstaggered grid (grid slot 0, nodes at i*dx).  s = x/dx - 1/2 in the
// division form the reference uses (exact multiply when dx is a power of two).
template <typename T>
struct QAxis {
  int base;
  T w[3], g[3];
  T xi0;  // base*dx - x (node offsets xi_s = xi0 + s*dx)
};

template <typename T>
__device__ __forceinline__ QAxis<T> quad_axis(T x, T dx, T inv_dx, int pow2) {
  QAxis<T> a;
  const T xd = over_dx(x, dx, inv_dx, pow2);
  const T fb = dfloor(sub_rn(xd, T(0.5)));
  a.base = static_cast<int>(fb);
  const T f = sub_rn(xd, T(a.base));  // [0.5, 1.5)
  const T t0 = sub_rn(T(1.5), f), t1 = sub_rn(f, T(1)), t2 = sub_rn(f, T(0.5));
  a.w[0] = mul_rn(mul_rn(T(0.5), t0), t0);
  a.w[1] = sub_rn(T(0.75), mul_rn(t1, t1));
  a.w[2] = mul_rn(mul_rn(T(0.5), t2), t2);
  a.g[0] = div_rn(-t0, dx);
  a.g[1] = div_rn(mul_rn(T(-2), t1), dx);
  a.g[2] = div_rn(t2, dx);
  a.xi0 = sub_rn(mul_rn(T(a.base), dx), x);
  return a;
}

// compute_apic_D over the 27-node quadratic stencil (transfer.hpp:101-116),
// separable: D_aa = M2_a S_b S_c, D_ab = M1_a M1_b S_c.
template <typename T>
__device__ __forceinline__ M3<T> apic_D_quad(const QAxis<T> (&q)[3], T dx) {
  T S[3], M1[3], M2[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    S[a] = M1[a] = M2[a] = T(0);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const T xi = q[a].xi0 + T(k) * dx;
      S[a] += q[a].w[k];
      M1[a] += q[a].w[k] * xi;
      M2[a] += q[a].w[k] * xi * xi;
    }
  }
  M3<T> D;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int c3 = 3 - a - b;
      D.a[a][b] = a == b ? M2[a] * S[(a + 1) % 3] * S[(a + 2) % 3] : M1[a] * M1[b] * S[c3];
    }
  return D;
}

// compute_apic_D (transfer.hpp:77-100) in separable form: with per-axis
// moments S = w0 + w1, M1 = w0 xi0 + w1 xi1, M2 = w0 xi0^2 + w1 xi1^2 the
// 16-node sum factorises exactly (D_aa = 1/2 sum_g M2_a S_b S_c, D_ab =
// 1/2 sum_g M1_a M1_b S_c); only the summation order differs from the
// reference's node loop.
template <typename T>
struct AxisMoments {
  T S, M1, M2;
};

template <typename T>
__device__ __forceinline__ AxisMoments<T> axis_moments(const Axis<T>& a, T dx) {
  const T x1 = a.xi0 + dx;
  return {a.w0 + a.w1, a.w0 * a.xi0 + a.w1 * x1, a.w0 * a.xi0 * a.xi0 + a.w1 * x1 * x1};
}

template <typename T>
__device__ __forceinline__ M3<T> apic_D(const Dual<T>& ds, T dx) {
  M3<T> D;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) D.a[i][j] = T(0);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const AxisMoments<T> m0 = axis_moments(ds.ax[g][0], dx), m1 = axis_moments(ds.ax[g][1], dx),
                         m2 = axis_moments(ds.ax[g][2], dx);
    D.a[0][0] += T(0.5) * m0.M2 * m1.S * m2.S;
    D.a[1][1] += T(0.5) * m1.M2 * m0.S * m2.S;
    D.a[2][2] += T(0.5) * m2.M2 * m0.S * m1.S;
    D.a[0][1] += T(0.5) * m0.M1 * m1.M1 * m2.S;
    D.a[0][2] += T(0.5) * m0.M1 * m2.M1 * m1.S;
    D.a[1][2] += T(0.5) * m1.M1 * m2.M1 * m0.S;
  }
  D.a[1][0] = D.a[0][1];
  D.a[2][0] = D.a[0][2];
  D.a[2][1] = D.a[1][2];
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

// mls_moment (transfer.hpp:127-150), separable form (see apic_D):
// M00 = 1/2 sum S S S, M0a = 1/2 sum M1_a S S, lower-right block = D.
template <typename T>
__device__ __forceinline__ void mls_moment(const Dual<T>& ds, T dx, T (&Mm)[4][4]) {
  const M3<T> D = apic_D(ds, dx);
  T m00 = T(0), m01 = T(0), m02 = T(0), m03 = T(0);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const AxisMoments<T> a = axis_moments(ds.ax[g][0], dx), b = axis_moments(ds.ax[g][1], dx),
                         c = axis_moments(ds.ax[g][2], dx);
    m00 += T(0.5) * a.S * b.S * c.S;
    m01 += T(0.5) * a.M1 * b.S * c.S;
    m02 += T(0.5) * b.M1 * a.S * c.S;
    m03 += T(0.5) * c.M1 * a.S * b.S;
  }
  Mm[0][0] = m00;
  Mm[0][1] = Mm[1][0] = m01;
  Mm[0][2] = Mm[2][0] = m02;
  Mm[0][3] = Mm[3][0] = m03;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Mm[1 + i][1 + j] = D.a[i][j];
}

template <typename T>
__device__ __forceinline__ M3<T> load_m3(const PState<T>& p, int k, uint64_t i) {
  M3<T> m;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) m.a[r][c] = __ldg(p.f + uint64_t(k + 3 * r + c) * p.stride + i);
  return m;
}

template <typename T>
__device__ __forceinline__ void store_m3(const PState<T>& p, int k, uint64_t i, const M3<T>& m) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) p.f[uint64_t(k + 3 * r + c) * p.stride + i] = m.a[r][c];
}


}  // namespace ckg
