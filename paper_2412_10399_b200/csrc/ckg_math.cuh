// ckg_math.cuh — register-resident 3x3 / 4x4 linear algebra for the CK-MPM
// transfer kernels (sm_100a).  Each routine restates the reference algorithm
// in proj/include/ckmpm/math.hpp (cited per function) so that results agree
// with the CPU engine to round-off; FMA contraction is allowed here (state
// parity is tolerance-based) — only the binning arithmetic in
// ckg_bin.cuh is pinned bit-exact with _rn intrinsics.
#pragma once

#include <cfloat>
#include <cstdint>

namespace ckg {

template <typename T>
struct V3 {
  T x, y, z;
  __device__ __forceinline__ T operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};

// Row-major 3x3 (math.hpp:62-115).
template <typename T>
struct M3 {
  T a[3][3];
};

template <typename T>
struct Lim;
template <>
struct Lim<double> {
  static constexpr double eps = DBL_EPSILON;
  static constexpr double tiny = DBL_MIN;
  static constexpr double ns_done = 1e-17;  // ||X^T X - I||^2 after which one more Newton-Schulz step is exact
};
template <>
struct Lim<float> {
  static constexpr float eps = FLT_EPSILON;
  static constexpr float tiny = FLT_MIN;
  static constexpr float ns_done = 1e-8f;
};

__device__ __forceinline__ double dsqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float dsqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double dabs(double x) { return fabs(x); }
__device__ __forceinline__ float dabs(float x) { return fabsf(x); }
__device__ __forceinline__ double dlog(double x) { return log(x); }
__device__ __forceinline__ float dlog(float x) { return logf(x); }
__device__ __forceinline__ double dexp(double x) { return exp(x); }
__device__ __forceinline__ float dexp(float x) { return expf(x); }
__device__ __forceinline__ double dpow(double x, double y) { return pow(x, y); }
__device__ __forceinline__ float dpow(float x, float y) { return powf(x, y); }
__device__ __forceinline__ double dfloor(double x) { return floor(x); }
__device__ __forceinline__ float dfloor(float x) { return floorf(x); }
__device__ __forceinline__ void dsincos(double x, double* s, double* c) { sincos(x, s, c); }
__device__ __forceinline__ void dsincos(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ bool dfinite(double x) { return isfinite(x); }
__device__ __forceinline__ bool dfinite(float x) { return isfinite(x); }

template <typename T>
__device__ __forceinline__ M3<T> m3_identity() {
  M3<T> m;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) m.a[i][j] = i == j ? T(1) : T(0);
  return m;
}

template <typename T>
__device__ __forceinline__ M3<T> mul(const M3<T>& x, const M3<T>& y) {
  M3<T> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r.a[i][j] = x.a[i][0] * y.a[0][j] + x.a[i][1] * y.a[1][j] + x.a[i][2] * y.a[2][j];
  return r;
}

// x * y^T without materialising the transpose.
template <typename T>
__device__ __forceinline__ M3<T> mul_bt(const M3<T>& x, const M3<T>& y) {
  M3<T> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r.a[i][j] = x.a[i][0] * y.a[j][0] + x.a[i][1] * y.a[j][1] + x.a[i][2] * y.a[j][2];
  return r;
}

template <typename T>
__device__ __forceinline__ V3<T> mul(const M3<T>& m, const V3<T>& v) {
  return {m.a[0][0] * v.x + m.a[0][1] * v.y + m.a[0][2] * v.z,
          m.a[1][0] * v.x + m.a[1][1] * v.y + m.a[1][2] * v.z,
          m.a[2][0] * v.x + m.a[2][1] * v.y + m.a[2][2] * v.z};
}

template <typename T>
__device__ __forceinline__ M3<T> transpose(const M3<T>& m) {
  M3<T> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.a[i][j] = m.a[j][i];
  return r;
}

template <typename T>
__device__ __forceinline__ M3<T> scale(T s, const M3<T>& m) {
  M3<T> r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.a[i][j] = m.a[i][j] * s;
  return r;
}

template <typename T>
__device__ __forceinline__ T det(const M3<T>& m) {  // math.hpp:128-132
  return m.a[0][0] * (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]) -
         m.a[0][1] * (m.a[1][0] * m.a[2][2] - m.a[1][2] * m.a[2][0]) +
         m.a[0][2] * (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]);
}

template <typename T>
__device__ __forceinline__ T frob2(const M3<T>& m) {
  T s = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) s += m.a[i][j] * m.a[i][j];
  return s;
}

template <typename T>
__device__ __forceinline__ T trace(const M3<T>& m) {
  return m.a[0][0] + m.a[1][1] + m.a[2][2];
}

template <typename T>
__device__ __forceinline__ T dot(const V3<T>& a, const V3<T>& b) {
  return a.x * b.x + a.y * b.y + a.z * b.z;
}

template <typename T>
__device__ __forceinline__ V3<T> cross(const V3<T>& a, const V3<T>& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// Adjugate (math.hpp:154-167); inverse = adj * (1/det).
template <typename T>
__device__ __forceinline__ M3<T> adjugate(const M3<T>& m) {
  M3<T> r;
  r.a[0][0] = m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1];
  r.a[0][1] = m.a[0][2] * m.a[2][1] - m.a[0][1] * m.a[2][2];
  r.a[0][2] = m.a[0][1] * m.a[1][2] - m.a[0][2] * m.a[1][1];
  r.a[1][0] = m.a[1][2] * m.a[2][0] - m.a[1][0] * m.a[2][2];
  r.a[1][1] = m.a[0][0] * m.a[2][2] - m.a[0][2] * m.a[2][0];
  r.a[1][2] = m.a[0][2] * m.a[1][0] - m.a[0][0] * m.a[1][2];
  r.a[2][0] = m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0];
  r.a[2][1] = m.a[0][1] * m.a[2][0] - m.a[0][0] * m.a[2][1];
  r.a[2][2] = m.a[0][0] * m.a[1][1] - m.a[0][1] * m.a[1][0];
  return r;
}

template <typename T>
__device__ __forceinline__ M3<T> inverse(const M3<T>& m) {
  return scale(T(1) / det(m), adjugate(m));
}

// One cyclic-Jacobi rotation on the (p,q) pair (math.hpp:202-230).
template <int p, int q, typename T>
__device__ __forceinline__ void jacobi_rotate(M3<T>& A, M3<T>& V) {
  if (A.a[p][q] == T(0)) return;
  constexpr int r = 3 - p - q;
  T theta = (A.a[q][q] - A.a[p][p]) / (T(2) * A.a[p][q]);
  T t = (theta >= T(0) ? T(1) : T(-1)) / (dabs(theta) + dsqrt(theta * theta + T(1)));
  T c = T(1) / dsqrt(t * t + T(1));
  T s = t * c;
  T app = A.a[p][p], aqq = A.a[q][q], apq = A.a[p][q];
  A.a[p][p] = c * c * app - T(2) * s * c * apq + s * s * aqq;
  A.a[q][q] = s * s * app + T(2) * s * c * apq + c * c * aqq;
  A.a[p][q] = A.a[q][p] = T(0);
  T arp = A.a[r][p], arq = A.a[r][q];
  A.a[r][p] = A.a[p][r] = c * arp - s * arq;
  A.a[r][q] = A.a[q][r] = s * arp + c * arq;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    T vip = V.a[i][p], viq = V.a[i][q];
    V.a[i][p] = c * vip - s * viq;
    V.a[i][q] = s * vip + c * viq;
  }
}

// sym_eigen3 (math.hpp:193-238): eigenvalues descending (ties keep index
// order, like libstdc++'s insertion sort for n=3), columns of V, det V = +1.
template <typename T>
__device__ __forceinline__ void sym_eigen3(M3<T> A, V3<T>& w_out, M3<T>& V_out) {
  M3<T> V = m3_identity<T>();
  for (int sweep = 0; sweep < 30; ++sweep) {
    T off = dabs(A.a[0][1]) + dabs(A.a[0][2]) + dabs(A.a[1][2]);
    T dg = dabs(A.a[0][0]) + dabs(A.a[1][1]) + dabs(A.a[2][2]);
    if (off <= Lim<T>::eps * (dg + Lim<T>::tiny)) break;
    jacobi_rotate<0, 1>(A, V);
    jacobi_rotate<0, 2>(A, V);
    jacobi_rotate<1, 2>(A, V);
  }
  T w0 = A.a[0][0], w1 = A.a[1][1], w2 = A.a[2][2];
  // Stable descending order of three values via a sorting network that
  // matches insertion sort's tie behaviour.
  int i0 = 0, i1 = 1, i2 = 2;
  T a0 = w0, a1 = w1, a2 = w2;
  if (a1 > a0) { T t = a0; a0 = a1; a1 = t; int ti = i0; i0 = i1; i1 = ti; }
  if (a2 > a1) {
    T t = a1; a1 = a2; a2 = t; int ti = i1; i1 = i2; i2 = ti;
    if (a1 > a0) { T t2 = a0; a0 = a1; a1 = t2; int tj = i0; i0 = i1; i1 = tj; }
  }
  w_out = {a0, a1, a2};
  M3<T> Vs;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    T c0 = V.a[r][0], c1 = V.a[r][1], c2 = V.a[r][2];
    Vs.a[r][0] = i0 == 0 ? c0 : (i0 == 1 ? c1 : c2);
    Vs.a[r][1] = i1 == 0 ? c0 : (i1 == 1 ? c1 : c2);
    Vs.a[r][2] = i2 == 0 ? c0 : (i2 == 1 ? c1 : c2);
  }
  if (det(Vs) < T(0)) {
#pragma unroll
    for (int r = 0; r < 3; ++r) Vs.a[r][2] = -Vs.a[r][2];
  }
  V_out = Vs;
}

// svd3 (math.hpp:249-292): F = U diag(sigma) V^T, det U = det V = +1.
// Kept out of line: it is called from several cold-or-warm sites (polar
// fallback, Drucker-Prager stress and return map, singular-value clamp) and
// inlining each copy would blow the instruction cache of the hot kernels.
template <typename T>
__device__ __noinline__ void svd3(const M3<T>& F, M3<T>& U, V3<T>& sigma, M3<T>& V) {
  M3<T> FtF;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      FtF.a[i][j] = F.a[0][i] * F.a[0][j] + F.a[1][i] * F.a[1][j] + F.a[2][i] * F.a[2][j];
  V3<T> w;
  sym_eigen3(FtF, w, V);
  V3<T> b[3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
    b[c] = {F.a[0][0] * V.a[0][c] + F.a[0][1] * V.a[1][c] + F.a[0][2] * V.a[2][c],
            F.a[1][0] * V.a[0][c] + F.a[1][1] * V.a[1][c] + F.a[1][2] * V.a[2][c],
            F.a[2][0] * V.a[0][c] + F.a[2][1] * V.a[1][c] + F.a[2][2] * V.a[2][c]};
  T sc = dsqrt(w.x < T(0) ? T(0) : w.x);
  T tiny = sc * T(1e-12) + Lim<T>::tiny;
  V3<T> u0 = b[0];
  T n0 = dsqrt(dot(u0, u0));
  if (n0 > tiny) {
    T s = T(1) / n0;
    u0 = {u0.x * s, u0.y * s, u0.z * s};
  } else {
    u0 = {T(1), T(0), T(0)};
  }
  T d = dot(b[1], u0);
  V3<T> u1 = {b[1].x - u0.x * d, b[1].y - u0.y * d, b[1].z - u0.z * d};
  T n1 = dsqrt(dot(u1, u1));
  if (n1 > tiny) {
    T s = T(1) / n1;
    u1 = {u1.x * s, u1.y * s, u1.z * s};
  } else {
    V3<T> seed = dabs(u0.x) < T(0.9) ? V3<T>{T(1), T(0), T(0)} : V3<T>{T(0), T(1), T(0)};
    u1 = cross(u0, seed);
    T s = T(1) / dsqrt(dot(u1, u1));
    u1 = {u1.x * s, u1.y * s, u1.z * s};
  }
  V3<T> u2 = cross(u0, u1);
  U.a[0][0] = u0.x; U.a[1][0] = u0.y; U.a[2][0] = u0.z;
  U.a[0][1] = u1.x; U.a[1][1] = u1.y; U.a[2][1] = u1.z;
  U.a[0][2] = u2.x; U.a[1][2] = u2.y; U.a[2][2] = u2.z;
  sigma = {dot(u0, b[0]), dot(u1, b[1]), dot(u2, b[2])};
}

// One Jacobi rotation on the (p,q) pair without the division by a_pq of
// jacobi_rotate: with d = a_qq - a_pp, t = tan of the rotation angle is
//   t = sgn(theta) 2|a_pq| / (|d| + sqrt(d^2 + 4 a_pq^2)),  theta = d / (2 a_pq)
// (the same root as math.hpp:211-213 multiplied through by |2 a_pq|, so a
// zero a_pq gives t = 0, the identity rotation, with no branch).
template <int p, int q, typename T>
__device__ __forceinline__ void jacobi_rotate_nb(M3<T>& A, M3<T>& V) {
  constexpr int r = 3 - p - q;
  const T app = A.a[p][p], aqq = A.a[q][q], apq = A.a[p][q];
  const T d = aqq - app, a2 = T(2) * dabs(apq);
  const T den = dabs(d) + dsqrt(d * d + a2 * a2);
  T t = den > T(0) ? a2 / den : T(0);
  if (d * apq < T(0)) t = -t;  // sgn(theta); theta = +-0 counts as positive (math.hpp:212)
  const T c = T(1) / dsqrt(t * t + T(1));
  const T sn = t * c;
  A.a[p][p] = c * c * app - T(2) * sn * c * apq + sn * sn * aqq;
  A.a[q][q] = sn * sn * app + T(2) * sn * c * apq + c * c * aqq;
  A.a[p][q] = A.a[q][p] = T(0);
  const T arp = A.a[r][p], arq = A.a[r][q];
  A.a[r][p] = A.a[p][r] = c * arp - sn * arq;
  A.a[r][q] = A.a[q][r] = sn * arp + c * arq;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const T vip = V.a[i][p], viq = V.a[i][q];
    V.a[i][p] = c * vip - sn * viq;
    V.a[i][q] = sn * vip + c * viq;
  }
}

// svd3 (math.hpp:249-292) for the hot path (Drucker-Prager return map in
// G2P): inlined and register-resident (no call, no by-reference outputs in
// local memory), the reference's cyclic Jacobi of F^T F with its stopping
// test before every sweep (a settled sand grain's F^T F is diagonal to
// round-off and exits at once; measured: four unconditional sweeps cost the
// 10M DP block's G2P 1.79 -> 2.68 ms) and branch-free rotations.  U, sigma
// follow svd3.
template <typename T>
__device__ __forceinline__ void svd3_inl(const M3<T>& F, M3<T>& U, V3<T>& sigma, M3<T>& V_out) {
  M3<T> A;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      A.a[i][j] = F.a[0][i] * F.a[0][j] + F.a[1][i] * F.a[1][j] + F.a[2][i] * F.a[2][j];
  M3<T> V = m3_identity<T>();
#pragma unroll 1
  for (int sweep = 0; sweep < 30; ++sweep) {
    const T off = dabs(A.a[0][1]) + dabs(A.a[0][2]) + dabs(A.a[1][2]);
    const T dg = dabs(A.a[0][0]) + dabs(A.a[1][1]) + dabs(A.a[2][2]);
    if (off <= Lim<T>::eps * (dg + Lim<T>::tiny)) break;
    jacobi_rotate_nb<0, 1>(A, V);
    jacobi_rotate_nb<0, 2>(A, V);
    jacobi_rotate_nb<1, 2>(A, V);
  }
  // descending eigenvalues (insertion-sort tie behaviour), det V = +1
  int i0 = 0, i1 = 1, i2 = 2;
  T a0 = A.a[0][0], a1 = A.a[1][1], a2 = A.a[2][2];
  if (a1 > a0) { T t = a0; a0 = a1; a1 = t; int ti = i0; i0 = i1; i1 = ti; }
  if (a2 > a1) {
    T t = a1; a1 = a2; a2 = t; int ti = i1; i1 = i2; i2 = ti;
    if (a1 > a0) { T t2 = a0; a0 = a1; a1 = t2; int tj = i0; i0 = i1; i1 = tj; }
  }
  M3<T> Vs;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const T c0 = V.a[r][0], c1 = V.a[r][1], c2 = V.a[r][2];
    Vs.a[r][0] = i0 == 0 ? c0 : (i0 == 1 ? c1 : c2);
    Vs.a[r][1] = i1 == 0 ? c0 : (i1 == 1 ? c1 : c2);
    Vs.a[r][2] = i2 == 0 ? c0 : (i2 == 1 ? c1 : c2);
  }
  if (det(Vs) < T(0)) {
#pragma unroll
    for (int r = 0; r < 3; ++r) Vs.a[r][2] = -Vs.a[r][2];
  }
  V_out = Vs;
  V3<T> b[3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
    b[c] = {F.a[0][0] * Vs.a[0][c] + F.a[0][1] * Vs.a[1][c] + F.a[0][2] * Vs.a[2][c],
            F.a[1][0] * Vs.a[0][c] + F.a[1][1] * Vs.a[1][c] + F.a[1][2] * Vs.a[2][c],
            F.a[2][0] * Vs.a[0][c] + F.a[2][1] * Vs.a[1][c] + F.a[2][2] * Vs.a[2][c]};
  const T sc = dsqrt(a0 < T(0) ? T(0) : a0);
  const T tiny = sc * T(1e-12) + Lim<T>::tiny;
  V3<T> u0 = b[0];
  const T n0 = dsqrt(dot(u0, u0));
  if (n0 > tiny) {
    const T s = T(1) / n0;
    u0 = {u0.x * s, u0.y * s, u0.z * s};
  } else {
    u0 = {T(1), T(0), T(0)};
  }
  const T d = dot(b[1], u0);
  V3<T> u1 = {b[1].x - u0.x * d, b[1].y - u0.y * d, b[1].z - u0.z * d};
  const T n1 = dsqrt(dot(u1, u1));
  if (n1 > tiny) {
    const T s = T(1) / n1;
    u1 = {u1.x * s, u1.y * s, u1.z * s};
  } else {
    const V3<T> seed = dabs(u0.x) < T(0.9) ? V3<T>{T(1), T(0), T(0)} : V3<T>{T(0), T(1), T(0)};
    u1 = cross(u0, seed);
    const T s = T(1) / dsqrt(dot(u1, u1));
    u1 = {u1.x * s, u1.y * s, u1.z * s};
  }
  const V3<T> u2 = cross(u0, u1);
  U.a[0][0] = u0.x; U.a[1][0] = u0.y; U.a[2][0] = u0.z;
  U.a[0][1] = u1.x; U.a[1][1] = u1.y; U.a[2][1] = u1.z;
  U.a[0][2] = u2.x; U.a[1][2] = u2.y; U.a[2][2] = u2.z;
  sigma = {dot(u0, b[0]), dot(u1, b[1]), dot(u2, b[2])};
}

// polar_rotation (math.hpp:300-321): scaled Newton R <- (gR + (gR)^-T)/2 with
// the reference's stopping rule; SVD construction for near-singular input.
template <typename T>
__device__ __noinline__ M3<T> polar_rotation(const M3<T>& F) {  // cold fallback: out of line
  T nf = dsqrt(frob2(F));
  T d = det(F);
  if (!(d > T(1e-10) * nf * nf * nf)) {
    M3<T> U, V;
    V3<T> s;
    svd3(F, U, s, V);
    return mul_bt(U, V);
  }
  const T tol = T(8) * Lim<T>::eps;
  M3<T> R = F;
  T prev = T(INFINITY);
  for (int it = 0; it < 40; ++it) {
    // (R^-1)^T = adj(R)^T / det(R)
    M3<T> adj = adjugate(R);
    T inv_det = T(1) / det(R);
    M3<T> Rit;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Rit.a[i][j] = adj.a[j][i] * inv_det;
    T g = dsqrt(dsqrt(frob2(Rit)) / dsqrt(frob2(R)));
    T ha = T(0.5) * g, hb = T(0.5) / g;
    M3<T> Rn;
    T diff2 = 0, rn2 = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        Rn.a[i][j] = ha * R.a[i][j] + hb * Rit.a[i][j];
        T dd = Rn.a[i][j] - R.a[i][j];
        diff2 += dd * dd;
        rn2 += Rn.a[i][j] * Rn.a[i][j];
      }
    T diff = dsqrt(diff2);
    R = Rn;
    if (diff <= tol * dsqrt(rn2) || diff >= prev) break;
    prev = diff;
  }
  return R;
}

// Same rotation factor as polar_rotation, cheaper near rotations: the
// Newton-Schulz iteration X <- X (3I - X^T X)/2 needs no inverse, square root
// or division and converges quadratically to the orthogonal polar factor while
// ||X^T X - I|| < 1 (every elastic state F = R(I + small strain)).  The final
// factor agrees with the reference's scaled Newton result to round-off; far
// from a rotation (or on non-convergence) the reference algorithm runs.
template <typename T>
__device__ __forceinline__ M3<T> polar_rotation_fast(const M3<T>& F) {
  M3<T> X = F;
  for (int it = 0; it < 8; ++it) {
    // E = X^T X - I (symmetric)
    M3<T> E;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i; j < 3; ++j) {
        T v = X.a[0][i] * X.a[0][j] + X.a[1][i] * X.a[1][j] + X.a[2][i] * X.a[2][j];
        if (i == j) v -= T(1);
        E.a[i][j] = v;
        E.a[j][i] = v;
      }
    const T e2 = frob2(E);
    if (!(e2 < T(0.25))) break;  // outside the comfortable convergence region
    // X <- X (I - E/2)
    M3<T> Y;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        Y.a[i][j] = X.a[i][j] - T(0.5) * (X.a[i][0] * E.a[0][j] + X.a[i][1] * E.a[1][j] + X.a[i][2] * E.a[2][j]);
    X = Y;
    // ||E|| ~ 1e-8 -> the step just taken leaves ~1.5e-16: converged.
    if (e2 < Lim<T>::ns_done) return X;
  }
  return polar_rotation(F);
}

// gauss_inverse4 with partial pivoting (math.hpp:360-385).  Returns false on
// a vanishing pivot.  Row swaps are done with predicated selects so the
// working set stays in registers.
template <typename T>
__device__ __forceinline__ bool gauss_inverse4(const T (&in)[4][4], T (&out)[4][4]) {
  T w[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) w[i][j] = j < 4 ? in[i][j] : (j - 4 == i ? T(1) : T(0));
#pragma unroll
  for (int col = 0; col < 4; ++col) {
    int piv = col;
    T best = dabs(w[col][col]);
#pragma unroll
    for (int r = col + 1; r < 4; ++r) {
      T v = dabs(w[r][col]);
      if (v > best) { best = v; piv = r; }
    }
    // Swap rows piv and col (selects over the static rows >= col).
#pragma unroll
    for (int r = col + 1; r < 4; ++r) {
      if (piv == r) {
#pragma unroll
        for (int j = 0; j < 8; ++j) { T t = w[r][j]; w[r][j] = w[col][j]; w[col][j] = t; }
      }
    }
    if (w[col][col] == T(0)) return false;
    T inv_p = T(1) / w[col][col];
#pragma unroll
    for (int j = 0; j < 8; ++j) w[col][j] *= inv_p;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (r == col) continue;
      T f = w[r][col];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[r][j] -= f * w[col][j];
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) out[i][j] = w[i][4 + j];
  return true;
}

}  // namespace ckg
