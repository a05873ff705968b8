/*
 * ckmpm_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference CK-MPM substep (Simulation<double>::step, deterministic mode).
 * See ckmpm_oracle.h.  Reference paths below are relative to
 * /root/reference/proj/include/ckmpm/.  Parity pinned bit-exact against the
 * compiled reference (oracle/_ref) by tests/test_oracle_pin.py.
 *
 * Conventions: Mat3 is row-major double[9]; expression trees follow the
 * reference's C++ operator evaluation order exactly (left-to-right sums,
 * scalar*matrix as element-wise multiply, Vec3/s as multiply by 1/s).
 */
#include "ckmpm_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define M(m, i, j) ((m)[3 * (i) + (j)])

static const double kPi = 3.141592653589793238462643383279502884;

/* ------------------------------------------------------------------ math */

/* Vec3 dot (math.hpp:43-45) */
static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static double norm3(const double* a) { return sqrt(dot3(a, a)); }
/* cross (math.hpp:48-50) */
static void cross3(const double* a, const double* b, double* r) {
  double x = a[1] * b[2] - a[2] * b[1], y = a[2] * b[0] - a[0] * b[2], z = a[0] * b[1] - a[1] * b[0];
  r[0] = x; r[1] = y; r[2] = z;
}
/* Mat3 * Mat3 (math.hpp:103-109) */
static void matmul(const double* x, const double* y, double* out) {
  double r[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r[3 * i + j] = M(x, i, 0) * M(y, 0, j) + M(x, i, 1) * M(y, 1, j) + M(x, i, 2) * M(y, 2, j);
  memcpy(out, r, sizeof r);
}
/* Mat3 * Vec3 (math.hpp:110-114) */
static void matvec(const double* m, const double* v, double* out) {
  double r0 = M(m, 0, 0) * v[0] + M(m, 0, 1) * v[1] + M(m, 0, 2) * v[2];
  double r1 = M(m, 1, 0) * v[0] + M(m, 1, 1) * v[1] + M(m, 1, 2) * v[2];
  double r2 = M(m, 2, 0) * v[0] + M(m, 2, 1) * v[1] + M(m, 2, 2) * v[2];
  out[0] = r0; out[1] = r1; out[2] = r2;
}
static void transpose3(const double* m, double* r) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[3 * i + j] = M(m, j, i);
  memcpy(r, t, sizeof t);
}
static void scale3(double s, const double* m, double* r) { for (int i = 0; i < 9; ++i) r[i] = m[i] * s; }
static void identity3(double* m) { memset(m, 0, 9 * sizeof(double)); m[0] = m[4] = m[8] = 1.0; }
static void diag3(double a, double b, double c, double* m) { memset(m, 0, 9 * sizeof(double)); m[0] = a; m[4] = b; m[8] = c; }
/* det (math.hpp:128-132) */
static double det3(const double* m) {
  return M(m, 0, 0) * (M(m, 1, 1) * M(m, 2, 2) - M(m, 1, 2) * M(m, 2, 1)) -
         M(m, 0, 1) * (M(m, 1, 0) * M(m, 2, 2) - M(m, 1, 2) * M(m, 2, 0)) +
         M(m, 0, 2) * (M(m, 1, 0) * M(m, 2, 1) - M(m, 1, 1) * M(m, 2, 0));
}
/* frobenius_norm (math.hpp:142-147) */
static double frob3(const double* m) {
  double s = 0;
  for (int i = 0; i < 9; ++i) s += m[i] * m[i];
  return sqrt(s);
}
/* inverse: adjugate * (1/det) (math.hpp:154-167) */
static void inverse3(const double* m, double* r) {
  double adj[9];
  adj[0] = M(m, 1, 1) * M(m, 2, 2) - M(m, 1, 2) * M(m, 2, 1);
  adj[1] = M(m, 0, 2) * M(m, 2, 1) - M(m, 0, 1) * M(m, 2, 2);
  adj[2] = M(m, 0, 1) * M(m, 1, 2) - M(m, 0, 2) * M(m, 1, 1);
  adj[3] = M(m, 1, 2) * M(m, 2, 0) - M(m, 1, 0) * M(m, 2, 2);
  adj[4] = M(m, 0, 0) * M(m, 2, 2) - M(m, 0, 2) * M(m, 2, 0);
  adj[5] = M(m, 0, 2) * M(m, 1, 0) - M(m, 0, 0) * M(m, 1, 2);
  adj[6] = M(m, 1, 0) * M(m, 2, 1) - M(m, 1, 1) * M(m, 2, 0);
  adj[7] = M(m, 0, 1) * M(m, 2, 0) - M(m, 0, 0) * M(m, 2, 1);
  adj[8] = M(m, 0, 0) * M(m, 1, 1) - M(m, 0, 1) * M(m, 1, 0);
  double s = 1.0 / det3(m);
  for (int i = 0; i < 9; ++i) r[i] = adj[i] * s;
}

/* sym_eigen3: cyclic Jacobi, <=30 sweeps, descending, det V = +1
 * (math.hpp:193-238). */
static void sym_eigen3(const double* Ain, double* w_out, double* V_out) {
  double A[9], V[9];
  memcpy(A, Ain, sizeof A);
  identity3(V);
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = fabs(M(A, 0, 1)) + fabs(M(A, 0, 2)) + fabs(M(A, 1, 2));
    double diag = fabs(M(A, 0, 0)) + fabs(M(A, 1, 1)) + fabs(M(A, 2, 2));
    if (off <= DBL_EPSILON * (diag + DBL_MIN)) break;
    for (int p = 0; p < 2; ++p) {
      for (int q = p + 1; q < 3; ++q) {
        if (M(A, p, q) == 0.0) continue;
        double theta = (M(A, q, q) - M(A, p, p)) / (2.0 * M(A, p, q));
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0);
        double s = t * c;
        double app = M(A, p, p), aqq = M(A, q, q), apq = M(A, p, q);
        M(A, p, p) = c * c * app - 2.0 * s * c * apq + s * s * aqq;
        M(A, q, q) = s * s * app + 2.0 * s * c * apq + c * c * aqq;
        M(A, p, q) = M(A, q, p) = 0.0;
        int r = 3 - p - q;
        double arp = M(A, r, p), arq = M(A, r, q);
        M(A, r, p) = M(A, p, r) = c * arp - s * arq;
        M(A, r, q) = M(A, q, r) = s * arp + c * arq;
        for (int i = 0; i < 3; ++i) {
          double vip = M(V, i, p), viq = M(V, i, q);
          M(V, i, p) = c * vip - s * viq;
          M(V, i, q) = s * vip + c * viq;
        }
      }
    }
  }
  /* std::sort of 3 indices by w descending: libstdc++ insertion sort for
   * n < 16, which keeps ties in index order. */
  int idx[3] = {0, 1, 2};
  double w[3] = {M(A, 0, 0), M(A, 1, 1), M(A, 2, 2)};
  for (int i = 1; i < 3; ++i) {
    int v = idx[i];
    int j = i;
    while (j > 0 && w[v] > w[idx[j - 1]]) { idx[j] = idx[j - 1]; --j; }
    idx[j] = v;
  }
  double Vs[9];
  for (int c = 0; c < 3; ++c) {
    w_out[c] = w[idx[c]];
    for (int r = 0; r < 3; ++r) M(Vs, r, c) = M(V, r, idx[c]);
  }
  if (det3(Vs) < 0.0)
    for (int r = 0; r < 3; ++r) M(Vs, r, 2) = -M(Vs, r, 2);
  memcpy(V_out, Vs, sizeof Vs);
}

/* svd3 via eig(F^T F) + Gram-Schmidt U (math.hpp:249-292). */
static void svd3(const double* F, double* U, double* sigma, double* Vout) {
  double Ft[9], FtF[9], w[3], V[9];
  transpose3(F, Ft);
  matmul(Ft, F, FtF);
  sym_eigen3(FtF, w, V);
  double b[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r)
      b[c][r] = M(F, r, 0) * M(V, 0, c) + M(F, r, 1) * M(V, 1, c) + M(F, r, 2) * M(V, 2, c);
  double scale = sqrt(w[0] < 0.0 ? 0.0 : w[0]); /* std::max(w0, T(0)) */
  double tiny = scale * 1e-12 + DBL_MIN;
  double u0[3] = {b[0][0], b[0][1], b[0][2]};
  double n0 = norm3(u0);
  if (n0 > tiny) { double s = 1.0 / n0; u0[0] *= s; u0[1] *= s; u0[2] *= s; }
  else { u0[0] = 1.0; u0[1] = 0.0; u0[2] = 0.0; }
  double d = dot3(b[1], u0);
  double u1[3] = {b[1][0] - u0[0] * d, b[1][1] - u0[1] * d, b[1][2] - u0[2] * d};
  double n1 = norm3(u1);
  if (n1 > tiny) { double s = 1.0 / n1; u1[0] *= s; u1[1] *= s; u1[2] *= s; }
  else {
    double seed[3] = {0, 0, 0};
    if (fabs(u0[0]) < 0.9) seed[0] = 1.0; else seed[1] = 1.0;
    cross3(u0, seed, u1);
    double s = 1.0 / norm3(u1);
    u1[0] *= s; u1[1] *= s; u1[2] *= s;
  }
  double u2[3];
  cross3(u0, u1, u2);
  for (int r = 0; r < 3; ++r) { M(U, r, 0) = u0[r]; M(U, r, 1) = u1[r]; M(U, r, 2) = u2[r]; }
  memcpy(Vout, V, sizeof V);
  sigma[0] = dot3(u0, b[0]);
  sigma[1] = dot3(u1, b[1]);
  sigma[2] = dot3(u2, b[2]);
}

/* polar_rotation: scaled Newton, <=40 iterations, SVD fallback
 * (math.hpp:300-321). */
static void polar_rotation(const double* F, double* Rout) {
  double nf = frob3(F);
  double d = det3(F);
  if (!(d > 1e-10 * nf * nf * nf)) {
    double U[9], s[3], V[9], Vt[9];
    svd3(F, U, s, V);
    transpose3(V, Vt);
    matmul(U, Vt, Rout);
    return;
  }
  double tol = 8.0 * DBL_EPSILON;
  double R[9];
  memcpy(R, F, sizeof R);
  double prev_diff = INFINITY;
  for (int it = 0; it < 40; ++it) {
    double Ri[9], Rit[9], Rn[9], a[9], b[9], dm[9];
    inverse3(R, Ri);
    transpose3(Ri, Rit);
    double g = sqrt(frob3(Rit) / frob3(R));
    scale3(0.5 * g, R, a);
    scale3(0.5 / g, Rit, b);
    for (int i = 0; i < 9; ++i) Rn[i] = a[i] + b[i];
    for (int i = 0; i < 9; ++i) dm[i] = Rn[i] - R[i];
    double diff = frob3(dm);
    memcpy(R, Rn, sizeof R);
    if (diff <= tol * frob3(R) || diff >= prev_diff) break;
    prev_diff = diff;
  }
  memcpy(Rout, R, sizeof R);
}

/* gauss_inverse4 with partial pivoting (math.hpp:360-385). */
static int gauss_inverse4(const double* in, double* out) {
  double w[4][8];
  memset(w, 0, sizeof w);
  for (int i = 0; i < 4; ++i) {
    for (int j = 0; j < 4; ++j) w[i][j] = in[4 * i + j];
    w[i][4 + i] = 1.0;
  }
  for (int col = 0; col < 4; ++col) {
    int piv = col;
    for (int r = col + 1; r < 4; ++r)
      if (fabs(w[r][col]) > fabs(w[piv][col])) piv = r;
    if (w[piv][col] == 0.0) return 0;
    if (piv != col) {
      double tmp[8];
      memcpy(tmp, w[piv], sizeof tmp);
      memcpy(w[piv], w[col], sizeof tmp);
      memcpy(w[col], tmp, sizeof tmp);
    }
    double inv_p = 1.0 / w[col][col];
    for (int j = 0; j < 8; ++j) w[col][j] *= inv_p;
    for (int r = 0; r < 4; ++r) {
      if (r == col) continue;
      double f = w[r][col];
      if (f == 0.0) continue;
      for (int j = 0; j < 8; ++j) w[r][j] -= f * w[col][j];
    }
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) out[4 * i + j] = w[i][4 + j];
  return 1;
}

/* ---------------------------------------------------------------- kernel */

static const double kTwoPi = 2.0 * 3.141592653589793238462643383279502884; /* two_pi_v (kernel.hpp:28) */
static double inv_two_pi(void) { return 1.0 / (2.0 * kPi); }             /* inv_two_pi_v (kernel.hpp:30) */

/* ck_weight_1d (kernel.hpp:77-82) */
double ckor_ck_weight_1d(double u) {
  double a = fabs(u);
  if (a >= 1.0) return 0.0;
  return 1.0 - a + sin(kTwoPi * a) * inv_two_pi();
}
/* ck_grad_1d (kernel.hpp:87-92) */
double ckor_ck_grad_1d(double u) {
  double a = fabs(u);
  if (a >= 1.0 || u == 0.0) return 0.0;
  double g = cos(kTwoPi * a) - 1.0;
  return u > 0.0 ? g : -g;
}

typedef struct { int base; double f, w0, w1, g0, g1; } axis_pair_t;

/* axis_pair: paired single-trig slice (kernel.hpp:114-137), hook disabled. */
static axis_pair_t axis_pair(double x, int k, double dx) {
  axis_pair_t p;
  double s = x / dx - (double)k * 0.25;
  double fb = floor(s);
  p.base = (int)fb;
  p.f = s - fb;
  double sn = sin(kTwoPi * p.f) * inv_two_pi();
  double cs = cos(kTwoPi * p.f);
  p.w0 = 1.0 - p.f + sn;
  p.w1 = p.f - sn;
  p.g0 = (cs - 1.0) / dx;
  p.g1 = -p.g0;
  return p;
}

void ckor_axis_pair(double x, int32_t k, double dx, int32_t* base, double* o) {
  axis_pair_t p = axis_pair(x, k, dx);
  *base = p.base;
  o[0] = p.f; o[1] = p.w0; o[2] = p.w1; o[3] = p.g0; o[4] = p.g1;
}

void ckor_polar_rotation(const double* F, double* R) { polar_rotation(F, R); }
void ckor_svd3(const double* F, double* U, double* s, double* V) { svd3(F, U, s, V); }

/* dual_stencil: grid 0 is k=-1, grid 1 is k=+1 (kernel.hpp:188-206) */
typedef struct { axis_pair_t ax[2][3]; } dual_stencil_t;
static int grid_tag(int g) { return g == 0 ? -1 : +1; }
static dual_stencil_t dual_stencil(const double* x, double dx) {
  dual_stencil_t d;
  for (int g = 0; g < 2; ++g)
    for (int a = 0; a < 3; ++a) d.ax[g][a] = axis_pair(x[a], grid_tag(g), dx);
  return d;
}
/* axis_geom: xi0 = (base + k/4) dx - xp (transfer.hpp:65-68) */
static void axis_geom(const axis_pair_t* ap, double xp, int k, double dx, double* xi) {
  xi[0] = ((double)ap->base + (double)k * 0.25) * dx - xp;
  xi[1] = xi[0] + dx;
}

/* ------------------------------------------------------------------ grid */

typedef struct { double mass, p[3]; } node_t;
typedef struct { int coord[3]; node_t nodes[128]; } block_t;

struct ckor_sim {
  ckg_config cfg;
  uint64_t n;
  ckg_particle_f64* ps;
  ckg_particle_f64* scratch;
  dual_stencil_t* ds;
  uint64_t* keys;
  uint64_t* counts;
  int D;
  int32_t* directory;
  block_t* blocks;
  uint64_t nblocks, cap_blocks;
  double vmax;
  double min_j[CKG_MAX_MATERIALS];
  uint64_t step_count;
};

static uint64_t dir_index(const ckor_sim* s, int bx, int by, int bz) {
  return ((uint64_t)bx * s->D + by) * s->D + bz;
}

/* mark_block: first-touch append (grid.hpp:266-272) */
static void mark_block(ckor_sim* s, int bx, int by, int bz) {
  int32_t* slot = &s->directory[dir_index(s, bx, by, bz)];
  if (*slot < 0) {
    if (s->nblocks == s->cap_blocks) {
      s->cap_blocks = s->cap_blocks ? 2 * s->cap_blocks : 1024;
      s->blocks = (block_t*)realloc(s->blocks, s->cap_blocks * sizeof(block_t));
    }
    *slot = (int32_t)s->nblocks;
    block_t* b = &s->blocks[s->nblocks++];
    b->coord[0] = bx; b->coord[1] = by; b->coord[2] = bz;
    memset(b->nodes, 0, sizeof b->nodes);
  }
}

/* node_by_index + node_offset (grid.hpp:164-175) */
static node_t* node_by_index(ckor_sim* s, int g, int i, int j, int k) {
  int32_t slot = s->directory[dir_index(s, i >> 2, j >> 2, k >> 2)];
  if (slot < 0) return NULL;
  return &s->blocks[slot].nodes[(g << 6) | ((i & 3) << 4) | ((j & 3) << 2) | (k & 3)];
}

typedef struct { int code, axis; uint64_t particle; char msg[256]; } err_t;

static int fail(err_t* e, int code, uint64_t particle, int axis, const char* msg) {
  e->code = code; e->particle = particle; e->axis = axis;
  snprintf(e->msg, sizeof e->msg, "%s", msg);
  return code == CKG_NUM_NONE ? 0 : 3;
}

/* activate: inset check + footprint + positive halo (grid.hpp:114-145) */
static int activate(ckor_sim* s, err_t* e) {
  for (uint64_t d = 0; d < (uint64_t)s->D * s->D * s->D; ++d) s->directory[d] = -1;
  s->nblocks = 0;
  const double dx = s->cfg.dx;
  const double inv_dx = 1.0 / dx;
  const int res = s->cfg.resolution;
  for (uint64_t pi = 0; pi < s->n; ++pi) {
    const double* x = s->ps[pi].x;
    int lo_b[3], hi_b[3];
    for (int a = 0; a < 3; ++a) {
      double sa = x[a] * inv_dx;
      if (!(sa >= 2.0 && sa <= (double)(res - 2))) {
        char m[128];
        snprintf(m, sizeof m, "particle %llu violates the 2-cell domain inset on axis %d",
                 (unsigned long long)pi, a);
        return fail(e, CKG_NUM_OUT_OF_DOMAIN, pi, a, m);
      }
      int base_plus = (int)floor(sa - 0.25);
      int base_minus = (int)floor(sa + 0.25);
      lo_b[a] = base_plus >> 2;
      hi_b[a] = ((base_minus + 1) >> 2) + 1;
    }
    for (int bi = lo_b[0]; bi <= hi_b[0]; ++bi)
      for (int bj = lo_b[1]; bj <= hi_b[1]; ++bj)
        for (int bk = lo_b[2]; bk <= hi_b[2]; ++bk) mark_block(s, bi, bj, bk);
  }
  return 0;
}

/* ------------------------------------------------------------- materials */

/* force_matrix: V0 * Kirchhoff stress (transfer.hpp:183-216, material.hpp:132-143) */
static int force_matrix(const ckg_particle_f64* p, const ckg_material* mat, double* A, err_t* e,
                        uint64_t pi) {
  switch (mat->model) {
    case CKG_MODEL_FIXED_COROTATED: {
      double J = det3(p->F);
      if (!(J > 0.0)) return fail(e, CKG_NUM_FC_STRESS_INVERTED, pi, 0, "fixed corotated stress: det F <= 0");
      double R[9], Ft[9], FmR[9], prod[9], t1[9], I[9], t2[9], tau[9];
      polar_rotation(p->F, R);
      transpose3(p->F, Ft);
      for (int i = 0; i < 9; ++i) FmR[i] = p->F[i] - R[i];
      matmul(FmR, Ft, prod);
      scale3(2.0 * mat->mu, prod, t1);
      identity3(I);
      scale3(mat->lambda * J * (J - 1.0), I, t2);
      for (int i = 0; i < 9; ++i) tau[i] = t1[i] + t2[i];
      scale3(p->volume0, tau, A);
      return 0;
    }
    case CKG_MODEL_DRUCKER_PRAGER: {
      double U[9], sg[3], V[9];
      svd3(p->F, U, sg, V);
      if (!(sg[2] > 0.0)) return fail(e, CKG_NUM_DP_STRESS_INVERTED, pi, 0, "granular stress: det F <= 0");
      double eps[3] = {log(sg[0]), log(sg[1]), log(sg[2])};
      double tr = eps[0] + eps[1] + eps[2];
      double td[3];
      for (int a = 0; a < 3; ++a) td[a] = 2.0 * mat->mu * eps[a] + mat->lambda * tr;
      double Dg[9], Ut[9], t[9], tau[9];
      diag3(td[0], td[1], td[2], Dg);
      transpose3(U, Ut);
      matmul(U, Dg, t);
      matmul(t, Ut, tau);
      scale3(p->volume0, tau, A);
      return 0;
    }
    case CKG_MODEL_J_FLUID: {
      /* stress_j_fluid + j_fluid_pressure (material.hpp:132-143) */
      if (!(p->J > 0.0)) return fail(e, CKG_NUM_FLUID_STATE_J, pi, 0, "fluid state: J must be > 0");
      double pr = mat->bulk * (pow(p->J, -mat->gamma) - 1.0);
      double sd = -p->J * pr;
      double Dg[9];
      diag3(sd, sd, sd, Dg);
      scale3(p->volume0, Dg, A);
      return 0;
    }
  }
  return fail(e, CKG_NUM_NONE, pi, 0, "force for reserved material tag");
}

/* compute_apic_D over both grids (transfer.hpp:77-100) */
static void compute_apic_D(const double* xp, const dual_stencil_t* ds, double dx, double* D) {
  memset(D, 0, 9 * sizeof(double));
  for (int g = 0; g < 2; ++g) {
    int k = grid_tag(g);
    const axis_pair_t* ax = ds->ax[g];
    double xix[2], xiy[2], xiz[2];
    axis_geom(&ax[0], xp[0], k, dx, xix);
    axis_geom(&ax[1], xp[1], k, dx, xiy);
    axis_geom(&ax[2], xp[2], k, dx, xiz);
    double wx[2] = {ax[0].w0, ax[0].w1}, wy[2] = {ax[1].w0, ax[1].w1}, wz[2] = {ax[2].w0, ax[2].w1};
    for (int s = 0; s < 2; ++s)
      for (int t = 0; t < 2; ++t)
        for (int u = 0; u < 2; ++u) {
          double w = 0.5 * wx[s] * wy[t] * wz[u];
          double xi[3] = {xix[s], xiy[t], xiz[u]};
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) D[3 * a + b] += w * xi[a] * xi[b];
        }
  }
}

/* apic_d_inverse with the degeneracy guard (transfer.hpp:222-229) */
static int apic_d_inverse(const double* D, double* Di, err_t* e, uint64_t pi) {
  double scale = (D[0] + D[4] + D[8]) / 3.0;
  double d = det3(D);
  if (!(d > scale * scale * scale * 1e-12)) return fail(e, CKG_NUM_NEAR_SINGULAR_D, pi, 0, "near-singular APIC D matrix");
  inverse3(D, Di);
  return 0;
}

/* mls_moment (transfer.hpp:127-150) */
static void mls_moment(const double* xp, const dual_stencil_t* ds, double dx, double* Mm) {
  memset(Mm, 0, 16 * sizeof(double));
  for (int g = 0; g < 2; ++g) {
    int k = grid_tag(g);
    const axis_pair_t* ax = ds->ax[g];
    double xix[2], xiy[2], xiz[2];
    axis_geom(&ax[0], xp[0], k, dx, xix);
    axis_geom(&ax[1], xp[1], k, dx, xiy);
    axis_geom(&ax[2], xp[2], k, dx, xiz);
    double wx[2] = {ax[0].w0, ax[0].w1}, wy[2] = {ax[1].w0, ax[1].w1}, wz[2] = {ax[2].w0, ax[2].w1};
    for (int s = 0; s < 2; ++s)
      for (int t = 0; t < 2; ++t)
        for (int u = 0; u < 2; ++u) {
          double w = 0.5 * wx[s] * wy[t] * wz[u];
          double P[4] = {1.0, xix[s], xiy[t], xiz[u]};
          for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) Mm[4 * a + b] += w * P[a] * P[b];
        }
  }
}

/* detail::scatter_one<false> over the dual stencil (transfer.hpp:235-283) */
static int scatter_one(ckor_sim* s, const ckg_particle_f64* p, const dual_stencil_t* ds,
                       const double* C, const double* A, double dt, err_t* e, uint64_t pi) {
  const double dx = s->cfg.dx;
  for (int g = 0; g < 2; ++g) {
    int k = grid_tag(g);
    const axis_pair_t* ax = ds->ax[g];
    double xix[2], xiy[2], xiz[2];
    axis_geom(&ax[0], p->x[0], k, dx, xix);
    axis_geom(&ax[1], p->x[1], k, dx, xiy);
    axis_geom(&ax[2], p->x[2], k, dx, xiz);
    double wx[2] = {ax[0].w0, ax[0].w1}, wy[2] = {ax[1].w0, ax[1].w1}, wz[2] = {ax[2].w0, ax[2].w1};
    double gx[2] = {ax[0].g0, ax[0].g1}, gy[2] = {ax[1].g0, ax[1].g1}, gz[2] = {ax[2].g0, ax[2].g1};
    for (int si = 0; si < 2; ++si)
      for (int t = 0; t < 2; ++t)
        for (int u = 0; u < 2; ++u) {
          double w = wx[si] * wy[t] * wz[u];
          node_t* nd = node_by_index(s, g, ax[0].base + si, ax[1].base + t, ax[2].base + u);
          if (!nd) return fail(e, CKG_NUM_INACTIVE_BLOCK, pi, 0, "access to inactive grid block");
          nd->mass += w * p->mass;
          double wm = w * p->mass;
          double mom[3] = {p->v[0] * wm, p->v[1] * wm, p->v[2] * wm};
          if (C) {
            double xi[3] = {xix[si], xiy[t], xiz[u]}, cx[3];
            matvec(C, xi, cx);
            for (int a = 0; a < 3; ++a) mom[a] += cx[a] * wm;
          }
          if (A) {
            double gw[3] = {gx[si] * wy[t] * wz[u], wx[si] * gy[t] * wz[u], wx[si] * wy[t] * gz[u]}, ag[3];
            matvec(A, gw, ag);
            for (int a = 0; a < 3; ++a) mom[a] -= ag[a] * dt;
          }
          nd->p[0] += mom[0];
          nd->p[1] += mom[1];
          nd->p[2] += mom[2];
        }
  }
  return 0;
}

/* detail::scatter_force_mls_one (transfer.hpp:335-369) */
static int scatter_force_mls_one(ckor_sim* s, const ckg_particle_f64* p, const dual_stencil_t* ds,
                                 const double* A, const double* Minv, double dt, err_t* e,
                                 uint64_t pi) {
  const double dx = s->cfg.dx;
  for (int g = 0; g < 2; ++g) {
    int k = grid_tag(g);
    const axis_pair_t* ax = ds->ax[g];
    double xix[2], xiy[2], xiz[2];
    axis_geom(&ax[0], p->x[0], k, dx, xix);
    axis_geom(&ax[1], p->x[1], k, dx, xiy);
    axis_geom(&ax[2], p->x[2], k, dx, xiz);
    double wx[2] = {ax[0].w0, ax[0].w1}, wy[2] = {ax[1].w0, ax[1].w1}, wz[2] = {ax[2].w0, ax[2].w1};
    for (int si = 0; si < 2; ++si)
      for (int t = 0; t < 2; ++t)
        for (int u = 0; u < 2; ++u) {
          double w = wx[si] * wy[t] * wz[u];
          double P[4] = {1.0, xix[si], xiy[t], xiz[u]}, q[4];
          for (int i = 0; i < 4; ++i) {
            double r = 0.0;
            for (int j = 0; j < 4; ++j) r += Minv[4 * i + j] * P[j];
            q[i] = r;
          }
          double gp[3] = {w * q[1], w * q[2], w * q[3]}, ag[3];
          matvec(A, gp, ag);
          double ndt = -dt;
          node_t* nd = node_by_index(s, g, ax[0].base + si, ax[1].base + t, ax[2].base + u);
          if (!nd) return fail(e, CKG_NUM_INACTIVE_BLOCK, pi, 0, "access to inactive grid block");
          nd->p[0] += ag[0] * ndt;
          nd->p[1] += ag[1] * ndt;
          nd->p[2] += ag[2] * ndt;
        }
  }
  return 0;
}

/* --------------------------------------------------------------- phases */

/* sort_particles: stable counting sort by G- block key (simulation.hpp:248-274) */
static void compute_keys(const ckor_sim* s, uint64_t* keys) {
  const double inv_dx = 1.0 / s->cfg.dx;
  const int D = s->D;
  for (uint64_t i = 0; i < s->n; ++i) {
    const double* x = s->ps[i].x;
    uint64_t kk[3];
    for (int a = 0; a < 3; ++a) {
      int b = ((int)floor(x[a] * inv_dx + 0.25)) >> 2;
      if (b < 0) b = 0;
      if (b > D - 1) b = D - 1;
      kk[a] = (uint64_t)b;
    }
    keys[i] = (kk[0] * D + kk[1]) * D + kk[2];
  }
}

static void stable_order(const ckor_sim* s, const uint64_t* keys, uint64_t* counts, uint32_t* order) {
  uint64_t nb = (uint64_t)s->D * s->D * s->D;
  memset(counts, 0, (nb + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < s->n; ++i) ++counts[keys[i] + 1];
  for (uint64_t b = 1; b <= nb; ++b) counts[b] += counts[b - 1];
  for (uint64_t i = 0; i < s->n; ++i) order[counts[keys[i]]++] = (uint32_t)i;
}

static void sort_particles(ckor_sim* s) {
  uint32_t* order = (uint32_t*)malloc(s->n * sizeof(uint32_t) + 1);
  compute_keys(s, s->keys);
  stable_order(s, s->keys, s->counts, order);
  for (uint64_t i = 0; i < s->n; ++i) s->scratch[i] = s->ps[order[i]];
  ckg_particle_f64* t = s->ps;
  s->ps = s->scratch;
  s->scratch = t;
  free(order);
}

void ckor_sort(const ckor_sim* s, uint32_t* keys_out, uint32_t* order) {
  uint64_t* keys = (uint64_t*)malloc(s->n * sizeof(uint64_t) + 8);
  uint64_t* counts = (uint64_t*)malloc(((uint64_t)s->D * s->D * s->D + 1) * sizeof(uint64_t));
  compute_keys(s, keys);
  stable_order(s, keys, counts, order);
  for (uint64_t i = 0; i < s->n; ++i) keys_out[i] = (uint32_t)keys[order[i]];
  free(keys);
  free(counts);
}

/* scatter_all, serial branch (simulation.hpp:279-337) */
static int scatter_all(ckor_sim* s, double dt, err_t* e) {
  const double dx = s->cfg.dx;
  for (uint64_t i = 0; i < s->n; ++i) {
    const ckg_particle_f64* p = &s->ps[i];
    const ckg_material* mat = &s->cfg.materials[p->material];
    double A[9];
    int rc = force_matrix(p, mat, A, e, i);
    if (rc || e->msg[0]) return rc ? rc : 2;
    dual_stencil_t* ds = &s->ds[i];
    *ds = dual_stencil(p->x, dx);
    if (s->cfg.scheme == CKG_SCHEME_PIC) {
      if ((rc = scatter_one(s, p, ds, NULL, A, dt, e, i))) return rc;
    } else {
      double D[9], Di[9], C[9];
      compute_apic_D(p->x, ds, dx, D);
      if ((rc = apic_d_inverse(D, Di, e, i))) return rc;
      matmul(p->B, Di, C);
      if (s->cfg.scheme == CKG_SCHEME_MLS) {
        if ((rc = scatter_one(s, p, ds, C, NULL, 0.0, e, i))) return rc;
        double Mm[16], Mi[16];
        mls_moment(p->x, ds, dx, Mm);
        if (!gauss_inverse4(Mm, Mi)) return fail(e, CKG_NUM_SINGULAR_MLS, i, 0, "singular MLS moment matrix");
        if ((rc = scatter_force_mls_one(s, p, ds, A, Mi, dt, e, i))) return rc;
      } else {
        if ((rc = scatter_one(s, p, ds, C, A, dt, e, i))) return rc;
      }
    }
  }
  return 0;
}

/* grid_update_block + BoundaryCondition::contains/apply (transfer.hpp:419-440, grid.hpp:34-55) */
static void grid_update(ckor_sim* s, double dt) {
  const double dx = s->cfg.dx;
  const double* gr = s->cfg.gravity;
  for (uint64_t b = 0; b < s->nblocks; ++b) {
    block_t* blk = &s->blocks[b];
    for (int g = 0; g < 2; ++g)
      for (int n = 0; n < 64; ++n) {
        node_t* nd = &blk->nodes[g * 64 + n];
        if (nd->mass > s->cfg.mass_eps) {
          double inv = 1.0 / nd->mass;
          for (int a = 0; a < 3; ++a) nd->p[a] = nd->p[a] * inv + gr[a] * dt;
          if (s->cfg.n_boundaries > 0) {
            int cell[3] = {(n >> 4) & 3, (n >> 2) & 3, n & 3};
            double off = ((double)grid_tag(g) * 0.25) * dx;
            double x[3];
            for (int a = 0; a < 3; ++a) x[a] = (double)(blk->coord[a] * 4 + cell[a]) * dx + off;
            for (int bi = 0; bi < s->cfg.n_boundaries; ++bi) {
              const ckg_boundary* bc = &s->cfg.boundaries[bi];
              if (!(x[0] >= bc->lo[0] && x[0] <= bc->hi[0] && x[1] >= bc->lo[1] && x[1] <= bc->hi[1] &&
                    x[2] >= bc->lo[2] && x[2] <= bc->hi[2]))
                continue;
              if (bc->kind == CKG_BC_STICKY) {
                double r[3] = {x[0] - bc->center[0], x[1] - bc->center[1], x[2] - bc->center[2]}, c[3];
                cross3(bc->omega, r, c);
                for (int a = 0; a < 3; ++a) nd->p[a] = bc->velocity[a] + c[a];
              } else if (bc->kind == CKG_BC_SLIP) {
                double vn = dot3(nd->p, bc->normal);
                double t[3] = {bc->normal[0] * vn, bc->normal[1] * vn, bc->normal[2] * vn};
                for (int a = 0; a < 3; ++a) nd->p[a] -= t[a];
              } else {
                double vn = dot3(nd->p, bc->normal);
                if (vn < 0.0) {
                  double t[3] = {bc->normal[0] * vn, bc->normal[1] * vn, bc->normal[2] * vn};
                  for (int a = 0; a < 3; ++a) nd->p[a] -= t[a];
                }
              }
            }
          }
        } else {
          nd->mass = 0.0;
          nd->p[0] = nd->p[1] = nd->p[2] = 0.0;
        }
      }
  }
}

/* clamp_singular_values (material.hpp:179-191) */
static void clamp_singular_values(double* F, double floor_value) {
  double U[9], sg[3], V[9];
  svd3(F, U, sg, V);
  int touched = 0;
  for (int i = 0; i < 3; ++i)
    if (sg[i] < floor_value) { sg[i] = floor_value; touched = 1; }
  if (!touched) return;
  double Dg[9], Vt[9], t[9];
  diag3(sg[0], sg[1], sg[2], Dg);
  transpose3(V, Vt);
  matmul(U, Dg, t);
  matmul(t, Vt, F);
}

/* return_map_drucker_prager (material.hpp:157-175) */
static int return_map_dp(double* F, double alpha, double mu, double lambda, err_t* e, uint64_t pi) {
  if (!(det3(F) > 0.0)) return fail(e, CKG_NUM_RETURN_MAP_INVERTED, pi, 0, "plastic return map: det F <= 0");
  double U[9], sg[3], V[9];
  svd3(F, U, sg, V);
  double eps[3] = {log(sg[0]), log(sg[1]), log(sg[2])};
  double tr = eps[0] + eps[1] + eps[2];
  if (tr > 0.0) {
    eps[0] = eps[1] = eps[2] = 0.0;
  } else {
    double t3 = tr / 3.0;
    double dev[3] = {eps[0] - t3, eps[1] - t3, eps[2] - t3};
    double dev_norm = norm3(dev);
    double dgamma = dev_norm + alpha * (3.0 * lambda + 2.0 * mu) / (2.0 * mu) * tr;
    if (dgamma <= 0.0) return 0;
    double f = dgamma / dev_norm;
    for (int a = 0; a < 3; ++a) eps[a] -= dev[a] * f;
  }
  double S[9], Vt[9], t[9];
  diag3(exp(eps[0]), exp(eps[1]), exp(eps[2]), S);
  transpose3(V, Vt);
  matmul(U, S, t);
  matmul(t, Vt, F);
  return 0;
}

typedef struct { double v[3], B[9], gradv[9]; } gather_t;

/* gather_one over the dual stencil: plain dual average (transfer.hpp:465-510) */
static int gather_one(ckor_sim* s, const double* xp, const dual_stencil_t* ds, gather_t* out,
                      err_t* e, uint64_t pi) {
  const double dx = s->cfg.dx;
  memset(out, 0, sizeof *out);
  for (int g = 0; g < 2; ++g) {
    int k = grid_tag(g);
    const axis_pair_t* ax = ds->ax[g];
    double xix[2], xiy[2], xiz[2];
    axis_geom(&ax[0], xp[0], k, dx, xix);
    axis_geom(&ax[1], xp[1], k, dx, xiy);
    axis_geom(&ax[2], xp[2], k, dx, xiz);
    double wx[2] = {ax[0].w0, ax[0].w1}, wy[2] = {ax[1].w0, ax[1].w1}, wz[2] = {ax[2].w0, ax[2].w1};
    double gx[2] = {ax[0].g0, ax[0].g1}, gy[2] = {ax[1].g0, ax[1].g1}, gz[2] = {ax[2].g0, ax[2].g1};
    for (int si = 0; si < 2; ++si)
      for (int t = 0; t < 2; ++t)
        for (int u = 0; u < 2; ++u) {
          node_t* nd = node_by_index(s, g, ax[0].base + si, ax[1].base + t, ax[2].base + u);
          if (!nd) return fail(e, CKG_NUM_INACTIVE_BLOCK, pi, 0, "access to inactive grid block");
          double w = wx[si] * wy[t] * wz[u];
          double hw = 0.5 * w;
          const double* vn = nd->p;
          for (int a = 0; a < 3; ++a) out->v[a] += vn[a] * hw;
          double xi[3] = {xix[si], xiy[t], xiz[u]};
          double gw[3] = {gx[si] * wy[t] * wz[u], wx[si] * gy[t] * wz[u], wx[si] * wy[t] * gz[u]};
          for (int a = 0; a < 3; ++a)
            for (int bb = 0; bb < 3; ++bb) {
              out->B[3 * a + bb] += hw * vn[a] * xi[bb];
              out->gradv[3 * a + bb] += 0.5 * vn[a] * gw[bb];
            }
        }
  }
  return 0;
}

/* update_particle_state (transfer.hpp:594-627) */
static int update_particle_state(ckor_sim* s, ckg_particle_f64* p, const gather_t* g,
                                 const ckg_material* mat, double dt, const double* mls_D, err_t* e,
                                 uint64_t pi) {
  memcpy(p->v, g->v, sizeof p->v);
  double local[9];
  memcpy(local, g->gradv, sizeof local);
  int scheme = s->cfg.scheme;
  if (scheme != CKG_SCHEME_PIC) {
    memcpy(p->B, g->B, sizeof p->B);
    if (scheme == CKG_SCHEME_MLS) {
      double Di[9];
      int rc = apic_d_inverse(mls_D, Di, e, pi);
      if (rc) return rc;
      matmul(p->B, Di, local);
    }
  }
  if (mat->model == CKG_MODEL_J_FLUID) {
    if (mat->viscosity > 0.0 && scheme != CKG_SCHEME_PIC) {
      /* viscous_deviatoric_factor (material.hpp:196-199) */
      double f = exp(-mat->viscosity * dt / (mat->density * s->cfg.dx * s->cfg.dx));
      double tb = (p->B[0] + p->B[4] + p->B[8]) / 3.0;
      double dev[9], Dg[9];
      memcpy(dev, p->B, sizeof dev);
      double t = (p->B[0] + p->B[4] + p->B[8]) / 3.0;
      dev[0] -= t; dev[4] -= t; dev[8] -= t;
      diag3(tb, tb, tb, Dg);
      for (int i = 0; i < 9; ++i) p->B[i] = Dg[i] + dev[i] * f;
    }
    p->J *= 1.0 + dt * (local[0] + local[4] + local[8]);
    if (!(p->J > 0.0)) return fail(e, CKG_NUM_FLUID_J, pi, 0, "fluid compression drove J <= 0");
  } else {
    double I[9], Ld[9], Fn[9];
    identity3(I);
    scale3(dt, local, Ld);
    for (int i = 0; i < 9; ++i) Ld[i] = I[i] + Ld[i];
    matmul(Ld, p->F, Fn);
    if (s->cfg.clamp_singular) clamp_singular_values(Fn, s->cfg.clamp_floor);
    if (mat->model == CKG_MODEL_DRUCKER_PRAGER) {
      int rc = return_map_dp(Fn, mat->dp_alpha, mat->mu, mat->lambda, e, pi);
      if (rc) return rc;
    } else if (!(det3(Fn) > 0.0)) {
      return fail(e, CKG_NUM_F_INVERTED, pi, 0, "deformation gradient inverted");
    }
    memcpy(p->F, Fn, sizeof Fn);
  }
  for (int a = 0; a < 3; ++a) p->x[a] += p->v[a] * dt;
  return 0;
}

/* gather_all with the vmax / min J / non-finite reductions (simulation.hpp:339-396) */
static int gather_all(ckor_sim* s, double dt, err_t* e) {
  double vm = 0.0;
  double mj[CKG_MAX_MATERIALS];
  for (int m = 0; m < CKG_MAX_MATERIALS; ++m) mj[m] = INFINITY;
  int bad = 0;
  for (uint64_t i = 0; i < s->n; ++i) {
    ckg_particle_f64* p = &s->ps[i];
    const dual_stencil_t* ds = &s->ds[i];
    gather_t g;
    int rc = gather_one(s, p->x, ds, &g, e, i);
    if (rc) return rc;
    const ckg_material* mat = &s->cfg.materials[p->material];
    if (s->cfg.scheme == CKG_SCHEME_MLS) {
      double D[9];
      compute_apic_D(p->x, ds, s->cfg.dx, D);
      rc = update_particle_state(s, p, &g, mat, dt, D, e, i);
    } else {
      rc = update_particle_state(s, p, &g, mat, dt, NULL, e, i);
    }
    if (rc) return rc;
    double s2 = dot3(p->v, p->v);
    vm = (vm < s2) ? s2 : vm; /* std::max(vm, s2) */
    if (mat->model == CKG_MODEL_J_FLUID) mj[p->material] = (p->J < mj[p->material]) ? p->J : mj[p->material];
    if (!isfinite(s2) || !isfinite(dot3(p->x, p->x))) bad = 1;
  }
  if (bad) {
    char m[128];
    snprintf(m, sizeof m, "non-finite particle state after step %llu", (unsigned long long)(s->step_count + 1));
    return fail(e, CKG_NUM_NONFINITE, 0, 0, m);
  }
  s->vmax = sqrt(vm);
  for (int m = 0; m < s->cfg.n_materials; ++m) s->min_j[m] = isfinite(mj[m]) ? mj[m] : 1.0;
  return 0;
}

/* ------------------------------------------------------------------- API */

ckor_sim* ckor_create(const ckg_config* cfg, const ckg_particle_f64* particles, uint64_t n) {
  ckor_sim* s = (ckor_sim*)calloc(1, sizeof(ckor_sim));
  s->cfg = *cfg;
  s->n = n;
  s->ps = (ckg_particle_f64*)malloc((n + 1) * sizeof(ckg_particle_f64));
  s->scratch = (ckg_particle_f64*)malloc((n + 1) * sizeof(ckg_particle_f64));
  s->ds = (dual_stencil_t*)malloc((n + 1) * sizeof(dual_stencil_t));
  s->keys = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  if (n) memcpy(s->ps, particles, n * sizeof(ckg_particle_f64));
  s->D = cfg->resolution / 4 + 2;
  uint64_t nb = (uint64_t)s->D * s->D * s->D;
  s->counts = (uint64_t*)malloc((nb + 1) * sizeof(uint64_t));
  s->directory = (int32_t*)malloc(nb * sizeof(int32_t));
  for (uint64_t d = 0; d < nb; ++d) s->directory[d] = -1;
  /* refresh_velocity_stats (simulation.hpp:234-243) */
  double vm = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    double v = norm3(s->ps[i].v);
    vm = vm < v ? v : vm;
  }
  s->vmax = vm;
  for (int m = 0; m < CKG_MAX_MATERIALS; ++m) s->min_j[m] = 1.0;
  for (uint64_t i = 0; i < n; ++i) {
    const ckg_particle_f64* p = &s->ps[i];
    if (cfg->materials[p->material].model == CKG_MODEL_J_FLUID && p->J < s->min_j[p->material])
      s->min_j[p->material] = p->J;
  }
  return s;
}

void ckor_destroy(ckor_sim* s) {
  if (!s) return;
  free(s->ps); free(s->scratch); free(s->ds); free(s->keys); free(s->counts);
  free(s->directory); free(s->blocks);
  free(s);
}

static void put(char* err, int32_t cap, const char* m) {
  if (err && cap > 0) snprintf(err, (size_t)cap, "%s", m);
}

/* Simulation::step (simulation.hpp:150-188) */
int32_t ckor_step_phases(ckor_sim* s, double dt, int32_t stop_after, ckg_step_out* out, char* err,
                         int32_t cap) {
  err_t e;
  memset(&e, 0, sizeof e);
  if (out) memset(out, 0, sizeof *out);
  put(err, cap, "");
  int rc = 0, phase = CKG_PHASE_SORT;
  sort_particles(s);
  if (stop_after >= CKG_PHASE_ACTIVATE) { phase = CKG_PHASE_ACTIVATE; rc = activate(s, &e); }
  if (!rc && stop_after >= CKG_PHASE_CLEAR) {
    phase = CKG_PHASE_CLEAR;
    for (uint64_t b = 0; b < s->nblocks; ++b) memset(s->blocks[b].nodes, 0, sizeof s->blocks[b].nodes);
  }
  if (!rc && stop_after >= CKG_PHASE_P2G) { phase = CKG_PHASE_P2G; rc = scatter_all(s, dt, &e); }
  if (!rc && stop_after >= CKG_PHASE_GRID) { phase = CKG_PHASE_GRID; grid_update(s, dt); }
  if (!rc && stop_after >= CKG_PHASE_G2P) { phase = CKG_PHASE_G2P; rc = gather_all(s, dt, &e); }
  if (out) {
    out->status = rc;
    out->error_code = e.code;
    out->error_axis = e.axis;
    out->error_particle = e.particle;
    out->error_phase = rc ? phase : 0;
    out->active_blocks = s->nblocks;
    out->vmax = s->vmax;
    for (int m = 0; m < CKG_MAX_MATERIALS; ++m) out->min_j[m] = s->min_j[m];
    uint64_t per = s->cfg.scheme == CKG_SCHEME_MLS ? 32 : 16;
    out->p2g_node_visits = per * s->n;
    out->g2p_node_visits = 16 * s->n;
    out->p2g_transfers = s->n;
    out->g2p_transfers = s->n;
  }
  if (rc) put(err, cap, e.msg);
  else if (stop_after >= CKG_PHASE_G2P) s->step_count++;
  return rc;
}

int32_t ckor_step(ckor_sim* s, double dt, ckg_step_out* out, char* err, int32_t cap) {
  return ckor_step_phases(s, dt, CKG_PHASE_G2P, out, err, cap);
}

uint64_t ckor_count(const ckor_sim* s) { return s->n; }
void ckor_particles(const ckor_sim* s, ckg_particle_f64* out) { memcpy(out, s->ps, s->n * sizeof(ckg_particle_f64)); }
double ckor_vmax(const ckor_sim* s) { return s->vmax; }
uint64_t ckor_active_blocks(const ckor_sim* s) { return s->nblocks; }

void ckor_grid(const ckor_sim* s, int32_t* coords, double* nodes, uint64_t nb) {
  uint64_t k = nb < s->nblocks ? nb : s->nblocks;
  for (uint64_t b = 0; b < k; ++b) {
    if (coords) for (int a = 0; a < 3; ++a) coords[3 * b + a] = s->blocks[b].coord[a];
    if (nodes)
      for (int n = 0; n < 128; ++n) {
        const node_t* nd = &s->blocks[b].nodes[n];
        double* o = nodes + (b * 128 + n) * 4;
        o[0] = nd->mass; o[1] = nd->p[0]; o[2] = nd->p[1]; o[3] = nd->p[2];
      }
  }
}

/* cfl_dt (simulation.hpp:134-145) with sound speeds (:73-81) */
double ckor_cfl_dt(const ckor_sim* s, double cfl, double max_dt, double remaining) {
  double cmax = 0.0;
  for (int mi = 0; mi < s->cfg.n_materials; ++mi) {
    const ckg_material* m = &s->cfg.materials[mi];
    double c = m->model == CKG_MODEL_J_FLUID
                   ? sqrt(m->bulk * m->gamma * pow(s->min_j[mi], 1.0 - m->gamma) / m->density)
                   : sqrt((m->lambda + 2.0 * m->mu) / m->density);
    cmax = cmax < c ? c : cmax;
  }
  double denom = s->vmax < cmax ? cmax : s->vmax;
  double dt = denom > 0.0 ? cfl * s->cfg.dx / denom : remaining;
  if (max_dt > 0.0) dt = dt < max_dt ? dt : max_dt;
  return dt < remaining ? dt : remaining;
}

/* compute_diagnostics (simulation.hpp:55-69) */
void ckor_diagnostics(const ckor_sim* s, ckg_diagnostics* o) {
  memset(o, 0, sizeof *o);
  for (uint64_t i = 0; i < s->n; ++i) {
    const ckg_particle_f64* p = &s->ps[i];
    double c[3];
    cross3(p->x, p->v, c);
    for (int a = 0; a < 3; ++a) {
      o->momentum[a] += p->v[a] * p->mass;
      o->angular[a] += c[a] * p->mass;
      o->momentum_massfree[a] += p->v[a];
    }
    o->kinetic_energy += 0.5 * p->mass * dot3(p->v, p->v);
    double v = norm3(p->v);
    o->vmax = o->vmax < v ? v : o->vmax;
  }
}
