/*
 * mcs_oracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE (see mcs_oracle.h).
 *
 * The plain CPU oracle of the hot path of arXiv 2504.18056, written from the
 * paper (PAPER.md, "P:n") step by step in the paper's order and notation, with
 * the readings of DESIGN.md §3 ("Rn") where the paper is silent.  fp64
 * throughout except the pinned fp32 correspondence-key path (R27), which must be
 * compiled WITHOUT floating-point contraction (-ffp-contract=off) so that every
 * a*b is a separately rounded product and every fmaf() a single rounding.
 *
 * Deliberately simple: per-point loops, a sorted cell list with binary search
 * for the voxel map, a textbook Cholesky for every linear solve, no blocking,
 * no fusion.  OpenMP only splits the independent per-particle loop (P:85:
 * "Each particle can be updated independently").
 */
#include "mcs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CELL_MIN (-1048576)  /* 21-bit signed cell range (R27) */
#define CELL_MAX (1048575)

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------------- */
/* small fp64 linear algebra                                                  */
/* ------------------------------------------------------------------------- */

static void skew(const double v[3], double M[9]) {
  M[0] = 0.0;   M[1] = -v[2]; M[2] = v[1];
  M[3] = v[2];  M[4] = 0.0;   M[5] = -v[0];
  M[6] = -v[1]; M[7] = v[0];  M[8] = 0.0;
}

static void mat3_mul(const double A[9], const double B[9], double C[9]) {
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
      for (int c = 0; c < 3; ++c) s += A[3 * a + c] * B[3 * c + b];
      C[3 * a + b] = s;
    }
}

static void cov6_to_mat(const double c[6], double M[9]) {
  M[0] = c[0]; M[1] = c[1]; M[2] = c[2];
  M[3] = c[1]; M[4] = c[3]; M[5] = c[4];
  M[6] = c[2]; M[7] = c[4]; M[8] = c[5];
}

/* Cholesky factorisation A = L L^T of an n x n SPD matrix (row-major).
 * returns 0 on success, 1 if a pivot is not strictly positive. */
static int cholesky(int n, const double* A, double* L) {
  memset(L, 0, sizeof(double) * n * n);
  for (int j = 0; j < n; ++j) {
    double d = A[j * n + j];
    for (int k = 0; k < j; ++k) d -= L[j * n + k] * L[j * n + k];
    if (!(d > 0.0)) return 1;
    L[j * n + j] = sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = A[i * n + j];
      for (int k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = s / L[j * n + j];
    }
  }
  return 0;
}

/* solve L L^T x = y given the Cholesky factor L */
static void chol_solve(int n, const double* L, const double* y, double* x) {
  double z[8];
  for (int i = 0; i < n; ++i) {
    double s = y[i];
    for (int k = 0; k < i; ++k) s -= L[i * n + k] * z[k];
    z[i] = s / L[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = z[i];
    for (int k = i + 1; k < n; ++k) s -= L[k * n + i] * x[k];
    x[i] = s / L[i * n + i];
  }
}

/* inverse of a 3x3 SPD matrix through its Cholesky factor; 1 if not PD */
static int spd3_inverse(const double C[9], double Cinv[9]) {
  double L[9];
  if (cholesky(3, C, L)) return 1;
  for (int col = 0; col < 3; ++col) {
    double y[3] = {0.0, 0.0, 0.0}, x[3];
    y[col] = 1.0;
    chol_solve(3, L, y, x);
    for (int row = 0; row < 3; ++row) Cinv[3 * row + col] = x[row];
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* SE(3): exp / log / compose (right-applied exp; R2)    */
/* ------------------------------------------------------------------------- */

void orc_se3_exp(const double xi[6], double T[12]) {
  const double* rho = xi;
  const double* phi = xi + 3;
  double th2 = phi[0] * phi[0] + phi[1] * phi[1] + phi[2] * phi[2];
  double th = sqrt(th2);
  double A, B, C; /* sin(th)/th, (1-cos th)/th^2, (th - sin th)/th^3 */
  if (th < 1e-4) {
    A = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    B = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
    C = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0;
  } else {
    A = sin(th) / th;
    B = (1.0 - cos(th)) / th2;
    C = (th - sin(th)) / (th2 * th);
  }
  double W[9], W2[9];
  skew(phi, W);
  mat3_mul(W, W, W2);
  double R[9], V[9];
  for (int k = 0; k < 9; ++k) {
    double I = (k % 4 == 0) ? 1.0 : 0.0;
    R[k] = I + A * W[k] + B * W2[k];
    V[k] = I + B * W[k] + C * W2[k];
  }
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) T[4 * a + b] = R[3 * a + b];
    T[4 * a + 3] = V[3 * a + 0] * rho[0] + V[3 * a + 1] * rho[1] + V[3 * a + 2] * rho[2];
  }
}

int orc_se3_log(const double T[12], double xi[6]) {
  double R[9], t[3];
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) R[3 * a + b] = T[4 * a + b];
    t[a] = T[4 * a + 3];
  }
  double c = 0.5 * (R[0] + R[4] + R[8] - 1.0);
  if (c > 1.0) c = 1.0;
  if (c < -1.0) c = -1.0;
  double th = acos(c);
  if (th > M_PI - 1e-6) return 1;
  double v[3] = {R[7] - R[5], R[2] - R[6], R[3] - R[1]}; /* (R - R^T)^vee * 2 */
  double k; /* phi = k * v */
  if (th < 1e-4) {
    k = 0.5 + th * th / 12.0 + 7.0 * th * th * th * th / 720.0;
  } else {
    k = th / (2.0 * sin(th));
  }
  double phi[3] = {k * v[0], k * v[1], k * v[2]};
  /* V^-1 = I - W/2 + (1/th^2) (1 - A/(2B)) W^2 */
  double W[9], W2[9];
  skew(phi, W);
  mat3_mul(W, W, W2);
  double g;
  if (th < 1e-4) {
    g = 1.0 / 12.0 + th * th / 720.0;
  } else {
    double A = sin(th) / th, B = (1.0 - cos(th)) / (th * th);
    g = (1.0 - A / (2.0 * B)) / (th * th);
  }
  for (int a = 0; a < 3; ++a) {
    double s = 0.0;
    for (int b = 0; b < 3; ++b) {
      double I = (a == b) ? 1.0 : 0.0;
      s += (I - 0.5 * W[3 * a + b] + g * W2[3 * a + b]) * t[b];
    }
    xi[a] = s;
    xi[3 + a] = phi[a];
  }
  return 0;
}

void orc_compose(const double A[12], const double B[12], double AB[12]) {
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 4; ++b) {
      double s = (b == 3) ? A[4 * a + 3] : 0.0;
      for (int c = 0; c < 3; ++c) s += A[4 * a + c] * B[4 * c + b];
      AB[4 * a + b] = s;
    }
  }
}

/* T <- T exp(xi) in fp64 from an fp32 pose, one Newton re-orthonormalisation
 * step R <- R (3I - R^T R) / 2 (R30), rounded back to fp32 (R23). */
static void pose32_right_update(float T32[12], const double xi[6]) {
  double T[12], E[12], TE[12];
  for (int k = 0; k < 12; ++k) T[k] = (double)T32[k];
  orc_se3_exp(xi, E);
  orc_compose(T, E, TE);
  double R[9], RtR[9], M[9], Rn[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) R[3 * a + b] = TE[4 * a + b];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
      for (int c = 0; c < 3; ++c) s += R[3 * c + a] * R[3 * c + b];
      RtR[3 * a + b] = s;
    }
  for (int k = 0; k < 9; ++k) M[k] = ((k % 4 == 0) ? 3.0 : 0.0) - RtR[k];
  mat3_mul(R, M, Rn);
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) T32[4 * a + b] = (float)(0.5 * Rn[3 * a + b]);
    T32[4 * a + 3] = (float)TE[4 * a + 3];
  }
}

/* ------------------------------------------------------------------------- */
/* keyframe voxel map ("voxel-based corresponding point search",        */
/* P:119; one aggregate per occupied cell: mean of means, mean of covs S:112)  */
/* ------------------------------------------------------------------------- */

typedef struct {
  int32_t c[3];
  int32_t count;
  double mean[3];
  double cov[6];
} orc_cell;

struct orc_map {
  int32_t n;
  float inv_r;
  orc_cell* cells; /* sorted lexicographically by (cx, cy, cz) */
  int32_t corr_mode; /* 0 CELL (R7), 1 NN27 (R33) */
  float nn_r2;       /* NN27: nn_radius * nn_radius in fp32 */
};

static int cell_cmp3(const int32_t* a, const int32_t* b) {
  for (int k = 0; k < 3; ++k) {
    if (a[k] < b[k]) return -1;
    if (a[k] > b[k]) return 1;
  }
  return 0;
}

typedef struct { int32_t c[3]; int32_t idx; } cell_idx;

static int cell_idx_cmp(const void* pa, const void* pb) {
  const cell_idx* a = (const cell_idx*)pa;
  const cell_idx* b = (const cell_idx*)pb;
  int r = cell_cmp3(a->c, b->c);
  if (r) return r;
  return (a->idx > b->idx) - (a->idx < b->idx); /* input order within a cell */
}

/* R27: the pinned fp32 cell of a point, floorf(q * inv_r) per axis with
 * inv_r = 1/r exact (r a power of two).  0 if outside the 21-bit range. */
int orc_cell_of(float qx, float qy, float qz, float inv_r, int32_t cell[3]) {
  float q[3] = {qx, qy, qz};
  for (int a = 0; a < 3; ++a) {
    float f = floorf(q[a] * inv_r);
    if (!(f >= (float)CELL_MIN && f <= (float)CELL_MAX)) return 0;
    cell[a] = (int32_t)f;
  }
  return 1;
}

orc_map* orc_map_build(const float* mean3, const float* cov6, int32_t n, float r) {
  orc_map* m = (orc_map*)calloc(1, sizeof(orc_map));
  m->inv_r = 1.0f / r;
  cell_idx* ci = (cell_idx*)malloc(sizeof(cell_idx) * (n > 0 ? n : 1));
  int32_t valid = 0;
  for (int32_t j = 0; j < n; ++j) {
    int32_t c[3];
    if (!orc_cell_of(mean3[3 * j], mean3[3 * j + 1], mean3[3 * j + 2], m->inv_r, c)) continue;
    memcpy(ci[valid].c, c, sizeof(c));
    ci[valid].idx = j;
    ++valid;
  }
  qsort(ci, valid, sizeof(cell_idx), cell_idx_cmp);
  m->cells = (orc_cell*)calloc(valid > 0 ? valid : 1, sizeof(orc_cell));
  int32_t nc = 0;
  for (int32_t s = 0; s < valid;) {
    int32_t e = s;
    while (e < valid && cell_cmp3(ci[e].c, ci[s].c) == 0) ++e;
    orc_cell* cell = &m->cells[nc++];
    memcpy(cell->c, ci[s].c, sizeof(cell->c));
    cell->count = e - s;
    for (int32_t k = s; k < e; ++k) {
      int32_t j = ci[k].idx;
      for (int a = 0; a < 3; ++a) cell->mean[a] += (double)mean3[3 * j + a];
      for (int a = 0; a < 6; ++a) cell->cov[a] += (double)cov6[6 * j + a];
    }
    for (int a = 0; a < 3; ++a) cell->mean[a] /= (double)cell->count;
    for (int a = 0; a < 6; ++a) cell->cov[a] /= (double)cell->count;
    s = e;
  }
  m->n = nc;
  free(ci);
  return m;
}

void orc_map_free(orc_map* m) {
  if (!m) return;
  free(m->cells);
  free(m);
}

int32_t orc_map_size(const orc_map* m) { return m->n; }

int32_t orc_map_cell(const orc_map* m, int32_t k, double mean[3], double cov6[6]) {
  if (k < 0 || k >= m->n) return 0;
  memcpy(mean, m->cells[k].mean, sizeof(double) * 3);
  memcpy(cov6, m->cells[k].cov, sizeof(double) * 6);
  return m->cells[k].count;
}

static int32_t map_find(const orc_map* m, const int32_t c[3]) {
  int32_t lo = 0, hi = m->n - 1;
  while (lo <= hi) {
    int32_t mid = lo + (hi - lo) / 2;
    int r = cell_cmp3(m->cells[mid].c, c);
    if (r == 0) return mid;
    if (r < 0) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

int32_t orc_map_lookup(const orc_map* m, int32_t cx, int32_t cy, int32_t cz,
                       double mean[3], double cov6[6]) {
  int32_t c[3] = {cx, cy, cz};
  int32_t k = map_find(m, c);
  if (k < 0) return 0;
  memcpy(mean, m->cells[k].mean, sizeof(double) * 3);
  memcpy(cov6, m->cells[k].cov, sizeof(double) * 6);
  return m->cells[k].count;
}

/* ------------------------------------------------------------------------- */
/* relative pose kT = (T_k)^-1 T_t  (Eq.4)                      */
/* ------------------------------------------------------------------------- */

void orc_relpose(const float Tk[12], const float Tt[12], float rel32[12], double rel64[12]) {
  /* (a) pinned fp32 key copy (R27): R_rel = Rk^T Rt, t_rel = Rk^T (t_t - t_k),
   * each entry as fmaf(x2, y2, fmaf(x1, y1, x0 * y0)). */
  float d[3];
  for (int a = 0; a < 3; ++a) d[a] = Tt[4 * a + 3] - Tk[4 * a + 3];
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) {
      float p0 = Tk[4 * 0 + a] * Tt[4 * 0 + b];
      rel32[4 * a + b] = fmaf(Tk[4 * 2 + a], Tt[4 * 2 + b], fmaf(Tk[4 * 1 + a], Tt[4 * 1 + b], p0));
    }
    float p0 = Tk[4 * 0 + a] * d[0];
    rel32[4 * a + 3] = fmaf(Tk[4 * 2 + a], d[2], fmaf(Tk[4 * 1 + a], d[1], p0));
  }
  /* (b) fp64 value copy from the same fp32 inputs */
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
      for (int c = 0; c < 3; ++c) s += (double)Tk[4 * c + a] * (double)Tt[4 * c + b];
      rel64[4 * a + b] = s;
    }
    double s = 0.0;
    for (int c = 0; c < 3; ++c)
      s += (double)Tk[4 * c + a] * ((double)Tt[4 * c + 3] - (double)Tk[4 * c + 3]);
    rel64[4 * a + 3] = s;
  }
}

/* pinned fp32 transform of the key path (R27):
 * q_a = fmaf(R[a][2], z, fmaf(R[a][1], y, fmaf(R[a][0], x, t_a))) */
static void key_transform(const float rel32[12], const float* mu, float q[3]) {
  for (int a = 0; a < 3; ++a)
    q[a] = fmaf(rel32[4 * a + 2], mu[2],
                fmaf(rel32[4 * a + 1], mu[1], fmaf(rel32[4 * a + 0], mu[0], rel32[4 * a + 3])));
}

void orc_map_set_corr(orc_map* m, int32_t mode, float nn_radius) {
  m->corr_mode = mode;
  m->nn_r2 = nn_radius * nn_radius;
}

/* CELL (R7): the single voxel containing q */
static int32_t cell_correspond(const orc_map* m, const float q[3]) {
  int32_t c[3];
  if (!orc_cell_of(q[0], q[1], q[2], m->inv_r, c)) return -1;
  return map_find(m, c);
}

/* NN27 (R33): among the 27 cells around q's cell, the cell representative (the fp32-rounded
 * mean of means) nearest to q within nn_radius.  Squared distance in the pinned fp32 order of
 * a1's distances, d = m32 - q32, d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx)); candidates need
 * d2 <= nn_radius^2 (fp32); ties -> lower enumeration index, enumerating (oz, oy, ox) in
 * {-1, 0, 1}^3 lexicographically.  With nn_radius <= r every representative within nn_radius
 * of q lies in this block, so this is the exact nearest neighbour. */
static int32_t nn27_correspond(const orc_map* m, const float q[3]) {
  int32_t c[3];
  if (!orc_cell_of(q[0], q[1], q[2], m->inv_r, c)) return -1;
  int32_t best = -1;
  float best_d2 = 0.0f;
  for (int oz = -1; oz <= 1; ++oz)
    for (int oy = -1; oy <= 1; ++oy)
      for (int ox = -1; ox <= 1; ++ox) {
        const int32_t nc[3] = {c[0] + ox, c[1] + oy, c[2] + oz};
        const int32_t k = map_find(m, nc);
        if (k < 0) continue;
        const float dx = (float)m->cells[k].mean[0] - q[0];
        const float dy = (float)m->cells[k].mean[1] - q[1];
        const float dz = (float)m->cells[k].mean[2] - q[2];
        const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        if (!(d2 <= m->nn_r2)) continue;
        if (best < 0 || d2 < best_d2) {
          best = k;
          best_d2 = d2;
        }
      }
  return best;
}

int32_t orc_map_correspond(const orc_map* m, const float q[3]) {
  return m->corr_mode == 1 ? nn27_correspond(m, q) : cell_correspond(m, q);
}

/* correspondence of scan point mu under rel32: index into the map's cell list or -1 */
static int32_t correspond(const orc_map* m, const float rel32[12], const float* mu) {
  float q[3];
  key_transform(rel32, mu, q);
  return orc_map_correspond(m, q);
}

/* ------------------------------------------------------------------------- */
/* Eqs.3-4 (likelihood) and Eq.6 (H, b, J) for one (particle, keyframe) pair   */
/* ------------------------------------------------------------------------- */

int orc_pair_linearize(const orc_map* m, const float* mean3, const float* cov6, int32_t S,
                       const float rel32[12], const double rel64[12],
                       double* l_out, double H[36], double b[6], int32_t* n_out, int32_t* corr) {
  double R[9], t[3];
  for (int a = 0; a < 3; ++a) {
    for (int c = 0; c < 3; ++c) R[3 * a + c] = rel64[4 * a + c];
    t[a] = rel64[4 * a + 3];
  }
  double l = 0.0;
  int32_t n = 0;
  memset(H, 0, sizeof(double) * 36);
  memset(b, 0, sizeof(double) * 6);
  for (int32_t j = 0; j < S; ++j) {
    const float* muf = mean3 + 3 * j;
    int32_t k = correspond(m, rel32, muf);
    if (corr) corr[j] = k;
    if (k < 0) continue; /* unmatched: skipped (R8) */
    const orc_cell* cell = &m->cells[k];
    double mu[3] = {muf[0], muf[1], muf[2]};
    double Sig[9], Sigp[9], RS[9], RSRt[9], C[9], Om[9];
    double c6[6];
    for (int a = 0; a < 6; ++a) c6[a] = (double)cov6[6 * j + a];
    cov6_to_mat(c6, Sig);
    cov6_to_mat(cell->cov, Sigp);
    /* e_j = mu'_j - kT mu_j  (Eq.4) */
    double e[3];
    for (int a = 0; a < 3; ++a) {
      double q = t[a];
      for (int c = 0; c < 3; ++c) q += R[3 * a + c] * mu[c];
      e[a] = cell->mean[a] - q;
    }
    /* Omega_j = (Sigma'_j + kR Sigma_j kR^T)^-1  (Eq.4) */
    mat3_mul(R, Sig, RS);
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (int d = 0; d < 3; ++d) s += RS[3 * a + d] * R[3 * c + d];
        RSRt[3 * a + c] = s;
      }
    for (int a = 0; a < 9; ++a) C[a] = Sigp[a] + RSRt[a];
    if (spd3_inverse(C, Om)) return 1;
    /* log p -= e^T Omega e  (Eq.3) */
    double Oe[3];
    for (int a = 0; a < 3; ++a) {
      Oe[a] = 0.0;
      for (int c = 0; c < 3; ++c) Oe[a] += Om[3 * a + c] * e[c];
    }
    l -= e[0] * Oe[0] + e[1] * Oe[1] + e[2] * Oe[2];
    /* J_j = de_j/d delta, right perturbation kT exp(delta) (Eq.6, R1-R2):
     * kT exp(delta) mu ~= kT mu + R rho - R [mu]x phi  =>  J = [ -R | R [mu]x ] */
    double Mx[9], RM[9], J[18];
    skew(mu, Mx);
    mat3_mul(R, Mx, RM);
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) {
        J[6 * a + c] = -R[3 * a + c];
        J[6 * a + 3 + c] = RM[3 * a + c];
      }
    /* H += J^T Omega J ; b += J^T Omega e  (Eq.6) */
    double OJ[18];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 6; ++c) {
        double s = 0.0;
        for (int d = 0; d < 3; ++d) s += Om[3 * a + d] * J[6 * d + c];
        OJ[6 * a + c] = s;
      }
    for (int r = 0; r < 6; ++r) {
      for (int c = 0; c < 6; ++c) {
        double s = 0.0;
        for (int d = 0; d < 3; ++d) s += J[6 * d + r] * OJ[6 * d + c];
        H[6 * r + c] += s;
      }
      double s = 0.0;
      for (int d = 0; d < 3; ++d) s += J[6 * d + r] * Oe[d];
      b[r] += s;
    }
    ++n;
  }
  *l_out = l;
  *n_out = n;
  return 0;
}

void orc_pair_omegas(const orc_map* m, const float* cov6, int32_t S, const double rel64[12],
                     const int32_t* corr, double* omega9) {
  double R[9];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) R[3 * a + c] = rel64[4 * a + c];
  for (int32_t j = 0; j < S; ++j) {
    if (corr[j] < 0) continue;
    double c6[6], Sig[9], Sigp[9], RS[9], C[9];
    for (int a = 0; a < 6; ++a) c6[a] = (double)cov6[6 * j + a];
    cov6_to_mat(c6, Sig);
    cov6_to_mat(m->cells[corr[j]].cov, Sigp);
    mat3_mul(R, Sig, RS);
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (int d = 0; d < 3; ++d) s += RS[3 * a + d] * R[3 * c + d];
        C[3 * a + c] = Sigp[3 * a + c] + s;
      }
    spd3_inverse(C, omega9 + 9 * j);
  }
}

double orc_pair_loglik_frozen(const orc_map* m, const float* mean3, int32_t S,
                              const double rel64[12], const int32_t* corr,
                              const double* omega9) {
  double l = 0.0;
  for (int32_t j = 0; j < S; ++j) {
    if (corr[j] < 0) continue;
    const orc_cell* cell = &m->cells[corr[j]];
    double e[3];
    for (int a = 0; a < 3; ++a) {
      double q = rel64[4 * a + 3];
      for (int c = 0; c < 3; ++c) q += rel64[4 * a + c] * (double)mean3[3 * j + c];
      e[a] = cell->mean[a] - q;
    }
    const double* Om = omega9 + 9 * j;
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) l -= e[a] * Om[3 * a + c] * e[c];
  }
  return l;
}

/* ------------------------------------------------------------------------- */
/* Eq.5 (+ damping and clamp, R1, R11)                                        */
/* ------------------------------------------------------------------------- */

int orc_gn_step(const double H[36], const double b[6], double damping_rel, double step_clamp,
                double psi[6], int32_t* clamped) {
  double A[36], L[36], nb[6];
  double tr = 0.0;
  for (int k = 0; k < 6; ++k) tr += H[7 * k];
  double lambda = damping_rel * tr / 6.0;
  memcpy(A, H, sizeof(A));
  for (int k = 0; k < 6; ++k) A[7 * k] += lambda;
  *clamped = 0;
  if (cholesky(6, A, L)) {
    for (int k = 0; k < 6; ++k) psi[k] = 0.0;
    return 1;
  }
  /* psi = -(H + lambda I)^-1 b: the Gauss-Newton ascent step on l (R1) */
  for (int k = 0; k < 6; ++k) nb[k] = -b[k];
  chol_solve(6, L, nb, psi);
  double nrm = 0.0;
  for (int k = 0; k < 6; ++k) nrm += psi[k] * psi[k];
  nrm = sqrt(nrm);
  if (nrm > step_clamp) {
    for (int k = 0; k < 6; ++k) psi[k] *= step_clamp / nrm;
    *clamped = 1;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Eqs.8-9: r_k = d(t_k, t_o) / d(t, t_o), d from the shared odometry path    */
/* length D (R14); keyframes t_o..latest (R15)                                */
/* ------------------------------------------------------------------------- */

int orc_propagation_ratio(const double* D, int32_t K, int32_t t_o, double D_now, double* r) {
  double den = D_now - D[t_o];
  if (!(den > 0.0)) return 1; /* no propagation */
  for (int32_t k = t_o; k < K; ++k) r[k - t_o] = (D[k] - D[t_o]) / den;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* per-particle steps 2-7                                                     */
/* ------------------------------------------------------------------------- */

static void one_particle(const orc_config* cfg, int32_t K, orc_map* const* maps,
                         const double* D, double D_now, float* Tt, float* Tk_all,
                         const float* scan_mean3, const float* scan_cov6, int32_t S,
                         int32_t apply_update, orc_particle_out* out, int32_t p) {
  const int32_t nbmax = cfg->neighbor_count;
  const int32_t nb = K < nbmax ? K : nbmax;
  const int32_t latest = K - 1;
  /* step 2: neighbour keyframes by translation distance, own T_k^i;
   * pinned fp32 squared distance (R6, R27); ties -> lower id */
  float dist[4096];
  for (int32_t k = 0; k < K; ++k) {
    const float* Tk = Tk_all + 12 * (size_t)k;
    float dx = Tk[3] - Tt[3], dy = Tk[7] - Tt[7], dz = Tk[11] - Tt[11];
    float dxx = dx * dx;
    dist[k] = fmaf(dz, dz, fmaf(dy, dy, dxx));
  }
  int32_t slot_kf[8];
  for (int32_t s = 0; s < nb; ++s) {
    int32_t best = -1;
    for (int32_t k = 0; k < K; ++k) {
      int taken = 0;
      for (int32_t u = 0; u < s; ++u) taken |= (slot_kf[u] == k);
      if (taken) continue;
      if (best < 0 || dist[k] < dist[best]) best = k; /* strict <: ties keep lower id */
    }
    slot_kf[s] = best;
  }
  /* loop detection: an "old" keyframe among the neighbours (R5) */
  int32_t loop = 0, t_o = slot_kf[0];
  int32_t old[8];
  for (int32_t s = 0; s < nb; ++s) {
    old[s] = (slot_kf[s] <= latest - cfg->loop_recency_gap);
    loop |= old[s];
    if (slot_kf[s] < t_o) t_o = slot_kf[s];
  }
  /* steps 3-4: relative pose, Eqs.2-4 and Eq.6 per neighbour */
  double l_sum = 0.0, H[36] = {0}, b[6] = {0};
  int32_t unmatched = 0;
  for (int32_t s = 0; s < nb; ++s) {
    float rel32[12];
    double rel64[12], ls, Hs[36], bs[6];
    int32_t ns;
    const float* Tk = Tk_all + 12 * (size_t)slot_kf[s];
    orc_relpose(Tk, Tt, rel32, rel64);
    orc_pair_linearize(maps[slot_kf[s]], scan_mean3, scan_cov6, S, rel32, rel64, &ls, Hs, bs,
                       &ns, NULL);
    if (out->slot_l) out->slot_l[(size_t)p * nbmax + s] = ls;
    if (out->slot_H36) memcpy(out->slot_H36 + ((size_t)p * nbmax + s) * 36, Hs, sizeof(Hs));
    if (out->slot_b6) memcpy(out->slot_b6 + ((size_t)p * nbmax + s) * 6, bs, sizeof(bs));
    if (out->slot_n) out->slot_n[(size_t)p * nbmax + s] = ns;
    if (out->slot_kf) out->slot_kf[(size_t)p * nbmax + s] = slot_kf[s];
    /* step 5: Eq.2 sum over all neighbours; H, b over the slots G that drive the update (R4) */
    l_sum += ls;
    unmatched += S - ns;
    int in_G = (cfg->gn_slots == 1) ? 1 : old[s];
    if (in_G) {
      for (int k = 0; k < 36; ++k) H[k] += Hs[k];
      for (int k = 0; k < 6; ++k) b[k] += bs[k];
    }
  }
  double l = l_sum - cfg->unmatched_penalty * (double)unmatched;
  uint8_t flags = loop ? 1u : 0u;
  double psi[6] = {0, 0, 0, 0, 0, 0};
  if (apply_update && loop) {
    /* step 6: Eq.5 + Eq.7, only for loop particles */
    int32_t clamped = 0;
    if (orc_gn_step(H, b, cfg->damping_rel, cfg->step_clamp, psi, &clamped)) {
      flags |= 4u; /* singular: no update */
    } else {
      if (clamped) flags |= 16u;
      int nonzero = 0;
      for (int k = 0; k < 6; ++k) nonzero |= (psi[k] != 0.0);
      if (nonzero) pose32_right_update(Tt, psi);
      flags |= 2u;
      /* step 7: Eqs.8-10, keyframes t_o..latest (R14-R16) */
      double r[4096];
      if (orc_propagation_ratio(D, K, t_o, D_now, r) == 0) {
        for (int32_t k = t_o; k <= latest; ++k) {
          double rk = r[k - t_o];
          if (rk == 0.0) continue; /* exp(0) = I: untouched (R15) */
          double xi[6];
          for (int c = 0; c < 6; ++c) xi[c] = rk * psi[c];
          pose32_right_update(Tk_all + 12 * (size_t)k, xi);
        }
      }
    }
  }
  out->loglik[p] = l;
  for (int k = 0; k < 6; ++k) out->grad6[6 * (size_t)p + k] = -2.0 * b[k]; /* dl/d delta */
  memcpy(out->hess36 + 36 * (size_t)p, H, sizeof(H));
  memcpy(out->psi6 + 6 * (size_t)p, psi, sizeof(psi));
  out->flags[p] = flags;
}

int orc_particles(const orc_config* cfg, int32_t K, orc_map* const* maps, const double* D,
                  double D_now, int32_t N, float* pose12, float* kf_pose12, int32_t kf_stride,
                  const float* scan_mean3, const float* scan_cov6, int32_t S,
                  const int32_t* idx, int32_t n_idx, int32_t apply_update,
                  orc_particle_out* out) {
  if (K < 1 || K > 4096 || cfg->neighbor_count < 1 || cfg->neighbor_count > 8) return 2;
  if (cfg->corr_mode != 0 && cfg->corr_mode != 1) return 2;
  if (cfg->corr_mode == 1 && !(cfg->nn_radius > 0.0f && cfg->nn_radius <= cfg->voxel_resolution))
    return 2;
  for (int32_t k = 0; k < K; ++k) orc_map_set_corr(maps[k], cfg->corr_mode, cfg->nn_radius);
  if (!idx) n_idx = N;
#pragma omp parallel for schedule(dynamic, 4)
  for (int32_t p = 0; p < n_idx; ++p) {
    int32_t i = idx ? idx[p] : p;
    one_particle(cfg, K, maps, D, D_now, pose12 + 12 * (size_t)i,
                 kf_pose12 + 12 * (size_t)i * kf_stride, scan_mean3, scan_cov6, S,
                 apply_update, out, p);
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Eq.11 in log space; dead set; respawn; representative      */
/* ------------------------------------------------------------------------- */

void orc_weights(int32_t N, double* L, const double* l, double* e, double* w,
                 double* m_out, double* S_out) {
  if (l)
    for (int32_t i = 0; i < N; ++i) L[i] += l[i]; /* log of Eq.11's product */
  double m = -INFINITY;
  for (int32_t i = 0; i < N; ++i) if (L[i] > m) m = L[i];
  double S = 0.0;
  for (int32_t i = 0; i < N; ++i) {
    e[i] = exp(L[i] - m);
    S += e[i];
  }
  for (int32_t i = 0; i < N; ++i) w[i] = e[i] / S;
  if (m_out) *m_out = m;
  if (S_out) *S_out = S;
}

int64_t orc_dead(int32_t N, const double* l, const double* w, double rel_floor,
                 double post_floor, uint8_t* dead) {
  double lstar = -INFINITY;
  for (int32_t i = 0; i < N; ++i) if (l[i] > lstar) lstar = l[i];
  int64_t D = 0;
  for (int32_t i = 0; i < N; ++i) {
    dead[i] = (uint8_t)((l[i] - lstar < rel_floor) || (w[i] < post_floor));
    D += dead[i];
  }
  return D;
}

/* ceil(num / den) for den > 0 in signed 128-bit */
static __int128 ceil_div128(__int128 num, __int128 den) {
  __int128 q = num / den; /* truncates toward zero */
  if (num > 0 && q * den != num) q += 1;
  return q;
}

/* n(c) = #{draws r in [0, D) : (r + U/2^32) Q / D < c}
 *      = clamp(ceil((c D 2^32 - U Q) / (Q 2^32)), 0, D)   (R18) */
static int64_t draws_below(uint64_t c, int64_t D, uint64_t Q, uint32_t U) {
  __int128 num = (__int128)c * (__int128)D * ((__int128)1 << 32) - (__int128)U * (__int128)Q;
  __int128 den = (__int128)Q * ((__int128)1 << 32);
  __int128 v = ceil_div128(num, den);
  if (v < 0) v = 0;
  if (v > D) v = D;
  return (int64_t)v;
}

int orc_resample(int32_t N, const double* e, const uint8_t* dead, uint32_t U, int32_t* donor) {
  uint64_t* C = (uint64_t*)malloc(sizeof(uint64_t) * (N > 0 ? N : 1));
  int64_t D = 0;
  uint64_t run = 0;
  for (int32_t i = 0; i < N; ++i) {
    /* survivors' ladder rungs q_i = floor(e_i 2^32); dead rungs 0 (R18) */
    uint64_t q = dead[i] ? 0u : (uint64_t)floor(e[i] * 4294967296.0);
    run += q;
    C[i] = run;
    D += dead[i];
    donor[i] = -1;
  }
  uint64_t Q = run;
  if (D == 0) { free(C); return 0; }
  if (Q == 0) { free(C); return 1; } /* every particle dead */
  /* r-th draw -> r-th dead slot in ascending order; donors ascending with multiplicity */
  int32_t* draw_donor = (int32_t*)malloc(sizeof(int32_t) * D);
  int64_t prev = 0;
  for (int32_t i = 0; i < N; ++i) {
    int64_t cur = draws_below(C[i], D, Q, U);
    for (int64_t r = prev; r < cur; ++r) draw_donor[r] = i;
    prev = cur;
  }
  int64_t r = 0;
  for (int32_t i = 0; i < N; ++i)
    if (dead[i]) donor[i] = draw_donor[r++];
  free(draw_donor);
  free(C);
  return 0;
}

int32_t orc_representative(int32_t N, const double* w) {
  int32_t best = 0;
  for (int32_t i = 1; i < N; ++i) if (w[i] > w[best]) best = i;
  return best;
}

/* ------------------------------------------------------------------------- */
/* the whole update: steps 2-11 in the paper's per-frame order          */
/* ------------------------------------------------------------------------- */

/* R35 (flag): the neighbour-particle diversity term — SVGD's kernel-gradient term with an RBF
 * kernel k(x, y) = exp(-|x - y|^2 / h) on the current-pose translations (the paper cites SVGD /
 * GN-SVGD for "preserving sample diversity through neighbor particle information", P:32, P:78,
 * and defines no term of its own).  Written as the definition: a plain double loop. */
void orc_diversity(int32_t N, const double* t, double h, double* d) {
  for (int32_t i = 0; i < N; ++i) {
    double acc[3] = {0.0, 0.0, 0.0};
    for (int32_t j = 0; j < N; ++j) {
      const double dx = t[3 * i] - t[3 * j], dy = t[3 * i + 1] - t[3 * j + 1],
                   dz = t[3 * i + 2] - t[3 * j + 2];
      const double k = exp(-(dx * dx + dy * dy + dz * dz) / h);
      acc[0] += dx * k;
      acc[1] += dy * k;
      acc[2] += dz * k;
    }
    for (int c = 0; c < 3; ++c) d[3 * i + c] = 2.0 / (h * (double)N) * acc[c];
  }
}

int orc_update(const orc_config* cfg, int32_t K, orc_map* const* maps, const double* D,
               double D_now, int32_t N, float* pose12, float* kf_pose12, int32_t kf_stride,
               double* L, const float* scan_mean3, const float* scan_cov6, int32_t S,
               uint32_t U, orc_update_out* out) {
  orc_particle_out po;
  memset(&po, 0, sizeof(po));
  po.loglik = out->loglik;
  po.grad6 = out->grad6;
  po.hess36 = out->hess36;
  po.psi6 = out->psi6;
  po.flags = out->flags;
  double* lw = (double*)malloc(sizeof(double) * (N > 0 ? N : 1));
  /* steps 2-7, repeated gn_iterations times (R12); the weighting l is the pre-update l of the
   * first iteration (R13) unless weight_after_update asks for a re-evaluation */
  const int32_t iters = cfg->gn_iterations > 0 ? cfg->gn_iterations : 1;
  /* R35: the translations the diversity term is taken at (the start of the update) */
  double* t0 = NULL;
  if (cfg->diversity_weight != 0.0) {
    t0 = (double*)malloc(sizeof(double) * 3 * (N > 0 ? N : 1));
    for (int32_t i = 0; i < N; ++i)
      for (int c = 0; c < 3; ++c) t0[3 * i + c] = (double)pose12[12 * (size_t)i + 4 * c + 3];
  }
  int rc = 0;
  for (int32_t it = 0; it < iters && rc == 0; ++it) {
    rc = orc_particles(cfg, K, maps, D, D_now, N, pose12, kf_pose12, kf_stride, scan_mean3,
                       scan_cov6, S, NULL, N, 1, &po);
    if (it == 0) memcpy(lw, out->loglik, sizeof(double) * N);
  }
  if (rc == 0 && t0) {
    /* after the GN step(s): t_i <- t_i + eta d_i in the world frame, rounded to fp32 (R35);
     * rotations, keyframe poses and weights untouched */
    double* d = (double*)malloc(sizeof(double) * 3 * (N > 0 ? N : 1));
    orc_diversity(N, t0, cfg->diversity_bandwidth, d);
    for (int32_t i = 0; i < N; ++i)
      for (int c = 0; c < 3; ++c) {
        float* tc = pose12 + 12 * (size_t)i + 4 * c + 3;
        *tc = (float)((double)*tc + cfg->diversity_weight * d[3 * i + c]);
      }
    free(d);
  }
  free(t0);
  if (rc == 0 && cfg->weight_after_update) {
    orc_particle_out pe;
    memset(&pe, 0, sizeof(pe));
    pe.loglik = lw;
    pe.grad6 = (double*)malloc(sizeof(double) * 6 * (size_t)N);
    pe.hess36 = (double*)malloc(sizeof(double) * 36 * (size_t)N);
    pe.psi6 = (double*)malloc(sizeof(double) * 6 * (size_t)N);
    pe.flags = (uint8_t*)malloc(N);
    rc = orc_particles(cfg, K, maps, D, D_now, N, pose12, kf_pose12, kf_stride, scan_mean3,
                       scan_cov6, S, NULL, N, 0, &pe);
    free(pe.grad6);
    free(pe.hess36);
    free(pe.psi6);
    free(pe.flags);
  }
  if (rc) {
    free(lw);
    return rc;
  }
  memcpy(out->loglik, lw, sizeof(double) * N);
  free(lw);
  double* e = (double*)malloc(sizeof(double) * N);
  uint8_t* dead = (uint8_t*)malloc(N);
  /* step 8: Eq.11 */
  orc_weights(N, L, out->loglik, e, out->weight, NULL, NULL);
  /* step 9: dead set */
  int64_t nd = orc_dead(N, out->loglik, out->weight, cfg->loglik_rel_floor,
                        cfg->posterior_floor, dead);
  if (out->n_dead) *out->n_dead = nd;
  for (int32_t i = 0; i < N; ++i) if (dead[i]) out->flags[i] |= 8u;
  /* step 10: respawn: clone T_t, every T_k and L of the donor (R19, R20) */
  rc = orc_resample(N, e, dead, U, out->donor);
  if (rc == 0) {
    if (cfg->clone_split) {
      /* R34: a donor with c clones shares its weight with them: all 1 + c get L - ln(1 + c) */
      int32_t* copies = (int32_t*)calloc(N > 0 ? N : 1, sizeof(int32_t));
      for (int32_t i = 0; i < N; ++i)
        if (out->donor[i] >= 0) ++copies[out->donor[i]];
      for (int32_t i = 0; i < N; ++i)
        if (copies[i] > 0) L[i] -= log((double)(1 + copies[i]));
      free(copies);
    }
    for (int32_t i = 0; i < N; ++i) {
      int32_t d = out->donor[i];
      if (d < 0) continue;
      memcpy(pose12 + 12 * (size_t)i, pose12 + 12 * (size_t)d, sizeof(float) * 12);
      memcpy(kf_pose12 + 12 * (size_t)i * kf_stride, kf_pose12 + 12 * (size_t)d * kf_stride,
             sizeof(float) * 12 * (size_t)K);
      L[i] = L[d];
    }
    /* re-normalise on the new L (step 10.7) */
    orc_weights(N, L, NULL, e, out->weight, NULL, NULL);
  }
  /* step 11: representative */
  if (out->representative) *out->representative = orc_representative(N, out->weight);
  free(e);
  free(dead);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw: "Parallel random numbers: as    */
/* easy as 1, 2, 3", SC'11): 10 rounds of two 32x32->64 multiplies + Weyl key */
/* ------------------------------------------------------------------------- */

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 8 standard normals for particle gi: two Philox blocks -> 8 uniforms in (0, 1] -> 4 Box-Muller
 * pairs, fp64 (R31) */
void orc_normals8(uint64_t seed, uint64_t frame, int64_t gi, double z[8]) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[8];
  for (uint32_t b = 0; b < 2; ++b) {
    const uint32_t ctr[4] = {b, (uint32_t)gi, (uint32_t)frame, (uint32_t)(frame >> 32)};
    orc_philox4x32_10(ctr, key, x + 4 * b);
  }
  for (int k = 0; k < 4; ++k) {
    const double u1 = ((double)x[2 * k] + 1.0) * 0x1.0p-32;
    const double u2 = ((double)x[2 * k + 1] + 1.0) * 0x1.0p-32;
    const double rr = sqrt(-2.0 * log(u1));
    const double th = 2.0 * M_PI * u2;
    z[2 * k] = rr * cos(th);
    z[2 * k + 1] = rr * sin(th);
  }
}

int orc_predict(int32_t N, float* pose12, const float dT12[12], const double cov36[36],
                uint64_t seed, uint64_t frame, int64_t gbase, double vertical_sigma) {
  /* delta ~ N(0, cov) as L z with cov = L L^T (Eq.1: "random noise in the tangent space") */
  double Lc[36];
  int zero = 1;
  for (int k = 0; k < 36; ++k) zero &= (cov36[k] == 0.0);
  if (zero) {
    memset(Lc, 0, sizeof(Lc));
  } else if (cholesky(6, cov36, Lc)) {
    return 1;
  }
  double dT[12];
  for (int k = 0; k < 12; ++k) dT[k] = (double)dT12[k];
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < N; ++i) {
    double z[8], delta[6], T[12], TdT[12];
    orc_normals8(seed, frame, gbase + i, z);
    for (int a = 0; a < 6; ++a) {
      double s = 0.0;
      for (int b = 0; b <= a; ++b) s += Lc[6 * a + b] * z[b];
      delta[a] = s;
    }
    float* P = pose12 + 12 * (size_t)i;
    for (int k = 0; k < 12; ++k) T[k] = (double)P[k];
    orc_compose(T, dT, TdT);
    /* T_{t-1} dT in fp64, then the right-applied exp with re-orthonormalisation (R30) */
    float tmp[12];
    for (int k = 0; k < 12; ++k) tmp[k] = 0.f;
    {
      double E[12], TE[12];
      orc_se3_exp(delta, E);
      orc_compose(TdT, E, TE);
      double R[9], RtR[9], M[9], Rn[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) R[3 * a + b] = TE[4 * a + b];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          double s = 0.0;
          for (int c = 0; c < 3; ++c) s += R[3 * c + a] * R[3 * c + b];
          RtR[3 * a + b] = s;
        }
      for (int k = 0; k < 9; ++k) M[k] = ((k % 4 == 0) ? 3.0 : 0.0) - RtR[k];
      mat3_mul(R, M, Rn);
      for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) tmp[4 * a + b] = (float)(0.5 * Rn[3 * a + b]);
        double ta = TE[4 * a + 3];
        if (a == 2) ta += vertical_sigma * z[6]; /* elevator: world-frame vertical walk */
        tmp[4 * a + 3] = (float)ta;
      }
    }
    memcpy(P, tmp, sizeof(tmp));
  }
  return 0;
}

double orc_overlap(const orc_map* m, const float* mean3, int32_t S, const float rel32[12]) {
  if (S <= 0) return 0.0;
  int64_t hit = 0;
  for (int32_t j = 0; j < S; ++j) {  /* occupancy of the containing voxel, whatever the rule */
    float q[3];
    key_transform(rel32, mean3 + 3 * j, q);
    hit += (cell_correspond(m, q) >= 0);
  }
  return (double)hit / (double)S;
}
