/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A deliberately plain CPU implementation of what the hot path computes,
 * written from the paper in its order and notation.  fp64 throughout,
 * compiled with -O2 -ffp-contract=off (no FMA contraction).  No blocking,
 * fusion or reordering beyond what each definition states.
 *
 *   P:L93-97   Eq. 7   GLL points xi_i, Legendre polynomials L_N, cardinal basis l_i
 *   P:L97-99   Eq. 8   tensor-product nodal basis u_ijk
 *   P:L101-105 Eq. 9   a(u,v) = sum_e v^T D^T G^e D u  (A^e = D^T G^e D)
 *   P:L107-111 Eq. 10  w_L = Q Q^T A_L u_L, Q^T Boolean gather, Q scatter
 *   P:L204-229 Alg. 1  gather-scatter split by processing element
 *   P:L257     sec. 4  Jacobi-preconditioned CG
 *
 * Readings where the paper is silent or garbled (Q1..Q22) are in DESIGN.md.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_PI 3.14159265358979323846

struct oracle_ctx {
  oracle_mesh m;
  int N, n, nranks, fully_periodic;
  int64_t E, n3, nslots, nglob;
  double *xi, *w, *D;          /* GLL rule and derivative matrix */
  double *X, *Y, *Z;           /* node coordinates per slot */
  double *G, *B;               /* geometric factors [E][6][n3], mass [E][n3] */
  double *dinv, *c;            /* Jacobi inverse diagonal, c = 1/mult */
  int64_t *gid;                /* global number per slot */
  int32_t *mult;               /* multiplicity per slot */
  uint8_t *mask;               /* 1 = Dirichlet slot */
  int32_t *rank_elem;          /* owning rank per element */
  int64_t *gs_off, *gs_slot;   /* slots of each gid, ascending (CSR) */
};

/* ------------------------------------------------------------------ */
/* Eq. 7: Legendre polynomial L_N and derivative by the three-term     */
/* recurrence (k+1) L_{k+1} = (2k+1) x L_k - k L_{k-1} and             */
/* L'_{k+1} = L'_{k-1} + (2k+1) L_k.                                   */
int oracle_legendre(int N, double x, double* L, double* dL) {
  if (N < 0) return -1;
  if (N == 0) { *L = 1.0; *dL = 0.0; return 0; }
  double Lm = 1.0, Lc = x, dLm = 0.0, dLc = 1.0;
  for (int k = 1; k < N; k++) {
    double Lp = ((2.0 * k + 1.0) * x * Lc - k * Lm) / (k + 1.0);
    double dLp = dLm + (2.0 * k + 1.0) * Lc;
    Lm = Lc; Lc = Lp;
    dLm = dLc; dLc = dLp;
  }
  *L = Lc; *dL = dLc;
  return 0;
}

/* Eq. 7: GLL points are the roots of (1 - xi^2) L_N'(xi).  Interior roots
   by Newton on L_N' from -cos(pi i/N) (reading Q1: seed, tolerance 1e-15,
   50 iterations), L_N'' from Legendre's equation; symmetrised.
   Weights w_i = 2 / (N (N+1) L_N(xi_i)^2). */
int oracle_gll(int N, double* xi, double* w) {
  if (N < 1) return -1;
  xi[0] = -1.0;
  xi[N] = 1.0;
  for (int i = 1; i < N; i++) {
    double x = -cos(ORACLE_PI * i / N);
    for (int it = 0; it < 50; it++) {
      double L, dL;
      oracle_legendre(N, x, &L, &dL);
      double d2L = (2.0 * x * dL - N * (N + 1.0) * L) / (1.0 - x * x);
      double dx = dL / d2L;
      x -= dx;
      if (fabs(dx) < 1e-15) break;
    }
    xi[i] = x;
  }
  for (int i = 0; i <= N / 2; i++) {
    double s = 0.5 * (xi[N - i] - xi[i]);
    xi[i] = -s;
    xi[N - i] = s;
  }
  if (N % 2 == 0) xi[N / 2] = 0.0;
  for (int i = 0; i <= N; i++) {
    double L, dL;
    oracle_legendre(N, xi[i], &L, &dL);
    w[i] = 2.0 / (N * (N + 1.0) * L * L);
  }
  return 0;
}

/* P:L105 "D the local derivatives of the operand at the GLL points":
   D_ij = l_j'(xi_i) = L_N(xi_i) / (L_N(xi_j) (xi_i - xi_j)) for i != j,
   D_ii = -sum_{j != i} D_ij (reading Q2, negative-sum diagonal). */
int oracle_deriv(int N, const double* xi, double* D) {
  if (N < 1) return -1;
  int n = N + 1;
  double* LN = (double*)malloc(sizeof(double) * n);
  if (!LN) return -5;
  for (int i = 0; i < n; i++) {
    double dL;
    oracle_legendre(N, xi[i], &LN[i], &dL);
  }
  for (int i = 0; i < n; i++) {
    double s = 0.0;
    for (int j = 0; j < n; j++) {
      if (j == i) continue;
      D[i * n + j] = LN[i] / (LN[j] * (xi[i] - xi[j]));
      s += D[i * n + j];
    }
    D[i * n + i] = -s;
  }
  free(LN);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Eq. 9 per element, as plain loops:                                  */
/*   ur = D_r u, us = D_s u, ut = D_t u                                 */
/*   w_a = sum_b G_ab u_b           (G symmetric, 6 stored factors)     */
/*   w   = D_r^T w_r + D_s^T w_s + D_t^T w_t                            */
int oracle_ax_raw(int64_t E, int N, const double* D, const double* G,
                  const double* u, double* w) {
  if (E < 0 || N < 1) return -1;
  const int n = N + 1;
  const int64_t n3 = (int64_t)n * n * n;
  int err = 0;
#pragma omp parallel
  {
    double* ur = (double*)malloc(sizeof(double) * 3 * n3);
    if (!ur) {
#pragma omp atomic write
      err = -5;
    }
#pragma omp for schedule(static)
    for (int64_t e = 0; e < E; e++) {
      if (!ur) continue;
      double* us = ur + n3;
      double* ut = us + n3;
      const double* ue = u + e * n3;
      const double* Ge = G + e * 6 * n3;
      double* we = w + e * n3;
      for (int k = 0; k < n; k++)
        for (int j = 0; j < n; j++)
          for (int i = 0; i < n; i++) {
            int64_t p = i + n * j + n * n * k;
            double r = 0.0, s = 0.0, t = 0.0;
            for (int m = 0; m < n; m++) {
              r += D[i * n + m] * ue[m + n * j + n * n * k];
              s += D[j * n + m] * ue[i + n * m + n * n * k];
              t += D[k * n + m] * ue[i + n * j + n * n * m];
            }
            const double grr = Ge[0 * n3 + p], gss = Ge[1 * n3 + p], gtt = Ge[2 * n3 + p];
            const double grs = Ge[3 * n3 + p], grt = Ge[4 * n3 + p], gst = Ge[5 * n3 + p];
            ur[p] = grr * r + grs * s + grt * t;
            us[p] = grs * r + gss * s + gst * t;
            ut[p] = grt * r + gst * s + gtt * t;
          }
      for (int k = 0; k < n; k++)
        for (int j = 0; j < n; j++)
          for (int i = 0; i < n; i++) {
            double a = 0.0, b = 0.0, cc = 0.0;
            for (int m = 0; m < n; m++) {
              a += D[m * n + i] * ur[m + n * j + n * n * k];
              b += D[m * n + j] * us[i + n * m + n * n * k];
              cc += D[m * n + k] * ut[i + n * j + n * n * m];
            }
            we[i + n * j + n * n * k] = a + b + cc;
          }
    }
    free(ur);
  }
  return err;
}

/* Diagonal of A^e = D^T G D at point (i,j,k) (reading Q14):
   sum_l D_li^2 G_rr(ljk) + sum_l D_lj^2 G_ss(ilk) + sum_l D_lk^2 G_tt(ijl)
   + 2 (G_rs D_ii D_jj + G_rt D_ii D_kk + G_st D_jj D_kk)(ijk). */
int oracle_diag_raw(int64_t E, int N, const double* D, const double* G, double* d) {
  if (E < 0 || N < 1) return -1;
  const int n = N + 1;
  const int64_t n3 = (int64_t)n * n * n;
  for (int64_t e = 0; e < E; e++) {
    const double* Ge = G + e * 6 * n3;
    for (int k = 0; k < n; k++)
      for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++) {
          int64_t p = i + n * j + n * n * k;
          double s = 0.0;
          for (int l = 0; l < n; l++)
            s += D[l * n + i] * D[l * n + i] * Ge[0 * n3 + l + n * j + n * n * k];
          for (int l = 0; l < n; l++)
            s += D[l * n + j] * D[l * n + j] * Ge[1 * n3 + i + n * l + n * n * k];
          for (int l = 0; l < n; l++)
            s += D[l * n + k] * D[l * n + k] * Ge[2 * n3 + i + n * j + n * n * l];
          s += 2.0 * (Ge[3 * n3 + p] * D[i * n + i] * D[j * n + j] +
                      Ge[4 * n3 + p] * D[i * n + i] * D[k * n + k] +
                      Ge[5 * n3 + p] * D[j * n + j] * D[k * n + k]);
          d[e * n3 + p] = s;
        }
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* node coordinates (reading Q4): reference lattice, optional          */
/* sinusoidal map after rescaling the box to (0, 2 pi)^3.               */
static void node_xyz(const oracle_mesh* m, const double* xi, int64_t ex, int64_t ey,
                     int64_t ez, int i, int j, int k, double* x, double* y, double* z) {
  double hx = (m->x1 - m->x0) / m->ex;
  double hy = (m->y1 - m->y0) / m->ey;
  double hz = (m->z1 - m->z0) / m->ez;
  double X = m->x0 + hx * (ex + 0.5 * (xi[i] + 1.0));
  double Y = m->y0 + hy * (ey + 0.5 * (xi[j] + 1.0));
  double Z = m->z0 + hz * (ez + 0.5 * (xi[k] + 1.0));
  if (m->deform) {
    double Xh = 2.0 * ORACLE_PI * (X - m->x0) / (m->x1 - m->x0);
    double Yh = 2.0 * ORACLE_PI * (Y - m->y0) / (m->y1 - m->y0);
    double Zh = 2.0 * ORACLE_PI * (Z - m->z0) / (m->z1 - m->z0);
    double dlt = m->deform_amp * sin(Xh) * sin(Yh) * sin(Zh);
    X += dlt * (m->x1 - m->x0) / (2.0 * ORACLE_PI);
    Y += dlt * (m->y1 - m->y0) / (2.0 * ORACLE_PI);
    Z += dlt * (m->z1 - m->z0) / (2.0 * ORACLE_PI);
  }
  *x = X; *y = Y; *z = Z;
}

/* P:L105 geometric factors (reading Q5): x_r etc. through D, J = det,
   inverse metric by cofactors / J, G_ab = J w_i w_j w_k sum_m r_a,m r_b,m,
   B = J w_i w_j w_k. */
static int geometry(oracle_ctx* c) {
  const int n = c->n;
  const int64_t n3 = c->n3;
  const double* D = c->D;
  for (int64_t e = 0; e < c->E; e++) {
    const double* xs[3] = {c->X + e * n3, c->Y + e * n3, c->Z + e * n3};
    double* Ge = c->G + e * 6 * n3;
    for (int k = 0; k < n; k++)
      for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++) {
          int64_t p = i + n * j + n * n * k;
          double M[3][3]; /* M[a][b] = d x_a / d r_b */
          for (int a = 0; a < 3; a++) {
            double dr = 0.0, ds = 0.0, dt = 0.0;
            for (int q = 0; q < n; q++) {
              dr += D[i * n + q] * xs[a][q + n * j + n * n * k];
              ds += D[j * n + q] * xs[a][i + n * q + n * n * k];
              dt += D[k * n + q] * xs[a][i + n * j + n * n * q];
            }
            M[a][0] = dr; M[a][1] = ds; M[a][2] = dt;
          }
          double J = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                     M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                     M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
          if (!(J > 0.0)) return -2;
          double R[3][3]; /* R[b][a] = d r_b / d x_a */
          R[0][0] = (M[1][1] * M[2][2] - M[1][2] * M[2][1]) / J;
          R[0][1] = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) / J;
          R[0][2] = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) / J;
          R[1][0] = (M[1][2] * M[2][0] - M[1][0] * M[2][2]) / J;
          R[1][1] = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) / J;
          R[1][2] = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) / J;
          R[2][0] = (M[1][0] * M[2][1] - M[1][1] * M[2][0]) / J;
          R[2][1] = (M[0][1] * M[2][0] - M[0][0] * M[2][1]) / J;
          R[2][2] = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) / J;
          double wq = c->w[i] * c->w[j] * c->w[k];
          double Jw = J * wq;
          const int ab[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
          for (int f = 0; f < 6; f++) {
            int a = ab[f][0], b = ab[f][1];
            double s = 0.0;
            for (int q = 0; q < 3; q++) s += R[a][q] * R[b][q];
            Ge[f * n3 + p] = Jw * s;
          }
          c->B[e * n3 + p] = Jw;
        }
  }
  return 0;
}

/* P:L107 "Each degree of freedom ... is assigned a unique global number"
   (reading Q6): lattice I = ex N + i (mod Ex N if periodic), likewise J, K;
   gid = I + Nx (J + Ny K). Mask (reading Q8): lattice index at a
   non-periodic box face. */
static void numbering(oracle_ctx* c) {
  const oracle_mesh* m = &c->m;
  const int N = c->N, n = c->n;
  int64_t Lx = (int64_t)m->ex * N, Ly = (int64_t)m->ey * N, Lz = (int64_t)m->ez * N;
  int64_t Nx = Lx + (m->periodic[0] ? 0 : 1);
  int64_t Ny = Ly + (m->periodic[1] ? 0 : 1);
  int64_t Nz = Lz + (m->periodic[2] ? 0 : 1);
  c->nglob = Nx * Ny * Nz;
  for (int64_t e = 0; e < c->E; e++) {
    int64_t ex = e % m->ex, ey = (e / m->ex) % m->ey, ez = e / ((int64_t)m->ex * m->ey);
    for (int k = 0; k < n; k++)
      for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++) {
          int64_t I = ex * N + i, J = ey * N + j, K = ez * N + k;
          int msk = 0;
          if (!m->periodic[0] && (I == 0 || I == Lx)) msk = 1;
          if (!m->periodic[1] && (J == 0 || J == Ly)) msk = 1;
          if (!m->periodic[2] && (K == 0 || K == Lz)) msk = 1;
          if (m->periodic[0]) I %= Lx;
          if (m->periodic[1]) J %= Ly;
          if (m->periodic[2]) K %= Lz;
          int64_t l = e * c->n3 + i + n * j + (int64_t)n * n * k;
          c->gid[l] = I + Nx * (J + Ny * K);
          c->mask[l] = (uint8_t)msk;
        }
  }
}

int oracle_setup(const oracle_mesh* m, int N, int nranks, oracle_ctx** out) {
  *out = NULL;
  if (!m || N < 1 || N > 11 || m->ex < 1 || m->ey < 1 || m->ez < 1) return -1;
  for (int a = 0; a < 3; a++) {
    int ea = a == 0 ? m->ex : (a == 1 ? m->ey : m->ez);
    if (m->periodic[a] && ea < 2) return -1; /* reading Q7 */
  }
  if (!(m->x1 > m->x0) || !(m->y1 > m->y0) || !(m->z1 > m->z0)) return -1;
  int64_t E = (int64_t)m->ex * m->ey * m->ez;
  if (nranks < 1 || nranks > E) return -1;

  oracle_ctx* c = (oracle_ctx*)calloc(1, sizeof(oracle_ctx));
  if (!c) return -5;
  c->m = *m;
  c->N = N;
  c->n = N + 1;
  c->nranks = nranks;
  c->E = E;
  c->n3 = (int64_t)c->n * c->n * c->n;
  c->nslots = E * c->n3;
  c->fully_periodic = m->periodic[0] && m->periodic[1] && m->periodic[2];
  int64_t ns = c->nslots;
  c->xi = (double*)malloc(sizeof(double) * c->n);
  c->w = (double*)malloc(sizeof(double) * c->n);
  c->D = (double*)malloc(sizeof(double) * c->n * c->n);
  c->X = (double*)malloc(sizeof(double) * ns);
  c->Y = (double*)malloc(sizeof(double) * ns);
  c->Z = (double*)malloc(sizeof(double) * ns);
  c->G = (double*)malloc(sizeof(double) * 6 * ns);
  c->B = (double*)malloc(sizeof(double) * ns);
  c->dinv = (double*)malloc(sizeof(double) * ns);
  c->c = (double*)malloc(sizeof(double) * ns);
  c->gid = (int64_t*)malloc(sizeof(int64_t) * ns);
  c->mult = (int32_t*)calloc(ns, sizeof(int32_t));
  c->mask = (uint8_t*)malloc(ns);
  c->rank_elem = (int32_t*)malloc(sizeof(int32_t) * E);
  c->gs_slot = (int64_t*)malloc(sizeof(int64_t) * ns);
  if (!c->xi || !c->w || !c->D || !c->X || !c->Y || !c->Z || !c->G || !c->B || !c->dinv ||
      !c->c || !c->gid || !c->mult || !c->mask || !c->rank_elem || !c->gs_slot) {
    oracle_free(c);
    return -5;
  }
  oracle_gll(N, c->xi, c->w);
  oracle_deriv(N, c->xi, c->D);

  /* lexicographic element partition: rank r owns [r E / P, (r+1) E / P) */
  for (int r = 0; r < nranks; r++) {
    int64_t lo = (int64_t)r * E / nranks, hi = (int64_t)(r + 1) * E / nranks;
    for (int64_t e = lo; e < hi; e++) c->rank_elem[e] = r;
  }

  for (int64_t e = 0; e < E; e++) {
    int64_t ex = e % m->ex, ey = (e / m->ex) % m->ey, ez = e / ((int64_t)m->ex * m->ey);
    for (int k = 0; k < c->n; k++)
      for (int j = 0; j < c->n; j++)
        for (int i = 0; i < c->n; i++) {
          int64_t l = e * c->n3 + i + c->n * j + (int64_t)c->n * c->n * k;
          node_xyz(m, c->xi, ex, ey, ez, i, j, k, &c->X[l], &c->Y[l], &c->Z[l]);
        }
  }
  int st = geometry(c);
  if (st) { oracle_free(c); return st; }
  numbering(c);

  /* slots of each gid in ascending slot order (counting sort) */
  c->gs_off = (int64_t*)calloc(c->nglob + 1, sizeof(int64_t));
  if (!c->gs_off) { oracle_free(c); return -5; }
  for (int64_t l = 0; l < ns; l++) c->gs_off[c->gid[l] + 1]++;
  for (int64_t g = 0; g < c->nglob; g++) c->gs_off[g + 1] += c->gs_off[g];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * c->nglob);
    if (!fill) { oracle_free(c); return -5; }
    memcpy(fill, c->gs_off, sizeof(int64_t) * c->nglob);
    for (int64_t l = 0; l < ns; l++) c->gs_slot[fill[c->gid[l]]++] = l;
    free(fill);
  }
  for (int64_t l = 0; l < ns; l++) {
    int64_t g = c->gid[l];
    c->mult[l] = (int32_t)(c->gs_off[g + 1] - c->gs_off[g]);
    c->c[l] = 1.0 / c->mult[l];
  }

  /* Jacobi: d = QQ^T diag(A_L), dinv = 0 on masked slots (reading Q14) */
  oracle_diag_raw(E, N, c->D, c->G, c->dinv);
  oracle_gs(c, c->dinv);
  for (int64_t l = 0; l < ns; l++) c->dinv[l] = c->mask[l] ? 0.0 : 1.0 / c->dinv[l];
  *out = c;
  return 0;
}

void oracle_free(oracle_ctx* c) {
  if (!c) return;
  free(c->xi); free(c->w); free(c->D);
  free(c->X); free(c->Y); free(c->Z);
  free(c->G); free(c->B); free(c->dinv); free(c->c);
  free(c->gid); free(c->mult); free(c->mask); free(c->rank_elem);
  free(c->gs_off); free(c->gs_slot);
  free(c);
}

int oracle_sizes(const oracle_ctx* c, int64_t* nslots, int64_t* E, int64_t* nglob) {
  if (!c) return -1;
  if (nslots) *nslots = c->nslots;
  if (E) *E = c->E;
  if (nglob) *nglob = c->nglob;
  return 0;
}

int oracle_get(const oracle_ctx* c, int which, double* dst) {
  if (!c || !dst) return -1;
  int64_t ns = c->nslots;
  switch (which) {
    case 0: memcpy(dst, c->xi, sizeof(double) * c->n); break;
    case 1: memcpy(dst, c->w, sizeof(double) * c->n); break;
    case 2: memcpy(dst, c->D, sizeof(double) * c->n * c->n); break;
    case 3: memcpy(dst, c->X, sizeof(double) * ns); break;
    case 4: memcpy(dst, c->Y, sizeof(double) * ns); break;
    case 5: memcpy(dst, c->Z, sizeof(double) * ns); break;
    case 6: memcpy(dst, c->G, sizeof(double) * 6 * ns); break;
    case 7: memcpy(dst, c->B, sizeof(double) * ns); break;
    case 8: memcpy(dst, c->dinv, sizeof(double) * ns); break;
    case 9: memcpy(dst, c->c, sizeof(double) * ns); break;
    default: return -1;
  }
  return 0;
}

int oracle_get_int(const oracle_ctx* c, int which, int64_t* dst) {
  if (!c || !dst) return -1;
  for (int64_t l = 0; l < c->nslots; l++) {
    switch (which) {
      case 0: dst[l] = c->gid[l]; break;
      case 1: dst[l] = c->mult[l]; break;
      case 2: dst[l] = c->mask[l]; break;
      case 3: dst[l] = c->rank_elem[l / c->n3]; break;
      default: return -1;
    }
  }
  return 0;
}

int oracle_ax(const oracle_ctx* c, const double* u, double* w) {
  if (!c) return -1;
  return oracle_ax_raw(c->E, c->N, c->D, c->G, u, w);
}

/* Eq. 10 + Alg. 1 (reading Q10): for each gid the slots are visited in
   ascending slot order; each processing element first forms its partial sum
   (Alg. 1 lines 6/8 "gather"), the partials are added in ascending rank
   order, and the total is scattered to every slot (lines 9/18). Ranks own
   contiguous element ranges, so ascending slots visit ranks in order. */
int oracle_gs(const oracle_ctx* c, double* u) {
  if (!c) return -1;
  for (int64_t g = 0; g < c->nglob; g++) {
    int64_t lo = c->gs_off[g], hi = c->gs_off[g + 1];
    if (hi - lo < 2) continue;
    int64_t s0 = c->gs_slot[lo];
    int cur = c->rank_elem[s0 / c->n3];
    double part = u[s0], total = 0.0;
    int have_total = 0;
    for (int64_t t = lo + 1; t < hi; t++) {
      int64_t s = c->gs_slot[t];
      int r = c->rank_elem[s / c->n3];
      if (r == cur) {
        part += u[s];
      } else {
        total = have_total ? total + part : part;
        have_total = 1;
        cur = r;
        part = u[s];
      }
    }
    total = have_total ? total + part : part;
    for (int64_t t = lo; t < hi; t++) u[c->gs_slot[t]] = total;
  }
  return 0;
}

int oracle_mask_apply(const oracle_ctx* c, double* u) {
  if (!c) return -1;
  for (int64_t l = 0; l < c->nslots; l++)
    if (c->mask[l]) u[l] = 0.0;
  return 0;
}

/* P:L111 "w_L = QQ^T A_L u_L", then the Dirichlet mask (reading Q8). */
int oracle_apply(const oracle_ctx* c, const double* u, double* w) {
  int st = oracle_ax(c, u, w);
  if (st) return st;
  oracle_gs(c, w);
  return oracle_mask_apply(c, w);
}

/* <a,b>_c = sum_l c_l a_l b_l, serial in slot order (c = 1/mult). */
double oracle_dot_c(const oracle_ctx* c, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t l = 0; l < c->nslots; l++) s += c->c[l] * a[l] * b[l];
  return s;
}

/* Eq. 6 right-hand side with collocated quadrature (reading Q12):
   b = mask(QQ^T (B .* f)); fully periodic: remove the unique-DOF mean
   (reading Q13) so that b lies in range(A). */
int oracle_rhs(const oracle_ctx* c, const double* f, double* b) {
  if (!c) return -1;
  for (int64_t l = 0; l < c->nslots; l++) b[l] = c->B[l] * f[l];
  oracle_gs(c, b);
  oracle_mask_apply(c, b);
  if (c->fully_periodic) {
    double sb = 0.0, sc = 0.0;
    for (int64_t l = 0; l < c->nslots; l++) {
      sb += c->c[l] * b[l];
      sc += c->c[l];
    }
    double mean = sb / sc;
    for (int64_t l = 0; l < c->nslots; l++) b[l] -= mean;
  }
  return 0;
}

/* NEXT-2: the Helmholtz operator of the velocity solves (P:L257
   "followed by a Helmholtz equation for each velocity components"; S:L294-302
   "h1*(stiffness action) + h2*(mass action), then gather-scatter add"), with
   the Dirichlet mask as for the Poisson operator (reading Q8):
   w = mask(QQ^T (h1 A_L u + h2 B_L u)). */
int oracle_helm_apply(const oracle_ctx* c, double h1, double h2, const double* u, double* w) {
  int st = oracle_ax(c, u, w);
  if (st) return st;
  for (int64_t l = 0; l < c->nslots; l++) w[l] = h1 * w[l] + h2 * (c->B[l] * u[l]);
  oracle_gs(c, w);
  return oracle_mask_apply(c, w);
}

/* b = mask(QQ^T (B .* f)) without the periodic projection (reading Q12): the
   right-hand side of the Helmholtz system, nonsingular for h2 > 0. */
int oracle_rhs_mass(const oracle_ctx* c, const double* f, double* b) {
  if (!c) return -1;
  for (int64_t l = 0; l < c->nslots; l++) b[l] = c->B[l] * f[l];
  oracle_gs(c, b);
  return oracle_mask_apply(c, b);
}

/* Jacobi for the Helmholtz operator (reading Q14 applied to h1 A + h2 B):
   d = QQ^T (h1 diag(A_L) + h2 B_L), dinv = 0 on masked slots, else 1/d. */
int oracle_helm_dinv(const oracle_ctx* c, double h1, double h2, double* dinv) {
  if (!c) return -1;
  oracle_diag_raw(c->E, c->N, c->D, c->G, dinv);
  for (int64_t l = 0; l < c->nslots; l++) dinv[l] = h1 * dinv[l] + h2 * c->B[l];
  oracle_gs(c, dinv);
  for (int64_t l = 0; l < c->nslots; l++) dinv[l] = c->mask[l] ? 0.0 : 1.0 / dinv[l];
  return 0;
}

/* operator of the PCG: helm = 0 -> Poisson (oracle_apply), 1 -> Helmholtz */
static int op_apply(const oracle_ctx* c, int helm, double h1, double h2, const double* u, double* w) {
  return helm ? oracle_helm_apply(c, h1, h2, u, w) : oracle_apply(c, u, w);
}

/* P:L257 "preconditioned Conjugate Gradient (CG) ... with a block Jacobi
   preconditioner", written step by step (readings Q14-Q17):
   x0 = 0; r = b; z = M^-1 r; p = z; rho = <r,z>_c
   for k = 1..maxit: w = A p; sigma = <p,w>_c; alpha = rho/sigma;
     x += alpha p; r -= alpha w; gamma = <r,r>_c; stop if sqrt(gamma) <= tol;
     z = M^-1 r; rho' = <r,z>_c; beta = rho'/rho; rho = rho'; p = z + beta p.
   hist[k] = sqrt(gamma) after iteration k (hist[0] = ||b||_c). */
static int pcg_core(const oracle_ctx* c, int helm, double h1, double h2, const double* dinv,
                    const double* b, double* x, double tol, int maxit, int* iters,
                    double* res_final, double* res_true, double* hist) {
  if (!c || maxit < 0) return -1;
  int64_t ns = c->nslots;
  double* r = (double*)malloc(sizeof(double) * ns);
  double* z = (double*)malloc(sizeof(double) * ns);
  double* p = (double*)malloc(sizeof(double) * ns);
  double* w = (double*)malloc(sizeof(double) * ns);
  if (!r || !z || !p || !w) { free(r); free(z); free(p); free(w); return -5; }
  int status = 1, k = 0;
  for (int64_t l = 0; l < ns; l++) {
    x[l] = 0.0;
    r[l] = b[l];
    z[l] = dinv[l] * r[l];
    p[l] = z[l];
  }
  double rho = oracle_dot_c(c, r, z);
  double gamma = oracle_dot_c(c, r, r);
  if (hist) hist[0] = sqrt(gamma);
  if (sqrt(gamma) <= tol) status = 0;
  while (status == 1 && k < maxit) {
    k++;
    op_apply(c, helm, h1, h2, p, w);
    double sigma = oracle_dot_c(c, p, w);
    if (!(sigma > 0.0)) { status = -6; break; }
    double alpha = rho / sigma;
    for (int64_t l = 0; l < ns; l++) {
      x[l] += alpha * p[l];
      r[l] -= alpha * w[l];
    }
    gamma = oracle_dot_c(c, r, r);
    if (hist) hist[k] = sqrt(gamma);
    if (sqrt(gamma) <= tol) { status = 0; break; }
    for (int64_t l = 0; l < ns; l++) z[l] = dinv[l] * r[l];
    double rho_new = oracle_dot_c(c, r, z);
    double beta = rho_new / rho;
    rho = rho_new;
    for (int64_t l = 0; l < ns; l++) p[l] = z[l] + beta * p[l];
  }
  if (iters) *iters = k;
  if (res_final) *res_final = sqrt(gamma);
  if (res_true) {
    op_apply(c, helm, h1, h2, x, w);
    for (int64_t l = 0; l < ns; l++) w[l] = b[l] - w[l];
    *res_true = sqrt(oracle_dot_c(c, w, w));
  }
  free(r); free(z); free(p); free(w);
  return status;
}

int oracle_pcg(const oracle_ctx* c, const double* b, double* x, double tol, int maxit,
               int* iters, double* res_final, double* res_true, double* hist) {
  if (!c) return -1;
  return pcg_core(c, 0, 0.0, 0.0, c->dinv, b, x, tol, maxit, iters, res_final, res_true, hist);
}

/* the same PCG on h1 A + h2 B with its own Jacobi diagonal (oracle_helm_dinv) */
int oracle_helm_pcg(const oracle_ctx* c, double h1, double h2, const double* b, double* x,
                    double tol, int maxit, int* iters, double* res_final, double* res_true,
                    double* hist) {
  if (!c) return -1;
  double* dinv = (double*)malloc(sizeof(double) * c->nslots);
  if (!dinv) return -5;
  oracle_helm_dinv(c, h1, h2, dinv);
  int st = pcg_core(c, 1, h1, h2, dinv, b, x, tol, maxit, iters, res_final, res_true, hist);
  free(dinv);
  return st;
}

/* Single-reduction PCG (Chronopoulos & Gear 1989; SURVEY 8(f) lower-ranked
   variant after NEXT-1..4, "addressed with non-blocking or pipelined
   Krylov solvers"), with the Jacobi preconditioner, reading Q34:
     x0 = 0, r0 = b, u0 = M r0, w0 = A u0, gamma0 = <r0,u0>_c, delta0 = <w0,u0>_c,
     eps0 = <r0,r0>_c; stop at once if sqrt(eps0) <= tol; alpha0 = gamma0/delta0, beta0 = 0;
     for i = 0, 1, ...:
       p_i = u_i + beta_i p_{i-1};  s_i = w_i + beta_i s_{i-1}   (s_i = A p_i)
       x_{i+1} = x_i + alpha_i p_i;  r_{i+1} = r_i - alpha_i s_i
       u_{i+1} = M r_{i+1};  w_{i+1} = A u_{i+1}
       gamma, delta, eps = <r,u>_c, <w,u>_c, <r,r>_c       (ONE global reduction)
       stop if sqrt(eps) <= tol (iterations = i + 1)
       beta_{i+1} = gamma_{i+1}/gamma_i;
       alpha_{i+1} = gamma_{i+1} / (delta_{i+1} - beta_{i+1} gamma_{i+1} / alpha_i)
   The iterates equal PCG's in exact arithmetic; hist[k] = sqrt(eps) after k updates. */
int oracle_cgcg(const oracle_ctx* c, const double* b, double* x, double tol, int maxit,
                int* iters, double* res_final, double* res_true, double* hist) {
  if (!c || maxit < 0) return -1;
  const int64_t ns = c->nslots;
  double* r = (double*)malloc(sizeof(double) * ns);
  double* u = (double*)malloc(sizeof(double) * ns);
  double* w = (double*)malloc(sizeof(double) * ns);
  double* p = (double*)calloc(ns, sizeof(double));
  double* s = (double*)calloc(ns, sizeof(double));
  if (!r || !u || !w || !p || !s) { free(r); free(u); free(w); free(p); free(s); return -5; }
  int status = 1, k = 0;
  for (int64_t l = 0; l < ns; l++) {
    x[l] = 0.0;
    r[l] = b[l];
    u[l] = c->dinv[l] * r[l];
  }
  oracle_apply(c, u, w);
  double gamma = oracle_dot_c(c, r, u);
  double delta = oracle_dot_c(c, w, u);
  double eps = oracle_dot_c(c, r, r);
  if (hist) hist[0] = sqrt(eps);
  if (sqrt(eps) <= tol) status = 0;
  double alpha = 0.0, beta = 0.0;
  if (status == 1) {
    if (!(delta > 0.0)) status = -6;
    else alpha = gamma / delta;
  }
  while (status == 1 && k < maxit) {
    for (int64_t l = 0; l < ns; l++) {
      p[l] = u[l] + beta * p[l];
      s[l] = w[l] + beta * s[l];
      x[l] += alpha * p[l];
      r[l] -= alpha * s[l];
      u[l] = c->dinv[l] * r[l];
    }
    k++;
    oracle_apply(c, u, w);
    const double gamma_new = oracle_dot_c(c, r, u);
    delta = oracle_dot_c(c, w, u);
    eps = oracle_dot_c(c, r, r);
    if (hist) hist[k] = sqrt(eps);
    if (sqrt(eps) <= tol) { status = 0; break; }
    beta = gamma_new / gamma;
    const double den = delta - beta * gamma_new / alpha;
    if (!(den > 0.0)) { status = -6; break; }
    alpha = gamma_new / den;
    gamma = gamma_new;
  }
  if (iters) *iters = k;
  if (res_final) *res_final = sqrt(eps);
  if (res_true) {
    oracle_apply(c, x, w);
    for (int64_t l = 0; l < ns; l++) w[l] = b[l] - w[l];
    *res_true = sqrt(oracle_dot_c(c, w, w));
  }
  free(r); free(u); free(w); free(p); free(s);
  return status;
}

/* ------------------------------------------------------------------ */
/* NEXT-3: restarted GMRES and solution projection (Table 2) */

/* Restarted GMRES(m) with right Jacobi preconditioning (readings Q25, Q26),
   Saad's algorithm step by step: x0 given; per cycle r = b - A x, beta = ||r||_c,
   v1 = r / beta; for j = 1..m: w = A M^-1 v_j (one iteration); modified Gram-
   Schmidt h_ij = <w, v_i>_c, w -= h_ij v_i, done twice (reorthogonalisation,
   h_ij summed over both passes); h_{j+1,j} = ||w||_c; v_{j+1} = w/h;
   previous Givens rotations applied to column j, a new one zeroes h_{j+1,j};
   |g_{j+1}| is the residual norm; stop when it is <= tol or at maxit; then
   y = H^-1 g (upper triangular), x += M^-1 V y.  hist[k] = |g| after iteration
   k (hist[0] = ||b - A x0||_c).  Returns 0 converged, 1 not converged. */
/* One Arnoldi step of right-Jacobi-preconditioned GMRES (Table 2,
   reading Q25): w = A M^-1 v_j, then modified Gram-Schmidt against
   v_0..v_j applied twice (one reorthogonalisation pass, which keeps the
   basis orthogonal over long cycles), H(0:j+1, j) and v_{j+1} = w / ||w||_c.
   Returns ||w||_c.  t, w: scratch of nslots. */
static double arnoldi_step(const oracle_ctx* c, double* V, int j, int m, double* t, double* w,
                           double* H) {
  const int64_t ns = c->nslots;
  double* vj = V + (int64_t)j * ns;
  for (int64_t l = 0; l < ns; l++) t[l] = c->dinv[l] * vj[l];
  oracle_apply(c, t, w);
  for (int i = 0; i <= j; i++) H[i * m + j] = 0.0;
  for (int pass = 0; pass < 2; pass++)
    for (int i = 0; i <= j; i++) {
      const double* vi = V + (int64_t)i * ns;
      const double h = oracle_dot_c(c, w, vi);
      H[i * m + j] += h;
      for (int64_t l = 0; l < ns; l++) w[l] -= h * vi[l];
    }
  const double hn = sqrt(oracle_dot_c(c, w, w));
  H[(j + 1) * m + j] = hn;
  double* vn = V + (int64_t)(j + 1) * ns;
  for (int64_t l = 0; l < ns; l++) vn[l] = hn > 0.0 ? w[l] / hn : 0.0;
  return hn;
}

/* test access: m Arnoldi steps from v_0 = b / ||b||_c with the same step as
   oracle_gmres; V [(m+1) x nslots], H [(m+1) x m] row-major (H[i*m + j]) */
int oracle_arnoldi(const oracle_ctx* c, const double* b, int m, double* V, double* H) {
  if (!c || m < 1) return -1;
  const int64_t ns = c->nslots;
  double* w = (double*)malloc(sizeof(double) * ns);
  double* t = (double*)malloc(sizeof(double) * ns);
  if (!w || !t) { free(w); free(t); return -5; }
  for (int i = 0; i < (m + 1) * m; i++) H[i] = 0.0;
  const double beta = sqrt(oracle_dot_c(c, b, b));
  for (int64_t l = 0; l < ns; l++) V[l] = b[l] / beta;
  for (int j = 0; j < m; j++) arnoldi_step(c, V, j, m, t, w, H);
  free(w); free(t);
  return 0;
}

int oracle_gmres(const oracle_ctx* c, const double* b, double* x, double tol, int maxit,
                 int restart, int* iters, double* res_final, double* res_true, double* hist) {
  if (!c || maxit < 0 || restart < 1) return -1;
  const int64_t ns = c->nslots;
  const int m = restart;
  double* V = (double*)malloc(sizeof(double) * ns * (m + 1));
  double* w = (double*)malloc(sizeof(double) * ns);
  double* t = (double*)malloc(sizeof(double) * ns);
  double* H = (double*)calloc((size_t)(m + 1) * m, sizeof(double));   /* H[i*m + j] */
  double* cs = (double*)malloc(sizeof(double) * m);
  double* sn = (double*)malloc(sizeof(double) * m);
  double* g = (double*)malloc(sizeof(double) * (m + 1));
  double* y = (double*)malloc(sizeof(double) * m);
  if (!V || !w || !t || !H || !cs || !sn || !g || !y) {
    free(V); free(w); free(t); free(H); free(cs); free(sn); free(g); free(y);
    return -5;
  }
  int k = 0, status = 1;
  double res = 0.0;
  for (int cycle = 0;; cycle++) {
    /* r = b - A x */
    oracle_apply(c, x, w);
    for (int64_t l = 0; l < ns; l++) V[l] = b[l] - w[l];
    const double beta = sqrt(oracle_dot_c(c, V, V));
    res = beta;
    if (cycle == 0 && hist) hist[0] = beta;
    if (beta <= tol) { status = 0; break; }
    if (k >= maxit) break;
    for (int64_t l = 0; l < ns; l++) V[l] /= beta;
    for (int i = 0; i <= m; i++) g[i] = 0.0;
    g[0] = beta;
    int j = 0;
    for (; j < m && k < maxit; j++) {
      const double hn = arnoldi_step(c, V, j, m, t, w, H);
      k++;
      for (int i = 0; i < j; i++) {   /* previous rotations */
        const double a = H[i * m + j], bb = H[(i + 1) * m + j];
        H[i * m + j] = cs[i] * a + sn[i] * bb;
        H[(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
      }
      const double a = H[j * m + j], bb = H[(j + 1) * m + j];
      const double r = sqrt(a * a + bb * bb);
      cs[j] = r > 0.0 ? a / r : 1.0;
      sn[j] = r > 0.0 ? bb / r : 0.0;
      H[j * m + j] = r;
      H[(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      res = fabs(g[j + 1]);
      if (hist) hist[k] = res;
      if (res <= tol || hn == 0.0) { j++; break; }
    }
    /* y = H(0:j,0:j)^-1 g(0:j), x += M^-1 V y */
    for (int i = j - 1; i >= 0; i--) {
      double sacc = g[i];
      for (int q = i + 1; q < j; q++) sacc -= H[i * m + q] * y[q];
      y[i] = sacc / H[i * m + i];
    }
    for (int64_t l = 0; l < ns; l++) {
      double vy = 0.0;
      for (int i = 0; i < j; i++) vy += V[(int64_t)i * ns + l] * y[i];
      x[l] += c->dinv[l] * vy;
    }
    if (res <= tol) { status = 0; break; }
    if (k >= maxit) break;
  }
  if (iters) *iters = k;
  if (res_final) *res_final = res;
  if (res_true) {
    oracle_apply(c, x, w);
    for (int64_t l = 0; l < ns; l++) w[l] = b[l] - w[l];
    *res_true = sqrt(oracle_dot_c(c, w, w));
  }
  free(V); free(w); free(t); free(H); free(cs); free(sn); free(g); free(y);
  return status;
}

/* Solution projection ("projections techniques as in Nek5000 [20] ...
   storing a set of previous solutions"; Fischer 1998, ref. [20]; readings Q26):
   up to m A-orthonormal directions z_i (with A z_i stored), <z_i, A z_j>_c = d_ij. */
struct oracle_proj {
  const oracle_ctx* c;
  const oracle_schwarz* schw;   /* NULL: Jacobi GMRES; else flexible GMRES + Schwarz */
  int m, k;
  double *Z, *AZ;   /* [m][nslots] */
};

int oracle_proj_create(const oracle_ctx* c, int m, oracle_proj** out) {
  if (!c || m < 1 || !out) return -1;
  oracle_proj* p = (oracle_proj*)calloc(1, sizeof(oracle_proj));
  if (!p) return -5;
  p->c = c;
  p->m = m;
  p->Z = (double*)malloc(sizeof(double) * c->nslots * m);
  p->AZ = (double*)malloc(sizeof(double) * c->nslots * m);
  if (!p->Z || !p->AZ) { free(p->Z); free(p->AZ); free(p); return -5; }
  *out = p;
  return 0;
}

void oracle_proj_free(oracle_proj* p) {
  if (!p) return;
  free(p->Z); free(p->AZ); free(p);
}

int oracle_proj_size(const oracle_proj* p) { return p ? p->k : -1; }


/* x_bar = sum_i <z_i, b>_c z_i, b_defl = b - sum_i <z_i, b>_c A z_i (= b - A x_bar) */
int oracle_proj_project(const oracle_proj* p, const double* b, double* xbar, double* bdefl) {
  const int64_t ns = p->c->nslots;
  for (int64_t l = 0; l < ns; l++) { xbar[l] = 0.0; bdefl[l] = b[l]; }
  for (int i = 0; i < p->k; i++) {
    const double* zi = p->Z + (int64_t)i * ns;
    const double* azi = p->AZ + (int64_t)i * ns;
    const double a = oracle_dot_c(p->c, zi, b);
    for (int64_t l = 0; l < ns; l++) {
      xbar[l] += a * zi[l];
      bdefl[l] -= a * azi[l];
    }
  }
  return 0;
}

/* append x: A-orthonormalise against the stored directions (modified Gram-
   Schmidt, two passes), skip if ||z||_A < 1e-12 ||x||_A; when the space is
   full it is reset to the single most recent solution.  Returns 1 if skipped. */
int oracle_proj_update(oracle_proj* p, const double* x) {
  const oracle_ctx* c = p->c;
  const int64_t ns = c->nslots;
  if (p->k == p->m) p->k = 0;   /* reset, keep the latest */
  double* z = p->Z + (int64_t)p->k * ns;
  double* az = p->AZ + (int64_t)p->k * ns;
  for (int64_t l = 0; l < ns; l++) z[l] = x[l];
  oracle_apply(c, z, az);
  const double nx = sqrt(fabs(oracle_dot_c(c, z, az)));
  for (int pass = 0; pass < 2; pass++)
    for (int i = 0; i < p->k; i++) {
      const double* zi = p->Z + (int64_t)i * ns;
      const double* azi = p->AZ + (int64_t)i * ns;
      const double a = oracle_dot_c(c, zi, az);   /* <z_i, z>_A */
      for (int64_t l = 0; l < ns; l++) {
        z[l] -= a * zi[l];
        az[l] -= a * azi[l];
      }
    }
  const double nz = sqrt(fabs(oracle_dot_c(c, z, az)));
  if (!(nz > 1e-12 * nx)) return 1;
  for (int64_t l = 0; l < ns; l++) {
    z[l] /= nz;
    az[l] /= nz;
  }
  p->k++;
  return 0;
}

/* the pressure-solve pipeline: project, GMRES(restart) on the deflated right-
   hand side from x = 0, x = x_bar + delta, append x to the space */
int oracle_proj_solve(oracle_proj* p, const double* b, double* x, double tol, int maxit,
                      int restart, int* iters, double* res_final) {
  const int64_t ns = p->c->nslots;
  double* xb = (double*)malloc(sizeof(double) * ns);
  double* bd = (double*)malloc(sizeof(double) * ns);
  if (!xb || !bd) { free(xb); free(bd); return -5; }
  oracle_proj_project(p, b, xb, bd);
  for (int64_t l = 0; l < ns; l++) x[l] = 0.0;
  int st = p->schw ? oracle_schwarz_gmres(p->schw, bd, x, tol, maxit, restart, iters,
                                          res_final, NULL, NULL)
                  : oracle_gmres(p->c, bd, x, tol, maxit, restart, iters, res_final, NULL, NULL);
  for (int64_t l = 0; l < ns; l++) x[l] += xb[l];
  if (st >= 0) oracle_proj_update(p, x);
  free(xb); free(bd);
  return st;
}

/* test access: A-inner products of the stored directions (k x k, row-major) */
int oracle_proj_gram(const oracle_proj* p, double* G) {
  const int64_t ns = p->c->nslots;
  for (int i = 0; i < p->k; i++)
    for (int j = 0; j < p->k; j++)
      G[i * p->k + j] = oracle_dot_c(p->c, p->Z + (int64_t)i * ns, p->AZ + (int64_t)j * ns);
  return 0;
}

/* ------------------------------------------------------------------ */
/* NEXT-1: two-level additive overlapping Schwarz preconditioner        */
/* (M0^-1 = R0^T A0^-1 R0 + sum_k R_k^T A~_k^-1 R_k; "the   */
/* coarse grid (on linear elements) is solved for using an approximate  */
/* Krylov solver, in essence performing few (~10) CG iterations").      */
/* Readings Q28-Q31:                                         */
/*  Q28 subdomain k = the closed node set of element k (overlap of one   */
/*      node layer into every neighbour, homogeneous Dirichlet on the    */
/*      next layer); A~_k = the separable operator                       */
/*      Bz (x) By (x) Ax + Bz (x) Ay (x) Bx + Az (x) By (x) Bx with the   */
/*      1-D SEM stiffness/mass of the element extended by the            */
/*      neighbours' end entries (element lengths = mean edge length).   */
/*      On Cartesian meshes this is exactly the principal submatrix of   */
/*      the assembled A on the element's unmasked nodes.                 */
/*  Q29 weights: c^(1/2) on input and output of the local sum, so M      */
/*      stays symmetric: z_loc = c^1/2 QQ^T (A~^-1 (c^1/2 r))_L          */
/*  Q30 coarse space: the N = 1 discretisation on the same mesh; R0^T    */
/*      interpolates vertex values trilinearly (J_ia = (1 -+ xi_i)/2),   */
/*      R0 is its transpose (c-weighted, then summed); periodic: the     */
/*      coarse right-hand side loses its unique-DOF mean.               */
/*  Q31 coarse solve: plain CG from 0, at most K0 iterations, stopped    */
/*      early when ||r||_c <= 1e-12 ||b0||_c or p^T A0 p <= 0.           */
/* The local inverse is computed from its definition: the dense          */
/* n^3 x n^3 matrix A~_k is assembled and Cholesky-factored.            */
struct oracle_schwarz {
  const oracle_ctx* c;
  oracle_ctx* c0;        /* the N = 1 coarse space on the same mesh */
  int K0;
  double* L;             /* [E][n3*n3] Cholesky factors (masked rows: identity) */
  double* sqc;           /* c^1/2 per slot */
};

/* 1-D reference stiffness Ah_ij = sum_q w_q D_qi D_qj (exact for degree 2N-2) */
static void ref_stiff_1d(const oracle_ctx* c, double* Ah) {
  const int n = c->n;
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) {
      double s = 0.0;
      for (int q = 0; q < n; q++) s += c->w[q] * c->D[q * n + i] * c->D[q * n + j];
      Ah[i * n + j] = s;
    }
}

/* mean length of element e along axis a: the four element edges parallel to
   a, straight vertex-to-vertex distances (reading Q28) */
static double elem_len(const oracle_ctx* c, int64_t e, int a) {
  const int n = c->n, N = c->N;
  double s = 0.0;
  for (int u = 0; u < 2; u++)
    for (int v = 0; v < 2; v++) {
      int i0[3], i1[3];
      int o1 = u * N, o2 = v * N;
      if (a == 0) { i0[0] = 0; i1[0] = N; i0[1] = i1[1] = o1; i0[2] = i1[2] = o2; }
      else if (a == 1) { i0[1] = 0; i1[1] = N; i0[0] = i1[0] = o1; i0[2] = i1[2] = o2; }
      else { i0[2] = 0; i1[2] = N; i0[0] = i1[0] = o1; i0[1] = i1[1] = o2; }
      int64_t l0 = e * c->n3 + i0[0] + n * i0[1] + (int64_t)n * n * i0[2];
      int64_t l1 = e * c->n3 + i1[0] + n * i1[1] + (int64_t)n * n * i1[2];
      double dx = c->X[l1] - c->X[l0], dy = c->Y[l1] - c->Y[l0], dz = c->Z[l1] - c->Z[l0];
      s += sqrt(dx * dx + dy * dy + dz * dz);
    }
  return 0.25 * s;
}

/* the extended 1-D operators of element e along axis a (n x n, mass diagonal) */
static void ext_1d(const oracle_ctx* c, const double* Ah, int64_t e, int a, double* A1,
                   double* B1) {
  const int n = c->n, N = c->N;
  const oracle_mesh* m = &c->m;
  const int64_t Ea[3] = {m->ex, m->ey, m->ez};
  int64_t idx[3] = {e % m->ex, (e / m->ex) % m->ey, e / ((int64_t)m->ex * m->ey)};
  const double h = elem_len(c, e, a);
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) A1[i * n + j] = (2.0 / h) * Ah[i * n + j];
  for (int i = 0; i < n; i++) B1[i] = 0.5 * h * c->w[i];
  for (int side = 0; side < 2; side++) {
    int64_t q = idx[a] + (side ? 1 : -1);
    if (q < 0 || q >= Ea[a]) {
      if (!m->periodic[a]) continue;      /* Dirichlet face: no neighbour */
      q = (q + Ea[a]) % Ea[a];
    }
    int64_t nb[3] = {idx[0], idx[1], idx[2]};
    nb[a] = q;
    const int64_t en = nb[0] + m->ex * (nb[1] + (int64_t)m->ey * nb[2]);
    const double hn = elem_len(c, en, a);
    if (side == 0) {   /* left neighbour: its node N coincides with our node 0 */
      A1[0] += (2.0 / hn) * Ah[N * n + N];
      B1[0] += 0.5 * hn * c->w[N];
    } else {
      A1[N * n + N] += (2.0 / hn) * Ah[0];
      B1[N] += 0.5 * hn * c->w[0];
    }
  }
}

/* dense A~_e (n3 x n3, row-major, p = i + n j + n^2 k); masked rows and
   columns are zero */
static void local_matrix(const oracle_ctx* c, const double* Ah, int64_t e, double* A) {
  const int n = c->n;
  const int64_t n3 = c->n3;
  double* A1 = (double*)malloc(sizeof(double) * 3 * n * n);
  double* B1 = (double*)malloc(sizeof(double) * 3 * n);
  for (int a = 0; a < 3; a++) ext_1d(c, Ah, e, a, A1 + a * n * n, B1 + a * n);
  const double *Ax = A1, *Ay = A1 + n * n, *Az = A1 + 2 * n * n;
  const double *Bx = B1, *By = B1 + n, *Bz = B1 + 2 * n;
  for (int64_t p = 0; p < n3; p++) {
    const int i = (int)(p % n), j = (int)((p / n) % n), k = (int)(p / ((int64_t)n * n));
    for (int64_t q = 0; q < n3; q++) {
      const int i2 = (int)(q % n), j2 = (int)((q / n) % n), k2 = (int)(q / ((int64_t)n * n));
      double v = 0.0;
      if (k == k2 && j == j2) v += Bz[k] * By[j] * Ax[i * n + i2];
      if (k == k2 && i == i2) v += Bz[k] * Ay[j * n + j2] * Bx[i];
      if (j == j2 && i == i2) v += Az[k * n + k2] * By[j] * Bx[i];
      const int mp = c->mask[e * n3 + p], mq = c->mask[e * n3 + q];
      A[p * n3 + q] = (mp || mq) ? 0.0 : v;
    }
  }
  free(A1);
  free(B1);
}

/* in-place Cholesky A = L L^T (lower triangle); returns -6 if not SPD */
static int cholesky(double* A, int64_t m) {
  for (int64_t j = 0; j < m; j++) {
    double d = A[j * m + j];
    for (int64_t k = 0; k < j; k++) d -= A[j * m + k] * A[j * m + k];
    if (!(d > 0.0)) return -6;
    const double ljj = sqrt(d);
    A[j * m + j] = ljj;
    for (int64_t i = j + 1; i < m; i++) {
      double s = A[i * m + j];
      for (int64_t k = 0; k < j; k++) s -= A[i * m + k] * A[j * m + k];
      A[i * m + j] = s / ljj;
    }
  }
  return 0;
}

int oracle_schwarz_create(const oracle_ctx* c, int coarse_iters, oracle_schwarz** out) {
  if (!c || !out || coarse_iters < 0) return -1;
  *out = NULL;
  oracle_schwarz* s = (oracle_schwarz*)calloc(1, sizeof(oracle_schwarz));
  if (!s) return -5;
  s->c = c;
  s->K0 = coarse_iters;
  const int64_t n3 = c->n3, E = c->E;
  s->L = (double*)malloc(sizeof(double) * E * n3 * n3);
  s->sqc = (double*)malloc(sizeof(double) * c->nslots);
  double* Ah = (double*)malloc(sizeof(double) * c->n * c->n);
  if (!s->L || !s->sqc || !Ah) { free(Ah); oracle_schwarz_free(s); return -5; }
  for (int64_t l = 0; l < c->nslots; l++) s->sqc[l] = sqrt(c->c[l]);
  ref_stiff_1d(c, Ah);
  int st = 0;
  for (int64_t e = 0; e < E && !st; e++) {
    double* A = s->L + e * n3 * n3;
    local_matrix(c, Ah, e, A);
    for (int64_t p = 0; p < n3; p++)
      if (c->mask[e * n3 + p]) A[p * n3 + p] = 1.0;
    st = cholesky(A, n3);
  }
  free(Ah);
  if (!st) st = oracle_setup(&c->m, 1, 1, &s->c0);
  if (st) { oracle_schwarz_free(s); return st; }
  *out = s;
  return 0;
}

void oracle_schwarz_free(oracle_schwarz* s) {
  if (!s) return;
  if (s->c0) oracle_free(s->c0);
  free(s->L); free(s->sqc); free(s);
}

int oracle_schwarz_local_matrix(const oracle_schwarz* s, int64_t e, double* A) {
  if (!s || e < 0 || e >= s->c->E) return -1;
  double* Ah = (double*)malloc(sizeof(double) * s->c->n * s->c->n);
  if (!Ah) return -5;
  ref_stiff_1d(s->c, Ah);
  local_matrix(s->c, Ah, e, A);
  free(Ah);
  return 0;
}

/* the coarse correction z_c = R0^T A0^-1 R0 r (readings Q30, Q31) */
static int coarse_correction(const oracle_schwarz* s, const double* r, double* zc) {
  const oracle_ctx* c = s->c;
  const oracle_ctx* c0 = s->c0;
  const int n = c->n;
  const int64_t n3 = c->n3, ns0 = c0->nslots;
  double J[2 * 12];   /* J[i*2 + a]: vertex a's linear basis at xi_i */
  for (int i = 0; i < n; i++) {
    J[i * 2 + 0] = 0.5 * (1.0 - c->xi[i]);
    J[i * 2 + 1] = 0.5 * (1.0 + c->xi[i]);
  }
  double* b0 = (double*)calloc(ns0, sizeof(double));
  double* x0 = (double*)calloc(ns0, sizeof(double));
  double* r0 = (double*)malloc(sizeof(double) * ns0);
  double* p0 = (double*)malloc(sizeof(double) * ns0);
  double* w0 = (double*)malloc(sizeof(double) * ns0);
  if (!b0 || !x0 || !r0 || !p0 || !w0) { free(b0); free(x0); free(r0); free(p0); free(w0); return -5; }
  /* R0 r: per element (J^T (x) J^T (x) J^T)(c r_e), then QQ^T on the coarse space, mask */
  for (int64_t e = 0; e < c->E; e++)
    for (int v = 0; v < 8; v++) {
      const int a = v & 1, b = (v >> 1) & 1, cc = v >> 2;
      double sacc = 0.0;
      for (int k = 0; k < n; k++)
        for (int j = 0; j < n; j++)
          for (int i = 0; i < n; i++) {
            const int64_t l = e * n3 + i + n * j + (int64_t)n * n * k;
            sacc += J[i * 2 + a] * J[j * 2 + b] * J[k * 2 + cc] * (c->c[l] * r[l]);
          }
      b0[e * 8 + v] = sacc;
    }
  oracle_gs(c0, b0);
  oracle_mask_apply(c0, b0);
  if (c0->fully_periodic) {   /* remove the unique-DOF mean (b0 in range(A0)) */
    double sb = 0.0, sc = 0.0;
    for (int64_t l = 0; l < ns0; l++) { sb += c0->c[l] * b0[l]; sc += c0->c[l]; }
    const double mean = sb / sc;
    for (int64_t l = 0; l < ns0; l++) b0[l] -= mean;
  }
  /* plain CG, x0 = 0, at most K0 iterations */
  for (int64_t l = 0; l < ns0; l++) { r0[l] = b0[l]; p0[l] = b0[l]; }
  double rho = oracle_dot_c(c0, r0, r0);
  const double stop = 1e-12 * sqrt(rho);
  for (int k = 0; k < s->K0 && rho > 0.0; k++) {
    oracle_apply(c0, p0, w0);
    const double sigma = oracle_dot_c(c0, p0, w0);
    if (!(sigma > 0.0)) break;
    const double alpha = rho / sigma;
    for (int64_t l = 0; l < ns0; l++) {
      x0[l] += alpha * p0[l];
      r0[l] -= alpha * w0[l];
    }
    const double gamma = oracle_dot_c(c0, r0, r0);
    if (sqrt(gamma) <= stop) break;
    const double beta = gamma / rho;
    rho = gamma;
    for (int64_t l = 0; l < ns0; l++) p0[l] = r0[l] + beta * p0[l];
  }
  /* R0^T x0: trilinear interpolation of the element's vertex values */
  for (int64_t e = 0; e < c->E; e++)
    for (int k = 0; k < n; k++)
      for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++) {
          double sacc = 0.0;
          for (int v = 0; v < 8; v++) {
            const int a = v & 1, b = (v >> 1) & 1, cc = v >> 2;
            sacc += J[i * 2 + a] * J[j * 2 + b] * J[k * 2 + cc] * x0[e * 8 + v];
          }
          zc[e * n3 + i + n * j + (int64_t)n * n * k] = sacc;
        }
  free(b0); free(x0); free(r0); free(p0); free(w0);
  return 0;
}

/* z = mask(c^1/2 QQ^T (A~^-1 c^1/2 r)_L + R0^T A0^-1 R0 r).  which: 1 local
   part only, 2 coarse part only, 3 both */
int oracle_schwarz_apply(const oracle_schwarz* s, const double* r, double* z, int which) {
  if (!s || which < 1 || which > 3) return -1;
  const oracle_ctx* c = s->c;
  const int64_t n3 = c->n3, ns = c->nslots;
  for (int64_t l = 0; l < ns; l++) z[l] = 0.0;
  if (which & 1) {
    double* y = (double*)malloc(sizeof(double) * n3);
    if (!y) return -5;
    for (int64_t e = 0; e < c->E; e++) {
      const double* L = s->L + e * n3 * n3;
      for (int64_t p = 0; p < n3; p++) {   /* forward: L y = c^1/2 r (0 on masked) */
        const int64_t l = e * n3 + p;
        double v = c->mask[l] ? 0.0 : s->sqc[l] * r[l];
        for (int64_t q = 0; q < p; q++) v -= L[p * n3 + q] * y[q];
        y[p] = v / L[p * n3 + p];
      }
      for (int64_t p = n3 - 1; p >= 0; p--) {   /* backward: L^T x = y */
        double v = y[p];
        for (int64_t q = p + 1; q < n3; q++) v -= L[q * n3 + p] * y[q];
        y[p] = v / L[p * n3 + p];
      }
      for (int64_t p = 0; p < n3; p++) z[e * n3 + p] = c->mask[e * n3 + p] ? 0.0 : y[p];
    }
    free(y);
    oracle_gs(c, z);
    for (int64_t l = 0; l < ns; l++) z[l] *= s->sqc[l];
  }
  if (which & 2) {
    double* zc = (double*)malloc(sizeof(double) * ns);
    if (!zc) return -5;
    int st = coarse_correction(s, r, zc);
    if (st) { free(zc); return st; }
    for (int64_t l = 0; l < ns; l++) z[l] += zc[l];
    free(zc);
  }
  oracle_mask_apply(c, z);
  return 0;
}

/* PCG with the Schwarz preconditioner.  The coarse solve is a fixed number of
   CG iterations, a nonlinear operator, so beta takes the flexible (Polak-
   Ribiere) form beta = <z', r' - r>_c / <z, r>_c = -alpha <z', w>_c / rho
   (reading Q32); otherwise the loop is pcg_core's. */
int oracle_schwarz_pcg(const oracle_schwarz* s, const double* b, double* x, double tol,
                       int maxit, int* iters, double* res_final, double* res_true, double* hist) {
  if (!s || maxit < 0) return -1;
  const oracle_ctx* c = s->c;
  const int64_t ns = c->nslots;
  double* r = (double*)calloc(ns, sizeof(double));
  double* z = (double*)malloc(sizeof(double) * ns);
  double* p = (double*)malloc(sizeof(double) * ns);
  double* w = (double*)malloc(sizeof(double) * ns);
  if (!r || !z || !p || !w) { free(r); free(z); free(p); free(w); return -5; }
  int status = 1, k = 0;
  for (int64_t l = 0; l < ns; l++) { x[l] = 0.0; r[l] = b[l]; }
  oracle_schwarz_apply(s, r, z, 3);
  for (int64_t l = 0; l < ns; l++) p[l] = z[l];
  double rho = oracle_dot_c(c, r, z);
  double gamma = oracle_dot_c(c, r, r);
  if (hist) hist[0] = sqrt(gamma);
  if (sqrt(gamma) <= tol) status = 0;
  while (status == 1 && k < maxit) {
    k++;
    oracle_apply(c, p, w);
    const double sigma = oracle_dot_c(c, p, w);
    if (!(sigma > 0.0)) { status = -6; break; }
    const double alpha = rho / sigma;
    for (int64_t l = 0; l < ns; l++) {
      x[l] += alpha * p[l];
      r[l] -= alpha * w[l];
    }
    gamma = oracle_dot_c(c, r, r);
    if (hist) hist[k] = sqrt(gamma);
    if (sqrt(gamma) <= tol) { status = 0; break; }
    oracle_schwarz_apply(s, r, z, 3);
    const double rho_new = oracle_dot_c(c, r, z);
    const double beta = -alpha * oracle_dot_c(c, w, z) / rho;
    rho = rho_new;
    for (int64_t l = 0; l < ns; l++) p[l] = z[l] + beta * p[l];
  }
  if (iters) *iters = k;
  if (res_final) *res_final = sqrt(gamma);
  if (res_true) {
    oracle_apply(c, x, w);
    for (int64_t l = 0; l < ns; l++) w[l] = b[l] - w[l];
    *res_true = sqrt(oracle_dot_c(c, w, w));
  }
  free(r); free(z); free(p); free(w);
  return status;
}

/* flexible restarted GMRES with the Schwarz preconditioner (right, variable:
   z_j = M v_j is stored and x += Z y, Saad's FGMRES); otherwise as oracle_gmres
   (two MGS passes, Givens rotations, the same stopping rule). */
int oracle_schwarz_gmres(const oracle_schwarz* s, const double* b, double* x, double tol,
                         int maxit, int restart, int* iters, double* res_final, double* res_true,
                         double* hist) {
  if (!s || maxit < 0 || restart < 1) return -1;
  const oracle_ctx* c = s->c;
  const int64_t ns = c->nslots;
  const int m = restart;
  double* V = (double*)malloc(sizeof(double) * ns * (m + 1));
  double* Zs = (double*)malloc(sizeof(double) * ns * m);
  double* w = (double*)malloc(sizeof(double) * ns);
  double* H = (double*)calloc((size_t)(m + 1) * m, sizeof(double));
  double* cs = (double*)malloc(sizeof(double) * m);
  double* sn = (double*)malloc(sizeof(double) * m);
  double* g = (double*)malloc(sizeof(double) * (m + 1));
  double* y = (double*)malloc(sizeof(double) * m);
  if (!V || !Zs || !w || !H || !cs || !sn || !g || !y) {
    free(V); free(Zs); free(w); free(H); free(cs); free(sn); free(g); free(y);
    return -5;
  }
  int k = 0, status = 1;
  double res = 0.0;
  for (int cycle = 0;; cycle++) {
    oracle_apply(c, x, w);
    for (int64_t l = 0; l < ns; l++) V[l] = b[l] - w[l];
    const double beta = sqrt(oracle_dot_c(c, V, V));
    res = beta;
    if (cycle == 0 && hist) hist[0] = beta;
    if (beta <= tol) { status = 0; break; }
    if (k >= maxit) break;
    for (int64_t l = 0; l < ns; l++) V[l] /= beta;
    for (int i = 0; i <= m; i++) g[i] = 0.0;
    g[0] = beta;
    int j = 0;
    for (; j < m && k < maxit; j++) {
      double* vj = V + (int64_t)j * ns;
      double* zj = Zs + (int64_t)j * ns;
      oracle_schwarz_apply(s, vj, zj, 3);
      oracle_apply(c, zj, w);
      k++;
      for (int i = 0; i <= j; i++) H[i * m + j] = 0.0;
      for (int pass = 0; pass < 2; pass++)
        for (int i = 0; i <= j; i++) {
          const double* vi = V + (int64_t)i * ns;
          const double h = oracle_dot_c(c, w, vi);
          H[i * m + j] += h;
          for (int64_t l = 0; l < ns; l++) w[l] -= h * vi[l];
        }
      const double hn = sqrt(oracle_dot_c(c, w, w));
      H[(j + 1) * m + j] = hn;
      double* vn = V + (int64_t)(j + 1) * ns;
      for (int64_t l = 0; l < ns; l++) vn[l] = hn > 0.0 ? w[l] / hn : 0.0;
      for (int i = 0; i < j; i++) {
        const double a = H[i * m + j], bb = H[(i + 1) * m + j];
        H[i * m + j] = cs[i] * a + sn[i] * bb;
        H[(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
      }
      const double a = H[j * m + j], bb = H[(j + 1) * m + j];
      const double rr = sqrt(a * a + bb * bb);
      cs[j] = rr > 0.0 ? a / rr : 1.0;
      sn[j] = rr > 0.0 ? bb / rr : 0.0;
      H[j * m + j] = rr;
      H[(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      res = fabs(g[j + 1]);
      if (hist) hist[k] = res;
      if (res <= tol || hn == 0.0) { j++; break; }
    }
    for (int i = j - 1; i >= 0; i--) {
      double sacc = g[i];
      for (int q = i + 1; q < j; q++) sacc -= H[i * m + q] * y[q];
      y[i] = sacc / H[i * m + i];
    }
    for (int64_t l = 0; l < ns; l++) {
      double zy = 0.0;
      for (int i = 0; i < j; i++) zy += Zs[(int64_t)i * ns + l] * y[i];
      x[l] += zy;
    }
    if (res <= tol) { status = 0; break; }
    if (k >= maxit) break;
  }
  if (iters) *iters = k;
  if (res_final) *res_final = res;
  if (res_true) {
    oracle_apply(c, x, w);
    for (int64_t l = 0; l < ns; l++) w[l] = b[l] - w[l];
    *res_true = sqrt(oracle_dot_c(c, w, w));
  }
  free(V); free(Zs); free(w); free(H); free(cs); free(sn); free(g); free(y);
  return status;
}

/* NEXT-1 pressure pipeline: projection + GMRES + Schwarz; NULL restores Jacobi */
int oracle_proj_set_schwarz(oracle_proj* p, const oracle_schwarz* s) {
  if (!p || (s && s->c != p->c)) return -1;
  p->schw = s;
  return 0;
}

/* ------------------------------------------------------------------ */
/* canonical plan export (P:L231 sorted tuples + variable blocks)       */
static int cmp_first(const void* a, const void* b) {
  int64_t x = ((const int64_t*)a)[0], y = ((const int64_t*)b)[0];
  return (x > y) - (x < y);
}

int oracle_plan(const oracle_ctx* c, int64_t* npairs, int64_t* nseg, int64_t* nsegslots,
                int64_t* pairs, int64_t* seg_off, int64_t* seg_slot) {
  if (!c) return -1;
  int64_t np = 0, nsg = 0, nss = 0;
  for (int64_t g = 0; g < c->nglob; g++) {
    int64_t cnt = c->gs_off[g + 1] - c->gs_off[g];
    if (cnt == 2) np++;
    else if (cnt >= 3) { nsg++; nss += cnt; }
  }
  *npairs = np; *nseg = nsg; *nsegslots = nss;
  if (!pairs || !seg_off || !seg_slot) return 0;
  /* pairs: (l_a, l_b), sorted by l_a */
  int64_t t = 0;
  for (int64_t g = 0; g < c->nglob; g++) {
    int64_t lo = c->gs_off[g];
    if (c->gs_off[g + 1] - lo == 2) {
      pairs[2 * t] = c->gs_slot[lo];
      pairs[2 * t + 1] = c->gs_slot[lo + 1];
      t++;
    }
  }
  qsort(pairs, (size_t)np, 2 * sizeof(int64_t), cmp_first);
  /* segments sorted by first slot: sort (first slot, gid) keys */
  int64_t* key = (int64_t*)malloc(sizeof(int64_t) * 2 * (nsg ? nsg : 1));
  if (!key) return -5;
  t = 0;
  for (int64_t g = 0; g < c->nglob; g++) {
    int64_t lo = c->gs_off[g];
    if (c->gs_off[g + 1] - lo >= 3) {
      key[2 * t] = c->gs_slot[lo];
      key[2 * t + 1] = g;
      t++;
    }
  }
  qsort(key, (size_t)nsg, 2 * sizeof(int64_t), cmp_first);
  seg_off[0] = 0;
  for (int64_t s = 0; s < nsg; s++) {
    int64_t g = key[2 * s + 1];
    int64_t lo = c->gs_off[g], hi = c->gs_off[g + 1];
    for (int64_t q = lo; q < hi; q++) seg_slot[seg_off[s] + (q - lo)] = c->gs_slot[q];
    seg_off[s + 1] = seg_off[s] + (hi - lo);
  }
  free(key);
  return 0;
}

int oracle_shared(const oracle_ctx* c, int r, int q, int64_t* count, int64_t* gids) {
  if (!c || r == q || r < 0 || q < 0 || r >= c->nranks || q >= c->nranks) return -1;
  int64_t cnt = 0;
  for (int64_t g = 0; g < c->nglob; g++) {
    int hr = 0, hq = 0;
    for (int64_t t = c->gs_off[g]; t < c->gs_off[g + 1]; t++) {
      int rk = c->rank_elem[c->gs_slot[t] / c->n3];
      if (rk == r) hr = 1;
      if (rk == q) hq = 1;
    }
    if (hr && hq) {
      if (gids) gids[cnt] = g;
      cnt++;
    }
  }
  *count = cnt;
  return 0;
}
