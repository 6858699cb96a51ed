/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the matrix-free SEM
 * pressure-Poisson hot path of Neko (arxiv 2107.01243).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no source with the CUDA product path
 * (paper_2107_01243_b200/csrc, include/sem.h) and neither side includes the
 * other.
 *
 * Citations: "P:L<n>" = /root/reference/PAPER.md line n; readings Q1..Q22 are
 * listed in DESIGN.md section 3 (they follow SURVEY.md section 8(c)).
 *
 * Conventions (reading Q3, the paper leaves them free):
 *   element  e = ex + Ex*(ey + Ey*ez)
 *   slot     l = e*n^3 + i + n*j + n^2*k      (n = N+1, i along x fastest)
 *   G        [E][6][n^3] in the order (rr, ss, tt, rs, rt, st)
 *
 * All functions return 0 on success, <0 on error:
 *   -1 invalid argument, -2 non-positive Jacobian, -5 out of memory,
 *   -6 CG breakdown (p^T A p <= 0); oracle_pcg returns 1 if not converged.
 */
#ifndef SEM_ORACLE_H
#define SEM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t ex, ey, ez;                 /* elements per axis */
  double x0, x1, y0, y1, z0, z1;      /* box extents */
  int32_t periodic[3];                /* 1 = periodic axis, 0 = homogeneous Dirichlet faces */
  int32_t deform;                     /* 0 = Cartesian, 1 = sinusoidal map (reading Q4) */
  double deform_amp;                  /* a in x_m = X_m + a sin X sin Y sin Z */
} oracle_mesh;

typedef struct oracle_ctx oracle_ctx;

/* 1-D building blocks (Eq. 7) */
int oracle_legendre(int N, double x, double* L, double* dL);
int oracle_gll(int N, double* xi, double* w);
int oracle_deriv(int N, const double* xi, double* D);        /* D[i*n+j] = l_j'(xi_i) */

/* raw element kernels on caller arrays (used by the pins with random G) */
int oracle_ax_raw(int64_t E, int N, const double* D, const double* G,
                  const double* u, double* w);               /* Eq. 9, no gs, no mask */
int oracle_diag_raw(int64_t E, int N, const double* D, const double* G,
                    double* d);                               /* diag of A^e (reading Q14) */

/* context: mesh + space + geometry + numbering + gs lists */
int oracle_setup(const oracle_mesh* m, int N, int nranks, oracle_ctx** out);
void oracle_free(oracle_ctx* c);
int oracle_sizes(const oracle_ctx* c, int64_t* nslots, int64_t* E, int64_t* nglob);
/* which: 0 xi, 1 w, 2 D, 3 X, 4 Y, 5 Z, 6 G, 7 B, 8 dinv, 9 c (=1/mult) */
int oracle_get(const oracle_ctx* c, int which, double* dst);
/* which: 0 gid, 1 mult, 2 mask, 3 rank of slot */
int oracle_get_int(const oracle_ctx* c, int which, int64_t* dst);

int oracle_ax(const oracle_ctx* c, const double* u, double* w);   /* w_L = A_L u_L */
int oracle_gs(const oracle_ctx* c, double* u);                      /* u <- QQ^T u */
int oracle_mask_apply(const oracle_ctx* c, double* u);
int oracle_apply(const oracle_ctx* c, const double* u, double* w); /* mask(QQ^T A_L u) */
int oracle_rhs(const oracle_ctx* c, const double* f, double* b);
double oracle_dot_c(const oracle_ctx* c, const double* a, const double* b);
int oracle_pcg(const oracle_ctx* c, const double* b, double* x, double tol, int maxit,
               int* iters, double* res_final, double* res_true, double* hist);

/* canonical gs plan (reading Q11): pairs (l_a<l_b) sorted by l_a, segments
   (>=3 slots, ascending) sorted by first slot. Call with NULL arrays to size. */
/* NEXT-2 Helmholtz h1 A + h2 B: operator, mass RHS without
   the periodic projection, Jacobi inverse diagonal, and the same PCG on it. */
int oracle_helm_apply(const oracle_ctx* c, double h1, double h2, const double* u, double* w);
int oracle_rhs_mass(const oracle_ctx* c, const double* f, double* b);
int oracle_helm_dinv(const oracle_ctx* c, double h1, double h2, double* dinv);
int oracle_helm_pcg(const oracle_ctx* c, double h1, double h2, const double* b, double* x,
                    double tol, int maxit, int* iters, double* res_final, double* res_true,
                    double* hist);
/* single-reduction (Chronopoulos-Gear) Jacobi PCG, reading Q34: same iterates
   as oracle_pcg in exact arithmetic, one global reduction per iteration */
int oracle_cgcg(const oracle_ctx* c, const double* b, double* x, double tol, int maxit,
                int* iters, double* res_final, double* res_true, double* hist);
/* NEXT-3 (Table 2): restarted GMRES with right Jacobi
   preconditioning, and the solution-projection space (Fischer 1998). */
/* test access: m Arnoldi steps (the oracle_gmres step) from b; V [(m+1) x nslots], H [(m+1) x m] */
int oracle_arnoldi(const oracle_ctx* c, const double* b, int m, double* V, double* H);
int oracle_gmres(const oracle_ctx* c, const double* b, double* x, double tol, int maxit,
                 int restart, int* iters, double* res_final, double* res_true, double* hist);
typedef struct oracle_proj oracle_proj;
int oracle_proj_create(const oracle_ctx* c, int m, oracle_proj** out);
void oracle_proj_free(oracle_proj* p);
int oracle_proj_size(const oracle_proj* p);
int oracle_proj_project(const oracle_proj* p, const double* b, double* xbar, double* bdefl);
int oracle_proj_update(oracle_proj* p, const double* x);
int oracle_proj_solve(oracle_proj* p, const double* b, double* x, double tol, int maxit,
                      int restart, int* iters, double* res_final);
int oracle_proj_gram(const oracle_proj* p, double* G);
/* NEXT-1: two-level additive overlapping Schwarz, readings Q28-Q32:
   element subdomains with one node of overlap (separable local operator, dense
   Cholesky here), N = 1 coarse space solved by <= coarse_iters plain CG steps. */
typedef struct oracle_schwarz oracle_schwarz;
int oracle_schwarz_create(const oracle_ctx* c, int coarse_iters, oracle_schwarz** out);
void oracle_schwarz_free(oracle_schwarz* s);
int oracle_schwarz_local_matrix(const oracle_schwarz* s, int64_t e, double* A);  /* n3 x n3 */
int oracle_schwarz_apply(const oracle_schwarz* s, const double* r, double* z, int which);
int oracle_schwarz_pcg(const oracle_schwarz* s, const double* b, double* x, double tol,
                       int maxit, int* iters, double* res_final, double* res_true, double* hist);
int oracle_schwarz_gmres(const oracle_schwarz* s, const double* b, double* x, double tol,
                         int maxit, int restart, int* iters, double* res_final, double* res_true,
                         double* hist);
int oracle_proj_set_schwarz(oracle_proj* p, const oracle_schwarz* s);
int oracle_plan(const oracle_ctx* c, int64_t* npairs, int64_t* nseg, int64_t* nsegslots,
                int64_t* pairs, int64_t* seg_off, int64_t* seg_slot);
/* gids shared between ranks r and q (r != q), ascending; NULL list to size. */
int oracle_shared(const oracle_ctx* c, int r, int q, int64_t* count, int64_t* gids);

#ifdef __cplusplus
}
#endif
#endif
