// Setup, gather-scatter and Krylov-vector kernels of libsem (sm_100a).
//   geometry       P:L105 "geometric factors for mapping to and from the reference element" (reading Q5)
//   gather-scatter P:L107-111 Eq. 10, Alg. 1, P:L231 (readings Q10, Q11)
//   Jacobi-PCG     P:L257 (readings Q14-Q17)
#include <cmath>

#include "dev_common.cuh"
#include "kernels.h"
#include "gs_dev.cuh"
#include "p2p_dev.cuh"
#include "sem_internal.h"

namespace sem {

static thread_local bool t_pdl = false;
void set_pdl(bool on) { t_pdl = on; }
bool pdl_on() { return t_pdl; }

namespace dev {

constexpr int kThreads = 256;

__device__ __forceinline__ double c_of(unsigned m) { return __drcp_rn((double)m); }

// ---------------------------------------------------------------- geometry
// Box and node_xyz (reading Q4) live in dev_common.cuh

// one thread per slot: dx_a/dr_b through D on the isoparametric coordinates,
// J = det, dr/dx by cofactors, G_ab = J w w w (dr_a/dx . dr_b/dx), B = J w w w
__global__ void geom_kernel(int n, int64_t nslots, const double* __restrict__ xi,
                            const double* __restrict__ wq, const double* __restrict__ D,
                            int64_t e_lo, int ex, int ey, int ez, Box b, int deform, double amp,
                            double* __restrict__ G, double* __restrict__ B, int* bad) {
  const int64_t n3 = (int64_t)n * n * n;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nslots;
       l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t el = l / n3;
    const int p = (int)(l - el * n3);
    const int i = p % n, j = (p / n) % n, k = p / (n * n);
    const int64_t e = e_lo + el;
    double M[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int m = 0; m < n; m++) {
      double xr[3], xs[3], xt[3];
      node_xyz(xi, ex, ey, ez, e, m, j, k, b, deform, amp, xr);
      node_xyz(xi, ex, ey, ez, e, i, m, k, b, deform, amp, xs);
      node_xyz(xi, ex, ey, ez, e, i, j, m, b, deform, amp, xt);
      const double di = D[i * n + m], dj = D[j * n + m], dk = D[k * n + m];
      for (int a = 0; a < 3; a++) {
        M[a][0] = fma(di, xr[a], M[a][0]);
        M[a][1] = fma(dj, xs[a], M[a][1]);
        M[a][2] = fma(dk, xt[a], M[a][2]);
      }
    }
    const double c00 = M[1][1] * M[2][2] - M[1][2] * M[2][1];
    const double c01 = M[1][2] * M[2][0] - M[1][0] * M[2][2];
    const double c02 = M[1][0] * M[2][1] - M[1][1] * M[2][0];
    const double J = M[0][0] * c00 + M[0][1] * c01 + M[0][2] * c02;
    if (!(J > 0.0)) {
      atomicMax(bad, 1);
      continue;
    }
    const double iJ = 1.0 / J;
    double R[3][3];  // R[b][a] = d r_b / d x_a = cof(M)[a][b] / J
    R[0][0] = c00 * iJ;
    R[1][0] = c01 * iJ;
    R[2][0] = c02 * iJ;
    R[0][1] = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) * iJ;
    R[1][1] = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) * iJ;
    R[2][1] = (M[0][1] * M[2][0] - M[0][0] * M[2][1]) * iJ;
    R[0][2] = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) * iJ;
    R[1][2] = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) * iJ;
    R[2][2] = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) * iJ;
    const double Jw = J * wq[i] * wq[j] * wq[k];
    const int ab[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
    for (int f = 0; f < 6; f++) {
      const int x = ab[f][0], y = ab[f][1];
      G[g_index(el, f, p, n)] = Jw * (R[x][0] * R[y][0] + R[x][1] * R[y][1] + R[x][2] * R[y][2]);
    }
    B[l] = Jw;
  }
}

__global__ void coords_kernel(int n, int64_t nslots, const double* __restrict__ xi, int64_t e_lo,
                              int ex, int ey, int ez, Box b, int deform, double amp,
                              double* X, double* Y, double* Z) {
  const int64_t n3 = (int64_t)n * n * n;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nslots;
       l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t el = l / n3;
    const int p = (int)(l - el * n3);
    double x[3];
    node_xyz(xi, ex, ey, ez, e_lo + el, p % n, (p / n) % n, p / (n * n), b, deform, amp, x);
    X[l] = x[0]; Y[l] = x[1]; Z[l] = x[2];
  }
}

// element diagonal of D^T G D (reading Q14)
__global__ void diag_kernel(int n, int64_t nslots, const double* __restrict__ D,
                            const double* __restrict__ G, double* __restrict__ d) {
  const int64_t n3 = (int64_t)n * n * n;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nslots;
       l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t el = l / n3;
    const int p = (int)(l - el * n3);
    const int i = p % n, j = (p / n) % n, k = p / (n * n);
    double s = 0.0;
    for (int m = 0; m < n; m++) {
      const double a = D[m * n + i], b2 = D[m * n + j], c = D[m * n + k];
      s = fma(a * a, G[g_index(el, 0, m + n * j + n * n * k, n)], s);
      s = fma(b2 * b2, G[g_index(el, 1, i + n * m + n * n * k, n)], s);
      s = fma(c * c, G[g_index(el, 2, i + n * j + n * n * m, n)], s);
    }
    const double dii = D[i * n + i], djj = D[j * n + j], dkk = D[k * n + k];
    s += 2.0 * (G[g_index(el, 3, p, n)] * dii * djj + G[g_index(el, 4, p, n)] * dii * dkk +
                G[g_index(el, 5, p, n)] * djj * dkk);
    d[l] = s;
  }
}

__device__ __forceinline__ bool slot_mask(const DevPlan& P, int64_t l) {
  const int n = P.n;
  const int64_t n3 = (int64_t)n * n * n;
  const int64_t el = l / n3;
  const int p = (int)(l - el * n3);
  return face_masked(P.bmask[el], p % n, (p / n) % n, p / (n * n), n - 1);
}

__global__ void invert_mask_kernel(const DevPlan P, double* d) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < P.n_local;
       l += (int64_t)gridDim.x * blockDim.x)
    d[l] = slot_mask(P, l) ? 0.0 : 1.0 / d[l];
}

__global__ void mask_kernel(const DevPlan P, double* u) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < P.n_local;
       l += (int64_t)gridDim.x * blockDim.x)
    if (slot_mask(P, l)) u[l] = 0.0;
}

__global__ void export_mask_kernel(const DevPlan P, uint8_t* m) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < P.n_local;
       l += (int64_t)gridDim.x * blockDim.x)
    m[l] = slot_mask(P, l) ? 1 : 0;
}

// Helmholtz Jacobi (NEXT-2): d = h1 d + h2 B on the element diagonals before gs
__global__ void helm_diag_kernel(double* __restrict__ d, const double* __restrict__ B, double h1,
                                 double h2, int64_t n) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x)
    d[l] = h1 * d[l] + h2 * B[l];
}

__global__ void scale_kernel(const double* __restrict__ B, const double* __restrict__ f,
                             double* __restrict__ b, int64_t n) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x)
    b[l] = B[l] * f[l];
}

// b = mask ? 0 : B f.  Masking before the gather-scatter equals masking after it
// (every copy of a Dirichlet global point is a Dirichlet slot), and reaches the
// boundary slots no gs entity touches (points of a single element).
__global__ void scale_mask_kernel(const DevPlan P, const double* __restrict__ B,
                                  const double* __restrict__ f, double* __restrict__ b) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < P.n_local;
       l += (int64_t)gridDim.x * blockDim.x)
    b[l] = slot_mask(P, l) ? 0.0 : B[l] * f[l];
}

__global__ void sub_scalar_kernel(double* a, const double* scal, int64_t n) {
  // scal[0] = sum_l c_l b_l, scal[1] = sum_l c_l  -> subtract the unique-DOF mean
  const double mean = scal[0] / scal[1];
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x)
    a[l] -= mean;
}

// ---------------------------------------------------------------- gather-scatter

// Multiplicity per slot (uint8): 1 everywhere, nin on entity points, the global
// incidence count on shared points.
__global__ void mult_kernel(const DevPlan P, uint8_t* mult) {
  const int n = P.n, N = n - 1;
  const int64_t nf = (int64_t)(N - 1) * (N - 1), ne = N - 1;
  const int64_t tF = P.nF * nf, tE = P.nEd * ne, tot = tF + tE + P.nV + P.nS;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < tF) {
      const int64_t f = t / nf;
      const int p = (int)(t - f * nf);
      const int ax = P.f_axis[f];
      const int off = (1 + p % (N - 1)) * f_s1(ax, n) + (1 + p / (N - 1)) * f_s2(ax, n);
      mult[P.f_base[2 * f] + off] = 2;
      mult[P.f_base[2 * f + 1] + off] = 2;
    } else if (t < tF + tE) {
      const int64_t q = t - tF, e = q / ne;
      const int p = (int)(q - e * ne);
      const int off = (1 + p) * e_sd(P.e_axis[e], n);
      for (int x = 0; x < P.e_nin[e]; x++) mult[P.e_base[4 * e + x] + off] = P.e_nin[e];
    } else if (t < tF + tE + P.nV) {
      const int64_t v = t - tF - tE;
      for (int x = 0; x < P.v_nin[v]; x++) mult[P.v_base[8 * v + x]] = P.v_nin[v];
    } else {
      const int64_t s = t - tF - tE - P.nV;
      for (int x = 0; x < P.s_nloc[s]; x++) mult[P.s_slot[(int64_t)x * P.nS + s]] = P.s_mult[s];
    }
  }
}

#ifndef SEM_GS_MINB
#define SEM_GS_MINB 1
#endif
#ifndef SEM_GS_GRIDX
#define SEM_GS_GRIDX 1   // grid = SEM_GS_GRIDX x resident blocks
#endif
template <int n, bool SWEEP>
__global__ void __launch_bounds__(256, SEM_GS_MINB) gs_local_kernel(const DevPlan P, double* __restrict__ u,
                                                       int apply_mask, unsigned long long base,
                                                       int ce, const GsSigma sig) {
  pdl_wait();
  pdl_trigger();
  // one-rank PCG: sigma = the Ax kernel's per-CTA partials, summed here (off the
  // CG update's critical path) by the last block, in the update's order
  if (sig.part && blockIdx.x == gridDim.x - 1) {
    __shared__ double scratch[32];
    const int G = *sig.count;
    double v = 0.0;
    for (int b = threadIdx.x; b < G; b += blockDim.x) v += __ldcg(&sig.part[b]);
    v = block_sum(v, scratch);
    if (threadIdx.x == 0) sig.st->sigma = v;
  }
  gs_local_body<n, SWEEP>(P, u, apply_mask, P.gs_ctr, base, ce);
}

// Alg. 1 lines 6-7: this rank's partial for every shared point (ascending local
// slots), copied into the send buffer of every neighbour that shares it.
__global__ void gs_pack_kernel(const DevPlan P, const double* __restrict__ u, double* part,
                               double* sendbuf) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < P.nS;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int nl = P.s_nloc[s];
#pragma unroll 1
    for (int x = 0; x < nl; x++) {
      const int32_t l = P.s_slot[(int64_t)x * P.nS + s];
      SEM_CHK(l >= 0 && l < P.n_local && (x == 0 || l > P.s_slot[(int64_t)(x - 1) * P.nS + s]));
    }
    double v = u[P.s_slot[s]];
    for (int x = 1; x < nl; x++) v += u[P.s_slot[(int64_t)x * P.nS + s]];
    part[s] = v;
    const int nr = P.s_nr[s];
    for (int x = 0; x < nr; x++) {
      const int o = P.s_off[(int64_t)x * P.nS + s];
      SEM_CHK(o < P.nbuf);
      if (o >= 0) sendbuf[o] = v;
    }
  }
}

// Alg. 1 lines 10-18: total = sum of the rank partials in ascending rank order
// (reading Q10, deterministic), scattered to every local slot.  Thread 0 also
// combines the split sigma partials of the PCG operator (fixed order).
__global__ void gs_unpack_kernel(const DevPlan P, double* __restrict__ u, const double* part,
                                 const double* recvbuf, int apply_mask, PcgState* st, int nparts) {
  if (st && blockIdx.x == 0 && threadIdx.x == 0) {
    double sg = st->sigma_part[0];
    for (int q = 1; q < nparts; q++) sg += st->sigma_part[q];
    st->loc[2] = sg;   // this rank's sigma; allreduced out-of-place into st->sigma
  }
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < P.nS;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int nr = P.s_nr[s];
    double tot = 0.0;
    for (int x = 0; x < nr; x++) {
      const int o = P.s_off[(int64_t)x * P.nS + s];
      SEM_CHK(o < P.nbuf);
      const double v = o < 0 ? part[s] : recvbuf[o];
      tot = x == 0 ? v : tot + v;
    }
    if (apply_mask && P.s_mask[s]) tot = 0.0;
    const int nl = P.s_nloc[s];
    for (int x = 0; x < nl; x++) {
      SEM_CHK(P.s_slot[(int64_t)x * P.nS + s] >= 0 && P.s_slot[(int64_t)x * P.nS + s] < P.n_local);
      u[P.s_slot[(int64_t)x * P.nS + s]] = tot;
    }
  }
}

// ---------------------------------------------------------------- reductions
__global__ void dot_c_kernel(int64_t n, const uint8_t* __restrict__ mult,
                             const double* __restrict__ a, const double* __restrict__ b,
                             double* partial, unsigned* ticket, double* out) {
  __shared__ double scratch[32];
  __shared__ int flag;
  double s = 0.0;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x)
    s = fma(c_of(mult[l]) * a[l], b[l], s);
  double v[1] = {s};
  grid_reduce<1>(v, partial, ticket, out, scratch, &flag);
}

// out2[0] = sum_l c_l a_l, out2[1] = sum_l c_l
__global__ void sum_c_kernel(int64_t n, const uint8_t* __restrict__ mult,
                             const double* __restrict__ a, double* partial, unsigned* ticket,
                             double* out2) {
  __shared__ double scratch[32];
  __shared__ int flag;
  double s0 = 0.0, s1 = 0.0;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x) {
    const double c = c_of(mult[l]);
    s0 = fma(c, a[l], s0);
    s1 += c;
  }
  double v[2] = {s0, s1};
  grid_reduce<2>(v, partial, ticket, out2, scratch, &flag);
}

// ---------------------------------------------------------------- Jacobi-PCG
// init: x = 0, r = b, p = z = dinv .* b; partials of <r,z>_c and <r,r>_c
__global__ void __launch_bounds__(kThreads) cg_init_kernel(int64_t n, const uint8_t* __restrict__ mult,
                               const double* __restrict__ dinv, const double* __restrict__ b,
                               double* __restrict__ x, double* __restrict__ r,
                               double* __restrict__ p, double* partial, PcgState* st,
                               double* out2, const PeerSync ps, int pzero) {
  __shared__ double scratch[32];
  __shared__ int flag;
  double rz = 0.0, rr = 0.0;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x) {
    const double bl = b[l], z = dinv[l] * bl, c = c_of(mult[l]);
    x[l] = 0.0;
    r[l] = bl;
    p[l] = pzero ? 0.0 : z;   // pzero: the fused Ax kernel forms p_0 = dinv r + 0 p
    rz = fma(c * bl, z, rz);
    rr = fma(c * bl, bl, rr);
  }
  double v[2] = {rz, rr};
  if (grid_reduce<2>(v, partial, &st->tickets[1], out2, scratch, &flag) && ps.c.P > 1 &&
      threadIdx.x == 0)
    ar_publish(ps.c, AR_RG, ps.e_pub, out2, 2);
}

__global__ void cg_start_kernel(PcgState* st, double* hist, const PeerSync ps) {
  if (ps.c.P > 1) {
    double g2[2];
    ar_wait_sum(ps.c, AR_RG, ps.e_wait, 2, g2);
    st->rho_new = g2[0];
    st->gamma = g2[1];
  }
  st->rho_old = st->rho_new;
  st->beta = 0.0;   // fused p update: p_0 = dinv r
  st->it = 0;
  const double g = sqrt(st->gamma);
  hist[0] = g;
  st->done = (g <= st->tol) ? 1 : (st->maxit == 0 ? 4 : 0);
  st->iters = 0;
}

// end of a PCG iteration from the reduced (rho', gamma) in the state:
// convergence test on sqrt(gamma) (reading Q15), NaN guard, beta = rho'/rho,
// rho <- rho', residual history (the p kernel's last block does the same)
__device__ __forceinline__ void pcg_end_iteration(PcgState* st, double* hist) {
  const double rho_new = st->rho_new, gamma = st->gamma;
  const double g = sqrt(gamma);
  const int it = st->it + 1;
  st->it = it;
  hist[it] = g;
  if (!(g == g) || !(rho_new == rho_new)) {
    st->done = 3;
    st->iters = it;
  } else if (g <= st->tol) {
    st->done = 1;
    st->iters = it;
  } else {
    st->beta = rho_new / st->rho_old;
    st->rho_old = rho_new;
    if (it >= st->maxit) {
      st->done = 4;
      st->iters = it;
    }
  }
}

// alpha = rho / sigma; r -= alpha w; partials of rho' = <r, dinv r>_c and
// gamma = <r, r>_c (z is never stored).  Unfused: x += alpha p is deferred to
// the p kernel, which streams p anyway (same operation, one pass less over p
// and x).  PF (one rank, p update fused into the next Ax kernel): x += alpha p
// here, and the last block ends the iteration -- convergence test on
// sqrt(gamma), beta = rho'/rho for the next Ax kernel, history -- as the p
// kernel's last block does otherwise (end_here = 0: NCCL / loopback, where
// cg_end_iter_kernel does it after the host-side allreduce).
//
// GN = n > 0 (SEM_OPT_PCG_GSU): w is the UNASSEMBLED A_L p and this kernel
// performs the gather-scatter on read.  A slot with multiplicity > 1 sums its
// point's incidences of w in ascending slot order -- the gs kernel's sum,
// bit for bit (v0 + v1 for faces, left to right for edges and vertices) --
// through the per-element incidence table gu; every other slot
// takes its own w.  The streamed vectors keep their coalesced pair access; only
// the partner values are gathered (mostly L2 hits: the partners lie in
// elements e +- 1, e +- ex, e +- ex ey of the slab).  The gs kernel and its
// write-back of w disappear; r, rho', gamma are bitwise the two-kernel ones.
// the point's incidence bases (all -1: take its own w) and offset along the
// entity; depends on the slot index only, so the table load issues with the
// streamed loads instead of after them
struct GuRef {
  int4 a, b;
  int off;
};
template <int n>
__device__ __forceinline__ GuRef gu_ref(const int32_t* __restrict__ gu, int64_t s) {
  constexpr int N = n - 1, n2 = n * n, n3 = n2 * n;
  const int64_t el = s / n3;
  const int l = (int)(s - el * n3);
  const int i = l % n, j = (l / n) % n, k = l / n2;
  const bool bi = i == 0 || i == N, bj = j == 0 || j == N, bk = k == 0 || k == N;
  const int nb = (int)bi + (int)bj + (int)bk;
  GuRef g;
  g.a = g.b = make_int4(-1, -1, -1, -1);
  g.off = 0;
  const int32_t* rec = gu + el * kGuInts;
  if (nb == 1) {   // face interior point: normal axis a
    const int a = bi ? 0 : (bj ? 1 : 2);
    const int ca = a == 0 ? i : (a == 1 ? j : k);
    const int2 bb = reinterpret_cast<const int2*>(rec)[2 * a + (ca == N)];
    g.a.x = bb.x;
    g.a.y = bb.y;
    g.off = l - ca * (a == 0 ? 1 : (a == 1 ? n : n2));
  } else if (nb == 2) {   // edge interior point: direction a, the other two fixed
    const int a = !bi ? 0 : (!bj ? 1 : 2);
    const int lo = a == 0 ? j : i, hi = a == 2 ? j : k;
    g.a = reinterpret_cast<const int4*>(rec + kGuEdge)[4 * a + (lo == N) + 2 * (hi == N)];
    g.off = a == 0 ? i : (a == 1 ? j * n : k * n2);
  } else if (nb == 3) {   // vertex: up to 8 incidences, two groups of 4
    const int sub = (i == N) + 2 * (j == N) + 4 * (k == N);
    g.a = reinterpret_cast<const int4*>(rec + kGuVert)[2 * sub];
    g.b = reinterpret_cast<const int4*>(rec + kGuVert)[2 * sub + 1];
  }
  return g;
}

// ascending incidences, summed left to right (the gs kernel's order); a point
// that is not on a local entity (interior, Dirichlet side, or shared with
// another rank) keeps its own value
__device__ __forceinline__ double gu_sum(const double* __restrict__ w, const GuRef& g,
                                         double own) {
  if (g.a.x < 0) return own;
  const int off = g.off;
  SEM_CHK(g.a.y > g.a.x && (g.a.z < 0 || g.a.z > g.a.y) && (g.a.w < 0 || g.a.w > g.a.z) &&
          (g.b.x < 0 || g.b.x > g.a.w));
  double acc = w[g.a.x + off];
  {
    const double v1 = w[g.a.y + off];
    const double v2 = g.a.z >= 0 ? w[g.a.z + off] : 0.0;
    const double v3 = g.a.w >= 0 ? w[g.a.w + off] : 0.0;
    acc += v1;
    if (g.a.z >= 0) acc += v2;
    if (g.a.w >= 0) acc += v3;
  }
  if (g.b.x >= 0) {
    const double v4 = w[g.b.x];
    const double v5 = g.b.y >= 0 ? w[g.b.y] : 0.0;
    const double v6 = g.b.z >= 0 ? w[g.b.z] : 0.0;
    const double v7 = g.b.w >= 0 ? w[g.b.w] : 0.0;
    acc += v4;
    if (g.b.y >= 0) acc += v5;
    if (g.b.z >= 0) acc += v6;
    if (g.b.w >= 0) acc += v7;
  }
  return acc;
}

template <bool PF, int GN>
__global__ void __launch_bounds__(kThreads, 4) cg_update_kernel(int64_t n, const uint8_t* __restrict__ mult,
                                 const double* __restrict__ dinv, double* __restrict__ r,
                                 const double* __restrict__ w, double* partial, PcgState* st,
                                 double* out2, const double* __restrict__ sig_part,
                                 const int* sig_count, const PeerSync ps_in,
                                 double* __restrict__ x, const double* __restrict__ p,
                                 double* hist, int end_here, const int32_t* __restrict__ gu) {
  __shared__ double scratch[32];
  __shared__ int flag;
  __shared__ double s_sig;
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  PeerSync ps = ps_in;
  if (ps.dev) {   // device-side epochs (graph-replayed iterations at P > 1)
    const uint64_t kit = (uint64_t)st->it + 1;
    ps.e_wait = st->ep0[1] + kit;
    ps.e_pub = st->ep0[2] + kit;
  }
  double sigma;
  if (ps.c.P > 1) {   // global sigma from the peers' mailboxes (rank-ordered sum)
    if (threadIdx.x == 0) ar_wait_sum(ps.c, AR_SIG, ps.e_wait, 1, &s_sig);
    __syncthreads();
    sigma = s_sig;
    if (blockIdx.x == 0 && threadIdx.x == 0) st->sigma = sigma;
  } else if (sig_part) {
    // sigma = sum of the Ax kernel's per-CTA partials in a fixed order (the same
    // in every block).  All threads load (<= 3 partials each, issued together):
    // one warp walking ~600 partials put ~5 dependent L2 round trips in front
    // of every block's streaming loop.
    const int G = *sig_count;
    double v = 0.0;
    for (int b = threadIdx.x; b < G; b += blockDim.x) v += __ldcg(&sig_part[b]);
    v = block_sum(v, scratch);
    if (threadIdx.x == 0) s_sig = v;
    __syncthreads();
    sigma = s_sig;
    if (blockIdx.x == 0 && threadIdx.x == 0) st->sigma = sigma;
  } else {
    sigma = st->sigma;
  }
  const bool ok = sigma > 0.0;   // breakdown guard (also catches NaN)
  const double alpha = ok ? st->rho_old / sigma : 0.0;
  double rz = 0.0, rr = 0.0;
  if (ok) {
    const int64_t n2 = n >> 1;
    const double2* w2 = reinterpret_cast<const double2*>(w);
    const double2* d2 = reinterpret_cast<const double2*>(dinv);
    double2* r2 = reinterpret_cast<double2*>(r);
    const uchar2* m2 = reinterpret_cast<const uchar2*>(mult);
    double2* x2 = reinterpret_cast<double2*>(x);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n2;
         q += (int64_t)gridDim.x * blockDim.x) {
      double2 wv = GN ? w2[q] : __ldcs(&w2[q]);
      const double2 dv = __ldcs(&d2[q]);
      double2 rv = __ldcs(&r2[q]);
      const uchar2 mv = m2[q];
      if (GN) {
        const GuRef g0 = gu_ref<GN ? GN : 2>(gu, 2 * q), g1 = gu_ref<GN ? GN : 2>(gu, 2 * q + 1);
        wv.x = gu_sum(w, g0, wv.x);
        wv.y = gu_sum(w, g1, wv.y);
      }
      if (PF) {
        const double2 pv = __ldcs(&p2[q]);
        double2 xv = __ldcs(&x2[q]);
        xv.x = fma(alpha, pv.x, xv.x);
        xv.y = fma(alpha, pv.y, xv.y);
        __stcs(&x2[q], xv);
      }
      rv.x = fma(-alpha, wv.x, rv.x);
      rv.y = fma(-alpha, wv.y, rv.y);
      __stcg(&r2[q], rv);
      const double c0 = c_of(mv.x), c1 = c_of(mv.y);
      rz = fma(c0 * rv.x, dv.x * rv.x, rz);
      rz = fma(c1 * rv.y, dv.y * rv.y, rz);
      rr = fma(c0 * rv.x, rv.x, rr);
      rr = fma(c1 * rv.y, rv.y, rr);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const int64_t l = n - 1;
      double wl = w[l];
      if (GN) wl = gu_sum(w, gu_ref<GN ? GN : 2>(gu, l), wl);
      const double rl = fma(-alpha, wl, r[l]);
      r[l] = rl;
      if (PF) x[l] = fma(alpha, p[l], x[l]);
      const double c = c_of(mult[l]);
      rz = fma(c * rl, dinv[l] * rl, rz);
      rr = fma(c * rl, rl, rr);
    }
  }
  double v[2] = {rz, rr};
  if (grid_reduce<2>(v, partial, &st->tickets[2], out2, scratch, &flag)) {
    if (threadIdx.x == 0 && !ok) {
      st->done = 2;
      st->iters = st->it + 1;
    }
    if (threadIdx.x == 0 && ps.c.P > 1) ar_publish(ps.c, AR_RG, ps.e_pub, out2, 2);
    if (PF && ok && end_here && threadIdx.x == 0) {
      // end of the iteration: one rank -- out2 is st->rho_new; peer memory --
      // the ranks' partials summed in ascending rank order first
      __threadfence();
      if (ps.c.P > 1) {
        double g2[2];
        ar_wait_sum(ps.c, AR_RG, ps.e_pub, 2, g2);
        st->rho_new = g2[0];
        st->gamma = g2[1];
      }
      pcg_end_iteration(st, hist);
    }
  }
}

// PF over NCCL / loopback: the end of the iteration after the host-side allreduce
__global__ void cg_end_iter_kernel(PcgState* st, double* hist) {
  if (st->done) return;
  pcg_end_iteration(st, hist);
}

// x += alpha p (this iteration's alpha, always); convergence test on
// sqrt(gamma); unless converged p = dinv .* r + beta p with beta = rho'/rho
__global__ void __launch_bounds__(kThreads) cg_p_kernel(int64_t n, const double* __restrict__ dinv,
                            const double* __restrict__ r, double* __restrict__ p,
                            double* __restrict__ x, PcgState* st, double* hist,
                            const PeerSync ps) {
  __shared__ int flag;
  __shared__ double s_rg[2];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  if (ps.c.P > 1) {   // global (rho', gamma) from the peers' mailboxes
    if (threadIdx.x == 0) ar_wait_sum(ps.c, AR_RG, ps.e_wait, 2, s_rg);
  } else if (threadIdx.x == 0) {
    s_rg[0] = st->rho_new;
    s_rg[1] = st->gamma;
  }
  __syncthreads();
  const double rho_new = s_rg[0], gamma = s_rg[1];
  const double sigma = st->sigma;
  const double alpha = st->rho_old / sigma;   // sigma > 0 (else the update ended the solve)
  const double g = sqrt(gamma);
  const bool conv = g <= st->tol;
  const bool bad = !(g == g) || !(rho_new == rho_new);
  const bool newp = !conv && !bad;
  const double beta = rho_new / st->rho_old;
  const int64_t n2 = n >> 1;
  const double2* r2 = reinterpret_cast<const double2*>(r);
  const double2* d2 = reinterpret_cast<const double2*>(dinv);
  double2* p2 = reinterpret_cast<double2*>(p);
  double2* x2 = reinterpret_cast<double2*>(x);
  if (newp) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n2;
         q += (int64_t)gridDim.x * blockDim.x) {
      const double2 rv = __ldcg(&r2[q]);
      const double2 dv = __ldcs(&d2[q]);
      double2 pv = __ldcs(&p2[q]);
      double2 xv = __ldcs(&x2[q]);
      xv.x = fma(alpha, pv.x, xv.x);
      xv.y = fma(alpha, pv.y, xv.y);
      __stcs(&x2[q], xv);
      pv.x = fma(beta, pv.x, dv.x * rv.x);
      pv.y = fma(beta, pv.y, dv.y * rv.y);
      p2[q] = pv;
    }
  } else {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n2;
         q += (int64_t)gridDim.x * blockDim.x) {
      const double2 pv = __ldcs(&p2[q]);
      double2 xv = __ldcs(&x2[q]);
      xv.x = fma(alpha, pv.x, xv.x);
      xv.y = fma(alpha, pv.y, xv.y);
      __stcs(&x2[q], xv);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    x[l] = fma(alpha, p[l], x[l]);
    if (newp) p[l] = fma(beta, p[l], dinv[l] * r[l]);
  }
  // last block advances the iteration state
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(&st->tickets[3], 1u);
    flag = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (flag && threadIdx.x == 0) {
    st->tickets[3] = 0u;
    st->rho_new = rho_new;
    st->gamma = gamma;
    const int it = st->it + 1;
    st->it = it;
    hist[it] = g;
    if (bad) {
      st->done = 3;
      st->iters = it;
    } else if (conv) {
      st->done = 1;
      st->iters = it;
    } else {
      st->rho_old = rho_new;
      if (it >= st->maxit) {
        st->done = 4;
        st->iters = it;
      }
    }
  }
}

// true residual: sqrt(sum c (b - A x)^2) -> st->res_true (after allreduce by the host)
__global__ void cg_residual_kernel(int64_t n, const uint8_t* __restrict__ mult,
                                   const double* __restrict__ b, const double* __restrict__ w,
                                   double* partial, PcgState* st, double* out1,
                                   const PeerSync ps) {
  __shared__ double scratch[32];
  __shared__ int flag;
  double s = 0.0;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x) {
    const double d = b[l] - w[l];
    s = fma(c_of(mult[l]) * d, d, s);
  }
  double v[1] = {s};
  if (grid_reduce<1>(v, partial, &st->tickets[4], out1, scratch, &flag) && ps.c.P > 1 &&
      threadIdx.x == 0)
    ar_publish(ps.c, AR_RES, ps.e_pub, out1, 1);
}

inline int grid_for(int64_t work, int cap = 148 * 8) {
  int64_t g = (work + kThreads - 1) / kThreads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace dev

using dev::kThreads;
using dev::grid_for;

cudaError_t launch_geom(const DevPlan& P, const double* xi, const double* wq, int64_t e_lo, int ex,
                        int ey, int ez, const double* box, int deform, double amp, double* G,
                        double* B, int* bad, cudaStream_t s) {
  dev::Box b{box[0], box[1], box[2], box[3], box[4], box[5]};
  dev::geom_kernel<<<grid_for(P.n_local), kThreads, 0, s>>>(P.n, P.n_local, xi, wq, P.D, e_lo, ex,
                                                            ey, ez, b, deform, amp, G, B, bad);
  return cudaGetLastError();
}

cudaError_t launch_coords(const DevPlan& P, const double* xi, int64_t e_lo, int ex, int ey, int ez,
                          const double* box, int deform, double amp, double* X, double* Y,
                          double* Z, cudaStream_t s) {
  dev::Box b{box[0], box[1], box[2], box[3], box[4], box[5]};
  dev::coords_kernel<<<grid_for(P.n_local), kThreads, 0, s>>>(P.n, P.n_local, xi, e_lo, ex, ey, ez,
                                                              b, deform, amp, X, Y, Z);
  return cudaGetLastError();
}

cudaError_t launch_diag(const DevPlan& P, const double* G, double* d, cudaStream_t s) {
  dev::diag_kernel<<<grid_for(P.n_local), kThreads, 0, s>>>(P.n, P.n_local, P.D, G, d);
  return cudaGetLastError();
}

cudaError_t launch_mult(const DevPlan& P, uint8_t* mult, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(mult, 1, (size_t)P.n_local, s);
  if (e != cudaSuccess) return e;
  const int64_t N = P.N;
  const int64_t tot = P.nF * (N - 1) * (N - 1) + P.nEd * (N - 1) + P.nV + P.nS;
  if (tot == 0) return cudaSuccess;
  dev::mult_kernel<<<grid_for(tot), kThreads, 0, s>>>(P, mult);
  return cudaGetLastError();
}

cudaError_t launch_invert_mask(const DevPlan& P, double* d, cudaStream_t s) {
  dev::invert_mask_kernel<<<grid_for(P.n_local), kThreads, 0, s>>>(P, d);
  return cudaGetLastError();
}

cudaError_t launch_mask(const DevPlan& P, double* u, cudaStream_t s) {
  dev::mask_kernel<<<grid_for(P.n_local), kThreads, 0, s>>>(P, u);
  return cudaGetLastError();
}

cudaError_t launch_export_mask(const DevPlan& P, uint8_t* m, cudaStream_t s) {
  dev::export_mask_kernel<<<grid_for(P.n_local), kThreads, 0, s>>>(P, m);
  return cudaGetLastError();
}

cudaError_t launch_helm_diag(double* d, const double* B, double h1, double h2, int64_t n,
                             cudaStream_t s) {
  dev::helm_diag_kernel<<<grid_for(n), kThreads, 0, s>>>(d, B, h1, h2, n);
  return cudaGetLastError();
}

cudaError_t launch_scale_mask(const DevPlan& P, const double* B, const double* f, double* b,
                              cudaStream_t s) {
  dev::scale_mask_kernel<<<grid_for(P.n_local), kThreads, 0, s>>>(P, B, f, b);
  return cudaGetLastError();
}

cudaError_t launch_scale(const double* B, const double* f, double* b, int64_t n, cudaStream_t s) {
  dev::scale_kernel<<<grid_for(n), kThreads, 0, s>>>(B, f, b, n);
  return cudaGetLastError();
}

cudaError_t launch_sub_scalar(double* a, const double* scal, int64_t n, cudaStream_t s) {
  dev::sub_scalar_kernel<<<grid_for(n), kThreads, 0, s>>>(a, scal, n);
  return cudaGetLastError();
}

cudaError_t launch_gs_local(const DevPlan& P, double* u, int apply_mask, uint64_t* base,
                            int mode, cudaStream_t s, const GsSigma* sig_in) {
  const GsSigma sig = sig_in ? *sig_in : GsSigma{};
  const int64_t N = P.N;
  const int64_t tot = P.nF * (N - 1) * (N - 1) + P.nEd * (N - 1) + P.nV;
  if (tot == 0 && !sig.part) return cudaSuccess;
  // co-resident grid (x SEM_GS_GRIDX); chunk mode: blocks pull element chunks
  static std::atomic<int> cache[kMaxDev][2];
  const int dev = device_index();
  int resident[2] = {cache[dev][0].load(std::memory_order_relaxed),
                     cache[dev][1].load(std::memory_order_relaxed)};
  if (resident[0] == 0 || resident[1] == 0) {
    int sms = 148, nb0 = 1, nb1 = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb0, dev::gs_local_kernel<8, false>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb1, dev::gs_local_kernel<8, true>, kThreads, 0);
    resident[0] = std::max(nb0, 1) * sms * SEM_GS_GRIDX;
    resident[1] = std::max(nb1, 1) * sms * SEM_GS_GRIDX;
    cache[dev][0].store(resident[0], std::memory_order_relaxed);
    cache[dev][1].store(resident[1], std::memory_order_relaxed);
  }
  const int ce = dev::gs_mode_ce(P, mode);
  // flat: enough threads for one round (F face points, FE edge points, one vertex each)
  const int64_t need = std::max(std::max<int64_t>((P.nF * (N - 1) * (N - 1) + dev::kGsF - 1) / dev::kGsF,
                                                 (P.nEd * (N - 1) + dev::kGsFE - 1) / dev::kGsFE),
                                (int64_t)P.nV);
  const int g = ce > 0 ? std::max(1, std::min(resident[1], (P.nloc + ce - 1) / ce))
                       : grid_for(need, resident[0]);
  const unsigned long long b = *base;
  *base += (uint64_t)dev::gs_sweep_tickets(P.nloc, ce, g);
#define GS_LAUNCH(k)                                                                        \
  return ce > 0 ? launch_k(dev::gs_local_kernel<k, true>, dim3(g), dim3(kThreads), 0, s, P, u, \
                           apply_mask, b, ce, sig)                                             \
                : launch_k(dev::gs_local_kernel<k, false>, dim3(g), dim3(kThreads), 0, s, P, u, \
                           apply_mask, b, ce, sig)
  switch (P.n) {
    case 2: GS_LAUNCH(2);
    case 3: GS_LAUNCH(3);
    case 4: GS_LAUNCH(4);
    case 5: GS_LAUNCH(5);
    case 6: GS_LAUNCH(6);
    case 7: GS_LAUNCH(7);
    case 8: GS_LAUNCH(8);
    case 9: GS_LAUNCH(9);
    case 10: GS_LAUNCH(10);
    case 11: GS_LAUNCH(11);
    case 12: GS_LAUNCH(12);
  }
#undef GS_LAUNCH
  return cudaGetLastError();
}

cudaError_t launch_gs_pack(const DevPlan& P, const double* u, double* part, double* sendbuf,
                           cudaStream_t s) {
  if (P.nS == 0) return cudaSuccess;
  dev::gs_pack_kernel<<<grid_for(P.nS), kThreads, 0, s>>>(P, u, part, sendbuf);
  return cudaGetLastError();
}

cudaError_t launch_gs_unpack(const DevPlan& P, double* u, const double* part, const double* recvbuf,
                             int apply_mask, PcgState* st, int nparts, cudaStream_t s) {
  dev::gs_unpack_kernel<<<grid_for(P.nS > 0 ? P.nS : 1), kThreads, 0, s>>>(P, u, part, recvbuf,
                                                                          apply_mask, st, nparts);
  return cudaGetLastError();
}

int cg_grid(int num_sms) { return num_sms * 4; }

cudaError_t launch_dot_c(const DevPlan& P, const uint8_t* mult, const double* a, const double* b,
                         double* partial, unsigned* ticket, double* out, int grid, cudaStream_t s) {
  dev::dot_c_kernel<<<grid, kThreads, 0, s>>>(P.n_local, mult, a, b, partial, ticket, out);
  return cudaGetLastError();
}

cudaError_t launch_sum_c(const DevPlan& P, const uint8_t* mult, const double* a, double* partial,
                         unsigned* ticket, double* out2, int grid, cudaStream_t s) {
  dev::sum_c_kernel<<<grid, kThreads, 0, s>>>(P.n_local, mult, a, partial, ticket, out2);
  return cudaGetLastError();
}

cudaError_t launch_cg_init(const DevPlan& P, const uint8_t* mult, const double* dinv, const double* b,
                           double* x, double* r, double* p, double* partial, PcgState* st,
                           double* out2, const PeerSync& ps, int grid, cudaStream_t s, int pzero) {
  dev::cg_init_kernel<<<grid, kThreads, 0, s>>>(P.n_local, mult, dinv, b, x, r, p, partial, st, out2,
                                                ps, pzero);
  return cudaGetLastError();
}

cudaError_t launch_cg_start(PcgState* st, double* hist, const PeerSync& ps, cudaStream_t s) {
  dev::cg_start_kernel<<<1, 1, 0, s>>>(st, hist, ps);
  return cudaGetLastError();
}

cudaError_t launch_cg_update(const DevPlan& P, const uint8_t* mult, const double* dinv, double* r,
                             const double* w, double* partial, PcgState* st, double* out2,
                             const double* sig_part, const int* sig_count, const PeerSync& ps,
                             int grid, cudaStream_t s, double* x, const double* p, double* hist,
                             int end_here, const int32_t* gu) {
  if (gu) {   // gather-scatter on read (PF iterations only)
    if (!x) return cudaErrorInvalidValue;
#define GUK(NN)                                                                                  \
  case NN:                                                                                       \
    return launch_k(dev::cg_update_kernel<true, NN>, dim3(grid), dim3(kThreads), 0, s, P.n_local, \
                    mult, dinv, r, w, partial, st, out2, sig_part, sig_count, ps, x, p, hist,    \
                    end_here, gu);
    switch (P.n) {
      GUK(2) GUK(3) GUK(4) GUK(5) GUK(6) GUK(7) GUK(8) GUK(9) GUK(10) GUK(11) GUK(12)
    }
#undef GUK
    return cudaErrorInvalidValue;
  }
  if (x)
    return launch_k(dev::cg_update_kernel<true, 0>, dim3(grid), dim3(kThreads), 0, s, P.n_local,
                    mult, dinv, r, w, partial, st, out2, sig_part, sig_count, ps, x, p, hist,
                    end_here, gu);
  return launch_k(dev::cg_update_kernel<false, 0>, dim3(grid), dim3(kThreads), 0, s, P.n_local,
                  mult, dinv, r, w, partial, st, out2, sig_part, sig_count, ps, x, p, hist,
                  end_here, gu);
}

cudaError_t launch_cg_end_iter(PcgState* st, double* hist, cudaStream_t s) {
  dev::cg_end_iter_kernel<<<1, 1, 0, s>>>(st, hist);
  return cudaGetLastError();
}

bool gs_flat(const DevPlan& P, int mode) { return dev::gs_mode_ce(P, mode) == 0; }

cudaError_t launch_cg_p(const DevPlan& P, const double* dinv, const double* r, double* p, double* x,
                        PcgState* st, double* hist, const PeerSync& ps, int grid, cudaStream_t s) {
  return launch_k(dev::cg_p_kernel, dim3(grid), dim3(kThreads), 0, s, P.n_local, dinv, r, p, x, st,
                  hist, ps);
}

cudaError_t launch_cg_residual(const DevPlan& P, const uint8_t* mult, const double* b,
                               const double* w, double* partial, PcgState* st, double* out1,
                               const PeerSync& ps, int grid, cudaStream_t s) {
  dev::cg_residual_kernel<<<grid, kThreads, 0, s>>>(P.n_local, mult, b, w, partial, st, out1, ps);
  return cudaGetLastError();
}

}  // namespace sem
