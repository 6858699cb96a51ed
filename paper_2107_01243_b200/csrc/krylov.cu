// Restarted GMRES and the solution-projection space on the device (SURVEY
// 8(f) NEXT-3; Table 2 "GMRES ... Projections 20"; Fischer
// 1998).  HBM-bound BLAS-1 work fused per pass:
//   * mdot: k c-weighted dots <a, V_i>_c of one vector against k basis vectors
//     in one read of a and the k vectors ((k+1)*8 B/pt), per-block partials
//     summed in a fixed order by the last block (deterministic);
//   * maxpy: y += alpha * D * sum_i coef_i V_i (D = dinv or 1), optionally with
//     the c-weighted squared norm of the result in the same pass;
//   * the Hessenberg / Givens bookkeeping runs in one device thread on a
//     device-resident state, so an Arnoldi step needs no host round trip.
// Arnoldi orthogonalisation is classical Gram-Schmidt applied twice (CGS2):
// two fused passes instead of the oracle's j+1 sequential MGS updates; equal
// in exact arithmetic, and as stable as MGS with the second pass.
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "dev_common.cuh"
#include "kernels.h"

namespace sem {
namespace dev {

constexpr int kKT = 256;   // threads per block of the vector kernels

__device__ __forceinline__ double c_of_k(uint8_t m) { return __drcp_rn((double)m); }

// fixed-order reduction of K per-block partials (part[b*K + i]) by the last
// block to arrive; returns true in that block (after out[] is written)
template <int KMAX>
__device__ __forceinline__ void reduce_cols(const double* acc, int K, double* part, unsigned* ticket,
                                            double* out, double* s_w) {
  __shared__ int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < KMAX; i++) {   // compile-time indices keep acc[] in registers
    if (i < K) {
      double v = warp_sum(acc[i]);
      if (lane == 0) s_w[warp * KMAX + i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double v = s_w[threadIdx.x];
    for (int q = 1; q < nw; q++) v += s_w[q * KMAX + threadIdx.x];
    part[(size_t)blockIdx.x * K + threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the last block sums the per-block partials of each column with all its
  // threads (a fixed block-to-thread assignment and a fixed tree: deterministic);
  // a single thread per column walking all blocks serialised ~600 L2 round trips
  for (int i = 0; i < K; i++) {
    double v = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
      v += __ldcg(&part[(size_t)b * K + i]);
    v = warp_sum(v);
    __syncthreads();   // s_w reuse
    if (lane == 0) s_w[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < nw; q++) t += s_w[q];
      out[i] = t;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// All vector kernels work on point PAIRS (16-byte loads and stores; ldv is
// even, see api.cu) and unroll the grid-stride loop UN times with every load
// of the unrolled body issued first: with one double per thread and
// iteration, a small K left only K+2 loads in flight per thread and the
// kernels ran at 1.1-2.4 TB/s (ncu, C3).  An odd n has its last point done by
// block 0 / thread 0.
__device__ __forceinline__ double2 ld2cs(const double* p, int64_t q) {
  return __ldcs(reinterpret_cast<const double2*>(p) + q);
}

// out[i] = <a, V_i>_c, i < K (V_i = V + i*ldv); skipped when *done
template <int KMAX, int UN>
__global__ void __launch_bounds__(kKT, 2) mdot_kernel(int64_t n, const uint8_t* __restrict__ mult,
                                                   const double* __restrict__ a,
                                                   const double* __restrict__ V, int64_t ldv, int K,
                                                   double* part, unsigned* ticket, double* out,
                                                   const int* done) {
  __shared__ double s_w[(kKT / 32) * KMAX];
  if (done && *done) return;
  double acc[KMAX];
#pragma unroll
  for (int i = 0; i < KMAX; i++) acc[i] = 0.0;
  const int64_t np = n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q0 < np; q0 += UN * stride) {
    double2 av[UN], vv[UN][KMAX];
    uchar2 mv[UN];
#pragma unroll
    for (int u = 0; u < UN; u++) {
      const int64_t q = q0 + u * stride;
      if (q < np) {
        av[u] = ld2cs(a, q);
        mv[u] = reinterpret_cast<const uchar2*>(mult)[q];
#pragma unroll
        for (int i = 0; i < KMAX; i++)
          if (i < K) vv[u][i] = ld2cs(V + i * ldv, q);
      }
    }
#pragma unroll
    for (int u = 0; u < UN; u++) {
      if (q0 + u * stride < np) {
        const double ca0 = c_of_k(mv[u].x) * av[u].x, ca1 = c_of_k(mv[u].y) * av[u].y;
#pragma unroll
        for (int i = 0; i < KMAX; i++)
          if (i < K) acc[i] = fma(ca1, vv[u][i].y, fma(ca0, vv[u][i].x, acc[i]));
      }
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    const double ca = c_of_k(mult[l]) * a[l];
#pragma unroll
    for (int i = 0; i < KMAX; i++)
      if (i < K) acc[i] = fma(ca, V[i * ldv + l], acc[i]);
  }
  reduce_cols<KMAX>(acc, K, part, ticket, out, s_w);
}

// y += alpha * (dinv ? dinv : 1) * sum_{i<K} coef[i] V_i ; NORM: out_norm = <y, y>_c
template <int KMAX, bool NORM, int UN>
__global__ void __launch_bounds__(kKT, 2) maxpy_kernel(int64_t n, double* __restrict__ y,
                                                    const double* __restrict__ V, int64_t ldv, int K,
                                                    const double* __restrict__ coef, double alpha,
                                                    const double* __restrict__ dinv,
                                                    const uint8_t* __restrict__ mult, double* part,
                                                    unsigned* ticket, double* out_norm,
                                                    const int* done) {
  __shared__ double s_w[(kKT / 32) * 1];
  __shared__ double s_c[KMAX];
  if (done && *done) return;
  if (threadIdx.x < K) s_c[threadIdx.x] = alpha * coef[threadIdx.x];
  __syncthreads();
  double nrm[1] = {0.0};
  const int64_t np = n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
  double2* y2 = reinterpret_cast<double2*>(y);
  for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q0 < np; q0 += UN * stride) {
    double2 yv[UN], dv[UN], vv[UN][KMAX];
    uchar2 mv[UN];
#pragma unroll
    for (int u = 0; u < UN; u++) {
      const int64_t q = q0 + u * stride;
      if (q < np) {
        yv[u] = y2[q];
        if (dinv) dv[u] = ld2cs(dinv, q);
        if (NORM) mv[u] = reinterpret_cast<const uchar2*>(mult)[q];
#pragma unroll
        for (int i = 0; i < KMAX; i++)
          if (i < K) vv[u][i] = ld2cs(V + i * ldv, q);
      }
    }
#pragma unroll
    for (int u = 0; u < UN; u++) {
      const int64_t q = q0 + u * stride;
      if (q < np) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int i = 0; i < KMAX; i++)
          if (i < K) {
            s0 = fma(s_c[i], vv[u][i].x, s0);
            s1 = fma(s_c[i], vv[u][i].y, s1);
          }
        double2 v;
        v.x = yv[u].x + (dinv ? dv[u].x * s0 : s0);
        v.y = yv[u].y + (dinv ? dv[u].y * s1 : s1);
        y2[q] = v;
        if (NORM) {
          nrm[0] = fma(c_of_k(mv[u].x) * v.x, v.x, nrm[0]);
          nrm[0] = fma(c_of_k(mv[u].y) * v.y, v.y, nrm[0]);
        }
      }
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    double sacc = 0.0;
    for (int i = 0; i < K; i++) sacc = fma(s_c[i], V[i * ldv + l], sacc);
    const double v = y[l] + (dinv ? dinv[l] * sacc : sacc);
    y[l] = v;
    if (NORM) nrm[0] = fma(c_of_k(mult[l]) * v, v, nrm[0]);
  }
  if (NORM) reduce_cols<1>(nrm, 1, part, ticket, out_norm, s_w);
}

// Fused CGS2 middle pass: y -= sum_i coef[i] V_i, then out[i] = <y_new, V_i>_c
// in the same sweep (each V_i is loaded once for both), so an Arnoldi step
// reads the basis three times instead of four.  K <= KMAX (no slicing: the
// dots need the final y).
template <int KMAX>
__global__ void __launch_bounds__(kKT, 1) maxpy_mdot_kernel(int64_t n, double* __restrict__ y,
                                                            const double* __restrict__ V,
                                                            int64_t ldv, int K,
                                                            const double* __restrict__ coef,
                                                            const uint8_t* __restrict__ mult,
                                                            double* part, unsigned* ticket,
                                                            double* out, const int* done) {
  __shared__ double s_w[(kKT / 32) * KMAX];
  __shared__ double s_c[KMAX];
  if (done && *done) return;
  if (threadIdx.x < K) s_c[threadIdx.x] = -coef[threadIdx.x];
  __syncthreads();
  double acc[KMAX];
#pragma unroll
  for (int i = 0; i < KMAX; i++) acc[i] = 0.0;
  const int64_t np = n >> 1, stride = (int64_t)gridDim.x * blockDim.x;
  double2* y2 = reinterpret_cast<double2*>(y);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < np; q += stride) {
    double2 vv[KMAX];
    const double2 yv = y2[q];
    const uchar2 mv = reinterpret_cast<const uchar2*>(mult)[q];
#pragma unroll
    for (int i = 0; i < KMAX; i++)
      if (i < K) vv[i] = ld2cs(V + i * ldv, q);
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int i = 0; i < KMAX; i++)
      if (i < K) {
        s0 = fma(s_c[i], vv[i].x, s0);
        s1 = fma(s_c[i], vv[i].y, s1);
      }
    const double2 v = make_double2(yv.x + s0, yv.y + s1);
    y2[q] = v;
    const double cv0 = c_of_k(mv.x) * v.x, cv1 = c_of_k(mv.y) * v.y;
#pragma unroll
    for (int i = 0; i < KMAX; i++)
      if (i < K) acc[i] = fma(cv1, vv[i].y, fma(cv0, vv[i].x, acc[i]));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    double sacc = 0.0;
    for (int i = 0; i < K; i++) sacc = fma(s_c[i], V[i * ldv + l], sacc);
    const double v = y[l] + sacc;
    y[l] = v;
    const double cv = c_of_k(mult[l]) * v;
#pragma unroll
    for (int i = 0; i < KMAX; i++)
      if (i < K) acc[i] = fma(cv, V[i * ldv + l], acc[i]);
  }
  reduce_cols<KMAX>(acc, K, part, ticket, out, s_w);
}

// v = (b - w) (restart residual) with its c-norm^2, or v = w with its c-norm^2
__global__ void __launch_bounds__(kKT) resid_kernel(int64_t n, const double* __restrict__ b,
                                                    const double* __restrict__ w,
                                                    double* __restrict__ v,
                                                    const uint8_t* __restrict__ mult, double* part,
                                                    unsigned* ticket, double* out, const int* done) {
  __shared__ double s_w[kKT / 32];
  if (done && *done) return;
  double acc[1] = {0.0};
  const int64_t np = n >> 1;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < np;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double2 wv = ld2cs(w, q);
    double2 rv = wv;
    if (b) {
      const double2 bv = ld2cs(b, q);
      rv.x = bv.x - wv.x;
      rv.y = bv.y - wv.y;
    }
    const uchar2 mv = reinterpret_cast<const uchar2*>(mult)[q];
    reinterpret_cast<double2*>(v)[q] = rv;
    acc[0] = fma(c_of_k(mv.x) * rv.x, rv.x, acc[0]);
    acc[0] = fma(c_of_k(mv.y) * rv.y, rv.y, acc[0]);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    const double r = b ? b[l] - w[l] : w[l];
    v[l] = r;
    acc[0] = fma(c_of_k(mult[l]) * r, r, acc[0]);
  }
  reduce_cols<1>(acc, 1, part, ticket, out, s_w);
}

// v = w / norm, t = dinv v (the next Arnoldi direction, preconditioned); v may be w
__global__ void __launch_bounds__(kKT) vnorm_kernel(int64_t n, const double* w, double* v,
                                                    double* __restrict__ t,
                                                    const double* __restrict__ dinv,
                                                    const GmresState* gs, const int* done) {
  if (done && *done) return;
  const double s = gs->inv_norm;
  const int64_t np = n >> 1;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < np;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double2 wv = reinterpret_cast<const double2*>(w)[q];
    const double2 x = make_double2(wv.x * s, wv.y * s);
    reinterpret_cast<double2*>(v)[q] = x;
    if (t) {
      const double2 dv = ld2cs(dinv, q);
      reinterpret_cast<double2*>(t)[q] = make_double2(dv.x * x.x, dv.y * x.y);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    const double x = w[l] * s;
    v[l] = x;
    if (t) t[l] = dinv[l] * x;
  }
}

// ---- single-reduction (Chronopoulos-Gear) Jacobi PCG (reading Q34)
// init: x = 0, r = b, u = dinv b, p = s = 0; partials of <r,u>_c and <r,r>_c
__global__ void __launch_bounds__(kKT) cgcg_init_kernel(int64_t n, const double* __restrict__ b,
                                                        const double* __restrict__ dinv,
                                                        const uint8_t* __restrict__ mult,
                                                        double* __restrict__ x, double* __restrict__ r,
                                                        double* __restrict__ u, double* __restrict__ p,
                                                        double* __restrict__ s, double* part,
                                                        unsigned* ticket, double* out2) {
  __shared__ double s_w[(kKT / 32) * 2];
  double acc[2] = {0.0, 0.0};
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x) {
    const double bl = b[l], ul = dinv[l] * bl, c = c_of_k(mult[l]);
    x[l] = 0.0;
    r[l] = bl;
    u[l] = ul;
    p[l] = 0.0;
    s[l] = 0.0;
    acc[0] = fma(c * bl, ul, acc[0]);
    acc[1] = fma(c * bl, bl, acc[1]);
  }
  reduce_cols<2>(acc, 2, part, ticket, out2, s_w);
}

// one pass: p = u + beta p; s = w + beta s; x += alpha p; r -= alpha s; u = dinv r;
// partials of gamma = <r,u>_c and eps = <r,r>_c.  Skipped when st->done.
__global__ void __launch_bounds__(kKT) cgcg_update_kernel(
    int64_t n, const double* __restrict__ dinv, const uint8_t* __restrict__ mult,
    double* __restrict__ u, const double* __restrict__ w, double* __restrict__ p,
    double* __restrict__ s, double* __restrict__ x, double* __restrict__ r, double* part,
    unsigned* ticket, double* out2, const PcgState* st) {
  __shared__ double s_w[(kKT / 32) * 2];
  if (st->done) return;
  const double alpha = st->alpha, beta = st->beta;
  double acc[2] = {0.0, 0.0};
  const int64_t np = n >> 1;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < np;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double2 uv = ld2cs(u, q), wv = ld2cs(w, q), dv = ld2cs(dinv, q);
    double2 pv = ld2cs(p, q), sv = ld2cs(s, q), xv = ld2cs(x, q), rv = ld2cs(r, q);
    const uchar2 mv = reinterpret_cast<const uchar2*>(mult)[q];
    pv.x = fma(beta, pv.x, uv.x);
    pv.y = fma(beta, pv.y, uv.y);
    sv.x = fma(beta, sv.x, wv.x);
    sv.y = fma(beta, sv.y, wv.y);
    xv.x = fma(alpha, pv.x, xv.x);
    xv.y = fma(alpha, pv.y, xv.y);
    rv.x = fma(-alpha, sv.x, rv.x);
    rv.y = fma(-alpha, sv.y, rv.y);
    const double2 un = make_double2(dv.x * rv.x, dv.y * rv.y);
    reinterpret_cast<double2*>(p)[q] = pv;
    reinterpret_cast<double2*>(s)[q] = sv;
    __stcs(reinterpret_cast<double2*>(x) + q, xv);
    reinterpret_cast<double2*>(r)[q] = rv;
    reinterpret_cast<double2*>(u)[q] = un;
    const double c0 = c_of_k(mv.x), c1 = c_of_k(mv.y);
    acc[0] = fma(c0 * rv.x, un.x, fma(c1 * rv.y, un.y, acc[0]));
    acc[1] = fma(c0 * rv.x, rv.x, fma(c1 * rv.y, rv.y, acc[1]));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t l = n - 1;
    const double pl = fma(beta, p[l], u[l]), sl = fma(beta, s[l], w[l]);
    p[l] = pl;
    s[l] = sl;
    x[l] = fma(alpha, pl, x[l]);
    const double rl = fma(-alpha, sl, r[l]), ul = dinv[l] * rl, c = c_of_k(mult[l]);
    r[l] = rl;
    u[l] = ul;
    acc[0] = fma(c * rl, ul, acc[0]);
    acc[1] = fma(c * rl, rl, acc[1]);
  }
  reduce_cols<2>(acc, 2, part, ticket, out2, s_w);
}

// scalars: cg3 = (gamma, eps, delta) of the current u, w.  stage 0: start;
// stage 1: after an update + operator application
__global__ void cgcg_scalar_kernel(int stage, PcgState* st, double* hist) {
  const double gamma = st->cg3[0], eps = st->cg3[1], delta = st->cg3[2];
  const double g = sqrt(eps);
  if (stage == 0) {
    st->it = 0;
    st->iters = 0;
    st->gamma = eps;
    hist[0] = g;
    st->beta = 0.0;
    st->rho_old = gamma;
    if (g <= st->tol) { st->done = 1; return; }
    if (!(delta > 0.0)) { st->done = 2; return; }
    st->alpha = gamma / delta;
    st->done = st->maxit == 0 ? 4 : 0;
    return;
  }
  if (st->done) return;
  const int it = st->it + 1;
  st->it = it;
  st->gamma = eps;
  hist[it] = g;
  if (!(g == g)) { st->done = 3; st->iters = it; return; }
  if (g <= st->tol) { st->done = 1; st->iters = it; return; }
  const double beta = gamma / st->rho_old;
  const double den = delta - beta * gamma / st->alpha;
  if (!(den > 0.0)) { st->done = 2; st->iters = it; return; }
  st->beta = beta;
  st->alpha = gamma / den;
  st->rho_old = gamma;
  if (it >= st->maxit) { st->done = 4; st->iters = it; }
}

// start of a cycle: beta = sqrt(norm2); converged if beta <= tol
__global__ void gm_start_kernel(GmresState* gs, PcgState* st, double* hist) {
  if (st->done) return;
  if (st->it == 0) gs->converged = 0;   // a new solve
  const double beta = sqrt(gs->norm2[0]);
  gs->j = 0;
  gs->g[0] = beta;
  for (int i = 1; i <= kGmMax; i++) gs->g[i] = 0.0;
  gs->res = beta;
  if (st->it == 0) hist[0] = beta;
  if (beta <= st->tol) {
    st->done = 1;
    st->iters = st->it;
    gs->cycle_done = 1;
    return;
  }
  if (st->it >= st->maxit) {
    st->done = 4;
    st->iters = st->it;
    gs->cycle_done = 1;
    return;
  }
  gs->inv_norm = 1.0 / beta;
  gs->cycle_done = 0;
}

// Arnoldi step j: H[0..j][j] = h1 + h2 (two CGS passes), H[j+1][j] = ||w||_c;
// Givens rotations; |g_{j+1}| = residual; cycle end at convergence, maxit or
// the restart length (the outer loop then solves H y = g and updates x)
__global__ void gm_arnoldi_kernel(GmresState* gs, PcgState* st, double* hist, int m) {
  if (st->done || gs->cycle_done) return;
  const int j = gs->j;
  double* H = gs->H;
  for (int i = 0; i <= j; i++) H[i * kGmMax + j] = gs->h1[i] + gs->h2[i];
  const double hn = sqrt(gs->norm2[0]);
  H[(j + 1) * kGmMax + j] = hn;
  for (int i = 0; i < j; i++) {
    const double a = H[i * kGmMax + j], b = H[(i + 1) * kGmMax + j];
    H[i * kGmMax + j] = gs->cs[i] * a + gs->sn[i] * b;
    H[(i + 1) * kGmMax + j] = -gs->sn[i] * a + gs->cs[i] * b;
  }
  const double a = H[j * kGmMax + j], b = H[(j + 1) * kGmMax + j];
  const double r = sqrt(a * a + b * b);
  gs->cs[j] = r > 0.0 ? a / r : 1.0;
  gs->sn[j] = r > 0.0 ? b / r : 0.0;
  H[j * kGmMax + j] = r;
  H[(j + 1) * kGmMax + j] = 0.0;
  gs->g[j + 1] = -gs->sn[j] * gs->g[j];
  gs->g[j] = gs->cs[j] * gs->g[j];
  const double res = fabs(gs->g[j + 1]);
  gs->res = res;
  const int it = st->it + 1;
  st->it = it;
  hist[it] = res;
  gs->j = j + 1;
  gs->inv_norm = hn > 0.0 ? 1.0 / hn : 0.0;
  const bool conv = res <= st->tol || hn == 0.0;
  if (conv || it >= st->maxit || j + 1 == m) gs->cycle_done = 1;
  if (conv) gs->converged = 1;
}

// y = H(0:j,0:j)^-1 g(0:j) (back substitution), jy = j; y beyond j zeroed
__global__ void gm_solve_kernel(GmresState* gs, PcgState* st, int m) {
  if (st->done) return;
  const int j = gs->j;
  for (int i = j; i < m; i++) gs->y[i] = 0.0;
  for (int i = j - 1; i >= 0; i--) {
    double s = gs->g[i];
    for (int q = i + 1; q < j; q++) s -= gs->H[i * kGmMax + q] * gs->y[q];
    gs->y[i] = s / gs->H[i * kGmMax + i];
  }
  gs->jy = j;
}

// after the x update: converged or out of iterations -> done
__global__ void gm_end_cycle_kernel(GmresState* gs, PcgState* st) {
  if (st->done) return;
  if (gs->converged) {
    st->done = 1;
    st->iters = st->it;
  } else if (st->it >= st->maxit) {
    st->done = 4;
    st->iters = st->it;
  }
}

}  // namespace dev

static int kgrid(int64_t n, int num_sms) {
  int64_t g = (n + dev::kKT - 1) / dev::kKT;
  const int cap = num_sms * 4;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

cudaError_t launch_mdot(int64_t n, const uint8_t* mult, const double* a, const double* V,
                        int64_t ldv, int K, double* part, unsigned* ticket, double* out,
                        const int* done, int num_sms, cudaStream_t s) {
  if (K > 1 && (ldv & 1)) return cudaErrorInvalidValue;   // pair accesses need an even ldv
  const int g = kgrid(n / 2 + 1, num_sms);
  for (int k0 = 0; k0 < K; k0 += 16) {   // > 16 vectors: slices of 16 (a is re-read)
    const int kk = std::min(16, K - k0);
    const double* Vk = V + k0 * ldv;
    if (kk <= 2)
      dev::mdot_kernel<2, 4><<<g, dev::kKT, 0, s>>>(n, mult, a, Vk, ldv, kk, part, ticket, out + k0,
                                                    done);
    else if (kk <= 8)
      dev::mdot_kernel<8, 2><<<g, dev::kKT, 0, s>>>(n, mult, a, Vk, ldv, kk, part, ticket, out + k0,
                                                    done);
    else
      dev::mdot_kernel<16, 1><<<g, dev::kKT, 0, s>>>(n, mult, a, Vk, ldv, kk, part, ticket,
                                                     out + k0, done);
  }
  return cudaGetLastError();
}

cudaError_t launch_maxpy(int64_t n, double* y, const double* V, int64_t ldv, int K,
                         const double* coef, double alpha, const double* dinv, const uint8_t* mult,
                         double* part, unsigned* ticket, double* out_norm, const int* done,
                         int num_sms, cudaStream_t s) {
  if (K > 1 && (ldv & 1)) return cudaErrorInvalidValue;
  const int g = kgrid(n / 2 + 1, num_sms);
  for (int k0 = 0; k0 < K; k0 += 16) {   // > 16 vectors: slices of 16 (y is re-read)
    const int kk = std::min(16, K - k0);
    const double* Vk = V + k0 * ldv;
    const double* ck = coef + k0;
    const bool nrm = out_norm != nullptr && k0 + 16 >= K;   // norm of the final y
    double* on = nrm ? out_norm : nullptr;
#define MAXPY(KM, UN)                                                                        \
  (nrm ? (dev::maxpy_kernel<KM, true, UN><<<g, dev::kKT, 0, s>>>(                             \
              n, y, Vk, ldv, kk, ck, alpha, dinv, mult, part, ticket, on, done),              \
          0)                                                                                 \
       : (dev::maxpy_kernel<KM, false, UN><<<g, dev::kKT, 0, s>>>(                            \
              n, y, Vk, ldv, kk, ck, alpha, dinv, mult, part, ticket, on, done),              \
          0))
    if (kk <= 2) MAXPY(2, 4);
    else if (kk <= 8) MAXPY(8, 2);
    else MAXPY(16, 1);
#undef MAXPY
  }
  return cudaGetLastError();
}

cudaError_t launch_maxpy_mdot(int64_t n, double* y, const double* V, int64_t ldv, int K,
                              const double* coef, const uint8_t* mult, double* part,
                              unsigned* ticket, double* out, const int* done, int num_sms,
                              cudaStream_t s) {
  if (K > 32 || (K > 1 && (ldv & 1))) return cudaErrorInvalidValue;
  const int g = kgrid(n / 2 + 1, num_sms);
  if (K <= 8)
    dev::maxpy_mdot_kernel<8><<<g, dev::kKT, 0, s>>>(n, y, V, ldv, K, coef, mult, part, ticket, out,
                                                     done);
  else if (K <= 16)
    dev::maxpy_mdot_kernel<16><<<g, dev::kKT, 0, s>>>(n, y, V, ldv, K, coef, mult, part, ticket,
                                                      out, done);
  else
    dev::maxpy_mdot_kernel<32><<<g, dev::kKT, 0, s>>>(n, y, V, ldv, K, coef, mult, part, ticket,
                                                      out, done);
  return cudaGetLastError();
}

cudaError_t launch_cgcg_init(int64_t n, const double* b, const double* dinv, const uint8_t* mult,
                             double* x, double* r, double* u, double* p, double* s, double* part,
                             unsigned* ticket, double* out2, int num_sms, cudaStream_t st) {
  dev::cgcg_init_kernel<<<kgrid(n, num_sms), dev::kKT, 0, st>>>(n, b, dinv, mult, x, r, u, p, s,
                                                                part, ticket, out2);
  return cudaGetLastError();
}

cudaError_t launch_cgcg_update(int64_t n, const double* dinv, const uint8_t* mult, double* u,
                               const double* w, double* p, double* s, double* x, double* r,
                               double* part, unsigned* ticket, double* out2, const PcgState* ps,
                               int num_sms, cudaStream_t st) {
  dev::cgcg_update_kernel<<<kgrid(n / 2 + 1, num_sms), dev::kKT, 0, st>>>(
      n, dinv, mult, u, w, p, s, x, r, part, ticket, out2, ps);
  return cudaGetLastError();
}

cudaError_t launch_cgcg_scalar(int stage, PcgState* ps, double* hist, cudaStream_t st) {
  dev::cgcg_scalar_kernel<<<1, 1, 0, st>>>(stage, ps, hist);
  return cudaGetLastError();
}

cudaError_t launch_resid(int64_t n, const double* b, const double* w, double* v,
                         const uint8_t* mult, double* part, unsigned* ticket, double* out,
                         const int* done, int num_sms, cudaStream_t s) {
  dev::resid_kernel<<<kgrid(n / 2 + 1, num_sms), dev::kKT, 0, s>>>(n, b, w, v, mult, part, ticket, out,
                                                          done);
  return cudaGetLastError();
}

cudaError_t launch_vnorm(int64_t n, const double* w, double* v, double* t, const double* dinv,
                         const GmresState* gs, const int* done, int num_sms, cudaStream_t s) {
  dev::vnorm_kernel<<<kgrid(n / 2 + 1, num_sms), dev::kKT, 0, s>>>(n, w, v, t, dinv, gs, done);
  return cudaGetLastError();
}

cudaError_t launch_gm_start(GmresState* gs, PcgState* st, double* hist, cudaStream_t s) {
  dev::gm_start_kernel<<<1, 1, 0, s>>>(gs, st, hist);
  return cudaGetLastError();
}

cudaError_t launch_gm_arnoldi(GmresState* gs, PcgState* st, double* hist, int m, cudaStream_t s) {
  dev::gm_arnoldi_kernel<<<1, 1, 0, s>>>(gs, st, hist, m);
  return cudaGetLastError();
}

cudaError_t launch_gm_solve(GmresState* gs, PcgState* st, int m, cudaStream_t s) {
  dev::gm_solve_kernel<<<1, 1, 0, s>>>(gs, st, m);
  return cudaGetLastError();
}

cudaError_t launch_gm_end_cycle(GmresState* gs, PcgState* st, cudaStream_t s) {
  dev::gm_end_cycle_kernel<<<1, 1, 0, s>>>(gs, st);
  return cudaGetLastError();
}

}  // namespace sem
