// Assembled coarse operator of the two-level Schwarz preconditioner (SURVEY
// 8(f) NEXT-1; "the coarse grid (on linear elements) is solved for
// using an approximate Krylov solver, in essence performing few (~10) CG
// iterations"; readings Q30, Q31, Q35 in DESIGN.md).
//
// On one rank (and on every rank of the replicated coarse level) the N = 1
// operator A0 is assembled once at setup on its unique unmasked vertices (ELL,
// <= 27 entries per row, api.cu coarse_assemble) and the ten CG steps run on
// those nu unknowns: per step one SpMV pass (12 B per entry) and three vector
// passes over nu values, instead of the N = 1 element operator, the
// gather-scatter of all 8 E slots and the c-weighted vector kernels over 8 nu
// slots.  Same Krylov iterates in exact arithmetic as the E-vector CG of
// kern.cu (the c-weighted dots over slots are the dots over unique points);
// all reductions deterministic (fixed-order grid reductions).
//
// Kernels (all no-ops once st->done; done = 5 when the gate says the outer
// iteration has converged, so a gated preconditioner costs ~20 empty launches):
//   init:    done = gate ? 5 : 0, it = 0
//   gather:  b[g] = sum of b0 over g's slots (ascending) ; sum_g b[g]
//   start:   r = b - mean (fully periodic: b in range(A0), reading Q30), x = 0,
//            p = r, gamma = <r, r>, tol = rtol sqrt(gamma)
//   spmv:    q = A0 p, sigma = <p, q>, alpha = gamma / sigma
//   update:  x += alpha p, r -= alpha q, gamma' = <r, r>, convergence, beta
//   p:       p = r + beta p
//   scatter: x0[slot] = x[g(slot)] (0 on masked slots)
#include <cstdint>

#include "dev_common.cuh"
#include "kernels.h"

namespace sem {
namespace dev {

constexpr int kCT = 256;

__global__ void casm_init_kernel(CoarseCg* st, const int* gate, int maxit) {
  st->done = (gate && *gate) ? 5 : 0;
  st->it = 0;
  st->maxit = maxit;
}

__global__ void __launch_bounds__(kCT) casm_gather_kernel(const CoarseAsm A, const double* __restrict__ b0) {
  __shared__ double scratch[32];
  __shared__ int flag;
  if (A.st->done) return;
  double s = 0.0;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < A.nu; g += gridDim.x * blockDim.x) {
    const int q0 = A.u2s_ptr[g], q1 = A.u2s_ptr[g + 1];
    SEM_CHK(q1 > q0 && q1 - q0 <= 8);
    for (int q = q0; q < q1; q++)
      SEM_CHK(A.u2s[q] >= 0 && A.u2s[q] < A.n0 && (q == q0 || A.u2s[q] > A.u2s[q - 1]));
    double v = b0[A.u2s[q0]];
    for (int q = q0 + 1; q < q1; q++) v += b0[A.u2s[q]];
    A.b[g] = v;
    s += v;
  }
  double v1[1] = {s};
  grid_reduce<1>(v1, A.partial, &A.st->ticket[0], &A.st->mean, scratch, &flag);
}

__global__ void __launch_bounds__(kCT) casm_start_kernel(const CoarseAsm A, double rtol) {
  __shared__ double scratch[32];
  __shared__ int flag;
  if (A.st->done) return;
  const double mean = A.periodic ? A.st->mean / (double)A.nu : 0.0;
  double gg = 0.0;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < A.nu; g += gridDim.x * blockDim.x) {
    const double r = A.b[g] - mean;
    A.r[g] = r;
    A.p[g] = r;
    A.x[g] = 0.0;
    gg = fma(r, r, gg);
  }
  double v1[1] = {gg};
  if (grid_reduce<1>(v1, A.partial, &A.st->ticket[1], &A.st->gamma, scratch, &flag) &&
      threadIdx.x == 0) {
    const double g = sqrt(A.st->gamma);
    A.st->tol = rtol * g;
    A.st->done = (g <= A.st->tol) ? 1 : (A.st->maxit == 0 ? 4 : 0);
  }
}

// q = A0 p (ELL, entries of a row in ascending column order), sigma = <p, q>
__global__ void __launch_bounds__(kCT) casm_spmv_kernel(const CoarseAsm A) {
  __shared__ double scratch[32];
  __shared__ int flag;
  if (A.st->done) return;
  double sg = 0.0;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < A.nu; g += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < A.K; k++) {
      const int64_t e = (int64_t)k * A.nu + g;
      SEM_CHK(A.col[e] >= 0 && A.col[e] < A.nu);
      acc = fma(A.val[e], A.p[A.col[e]], acc);
    }
    A.q[g] = acc;
    sg = fma(A.p[g], acc, sg);
  }
  double v1[1] = {sg};
  if (grid_reduce<1>(v1, A.partial, &A.st->ticket[2], &A.st->sigma, scratch, &flag) &&
      threadIdx.x == 0) {
    const double sigma = A.st->sigma;
    if (sigma > 0.0) {
      A.st->alpha = A.st->gamma / sigma;
    } else {   // breakdown guard (also NaN): stop with the current iterate
      A.st->done = 2;
    }
  }
}

__global__ void __launch_bounds__(kCT) casm_update_kernel(const CoarseAsm A) {
  __shared__ double scratch[32];
  __shared__ int flag;
  if (A.st->done) return;
  const double alpha = A.st->alpha;
  double gg = 0.0;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < A.nu; g += gridDim.x * blockDim.x) {
    A.x[g] = fma(alpha, A.p[g], A.x[g]);
    const double r = fma(-alpha, A.q[g], A.r[g]);
    A.r[g] = r;
    gg = fma(r, r, gg);
  }
  double v1[1] = {gg};
  if (grid_reduce<1>(v1, A.partial, &A.st->ticket[3], &A.st->red, scratch, &flag) &&
      threadIdx.x == 0) {
    CoarseCg* st = A.st;
    const double gn = st->red;
    st->it++;
    if (!(gn == gn)) {
      st->done = 3;
    } else if (sqrt(gn) <= st->tol) {
      st->done = 1;
    } else {
      st->beta = gn / st->gamma;
      st->gamma = gn;
      if (st->it >= st->maxit) st->done = 4;
    }
  }
}

__global__ void __launch_bounds__(kCT) casm_p_kernel(const CoarseAsm A) {
  if (A.st->done) return;
  const double beta = A.st->beta;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < A.nu; g += gridDim.x * blockDim.x)
    A.p[g] = fma(beta, A.p[g], A.r[g]);
}

__global__ void __launch_bounds__(kCT) casm_scatter_kernel(const CoarseAsm A, double* __restrict__ x0) {
  if (A.st->done == 5) return;   // gated: the preconditioner application is a no-op
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < A.n0;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int g = A.uidx[s];
    SEM_CHK(g >= -1 && g < A.nu);
    x0[s] = g >= 0 ? A.x[g] : 0.0;
  }
}

}  // namespace dev

int coarse_asm_grid(int nu, int num_sms) {
  const int g = (nu + dev::kCT - 1) / dev::kCT;
  return g < 1 ? 1 : (g > 4 * num_sms ? 4 * num_sms : g);
}

cudaError_t launch_coarse_asm_solve(const CoarseAsm& A, const double* b0, double* x0,
                                    const int* gate, int maxit, double rtol, int grid,
                                    cudaStream_t s, int64_t* launches) {
  const int gs = (int)((A.n0 + dev::kCT - 1) / dev::kCT) < 4 * grid
                     ? (int)((A.n0 + dev::kCT - 1) / dev::kCT) : 4 * grid;
  dev::casm_init_kernel<<<1, 1, 0, s>>>(A.st, gate, maxit);
  dev::casm_gather_kernel<<<grid, dev::kCT, 0, s>>>(A, b0);
  dev::casm_start_kernel<<<grid, dev::kCT, 0, s>>>(A, rtol);
  for (int q = 0; q < maxit; q++) {
    dev::casm_spmv_kernel<<<grid, dev::kCT, 0, s>>>(A);
    dev::casm_update_kernel<<<grid, dev::kCT, 0, s>>>(A);
    if (q + 1 < maxit) dev::casm_p_kernel<<<grid, dev::kCT, 0, s>>>(A);
  }
  dev::casm_scatter_kernel<<<gs < 1 ? 1 : gs, dev::kCT, 0, s>>>(A, x0);
  if (launches) *launches += 4 + 3 * (int64_t)maxit - (maxit > 0 ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace sem
