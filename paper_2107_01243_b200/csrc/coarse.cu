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

// ---- small coarse problems: the whole solve on ONE thread-block cluster
// (SEM_COARSE_CLUSTER): kCC CTAs of kCT2 threads, hardware cluster barriers
// between the phases, reductions through distributed shared memory (every CTA
// sums the CTAs' partials in rank order, so all take the same scalars and the
// same branch).  The unknowns' vectors stay in global memory (L2-resident).
constexpr int kCC = 8, kCT2 = 1024;

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ double cl_ld_remote(const double* local, unsigned rank) {
  unsigned a = (unsigned)__cvta_generic_to_shared(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
  return v;
}
// cluster total of v (slot h of the partial array); identical in every CTA
__device__ __forceinline__ double cl_reduce(double v, double* s_part, int h, double* scratch,
                                            double* s_tot) {
  const double bs = block_sum(v, scratch);
  if (threadIdx.x == 0) s_part[h] = bs;
  cl_sync();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (unsigned q = 0; q < kCC; q++) t += cl_ld_remote(&s_part[h], q);
    *s_tot = t;
  }
  __syncthreads();
  return *s_tot;
}

__global__ void __launch_bounds__(kCT2) casm_cluster_kernel(const CoarseAsm A, const double* __restrict__ b0,
                                                            double* __restrict__ x0, const int* gate,
                                                            int maxit, double rtol) {
  __shared__ double scratch[32];
  __shared__ double s_part[2];
  __shared__ double s_tot;
  if (gate && *gate) return;   // every CTA of the cluster alike
  const int tid = (int)cl_rank() * blockDim.x + threadIdx.x, nth = kCC * blockDim.x;
  int h = 0;
  double s = 0.0;
  for (int g = tid; g < A.nu; g += nth) {
    const int q0 = A.u2s_ptr[g], q1 = A.u2s_ptr[g + 1];
    SEM_CHK(q1 > q0 && q1 - q0 <= 8);
    double v = b0[A.u2s[q0]];
    for (int q = q0 + 1; q < q1; q++) v += b0[A.u2s[q]];
    A.b[g] = v;
    s += v;
  }
  const double sum = cl_reduce(s, s_part, h, scratch, &s_tot);
  h ^= 1;
  const double mean = A.periodic ? sum / (double)A.nu : 0.0;
  double gg = 0.0;
  for (int g = tid; g < A.nu; g += nth) {
    const double r = A.b[g] - mean;
    A.r[g] = r;
    A.p[g] = r;
    A.x[g] = 0.0;
    gg = fma(r, r, gg);
  }
  double gamma = cl_reduce(gg, s_part, h, scratch, &s_tot);
  h ^= 1;
  const double tol = rtol * sqrt(gamma);
  const bool run = !(sqrt(gamma) <= tol) && maxit > 0;
  for (int it = 0; run && it < maxit; it++) {
    double sg = 0.0;
    for (int g = tid; g < A.nu; g += nth) {
      double acc = 0.0;
      for (int k = 0; k < A.K; k++) {
        const int64_t e = (int64_t)k * A.nu + g;
        acc = fma(A.val[e], A.p[A.col[e]], acc);
      }
      A.q[g] = acc;
      sg = fma(A.p[g], acc, sg);
    }
    const double sigma = cl_reduce(sg, s_part, h, scratch, &s_tot);
    h ^= 1;
    if (!(sigma > 0.0)) break;   // breakdown: keep the current iterate
    const double alpha = gamma / sigma;
    double gn = 0.0;
    for (int g = tid; g < A.nu; g += nth) {
      A.x[g] = fma(alpha, A.p[g], A.x[g]);
      const double r = fma(-alpha, A.q[g], A.r[g]);
      A.r[g] = r;
      gn = fma(r, r, gn);
    }
    const double gnew = cl_reduce(gn, s_part, h, scratch, &s_tot);
    h ^= 1;
    if (!(gnew == gnew) || sqrt(gnew) <= tol || it + 1 >= maxit) break;
    const double beta = gnew / gamma;
    gamma = gnew;
    for (int g = tid; g < A.nu; g += nth) A.p[g] = fma(beta, A.p[g], A.r[g]);
    cl_sync();   // p complete before the next product
  }
  cl_sync();     // x complete (and no CTA exits while others read its shared partials)
  for (int64_t q = tid; q < A.n0; q += nth) {
    const int g = A.uidx[q];
    x0[q] = g >= 0 ? A.x[g] : 0.0;
  }
}

}  // namespace dev

bool coarse_asm_cluster_ok(int nu) { return nu <= kCoarseClusterMax; }

cudaError_t launch_coarse_asm_cluster(const CoarseAsm& A, const double* b0, double* x0,
                                      const int* gate, int maxit, double rtol, cudaStream_t s,
                                      int64_t* launches) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(dev::kCC);
  cfg.blockDim = dim3(dev::kCT2);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = dev::kCC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (launches) *launches += 1;
  return cudaLaunchKernelEx(&cfg, dev::casm_cluster_kernel, A, b0, x0, gate, maxit, rtol);
}

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
