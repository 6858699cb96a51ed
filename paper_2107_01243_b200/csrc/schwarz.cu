// Two-level additive overlapping Schwarz preconditioner on the device (SURVEY
// 8(f) NEXT-1; "M0^-1 = R0^T A0^-1 R0 + sum_k R_k^T A~_k^-1 R_k",
// "the coarse grid (on linear elements) is solved for using an approximate
// Krylov solver, in essence performing few (~10) CG iterations"; readings
// Q28-Q32 in DESIGN.md).
//
// Local solves by fast diagonalisation (Lynch-Rice-Thomas; Fischer 1997,
// ref. [19]): the subdomain operator of element e is separable,
//   A~ = Bz (x) By (x) Ax + Bz (x) Ay (x) Bx + Az (x) By (x) Bx,
// with the element's 1-D SEM stiffness/mass extended by the neighbours' end
// entries (one node of overlap, Dirichlet beyond).  With the generalised
// eigenvectors S_d (S^T B S = I, S^T A S = Lambda) its inverse is
//   A~^-1 = (Sz (x) Sy (x) Sx) diag(1 / (lx_a + ly_b + lz_c)) (Sz (x) Sy (x) Sx)^T,
// six n x n contractions per element instead of an n^3 x n^3 solve.  The
// 1-D eigenproblems are solved once at setup on the device (cyclic Jacobi on
// B^-1/2 A B^-1/2, one thread per element and axis).  A node on a Dirichlet
// face is dropped from its 1-D problem (zero row and column of S), so the
// local solve ignores and returns zero on masked slots without a mask test.
//
// The same pass over r also forms the element's coarse restriction
// (J^T (x) J^T (x) J^T)(c r_e), J_ia = (1 -+ xi_i)/2 (8 values per element):
// r is read once for both levels.  The combine kernel scales the assembled
// local part by c^1/2 (reading Q29), adds the trilinear prolongation of the
// coarse solution and optionally forms the flexible-CG dots <z,r>_c, <z,w>_c.
//
// Roofline: HBM.  fdm_kernel moves 8 (r) + 1 (mult) + 8 (y) B/pt plus
// 24 (n^2 + n) B per element of factors; combine 8 + 8 + 1 (+16) B/pt.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "dev_common.cuh"
#include "kernels.h"

namespace sem {
namespace dev {

constexpr int kFT = 256;   // threads per block of the Schwarz kernels

// mean length of global element eg along axis a: the four element edges
// parallel to a, straight vertex-to-vertex distances (reading Q28)
__device__ double elem_len(const double* xi, int N, int ex, int ey, int ez, int64_t eg, int a,
                           const Box& b, int deform, double amp) {
  double s = 0.0;
  for (int u = 0; u < 2; u++)
    for (int v = 0; v < 2; v++) {
      int i0[3], i1[3];
      const int o1 = u * N, o2 = v * N;
      for (int d = 0; d < 3; d++) i0[d] = i1[d] = 0;
      i0[a] = 0;
      i1[a] = N;
      const int d1 = a == 0 ? 1 : 0, d2 = a == 2 ? 1 : 2;
      i0[d1] = i1[d1] = o1;
      i0[d2] = i1[d2] = o2;
      double p0[3], p1[3];
      node_xyz(xi, ex, ey, ez, eg, i0[0], i0[1], i0[2], b, deform, amp, p0);
      node_xyz(xi, ex, ey, ez, eg, i1[0], i1[1], i1[2], b, deform, amp, p1);
      const double dx = p1[0] - p0[0], dy = p1[1] - p0[1], dz = p1[2] - p0[2];
      s += sqrt(dx * dx + dy * dy + dz * dz);
    }
  return 0.25 * s;
}

// one thread per (local element, axis): extended 1-D operators, generalised
// eigenvectors S[el][a][i*n + mode] and eigenvalues lam[el][a][mode]
__global__ void fdm_setup_kernel(int n, int nloc, int64_t e_lo, int ex, int ey, int ez, Box b,
                                 int deform, double amp, int per0, int per1, int per2,
                                 const double* __restrict__ xi, const double* __restrict__ wq,
                                 const double* __restrict__ D, double* __restrict__ Sg,
                                 double* __restrict__ lamg) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * nloc) return;
  const int el = t / 3, a = t - 3 * el;
  const int N = n - 1;
  const int64_t eg = e_lo + el;
  const int64_t idx[3] = {eg % ex, (eg / ex) % ey, eg / ((int64_t)ex * ey)};
  const int64_t Ea[3] = {ex, ey, ez};
  const int per[3] = {per0, per1, per2};
  double M[144], V[144], Bd[12];
  const double h = elem_len(xi, N, ex, ey, ez, eg, a, b, deform, amp);
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) {
      double s = 0.0;
      for (int q = 0; q < n; q++) s += wq[q] * D[q * n + i] * D[q * n + j];
      M[i * n + j] = (2.0 / h) * s;
    }
  for (int i = 0; i < n; i++) Bd[i] = 0.5 * h * wq[i];
  bool keep[2] = {false, false};
  for (int side = 0; side < 2; side++) {
    int64_t q = idx[a] + (side ? 1 : -1);
    if (q < 0 || q >= Ea[a]) {
      if (!per[a]) continue;   // Dirichlet face: the end node is dropped
      q = (q + Ea[a]) % Ea[a];
    }
    keep[side] = true;
    int64_t nb[3] = {idx[0], idx[1], idx[2]};
    nb[a] = q;
    const int64_t en = nb[0] + ex * (nb[1] + (int64_t)ey * nb[2]);
    const double hn = elem_len(xi, N, ex, ey, ez, en, a, b, deform, amp);
    double s = 0.0;   // the neighbour's stiffness entry at its shared end node
    const int m = side ? 0 : N;
    for (int q2 = 0; q2 < n; q2++) s += wq[q2] * D[q2 * n + m] * D[q2 * n + m];
    const int e = side ? N : 0;
    M[e * n + e] += (2.0 / hn) * s;
    Bd[e] += 0.5 * hn * wq[m];
  }
  // B^-1/2 A B^-1/2 with the dropped nodes decoupled (zero rows and columns)
  for (int i = 0; i < n; i++) {
    const bool di = (i == 0 && !keep[0]) || (i == N && !keep[1]);
    for (int j = 0; j < n; j++) {
      const bool dj = (j == 0 && !keep[0]) || (j == N && !keep[1]);
      M[i * n + j] = (di || dj) ? 0.0 : M[i * n + j] / sqrt(Bd[i] * Bd[j]);
      V[i * n + j] = i == j ? 1.0 : 0.0;
    }
  }
  // cyclic Jacobi (Golub-Van Loan 8.5.3)
  for (int sweep = 0; sweep < 30; sweep++) {
    double off = 0.0, dia = 0.0;
    for (int i = 0; i < n; i++)
      for (int j = 0; j < n; j++)
        if (i != j) off += M[i * n + j] * M[i * n + j];
        else dia += M[i * n + j] * M[i * n + j];
    if (off <= 1e-34 * dia) break;
    for (int p = 0; p < n - 1; p++)
      for (int q = p + 1; q < n; q++) {
        const double apq = M[p * n + q];
        if (fabs(apq) < 1e-300) continue;
        const double tau = (M[q * n + q] - M[p * n + p]) / (2.0 * apq);
        const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + tt * tt), s = tt * c;
        for (int k = 0; k < n; k++) {
          const double mkp = M[k * n + p], mkq = M[k * n + q];
          M[k * n + p] = c * mkp - s * mkq;
          M[k * n + q] = s * mkp + c * mkq;
        }
        for (int k = 0; k < n; k++) {
          const double mpk = M[p * n + k], mqk = M[q * n + k];
          M[p * n + k] = c * mpk - s * mqk;
          M[q * n + k] = s * mpk + c * mqk;
        }
        for (int k = 0; k < n; k++) {
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  double* S = Sg + ((size_t)el * 3 + a) * n * n;
  double* lam = lamg + ((size_t)el * 3 + a) * n;
  for (int mode = 0; mode < n; mode++) {
    // a dropped node keeps its own (never rotated) mode: zero column, lambda 1
    const bool dm = (mode == 0 && !keep[0]) || (mode == N && !keep[1]);
    lam[mode] = dm ? 1.0 : M[mode * n + mode];
    for (int i = 0; i < n; i++) {
      const bool di = (i == 0 && !keep[0]) || (i == N && !keep[1]);
      S[i * n + mode] = (dm || di) ? 0.0 : V[i * n + mode] / sqrt(Bd[i]);
    }
  }
}

// 1/x for the (positive, well-scaled) eigenvalue sums: approximate reciprocal
// and two Newton steps (within an ulp of 1/x; a division costs ~5x the
// instructions and a subroutine call on its slow path)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
}

// y_e = A~_e^-1 (c^1/2 r)_e (fast diagonalisation) and b0_e = (J^T)^3 (c r)_e;
// either output may be null.  Skipped when *gate.
template <int n>
__global__ void __launch_bounds__(kFT) fdm_kernel(int nloc, const double* __restrict__ r,
                                                  const uint8_t* __restrict__ mult,
                                                  const double* __restrict__ Sg,
                                                  const double* __restrict__ lamg,
                                                  const double* __restrict__ xi,
                                                  double* __restrict__ y, double* __restrict__ b0,
                                                  const int* gate) {
  constexpr int n2 = n * n, n3 = n2 * n;
  __shared__ double u[n3], t[n3];
  __shared__ double S[3][n2], lam[3][n], J[n][2];
  __shared__ double red[kFT / 32][8];
  if (gate && *gate) return;
  const int tid = threadIdx.x;
  if (tid < n) {
    J[tid][0] = 0.5 * (1.0 - xi[tid]);
    J[tid][1] = 0.5 * (1.0 + xi[tid]);
  }
  for (int el = blockIdx.x; el < nloc; el += gridDim.x) {
    const double* re = r + (int64_t)el * n3;
    const uint8_t* me = mult + (int64_t)el * n3;
    __syncthreads();   // J ready; the previous element is done with u, t, S
    double acc[8];
#pragma unroll
    for (int v = 0; v < 8; v++) acc[v] = 0.0;
    for (int p = tid; p < n3; p += kFT) {
      const double rv = __ldcs(&re[p]);
      const double c = __drcp_rn((double)me[p]);
      u[p] = sqrt(c) * rv;
      if (b0) {
        const int i = p % n, j = (p / n) % n, k = p / n2;
        const double cr = c * rv;
#pragma unroll
        for (int v = 0; v < 8; v++)
          acc[v] = fma(J[i][v & 1] * J[j][(v >> 1) & 1] * J[k][v >> 2], cr, acc[v]);
      }
    }
    if (y) {
      const double* Se = Sg + (size_t)el * 3 * n2;
      const double* le = lamg + (size_t)el * 3 * n;
      for (int q = tid; q < 3 * n2; q += kFT) (&S[0][0])[q] = __ldcs(&Se[q]);
      for (int q = tid; q < 3 * n; q += kFT) (&lam[0][0])[q] = __ldcs(&le[q]);
    }
    if (b0) {
      const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
      for (int v = 0; v < 8; v++) {
        const double s = warp_sum(acc[v]);
        if (lane == 0) red[wid][v] = s;
      }
    }
    __syncthreads();
    if (b0 && tid < 8) {
      double s = 0.0;
      for (int w = 0; w < kFT / 32; w++) s += red[w][tid];
      b0[(int64_t)el * 8 + tid] = s;
    }
    if (!y) continue;
    // forward transform: t = (Sx^T) u along i, u = (Sy^T) t along j, t = (Sz^T) u / Lambda
    for (int p = tid; p < n3; p += kFT) {
      const int a = p % n, jk = p / n;
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < n; i++) s = fma(S[0][i * n + a], u[i + n * jk], s);
      t[p] = s;
    }
    __syncthreads();
    for (int p = tid; p < n3; p += kFT) {
      const int a = p % n, b = (p / n) % n, k = p / n2;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < n; j++) s = fma(S[1][j * n + b], t[a + n * j + n2 * k], s);
      u[p] = s;
    }
    __syncthreads();
    for (int p = tid; p < n3; p += kFT) {
      const int a = p % n, b = (p / n) % n, c = p / n2;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < n; k++) s = fma(S[2][k * n + c], u[a + n * b + n2 * k], s);
      t[p] = s * rcp_nr(lam[0][a] + lam[1][b] + lam[2][c]);
    }
    __syncthreads();
    // backward: u = Sz t along c, t = Sy u along b, y = Sx t along a
    for (int p = tid; p < n3; p += kFT) {
      const int ab = p % n2, k = p / n2;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < n; c++) s = fma(S[2][k * n + c], t[ab + n2 * c], s);
      u[p] = s;
    }
    __syncthreads();
    for (int p = tid; p < n3; p += kFT) {
      const int a = p % n, j = (p / n) % n, k = p / n2;
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < n; b++) s = fma(S[1][j * n + b], u[a + n * b + n2 * k], s);
      t[p] = s;
    }
    __syncthreads();
    double* ye = y + (int64_t)el * n3;
    for (int p = tid; p < n3; p += kFT) {
      const int i = p % n, jk = p / n;
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < n; a++) s = fma(S[0][i * n + a], t[a + n * jk], s);
      __stcs(&ye[p], s);
    }
  }
}

// ---- n = 8 (N = 7): the six contractions on the fp64 tensor cores.
// One warp per element; every stage is 8 tiles x 2 k-steps of DMMA m8n8k4
// (D[8x8] += A[8x4] B[4x8]).  The S factors are operands held in registers
// (2 per stage per lane, read once from global/L2); the element's data moves
// between two shared-memory buffers with the padded layout
// a(i,j,k) = (i ^ 4 [bit 2 of j != bit 2 of k]) + 12 j + 100 k (pad8), which
// makes every fragment load and store of the six stages (strides 1/12/100
// against the lane fields g = lane/4, q = lane%4 and the accumulator columns
// 2q+e) conflict-free.  The same smem traffic as one CUDA-core stage moves
// 8x the arithmetic, which is what takes the kernel from shared-memory bound
// (15 % of HBM bandwidth) towards the HBM roofline.
constexpr int kF8W = 4;          // warps (elements in flight) per CTA
constexpr int kF8Buf = 800;      // doubles per padded buffer (max index 791)
constexpr int kF8Smem = kF8W * 2 * kF8Buf + 2 * 256;   // + 1/m and (1/m)^1/2 tables

// swizzled padded layout: i is XOR-ed with 4 when bit 2 of j and bit 2 of k
// differ.  The plain pad i + 12 j + 100 k made every fragment LOAD of the six
// stages conflict-free but the accumulator STORES (columns 2q + e) 2-way
// conflicted within each half warp (lanes q and q + 2 on one bank pair):
// ~8 M excess wavefronts per C3 launch in ncu.  The swizzle makes loads and
// stores hit 16 distinct bank pairs per half warp (checked for every stage
// pattern and for the 128-bit load / store phases) in the same 792 doubles.
__device__ __forceinline__ int pad8(int i, int j, int k) {
  return (i ^ (4 * (((j >> 2) ^ (k >> 2)) & 1))) + 12 * j + 100 * k;
}

// not volatile: the tiles of a stage are independent and the scheduler may
// interleave their DMMAs (a volatile asm keeps program order)
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// One contraction stage: 8 output tiles, two k-steps each.  All operand loads
// of a group of tiles are issued first, then the k-step-0 DMMAs of every tile,
// then the k-step-1 DMMAs, then the stores: independent accumulation chains
// interleave (the straightforward per-tile order serialised load -> DMMA ->
// DMMA -> store eight times per stage).
template <class L0, class L1, class MM, class ST>
__device__ __forceinline__ void f8_stage(L0 l0, L1 l1, MM mm, ST st) {
  constexpr int TG = 4;   // tiles per group
#pragma unroll
  for (int h = 0; h < 8; h += TG) {
    double x0[TG], x1[TG], d0[TG], d1[TG];
#pragma unroll
    for (int u = 0; u < TG; u++) {
      x0[u] = l0(h + u);
      x1[u] = l1(h + u);
    }
#pragma unroll
    for (int u = 0; u < TG; u++) {
      d0[u] = 0.0;
      d1[u] = 0.0;
      mm(d0[u], d1[u], 0, x0[u]);
    }
#pragma unroll
    for (int u = 0; u < TG; u++) mm(d0[u], d1[u], 1, x1[u]);
#pragma unroll
    for (int u = 0; u < TG; u++) st(h + u, d0[u], d1[u]);
  }
}

__global__ void __launch_bounds__(kF8W * 32) fdm8_kernel(
    int nloc, const double* __restrict__ r, const uint8_t* __restrict__ mult,
    const double* __restrict__ Sg, const double* __restrict__ lamg, const double* __restrict__ xi,
    double* __restrict__ y, double* __restrict__ b0, const int* gate) {
  extern __shared__ double f8smem[];
  if (gate && *gate) return;
  // warp index broadcast from lane 0: provably warp-uniform, so the element
  // loop and its mma.sync need no divergence handling
  const int lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
  const int g = lane >> 2, q = lane & 3;
  double* U = f8smem + warp * 2 * kF8Buf;
  double* T = U + kF8Buf;
  double* cinv = f8smem + kF8W * 2 * kF8Buf;   // [256]: 1/m (as __drcp_rn), then its sqrt
  double* csq = cinv + 256;
  for (int m = threadIdx.x; m < 256; m += blockDim.x) {
    const double c = __drcp_rn((double)(m > 0 ? m : 1));
    cinv[m] = c;
    csq[m] = sqrt(c);
  }
  // this lane's point pair in the load / store phases: pair q of plane m
  // (points 2q, 2q + 1: i = 2 (q % 4), j = q / 4, k = m).  The lane -> pair map
  // is a permutation within the warp's 512-B segment (still one coalesced
  // access) chosen so that the eight lanes of every quarter warp hit eight
  // distinct 16-B bank groups of the padded buffer (pad8 = i + 12 j + 100 k):
  // quarter warp G takes the rows j in {jt[G], jt[G] + 2}, jt = {0, 1, 4, 5}
  // (the identity map, j = lane / 4, put two lanes on every group: 2-way
  // conflicts on the LDS.128 / STS of these phases, ~9 M excess wavefronts
  // per C3 launch in ncu).  The restriction weights J_ia J_jb J_kc factor per lane.
  const int qp = ((lane >> 3) == 0 ? 0 : (lane >> 3) == 1 ? 1 : (lane >> 3) == 2 ? 4 : 5) * 4 +
                 ((lane >> 2) & 1) * 8 + (lane & 3);
  const int i0 = 2 * (qp & 3), j0 = qp >> 2;
  const double xa = __ldg(&xi[i0]), xb = __ldg(&xi[i0 + 1]), xj = __ldg(&xi[j0]);
  const double ja[2] = {0.5 * (1.0 - xa), 0.5 * (1.0 + xa)};
  const double jb[2] = {0.5 * (1.0 - xb), 0.5 * (1.0 + xb)};
  const double jj[2] = {0.5 * (1.0 - xj), 0.5 * (1.0 + xj)};
  __syncthreads();
  for (int el = blockIdx.x * kF8W + warp; el < nloc; el += gridDim.x * kF8W) {
    // every global load of the element first: r, mult, the S fragments, lambda
    const double2* r2 = reinterpret_cast<const double2*>(r + (int64_t)el * 512);
    const uchar2* m2 = reinterpret_cast<const uchar2*>(mult + (int64_t)el * 512);
    double2 rv[8];
    uchar2 mv[8];
#pragma unroll
    for (int m = 0; m < 8; m++) {
      rv[m] = __ldcs(&r2[qp + 32 * m]);
      mv[m] = m2[qp + 32 * m];
    }
    const double* Sx = Sg + (size_t)el * 192;
    const double* Sy = Sx + 64;
    const double* Sz = Sx + 128;
    const double* lx = lamg + (size_t)el * 24;
    const double AX0 = __ldcs(&Sx[q * 8 + g]), AX1 = __ldcs(&Sx[(4 + q) * 8 + g]);
    const double BY0 = __ldcs(&Sy[q * 8 + g]), BY1 = __ldcs(&Sy[(4 + q) * 8 + g]);
    const double BZ0 = __ldcs(&Sz[q * 8 + g]), BZ1 = __ldcs(&Sz[(4 + q) * 8 + g]);
    const double CZ0 = __ldcs(&Sz[g * 8 + q]), CZ1 = __ldcs(&Sz[g * 8 + 4 + q]);
    const double CY0 = __ldcs(&Sy[g * 8 + q]), CY1 = __ldcs(&Sy[g * 8 + 4 + q]);
    const double CX0 = __ldcs(&Sx[g * 8 + q]), CX1 = __ldcs(&Sx[g * 8 + 4 + q]);
    const double lxg = __ldcs(&lx[g]);
    const double lz0 = __ldcs(&lx[16 + 2 * q]), lz1 = __ldcs(&lx[17 + 2 * q]);
    // c^1/2 r into U (padded), restriction partials of (J^T)^3 (c r)
    double acc[8];
#pragma unroll
    for (int v = 0; v < 8; v++) acc[v] = 0.0;
#pragma unroll
    for (int m = 0; m < 8; m++) {
      U[pad8(i0, j0, m)] = csq[mv[m].x] * rv[m].x;
      U[pad8(i0 + 1, j0, m)] = csq[mv[m].y] * rv[m].y;
      if (b0) {   // separable: sum over the pair along i first, then weight by J_j J_k
        const double xk = __ldg(&xi[m]);
        const double jk[2] = {0.5 * (1.0 - xk), 0.5 * (1.0 + xk)};
        const double cr0 = cinv[mv[m].x] * rv[m].x, cr1 = cinv[mv[m].y] * rv[m].y;
        const double si[2] = {fma(ja[0], cr0, jb[0] * cr1), fma(ja[1], cr0, jb[1] * cr1)};
#pragma unroll
        for (int v = 0; v < 8; v++)
          acc[v] = fma(si[v & 1], jj[(v >> 1) & 1] * jk[v >> 2], acc[v]);
      }
    }
    if (b0) {
#pragma unroll
      for (int v = 0; v < 8; v++) acc[v] = warp_sum(acc[v]);
      if (lane < 8) {
        double o = acc[0];
#pragma unroll
        for (int v = 1; v < 8; v++) o = lane == v ? acc[v] : o;
        b0[(int64_t)el * 8 + lane] = o;
      }
    }
    __syncwarp();
    // 1. T[a][j][k] = sum_i Sx[i][a] U[i][j][k]   (S as the A operand)
    f8_stage([&](int t) { return U[pad8(q, g, t)]; }, [&](int t) { return U[pad8(4 + q, g, t)]; },
             [&](double& d0, double& d1, int s, double x) { dmma884(d0, d1, s ? AX1 : AX0, x); },
             [&](int t, double d0, double d1) {
               T[pad8(g, 2 * q, t)] = d0;
               T[pad8(g, 2 * q + 1, t)] = d1;
             });
    __syncwarp();
    // 2. U[a][b][k] = sum_j T[a][j][k] Sy[j][b]   (S as the B operand)
    f8_stage([&](int t) { return T[pad8(g, q, t)]; }, [&](int t) { return T[pad8(g, 4 + q, t)]; },
             [&](double& d0, double& d1, int s, double x) { dmma884(d0, d1, x, s ? BY1 : BY0); },
             [&](int t, double d0, double d1) {
               U[pad8(g, 2 * q, t)] = d0;
               U[pad8(g, 2 * q + 1, t)] = d1;
             });
    __syncwarp();
    // 3. T[a][b][c] = sum_k U[a][b][k] Sz[k][c] / (lx_a + ly_b + lz_c)
    f8_stage([&](int t) { return U[pad8(g, t, q)]; }, [&](int t) { return U[pad8(g, t, 4 + q)]; },
             [&](double& d0, double& d1, int s, double x) { dmma884(d0, d1, x, s ? BZ1 : BZ0); },
             [&](int t, double d0, double d1) {
               const double lyt = __ldg(&lx[8 + t]);
               T[pad8(g, t, 2 * q)] = d0 * rcp_nr(lxg + lyt + lz0);
               T[pad8(g, t, 2 * q + 1)] = d1 * rcp_nr(lxg + lyt + lz1);
             });
    __syncwarp();
    // 4. U[a][b][k] = sum_c T[a][b][c] Sz[k][c]
    f8_stage([&](int t) { return T[pad8(g, t, q)]; }, [&](int t) { return T[pad8(g, t, 4 + q)]; },
             [&](double& d0, double& d1, int s, double x) { dmma884(d0, d1, x, s ? CZ1 : CZ0); },
             [&](int t, double d0, double d1) {
               U[pad8(g, t, 2 * q)] = d0;
               U[pad8(g, t, 2 * q + 1)] = d1;
             });
    __syncwarp();
    // 5. T[a][j][k] = sum_b U[a][b][k] Sy[j][b]
    f8_stage([&](int t) { return U[pad8(g, q, t)]; }, [&](int t) { return U[pad8(g, 4 + q, t)]; },
             [&](double& d0, double& d1, int s, double x) { dmma884(d0, d1, x, s ? CY1 : CY0); },
             [&](int t, double d0, double d1) {
               T[pad8(g, 2 * q, t)] = d0;
               T[pad8(g, 2 * q + 1, t)] = d1;
             });
    __syncwarp();
    // 6. U[i][j][k] = sum_a Sx[i][a] T[a][j][k]
    f8_stage([&](int t) { return T[pad8(q, g, t)]; }, [&](int t) { return T[pad8(4 + q, g, t)]; },
             [&](double& d0, double& d1, int s, double x) { dmma884(d0, d1, s ? CX1 : CX0, x); },
             [&](int t, double d0, double d1) {
               U[pad8(g, 2 * q, t)] = d0;
               U[pad8(g, 2 * q + 1, t)] = d1;
             });
    __syncwarp();
    double2* y2 = reinterpret_cast<double2*>(y + (int64_t)el * 512);
#pragma unroll
    for (int m = 0; m < 8; m++)
      __stcs(&y2[qp + 32 * m], make_double2(U[pad8(i0, j0, m)], U[pad8(i0 + 1, j0, m)]));
    __syncwarp();   // U is refilled by the next element
  }
}

// z = c^1/2 y + (J (x) J (x) J) x0_e (either part may be null).  DOTS: the
// flexible-CG dots <z, r>_c and <z, w>_c into dots[0..1] (deterministic grid
// reduction).  Flat over point pairs (16-byte accesses); a shared table maps
// the in-element index p to its (i, j, k) and holds the J factors, so a point
// costs no integer division beyond one per pair.  Skipped when *gate.
template <bool DOTS>
__global__ void __launch_bounds__(kFT) schwarz_combine_kernel(
    int n, int nloc, const double* __restrict__ y, const double* __restrict__ x0,
    const uint8_t* __restrict__ mult, const double* __restrict__ xi, double* __restrict__ z,
    const double* __restrict__ r, const double* __restrict__ w, double* partial,
    unsigned* ticket, double* dots, const int* gate) {
  __shared__ double scratch[32];
  __shared__ int flag;
  __shared__ uint32_t ijk[1728];
  __shared__ double Js[12][2];
  __shared__ double cinv[256], csq[256];   // 1/m (as __drcp_rn) and its square root
  if (gate && *gate) return;
  const int n3 = n * n * n;
  for (int m = threadIdx.x; m < 256; m += blockDim.x) {
    const double c = __drcp_rn((double)(m > 0 ? m : 1));
    cinv[m] = c;
    csq[m] = sqrt(c);
  }
  for (int p = threadIdx.x; p < n3; p += blockDim.x)
    ijk[p] = (uint32_t)(p % n) | ((uint32_t)((p / n) % n) << 8) | ((uint32_t)(p / (n * n)) << 16);
  if (threadIdx.x < n) {
    Js[threadIdx.x][0] = 0.5 * (1.0 - xi[threadIdx.x]);
    Js[threadIdx.x][1] = 0.5 * (1.0 + xi[threadIdx.x]);
  }
  __syncthreads();
  const int64_t nslots = (int64_t)nloc * n3;
  const int64_t npair = nslots >> 1;
  double zr = 0.0, zw = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < npair;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = 2 * q;
    int64_t el = l / n3;
    int p = (int)(l - el * n3);
    const uchar2 mv = *reinterpret_cast<const uchar2*>(mult + l);
    const double c0 = cinv[mv.x], c1 = cinv[mv.y];
    double v0 = 0.0, v1 = 0.0;
    if (y) {
      const double2 yv = __ldcs(reinterpret_cast<const double2*>(y) + q);
      v0 = csq[mv.x] * yv.x;
      v1 = csq[mv.y] * yv.y;
    }
    if (x0) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        if (h == 1 && ++p == n3) {   // the pair straddles two elements (odd n)
          p = 0;
          el++;
        }
        const uint32_t t = ijk[p];
        const int i = t & 255, j = (t >> 8) & 255, k = t >> 16;
        const double2* xe = reinterpret_cast<const double2*>(x0 + el * 8);
        const double2 a01 = __ldg(xe), a23 = __ldg(xe + 1), a45 = __ldg(xe + 2), a67 = __ldg(xe + 3);
        const double xv[8] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y};
        const double ji[2] = {Js[i][0], Js[i][1]}, jj[2] = {Js[j][0], Js[j][1]};
        const double jk[2] = {Js[k][0], Js[k][1]};
        double s = 0.0;
#pragma unroll
        for (int v = 0; v < 8; v++) s = fma(ji[v & 1] * jj[(v >> 1) & 1] * jk[v >> 2], xv[v], s);
        if (h == 0) v0 += s;
        else v1 += s;
      }
    }
    reinterpret_cast<double2*>(z)[q] = make_double2(v0, v1);
    if (DOTS) {
      const double2 rv = __ldcs(reinterpret_cast<const double2*>(r) + q);
      const double2 wv = __ldcs(reinterpret_cast<const double2*>(w) + q);
      zr = fma(c0 * v0, rv.x, zr);
      zr = fma(c1 * v1, rv.y, zr);
      zw = fma(c0 * v0, wv.x, zw);
      zw = fma(c1 * v1, wv.y, zw);
    }
  }
  if ((nslots & 1) && blockIdx.x == 0 && threadIdx.x == 0) {   // odd tail point
    const int64_t l = nslots - 1;
    const int64_t el = l / n3;
    const int p = (int)(l - el * n3);
    const double c = __drcp_rn((double)mult[l]);
    double v = y ? sqrt(c) * y[l] : 0.0;
    if (x0) {
      const uint32_t t = ijk[p];
      const int i = t & 255, j = (t >> 8) & 255, k = t >> 16;
      double s = 0.0;
      for (int vv = 0; vv < 8; vv++)
        s = fma(Js[i][vv & 1] * Js[j][(vv >> 1) & 1] * Js[k][vv >> 2], x0[el * 8 + vv], s);
      v += s;
    }
    z[l] = v;
    if (DOTS) {
      zr = fma(c * v, r[l], zr);
      zw = fma(c * v, w[l], zw);
    }
  }
  if (DOTS) {
    double vv[2] = {zr, zw};
    grid_reduce<2>(vv, partial, ticket, dots, scratch, &flag);
  }
}

// ---- flexible PCG scalars (device-resident, one thread)
// stage 0: start (rho = <r,z>, gamma = <r,r> reduced into st->rho_new, st->gamma)
// stage 1: alpha = rho / sigma (breakdown if sigma <= 0)
// stage 2: iteration count, history, convergence on sqrt(gamma)
// stage 3: beta = -alpha <z', w>_c / rho, rho = <z', r'>_c; maxit
__global__ void fcg_scalar_kernel(int stage, PcgState* st, double* hist) {
  if (stage == 0) {
    st->rho_old = st->rho_new;
    st->it = 0;
    st->iters = 0;
    const double g = sqrt(st->gamma);
    hist[0] = g;
    st->done = (g <= st->tol) ? 1 : (st->maxit == 0 ? 4 : 0);
    return;
  }
  if (st->done) return;
  if (stage == 1) {
    const double sigma = st->sigma;
    if (!(sigma > 0.0)) {
      st->done = 2;
      st->iters = st->it + 1;
      return;
    }
    st->alpha = st->rho_old / sigma;
  } else if (stage == 2) {
    const int it = st->it + 1;
    st->it = it;
    const double g = sqrt(st->gamma);
    hist[it] = g;
    if (!(g == g)) {
      st->done = 3;
      st->iters = it;
    } else if (g <= st->tol) {
      st->done = 1;
      st->iters = it;
    }
  } else {
    st->beta = -st->alpha * st->dz[1] / st->rho_old;
    st->rho_old = st->dz[0];
    if (!(st->beta == st->beta)) {
      st->done = 3;
      st->iters = st->it;
    } else if (st->it >= st->maxit) {
      st->done = 4;
      st->iters = st->it;
    }
  }
}

// p = z + beta p (skipped when *done)
__global__ void __launch_bounds__(kFT) xpay_kernel(int64_t n, double* __restrict__ p,
                                                   const double* __restrict__ z,
                                                   const PcgState* st) {
  if (st->done) return;
  const double beta = st->beta;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < n;
       l += (int64_t)gridDim.x * blockDim.x)
    p[l] = fma(beta, p[l], z[l]);
}

// coarse solve gate: a finished outer iteration makes the coarse CG a no-op
__global__ void gate_state_kernel(PcgState* st, const int* gate) {
  if (gate && *gate) st->done = 5;
}

// relative stopping rule of the coarse CG (reading Q31): tol = rtol ||b0||_c
__global__ void rel_tol_kernel(PcgState* st, double rtol) {
  const double g = sqrt(st->gamma);
  st->tol = rtol * g;
  st->done = (g <= st->tol) ? 1 : (st->maxit == 0 ? 4 : 0);
}

// the coarse-graph gate slot: *dst = gate ? *gate : 0
__global__ void copy_gate_kernel(int* dst, const int* gate) { *dst = gate ? *gate : 0; }

}  // namespace dev

cudaError_t launch_copy_gate(int* dst, const int* gate, cudaStream_t s) {
  dev::copy_gate_kernel<<<1, 1, 0, s>>>(dst, gate);
  return cudaGetLastError();
}

cudaError_t launch_fdm_setup(int n, int nloc, int64_t e_lo, int ex, int ey, int ez,
                             const double* box, int deform, double amp, const int* per,
                             const double* xi, const double* wq, const double* D, double* S,
                             double* lam, cudaStream_t s) {
  dev::Box b{box[0], box[1], box[2], box[3], box[4], box[5]};
  const int nt = 3 * nloc;
  if (nt == 0) return cudaSuccess;
  dev::fdm_setup_kernel<<<(nt + 63) / 64, 64, 0, s>>>(n, nloc, e_lo, ex, ey, ez, b, deform, amp,
                                                      per[0], per[1], per[2], xi, wq, D, S, lam);
  return cudaGetLastError();
}

cudaError_t launch_fdm(int n, int nloc, const double* r, const uint8_t* mult, const double* S,
                       const double* lam, const double* xi, double* y, double* b0,
                       const int* gate, int num_sms, bool tensor_cores, cudaStream_t s) {
  if (nloc == 0) return cudaSuccess;
  if (n == 8 && y && tensor_cores) {   // fp64 tensor-core path (N = 7)
    const size_t smem = (size_t)dev::kF8Smem * sizeof(double);
    static std::atomic<bool> attr[kMaxDev];   // function attributes are per device
    const int d = device_index();
    if (!attr[d].load(std::memory_order_relaxed)) {
      cudaError_t e = cudaFuncSetAttribute(dev::fdm8_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr[d].store(true, std::memory_order_relaxed);
    }
    const int grid8 = std::min((nloc + dev::kF8W - 1) / dev::kF8W, num_sms * 4);
    dev::fdm8_kernel<<<grid8, dev::kF8W * 32, smem, s>>>(nloc, r, mult, S, lam, xi, y, b0, gate);
    return cudaGetLastError();
  }
  const int grid = std::min(nloc, num_sms * 8);
#define FDM_CASE(NN)                                                                        \
  case NN:                                                                                  \
    dev::fdm_kernel<NN><<<grid, dev::kFT, 0, s>>>(nloc, r, mult, S, lam, xi, y, b0, gate); \
    break;
  switch (n) {
    FDM_CASE(2) FDM_CASE(3) FDM_CASE(4) FDM_CASE(5) FDM_CASE(6) FDM_CASE(7) FDM_CASE(8)
    FDM_CASE(9) FDM_CASE(10) FDM_CASE(11) FDM_CASE(12)
    default: return cudaErrorInvalidValue;
  }
#undef FDM_CASE
  return cudaGetLastError();
}

cudaError_t launch_schwarz_combine(int n, int nloc, const double* y, const double* x0,
                                   const uint8_t* mult, const double* xi, double* z,
                                   const double* r, const double* w, double* partial,
                                   unsigned* ticket, double* dots, const int* gate, int num_sms,
                                   cudaStream_t s) {
  const int64_t npair = ((int64_t)nloc * n * n * n) / 2;
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((npair + dev::kFT - 1) / dev::kFT, (int64_t)num_sms * 8));
  if (dots)
    dev::schwarz_combine_kernel<true><<<grid, dev::kFT, 0, s>>>(n, nloc, y, x0, mult, xi, z, r, w,
                                                                partial, ticket, dots, gate);
  else
    dev::schwarz_combine_kernel<false><<<grid, dev::kFT, 0, s>>>(n, nloc, y, x0, mult, xi, z, r, w,
                                                                 partial, ticket, dots, gate);
  return cudaGetLastError();
}

cudaError_t launch_fcg_scalar(int stage, PcgState* st, double* hist, cudaStream_t s) {
  dev::fcg_scalar_kernel<<<1, 1, 0, s>>>(stage, st, hist);
  return cudaGetLastError();
}

cudaError_t launch_xpay(int64_t n, double* p, const double* z, const PcgState* st, int num_sms,
                        cudaStream_t s) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + dev::kFT - 1) / dev::kFT,
                                                                (int64_t)num_sms * 8));
  dev::xpay_kernel<<<grid, dev::kFT, 0, s>>>(n, p, z, st);
  return cudaGetLastError();
}

cudaError_t launch_gate_state(PcgState* st, const int* gate, cudaStream_t s) {
  dev::gate_state_kernel<<<1, 1, 0, s>>>(st, gate);
  return cudaGetLastError();
}

cudaError_t launch_rel_tol(PcgState* st, double rtol, cudaStream_t s) {
  dev::rel_tol_kernel<<<1, 1, 0, s>>>(st, rtol);
  return cudaGetLastError();
}

}  // namespace sem
