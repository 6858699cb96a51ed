// Element stiffness operator  w_L = A_L u_L,  A^e = D^T G^e D  (Eq. 9),
// optionally fused with the gather-scatter QQ^T (Eq. 10), the
// Dirichlet mask and the CG inner product <p, A p>.
//
// Design, sm_100a, fp64 on the CUDA cores:
//  * persistent grid; each CTA walks element groups (NE elements of n^3 points)
//    with a 2-stage ring: the 6 geometric factors of the next group (and u when
//    n is even) are fetched by the TMA bulk-copy engine (cp.async.bulk ->
//    UBLKCP) into shared memory, completion tracked on mbarriers, while the
//    current group is computed;
//  * thread (i,j) owns the k-column of its element: u_(i,j,:) and the
//    t-direction contributions live in registers; the r and s contractions read
//    shared memory (padded D to avoid bank conflicts); w_r, w_s overwrite the
//    consumed G_rr, G_ss slots of the stage in place (no extra smem);
//  * AX_APPLY / AX_PCG: after writing w_e, the CTA "arrives" on each face /
//    edge / vertex entity of the element (one atomic ticket per entity per
//    call); the last arriver sums the entity's slots in ascending slot order
//    (reading Q10) while they are still L2-resident, writes the sum (or 0 on
//    Dirichlet points) to every slot, and resets the ticket.  The gather-
//    scatter therefore costs no separate pass over HBM;
//  * AX_PCG also accumulates sigma = sum_l p_l (A_L p)_l = p^T A p (valid for a
//    continuous p that vanishes on Dirichlet slots) and reduces it
//    deterministically (fixed element->CTA map, fixed-order final sum).
#include <algorithm>

#include "dev_common.cuh"
#include "kernels.h"
#include "sem_internal.h"

namespace sem {
namespace dev {

template <int n>
struct AxCfg;
// elements per CTA group: keep ~64-160 threads per CTA and the 2-stage ring
// inside shared memory
template <> struct AxCfg<2> { static constexpr int NE = 16; };
template <> struct AxCfg<3> { static constexpr int NE = 8; };
template <> struct AxCfg<4> { static constexpr int NE = 4; };
template <> struct AxCfg<5> { static constexpr int NE = 2; };
template <> struct AxCfg<6> { static constexpr int NE = 2; };
template <> struct AxCfg<7> { static constexpr int NE = 1; };
template <> struct AxCfg<8> { static constexpr int NE = 1; };
template <> struct AxCfg<9> { static constexpr int NE = 1; };
template <> struct AxCfg<10> { static constexpr int NE = 1; };
template <> struct AxCfg<11> { static constexpr int NE = 1; };
template <> struct AxCfg<12> { static constexpr int NE = 1; };

template <int n>
struct AxShape {
  static constexpr int NE = AxCfg<n>::NE;
  static constexpr int n2 = n * n, n3 = n2 * n;
  static constexpr int TC = NE * n2;               // computing threads
  static constexpr int T = (TC + 31) / 32 * 32;    // launched threads
  static constexpr int S = 2;                      // ring stages
  static constexpr bool kBulkU = (n % 2) == 0;     // u block 16-B aligned for any element
  static constexpr int stage_dbl = NE * 6 * n3 + (kBulkU ? NE * n3 : 0);
  static constexpr int plainu_dbl = kBulkU ? 0 : NE * n3;
  static constexpr int dpad = n + 1;
  static constexpr int kMaxList = NE * kRefsPerElem;
  static constexpr size_t smem_bytes =
      sizeof(double) * ((size_t)S * stage_dbl + plainu_dbl + 2 * n * dpad + 32) +
      sizeof(uint64_t) * S + sizeof(int) * (kMaxList + 8);
};

__device__ __forceinline__ int face_s1(int axis, int n) { return axis == 0 ? n : 1; }
__device__ __forceinline__ int face_s2(int axis, int n) { return axis == 2 ? n : n * n; }
__device__ __forceinline__ int edge_stride(int axis, int n) {
  return axis == 0 ? 1 : (axis == 1 ? n : n * n);
}

// Sum one entity point over its incidences (ascending slots), write the total.
__device__ __forceinline__ void sum_point(double* __restrict__ w, const int32_t* base, int nin,
                                          int off, bool masked) {
  double v[8];
#pragma unroll
  for (int t = 0; t < 8; t++)
    if (t < nin) v[t] = __ldcg(&w[base[t] + off]);
  double s = v[0];
#pragma unroll
  for (int t = 1; t < 8; t++)
    if (t < nin) s += v[t];
  if (masked) s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; t++)
    if (t < nin) __stcg(&w[base[t] + off], s);
}

template <int n, int MODE, bool FUSE>
__global__ void __launch_bounds__(AxShape<n>::T)
    ax_kernel(const DevPlan P, const AxLaunch a) {
  using Sh = AxShape<n>;
  constexpr int NE = Sh::NE, n2 = Sh::n2, n3 = Sh::n3, T = Sh::T, S = Sh::S;
  constexpr int dp = Sh::dpad;
  constexpr bool kBulkU = Sh::kBulkU;
  constexpr bool kMask = MODE != AX_ONLY;   // Dirichlet mask in the epilogue
  constexpr bool kGs = kMask && FUSE;         // last-arriver gather-scatter in-kernel

  if (MODE == AX_PCG && *a.done) return;

  extern __shared__ __align__(128) double smem[];
  double* stage0 = smem;
  double* su_plain = smem + S * Sh::stage_dbl;
  double* sD = su_plain + Sh::plainu_dbl;   // sD[i*dp+m]  = D[i][m]
  double* sDt = sD + n * dp;                // sDt[i*dp+m] = D[m][i]
  double* s_red = sDt + n * dp;             // 32 doubles
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_red + 32);
  int* s_list = reinterpret_cast<int*>(bar + S);
  int* s_misc = s_list + Sh::kMaxList;      // [0] list length, [1] last-block flag

  const int tid = threadIdx.x;
  const int el = tid / n2, ij = tid - (tid / n2) * n2;
  const int i = ij % n, j = ij / n;

  for (int q = tid; q < n2; q += T) {
    const int r = q / n, c = q % n;
    const double d = P.D[q];
    sD[r * dp + c] = d;
    sDt[c * dp + r] = d;
  }
  if (tid == 0) {
    for (int s = 0; s < S; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int n0 = a.r0hi - a.r0lo, n1 = a.r1hi - a.r1lo;
  const int ng0 = (n0 + NE - 1) / NE, ng1 = (n1 + NE - 1) / NE, ng = ng0 + ng1;
  auto group = [&](int g, int& e0, int& cnt) {
    if (g < ng0) {
      e0 = a.r0lo + g * NE;
      cnt = min(NE, a.r0hi - e0);
    } else {
      e0 = a.r1lo + (g - ng0) * NE;
      cnt = min(NE, a.r1hi - e0);
    }
  };
  const uint64_t pol_G = policy_evict_first();
  auto issue = [&](int g, int s) {
    int e0, cnt;
    group(g, e0, cnt);
    double* st = stage0 + s * Sh::stage_dbl;
    const uint32_t bG = (uint32_t)cnt * 6u * n3 * 8u;
    const uint32_t bU = kBulkU ? (uint32_t)cnt * n3 * 8u : 0u;
    mbar_arrive_expect_tx(&bar[s], bG + bU);
    bulk_g2s_hint(st, a.G + (size_t)e0 * 6 * n3, bG, &bar[s], pol_G);
    if (kBulkU) bulk_g2s(st + NE * 6 * n3, a.u + (size_t)e0 * n3, bU, &bar[s]);
  };
  if (tid == 0)
    for (int s = 0; s < S; s++) {
      const int g = blockIdx.x + s * gridDim.x;
      if (g < ng) issue(g, s);
    }

  double acc = 0.0;  // sigma partial (AX_PCG)
  int it = 0;
  for (int g = blockIdx.x; g < ng; g += gridDim.x, ++it) {
    const int s = it % S;
    const uint32_t ph = (uint32_t)(it / S) & 1u;
    int e0, cnt;
    group(g, e0, cnt);
    const bool active = el < cnt;
    double* st = stage0 + s * Sh::stage_dbl;
    double* sG = st + el * 6 * n3;
    const double* sU;
    if (kBulkU) {
      sU = st + NE * 6 * n3 + el * n3;
    } else {
      double* su = su_plain + el * n3;
      if (active) {
        const double* ug = a.u + (size_t)(e0 + el) * n3;
#pragma unroll
        for (int k = 0; k < n; k++) su[ij + n2 * k] = ug[ij + n2 * k];
      }
      __syncthreads();
      sU = su;
    }
    mbar_wait(&bar[s], ph);

    double ru[n], rw[n];
    if (active) {
#pragma unroll
      for (int k = 0; k < n; k++) {
        ru[k] = sU[ij + n2 * k];
        rw[k] = 0.0;
      }
#pragma unroll
      for (int k = 0; k < n; k++) {
        double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
        for (int m = 0; m < n; m++) {
          ur = fma(sD[i * dp + m], sU[m + n * j + n2 * k], ur);
          us = fma(sD[j * dp + m], sU[i + n * m + n2 * k], us);
          ut = fma(sD[k * dp + m], ru[m], ut);
        }
        const int pt = ij + n2 * k;
        const double grr = sG[0 * n3 + pt], gss = sG[1 * n3 + pt], gtt = sG[2 * n3 + pt];
        const double grs = sG[3 * n3 + pt], grt = sG[4 * n3 + pt], gst = sG[5 * n3 + pt];
        const double wr = grr * ur + grs * us + grt * ut;
        const double ws = grs * ur + gss * us + gst * ut;
        const double wt = grt * ur + gst * us + gtt * ut;
        sG[0 * n3 + pt] = wr;   // own point only: safe without a barrier
        sG[1 * n3 + pt] = ws;
#pragma unroll
        for (int m = 0; m < n; m++) rw[m] = fma(sD[k * dp + m], wt, rw[m]);
      }
    }
    __syncthreads();
    if (active) {
      const double* swr = sG;
      const double* sws = sG + n3;
      const int e = e0 + el;
      double* wg = a.w + (size_t)e * n3;
      const unsigned bm = kMask ? P.bmask[e] : 0u;
#pragma unroll
      for (int k = 0; k < n; k++) {
        double v = rw[k];
#pragma unroll
        for (int m = 0; m < n; m++) {
          v = fma(sDt[i * dp + m], swr[m + n * j + n2 * k], v);
          v = fma(sDt[j * dp + m], sws[i + n * m + n2 * k], v);
        }
        if (kMask && face_masked(bm, i, j, k, n - 1)) v = 0.0;
        if (MODE == AX_PCG) acc = fma(ru[k], v, acc);
        wg[ij + n2 * k] = v;
      }
    }

    if (kGs) {
      // ---- arrive on this group's entities; the last arriver sums them ----
      if (tid == 0) s_misc[0] = 0;
      __syncthreads();   // all w_e stores of the group issued; list reset visible
      for (int q = tid; q < cnt * kRefsPerElem; q += T) {
        const int e = e0 + q / kRefsPerElem;
        const int ref = P.eref[(size_t)e * kRefsPerElem + q % kRefsPerElem];
        if (ref >= 0) {
          const int cls = ref >> kClsShift, idx = ref & ((1 << kClsShift) - 1);
          const unsigned nin = cls == CLS_FACE ? 2u : (cls == CLS_EDGE ? P.e_nin[idx] : P.v_nin[idx]);
          unsigned* tk = P.cnt + (cls == CLS_FACE ? idx : (cls == CLS_EDGE ? P.nF + idx : P.nF + P.nEd + idx));
          // acq_rel: releases this CTA's w stores (ordered before by the barrier),
          // acquires the other incidences' stores when this is the last arrival
          const unsigned old = atom_add_acq_rel_gpu(tk, 1u);
          if (old == nin - 1u) {
            *tk = 0u;
            s_list[atomicAdd(&s_misc[0], 1)] = ref;
          }
        }
      }
      __syncthreads();
      const int nl = s_misc[0];
      if (nl > 0) {
        constexpr int NW = T / 32;
        const int lane = tid & 31, wid = tid >> 5;
        const int N = n - 1, nf = (N - 1) * (N - 1), ne = N - 1;
        for (int q = wid; q < nl; q += NW) {
          const int ref = s_list[q];
          const int cls = ref >> kClsShift, idx = ref & ((1 << kClsShift) - 1);
          int32_t base[8];
          if (n > 2 && cls == CLS_FACE) {
            base[0] = P.f_base[2 * idx];
            base[1] = P.f_base[2 * idx + 1];
            const int ax = P.f_axis[idx];
            const int s1 = face_s1(ax, n), s2 = face_s2(ax, n);
            constexpr int Nm1 = n > 2 ? n - 2 : 1;
            for (int p = lane; p < nf; p += 32) {
              const int off = (1 + p % Nm1) * s1 + (1 + p / Nm1) * s2;
              sum_point(a.w, base, 2, off, false);
            }
          } else if (n > 2 && cls == CLS_EDGE) {
            const int nin = P.e_nin[idx];
#pragma unroll
            for (int t = 0; t < 4; t++) base[t] = P.e_base[4 * idx + t];
            const int sd = edge_stride(P.e_axis[idx], n);
            const bool mk = P.e_mask[idx];
            for (int p = lane; p < ne; p += 32) sum_point(a.w, base, nin, (1 + p) * sd, mk);
          } else if (cls == CLS_VERT) {
            const int nin = P.v_nin[idx];
#pragma unroll
            for (int t = 0; t < 8; t++) base[t] = P.v_base[8 * idx + t];
            if (lane == 0) sum_point(a.w, base, nin, 0, P.v_mask[idx]);
          }
        }
      }
    }

    // release the stage to the bulk-copy engine (WAW with the in-place w_r/w_s)
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const int gn = g + S * gridDim.x;
      if (gn < ng) issue(gn, s);
    }
  }

  if (MODE == AX_PCG) {
    double v[1] = {acc};
    grid_reduce<1>(v, a.red_partial, a.red_ticket, a.red_out, s_red, &s_misc[1]);
  }
}

template <int n, int MODE, bool FUSE>
static cudaError_t launch_n(const DevPlan& P, const AxLaunch& a, int grid, cudaStream_t s) {
  using Sh = AxShape<n>;
  auto kern = ax_kernel<n, MODE, FUSE>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Sh::smem_bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<grid, Sh::T, Sh::smem_bytes, s>>>(P, a);
  return cudaGetLastError();
}

template <int n, int MODE>
static int occupancy_n() {
  using Sh = AxShape<n>;
  auto kern = ax_kernel<n, MODE, true>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::smem_bytes);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, Sh::T, Sh::smem_bytes) != cudaSuccess)
    return 1;
  return std::max(nb, 1);
}

template <int MODE, bool FUSE>
static cudaError_t dispatch(const DevPlan& P, const AxLaunch& a, int grid, cudaStream_t s) {
  switch (P.n) {
    case 2: return launch_n<2, MODE, FUSE>(P, a, grid, s);
    case 3: return launch_n<3, MODE, FUSE>(P, a, grid, s);
    case 4: return launch_n<4, MODE, FUSE>(P, a, grid, s);
    case 5: return launch_n<5, MODE, FUSE>(P, a, grid, s);
    case 6: return launch_n<6, MODE, FUSE>(P, a, grid, s);
    case 7: return launch_n<7, MODE, FUSE>(P, a, grid, s);
    case 8: return launch_n<8, MODE, FUSE>(P, a, grid, s);
    case 9: return launch_n<9, MODE, FUSE>(P, a, grid, s);
    case 10: return launch_n<10, MODE, FUSE>(P, a, grid, s);
    case 11: return launch_n<11, MODE, FUSE>(P, a, grid, s);
    case 12: return launch_n<12, MODE, FUSE>(P, a, grid, s);
  }
  return cudaErrorInvalidValue;
}

template <int MODE>
static int occ_dispatch(int n) {
  switch (n) {
    case 2: return occupancy_n<2, MODE>();
    case 3: return occupancy_n<3, MODE>();
    case 4: return occupancy_n<4, MODE>();
    case 5: return occupancy_n<5, MODE>();
    case 6: return occupancy_n<6, MODE>();
    case 7: return occupancy_n<7, MODE>();
    case 8: return occupancy_n<8, MODE>();
    case 9: return occupancy_n<9, MODE>();
    case 10: return occupancy_n<10, MODE>();
    case 11: return occupancy_n<11, MODE>();
    case 12: return occupancy_n<12, MODE>();
  }
  return 1;
}

}  // namespace dev

static int ne_of(int n) {
  switch (n) {
    case 2: return dev::AxCfg<2>::NE;
    case 3: return dev::AxCfg<3>::NE;
    case 4: return dev::AxCfg<4>::NE;
    case 5: return dev::AxCfg<5>::NE;
    case 6: return dev::AxCfg<6>::NE;
    default: return 1;
  }
}

int ax_groups(int N, int nelem) {
  const int ne = ne_of(N + 1);
  return (nelem + ne - 1) / ne;
}

int ax_occupancy(int N, int mode) {
  const int n = N + 1;
  if (mode == AX_ONLY) return dev::occ_dispatch<AX_ONLY>(n);
  if (mode == AX_APPLY) return dev::occ_dispatch<AX_APPLY>(n);
  return dev::occ_dispatch<AX_PCG>(n);
}

cudaError_t launch_ax(const DevPlan& P, const AxLaunch& a, int mode, int grid, cudaStream_t s,
                      bool fuse_gs) {
  if (grid < 1) grid = 1;
  if (mode == AX_ONLY) return dev::dispatch<AX_ONLY, false>(P, a, grid, s);
  if (mode == AX_APPLY)
    return fuse_gs ? dev::dispatch<AX_APPLY, true>(P, a, grid, s)
                   : dev::dispatch<AX_APPLY, false>(P, a, grid, s);
  return fuse_gs ? dev::dispatch<AX_PCG, true>(P, a, grid, s)
                 : dev::dispatch<AX_PCG, false>(P, a, grid, s);
}

}  // namespace sem
