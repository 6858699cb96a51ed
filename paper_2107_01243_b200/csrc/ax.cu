// Element stiffness operator  w_L = A_L u_L,  A^e = D^T G^e D  (Eq. 9),
// optionally with the Dirichlet mask and the CG inner product <p, A p>
// fused in; the gather-scatter QQ^T (Eq. 10) follows in kern.cu.
//
// Design, sm_100a, fp64 on the CUDA cores (the
// contraction is HBM-bound: 1.7 flop/B at N=7, far below the fp64 ridge):
//  * warp-specialised persistent CTAs: one producer warp drives the TMA
//    bulk-copy engine (cp.async.bulk -> UBLKCP), the compute warps only
//    compute.  The producer streams, for the CTA's element sequence, each
//    element's u block and then its k-planes of geometric factors (plane-major
//    layout G[e][k][f][ij]: one 48 n^2-byte copy per plane) into two mbarrier
//    rings (full/empty), so ~tens of KB per SM are in flight without holding
//    registers and the compute warps never issue a global load;
//  * thread (i,j) owns the k-column of its element: u_(i,j,:) and the
//    t-direction accumulation live in registers; the r and s contractions read
//    shared memory (padded D and padded w_r/w_s scratch avoid bank conflicts);
//  * epilogue: mask (per-thread precomputed bits), sigma = sum_l p_l (A_L p)_l
//    (= p^T A p for a continuous p vanishing on Dirichlet slots), store w.
//    (A variant with the gather-scatter fused in -- the last CTA to finish an
//    element of a shared face/edge/vertex summing it -- was measured ~3x
//    slower than the separate gather-scatter kernel and was removed.)
#include <algorithm>

#include "dev_common.cuh"
#include "kernels.h"
#include "sem_internal.h"

namespace sem {
namespace dev {

template <int n>
struct AxCfg;
// NE: elements computed together by one CTA (64-160 compute threads)
// NSG: depth of the G plane ring (planes in flight per CTA)
#ifndef SEM_AX_SMEM_PAD
#define SEM_AX_SMEM_PAD 0   // tuning experiments only: extra smem to force lower residency
#endif
// PPC: k-planes per bulk copy (divides n).  n=8 tuned with tools/ubench_ax.cu
// on B200 (NSG=3, PPC=4: 6.2 TB/s on 32^3 elements); n=7, 9, 11, 12 with
// tools/measure.py sweep over build variants (profiles/r01_measure.md); n=2, 3,
// 5, 6, 10 likewise (profiles/r01d_ax_tuning: NE filling whole warps wins for
// small n); n=4 follows the rule of ~2 copies per element and a 2-3 slot ring
// within ~60 KB of smem.
#ifndef SEM_AX8_NE
#define SEM_AX8_NE 1
#endif
#ifndef SEM_AX8_NSG
#define SEM_AX8_NSG 3
#endif
#ifndef SEM_AX8_PPC
#define SEM_AX8_PPC 4
#endif
#ifndef SEM_AX2_NE
#define SEM_AX2_NE 32
#endif
#ifndef SEM_AX2_NSG
#define SEM_AX2_NSG 3
#endif
#ifndef SEM_AX2_PPC
#define SEM_AX2_PPC 2
#endif
template <> struct AxCfg<2> {
  static constexpr int NE = SEM_AX2_NE, NSG = SEM_AX2_NSG, PPC = SEM_AX2_PPC;
};
#ifndef SEM_AX3_NE
#define SEM_AX3_NE 14
#endif
#ifndef SEM_AX3_NSG
#define SEM_AX3_NSG 3
#endif
#ifndef SEM_AX3_PPC
#define SEM_AX3_PPC 3
#endif
template <> struct AxCfg<3> {
  static constexpr int NE = SEM_AX3_NE, NSG = SEM_AX3_NSG, PPC = SEM_AX3_PPC;
};
template <> struct AxCfg<4> { static constexpr int NE = 4, NSG = 3, PPC = 2; };
#ifndef SEM_AX5_NE
#define SEM_AX5_NE 5
#endif
#ifndef SEM_AX5_NSG
#define SEM_AX5_NSG 3
#endif
#ifndef SEM_AX5_PPC
#define SEM_AX5_PPC 5
#endif
template <> struct AxCfg<5> {
  static constexpr int NE = SEM_AX5_NE, NSG = SEM_AX5_NSG, PPC = SEM_AX5_PPC;
};
#ifndef SEM_AX6_NE
#define SEM_AX6_NE 2
#endif
#ifndef SEM_AX6_NSG
#define SEM_AX6_NSG 3
#endif
#ifndef SEM_AX6_PPC
#define SEM_AX6_PPC 3
#endif
template <> struct AxCfg<6> {
  static constexpr int NE = SEM_AX6_NE, NSG = SEM_AX6_NSG, PPC = SEM_AX6_PPC;
};
#ifndef SEM_AX7_NE
#define SEM_AX7_NE 3
#endif
#ifndef SEM_AX7_NSG
#define SEM_AX7_NSG 6
#endif
#ifndef SEM_AX7_PPC
#define SEM_AX7_PPC 1
#endif
template <> struct AxCfg<7> {
  static constexpr int NE = SEM_AX7_NE, NSG = SEM_AX7_NSG, PPC = SEM_AX7_PPC;
};
template <> struct AxCfg<8> {
  static constexpr int NE = SEM_AX8_NE, NSG = SEM_AX8_NSG, PPC = SEM_AX8_PPC;
};
#ifndef SEM_AX9_NSG
#define SEM_AX9_NSG 6
#endif
#ifndef SEM_AX9_PPC
#define SEM_AX9_PPC 1
#endif
#ifndef SEM_AX9_NE
#define SEM_AX9_NE 1
#endif
template <> struct AxCfg<9> { static constexpr int NE = SEM_AX9_NE, NSG = SEM_AX9_NSG, PPC = SEM_AX9_PPC; };
#ifndef SEM_AX10_NSG
#define SEM_AX10_NSG 4
#endif
#ifndef SEM_AX10_PPC
#define SEM_AX10_PPC 2
#endif
template <> struct AxCfg<10> { static constexpr int NE = 1, NSG = SEM_AX10_NSG, PPC = SEM_AX10_PPC; };
#ifndef SEM_AX11_NSG
#define SEM_AX11_NSG 6
#endif
template <> struct AxCfg<11> { static constexpr int NE = 1, NSG = SEM_AX11_NSG, PPC = 1; };
#ifndef SEM_AX12_NSG
#define SEM_AX12_NSG 2
#endif
template <> struct AxCfg<12> { static constexpr int NE = 1, NSG = SEM_AX12_NSG, PPC = 3; };

// PF (one-rank Jacobi-PCG with the p update fused in): the u ring carries p_old,
// r and dinv (NU = 3 blocks per slot); at n = 8 the G ring is 4 slots of 2
// planes (3 CTAs per SM; best of 3x2, 3x4, 4x1, 4x2, 5x1, 2x2 on C2 and C3,
// profiles/r02_experiments/pcg_fuse_ab.jsonl)
#ifndef SEM_AX8PF_NSG
#define SEM_AX8PF_NSG 4
#endif
#ifndef SEM_AX8PF_PPC
#define SEM_AX8PF_PPC 2
#endif
template <int n, bool PF = false>
struct AxShape {
  static constexpr int NE = AxCfg<n>::NE;
  static constexpr int NSG = (PF && n == 8) ? SEM_AX8PF_NSG : AxCfg<n>::NSG;
  static constexpr int PPC = (PF && n == 8) ? SEM_AX8PF_PPC : AxCfg<n>::PPC;
  static constexpr int NU = PF ? 3 : 1;            // blocks per u slot (p_old, r, dinv)
  static_assert(n % PPC == 0, "planes per copy must divide n");
  static constexpr int n2 = n * n, n3 = n2 * n;
  static constexpr int TC = NE * n2;               // computing threads
  static constexpr int TCW = (TC + 31) / 32 * 32;  // compute warps x 32
  static constexpr int NWC = TCW / 32;             // compute warps
  static constexpr int T = TCW + 32;               // + producer warp
  static constexpr int NSU = 2;                    // u ring depth
  static constexpr bool kBulkU = (n % 2) == 0;     // u block 16-B aligned for any element
  // doubles per u slot (odd n: +2 so the 16-B aligned body can be shifted by one
  // double, rounded to an even count so every slot starts 16-B aligned)
  static constexpr int uslot = kBulkU ? NE * n3 : (NE * n3 + 3) / 2 * 2;
  static_assert(uslot % 2 == 0, "u slots must stay 16-B aligned");
  static constexpr int gslot = NE * PPC * 6 * n2;  // doubles per G slot (PPC planes x NE)
  // row pitch of w_r / w_s: odd, so the transposed-contraction reads
  // w_r[k][j][m] (j across the warp) spread over distinct banks
  static constexpr int rp = (n % 2) ? n : n + 1;
  static constexpr int wpl = n * rp;               // padded plane pitch
  static constexpr int wel = n * wpl;              // per element
  static constexpr int dpad = n + 1;
  static constexpr int nbar = 2 * NSG + 2 * NSU;
  static constexpr size_t smem_bytes =
      sizeof(double) * ((size_t)NSU * NU * uslot + (size_t)NSG * gslot + 2 * NE * wel + 2 * n * dpad + 32) +
      sizeof(uint64_t) * nbar + sizeof(int) * 8 + SEM_AX_SMEM_PAD;
  // CTAs per SM the shared memory allows; the register budget is sized to match
  static constexpr int MINB0 = (int)((227u * 1024u) / (smem_bytes + 1024u));
  // n >= 7: keep 168 registers per thread -- the contraction
  // state does not fit fewer without spilling, which costs far more than residency
#ifndef SEM_AX10_REGS
#define SEM_AX10_REGS 168
#endif
  static constexpr int kRegs = n == 10 ? SEM_AX10_REGS : 168;
  static constexpr int MINBR = n >= 7 ? 65536 / (T * kRegs) : 8;
  static constexpr int MINB1 = MINB0 < MINBR ? MINB0 : MINBR;
  static constexpr int MINB = MINB1 < 1 ? 1 : (MINB1 > 8 ? 8 : MINB1);
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// named barrier over the compute warps only (the producer warp never joins)
template <int NT>
__device__ __forceinline__ void compute_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

template <int n, int MODE, bool HELM = false, bool PF = false>
__global__ void __launch_bounds__(AxShape<n, PF>::T, AxShape<n, PF>::MINB)
    ax_kernel(const DevPlan P, const AxLaunch a) {
  using Sh = AxShape<n, PF>;
  static_assert(!PF || MODE == AX_PCG, "the fused p update is a PCG-iteration mode");
  constexpr int NU = Sh::NU;
  constexpr int NE = Sh::NE, n2 = Sh::n2, n3 = Sh::n3, TCW = Sh::TCW;
  constexpr int NSG = Sh::NSG, NSU = Sh::NSU, PPC = Sh::PPC;
  constexpr int dp = Sh::dpad, rp = Sh::rp, wpl = Sh::wpl;
  constexpr bool kBulkU = Sh::kBulkU;
  constexpr bool kMask = MODE != AX_ONLY;   // Dirichlet mask in the epilogue
#ifndef SEM_DREG_MAX
#define SEM_DREG_MAX 12
#endif
  constexpr bool kDreg = n <= SEM_DREG_MAX;   // D rows in registers (else shared memory)
#ifndef SEM_DT_REG
#define SEM_DT_REG 1
#endif
  constexpr bool kDtreg = kDreg && SEM_DT_REG; // transposed-contraction D columns in registers

  extern __shared__ __align__(128) double smem[];
  double* sU = smem;                                   // [NSU][NE*n3]
  double* sG = sU + NSU * NU * Sh::uslot;              // [NSG][NE][6][n2]
  double* sWr = sG + NSG * Sh::gslot;                  // [NE][n][n][rp]
  double* sWs = sWr + NE * Sh::wel;
  double* sD = sWs + NE * Sh::wel;                     // sD[i*dp+m]  = D[i][m]
  double* sDt = sD + n * dp;                           // sDt[i*dp+m] = D[m][i]
  double* s_red = sDt + n * dp;                        // 32 doubles
  uint64_t* fullG = reinterpret_cast<uint64_t*>(s_red + 32);
  uint64_t* emptyG = fullG + NSG;
  uint64_t* fullU = emptyG + NSG;
  uint64_t* emptyU = fullU + NSU;
  int* s_misc = reinterpret_cast<int*>(emptyU + NSU);  // [1] last-block flag

  const int tid = threadIdx.x;
  const bool producer = tid >= TCW && tid < TCW + 32;

  for (int q = tid; q < n2; q += Sh::T) {
    const int r = q / n, c = q % n;
    const double d = P.D[q];
    sD[r * dp + c] = d;
    sDt[c * dp + r] = d;
  }
  if (tid == 0) {
    for (int s = 0; s < NSG; s++) {
      mbar_init(&fullG[s], 1);
      mbar_init(&emptyG[s], Sh::NWC);
    }
    for (int s = 0; s < NSU; s++) {
      mbar_init(&fullU[s], kBulkU ? 1 : 2);
      mbar_init(&emptyU[s], Sh::NWC);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int r0lo = a.r0lo, r0hi = a.r0hi, r1lo = a.r1lo, r1hi = a.r1hi;
  const int ng0 = (r0hi - r0lo + NE - 1) / NE, ng1 = (r1hi - r1lo + NE - 1) / NE, ng = ng0 + ng1;
  auto group = [=](int g, int& e0, int& cnt) {
    if (g < ng0) {
      e0 = r0lo + g * NE;
      cnt = min(NE, r0hi - e0);
    } else {
      e0 = r1lo + (g - ng0) * NE;
      cnt = min(NE, r1hi - e0);
    }
  };
  // programmatic dependent launch (a.pdl_pref): G does not depend on the
  // preceding kernel, so the producer streams the first group's G planes into
  // the (initially free) ring slots BEFORE waiting for the preceding grid --
  // the ring fill overlaps that kernel's tail.  Only when the group's planes
  // fit the ring (no wait on a consumer that itself waits for u).
  constexpr int kPrefPlanes = (n / PPC <= NSG) ? n / PPC : 0;
  const bool pref = a.pdl_pref && kPrefPlanes > 0 && blockIdx.x < ng;
  if (pref && producer && tid == TCW) {
    int e0, cnt;
    group(blockIdx.x, e0, cnt);
    const uint64_t pol = policy_evict_first();
    const uint32_t bP = PPC * 6u * n2 * 8u;
    for (int kb = 0; kb < kPrefPlanes; kb++) {
      mbar_arrive_expect_tx(&fullG[kb], bP * (uint32_t)cnt);
      for (int x = 0; x < cnt; x++)
        bulk_g2s_hint(sG + kb * Sh::gslot + x * PPC * 6 * n2,
                      a.G + ((size_t)(e0 + x) * n + kb * PPC) * 6 * n2, bP, &fullG[kb], pol);
    }
  }
  pdl_wait();   // u (= p) and the done flag come from the preceding kernel
  pdl_trigger();
  if ((MODE == AX_PCG || a.gate) && *a.done) {
    // no bulk copy may still target this CTA's shared memory when it exits
    if (pref && producer && tid == TCW)
      for (int kb = 0; kb < kPrefPlanes; kb++) mbar_wait(&fullG[kb], 0u);
    return;
  }

  double acc = 0.0;  // sigma partial (AX_PCG)
  const double beta = PF ? *a.beta : 0.0;   // written by the preceding CG update

  if (producer) {
    // ======================= producer warp: TMA bulk copies =======================
    const int lane = tid - TCW;
    const uint64_t pol = policy_evict_first();
    int su = 0, sg = 0;
    uint32_t phu = 0, phg = 0;
    bool first = pref;   // the first group's G planes are already in flight
    for (int g = blockIdx.x; g < ng; g += gridDim.x) {
      int e0, cnt;
      group(g, e0, cnt);
      // u block of the group (PF: p_old, r and dinv blocks)
      const double* usrc[3] = {a.u, a.rr, a.dinv};
      mbar_wait(&emptyU[su], phu ^ 1u);
      if (kBulkU) {
        if (lane == 0) {
          const uint32_t bU = (uint32_t)cnt * n3 * 8u;
          mbar_arrive_expect_tx(&fullU[su], bU * NU);
#pragma unroll
          for (int b = 0; b < NU; b++)
            bulk_g2s(sU + (su * NU + b) * Sh::uslot, usrc[b] + (size_t)e0 * n3, bU, &fullU[su]);
        }
      } else {
        // odd n: the group's u block starts 8 mod 16 for every other element.
        // Bulk-copy its 16-B aligned body; lane 1 copies the (at most two) end
        // doubles.  The block lands h doubles into the slot (h = source
        // misalignment), which keeps the bulk destination 16-B aligned.
        // (PF: the three arrays share the allocation alignment, hence h)
        const int h = (int)((reinterpret_cast<uintptr_t>(a.u + (size_t)e0 * n3) >> 3) & 1u);
        const int cntd = cnt * n3, nb = ((cntd - h) >> 1) << 1;
        if (lane == 0) mbar_arrive_expect_tx(&fullU[su], (uint32_t)nb * 8u * NU);
#pragma unroll
        for (int b = 0; b < NU; b++) {
          const double* src = usrc[b] + (size_t)e0 * n3;
          double* dst = sU + (su * NU + b) * Sh::uslot + h;
          if (lane == 0) {
            bulk_g2s(dst + h, src + h, (uint32_t)nb * 8u, &fullU[su]);
          } else if (lane == 1) {
            if (h) dst[0] = __ldg(src);
            if (h + nb < cntd) dst[cntd - 1] = __ldg(src + cntd - 1);
          }
        }
        if (lane == 1) mbar_arrive(&fullU[su]);   // release: this lane's stores
      }
      if (++su == NSU) { su = 0; phu ^= 1u; }
      // k-planes of the geometric factors
      for (int kb = 0; kb < n / PPC; kb++) {
        if (first) {   // prefetched before griddepcontrol.wait
          if (++sg == NSG) { sg = 0; phg ^= 1u; }
          continue;
        }
        mbar_wait(&emptyG[sg], phg ^ 1u);
        if (lane == 0) {
          const uint32_t bP = PPC * 6u * n2 * 8u;
          mbar_arrive_expect_tx(&fullG[sg], bP * (uint32_t)cnt);
          for (int x = 0; x < cnt; x++)
            bulk_g2s_hint(sG + sg * Sh::gslot + x * PPC * 6 * n2,
                          a.G + ((size_t)(e0 + x) * n + kb * PPC) * 6 * n2, bP, &fullG[sg], pol);
        }
        if (++sg == NSG) { sg = 0; phg ^= 1u; }
      }
      first = false;
    }
  } else {
    // ======================= compute warps =======================
    const int el = tid / n2, ij = tid - (tid / n2) * n2;
    const int i = ij % n, j = ij / n;
    const int lane = tid & 31;
    // D rows/columns this thread contracts with, in registers (the uniform
    // D[k][m] operands come straight from the kernel-parameter constant bank)
    // (loaded from shared memory per group, right before the phase that uses
    // them, so rows and columns are never live at the same time)
    double Di[n], Dj[n], Dti[n], Dtj[n];
    int su = 0, sg = 0;
    uint32_t phu = 0, phg = 0;
    for (int g = blockIdx.x; g < ng; g += gridDim.x) {
      int e0, cnt;
      group(g, e0, cnt);
      const bool active = el < cnt;
      // the element's Dirichlet face bits, fetched now, used by the epilogue
      const unsigned bm = (kMask && active) ? (unsigned)__ldg(P.bmask + e0 + el) : 0u;
      const int uoff = kBulkU ? 0 : (int)((reinterpret_cast<uintptr_t>(a.u + (size_t)e0 * n3) >> 3) & 1u);
      double* sUe = sU + su * NU * Sh::uslot + uoff + el * n3;   // (PF: p_old, then r, dinv)
      double* wr_s = sWr + el * Sh::wel;
      double* ws_s = sWs + el * Sh::wel;
      mbar_wait(&fullU[su], phu);
#pragma unroll
      for (int m = 0; m < n; m++) {
        Di[m] = kDreg ? sD[i * dp + m] : 0.0;
        Dj[m] = kDreg ? sD[j * dp + m] : 0.0;
      }

      // Helmholtz: this thread's mass column (coalesced per plane), prefetched into
      // registers where they are free (else loaded by the epilogue; no spills either way)
#ifndef SEM_HELM_PRE
#define SEM_HELM_PRE 1
#endif
      constexpr bool kBpre = SEM_HELM_PRE && HELM && (n <= 3 || (n >= 5 && n <= 9));
      double ru[n], rw[n], rb[kBpre ? n : 1];
      const double* Bc = HELM ? a.B + (size_t)(e0 + el) * n3 + ij : nullptr;
      if (kBpre) {
#pragma unroll
        for (int k = 0; k < n; k++) rb[kBpre ? k : 0] = active ? __ldg(Bc + n2 * k) : 0.0;
      }
      if (PF) {
        // fused p update (one-rank PCG): p = dinv r + beta p_old for this thread's
        // column, in place in the slot's p part (the contractions read it across
        // threads) and to global memory; beta = 0 on the first iteration (p_old = 0)
        const double* sRe = sUe + Sh::uslot;
        const double* sDe = sUe + 2 * Sh::uslot;
        double* pg = a.pout + (size_t)(e0 + el) * n3 + ij;
#pragma unroll
        for (int k = 0; k < n; k++) {
          double pn = 0.0;
          if (active) {
            const int l = ij + n2 * k;
            pn = fma(beta, sUe[l], sDe[l] * sRe[l]);
            sUe[l] = pn;
            pg[n2 * k] = pn;
          }
          ru[k] = pn;
          rw[k] = 0.0;
        }
        compute_sync<TCW>();   // the whole group's p in shared memory
      } else {
#pragma unroll
        for (int k = 0; k < n; k++) {
          ru[k] = active ? sUe[ij + n2 * k] : 0.0;
          rw[k] = 0.0;
        }
      }
#ifndef SEM_KU
#define SEM_KU 2
#endif
      // plane loop: partial unrolling keeps the live range (and registers) bounded
      constexpr int kKU = SEM_KU;
#pragma unroll(kKU)
      for (int k = 0; k < n; k++) {
        if (k % PPC == 0) mbar_wait(&fullG[sg], phg);
        const double* gp = sG + sg * Sh::gslot + (el * PPC + k % PPC) * 6 * n2 + ij;
        double gk[6];
#pragma unroll
        for (int f = 0; f < 6; f++) gk[f] = active ? gp[f * n2] : 0.0;
        if (active) {
          double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
          for (int m = 0; m < n; m++) {
            ur = fma(kDreg ? Di[m] : sD[i * dp + m], sUe[m + n * j + n2 * k], ur);
            us = fma(kDreg ? Dj[m] : sD[j * dp + m], sUe[i + n * m + n2 * k], us);
            ut = fma(a.Dm[k * n + m], ru[m], ut);
          }
          // G order (rr, ss, tt, rs, rt, st)
          const double wr = gk[0] * ur + gk[3] * us + gk[4] * ut;
          const double ws = gk[3] * ur + gk[1] * us + gk[5] * ut;
          const double wt = gk[4] * ur + gk[5] * us + gk[2] * ut;
          wr_s[i + rp * j + wpl * k] = wr;
          ws_s[i + rp * j + wpl * k] = ws;
#pragma unroll
          for (int m = 0; m < n; m++) rw[m] = fma(a.Dm[k * n + m], wt, rw[m]);
        }
        // release the G slot only after its last plane was consumed: the w_r / w_s
        // shared stores above depend on the loaded factors and the arrive's memory
        // clobber keeps them before it, so no shared-memory read of the slot is
        // still in flight when the producer's TMA may overwrite it (WAR hazard)
        if (k % PPC == PPC - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&emptyG[sg]);
          if (++sg == NSG) { sg = 0; phg ^= 1u; }
        }
      }
      // PF wrote the slot with generic stores: order them before the producer's
      // next bulk copy (async proxy) into it
      if (PF) fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptyU[su]);   // u slot consumed
      if (++su == NSU) { su = 0; phu ^= 1u; }
      compute_sync<TCW>();                       // w_r / w_s of the group complete
#pragma unroll
      for (int m = 0; m < n; m++) {
        Dti[m] = kDtreg ? sDt[i * dp + m] : 0.0;
        Dtj[m] = kDtreg ? sDt[j * dp + m] : 0.0;
      }
      if (active) {
        const int e = e0 + el;
        double* wg = a.w + (size_t)e * n3;
        uint32_t kmask = 0u;   // bit k set: slot (i,j,k) is a Dirichlet slot
        if (kMask) {
          const bool mij = ((i == 0) && (bm & 1u)) || ((i == n - 1) && (bm & 2u)) ||
                           ((j == 0) && (bm & 4u)) || ((j == n - 1) && (bm & 8u));
          kmask = mij ? 0xffffffffu
                      : (((bm & 16u) ? 1u : 0u) | ((bm & 32u) ? (1u << (n - 1)) : 0u));
        }
#pragma unroll
        for (int k = 0; k < n; k++) {
          double v = rw[k];
#pragma unroll
          for (int m = 0; m < n; m++) {
            v = fma(kDtreg ? Dti[m] : sDt[i * dp + m], wr_s[m + rp * j + wpl * k], v);
            v = fma(kDtreg ? Dtj[m] : sDt[j * dp + m], ws_s[i + rp * m + wpl * k], v);
          }
          if (HELM)   // h1 A_L u + h2 B_L u
            v = a.h1 * v + a.h2 * ((kBpre ? rb[kBpre ? k : 0] : __ldg(Bc + n2 * k)) * ru[k]);
          if (kMask && ((kmask >> k) & 1u)) v = 0.0;
          if (MODE == AX_PCG) acc = fma(ru[k], v, acc);
          wg[ij + n2 * k] = v;
        }
      }

      compute_sync<TCW>();   // w_r / w_s scratch free for the next group
    }
  }

  if (MODE == AX_PCG) {
    if (a.red_out) {
      double v[1] = {acc};
      grid_reduce<1>(v, a.red_partial, a.red_ticket, a.red_out, s_red, &s_misc[1]);
    } else {   // partials only; the consumer kernel sums them (no last-block tail)
      const double bs = block_sum(acc, s_red);
      if (tid == 0) {
        a.red_partial[blockIdx.x] = bs;
        if (blockIdx.x == 0) *a.red_count = gridDim.x;
      }
    }
  }
}

// persistent launch: grid = min(work groups, resident CTAs x SMs) of this variant
template <int n, int MODE, bool HELM, bool PF>
static cudaError_t launch_n(const DevPlan& P, const AxLaunch& a, int groups, cudaStream_t s) {
  using Sh = AxShape<n, PF>;
  auto kern = ax_kernel<n, MODE, HELM, PF>;
  static std::atomic<int> cache[kMaxDev];   // resident CTAs on each device
  const int dev = device_index();
  int resident = cache[dev].load(std::memory_order_relaxed);
  if (resident == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Sh::smem_bytes);
    if (e != cudaSuccess) return e;
    int sms = 148, nb = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, Sh::T, Sh::smem_bytes) != cudaSuccess)
      nb = 1;
    resident = std::max(nb, 1) * sms;
    cache[dev].store(resident, std::memory_order_relaxed);
  }
  const int grid = std::max(1, std::min(groups, resident));
  return launch_k(kern, dim3(grid), dim3(Sh::T), Sh::smem_bytes, s, P, a);
}

template <int n, int MODE>
static int occupancy_n() {
  using Sh = AxShape<n>;
  auto kern = ax_kernel<n, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::smem_bytes);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, Sh::T, Sh::smem_bytes) != cudaSuccess)
    return 1;
  return std::max(nb, 1);
}

template <int MODE, bool HELM = false, bool PF = false>
static cudaError_t dispatch(const DevPlan& P, const AxLaunch& a, int grid, cudaStream_t s) {
#ifdef SEM_AX_ONLY_N8
  if (P.n == 8) return launch_n<8, MODE, HELM, PF>(P, a, grid, s);
  return cudaErrorInvalidValue;
#endif
  switch (P.n) {
    case 2: return launch_n<2, MODE, HELM, PF>(P, a, grid, s);
    case 3: return launch_n<3, MODE, HELM, PF>(P, a, grid, s);
    case 4: return launch_n<4, MODE, HELM, PF>(P, a, grid, s);
    case 5: return launch_n<5, MODE, HELM, PF>(P, a, grid, s);
    case 6: return launch_n<6, MODE, HELM, PF>(P, a, grid, s);
    case 7: return launch_n<7, MODE, HELM, PF>(P, a, grid, s);
    case 8: return launch_n<8, MODE, HELM, PF>(P, a, grid, s);
    case 9: return launch_n<9, MODE, HELM, PF>(P, a, grid, s);
    case 10: return launch_n<10, MODE, HELM, PF>(P, a, grid, s);
    case 11: return launch_n<11, MODE, HELM, PF>(P, a, grid, s);
    case 12: return launch_n<12, MODE, HELM, PF>(P, a, grid, s);
  }
  return cudaErrorInvalidValue;
}

template <int MODE>
static int occ_dispatch(int n) {
#ifdef SEM_AX_ONLY_N8
  return occupancy_n<8, MODE>();
#endif
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
    case 7: return dev::AxCfg<7>::NE;
    case 8: return dev::AxCfg<8>::NE;
    case 9: return dev::AxCfg<9>::NE;
    case 10: return dev::AxCfg<10>::NE;
    case 11: return dev::AxCfg<11>::NE;
    case 12: return dev::AxCfg<12>::NE;
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
                      bool helm, bool pf) {
  if (grid < 1) grid = 1;
  if (pf) {   // one-rank PCG iteration with the p update fused in
    if (mode != AX_PCG) return cudaErrorInvalidValue;
    return helm ? dev::dispatch<AX_PCG, true, true>(P, a, grid, s)
                : dev::dispatch<AX_PCG, false, true>(P, a, grid, s);
  }
  if (helm) {   // Helmholtz: h1 A + h2 B
    if (mode == AX_APPLY) return dev::dispatch<AX_APPLY, true>(P, a, grid, s);
    if (mode == AX_PCG) return dev::dispatch<AX_PCG, true>(P, a, grid, s);
    return cudaErrorInvalidValue;
  }
  if (mode == AX_ONLY) return dev::dispatch<AX_ONLY>(P, a, grid, s);
  if (mode == AX_APPLY) return dev::dispatch<AX_APPLY>(P, a, grid, s);
  return dev::dispatch<AX_PCG>(P, a, grid, s);
}

}  // namespace sem
