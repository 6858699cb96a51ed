// Rank-local gather-scatter over the entity plan (shared by kern.cu and p2p.cu).
#pragma once
#include <cstdint>

#include "kernels.h"
#include "sem_internal.h"

#ifndef SEM_GS_F
#define SEM_GS_F 2       // face points per thread per round (loads issued together)
#endif
#ifndef SEM_GS_CG
#define SEM_GS_CG 0      // 1: L2-only loads/stores (ld/st .cg)
#endif

namespace sem {
namespace dev {

__device__ __forceinline__ double gs_ld(const double* p) {
#if SEM_GS_CG
  return __ldcg(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ void gs_st(double* p, double v) {
#if SEM_GS_CG
  __stcg(p, v);
#else
  *p = v;
#endif
}

__device__ __forceinline__ int f_s1(int axis, int n) { return axis == 0 ? n : 1; }
__device__ __forceinline__ int f_s2(int axis, int n) { return axis == 2 ? n : n * n; }
__device__ __forceinline__ int e_sd(int axis, int n) { return axis == 0 ? 1 : (axis == 1 ? n : n * n); }

// Flat schedule (w L2-resident or moderately larger): each entity class is
// spread over the whole grid.  The kernel is latency bound (scattered 8-byte
// accesses), so every thread issues ALL its loads of a round before any use:
// the index records of F face points and FE edge points first, then their
// 2F + 4FE data loads, then the sums and the broadcast stores (fire and
// forget).  A round covers nth*F face points and nth*FE edge points
// (consecutive threads on consecutive points of an entity: coalesced where
// the layout allows); vertices (few) follow in a grid-stride loop.  F = 3,
// FE = 1 measured best of (2,1), (3,1), (4,1), (6,2), (8,2) and of the
// round-1 faces-then-edges loop, inside the PCG iteration on C2 and C3
// (profiles/r02_experiments/gs_flat_ab.jsonl).
#ifndef SEM_GS_FF
#define SEM_GS_FF 3
#endif
#ifndef SEM_GS_FFE
#define SEM_GS_FFE 1
#endif
constexpr int kGsF = SEM_GS_FF, kGsFE = SEM_GS_FFE;
// the rounds over the entity ranges [f0, f0 + nFr), [e0, e0 + nEr), [v0, v0 + nVr)
// by threads tid of nth (the flat schedule: every entity, the whole grid; the
// chunk schedule: one chunk's entities, one block)
template <int n, int F = kGsF, int FE = kGsFE>
__device__ __forceinline__ void gs_round_body(const DevPlan& P, double* __restrict__ u,
                                              int apply_mask, int tid, int nth, int f0, int nFr,
                                              int e0, int nEr, int v0, int nVr) {
  constexpr int N = n - 1;
  constexpr int nf = (N - 1) * (N - 1), ne = N - 1;
  constexpr int Nm1 = N > 1 ? N - 1 : 1;
  constexpr int nfd = nf > 0 ? nf : 1, ned = ne > 0 ? ne : 1;
  const int tF = nFr * nf, tE = nEr * ne;
  const int rF = nf > 0 ? (tF + nth * F - 1) / (nth * F) : 0;
  const int rE = ne > 0 ? (tE + nth * FE - 1) / (nth * FE) : 0;
  const int rounds = rF > rE ? rF : rE;
  for (int r = 0; r < rounds; r++) {
    int a0[F], a1[F];
    bool fok[F];
    int eb[FE][4], eoff[FE], enin[FE];
    bool emk[FE];
#pragma unroll
    for (int q = 0; q < F; q++) {
      const int t = (r * F + q) * nth + tid;
      fok[q] = nf > 0 && t < tF;
      const int fl = fok[q] ? t / nfd : 0;
      const int p = t - fl * nf;
      const int f = f0 + fl;
      const int ax = fok[q] ? P.f_axis[f] : 0;
      const int off = (1 + p % Nm1) * f_s1(ax, n) + (1 + p / Nm1) * f_s2(ax, n);
      const int2 b2 = fok[q] ? reinterpret_cast<const int2*>(P.f_base)[f] : make_int2(0, 0);
      a0[q] = b2.x + off;
      a1[q] = b2.y + off;
      SEM_CHK(!fok[q] || (a0[q] >= 0 && a0[q] < a1[q] && a1[q] < P.n_local));
    }
#pragma unroll
    for (int q = 0; q < FE; q++) {
      const int t = (r * FE + q) * nth + tid;
      const bool ok = ne > 0 && t < tE;
      const int el = ok ? t / ned : 0;
      const int p = t - el * ne;
      const int e = e0 + el;
      enin[q] = ok ? P.e_nin[e] : 0;
      eoff[q] = ok ? (1 + p) * e_sd(P.e_axis[e], n) : 0;
      emk[q] = ok && P.e_mask[e];
      const int4 b4 = ok ? reinterpret_cast<const int4*>(P.e_base)[e] : make_int4(0, 0, 0, 0);
      eb[q][0] = b4.x; eb[q][1] = b4.y; eb[q][2] = b4.z; eb[q][3] = b4.w;
#pragma unroll
      for (int x = 0; x < 4; x++)
        SEM_CHK(x >= enin[q] || (eb[q][x] + eoff[q] >= 0 && eb[q][x] + eoff[q] < P.n_local &&
                                 (x == 0 || eb[q][x] > eb[q][x - 1])));
    }
    double v0[F], v1[F], ve[FE][4];
#pragma unroll
    for (int q = 0; q < F; q++)
      if (fok[q]) {
        v0[q] = gs_ld(&u[a0[q]]);
        v1[q] = gs_ld(&u[a1[q]]);
      }
#pragma unroll
    for (int q = 0; q < FE; q++)
#pragma unroll
      for (int x = 0; x < 4; x++)
        if (x < enin[q]) ve[q][x] = gs_ld(&u[eb[q][x] + eoff[q]]);
#pragma unroll
    for (int q = 0; q < F; q++)
      if (fok[q]) {
        const double s = v0[q] + v1[q];
        gs_st(&u[a0[q]], s);
        gs_st(&u[a1[q]], s);
      }
#pragma unroll
    for (int q = 0; q < FE; q++) {
      if (enin[q] == 0) continue;
      double s = ve[q][0];
#pragma unroll
      for (int x = 1; x < 4; x++)
        if (x < enin[q]) s += ve[q][x];
      if (apply_mask && emk[q]) s = 0.0;
#pragma unroll
      for (int x = 0; x < 4; x++)
        if (x < enin[q]) gs_st(&u[eb[q][x] + eoff[q]], s);
    }
  }
  for (int vl = tid; vl < nVr; vl += nth) {
    const int v = v0 + vl;
    const int nin = P.v_nin[v];
    const int4 b0 = reinterpret_cast<const int4*>(P.v_base)[2 * v];
    const int4 b1 = reinterpret_cast<const int4*>(P.v_base)[2 * v + 1];
    const int base[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int x = 0; x < 8; x++)
      SEM_CHK(x >= nin || (base[x] >= 0 && base[x] < P.n_local && (x == 0 || base[x] > base[x - 1])));
    double vv[8];
#pragma unroll
    for (int x = 0; x < 8; x++)
      if (x < nin) vv[x] = gs_ld(&u[base[x]]);
    double s = vv[0];
#pragma unroll
    for (int x = 1; x < 8; x++)
      if (x < nin) s += vv[x];
    if (apply_mask && P.v_mask[v]) s = 0.0;
#pragma unroll
    for (int x = 0; x < 8; x++)
      if (x < nin) gs_st(&u[base[x]], s);
  }
}

template <int n>
__device__ __forceinline__ void gs_flat_body(const DevPlan& P, double* __restrict__ u,
                                             int apply_mask, int tid, int nth) {
  gs_round_body<n>(P, u, apply_mask, tid, nth, 0, P.nF, 0, P.nEd, 0, P.nV);
}

// Rank-local gather-scatter, one sweep in element order.  The planner creates
// every entity from its smallest local element, in element order, so the faces,
// edges and vertices created by elements [e0, e1) are three contiguous index
// ranges.  A block processes one chunk of ce elements (all three classes
// together, while their rows are in L2) and grabs chunks dynamically, so at any
// moment the GPU works on a window of consecutive elements and each element's w
// is streamed from DRAM about once (the earlier class-by-class sweeps read it
// three times).  Per gid: ascending-slot sum, broadcast write, no atomics, so
// the result does not depend on which block did the work.
#ifndef SEM_GS_CHUNK_PTS
#define SEM_GS_CHUNK_PTS 2048   // entity points per chunk (sets ce from N)
#endif
// elements per chunk: ~SEM_GS_CHUNK_PTS entity points (3 faces, 3 edges and one
// vertex per element in the interior of a box)
#ifndef SEM_GS_FLAT_BYTES
#define SEM_GS_FLAT_BYTES (256ll << 20)   // auto mode: flat schedule up to 256 MB of w (C3: 134 MB)
#endif
// mode 0 auto, 1 flat, 2 element-ordered chunks -> ce (0 = flat)
int gs_chunk_elems(int N);
inline int gs_mode_ce(const DevPlan& P, int mode) {
  const bool sweep = mode == 2 || (mode == 0 && P.n_local * 8ll > SEM_GS_FLAT_BYTES);
  return sweep ? gs_chunk_elems(P.N) : 0;
}
inline int gs_chunk_elems(int N) {
  const int w = 3 * (N - 1) * (N - 1) + 3 * (N - 1) + 1;
  const int ce = (SEM_GS_CHUNK_PTS + w - 1) / w;
  return ce < 1 ? 1 : ce;
}

template <int n>
__device__ __forceinline__ void gs_chunk_body(const DevPlan& P, double* __restrict__ u,
                                              int apply_mask, int e0, int e1) {
  constexpr int N = n - 1;
  constexpr int nf = (N - 1) * (N - 1), ne = N - 1;
  constexpr int Nm1 = N > 1 ? N - 1 : 1;
  constexpr int F = SEM_GS_F;
  const int T = blockDim.x;
  // faces: 2 incidences, F points per thread with all 2F loads issued first
  if (nf > 0) {
    const int f0 = P.f_start[e0], tF = (P.f_start[e1] - f0) * nf;
    for (int t0 = threadIdx.x; t0 < tF; t0 += T * F) {
      int a0[F], a1[F];
      bool ok[F];
#pragma unroll
      for (int q = 0; q < F; q++) {
        const int t = t0 + q * T;
        ok[q] = t < tF;
        const int fl = ok[q] ? t / (nf > 0 ? nf : 1) : 0;
        const int p = t - fl * nf;
        const int f = f0 + fl;
        const int ax = P.f_axis[f];
        const int off = (1 + p % Nm1) * f_s1(ax, n) + (1 + p / Nm1) * f_s2(ax, n);
        const int2 b2 = reinterpret_cast<const int2*>(P.f_base)[f];
        a0[q] = b2.x + off;
        a1[q] = b2.y + off;
        SEM_CHK(!ok[q] || (a0[q] >= 0 && a0[q] < a1[q] && a1[q] < P.n_local));
      }
      double v0[F], v1[F];
#pragma unroll
      for (int q = 0; q < F; q++)
        if (ok[q]) {
          v0[q] = gs_ld(&u[a0[q]]);
          v1[q] = gs_ld(&u[a1[q]]);
        }
#pragma unroll
      for (int q = 0; q < F; q++)
        if (ok[q]) {
          const double s = v0[q] + v1[q];
          gs_st(&u[a0[q]], s);
          gs_st(&u[a1[q]], s);
        }
    }
  }
  // edges (N-1 points, 2-4 incidences) and vertices (2-8 incidences): one per thread
  const int ed0 = P.e_start[e0], tE = (P.e_start[e1] - ed0) * ne;
  const int v0i = P.v_start[e0], tot = tE + (P.v_start[e1] - v0i);
  for (int t = threadIdx.x; t < tot; t += T) {
    int32_t base[8];
    int nin, off;
    bool mk = false;
    if (ne > 0 && t < tE) {
      const int q = t / (ne > 0 ? ne : 1);
      const int e = ed0 + q;
      const int p = t - q * ne;
      off = (1 + p) * e_sd(P.e_axis[e], n);
      nin = P.e_nin[e];
      const int4 b4 = reinterpret_cast<const int4*>(P.e_base)[e];
      base[0] = b4.x; base[1] = b4.y; base[2] = b4.z; base[3] = b4.w;
      mk = P.e_mask[e];
    } else {
      const int v = v0i + (t - tE);
      off = 0;
      nin = P.v_nin[v];
      const int4 b0 = reinterpret_cast<const int4*>(P.v_base)[2 * v];
      const int4 b1 = reinterpret_cast<const int4*>(P.v_base)[2 * v + 1];
      base[0] = b0.x; base[1] = b0.y; base[2] = b0.z; base[3] = b0.w;
      base[4] = b1.x; base[5] = b1.y; base[6] = b1.z; base[7] = b1.w;
      mk = P.v_mask[v];
    }
#pragma unroll
    for (int x = 0; x < 8; x++)
      SEM_CHK(x >= nin || (base[x] + off >= 0 && base[x] + off < P.n_local &&
                           (x == 0 || base[x] > base[x - 1])));
    double v[8];
#pragma unroll
    for (int x = 0; x < 8; x++)
      if (x < nin) v[x] = gs_ld(&u[base[x] + off]);
    double s = v[0];
#pragma unroll
    for (int x = 1; x < 8; x++)
      if (x < nin) s += v[x];
    if (apply_mask && mk) s = 0.0;
#pragma unroll
    for (int x = 0; x < 8; x++)
      if (x < nin) gs_st(&u[base[x] + off], s);
  }
}

// Every block grabs chunks from *ctr until they run out.  The counter is never
// reset: a launch starts at `base` and takes exactly nchunks + gridDim.x tickets
// (each block's last grab fails), which the host adds to its copy of base.
// The next ticket is requested before the current chunk is processed and read
// after it, so the atomic's latency hides behind the chunk's loads.
template <int n>
__device__ __forceinline__ void gs_sweep_body(const DevPlan& P, double* __restrict__ u,
                                              int apply_mask, unsigned long long* ctr,
                                              unsigned long long base, int ce) {
  __shared__ long long s_next;
  const long long nch = (P.nloc + ce - 1) / ce;
  if (threadIdx.x == 0) s_next = (long long)(atomicAdd(ctr, 1ull) - base);
  __syncthreads();
  long long c = s_next;
  __syncthreads();
  while (c < nch) {
    unsigned long long nx = 0;
    if (threadIdx.x == 0) nx = atomicAdd(ctr, 1ull);
    const int e0 = (int)c * ce;
    // (the flat schedule's load-all-first rounds over the chunk's entity ranges were
    // measured 10-40 % slower here: profiles/r02_experiments/gs_chunk_rounds.jsonl)
    gs_chunk_body<n>(P, u, apply_mask, e0, min(e0 + ce, P.nloc));
    if (threadIdx.x == 0) s_next = (long long)(nx - base);
    __syncthreads();
    c = s_next;
    __syncthreads();
  }
}

inline long long gs_sweep_tickets(int nloc, int ce, int grid) {
  return ce > 0 ? (nloc + ce - 1) / ce + grid : 0;
}

// SWEEP: element-ordered chunk sweep (ce elements per chunk); else flat
template <int n, bool SWEEP>
__device__ __forceinline__ void gs_local_body(const DevPlan& P, double* __restrict__ u,
                                              int apply_mask, unsigned long long* ctr,
                                              unsigned long long base, int ce) {
  if (SWEEP)
    gs_sweep_body<n>(P, u, apply_mask, ctr, base, ce);
  else
    gs_flat_body<n>(P, u, apply_mask, blockIdx.x * blockDim.x + threadIdx.x,
                    gridDim.x * blockDim.x);
}

}  // namespace dev
}  // namespace sem
