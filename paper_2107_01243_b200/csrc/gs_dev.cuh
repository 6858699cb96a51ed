// Rank-local gather-scatter over the entity plan (shared by kern.cu and p2p.cu).
#pragma once
#include <cstdint>

#include "kernels.h"
#include "sem_internal.h"

namespace sem {
namespace dev {

__device__ __forceinline__ int f_s1(int axis, int n) { return axis == 0 ? n : 1; }
__device__ __forceinline__ int f_s2(int axis, int n) { return axis == 2 ? n : n * n; }
__device__ __forceinline__ int e_sd(int axis, int n) { return axis == 0 ? 1 : (axis == 1 ? n : n * n); }

// standalone gs over the rank-local entities: ascending-slot sum, broadcast
// write, no atomics.  Templated on n so the point -> (entity, offset)
// decomposition is a constant division.  Face points (2 incidences, ~85% of
// the points) are processed F = 4 per thread with all 2F loads issued before any
// use (the kernel is L2-latency bound); edges and vertices one per thread.
template <int n>
__device__ __forceinline__ void gs_local_body(const DevPlan& P, double* __restrict__ u,
                                              int apply_mask, int tid, int nth) {
  constexpr int N = n - 1;
  constexpr int nf = (N - 1) * (N - 1), ne = N - 1;
  constexpr int Nm1 = N > 1 ? N - 1 : 1;
  constexpr int F = 4;
  const int tF = P.nF * nf, tE = P.nEd * ne, tot = tF + tE + P.nV;
  if (nf > 0) {
    for (int t0 = tid; t0 < tF; t0 += nth * F) {
      int a0[F], a1[F];
      bool ok[F];
#pragma unroll
      for (int q = 0; q < F; q++) {
        const int t = t0 + q * nth;
        ok[q] = t < tF;
        const int f = ok[q] ? t / (nf > 0 ? nf : 1) : 0;
        const int p = t - f * nf;
        const int ax = P.f_axis[f];
        const int off = (1 + p % Nm1) * f_s1(ax, n) + (1 + p / Nm1) * f_s2(ax, n);
        const int2 b2 = reinterpret_cast<const int2*>(P.f_base)[f];
        a0[q] = b2.x + off;
        a1[q] = b2.y + off;
      }
      double v0[F], v1[F];
#pragma unroll
      for (int q = 0; q < F; q++)
        if (ok[q]) {
          v0[q] = u[a0[q]];
          v1[q] = u[a1[q]];
        }
#pragma unroll
      for (int q = 0; q < F; q++)
        if (ok[q]) {
          const double s = v0[q] + v1[q];
          u[a0[q]] = s;
          u[a1[q]] = s;
        }
    }
  }
  for (int t = tF + tid; t < tot; t += nth) {
    int32_t base[8];
    int nin, off;
    bool mk = false;
    if (ne > 0 && t < tF + tE) {
      const int q = t - tF, e = q / (ne > 0 ? ne : 1);
      const int p = q - e * ne;
      off = (1 + p) * e_sd(P.e_axis[e], n);
      nin = P.e_nin[e];
      const int4 b4 = reinterpret_cast<const int4*>(P.e_base)[e];
      base[0] = b4.x; base[1] = b4.y; base[2] = b4.z; base[3] = b4.w;
      mk = P.e_mask[e];
    } else {
      const int v = t - tF - tE;
      off = 0;
      nin = P.v_nin[v];
      const int4 b0 = reinterpret_cast<const int4*>(P.v_base)[2 * v];
      const int4 b1 = reinterpret_cast<const int4*>(P.v_base)[2 * v + 1];
      base[0] = b0.x; base[1] = b0.y; base[2] = b0.z; base[3] = b0.w;
      base[4] = b1.x; base[5] = b1.y; base[6] = b1.z; base[7] = b1.w;
      mk = P.v_mask[v];
    }
    double v[8];
#pragma unroll
    for (int x = 0; x < 8; x++)
      if (x < nin) v[x] = u[base[x] + off];
    double s = v[0];
#pragma unroll
    for (int x = 1; x < 8; x++)
      if (x < nin) s += v[x];
    if (apply_mask && mk) s = 0.0;
#pragma unroll
    for (int x = 0; x < 8; x++)
      if (x < nin) u[base[x] + off] = s;
  }
}

}  // namespace dev
}  // namespace sem
