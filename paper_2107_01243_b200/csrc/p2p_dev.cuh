// Device helpers of the NVLink peer-memory collectives (see p2p.cu).
#pragma once
#include <cstdint>

#include "kernels.h"

namespace sem {
namespace dev {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_volatile(const double* p) {
  double v;
  asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// spin until *flag >= epoch (bounded); returns false on timeout
__device__ __forceinline__ bool wait_flag(const uint64_t* flag, uint64_t epoch, int* err) {
  if (ld_acquire_sys(flag) >= epoch) return true;
  const long long t0 = clock64();
  while (ld_acquire_sys(flag) < epoch) {
    if (clock64() - t0 > (1ll << 33)) {   // ~4 s at 2 GHz
      atomicExch(err, 1);
      return false;
    }
  }
  return true;
}

__device__ __forceinline__ double* mb_slot(char* mb, int site, uint64_t epoch, int r) {
  return reinterpret_cast<double*>(mb + P2P::kSlotOff) +
         (((size_t)site * 2 + (epoch & 1)) * P2P::kMaxP + r) * 4;
}
__device__ __forceinline__ uint64_t* mb_arflag(char* mb, int site, int r) {
  return reinterpret_cast<uint64_t*>(mb + P2P::kArFlagOff) + (size_t)site * P2P::kMaxP + r;
}
__device__ __forceinline__ uint64_t* mb_gsflag(char* mb, int r) {
  return reinterpret_cast<uint64_t*>(mb + P2P::kGsFlagOff) + r;
}
__device__ __forceinline__ uint64_t* mb_gsack(char* mb, int r) {
  return reinterpret_cast<uint64_t*>(mb + P2P::kGsAckOff) + r;
}
__device__ __forceinline__ double* mb_recv(char* mb) {
  return reinterpret_cast<double*>(mb + P2P::kRecvOff);
}

// one thread: publish K partials of this rank to every rank
__device__ __forceinline__ void ar_publish(const P2P& c, int site, uint64_t epoch, const double* v, int K) {
  for (int q = 0; q < c.P; q++) {
    double* dst = mb_slot(c.peers[q], site, epoch, c.me);
    for (int k = 0; k < K; k++) dst[k] = v[k];
  }
  __threadfence_system();
  for (int q = 0; q < c.P; q++) st_release_sys(mb_arflag(c.peers[q], site, c.me), epoch);
}

// one thread: wait for all ranks' partials of (site, epoch); sum in ascending rank order
__device__ __forceinline__ void ar_wait_sum(const P2P& c, int site, uint64_t epoch, int K, double* out) {
  for (int r = 0; r < c.P; r++) wait_flag(mb_arflag(c.local, site, r), epoch, c.err);
  for (int k = 0; k < K; k++) out[k] = 0.0;
  for (int r = 0; r < c.P; r++) {
    const double* src = mb_slot(c.local, site, epoch, r);
    for (int k = 0; k < K; k++) out[k] = r == 0 ? ld_volatile(&src[k]) : out[k] + ld_volatile(&src[k]);
  }
}

}  // namespace dev
}  // namespace sem
