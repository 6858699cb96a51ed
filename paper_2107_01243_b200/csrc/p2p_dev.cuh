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

// has any wait of this rank already timed out?  (checked only on the slow path:
// after one timeout every later wait gives up at once, so a rank whose peer
// never arrives fails in ~4 s instead of ~4 s per wait)
__device__ __forceinline__ bool p2p_failed(const int* err) {
  return *reinterpret_cast<const volatile int*>(err) != 0;
}

// spin until *flag >= epoch (bounded); returns false on timeout
__device__ __forceinline__ bool wait_flag(const uint64_t* flag, uint64_t epoch, int* err) {
  if (ld_acquire_sys(flag) >= epoch) return true;
  const long long t0 = clock64();
  while (ld_acquire_sys(flag) < epoch) {
    if (p2p_failed(err)) return false;
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
__device__ __forceinline__ uint64_t* mb_ping(char* mb, int r) {
  return reinterpret_cast<uint64_t*>(mb + P2P::kPingOff) + r;
}
// receive entry o of the gather-scatter exchange with the given epoch parity
__device__ __forceinline__ uint4* mb_ll(char* mb, int64_t o, uint64_t epoch) {
  return reinterpret_cast<uint4*>(mb + P2P::kRecvOff) + 2 * o + (epoch & 1);
}
// "LL" store: the 16-byte record is two 8-byte halves, each packing 32 data
// bits with the 32-bit epoch flag as ONE u64 element ((flag << 32) | data).
// st.volatile.v2.u64 makes each half an aligned 8-byte element access, which
// the PTX memory model makes single-copy atomic, so a reader that sees both
// flags equal to the epoch holds both halves of this epoch's value -- no
// fence and no separate flag are needed
__device__ __forceinline__ void ll_store(uint4* p, double v, uint32_t flag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long h0 = ((unsigned long long)flag << 32) | (b & 0xffffffffull);
  const unsigned long long h1 = ((unsigned long long)flag << 32) | (b >> 32);
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(h0), "l"(h1) : "memory");
}
// spin until the record carries this epoch (bounded; on timeout raise err, return 0)
__device__ __forceinline__ double ll_load(const uint4* p, uint32_t flag, int* err) {
  unsigned long long h0, h1;
  long long t0 = -1;
  for (;;) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(h0), "=l"(h1) : "l"(p) : "memory");
    if ((uint32_t)(h0 >> 32) == flag && (uint32_t)(h1 >> 32) == flag) break;
    if (t0 < 0) t0 = clock64();
    else if (p2p_failed(err)) return 0.0;
    else if (clock64() - t0 > (1ll << 33)) {
      atomicExch(err, 1);
      return 0.0;
    }
  }
  return __longlong_as_double((long long)(((h1 & 0xffffffffull) << 32) | (h0 & 0xffffffffull)));
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
