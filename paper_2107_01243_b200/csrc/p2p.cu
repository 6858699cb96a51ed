// Multi-GPU communication of the hot path over NVLink peer memory (P:L204-229
// Alg. 1 gather-scatter exchange; P:L353, P:L367 the CG dot-product
// allreduce), without NCCL in the iteration.
//
// Every rank owns a "mailbox" (device memory, CUDA-IPC mapped into every peer):
//   * allreduce slots: [site][epoch parity][sender rank][4] doubles + one epoch
//     flag per (site, sender).  A publisher writes its partials into the slot
//     reserved for it in EVERY rank's mailbox (itself included), then, after a
//     system-scope fence, releases the flag with the epoch.  Consumers acquire
//     all P flags of their own mailbox and sum the partials in ascending rank
//     order -- identical operands and order on every rank, so all ranks hold
//     the bit-identical global value (reading Q10 applied to dot products).
//   * gather-scatter receive entries, one per (shared point, sending neighbour),
//     as 16-byte "LL" records {lo32, epoch, hi32, epoch} with the two epoch
//     parities interleaved.  The packing thread stores its rank's partial
//     straight into the neighbour's entry; the unpacking thread of the
//     neighbour spins on that one entry until both halves carry the epoch.  No
//     fence, flag or ticket sits on the path.  Parity double buffering makes an
//     acknowledgement unnecessary: a rank writes parity e&1 again only at epoch
//     e+2, after it received the neighbour's epoch-(e+1) entries, which the
//     neighbour packed after it had finished reading epoch e (the neighbour
//     relation is symmetric and kernels of one rank run in stream order).
// Spin-waits are bounded (~4 s); on timeout an error flag is raised instead
// of hanging the GPU.  One rank per GPU: every waiting kernel depends only on
// kernels of other GPUs that never wait on it in the same phase.
#include <algorithm>
#include <cstdint>

#include "dev_common.cuh"
#include "gs_dev.cuh"
#include "kernels.h"
#include "p2p_dev.cuh"
#include "sem_internal.h"

namespace sem {
namespace dev {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// per-block phase timestamps of the exchange kernel (instrumentation, read with
// sem_debug_read): [phase][block], phases 0 start, 1 packed, 2 local gs done,
// 3 unpack done, 4 end
constexpr int kXtsBlocks = 2048;
__device__ unsigned long long g_xts[5 * kXtsBlocks];
#ifndef SEM_XUNPACK
#define SEM_XUNPACK 1   // exchange kernel: the non-packer blocks unpack (0: the packers)
#endif
#define XTS(ph) \
  do { if (threadIdx.x == 0 && blockIdx.x < kXtsBlocks) g_xts[(ph) * kXtsBlocks + blockIdx.x] = gtimer(); } while (0)

// ---------------------------------------------------------------- gather-scatter exchange
// this rank's partial of shared point s (ascending local slots), also sent to
// every other rank sharing s
__device__ __forceinline__ void pack_point(const DevPlan& P, const double* u, double* part,
                                           const P2P& c, uint64_t epoch, int s) {
  const int nl = P.s_nloc[s];
  for (int x = 0; x < nl; x++)
    SEM_CHK(P.s_slot[(int64_t)x * P.nS + s] >= 0 && P.s_slot[(int64_t)x * P.nS + s] < P.n_local &&
            (x == 0 || P.s_slot[(int64_t)x * P.nS + s] > P.s_slot[(int64_t)(x - 1) * P.nS + s]));
  double v = u[P.s_slot[s]];
  for (int x = 1; x < nl; x++) v += u[P.s_slot[(int64_t)x * P.nS + s]];
  part[s] = v;
  const int nr = P.s_nr[s];
  for (int x = 0; x < nr; x++) {
    const int q = P.s_rank[(int64_t)x * P.nS + s];
    if (q == c.me) continue;
    ll_store(mb_ll(c.peers[q], P.s_off[(int64_t)x * P.nS + s] + c.rdelta[q], epoch), v,
             (uint32_t)epoch);
  }
}

// the rank partials of s in ascending rank order, masked, scattered to its slots
// (OWN: this rank's partial recomputed from its slots, in pack_point's order,
// instead of read from part[] -- the slots are unchanged until this write)
template <bool OWN = false>
__device__ __forceinline__ void unpack_point(const DevPlan& P, double* u, const double* part,
                                             const P2P& c, uint64_t epoch, int apply_mask, int s) {
  const int nr = P.s_nr[s];
  const int nl = P.s_nloc[s];
  double self = 0.0;
  if (OWN) {
    self = u[P.s_slot[s]];
    for (int x = 1; x < nl; x++) self += u[P.s_slot[(int64_t)x * P.nS + s]];
  }
  double tot = 0.0;
  for (int x = 0; x < nr; x++) {
    const int o = P.s_off[(int64_t)x * P.nS + s];
    SEM_CHK(o < P.nbuf);
    const double v = o < 0 ? (OWN ? self : part[s])
                           : ll_load(mb_ll(c.local, o, epoch), (uint32_t)epoch, c.err);
    tot = x == 0 ? v : tot + v;
  }
  if (apply_mask && P.s_mask[s]) tot = 0.0;
  for (int x = 0; x < nl; x++) u[P.s_slot[(int64_t)x * P.nS + s]] = tot;
}

// PCG: this rank's sigma (fixed-order sum of its partials) to every rank's
// mailbox, one warp.  The partials come from kernels earlier in the stream.
__device__ __forceinline__ void publish_sigma(const P2P& c, PcgState* st, int nparts,
                                              uint64_t e_sig, const double* sig_part,
                                              const int* sig_count) {
  double sg;
  if (sig_part) {   // the Ax kernel's per-CTA partials
    const int G = *sig_count;
    double v = 0.0;
    for (int b0 = threadIdx.x; b0 < G; b0 += 32 * 8) {   // 8 loads in flight per lane
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int b = b0 + 32 * u;
        t[u] = b < G ? __ldcg(&sig_part[b]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) v += t[u];
    }
    sg = warp_sum(v);
  } else {
    sg = st->sigma_part[0];
    for (int q = 1; q < nparts; q++) sg += st->sigma_part[q];
  }
  if (threadIdx.x == 0) {
    st->loc[2] = sg;
    ar_publish(c, AR_SIG, e_sig, &sg, 1);
  }
}

__global__ void gs_pack_p2p_kernel(const DevPlan P, const double* __restrict__ u, double* part,
                                   const P2P c, uint64_t epoch) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < P.nS; s += gridDim.x * blockDim.x)
    pack_point(P, u, part, c, epoch, s);
}

__global__ void gs_unpack_p2p_kernel(const DevPlan P, double* __restrict__ u, const double* part,
                                     const P2P c, uint64_t epoch, int apply_mask, PcgState* st,
                                     int nparts, uint64_t e_sig) {
  if (st && blockIdx.x == gridDim.x - 1 && threadIdx.x < 32)
    publish_sigma(c, st, nparts, e_sig, nullptr, nullptr);
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < P.nS; s += gridDim.x * blockDim.x)
    unpack_point(P, u, part, c, epoch, apply_mask, s);
}

// One kernel per operator application for nranks > 1 (Alg. 1 over NVLink):
//  1. pack: the first npb blocks send this rank's partial of every shared point
//     into the neighbours' receive entries;
//  2. rank-local gather-scatter (slots disjoint from the shared points') while
//     the partials travel;
//  3. the same threads unpack the points they packed (so no block overwrites a
//     slot another block still has to read), waiting per entry.
// Inside PCG the last block publishes this rank's sigma first.  Every block is
// co-resident (grid capped at residency by the launcher), so the waits cannot
// starve a block that has yet to pack.
template <int n, bool SWEEP>
__global__ void __launch_bounds__(256) gs_exchange_p2p_kernel(const DevPlan P,
                                                              double* __restrict__ u, double* part,
                                                              const P2P c, uint64_t epoch,
                                                              int apply_mask, PcgState* st,
                                                              int nparts, uint64_t e_sig,
                                                              const double* sig_part,
                                                              const int* sig_count,
                                                              unsigned long long base, int ce) {
  pdl_wait();
  pdl_trigger();
  XTS(0);
  if (st) {   // PCG iteration: a finished solve consumes no epochs (same on every rank);
              // the chunk schedule must still take its tickets (host-tracked base)
    if (!SWEEP && st->done) return;
    if (epoch == 0) {   // device-side epochs (graph-replayed iterations)
      const uint64_t k = (uint64_t)st->it + 1;
      epoch = st->ep0[0] + k;
      e_sig = st->ep0[1] + k;
    }
  }
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (st && blockIdx.x == gridDim.x - 1 && threadIdx.x < 32)
    publish_sigma(c, st, nparts, e_sig, sig_part, sig_count);
  const int npb = min((int)gridDim.x, (P.nS + (int)blockDim.x - 1) / (int)blockDim.x);
  const int nthp = npb * blockDim.x;
  const bool packer = blockIdx.x < npb;
  // unpack by the non-packer blocks (they finish their local gs share first;
  // the packers' share starts after the pack), each point once its packer block
  // has released the epoch of its finished pack (the pack reads the slots the
  // unpack overwrites); with no non-packer block the packers unpack their own
  const int nun = (int)gridDim.x - npb;
  const bool xun = SEM_XUNPACK && nun > 0 && c.xflag && npb <= P2P::kXflags;
  if (packer) {
    for (int s = tid; s < P.nS; s += nthp) pack_point(P, u, part, c, epoch, s);
    if (xun) {
      // the block's slot reads have returned (their values went into the remote
      // stores) before the barrier, so a plain flag store after it is enough for
      // the unpacker's later overwrite; no fence (a fence here would wait for the
      // NVLink stores: +4-5 us per pack measured).  The unpacker recomputes this
      // rank's partial from the slots instead of reading part[].
      __syncthreads();
      if (threadIdx.x == 0)
        *reinterpret_cast<volatile unsigned long long*>(&c.xflag[blockIdx.x]) = epoch;
    }
  }
  XTS(1);
  gs_local_body<n, SWEEP>(P, u, apply_mask, P.gs_ctr + 1, base, ce);
  XTS(2);
  if (xun) {
    if (!packer)
      for (int s = (blockIdx.x - npb) * blockDim.x + threadIdx.x; s < P.nS; s += nun * blockDim.x) {
        wait_flag(&c.xflag[(s % nthp) / blockDim.x], epoch, c.err);
        unpack_point<true>(P, u, part, c, epoch, apply_mask, s);
      }
  } else if (packer) {
    for (int s = tid; s < P.nS; s += nthp) unpack_point(P, u, part, c, epoch, apply_mask, s);
  }
  XTS(3);
  XTS(4);
}

// ---------------------------------------------------------------- interconnect probes
// Ping-pong between this rank and `peer` through their mailboxes: the lower rank
// releases a flag in the peer's mailbox and waits for the answer in its own; the
// other rank answers.  Round-trip time per sample from %globaltimer (P:L373 samples
// 10,000 ping-pongs for alpha*).
__global__ void p2p_pingpong_kernel(const P2P c, int peer, int iters, uint64_t e0, long long* out) {
  uint64_t* mine = mb_ping(c.local, peer);
  uint64_t* theirs = mb_ping(c.peers[peer], c.me);
  const bool ping = c.me < peer;
  for (int it = 0; it < iters; it++) {
    const uint64_t e = e0 + it + 1;
    if (ping) {
      const unsigned long long t0 = gtimer();
      st_release_sys(theirs, e);
      wait_flag(mine, e, c.err);
      out[it] = (long long)(gtimer() - t0);
    } else {
      wait_flag(mine, e, c.err);
      st_release_sys(theirs, e);
    }
  }
}

// one-sided bandwidth probe: n doubles written into the peer's receive area
// (wrapping at cap doubles), reps times, 16-B vector stores
__global__ void p2p_write_kernel(const P2P c, int peer, const double2* __restrict__ src, int64_t n2,
                                 int64_t cap2, int reps) {
  double2* dst = reinterpret_cast<double2*>(c.peers[peer] + P2P::kRecvOff);
  for (int r = 0; r < reps; r++)
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n2;
         q += (int64_t)gridDim.x * blockDim.x)
      dst[q % cap2] = src[q];
  __threadfence_system();
}

// publish k values from device memory (one thread)
__global__ void ar_publish_kernel(const P2P c, int site, uint64_t epoch, const double* v, int K) {
  double t[4];
  for (int k = 0; k < K; k++) t[k] = v[k];
  ar_publish(c, site, epoch, t, K);
}

// wait and write the global sums (one thread)
__global__ void ar_finish_kernel(const P2P c, int site, uint64_t epoch, double* out, int K) {
  double t[4];
  ar_wait_sum(c, site, epoch, K, t);
  for (int k = 0; k < K; k++) out[k] = t[k];
}

}  // namespace dev

int p2p_debug_read_blocks(unsigned long long* out, int n) {
  if (n > 5 * dev::kXtsBlocks) n = 5 * dev::kXtsBlocks;
  return cudaMemcpyFromSymbol(out, dev::g_xts, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -3;
}

cudaError_t launch_gs_pack_p2p(const DevPlan& P, const double* u, double* part, const P2P& c,
                               uint64_t epoch, cudaStream_t s) {
  int g = (int)((P.nS + 255) / 256);
  g = g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g);
  dev::gs_pack_p2p_kernel<<<g, 256, 0, s>>>(P, u, part, c, epoch);
  return cudaGetLastError();
}

cudaError_t launch_gs_unpack_p2p(const DevPlan& P, double* u, const double* part, const P2P& c,
                                 uint64_t epoch, int apply_mask, PcgState* st, int nparts,
                                 uint64_t e_sig, cudaStream_t s) {
  int g = (int)((P.nS + 255) / 256);
  g = g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g);
  dev::gs_unpack_p2p_kernel<<<g, 256, 0, s>>>(P, u, part, c, epoch, apply_mask, st, nparts,
                                              e_sig);
  return cudaGetLastError();
}

template <int n>
static cudaError_t launch_exchange_n(const DevPlan& P, double* u, double* part, const P2P& c,
                                     uint64_t epoch, int apply_mask, PcgState* st, int nparts,
                                     uint64_t e_sig, const double* sig_part, const int* sig_count,
                                     uint64_t* base, int mode, cudaStream_t s) {
  static std::atomic<int> cache[kMaxDev][2];
  const int dev = device_index();
  int resident[2] = {cache[dev][0].load(std::memory_order_relaxed),
                     cache[dev][1].load(std::memory_order_relaxed)};
  if (resident[0] == 0 || resident[1] == 0) {
    int sms = 148, nb0 = 1, nb1 = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb0, dev::gs_exchange_p2p_kernel<n, false>, 256, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb1, dev::gs_exchange_p2p_kernel<n, true>, 256, 0);
    resident[0] = std::max(nb0, 1) * sms;
    resident[1] = std::max(nb1, 1) * sms;
    cache[dev][0].store(resident[0], std::memory_order_relaxed);
    cache[dev][1].store(resident[1], std::memory_order_relaxed);
  }
  const int ce = dev::gs_mode_ce(P, mode);
  // co-resident grid (the waits must not starve unscheduled blocks)
  const int g = resident[ce > 0 ? 1 : 0];
  const unsigned long long b = *base;
  *base += (uint64_t)dev::gs_sweep_tickets(P.nloc, ce, g);
  // The packers' receive-record waits need every CTA co-resident: the grid is
  // capped at the occupancy-computed residency.  A cooperative launch (the
  // runtime's guarantee) was measured 10 us slower per exchange (C2, 2 GPUs:
  // 39.4 vs 29.4 us, profiles/r02_experiments/coop_launch.txt); a kernel that
  // cannot become co-resident (another stream occupying the SMs) times out
  // after ~4 s and the call returns SEM_ENCCL instead of hanging.
  if (ce > 0)
    return launch_k(dev::gs_exchange_p2p_kernel<n, true>, dim3(g), dim3(256), 0, s, P, u, part, c,
                    epoch, apply_mask, st, nparts, e_sig, sig_part, sig_count, b, ce);
  return launch_k(dev::gs_exchange_p2p_kernel<n, false>, dim3(g), dim3(256), 0, s, P, u, part, c,
                  epoch, apply_mask, st, nparts, e_sig, sig_part, sig_count, b, ce);
}

cudaError_t launch_gs_exchange_p2p(const DevPlan& P, double* u, double* part, const P2P& c,
                                   uint64_t epoch, int apply_mask, PcgState* st, int nparts,
                                   uint64_t e_sig, const double* sig_part, const int* sig_count,
                                   uint64_t* base, int mode, cudaStream_t s) {
  switch (P.n) {
    case 2: return launch_exchange_n<2>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 3: return launch_exchange_n<3>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 4: return launch_exchange_n<4>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 5: return launch_exchange_n<5>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 6: return launch_exchange_n<6>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 7: return launch_exchange_n<7>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 8: return launch_exchange_n<8>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 9: return launch_exchange_n<9>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 10: return launch_exchange_n<10>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 11: return launch_exchange_n<11>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
    case 12: return launch_exchange_n<12>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig,
                                        sig_part, sig_count, base, mode, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_p2p_pingpong(const P2P& c, int peer, int iters, uint64_t e0, long long* out,
                                cudaStream_t s) {
  dev::p2p_pingpong_kernel<<<1, 1, 0, s>>>(c, peer, iters, e0, out);
  return cudaGetLastError();
}

cudaError_t launch_p2p_write(const P2P& c, int peer, const double* src, int64_t n, int64_t cap,
                             int reps, cudaStream_t s) {
  dev::p2p_write_kernel<<<148 * 4, 256, 0, s>>>(c, peer, reinterpret_cast<const double2*>(src),
                                                 n / 2, cap / 2, reps);
  return cudaGetLastError();
}

cudaError_t launch_ar_publish(const P2P& c, int site, uint64_t epoch, const double* v, int K,
                              cudaStream_t s) {
  dev::ar_publish_kernel<<<1, 1, 0, s>>>(c, site, epoch, v, K);
  return cudaGetLastError();
}

cudaError_t launch_ar_finish(const P2P& c, int site, uint64_t epoch, double* out, int K,
                             cudaStream_t s) {
  dev::ar_finish_kernel<<<1, 1, 0, s>>>(c, site, epoch, out, K);
  return cudaGetLastError();
}

}  // namespace sem
