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
//   * gather-scatter: the pack kernel writes this rank's partial of every shared
//     point straight into each neighbour's receive buffer (at the neighbour's
//     offset for this rank), the last block releases one epoch flag per
//     neighbour; the unpack kernel acquires its neighbours' flags, adds the rank
//     partials in ascending rank order, scatters, and its last block
//     acknowledges (the neighbours' next pack waits for that acknowledgement,
//     so a receive buffer is never overwritten while being read).
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

// phase timestamps (ns, %globaltimer) of the exchange kernels, block 0 thread 0;
// read with sem_debug_read (instrumentation only)
__device__ unsigned long long g_p2p_ts[16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define P2P_TS(slot) \
  do { if (blockIdx.x == 0 && threadIdx.x == 0) g_p2p_ts[slot] = gtimer(); } while (0)

// ---------------------------------------------------------------- gather-scatter exchange
__global__ void gs_pack_p2p_kernel(const DevPlan P, const double* __restrict__ u, double* part,
                                   const P2P c, uint64_t epoch) {
  __shared__ int last;
  P2P_TS(0);
  if (threadIdx.x < c.nnbr)   // the neighbours finished reading the previous exchange
    wait_flag(mb_gsack(c.local, c.nbrs[threadIdx.x]), epoch - 1, c.err);
  __syncthreads();
  P2P_TS(1);
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < P.nS;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int nl = P.s_nloc[s];
    double v = u[P.s_slot[s]];
    for (int x = 1; x < nl; x++) v += u[P.s_slot[(int64_t)x * P.nS + s]];
    part[s] = v;
    const int nr = P.s_nr[s];
    for (int x = 0; x < nr; x++) {
      const int q = P.s_rank[(int64_t)x * P.nS + s];
      if (q == c.me) continue;
      const int o = P.s_off[(int64_t)x * P.nS + s];
      mb_recv(c.peers[q])[o + c.rdelta[q]] = v;   // NVLink store into the neighbour
    }
  }
  // one system-scope fence per block, cumulative over the block's NVLink
  // stores (ordered before it by the barrier), then the last-block ticket
  __syncthreads();
  P2P_TS(2);
  if (threadIdx.x == 0) {
    __threadfence_system();
    last = (atomicAdd(&c.tick[0], 1u) == gridDim.x - 1);
  }
  __syncthreads();
  P2P_TS(3);
  if (last) {
    if (threadIdx.x == 0) {
      __threadfence_system();
      c.tick[0] = 0u;
      g_p2p_ts[4] = gtimer();
      g_p2p_ts[5] = gridDim.x;
    }
    __syncthreads();
    if (threadIdx.x < c.nnbr) st_release_sys(mb_gsflag(c.peers[c.nbrs[threadIdx.x]], c.me), epoch);
  }
}

__global__ void gs_unpack_p2p_kernel(const DevPlan P, double* __restrict__ u, const double* part,
                                     const P2P c, uint64_t epoch, int apply_mask, PcgState* st,
                                     int nparts, uint64_t e_sig) {
  __shared__ int last;
  P2P_TS(8);
  if (st && blockIdx.x == 0 && threadIdx.x == 0) {
    double sg = st->sigma_part[0];
    for (int q = 1; q < nparts; q++) sg += st->sigma_part[q];
    st->loc[2] = sg;
  }
  if (threadIdx.x < c.nnbr) wait_flag(mb_gsflag(c.local, c.nbrs[threadIdx.x]), epoch, c.err);
  __syncthreads();
  P2P_TS(9);
  const double* recv = mb_recv(c.local);
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < P.nS;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int nr = P.s_nr[s];
    double tot = 0.0;
    for (int x = 0; x < nr; x++) {
      const int o = P.s_off[(int64_t)x * P.nS + s];
      const double v = o < 0 ? part[s] : ld_volatile(&recv[o]);
      tot = x == 0 ? v : tot + v;
    }
    if (apply_mask && P.s_mask[s]) tot = 0.0;
    const int nl = P.s_nloc[s];
    for (int x = 0; x < nl; x++) u[P.s_slot[(int64_t)x * P.nS + s]] = tot;
  }
  __syncthreads();
  P2P_TS(10);
  if (threadIdx.x == 0) {
    __threadfence();
    last = (atomicAdd(&c.tick[1], 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {   // acknowledge: the receive buffer may be overwritten
    if (threadIdx.x < c.nnbr) st_release_sys(mb_gsack(c.peers[c.nbrs[threadIdx.x]], c.me), epoch);
    if (threadIdx.x == 0) {
      c.tick[1] = 0u;
      if (st) {   // PCG: this rank's sigma to every rank's mailbox
        __threadfence();
        const double v = *(volatile double*)&st->loc[2];
        ar_publish(c, AR_SIG, e_sig, &v, 1);
      }
    }
  }
}

// One kernel per operator application for nranks > 1 (Alg. 1 over NVLink):
//  1. pack: this rank's partial of every shared point into the neighbours'
//     receive buffers; the last block to finish releases the neighbours' flags
//     and this rank's own "pack done" flag;
//  2. rank-local gather-scatter (disjoint slots) while the partials travel;
//  3. acquire the neighbours' flags and the own pack-done flag (no block may
//     overwrite a shared slot before every block has packed it), add the rank
//     partials in ascending rank order, scatter; the last block acknowledges
//     and, inside PCG, publishes this rank's sigma.
// Every block is co-resident (grid capped at residency by the launcher), so the
// in-kernel waits cannot starve the blocks they wait for.
template <int n>
__global__ void __launch_bounds__(256) gs_exchange_p2p_kernel(const DevPlan P,
                                                              double* __restrict__ u, double* part,
                                                              const P2P c, uint64_t epoch,
                                                              int apply_mask, PcgState* st,
                                                              int nparts, uint64_t e_sig,
                                                              const double* sig_part,
                                                              const int* sig_count) {
  __shared__ int last;
  const int nth = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
  // ---- 1. pack (only the first npb blocks own shared points; the others go
  //      straight to the local phase and skip the system-scope fence)
  const int npb = min((int)gridDim.x, (P.nS + (int)blockDim.x - 1) / (int)blockDim.x);
  const int nthp = npb * blockDim.x;
  if (blockIdx.x < npb) {
  if (threadIdx.x < c.nnbr) wait_flag(mb_gsack(c.local, c.nbrs[threadIdx.x]), epoch - 1, c.err);
  __syncthreads();
  for (int s = tid; s < P.nS; s += nthp) {
    const int nl = P.s_nloc[s];
    double v = u[P.s_slot[s]];
    for (int x = 1; x < nl; x++) v += u[P.s_slot[(int64_t)x * P.nS + s]];
    part[s] = v;
    const int nr = P.s_nr[s];
    for (int x = 0; x < nr; x++) {
      const int q = P.s_rank[(int64_t)x * P.nS + s];
      if (q == c.me) continue;
      mb_recv(c.peers[q])[P.s_off[(int64_t)x * P.nS + s] + c.rdelta[q]] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    last = (atomicAdd(&c.tick[0], 1u) == (unsigned)npb - 1);
  }
  __syncthreads();
  if (last) {
    if (threadIdx.x == 0) {
      __threadfence_system();
      c.tick[0] = 0u;
    }
    __syncthreads();
    if (threadIdx.x < c.nnbr) st_release_sys(mb_gsflag(c.peers[c.nbrs[threadIdx.x]], c.me), epoch);
    if (threadIdx.x == 32) st_release_sys(mb_gsflag(c.local, c.me), epoch);   // own pack done
  }
  }
  // ---- 2. rank-local entities
  gs_local_body<n>(P, u, apply_mask, tid, nth);
  // ---- 3. unpack
  if (st && blockIdx.x == 0 && threadIdx.x < 32) {
    double sg;
    if (sig_part) {   // this rank's sigma from the Ax kernel's per-CTA partials (fixed order)
      const int G = *sig_count;
      double v = 0.0;
      for (int b = threadIdx.x; b < G; b += 32) v += sig_part[b];
      sg = warp_sum(v);
    } else {
      sg = st->sigma_part[0];
      for (int q = 1; q < nparts; q++) sg += st->sigma_part[q];
    }
    if (threadIdx.x == 0) st->loc[2] = sg;
  }
  if (threadIdx.x < c.nnbr) wait_flag(mb_gsflag(c.local, c.nbrs[threadIdx.x]), epoch, c.err);
  if (threadIdx.x == 32) wait_flag(mb_gsflag(c.local, c.me), epoch, c.err);
  __syncthreads();
  const double* recv = mb_recv(c.local);
  for (int s = tid; s < P.nS; s += nth) {
    const int nr = P.s_nr[s];
    double tot = 0.0;
    for (int x = 0; x < nr; x++) {
      const int o = P.s_off[(int64_t)x * P.nS + s];
      const double v = o < 0 ? __ldcg(&part[s]) : ld_volatile(&recv[o]);
      tot = x == 0 ? v : tot + v;
    }
    if (apply_mask && P.s_mask[s]) tot = 0.0;
    const int nl = P.s_nloc[s];
    for (int x = 0; x < nl; x++) u[P.s_slot[(int64_t)x * P.nS + s]] = tot;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = (atomicAdd(&c.tick[1], 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    if (threadIdx.x < c.nnbr) st_release_sys(mb_gsack(c.peers[c.nbrs[threadIdx.x]], c.me), epoch);
    if (threadIdx.x == 0) {
      c.tick[1] = 0u;
      if (st) {
        __threadfence();
        const double v = *(volatile double*)&st->loc[2];
        ar_publish(c, AR_SIG, e_sig, &v, 1);
      }
    }
  }
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

int p2p_debug_read(unsigned long long* out, int n) {
  if (n > 16) n = 16;
  return cudaMemcpyFromSymbol(out, dev::g_p2p_ts, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -3;
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
                                     cudaStream_t s) {
  static int resident = 0;
  if (resident == 0) {
    int dev = 0, sms = 148, nb = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dev::gs_exchange_p2p_kernel<n>, 256, 0);
    resident = std::max(nb, 1) * sms;
  }
  const int g = resident;   // co-resident grid (the local-gs phase is latency bound)
  dev::gs_exchange_p2p_kernel<n><<<g, 256, 0, s>>>(P, u, part, c, epoch, apply_mask, st, nparts,
                                                   e_sig, sig_part, sig_count);
  return cudaGetLastError();
}

cudaError_t launch_gs_exchange_p2p(const DevPlan& P, double* u, double* part, const P2P& c,
                                   uint64_t epoch, int apply_mask, PcgState* st, int nparts,
                                   uint64_t e_sig, const double* sig_part, const int* sig_count,
                                   cudaStream_t s) {
  switch (P.n) {
    case 2: return launch_exchange_n<2>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 3: return launch_exchange_n<3>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 4: return launch_exchange_n<4>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 5: return launch_exchange_n<5>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 6: return launch_exchange_n<6>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 7: return launch_exchange_n<7>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 8: return launch_exchange_n<8>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 9: return launch_exchange_n<9>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 10: return launch_exchange_n<10>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 11: return launch_exchange_n<11>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
    case 12: return launch_exchange_n<12>(P, u, part, c, epoch, apply_mask, st, nparts, e_sig, sig_part,
                                       sig_count, s);
  }
  return cudaErrorInvalidValue;
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
