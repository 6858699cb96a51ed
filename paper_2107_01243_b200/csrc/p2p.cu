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
#include <cstdint>

#include "dev_common.cuh"
#include "kernels.h"
#include "p2p_dev.cuh"
#include "sem_internal.h"

namespace sem {
namespace dev {

// ---------------------------------------------------------------- gather-scatter exchange
__global__ void gs_pack_p2p_kernel(const DevPlan P, const double* __restrict__ u, double* part,
                                   const P2P c, uint64_t epoch) {
  __shared__ int last;
  if (threadIdx.x < c.nnbr)   // the neighbours finished reading the previous exchange
    wait_flag(mb_gsack(c.local, c.nbrs[threadIdx.x]), epoch - 1, c.err);
  __syncthreads();
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
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&c.tick[0], 1u) == gridDim.x - 1);
  __syncthreads();
  if (last) {
    __threadfence_system();
    if (threadIdx.x < c.nnbr) st_release_sys(mb_gsflag(c.peers[c.nbrs[threadIdx.x]], c.me), epoch);
    if (threadIdx.x == 0) c.tick[0] = 0u;
  }
}

__global__ void gs_unpack_p2p_kernel(const DevPlan P, double* __restrict__ u, const double* part,
                                     const P2P c, uint64_t epoch, int apply_mask, PcgState* st,
                                     int nparts, uint64_t e_sig) {
  __shared__ int last;
  if (st && blockIdx.x == 0 && threadIdx.x == 0) {
    double sg = st->sigma_part[0];
    for (int q = 1; q < nparts; q++) sg += st->sigma_part[q];
    st->loc[2] = sg;
  }
  if (threadIdx.x < c.nnbr) wait_flag(mb_gsflag(c.local, c.nbrs[threadIdx.x]), epoch, c.err);
  __syncthreads();
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
