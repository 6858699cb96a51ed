// C ABI of libsem (include/sem.h): context setup, the hot-path entry points
// (sem_ax, sem_gs, sem_apply, sem_pcg_solve, ...) and the multi-rank plumbing.
//
// The operator w = mask(QQ^T A_L u) is two kernels: the Ax kernel (ax.cu; mask
// and the CG sigma partials in its epilogue) and the gather-scatter kernel
// (kern.cu / gs_dev.cuh).  Multi-GPU (Alg. 1, P:L367 allreduce):
// one process per GPU, three transports for the entities shared with other
// ranks and for the CG inner products, all summing in ascending rank order:
//   * NVLink peer memory (default): ONE exchange kernel (p2p.cu) packs this
//     rank's partials straight into the neighbours' IPC-mapped receive
//     records, runs the rank-local gs while they travel and unpacks; the
//     allreduces are mailbox publishes fused into the CG kernels;
//   * NCCL (SEM_OPT_P2P = 0, or when peer mapping fails): Alg. 1 with Ax on
//     the boundary elements, pack, ncclSend/ncclRecv on a communication stream
//     overlapped with Ax on the interior elements and the local gs, unpack;
//     ncclAllReduce for the dots;
//   * loopback (sem_loopback_*; tests): P rank contexts on ONE device in one
//     process, the NCCL transport's pack / copy / unpack and rank-ordered
//     reductions with device copies instead of NCCL (loopback.cu).
// The host never synchronises inside a CG iteration: scalars stay on the
// device and the host polls a "done" flag every kBatch iterations.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.h"
#include "sem_internal.h"

namespace sem {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

}  // namespace sem

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      sem::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                \
      return SEM_ECUDA;                                                                  \
    }                                                                                    \
  } while (0)

#define NCCL_TRY(expr)                                                                   \
  do {                                                                                   \
    ncclResult_t _r = (expr);                                                            \
    if (_r != ncclSuccess) {                                                             \
      sem::set_error(std::string(#expr) + ": " + ncclGetErrorString(_r));                \
      return SEM_ENCCL;                                                                  \
    }                                                                                    \
  } while (0)

#define SEM_TRY(expr)           \
  do {                          \
    int _s = (expr);            \
    if (_s != SEM_OK) return _s; \
  } while (0)

namespace {

constexpr int kBatch = 8;            // iterations enqueued between host polls
constexpr int kTimerClasses = 10;

struct Timer {
  std::vector<cudaEvent_t> pool;     // pairs
  std::vector<int> cls;              // class of each recorded pair
  size_t used = 0;
};

}  // namespace

struct sem_ctx {
  sem::HostPlan hp;
  sem::DevPlan dp;
  int dev = 0, num_sms = 148;
  cudaStream_t stream = nullptr, comm = nullptr;
  ncclComm_t nccl = nullptr;
  sem::LoopComm* loop = nullptr;   // loopback transport (tests), else NCCL / peer memory
  // device data
  double *d_xi = nullptr, *d_w = nullptr, *d_D = nullptr, *d_G = nullptr, *d_B = nullptr,
         *d_dinv = nullptr;
  uint8_t *d_mult = nullptr, *d_bmask = nullptr;
  int32_t *d_fb = nullptr, *d_eb = nullptr, *d_vb = nullptr;
  uint8_t *d_fax = nullptr, *d_eax = nullptr, *d_enin = nullptr, *d_emask = nullptr,
          *d_vnin = nullptr, *d_vmask = nullptr;
  int32_t *d_fst = nullptr, *d_est = nullptr, *d_vst = nullptr;
  unsigned long long* d_gsctr = nullptr;   // gs chunk counters (never reset)
  uint64_t gs_base[2] = {0, 0};            // host copies: tickets taken so far
  int gs_mode = 0;                         // SEM_OPT_GS_MODE
  // NEXT-3: GMRES work space, projection space
  const int* ax_gate = nullptr;            // Ax early-exit flag of GMRES Arnoldi steps
  double *d_V = nullptr, *d_gt = nullptr, *d_kpart = nullptr;
  sem::GmresState* d_gs = nullptr;
  unsigned* d_ktick = nullptr;
  int gm_cap = 0;
  // leading dimension of the multi-vector blocks (V, Z, projection space):
  // n rounded up plus an odd multiple of 128 B, so the k streams a multi-dot
  // reads concurrently do not start at the same power-of-two offset
  int64_t ldv = 0;
  double *d_Z = nullptr, *d_AZ = nullptr, *d_pdelta = nullptr, *d_pbd = nullptr;
  int proj_m = 0, proj_k = 0;
  // NEXT-1: two-level Schwarz (schwarz.cu); the coarse space is a second
  // context at N = 1 on the same mesh and partition
  int precond = SEM_PRECOND_JACOBI;
  int coarse_iters = 10;
  sem_ctx* c0 = nullptr;
  double *d_fS = nullptr, *d_flam = nullptr;     // [nloc][3][n*n], [nloc][3][n]
  double *d_sy = nullptr;                        // local solves (then assembled)
  double *d_b0 = nullptr, *d_x0 = nullptr, *d_dinv0 = nullptr;   // coarse vectors
  sem::PcgState* d_st0 = nullptr;                // coarse CG start state
  double *d_rw = nullptr, *d_z = nullptr;        // flexible PCG: [r | w], z
  double* d_Zs = nullptr;                        // flexible GMRES: M v_j
  int zs_cap = 0;
  // single rank: the coarse solve replayed as one CUDA graph (its launches are
  // argument-stable: flat gs schedule, no peer epochs); gate copied to d_gate
  bool coarse_graph = true;
  int coarse_replicate = -1;   // SEM_OPT_COARSE_REPLICATE: -1 auto, 0 distributed, 1 replicated
  bool c0_repl = false;        // the coarse context in use is the replicated one
  // SEM_OPT_COARSE_ASM: the one-rank coarse level as an assembled operator on
  // its unique vertices (coarse.cu); -1 auto = on whenever the coarse level is single-rank
  int coarse_asm = -1;
  bool casm_ok = false;
  sem::CoarseAsm casm;
  int casm_grid = 1;
  int32_t *d_ccol = nullptr, *d_cu2sp = nullptr, *d_cu2s = nullptr, *d_cuidx = nullptr;
  double *d_cval = nullptr, *d_cvec = nullptr, *d_cpart = nullptr;
  sem::CoarseCg* d_ccg = nullptr;
  bool ax_pdl = true;      // SEM_OPT_AX_PDL (C2: 123.0 -> 121.6 us per PCG iteration)
  bool ax_pdl_now = false; // set around the PCG iteration's Ax launch
  // SEM_OPT_PCG_FUSE: Jacobi-PCG (every P) with the p update fused into the Ax
  // kernel (and x += alpha p into the CG update): three kernels per iteration
  bool pcg_fuse = true;
  bool pf_now = false;            // set around the PCG iteration's Ax launch
  const double* pf_dinv = nullptr;
  // SEM_OPT_PCG_GSU: one-rank fused PCG with the gather-scatter performed on
  // read by the r update (per-element incidence table d_gu, built on first use);
  // -1 auto: when w exceeds the L2
  int pcg_gsu = -1;
  bool gsu_now = false;           // set around the PCG iteration's operator
  bool gs_sigma_now = false;      // the gs kernel of this PCG iteration sums sigma
  int32_t* d_gu = nullptr;
  int pcg_variant = 0;     // SEM_OPT_PCG_VARIANT: 0 standard, 1 single-reduction (Chronopoulos-Gear)
  bool fdm_tc = true;   // SEM_OPT_FDM_TC: n = 8 local solves on the fp64 tensor cores (DMMA)
  cudaGraphExec_t g0exec = nullptr;
  // SEM_OPT_PCG_GRAPH: one-rank PCG batches replayed as a CUDA graph
  bool pcg_graph = true;
  cudaGraphExec_t pg_exec = nullptr;
  double pg_key[4] = {0, 0, 0, 0};
  // SEM_OPT_SCHWARZ_GRAPH: one-rank flexible-PCG (Schwarz) batches replayed as a
  // CUDA graph (the coarse solve's kernels inlined into it)
  bool sw_graph = true;
  bool sw_capturing = false;
  cudaGraphExec_t sw_exec = nullptr;
  double sw_key[6] = {0, 0, 0, 0, 0, 0};
  int64_t sw_launches = 0;
  // SEM_OPT_GMRES_GRAPH: one-rank GMRES restart cycles replayed as a CUDA graph
  bool gm_graph = true;
  cudaGraphExec_t gm_exec = nullptr;
  double gm_key[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  int64_t gm_launches = 0;
  int64_t pg_launches = 0;
  int g0_iters = -1;
  int64_t g0_launches = 0;
  int* d_gate = nullptr;
  cudaStream_t cap_stream = nullptr;   // capture stream (the legacy stream cannot capture)
  // Helmholtz (NEXT-2): operator in use by apply_op / pcg_run, and its Jacobi cache
  bool helm = false;
  double h1 = 1.0, h2 = 0.0;
  double* d_dinv_helm = nullptr;
  double helm_key[2] = {0.0, -1.0};
  int32_t *d_sslot = nullptr, *d_soff = nullptr;
  uint8_t *d_snloc = nullptr, *d_snr = nullptr, *d_smask = nullptr, *d_smult = nullptr;
  int8_t* d_srank = nullptr;
  double *d_part = nullptr, *d_send = nullptr, *d_recv = nullptr;
  // work
  double *d_r = nullptr, *d_p = nullptr, *d_wv = nullptr, *d_tmp = nullptr;
  double* d_partial = nullptr;        // reduction partials
  double* d_partial_ax = nullptr;     // per-CTA sigma partials of the Ax kernel
  int* d_nsig = nullptr;              // their count
  unsigned* d_tickets = nullptr;      // misc tickets
  double* d_scal = nullptr;           // misc scalars
  sem::PcgState* d_st = nullptr;
  sem::PcgState* h_st = nullptr;      // pinned
  double* d_hist = nullptr;
  int hist_cap = 0;
  int last_hist = 0;
  cudaEvent_t ev_pack = nullptr, ev_comm = nullptr, ev_poll = nullptr;
  int ax_grid = 148;
  int red_grid = 592;
  int64_t launches = 0;
  bool timing = false;
  Timer timer;
  double t_ms[kTimerClasses] = {};
  int64_t t_cnt[kTimerClasses] = {};
  bool overlap = false;  // SEM_OPT_OVERLAP: Alg. 1 boundary/interior split (measured slower
                         // on NVLink: the exchange is ~200 KB, the split costs a launch)
  // NVLink peer-memory transport (nranks > 1)
  bool p2p_ok = false, use_p2p = true;
  sem::P2P p2p;
  char* d_mbox = nullptr;
  char** d_peers = nullptr;
  int64_t* d_rdelta = nullptr;
  int32_t* d_nbrs = nullptr;
  int* d_perr = nullptr;
  uint64_t* d_xflag = nullptr;   // exchange kernel: per packer block, the epoch of its finished pack
  std::vector<char*> ipc_opened;
  uint64_t ep_gs = 0, ep_ar[sem::P2P::kSites] = {0, 0, 0, 0};
  std::vector<uint64_t> ep_ping;   // per peer: ping-pong flag epochs
  uint64_t cur_e_sig = 0;   // sigma epoch published by the last PCG apply
  // PCG at P > 1 over peer memory, graph-replayed: the iteration kernels take
  // their epochs from the device state (PcgState::ep0 + iteration) instead of
  // kernel arguments, so a captured batch is argument-stable
  bool dev_ep = false;
};

namespace {

template <typename T>
int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) {
    sem::set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SEM_ENOMEM : SEM_ECUDA;
  }
#if SEM_CHECKED || SEM_POISON   // poison (checked builds): NaN doubles, -1 indices
  // (completed before returning: the caller's stream may be a non-blocking one
  // that does not order after the legacy stream the memset runs on)
  cudaMemset(*p, 0xFF, count * sizeof(T));
  cudaDeviceSynchronize();
#endif
  return SEM_OK;
}

template <typename T>
int upload(T** p, const std::vector<T>& v, cudaStream_t s) {
  SEM_TRY(dalloc(p, v.size()));
  if (!v.empty()) CUDA_TRY(cudaMemcpyAsync(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return SEM_OK;
}

// timing hooks around kernel launches (sem_timing)
int timer_begin(sem_ctx* c, int cls) {
  if (!c->timing) return -1;
  Timer& t = c->timer;
  if (t.used + 2 > t.pool.size()) {
    for (int q = 0; q < 256; q++) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return -1;
      t.pool.push_back(e);
    }
  }
  int idx = (int)t.used;
  t.used += 2;
  t.cls.push_back(cls);
  cudaEventRecord(t.pool[idx], c->stream);
  return idx;
}

void timer_end(sem_ctx* c, int idx) {
  if (idx < 0) return;
  cudaEventRecord(c->timer.pool[idx + 1], c->stream);
}

void timer_collect(sem_ctx* c) {
  Timer& t = c->timer;
  if (t.used == 0) return;
  cudaEventSynchronize(t.pool[t.used - 1]);
  for (size_t q = 0; q < t.cls.size(); q++) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.pool[2 * q], t.pool[2 * q + 1]);
    c->t_ms[t.cls[q]] += ms;
    c->t_cnt[t.cls[q]] += 1;
  }
  t.used = 0;
  t.cls.clear();
}

int check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    sem::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return SEM_ECUDA;
  }
  return SEM_OK;
}

// ---- collectives: NCCL, or the loopback transport (loopback.cu)
int coll_allreduce(sem_ctx* c, const double* in, double* out, size_t count, cudaStream_t s) {
  if (c->loop) return sem::loop_allreduce(c->loop, in, out, count, s);
  NCCL_TRY(ncclAllReduce(in, out, count, ncclDouble, ncclSum, c->nccl, s));
  return SEM_OK;
}

int coll_allgather(sem_ctx* c, const double* in, double* out, size_t count, cudaStream_t s) {
  if (c->loop) return sem::loop_allgather(c->loop, in, out, count * sizeof(double), s);
  NCCL_TRY(ncclAllGather(in, out, count, ncclDouble, c->nccl, s));
  return SEM_OK;
}

// ---- the operator ----------------------------------------------------------
int run_ax(sem_ctx* c, const double* u, double* w, int mode, int r0lo, int r0hi, int r1lo,
           int r1hi, double* red_out) {
  sem::AxLaunch a{};
  a.u = u;
  a.w = w;
  a.G = c->d_G;
  a.r0lo = r0lo; a.r0hi = r0hi; a.r1lo = r1lo; a.r1hi = r1hi;
  a.red_partial = red_out ? c->d_partial : c->d_partial_ax;
  a.red_count = c->d_nsig;
  a.red_ticket = &c->d_st->tickets[0];
  a.red_out = red_out;
  a.done = c->ax_gate ? c->ax_gate : &c->d_st->done;
  a.gate = c->ax_gate ? 1 : 0;
  std::copy(c->hp.D.begin(), c->hp.D.end(), a.Dm);
  a.B = c->d_B;
  a.h1 = c->h1;
  a.h2 = c->h2;
  const int ng = sem::ax_groups(c->hp.N, (r0hi - r0lo)) + sem::ax_groups(c->hp.N, (r1hi - r1lo));
  const int groups = std::max(ng, 1);   // the launcher caps the grid at residency
  int tk = timer_begin(c, mode == sem::AX_ONLY ? 3 : (c->pf_now && mode == sem::AX_PCG ? 9 : 0));
  // PCG iterations: programmatic dependent launch of the Ax kernel alone, its
  // producer prefetching G before waiting for the preceding kernel (SEM_OPT_AX_PDL)
  const bool pdl = c->ax_pdl_now && !c->timing;
  const bool pdl_set = pdl && !sem::pdl_on();   // (already on: every iteration kernel uses PDL)
  a.pdl_pref = pdl ? 1 : 0;
  if (pdl_set) sem::set_pdl(true);
  const bool pf = c->pf_now && mode == sem::AX_PCG;
  if (pf) {   // u is p: p_old in, p_new out (in place)
    a.rr = c->d_r;
    a.dinv = c->pf_dinv;
    a.pout = const_cast<double*>(u);
    a.beta = &c->d_st->beta;
  }
  cudaError_t e = sem::launch_ax(c->dp, a, mode, groups, c->stream,
                                 c->helm && mode != sem::AX_ONLY, pf);
  if (pdl_set) sem::set_pdl(false);
  timer_end(c, tk);
  c->launches++;
  return check(e, "ax kernel");
}

// exchange the shared partials (Alg. 1 lines 1-5, 7, 10-17) on the comm stream
int exchange(sem_ctx* c) {
  CUDA_TRY(cudaEventRecord(c->ev_pack, c->stream));
  CUDA_TRY(cudaStreamWaitEvent(c->comm, c->ev_pack, 0));
  if (c->loop) {
    SEM_TRY(sem::loop_sendrecv(c->loop, c->d_send, c->d_recv, c->hp.nbr_rank, c->hp.nbr_off,
                               c->hp.nbr_cnt, c->comm));
    CUDA_TRY(cudaEventRecord(c->ev_comm, c->comm));
    return SEM_OK;
  }
  NCCL_TRY(ncclGroupStart());
  for (size_t q = 0; q < c->hp.nbr_rank.size(); q++) {
    const int peer = c->hp.nbr_rank[q];
    const size_t off = (size_t)c->hp.nbr_off[q], cnt = (size_t)c->hp.nbr_cnt[q];
    NCCL_TRY(ncclSend(c->d_send + off, cnt, ncclDouble, peer, c->nccl, c->comm));
    NCCL_TRY(ncclRecv(c->d_recv + off, cnt, ncclDouble, peer, c->nccl, c->comm));
  }
  NCCL_TRY(ncclGroupEnd());
  CUDA_TRY(cudaEventRecord(c->ev_comm, c->comm));
  return SEM_OK;
}

// rank-local gather-scatter pass of the operator (masked slots are already
// zero, so every masked entity point sums to zero)
#ifndef SEM_GS_SIGMA
#define SEM_GS_SIGMA 1   // one-rank fused PCG: sigma summed by the gs kernel's last block
#endif
int gs_pass(sem_ctx* c, double* w) {
  int tk = timer_begin(c, 4);
  sem::GsSigma sig;
  if (c->gs_sigma_now) {
    sig.part = c->d_partial_ax;
    sig.count = c->d_nsig;
    sig.st = c->d_st;
  }
  cudaError_t e = sem::launch_gs_local(c->dp, w, 0, &c->gs_base[0], c->gs_mode, c->stream,
                                       c->gs_sigma_now ? &sig : nullptr);
  timer_end(c, tk);
  c->launches++;
  return check(e, "gs kernel");
}

bool p2p(const sem_ctx* c) { return c->p2p_ok && c->use_p2p; }


// global sum of K device doubles (this rank's partials at loc) into glob:
// NVLink mailboxes (publish + rank-ordered sum) or NCCL allreduce
int allreduce_site(sem_ctx* c, int site, const double* loc, double* glob, int K) {
  if (c->hp.nranks == 1) return SEM_OK;
  if (p2p(c)) {
    const uint64_t e = ++c->ep_ar[site];
    CUDA_TRY(sem::launch_ar_publish(c->p2p, site, e, loc, K, c->stream));
    CUDA_TRY(sem::launch_ar_finish(c->p2p, site, e, glob, K, c->stream));
    c->launches += 2;
    return SEM_OK;
  }
  return coll_allreduce(c, loc, glob, (size_t)K, c->stream);
}

// w = mask(QQ^T A_L u) (mode AX_APPLY) or the same plus sigma (AX_PCG)
int apply_op(sem_ctx* c, const double* u, double* w, int mode) {
  const sem::HostPlan& h = c->hp;
  sem::PcgState* st = c->d_st;
  if (h.nranks > 1 && h.nS > 0 && p2p(c) && !c->overlap) {
    // one Ax launch, then ONE exchange kernel: pack into the neighbours'
    // receive buffers, rank-local gs while the partials travel, unpack
    const bool dev_ep = c->dev_ep && mode == sem::AX_PCG;   // epochs from the device state
    const uint64_t e = dev_ep ? 0 : ++c->ep_gs;
    // PCG: the Ax kernel leaves per-CTA sigma partials; the exchange kernel sums them
    SEM_TRY(run_ax(c, u, w, mode, 0, (int)h.nloc, 0, 0, nullptr));
    c->cur_e_sig = mode == sem::AX_PCG ? (dev_ep ? 0 : ++c->ep_ar[sem::AR_SIG]) : 0;
    int tk = timer_begin(c, 4);
    CUDA_TRY(sem::launch_gs_exchange_p2p(c->dp, w, c->d_part, c->p2p, e, 1,
                                         mode == sem::AX_PCG ? st : nullptr, 1, c->cur_e_sig,
                                         c->d_partial_ax, c->d_nsig, &c->gs_base[1], c->gs_mode,
                                         c->stream));
    timer_end(c, tk);
    c->launches++;
    return SEM_OK;
  }
  if (h.nranks > 1 && h.nS > 0 && p2p(c)) {
    // Alg. 1 over NVLink: boundary elements, pack straight into the
    // neighbours' receive buffers, interior elements meanwhile, local gs,
    // then the rank-ordered unpack.
    const uint64_t e = ++c->ep_gs;
    int nparts = 1;
    int tk;
    if (c->overlap && h.ihi > h.ilo) {
      SEM_TRY(run_ax(c, u, w, mode, (int)h.b0lo, (int)h.b0hi, (int)h.b1lo, (int)h.b1hi,
                     &st->sigma_part[0]));
      tk = timer_begin(c, 5);
      CUDA_TRY(sem::launch_gs_pack_p2p(c->dp, w, c->d_part, c->p2p, e, c->stream));
      timer_end(c, tk);
      SEM_TRY(run_ax(c, u, w, mode, (int)h.ilo, (int)h.ihi, 0, 0, &st->sigma_part[1]));
      nparts = 2;
    } else {
      SEM_TRY(run_ax(c, u, w, mode, 0, (int)h.nloc, 0, 0, &st->sigma_part[0]));
      tk = timer_begin(c, 5);
      CUDA_TRY(sem::launch_gs_pack_p2p(c->dp, w, c->d_part, c->p2p, e, c->stream));
      timer_end(c, tk);
    }
    SEM_TRY(gs_pass(c, w));
    // PCG: the unpack also publishes this rank's sigma; the CG update sums it
    c->cur_e_sig = mode == sem::AX_PCG ? ++c->ep_ar[sem::AR_SIG] : 0;
    tk = timer_begin(c, 6);
    CUDA_TRY(sem::launch_gs_unpack_p2p(c->dp, w, c->d_part, c->p2p, e, 1,
                                       mode == sem::AX_PCG ? st : nullptr, nparts, c->cur_e_sig,
                                       c->stream));
    timer_end(c, tk);
    c->launches += 2;
    return SEM_OK;
  }
  if (h.nranks == 1 || h.nS == 0) {
    // single rank: the CG update kernel sums the per-CTA sigma partials itself
    SEM_TRY(run_ax(c, u, w, mode, 0, (int)h.nloc, 0, 0,
                   (mode == sem::AX_PCG && h.nranks == 1) ? nullptr : &st->sigma));
    // SEM_OPT_PCG_GSU: w stays unassembled, the r update gathers on read
    if (!(c->gsu_now && mode == sem::AX_PCG)) SEM_TRY(gs_pass(c, w));
    return SEM_OK;
  }
  int nparts = 1;
  if (h.ihi > h.ilo) {
    SEM_TRY(run_ax(c, u, w, mode, (int)h.b0lo, (int)h.b0hi, (int)h.b1lo, (int)h.b1hi,
                   &st->sigma_part[0]));
    CUDA_TRY(sem::launch_gs_pack(c->dp, w, c->d_part, c->d_send, c->stream));
    c->launches++;
    SEM_TRY(exchange(c));
    SEM_TRY(run_ax(c, u, w, mode, (int)h.ilo, (int)h.ihi, 0, 0, &st->sigma_part[1]));
    nparts = 2;
  } else {
    SEM_TRY(run_ax(c, u, w, mode, 0, (int)h.nloc, 0, 0, &st->sigma_part[0]));
    CUDA_TRY(sem::launch_gs_pack(c->dp, w, c->d_part, c->d_send, c->stream));
    c->launches++;
    SEM_TRY(exchange(c));
  }
  SEM_TRY(gs_pass(c, w));
  CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_comm, 0));
  CUDA_TRY(sem::launch_gs_unpack(c->dp, w, c->d_part, c->d_recv, 1,
                                 mode == sem::AX_PCG ? st : nullptr, nparts, c->stream));
  c->launches++;
  if (mode == sem::AX_PCG) SEM_TRY(coll_allreduce(c, &st->loc[2], &st->sigma, 1, c->stream));
  return SEM_OK;
}

// standalone gs (no mask unless asked): local entities + shared exchange
int gs_op(sem_ctx* c, double* u, int apply_mask) {
  const bool shared = c->hp.nranks > 1 && c->hp.nS > 0;
  if (shared && p2p(c)) {   // one kernel: pack, local entities, unpack
    const uint64_t e = ++c->ep_gs;
    CUDA_TRY(sem::launch_gs_exchange_p2p(c->dp, u, c->d_part, c->p2p, e, apply_mask, nullptr, 1,
                                         0, nullptr, nullptr, &c->gs_base[1], c->gs_mode,
                                         c->stream));
    c->launches++;
    return SEM_OK;
  }
  CUDA_TRY(sem::launch_gs_local(c->dp, u, apply_mask, &c->gs_base[0], c->gs_mode, c->stream));
  c->launches++;
  if (shared) {
    CUDA_TRY(sem::launch_gs_pack(c->dp, u, c->d_part, c->d_send, c->stream));
    c->launches++;
    SEM_TRY(exchange(c));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_comm, 0));
    CUDA_TRY(sem::launch_gs_unpack(c->dp, u, c->d_part, c->d_recv, apply_mask, nullptr, 1, c->stream));
    c->launches++;
  }
  return SEM_OK;
}

int allreduce(sem_ctx* c, double* p, size_t count) {
  if (c->hp.nranks > 1) return coll_allreduce(c, p, p, count, c->stream);
  return SEM_OK;
}

// out-of-place reduction of this rank's partials into the global scalars: safe
// to repeat (kernels of converged iterations are no-ops but the collectives
// still run, re-reducing the same partials)
int allreduce_to(sem_ctx* c, const double* loc, double* glob, size_t count) {
  if (c->hp.nranks > 1) return coll_allreduce(c, loc, glob, count, c->stream);
  return SEM_OK;
}

int ensure_hist(sem_ctx* c, int maxit) {
  if (maxit + 2 <= c->hist_cap) return SEM_OK;
  if (c->d_hist) cudaFree(c->d_hist);
  c->hist_cap = maxit + 2;
  return dalloc(&c->d_hist, (size_t)c->hist_cap);
}

void casm_free(sem_ctx* c) {
  void* ptrs[] = {c->d_ccol, c->d_cu2sp, c->d_cu2s, c->d_cuidx, c->d_cval, c->d_cvec, c->d_cpart,
                  c->d_ccg};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  c->d_ccol = c->d_cu2sp = c->d_cu2s = c->d_cuidx = nullptr;
  c->d_cval = c->d_cvec = c->d_cpart = nullptr;
  c->d_ccg = nullptr;
  c->casm_ok = false;
}

void free_ctx(sem_ctx* c) {
  if (!c) return;
  void* ptrs[] = {c->d_xi, c->d_w, c->d_D, c->d_G, c->d_B, c->d_dinv, c->d_mult, c->d_bmask,
                  c->d_fb, c->d_eb, c->d_vb, c->d_fax, c->d_eax, c->d_enin,
                  c->d_emask, c->d_vnin, c->d_vmask, c->d_sslot, c->d_soff,
                  c->d_snloc, c->d_snr, c->d_smask, c->d_smult, c->d_part, c->d_send,
                  c->d_recv, c->d_r, c->d_p, c->d_wv, c->d_tmp, c->d_partial, c->d_tickets,
                  c->d_scal, c->d_st, c->d_hist, c->d_partial_ax, c->d_nsig, c->d_srank, c->d_fst, c->d_est,
                  c->d_vst, c->d_gsctr, c->d_dinv_helm,
                  c->d_V, c->d_gt, c->d_kpart, c->d_Z, c->d_AZ, c->d_pdelta, c->d_pbd,
                  c->d_fS, c->d_flam, c->d_sy, c->d_b0, c->d_x0, c->d_dinv0, c->d_st0,
                  c->d_rw, c->d_z, c->d_Zs};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->d_gs) cudaFree(c->d_gs);
  if (c->d_ktick) cudaFree(c->d_ktick);
  if (c->d_gu) cudaFree(c->d_gu);
  casm_free(c);
  if (c->c0) free_ctx(c->c0);
  if (c->g0exec) cudaGraphExecDestroy(c->g0exec);
  if (c->pg_exec) cudaGraphExecDestroy(c->pg_exec);
  if (c->sw_exec) cudaGraphExecDestroy(c->sw_exec);
  if (c->gm_exec) cudaGraphExecDestroy(c->gm_exec);
  if (c->d_gate) cudaFree(c->d_gate);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->h_st) cudaFreeHost(c->h_st);
  for (char* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  void* p2ps[] = {c->d_mbox, c->d_peers, c->d_rdelta, c->d_nbrs, c->d_perr, c->d_xflag};
  for (void* p : p2ps)
    if (p) cudaFree(p);
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  if (c->ev_poll) cudaEventDestroy(c->ev_poll);
  for (cudaEvent_t e : c->timer.pool) cudaEventDestroy(e);
  if (c->comm) cudaStreamDestroy(c->comm);
  delete c;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Map every rank's mailbox into this process (CUDA IPC over NVLink); handles and
// receive-buffer offsets are exchanged once with NCCL all-gathers.  Returns
// SEM_OK with c->p2p_ok = false (NCCL transport) if peer mapping is unavailable.
int p2p_setup(sem_ctx* c) {
  const sem::HostPlan& h = c->hp;
  const int P = h.nranks, me = h.rank;
  cudaStream_t s = c->stream;
  if (P > sem::P2P::kMaxP) return SEM_OK;
  // receive entries: 16-byte records, two epoch parities each
  const size_t bytes =
      sem::P2P::kRecvOff + (size_t)std::max<int64_t>(h.nbuf + 1, sem::P2P::kMinRecv) * 2 * 16;
  SEM_TRY(dalloc(&c->d_mbox, bytes));
  CUDA_TRY(cudaMemsetAsync(c->d_mbox, 0, bytes, s));
  // a rank that cannot export its mailbox still runs every collective below
  // (with a zeroed handle), so all ranks reach the agreement allreduce and
  // fall back to NCCL together
  bool ok = true;
  cudaIpcMemHandle_t mine;
  if (cudaIpcGetMemHandle(&mine, c->d_mbox) != cudaSuccess) {
    cudaGetLastError();
    std::memset(&mine, 0, sizeof(mine));
    ok = false;
  }
  char* dh = nullptr;
  SEM_TRY(dalloc(&dh, (size_t)64 * (P + 1)));
  CUDA_TRY(cudaMemcpyAsync(dh, &mine, 64, cudaMemcpyHostToDevice, s));
  NCCL_TRY(ncclAllGather(dh, dh + 64, 64, ncclChar, c->nccl, s));
  std::vector<cudaIpcMemHandle_t> all(P);
  CUDA_TRY(cudaMemcpyAsync(all.data(), dh + 64, (size_t)64 * P, cudaMemcpyDeviceToHost, s));
  // receive-buffer offsets: mine[q] = where q's data lands in my buffer
  std::vector<int64_t> myoff(P, -1);
  for (size_t k = 0; k < h.nbr_rank.size(); k++) myoff[h.nbr_rank[k]] = h.nbr_off[k];
  int64_t* doff = nullptr;
  SEM_TRY(dalloc(&doff, (size_t)P * (P + 1)));
  CUDA_TRY(cudaMemcpyAsync(doff, myoff.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, s));
  NCCL_TRY(ncclAllGather(doff, doff + P, P, ncclInt64, c->nccl, s));
  std::vector<int64_t> alloff((size_t)P * P);
  CUDA_TRY(cudaMemcpyAsync(alloff.data(), doff + P, sizeof(int64_t) * P * P, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  cudaFree(dh);
  cudaFree(doff);
  std::vector<char*> peers(P, nullptr);
  for (int q = 0; q < P && ok; q++) {
    if (q == me) { peers[q] = c->d_mbox; continue; }
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      break;
    }
    peers[q] = static_cast<char*>(ptr);
    c->ipc_opened.push_back(peers[q]);
  }
  // every rank must agree (otherwise all fall back to NCCL)
  {
    double flag = ok ? 0.0 : 1.0;
    double* df = nullptr;
    SEM_TRY(dalloc(&df, 1));
    CUDA_TRY(cudaMemcpyAsync(df, &flag, sizeof(double), cudaMemcpyHostToDevice, s));
    NCCL_TRY(ncclAllReduce(df, df, 1, ncclDouble, ncclSum, c->nccl, s));
    CUDA_TRY(cudaMemcpyAsync(&flag, df, sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(df);
    if (flag > 0.0) return SEM_OK;
  }
  std::vector<int64_t> rdelta(P, 0);
  for (int q = 0; q < P; q++)
    if (myoff[q] >= 0) rdelta[q] = alloff[(size_t)q * P + me] - myoff[q];
  SEM_TRY(upload(reinterpret_cast<char***>(&c->d_peers), peers, s));
  SEM_TRY(upload(&c->d_rdelta, rdelta, s));
  SEM_TRY(upload(&c->d_nbrs, h.nbr_rank, s));
  SEM_TRY(dalloc(&c->d_perr, 1));
  CUDA_TRY(cudaMemsetAsync(c->d_perr, 0, sizeof(int), s));
  SEM_TRY(dalloc(&c->d_xflag, sem::P2P::kXflags));
  CUDA_TRY(cudaMemsetAsync(c->d_xflag, 0, sizeof(uint64_t) * sem::P2P::kXflags, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  sem::P2P& p = c->p2p;
  p.P = P; p.me = me; p.nnbr = (int)h.nbr_rank.size();
  p.local = c->d_mbox; p.peers = c->d_peers; p.rdelta = c->d_rdelta; p.nbrs = c->d_nbrs;
  p.err = c->d_perr;
  p.xflag = c->d_xflag;
  c->ep_ping.assign(P, 0);
  c->p2p_ok = true;
  return SEM_OK;
}

int p2p_check(sem_ctx* c) {
  if (!c->p2p_ok) return SEM_OK;
  int err = 0;
  CUDA_TRY(cudaMemcpy(&err, c->d_perr, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) {
    sem::set_error("peer-memory wait timed out (a rank did not reach the collective)");
    return SEM_ENCCL;
  }
  return SEM_OK;
}

}  // namespace

// =============================================================== C ABI
extern "C" const char* sem_last_error(void) { return sem::g_err.c_str(); }

extern "C" int sem_setup(const sem_mesh* m, int N, sem_ctx** out) {
  if (!m || !out) { sem::set_error("NULL argument"); return SEM_EINVAL; }
  *out = nullptr;
  if (m->nranks > 1 && !m->nccl_comm) { sem::set_error("nranks > 1 needs nccl_comm"); return SEM_EINVAL; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    sem::set_error("no CUDA device (libsem has no CPU fallback)");
    return SEM_ECUDA;
  }
  sem_ctx* c = new (std::nothrow) sem_ctx();
  if (!c) return SEM_ENOMEM;
  int st = sem::build_plan(m, N, &c->hp);
  if (st != SEM_OK) { delete c; return st; }
  const sem::HostPlan& h = c->hp;
  c->stream = static_cast<cudaStream_t>(m->stream);
  auto fail = [&](int s) { free_ctx(c); return s; };
  c->loop = sem::loop_lookup(m->nccl_comm);
  if (c->loop) {
    if (sem::loop_rank(c->loop) != m->rank || sem::loop_size(c->loop) != m->nranks) {
      sem::set_error("loopback communicator rank/size differ from the mesh's rank/nranks");
      return fail(SEM_EINVAL);
    }
  } else {
    c->nccl = static_cast<ncclComm_t>(m->nccl_comm);
  }
#define SETUP_TRY(expr)             \
  do {                              \
    int _s = (expr);                \
    if (_s != SEM_OK) return fail(_s); \
  } while (0)
#define SETUP_CUDA(expr) SETUP_TRY(check((expr), #expr))
  SETUP_CUDA(cudaGetDevice(&c->dev));
  SETUP_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->dev));
  SETUP_CUDA(cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking));
  SETUP_CUDA(cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
  SETUP_CUDA(cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));
  SETUP_CUDA(cudaEventCreateWithFlags(&c->ev_poll, cudaEventDisableTiming));
  cudaStream_t s = c->stream;

  SETUP_TRY(upload(&c->d_xi, h.xi, s));
  SETUP_TRY(upload(&c->d_w, h.w, s));
  SETUP_TRY(upload(&c->d_D, h.D, s));
  SETUP_TRY(upload(&c->d_bmask, h.bmask, s));
  SETUP_TRY(upload(&c->d_fb, h.f_base, s));
  SETUP_TRY(upload(&c->d_fax, h.f_axis, s));
  SETUP_TRY(upload(&c->d_eb, h.e_base, s));
  SETUP_TRY(upload(&c->d_eax, h.e_axis, s));
  SETUP_TRY(upload(&c->d_enin, h.e_nin, s));
  SETUP_TRY(upload(&c->d_emask, h.e_mask, s));
  SETUP_TRY(upload(&c->d_vb, h.v_base, s));
  SETUP_TRY(upload(&c->d_vnin, h.v_nin, s));
  SETUP_TRY(upload(&c->d_vmask, h.v_mask, s));
  SETUP_TRY(upload(&c->d_fst, h.f_start, s));
  SETUP_TRY(upload(&c->d_est, h.e_start, s));
  SETUP_TRY(upload(&c->d_vst, h.v_start, s));
  SETUP_TRY(dalloc(&c->d_gsctr, 2));
  SETUP_CUDA(cudaMemsetAsync(c->d_gsctr, 0, 2 * sizeof(unsigned long long), s));
  SETUP_TRY(upload(&c->d_sslot, h.s_slot, s));
  SETUP_TRY(upload(&c->d_soff, h.s_off, s));
  SETUP_TRY(upload(&c->d_snloc, h.s_nloc, s));
  SETUP_TRY(upload(&c->d_snr, h.s_nr, s));
  SETUP_TRY(upload(&c->d_smask, h.s_mask, s));
  SETUP_TRY(upload(&c->d_smult, h.s_mult, s));
  SETUP_TRY(upload(&c->d_srank, h.s_rank, s));
  SETUP_TRY(dalloc(&c->d_part, (size_t)h.nS));
  SETUP_TRY(dalloc(&c->d_send, (size_t)h.nbuf));
  SETUP_TRY(dalloc(&c->d_recv, (size_t)h.nbuf));
  const size_t nl = (size_t)h.n_local;
  c->ldv = ((h.n_local + 255) / 256) * 256 + 304;   // + 2432 B = 19 x 128 B
  SETUP_TRY(dalloc(&c->d_G, 6 * nl));
  SETUP_TRY(dalloc(&c->d_B, nl));
  SETUP_TRY(dalloc(&c->d_dinv, nl));
  SETUP_TRY(dalloc(&c->d_mult, nl + 2));
  SETUP_TRY(dalloc(&c->d_r, nl));
  SETUP_TRY(dalloc(&c->d_p, nl));
  SETUP_TRY(dalloc(&c->d_wv, nl));
  SETUP_TRY(dalloc(&c->d_st, 1));
  SETUP_CUDA(cudaMemsetAsync(c->d_st, 0, sizeof(sem::PcgState), s));
  SETUP_CUDA(cudaMallocHost(&c->h_st, sizeof(sem::PcgState)));
  SETUP_TRY(ensure_hist(c, 1000));

  sem::DevPlan& P = c->dp;
  P.N = h.N; P.n = h.n; P.nloc = (int)h.nloc; P.n_local = h.n_local;
  P.nF = (int)h.nF; P.nEd = (int)h.nEd; P.nV = (int)h.nV; P.nS = (int)h.nS; P.nbuf = h.nbuf;
  P.D = c->d_D; P.bmask = c->d_bmask;
  P.f_base = c->d_fb; P.f_axis = c->d_fax;
  P.e_base = c->d_eb; P.e_axis = c->d_eax; P.e_nin = c->d_enin; P.e_mask = c->d_emask;
  P.v_base = c->d_vb; P.v_nin = c->d_vnin; P.v_mask = c->d_vmask;
  P.f_start = c->d_fst; P.e_start = c->d_est; P.v_start = c->d_vst; P.gs_ctr = c->d_gsctr;
  P.s_slot = c->d_sslot; P.s_off = c->d_soff; P.s_nloc = c->d_snloc; P.s_nr = c->d_snr;
  P.s_mask = c->d_smask; P.s_mult = c->d_smult;

  // launch geometry (persistent grids sized to the SM count x residency)
  c->ax_grid = c->num_sms * sem::ax_occupancy(h.N, sem::AX_PCG);
  c->red_grid = sem::cg_grid(c->num_sms);
  SETUP_TRY(dalloc(&c->d_partial, (size_t)2 * std::max(c->num_sms * 32, c->red_grid)));
  SETUP_TRY(dalloc(&c->d_partial_ax, (size_t)c->num_sms * 32 + 8));   // >= any Ax grid
  SETUP_TRY(dalloc(&c->d_nsig, 1));
  SETUP_TRY(dalloc(&c->d_tickets, 8));
  SETUP_CUDA(cudaMemsetAsync(c->d_tickets, 0, 8 * sizeof(unsigned), s));
  SETUP_TRY(dalloc(&c->d_scal, 8));

  if (h.nranks > 1 && !c->loop) SETUP_TRY(p2p_setup(c));   // loopback: device copies only
  c->dp.s_rank = c->d_srank;

  // geometry on the device
  int* d_bad = nullptr;
  SETUP_TRY(dalloc(&d_bad, 1));
  SETUP_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
  const double box[6] = {m->x0, m->x1, m->y0, m->y1, m->z0, m->z1};
  SETUP_CUDA(sem::launch_geom(P, c->d_xi, c->d_w, h.e_lo, m->ex, m->ey, m->ez, box, m->deform,
                              m->deform_amp, c->d_G, c->d_B, d_bad, s));
  int bad = 0;
  SETUP_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  SETUP_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_bad);
  // all ranks must agree on a geometry failure before returning
  if (h.nranks > 1) {
    double flag = bad ? 1.0 : 0.0;
    SETUP_CUDA(cudaMemcpyAsync(c->d_scal, &flag, sizeof(double), cudaMemcpyHostToDevice, s));
    SETUP_TRY(coll_allreduce(c, c->d_scal, c->d_scal, 1, s));
    SETUP_CUDA(cudaMemcpyAsync(&flag, c->d_scal, sizeof(double), cudaMemcpyDeviceToHost, s));
    SETUP_CUDA(cudaStreamSynchronize(s));
    bad = flag > 0.0;
  }
  if (bad) {
    sem::set_error("non-positive Jacobian at some GLL point");
    return fail(SEM_EGEOM);
  }
  // multiplicity and Jacobi: d = QQ^T diag(A_L); dinv = mask ? 0 : 1/d (reading Q14)
  SETUP_CUDA(sem::launch_mult(P, c->d_mult, s));
  SETUP_CUDA(sem::launch_diag(P, c->d_G, c->d_dinv, s));
  SETUP_TRY(gs_op(c, c->d_dinv, 0));
  SETUP_CUDA(sem::launch_invert_mask(P, c->d_dinv, s));
  SETUP_CUDA(cudaStreamSynchronize(s));
#undef SETUP_TRY
#undef SETUP_CUDA
  *out = c;
  return SEM_OK;
}

extern "C" int sem_destroy(sem_ctx* c) {
  if (c) {
    cudaStreamSynchronize(c->stream);
    free_ctx(c);
  }
  return SEM_OK;
}

extern "C" int sem_sizes(const sem_ctx* c, int64_t* n_local, int64_t* e_local, int64_t* n_glob) {
  if (!c) { sem::set_error("NULL context"); return SEM_EINVAL; }
  if (n_local) *n_local = c->hp.n_local;
  if (e_local) *e_local = c->hp.nloc;
  if (n_glob) *n_glob = c->hp.nglob;
  return SEM_OK;
}

extern "C" int sem_ax(sem_ctx* c, const double* u, double* w) {
  if (!c || !u || !w || !aligned16(u) || !aligned16(w) || u == w) {
    sem::set_error("sem_ax: bad arguments (NULL, misaligned or aliased pointers)");
    return SEM_EINVAL;
  }
  return run_ax(c, u, w, sem::AX_ONLY, 0, (int)c->hp.nloc, 0, 0, nullptr);
}

extern "C" int sem_gs(sem_ctx* c, double* u) {
  if (!c || !u) { sem::set_error("sem_gs: NULL argument"); return SEM_EINVAL; }
  return gs_op(c, u, 0);
}

extern "C" int sem_apply(sem_ctx* c, const double* u, double* w) {
  if (!c || !u || !w || !aligned16(u) || !aligned16(w) || u == w) {
    sem::set_error("sem_apply: bad arguments (NULL, misaligned or aliased pointers)");
    return SEM_EINVAL;
  }
  return apply_op(c, u, w, sem::AX_APPLY);
}

extern "C" int sem_coords(sem_ctx* c, double* X, double* Y, double* Z) {
  if (!c || !X || !Y || !Z) { sem::set_error("sem_coords: NULL argument"); return SEM_EINVAL; }
  const sem_mesh& m = c->hp.m;
  const double box[6] = {m.x0, m.x1, m.y0, m.y1, m.z0, m.z1};
  CUDA_TRY(sem::launch_coords(c->dp, c->d_xi, c->hp.e_lo, m.ex, m.ey, m.ez, box, m.deform,
                              m.deform_amp, X, Y, Z, c->stream));
  c->launches++;
  return SEM_OK;
}

extern "C" int sem_rhs(sem_ctx* c, const double* f, double* b) {
  if (!c || !f || !b) { sem::set_error("sem_rhs: NULL argument"); return SEM_EINVAL; }
  CUDA_TRY(sem::launch_scale_mask(c->dp, c->d_B, f, b, c->stream));
  c->launches++;
  SEM_TRY(gs_op(c, b, 1));
  if (c->hp.fully_periodic) {
    CUDA_TRY(sem::launch_sum_c(c->dp, c->d_mult, b, c->d_partial, &c->d_tickets[0], c->d_scal,
                               c->red_grid, c->stream));
    SEM_TRY(allreduce(c, c->d_scal, 2));
    CUDA_TRY(sem::launch_sub_scalar(b, c->d_scal, c->hp.n_local, c->stream));
    c->launches += 2;
  }
  return SEM_OK;
}

// ---- PCG building blocks (pcg_run and the Schwarz coarse solve)
struct PcgCtl {
  bool dist = false, pp = false;
  bool pf = false;   // p update fused into the Ax kernel
  bool gu = false;   // one rank: gather-scatter on read in the r update
  double* rg_out = nullptr;
};

// SEM_OPT_PCG_GSU auto: gather on read when w (8 B per slot) exceeds 64 MiB --
// below, the gs kernel runs on an L2-resident w and the separate pass is
// cheaper (C2, 34 MB: 115 vs 123 us per iteration) -- and one z-layer of
// elements holds at most 8 MiB of w: the update streams ~7x the w bytes
// (57 B per slot) between an element and its +z neighbour, whose face
// partners must still be in the L2 then.  N = 7 measurements
// (profiles/r02_experiments/gsu_ab*.jsonl): 32^3 (4 MiB layers) 451 -> 441 us,
// 40^3 (6.5 MiB) -5.7 %, 48^3 (9.4 MiB) -0.7 %, 64x64x32 and C4 (16.8 MiB)
// +9 / +13 %.
constexpr int64_t kGsuAutoBytes = 64ll << 20, kGsuLayerBytes = 8ll << 20;

// x = 0, r = b, p = dinv b, (rho, gamma), start state; the host wrote tol/maxit
static int pcg_enqueue_init(sem_ctx* c, const double* dinv, const double* b, double* x,
                            PcgCtl* k) {
  cudaStream_t s = c->stream;
  sem::PcgState* st = c->d_st;
  k->dist = c->hp.nranks > 1;
  k->pf = c->pcg_fuse;
  k->gu = k->pf && c->hp.nranks == 1 &&
          (c->pcg_gsu > 0 ||
           (c->pcg_gsu < 0 && c->hp.n_local * 8 > kGsuAutoBytes &&
            (int64_t)c->hp.m.ex * c->hp.m.ey * c->hp.n3 * 8 <= kGsuLayerBytes));
  if (k->gu && !c->d_gu) {   // the incidence table, once per context
    std::vector<int32_t> tab;
    sem::build_gu_table(c->hp, &tab);
    CUDA_TRY(cudaMalloc(&c->d_gu, std::max<size_t>(tab.size(), 1) * sizeof(int32_t)));
    CUDA_TRY(cudaMemcpy(c->d_gu, tab.data(), tab.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  k->rg_out = k->dist ? &st->loc[0] : &st->rho_new;   // (rho_new, gamma)
  // peer-memory allreduces fused into the CG kernels (nranks > 1 with NVLink mailboxes)
  k->pp = p2p(c);
  sem::PeerSync ps;
  if (k->pp) ps.c = c->p2p;
  ps.e_pub = ps.e_wait = k->pp ? ++c->ep_ar[sem::AR_RG] : 0;
  CUDA_TRY(sem::launch_cg_init(c->dp, c->d_mult, dinv, b, x, c->d_r, c->d_p, c->d_partial,
                               st, k->rg_out, ps, c->red_grid, s, k->pf ? 1 : 0));
  if (!k->pp) SEM_TRY(allreduce_site(c, sem::AR_RG, &st->loc[0], &st->rho_new, 2));
  CUDA_TRY(sem::launch_cg_start(st, c->d_hist, ps, s));
  c->launches += 2;
  return SEM_OK;
}

// one PCG iteration: w = A p (+ sigma), update (r, rho', gamma), x and p
static int pcg_enqueue_iter(sem_ctx* c, const double* dinv, double* x, const PcgCtl& k) {
  cudaStream_t s = c->stream;
  sem::PcgState* st = c->d_st;
  c->ax_pdl_now = c->ax_pdl;
  c->pf_now = k.pf;
  c->pf_dinv = dinv;
  c->gsu_now = k.gu;
  // one rank, separate gs kernel: sigma summed there, the update reads st->sigma
  const bool gsig = SEM_GS_SIGMA && k.pf && !k.dist && !k.gu;
  c->gs_sigma_now = gsig;
  const int sa = apply_op(c, c->d_p, c->d_wv, sem::AX_PCG);
  c->ax_pdl_now = false;
  c->pf_now = false;
  c->gsu_now = false;
  c->gs_sigma_now = false;
  SEM_TRY(sa);
  if (k.pf) {   // r, x updates and (one rank, peer memory) the end of the iteration
    sem::PeerSync ps;
    if (k.pp) {
      ps.c = c->p2p;
      if (c->dev_ep) {
        ps.dev = st;
      } else {
        ps.e_wait = c->cur_e_sig;
        ps.e_pub = ++c->ep_ar[sem::AR_RG];
      }
    }
    const bool end_here = !k.dist || k.pp;
    int tk = timer_begin(c, 1);
    CUDA_TRY(sem::launch_cg_update(c->dp, c->d_mult, dinv, c->d_r, c->d_wv, c->d_partial, st,
                                   k.rg_out, (k.dist || gsig) ? nullptr : c->d_partial_ax,
                                   c->d_nsig, ps, c->red_grid, s, x, c->d_p, c->d_hist,
                                   end_here ? 1 : 0, k.gu ? c->d_gu : nullptr));
    timer_end(c, tk);
    c->launches++;
    if (!end_here) {   // NCCL / loopback: reduce (rho', gamma), then end the iteration
      SEM_TRY(allreduce_site(c, sem::AR_RG, &st->loc[0], &st->rho_new, 2));
      CUDA_TRY(sem::launch_cg_end_iter(st, c->d_hist, s));
      c->launches++;
    }
    return SEM_OK;
  }
  sem::PeerSync psu, psp;
  if (k.pp) {
    psu.c = psp.c = c->p2p;
    psu.e_wait = c->cur_e_sig;
    psu.e_pub = psp.e_wait = ++c->ep_ar[sem::AR_RG];
  }
  int tk = timer_begin(c, 1);
  CUDA_TRY(sem::launch_cg_update(c->dp, c->d_mult, dinv, c->d_r, c->d_wv, c->d_partial, st,
                                 k.rg_out, k.dist ? nullptr : c->d_partial_ax, c->d_nsig, psu,
                                 c->red_grid, s));
  timer_end(c, tk);
  if (!k.pp) SEM_TRY(allreduce_site(c, sem::AR_RG, &st->loc[0], &st->rho_new, 2));
  tk = timer_begin(c, 2);
  CUDA_TRY(sem::launch_cg_p(c->dp, dinv, c->d_r, c->d_p, x, st, c->d_hist, psp, c->red_grid, s));
  timer_end(c, tk);
  c->launches += 2;
  return SEM_OK;
}

// true residual once at the end (reading Q17), status and result of a PCG solve
static int pcg_finish(sem_ctx* c, const double* b, const double* x, sem_pcg_result* res) {
  cudaStream_t s = c->stream;
  sem::PcgState* st = c->d_st;
  const bool dist = c->hp.nranks > 1;
  const bool pp = p2p(c);
  SEM_TRY(apply_op(c, x, c->d_wv, sem::AX_APPLY));
  sem::PeerSync psr;
  if (pp) {
    psr.c = c->p2p;
    psr.e_pub = ++c->ep_ar[sem::AR_RES];
  }
  CUDA_TRY(sem::launch_cg_residual(c->dp, c->d_mult, b, c->d_wv, c->d_partial, st,
                                   dist ? &st->loc[3] : &st->res_true, psr, c->red_grid, s));
  c->launches++;
  if (pp) {
    CUDA_TRY(sem::launch_ar_finish(c->p2p, sem::AR_RES, psr.e_pub, &st->res_true, 1, s));
    c->launches++;
  } else {
    SEM_TRY(allreduce_site(c, sem::AR_RES, &st->loc[3], &st->res_true, 1));
  }
  CUDA_TRY(cudaMemcpyAsync(c->h_st, st, sizeof(sem::PcgState), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  timer_collect(c);
  SEM_TRY(p2p_check(c));
  const sem::PcgState& hs = *c->h_st;
  c->last_hist = hs.iters;
  if (res) {
    res->iters = hs.iters;
    res->res_final = std::sqrt(hs.gamma);
    res->res_true = std::sqrt(hs.res_true);
  }
  int status;
  if (hs.done == 1) status = SEM_OK;
  else if (hs.done == 2 || hs.done == 3) {
    sem::set_error(hs.done == 2 ? "CG breakdown: p^T A p <= 0" : "CG produced NaN");
    status = SEM_EBREAKDOWN;
  } else status = SEM_NOT_CONVERGED;
  if (res) res->status = status;
  return status;
}


// gate of the operator's Ax kernel (any mode returns early when *g)
struct GateScope {
  sem_ctx* c;
  GateScope(sem_ctx* ctx, const int* g) : c(ctx) { c->ax_gate = g; }
  ~GateScope() { c->ax_gate = nullptr; }
};

// single-reduction (Chronopoulos-Gear) Jacobi PCG (reading Q34): one global
// reduction per iteration -- (gamma, eps) from the update pass and delta from the
// operator application are reduced together (one allreduce at P > 1)
static int cgcg_run(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                    sem_pcg_result* res) {
  if (maxit < 0 || !(tol >= 0.0)) { sem::set_error("bad tol/maxit"); return SEM_EINVAL; }
  SEM_TRY(ensure_hist(c, maxit));
  const sem::HostPlan& h = c->hp;
  const int64_t n = h.n_local;
  cudaStream_t s = c->stream;
  const int sms = c->num_sms;
  const bool dist = h.nranks > 1;
  if (!c->d_rw) SEM_TRY(dalloc(&c->d_rw, 2 * (size_t)c->ldv));
  double *u = c->d_rw, *sv = c->d_rw + c->ldv, *p = c->d_p, *r = c->d_r, *w = c->d_wv;
  const double* dinv = c->helm ? c->d_dinv_helm : c->d_dinv;
  sem::PcgState* st = c->d_st;
  const int* done = &st->done;
  double* out3 = dist ? st->cg3_loc : st->cg3;
  sem::PcgState init{};
  init.tol = tol;
  init.maxit = maxit;
  std::memcpy(c->h_st, &init, sizeof(init));
  CUDA_TRY(cudaMemcpyAsync(st, c->h_st, sizeof(init), cudaMemcpyHostToDevice, s));
  auto op = [&]() -> int {   // w = A u and delta = <w, u>
    GateScope g(c, done);
    if (!dist) {
      SEM_TRY(run_ax(c, u, w, sem::AX_PCG, 0, (int)h.nloc, 0, 0, &st->cg3[2]));
      SEM_TRY(gs_pass(c, w));
    } else {
      SEM_TRY(apply_op(c, u, w, sem::AX_APPLY));
      CUDA_TRY(sem::launch_mdot(n, c->d_mult, u, w, n, 1, c->d_partial, &c->d_tickets[6],
                                &out3[2], done, sms, s));
      c->launches++;
    }
    if (dist) SEM_TRY(allreduce_to(c, st->cg3_loc, st->cg3, 3));   // the one reduction
    return SEM_OK;
  };
  CUDA_TRY(sem::launch_cgcg_init(n, b, dinv, c->d_mult, x, r, u, p, sv, c->d_partial,
                                 &c->d_tickets[6], out3, sms, s));
  SEM_TRY(op());
  CUDA_TRY(sem::launch_cgcg_scalar(0, st, c->d_hist, s));
  c->launches += 2;
  int hd = 0;
  for (int it = 0; it < maxit && !hd; it += kBatch) {
    const int nb = std::min(kBatch, maxit - it);
    for (int q = 0; q < nb; q++) {
      int tk = timer_begin(c, 1);
      CUDA_TRY(sem::launch_cgcg_update(n, dinv, c->d_mult, u, w, p, sv, x, r, c->d_partial,
                                       &c->d_tickets[6], out3, st, sms, s));
      timer_end(c, tk);
      SEM_TRY(op());
      CUDA_TRY(sem::launch_cgcg_scalar(1, st, c->d_hist, s));
      c->launches += 2;
    }
    CUDA_TRY(cudaMemcpyAsync(&c->h_st->done, done, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    hd = c->h_st->done;
  }
  return pcg_finish(c, b, x, res);
}

// One rank, flat gather-scatter schedule: the kernels of kBatch PCG iterations
// have fixed arguments (no gs chunk tickets, no peer-memory epochs), so the
// batch is captured once into a CUDA graph (SEM_OPT_PCG_GRAPH) and replayed;
// the graph is keyed by the operands that enter the kernel arguments.
// Returns nullptr (plain stream launches) when not applicable.
static cudaGraphExec_t pcg_batch_graph(sem_ctx* c, const double* dinv, double* x, const PcgCtl& k) {
  if (!c->pcg_graph || (c->hp.nranks > 1 && !c->dev_ep) || c->timing || c->ax_gate ||
      !sem::gs_flat(c->dp, c->gs_mode))
    return nullptr;
  const double key[4] = {(double)(uintptr_t)x, (double)(uintptr_t)dinv, c->helm ? c->h1 : -1.0,
                         c->helm ? c->h2 : -1.0};
  if (c->pg_exec && std::memcmp(key, c->pg_key, sizeof(key)) == 0) return c->pg_exec;
  if (c->pg_exec) cudaGraphExecDestroy(c->pg_exec);
  c->pg_exec = nullptr;
  if (!c->cap_stream && cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  // capture on a private stream (the context stream may be the legacy one)
  cudaStream_t s_save = c->stream;
  c->stream = c->cap_stream;
  const int64_t l0 = c->launches;
  cudaGraph_t graph = nullptr;
  int st = SEM_OK;
  if (cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    for (int q = 0; q < kBatch && st == SEM_OK; q++) st = pcg_enqueue_iter(c, dinv, x, k);
    if (cudaStreamEndCapture(c->cap_stream, &graph) != cudaSuccess) st = SEM_ECUDA;
  } else {
    st = SEM_ECUDA;
  }
  c->stream = s_save;
  c->pg_launches = c->launches - l0;
  c->launches = l0;
  cudaGraphExec_t ge = nullptr;
  if (st == SEM_OK && graph && cudaGraphInstantiate(&ge, graph, 0) != cudaSuccess) ge = nullptr;
  if (graph) cudaGraphDestroy(graph);
  cudaGetLastError();
  if (!ge) {
    c->pcg_graph = false;   // not capturable here: plain stream launches from now on
    return nullptr;
  }
  c->pg_exec = ge;
  std::memcpy(c->pg_key, key, sizeof(key));
  return ge;
}

static int pcg_run(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                   sem_pcg_result* res) {
  if (maxit < 0 || !(tol >= 0.0)) { sem::set_error("bad tol/maxit"); return SEM_EINVAL; }
  if (c->pcg_variant == 1) return cgcg_run(c, b, x, tol, maxit, res);
  SEM_TRY(ensure_hist(c, maxit));
  cudaStream_t s = c->stream;
  sem::PcgState* st = c->d_st;
  // scalars: tol, maxit
  sem::PcgState init{};
  init.tol = tol;
  init.maxit = maxit;
  std::memcpy(c->h_st, &init, sizeof(init));   // h_st is idle: every solve ends synchronised
  CUDA_TRY(cudaMemcpyAsync(st, c->h_st, sizeof(init), cudaMemcpyHostToDevice, s));
  const double* dinv = c->helm ? c->d_dinv_helm : c->d_dinv;   // Jacobi of the operator in use
  static_assert(offsetof(sem::PcgState, done) == offsetof(sem::PcgState, it) + sizeof(int),
                "the host polls (it, done) with one copy");
  PcgCtl k;
  c->dev_ep = false;
  SEM_TRY(pcg_enqueue_init(c, dinv, b, x, &k));
  // P > 1 over peer memory with graph replay: device-side epochs from here on
  c->dev_ep = k.pp && k.pf && c->pcg_graph && !c->timing && !c->ax_gate && !c->overlap &&
              sem::gs_flat(c->dp, c->gs_mode);
  if (c->dev_ep) {
    c->h_st->ep0[0] = c->ep_gs;
    c->h_st->ep0[1] = c->ep_ar[sem::AR_SIG];
    c->h_st->ep0[2] = c->ep_ar[sem::AR_RG];
    CUDA_TRY(cudaMemcpyAsync(st->ep0, c->h_st->ep0, sizeof(st->ep0), cudaMemcpyHostToDevice, s));
  }
  int done = 0;
  for (int it = 0; it < maxit && !done; it += kBatch) {
    const int nb = std::min(kBatch, maxit - it);
    cudaGraphExec_t ge = nb == kBatch ? pcg_batch_graph(c, dinv, x, k) : nullptr;
    if (ge) {
      CUDA_TRY(cudaGraphLaunch(ge, s));
      c->launches += c->pg_launches;
    } else {
      for (int q = 0; q < nb; q++) SEM_TRY(pcg_enqueue_iter(c, dinv, x, k));
    }
    // (it, done) adjacent in the state: the iteration count advances the epochs
    CUDA_TRY(cudaMemcpyAsync(&c->h_st->it, &st->it, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaEventRecord(c->ev_poll, s));
    CUDA_TRY(cudaEventSynchronize(c->ev_poll));
    done = c->h_st->done;
  }
  if (c->dev_ep) {   // the host's epoch counters continue after the device-side ones
    const uint64_t kit = (uint64_t)c->h_st->it;
    c->ep_gs = c->h_st->ep0[0] + kit;
    c->ep_ar[sem::AR_SIG] = c->h_st->ep0[1] + kit;
    c->ep_ar[sem::AR_RG] = c->h_st->ep0[2] + kit;
    c->dev_ep = false;
  }
  return pcg_finish(c, b, x, res);
}


// ---------------------------------------------------------------- NEXT-1: Schwarz
// two-level additive overlapping Schwarz (readings Q28-Q32;
// kernels in schwarz.cu).  The coarse space is a second context at N = 1 on
// the same mesh and element partition (its operator, gather-scatter, PCG
// kernels and multi-GPU transports are the fine level's, at n = 2).
// replicated coarse solve (nranks > 1): every rank all-gathers the restricted
// right-hand side and solves the whole N = 1 problem itself (one NCCL
// all-gather instead of a gather-scatter exchange and two allreduces in each
// of the ten coarse CG steps; graph-replayable like one rank).  Auto: when the
// coarse problem is small (<= kReplicateSlots coarse slots) and the element
// partition is even (equal all-gather blocks).
// With the assembled coarse operator (Q35) the replicated solve is cheap up to
// the assembly bound: C4 (2.1 M coarse slots) Schwarz PCG 134.0 -> 126.8 ms at
// 2 GPUs, 81.7 -> 75.7 ms at 4 (profiles/r02_schwarz_scale/); it was 2^20
// slots with the E-vector coarse CG.
constexpr int64_t kReplicateSlots = int64_t(1) << 26;
static bool coarse_replicated(const sem_ctx* c) {
  const sem::HostPlan& h = c->hp;
  if (h.nranks == 1 || h.E % h.nranks != 0) return false;
  if (c->coarse_replicate >= 0) return c->coarse_replicate == 1;
  return h.E * 8 <= kReplicateSlots;
}

static int coarse_assemble(sem_ctx* c);
#ifndef SEM_COARSE_CLUSTER
#define SEM_COARSE_CLUSTER 1   // small assembled coarse problems on one thread-block cluster
#endif

static int schwarz_setup(sem_ctx* c) {
  if (c->c0) return SEM_OK;
  const sem::HostPlan& h = c->hp;
  cudaStream_t s = c->stream;
  sem_ctx* c0 = nullptr;
  c->c0_repl = coarse_replicated(c);
  if (c->c0_repl) {   // the whole coarse mesh on this rank
    sem_mesh m0 = h.m;
    m0.rank = 0;
    m0.nranks = 1;
    m0.nccl_comm = nullptr;
    SEM_TRY(sem_setup(&m0, 1, &c0));
  } else {
    SEM_TRY(sem_setup(&h.m, 1, &c0));   // collective for nranks > 1
  }
  c->c0 = c0;
  if (c0->hp.nranks == 1) c0->gs_mode = 1;   // flat schedule: graph-stable launches (bit-identical)
  const size_t nloc = (size_t)h.nloc, n = (size_t)h.n;
  if (!c->d_fS) {
    SEM_TRY(dalloc(&c->d_fS, nloc * 3 * n * n));
    SEM_TRY(dalloc(&c->d_flam, nloc * 3 * n));
    SEM_TRY(dalloc(&c->d_sy, (size_t)h.n_local));
    const sem_mesh& m = h.m;
    const double box[6] = {m.x0, m.x1, m.y0, m.y1, m.z0, m.z1};
    CUDA_TRY(sem::launch_fdm_setup(h.n, (int)h.nloc, h.e_lo, m.ex, m.ey, m.ez, box, m.deform,
                                   m.deform_amp, m.periodic, c->d_xi, c->d_w, c->d_D, c->d_fS,
                                   c->d_flam, s));
    c->launches++;
  }
  const size_t n0 = (size_t)c0->hp.n_local;
  SEM_TRY(dalloc(&c->d_b0, n0));
  SEM_TRY(dalloc(&c->d_x0, n0));
  if (!c->d_st0) SEM_TRY(dalloc(&c->d_st0, 1));
  // plain CG on the coarse level: the "Jacobi" vector is 1 on unmasked slots
  std::vector<double> ones(n0, 1.0);
  SEM_TRY(upload(&c->d_dinv0, ones, s));
  CUDA_TRY(sem::launch_invert_mask(c0->dp, c->d_dinv0, s));
  c->launches++;
  CUDA_TRY(cudaStreamSynchronize(s));
  return coarse_assemble(c);
}

// The single-rank coarse level as an assembled operator (coarse.cu, reading
// Q35): the element matrices A_e of the N = 1 operator, column by column
// (A_e e_a through the element kernel, no gs, no mask), summed on the host in
// ascending element order into A0 on the unmasked unique vertices (ascending
// global lattice number); ELL on the device with each row's entries in
// ascending column order.  Plus the slot <-> unique maps for the restriction
// (ascending-slot sums) and the prolongation.
static int coarse_assemble(sem_ctx* c) {
  sem_ctx* c0 = c->c0;
  if (!c0 || c->casm_ok || c0->hp.nranks != 1 || c->coarse_asm == 0) return SEM_OK;
  const sem::HostPlan& h0 = c0->hp;
  const int64_t n0 = h0.n_local, E = h0.nloc;
  // the host assembly holds the 8 columns of every element matrix (64 B per
  // coarse slot): beyond 2^26 slots the coarse level stays in E-vector form
  if (n0 > (int64_t(1) << 26)) return SEM_OK;
  cudaStream_t s = c0->stream;
  double *du = nullptr, *dw = nullptr;
  SEM_TRY(dalloc(&du, (size_t)n0));
  int st = dalloc(&dw, (size_t)n0);
  std::vector<double> u((size_t)n0), Ae((size_t)8 * n0);
  for (int a = 0; a < 8 && st == SEM_OK; a++) {
    for (int64_t q = 0; q < n0; q++) u[q] = (q % 8 == a) ? 1.0 : 0.0;
    if (cudaMemcpyAsync(du, u.data(), n0 * sizeof(double), cudaMemcpyHostToDevice, s) != cudaSuccess)
      st = SEM_ECUDA;
    if (st == SEM_OK) st = sem_ax(c0, du, dw);
    if (st == SEM_OK &&
        (cudaMemcpyAsync(Ae.data() + (size_t)a * n0, dw, n0 * sizeof(double), cudaMemcpyDeviceToHost,
                         s) != cudaSuccess ||
         cudaStreamSynchronize(s) != cudaSuccess))
      st = SEM_ECUDA;
  }
  cudaFree(du);
  cudaFree(dw);
  if (st != SEM_OK) {
    cudaGetLastError();
    sem::set_error("coarse_assemble: element matrices");
    return st;
  }
  // unique numbering of the unmasked vertices, ascending global number
  std::vector<int64_t> gid((size_t)n0);
  std::vector<int32_t> cidx((size_t)h0.nglob, -1), uidx((size_t)n0, -1);
  for (int64_t el = 0; el < E; el++)
    for (int a = 0; a < 8; a++) {
      const int i = a & 1, j = (a >> 1) & 1, k = a >> 2;
      const int64_t sl = el * 8 + a;
      gid[sl] = sem::lattice_gid(h0, h0.e_lo + el, i, j, k);
      if (sem::slot_masked(h0, h0.e_lo + el, i, j, k)) gid[sl] = -1;
      else cidx[gid[sl]] = -2;
    }
  int nu = 0;
  for (int64_t g = 0; g < h0.nglob; g++)
    if (cidx[g] == -2) cidx[g] = nu++;
  std::vector<int32_t> u2sp((size_t)nu + 1, 0), u2s;
  for (int64_t sl = 0; sl < n0; sl++)
    if (gid[sl] >= 0) {
      uidx[sl] = cidx[gid[sl]];
      u2sp[uidx[sl] + 1]++;
    }
  for (int g = 0; g < nu; g++) u2sp[g + 1] += u2sp[g];
  u2s.assign((size_t)u2sp[nu], 0);
  {
    std::vector<int32_t> fill(u2sp.begin(), u2sp.end() - 1);
    for (int64_t sl = 0; sl < n0; sl++)   // ascending slots per unique vertex
      if (uidx[sl] >= 0) u2s[fill[uidx[sl]]++] = (int32_t)sl;
  }
  // A0 rows: <= 27 distinct columns on the vertex lattice
  constexpr int kW = 27;
  std::vector<int32_t> rc((size_t)nu * kW, -1);
  std::vector<double> rv((size_t)nu * kW, 0.0);
  std::vector<uint8_t> rn((size_t)nu, 0);
  for (int64_t el = 0; el < E; el++)
    for (int b = 0; b < 8; b++) {
      const int row = uidx[el * 8 + b];
      if (row < 0) continue;
      int32_t* cr = &rc[(size_t)row * kW];
      double* vr = &rv[(size_t)row * kW];
      for (int a = 0; a < 8; a++) {
        const int col = uidx[el * 8 + a];
        if (col < 0) continue;
        const double v = Ae[(size_t)a * n0 + el * 8 + b];
        int q = 0;
        while (q < rn[row] && cr[q] != col) q++;
        if (q == rn[row]) {
          if (q == kW) {
            sem::set_error("coarse_assemble: more than 27 columns in a row");
            return SEM_EINVAL;
          }
          cr[q] = col;
          vr[q] = v;
          rn[row]++;
        } else {
          vr[q] += v;
        }
      }
    }
  int K = 1;
  for (int g = 0; g < nu; g++) K = std::max<int>(K, rn[g]);
  std::vector<int32_t> ecol((size_t)K * nu);
  std::vector<double> eval((size_t)K * nu);
  for (int g = 0; g < nu; g++) {
    int ord[kW];
    const int m = rn[g];
    for (int q = 0; q < m; q++) ord[q] = q;
    const int32_t* cr = &rc[(size_t)g * kW];
    std::sort(ord, ord + m, [&](int x, int y) { return cr[x] < cr[y]; });
    for (int q = 0; q < K; q++) {
      ecol[(size_t)q * nu + g] = q < m ? cr[ord[q]] : g;
      eval[(size_t)q * nu + g] = q < m ? rv[(size_t)g * kW + ord[q]] : 0.0;
    }
  }
  cudaStream_t sc = c->stream;
  c->casm_grid = sem::coarse_asm_grid(nu, c->num_sms);
  SEM_TRY(upload(&c->d_ccol, ecol, sc));
  SEM_TRY(upload(&c->d_cval, eval, sc));
  SEM_TRY(upload(&c->d_cu2sp, u2sp, sc));
  SEM_TRY(upload(&c->d_cu2s, u2s, sc));
  SEM_TRY(upload(&c->d_cuidx, uidx, sc));
  SEM_TRY(dalloc(&c->d_cvec, (size_t)5 * std::max(nu, 1)));
  SEM_TRY(dalloc(&c->d_cpart, (size_t)c->casm_grid));
  SEM_TRY(dalloc(&c->d_ccg, 1));
  CUDA_TRY(cudaMemsetAsync(c->d_ccg, 0, sizeof(sem::CoarseCg), sc));
  CUDA_TRY(cudaStreamSynchronize(sc));
  sem::CoarseAsm& A = c->casm;
  A.nu = nu;
  A.K = K;
  A.n0 = n0;
  A.periodic = h0.fully_periodic ? 1 : 0;
  A.col = c->d_ccol;
  A.val = c->d_cval;
  A.u2s_ptr = c->d_cu2sp;
  A.u2s = c->d_cu2s;
  A.uidx = c->d_cuidx;
  A.b = c->d_cvec;
  A.x = A.b + nu;
  A.r = A.x + nu;
  A.p = A.r + nu;
  A.q = A.p + nu;
  A.partial = c->d_cpart;
  A.st = c->d_ccg;
  c->casm_ok = true;
  return SEM_OK;
}

// drop the coarse level (rebuilt by the next schwarz_setup)
static void schwarz_drop_coarse(sem_ctx* c) {
  if (!c->c0) return;
  cudaStreamSynchronize(c->stream);
  free_ctx(c->c0);
  c->c0 = nullptr;
  double* bufs[3] = {c->d_b0, c->d_x0, c->d_dinv0};
  for (double* p : bufs)
    if (p) cudaFree(p);
  c->d_b0 = c->d_x0 = c->d_dinv0 = nullptr;
  casm_free(c);
  if (c->sw_exec) cudaGraphExecDestroy(c->sw_exec);
  c->sw_exec = nullptr;
  if (c->gm_exec) cudaGraphExecDestroy(c->gm_exec);
  c->gm_exec = nullptr;
  if (c->g0exec) cudaGraphExecDestroy(c->g0exec);
  c->g0exec = nullptr;
  c->g0_iters = -1;
}

// coarse start state: tol set from ||b0|| on the device, at most K0 iterations
static int coarse_state(sem_ctx* c) {
  sem::PcgState init{};
  init.maxit = c->coarse_iters;
  CUDA_TRY(cudaMemcpyAsync(c->d_st0, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  SEM_TRY(ensure_hist(c->c0, c->coarse_iters));
  return SEM_OK;
}

// x0 = A0^-1 b0 by <= K0 plain CG steps (reading Q31); no-op when *gate
static int coarse_body(sem_ctx* c, const int* gate) {
  sem_ctx* c0 = c->c0;
  cudaStream_t s = c0->stream;
  if (c->casm_ok && c->coarse_asm != 0) {   // assembled operator on the unique vertices
    if (SEM_COARSE_CLUSTER && c->coarse_asm != 2 && sem::coarse_asm_cluster_ok(c->casm.nu))
      CUDA_TRY(sem::launch_coarse_asm_cluster(c->casm, c->d_b0, c->d_x0, gate, c->coarse_iters,
                                              1e-12, s, &c0->launches));
    else
      CUDA_TRY(sem::launch_coarse_asm_solve(c->casm, c->d_b0, c->d_x0, gate, c->coarse_iters,
                                            1e-12, c->casm_grid, s, &c0->launches));
    return SEM_OK;
  }
  SEM_TRY(gs_op(c0, c->d_b0, 1));
  if (c0->hp.fully_periodic) {   // b0 in range(A0): remove the unique-DOF mean
    CUDA_TRY(sem::launch_sum_c(c0->dp, c0->d_mult, c->d_b0, c0->d_partial, &c0->d_tickets[0],
                               c0->d_scal, c0->red_grid, s));
    SEM_TRY(allreduce(c0, c0->d_scal, 2));
    CUDA_TRY(sem::launch_sub_scalar(c->d_b0, c0->d_scal, c0->hp.n_local, s));
    c0->launches += 2;
  }
  CUDA_TRY(cudaMemcpyAsync(c0->d_st, c->d_st0, sizeof(sem::PcgState), cudaMemcpyDeviceToDevice, s));
  PcgCtl k;
  SEM_TRY(pcg_enqueue_init(c0, c->d_dinv0, c->d_b0, c->d_x0, &k));
  CUDA_TRY(sem::launch_rel_tol(c0->d_st, 1e-12, s));
  CUDA_TRY(sem::launch_gate_state(c0->d_st, gate, s));
  c0->launches += 2;
  for (int q = 0; q < c->coarse_iters; q++) SEM_TRY(pcg_enqueue_iter(c0, c->d_dinv0, c->d_x0, k));
  return SEM_OK;
}

static bool coarse_is_one_kernel(const sem_ctx* c) {
  return SEM_COARSE_CLUSTER && c->casm_ok && c->coarse_asm != 0 && c->coarse_asm != 2 &&
         sem::coarse_asm_cluster_ok(c->casm.nu);
}

static int coarse_solve(sem_ctx* c, const int* gate) {
  // (inside the captured Schwarz batch the coarse kernels are captured inline; a
  // coarse solve that is a single cluster kernel needs no graph of its own)
  if (c->c0->hp.nranks > 1 || !c->coarse_graph || c->timing || c->sw_capturing ||
      coarse_is_one_kernel(c))
    return coarse_body(c, gate);
  cudaStream_t s = c->stream;
  if (!c->g0exec || c->g0_iters != c->coarse_iters) {
    if (c->g0exec) cudaGraphExecDestroy(c->g0exec);
    c->g0exec = nullptr;
    if (!c->d_gate) SEM_TRY(dalloc(&c->d_gate, 1));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (!c->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    const int64_t l0 = c->launches + c->c0->launches;
    cudaGraph_t graph = nullptr;
    // capture on a private stream (the context stream may be the legacy one)
    cudaStream_t s_save = c->stream, s0_save = c->c0->stream;
    c->stream = c->c0->stream = c->cap_stream;
    if (cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      c->stream = s_save;
      c->c0->stream = s0_save;
      c->coarse_graph = false;
      return coarse_body(c, gate);
    }
    const int st = coarse_body(c, c->d_gate);
    const cudaError_t ec = cudaStreamEndCapture(c->cap_stream, &graph);
    c->stream = s_save;
    c->c0->stream = s0_save;
    if (st != SEM_OK || ec != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      c->coarse_graph = false;   // fall back to stream launches
      return coarse_body(c, gate);
    }
    const cudaError_t ei = cudaGraphInstantiate(&c->g0exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
      cudaGetLastError();
      c->g0exec = nullptr;
      c->coarse_graph = false;
      return coarse_body(c, gate);
    }
    c->g0_launches = c->launches + c->c0->launches - l0;
    c->g0_iters = c->coarse_iters;
  }
  CUDA_TRY(sem::launch_copy_gate(c->d_gate, gate, s));
  CUDA_TRY(cudaGraphLaunch(c->g0exec, s));
  c->launches += 1 + c->g0_launches;
  return SEM_OK;
}

// z = M r (which: 1 local, 2 coarse, 3 both); dots (flexible PCG): <z, r>_c and
// <z, w>_c into st->dz; every kernel is a no-op when *gate
static int schwarz_apply(sem_ctx* c, const double* r, double* z, int which, const int* gate,
                         const double* w_dot) {
  const sem::HostPlan& h = c->hp;
  cudaStream_t s = c->stream;
  double* y = (which & 1) ? c->d_sy : nullptr;
  // replicated coarse level: this rank's elements are the block at e_lo
  const int64_t off0 = c->c0_repl ? h.e_lo * 8 : 0;
  double* b0 = (which & 2) ? c->d_b0 + off0 : nullptr;
  int tk = timer_begin(c, 7);
  CUDA_TRY(sem::launch_fdm(h.n, (int)h.nloc, r, c->d_mult, c->d_fS, c->d_flam, c->d_xi, y, b0,
                           gate, c->num_sms, c->fdm_tc, s));
  timer_end(c, tk);
  c->launches++;
  if (y) SEM_TRY(gs_op(c, y, 0));
  if (b0) {
    if (c->c0_repl)   // in place: every rank's restricted block -> the whole b0
      SEM_TRY(coll_allgather(c, b0, c->d_b0, (size_t)h.nloc * 8, s));
    SEM_TRY(coarse_solve(c, gate));
  }
  sem::PcgState* st = c->d_st;
  const bool dist = h.nranks > 1;
  double* dots = w_dot ? (dist ? st->loc_dz : st->dz) : nullptr;
  tk = timer_begin(c, 8);
  CUDA_TRY(sem::launch_schwarz_combine(h.n, (int)h.nloc, y, b0 ? c->d_x0 + off0 : nullptr, c->d_mult,
                                       c->d_xi, z, r, w_dot, c->d_partial, &c->d_tickets[5], dots,
                                       gate, c->num_sms, s));
  timer_end(c, tk);
  c->launches++;
  if (dots && dist) SEM_TRY(allreduce_to(c, st->loc_dz, st->dz, 2));
  return SEM_OK;
}

// flexible PCG with the Schwarz preconditioner (reading Q32); scalars stay on
// the device, the host polls every kBatch iterations
// One rank, flat gather-scatter schedule: the kernels of kBatch flexible-PCG
// iterations (operator, gs, scalar and vector kernels, the preconditioner with
// its coarse solve inlined) have fixed arguments, so the batch is captured once
// and replayed (SEM_OPT_SCHWARZ_GRAPH); keyed by x and the preconditioner's
// configuration.  nullptr: plain stream launches.
template <class F>
static cudaGraphExec_t schwarz_batch_graph(sem_ctx* c, double* x, F& iteration) {
  if (!c->sw_graph || c->hp.nranks > 1 || c->timing || !sem::gs_flat(c->dp, c->gs_mode) ||
      !c->c0 || c->c0->hp.nranks > 1 || !sem::gs_flat(c->c0->dp, c->c0->gs_mode))
    return nullptr;
  const double key[6] = {(double)(uintptr_t)x, (double)(uintptr_t)c->c0, (double)c->coarse_iters,
                         c->fdm_tc ? 1.0 : 0.0, (c->casm_ok && c->coarse_asm != 0) ? 1.0 : 0.0,
                         (double)(uintptr_t)c->d_b0};
  if (c->sw_exec && std::memcmp(key, c->sw_key, sizeof(key)) == 0) return c->sw_exec;
  if (c->sw_exec) cudaGraphExecDestroy(c->sw_exec);
  c->sw_exec = nullptr;
  if (!c->cap_stream && cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  cudaStream_t s_save = c->stream, s0_save = c->c0->stream;
  c->stream = c->c0->stream = c->cap_stream;
  c->sw_capturing = true;
  const int64_t l_c = c->launches, l_c0 = c->c0->launches;
  cudaGraph_t graph = nullptr;
  int st = SEM_OK;
  if (cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    for (int q = 0; q < kBatch && st == SEM_OK; q++) st = iteration();
    if (cudaStreamEndCapture(c->cap_stream, &graph) != cudaSuccess) st = SEM_ECUDA;
  } else {
    st = SEM_ECUDA;
  }
  c->sw_capturing = false;
  c->stream = s_save;
  c->c0->stream = s0_save;
  // kernels per replay (the coarse context's counted into this one's); the
  // capture itself launched nothing
  c->sw_launches = (c->launches - l_c) + (c->c0->launches - l_c0);
  c->launches = l_c;
  c->c0->launches = l_c0;
  cudaGraphExec_t ge = nullptr;
  if (st == SEM_OK && graph && cudaGraphInstantiate(&ge, graph, 0) != cudaSuccess) ge = nullptr;
  if (graph) cudaGraphDestroy(graph);
  cudaGetLastError();
  if (!ge) {
    c->sw_graph = false;   // not capturable here: stream launches from now on
    return nullptr;
  }
  c->sw_exec = ge;
  std::memcpy(c->sw_key, key, sizeof(key));
  return ge;
}

static int schwarz_pcg_run(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                           sem_pcg_result* res) {
  if (maxit < 0 || !(tol >= 0.0)) { sem::set_error("bad tol/maxit"); return SEM_EINVAL; }
  SEM_TRY(ensure_hist(c, maxit));
  const sem::HostPlan& h = c->hp;
  const int64_t n = h.n_local;
  cudaStream_t s = c->stream;
  const int sms = c->num_sms;
  // r and w 16-byte aligned (the vector kernels move point pairs)
  if (!c->d_rw) SEM_TRY(dalloc(&c->d_rw, 2 * (size_t)c->ldv));
  if (!c->d_z) SEM_TRY(dalloc(&c->d_z, (size_t)n));
  double *r = c->d_rw, *w = c->d_rw + c->ldv, *z = c->d_z, *p = c->d_p;
  sem::PcgState* st = c->d_st;
  const int* done = &st->done;
  const bool dist = h.nranks > 1;
  double* part = c->d_partial;
  unsigned* tk = &c->d_tickets[6];
  sem::PcgState init{};
  init.tol = tol;
  init.maxit = maxit;
  std::memcpy(c->h_st, &init, sizeof(init));
  CUDA_TRY(cudaMemcpyAsync(st, c->h_st, sizeof(init), cudaMemcpyHostToDevice, s));
  SEM_TRY(coarse_state(c));
  CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  CUDA_TRY(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(cudaMemsetAsync(w, 0, sizeof(double) * n, s));
  // z = M r, p = z, rho = <r, z>_c, gamma = <r, r>_c
  SEM_TRY(schwarz_apply(c, r, z, 3, nullptr, w));
  CUDA_TRY(cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(sem::launch_mdot(n, c->d_mult, r, r, n, 1, part, tk, dist ? &st->loc[1] : &st->gamma,
                            nullptr, sms, s));
  if (dist) SEM_TRY(allreduce_to(c, &st->loc[1], &st->gamma, 1));
  CUDA_TRY(cudaMemcpyAsync(&st->rho_new, &st->dz[0], sizeof(double), cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(sem::launch_fcg_scalar(0, st, c->d_hist, s));
  c->launches += 2;
  int hd = 0;
  auto iteration = [&]() -> int {
      cudaStream_t s = c->stream;   // (the capture stream while a batch is captured)
      if (!dist) {
        // w = A p with sigma = sum_l p_l (A_L p)_l reduced by the Ax kernel itself
        // (reading Q23: equals <p, w>_c for the continuous, masked p)
        GateScope g(c, done);
        SEM_TRY(run_ax(c, p, w, sem::AX_PCG, 0, (int)h.nloc, 0, 0, &st->sigma));
        SEM_TRY(gs_pass(c, w));
      } else {
        {
          GateScope g(c, done);
          SEM_TRY(apply_op(c, p, w, sem::AX_APPLY));   // w = A p
        }
        CUDA_TRY(sem::launch_mdot(n, c->d_mult, p, w, n, 1, part, tk,
                                  dist ? &st->loc[2] : &st->sigma, done, sms, s));
        if (dist) SEM_TRY(allreduce_to(c, &st->loc[2], &st->sigma, 1));
      }
      CUDA_TRY(sem::launch_fcg_scalar(1, st, c->d_hist, s));       // alpha
      CUDA_TRY(sem::launch_maxpy(n, x, p, n, 1, &st->alpha, 1.0, nullptr, c->d_mult, part, tk,
                                 nullptr, done, sms, s));           // x += alpha p
      CUDA_TRY(sem::launch_maxpy(n, r, w, n, 1, &st->alpha, -1.0, nullptr, c->d_mult, part, tk,
                                 dist ? &st->loc[1] : &st->gamma, done, sms, s));   // r -= alpha w
      if (dist) SEM_TRY(allreduce_to(c, &st->loc[1], &st->gamma, 1));
      CUDA_TRY(sem::launch_fcg_scalar(2, st, c->d_hist, s));       // convergence
      SEM_TRY(schwarz_apply(c, r, z, 3, done, w));                  // z = M r, dots
      CUDA_TRY(sem::launch_fcg_scalar(3, st, c->d_hist, s));       // beta
      CUDA_TRY(sem::launch_xpay(n, p, z, st, sms, s));              // p = z + beta p
      c->launches += 7;
      return SEM_OK;
  };
  for (int it = 0; it < maxit && !hd; it += kBatch) {
    const int nb = std::min(kBatch, maxit - it);
    cudaGraphExec_t ge = nb == kBatch ? schwarz_batch_graph(c, x, iteration) : nullptr;
    if (ge) {
      CUDA_TRY(cudaGraphLaunch(ge, s));
      c->launches += c->sw_launches;
    } else {
      for (int q = 0; q < nb; q++) SEM_TRY(iteration());
    }
    CUDA_TRY(cudaMemcpyAsync(&c->h_st->done, done, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    hd = c->h_st->done;
  }
  return pcg_finish(c, b, x, res);
}

extern "C" int sem_schwarz_apply(sem_ctx* c, const double* r, double* z, int32_t which) {
  if (!c || !r || !z || r == z || which < 1 || which > 3) {
    sem::set_error("sem_schwarz_apply: bad arguments");
    return SEM_EINVAL;
  }
  SEM_TRY(schwarz_setup(c));
  SEM_TRY(coarse_state(c));
  return schwarz_apply(c, r, z, which, nullptr, nullptr);
}

// the preconditioner selected by SEM_OPT_PRECOND (sem_pcg_solve and sem_pcg_solve_host)
static int pcg_dispatch(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                        sem_pcg_result* res) {
  if (c->precond == SEM_PRECOND_SCHWARZ) {
    SEM_TRY(schwarz_setup(c));
    return schwarz_pcg_run(c, b, x, tol, maxit, res);
  }
  return pcg_run(c, b, x, tol, maxit, res);
}

extern "C" int sem_pcg_solve(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                             sem_pcg_result* res) {
  if (!c || !b || !x || !aligned16(b) || !aligned16(x) || b == x) {
    sem::set_error("sem_pcg_solve: bad arguments");
    return SEM_EINVAL;
  }
  return pcg_dispatch(c, b, x, tol, maxit, res);
}

// ---------------------------------------------------------------- NEXT-2: Helmholtz
// h1 A + h2 B (P:L257 velocity solves); the context switches to
// the Helmholtz operator for the duration of one call
struct HelmScope {
  sem_ctx* c;
  HelmScope(sem_ctx* ctx, double h1, double h2) : c(ctx) {
    c->helm = true;
    c->h1 = h1;
    c->h2 = h2;
  }
  ~HelmScope() {
    c->helm = false;
    c->h1 = 1.0;
    c->h2 = 0.0;
  }
};

extern "C" int sem_helm_apply(sem_ctx* c, double h1, double h2, const double* u, double* w) {
  if (!c || !u || !w || !aligned16(u) || !aligned16(w) || u == w) {
    sem::set_error("sem_helm_apply: bad arguments (NULL, misaligned or aliased pointers)");
    return SEM_EINVAL;
  }
  HelmScope hs(c, h1, h2);
  return apply_op(c, u, w, sem::AX_APPLY);
}

extern "C" int sem_rhs_mass(sem_ctx* c, const double* f, double* b) {
  if (!c || !f || !b) { sem::set_error("sem_rhs_mass: NULL argument"); return SEM_EINVAL; }
  CUDA_TRY(sem::launch_scale_mask(c->dp, c->d_B, f, b, c->stream));
  c->launches++;
  return gs_op(c, b, 1);
}

// Jacobi of h1 A + h2 B: dinv = mask ? 0 : 1 / QQ^T(h1 diag(A_L) + h2 B_L), cached per (h1, h2)
static int helm_jacobi(sem_ctx* c, double h1, double h2) {
  if (c->d_dinv_helm && c->helm_key[0] == h1 && c->helm_key[1] == h2) return SEM_OK;
  if (!c->d_dinv_helm) SEM_TRY(dalloc(&c->d_dinv_helm, (size_t)c->hp.n_local));
  CUDA_TRY(sem::launch_diag(c->dp, c->d_G, c->d_dinv_helm, c->stream));
  CUDA_TRY(sem::launch_helm_diag(c->d_dinv_helm, c->d_B, h1, h2, c->hp.n_local, c->stream));
  SEM_TRY(gs_op(c, c->d_dinv_helm, 0));
  CUDA_TRY(sem::launch_invert_mask(c->dp, c->d_dinv_helm, c->stream));
  c->launches += 3;
  c->helm_key[0] = h1;
  c->helm_key[1] = h2;
  return SEM_OK;
}

extern "C" int sem_helm_pcg_solve(sem_ctx* c, double h1, double h2, const double* b, double* x,
                                  double tol, int32_t maxit, sem_pcg_result* res) {
  if (!c || !b || !x || !aligned16(b) || !aligned16(x) || b == x) {
    sem::set_error("sem_helm_pcg_solve: bad arguments");
    return SEM_EINVAL;
  }
  if (!(h1 >= 0.0) || !(h2 >= 0.0) || (h1 == 0.0 && h2 == 0.0)) {
    sem::set_error("sem_helm_pcg_solve: need h1 >= 0, h2 >= 0, not both 0");
    return SEM_EINVAL;
  }
  SEM_TRY(helm_jacobi(c, h1, h2));
  HelmScope hs(c, h1, h2);
  return pcg_run(c, b, x, tol, maxit, res);
}

// ---------------------------------------------------------------- NEXT-3: GMRES, projection
// restarted GMRES(m) with right Jacobi preconditioning (readings Q25, Q26);
// device-resident: the host enqueues 8 Arnoldi steps per poll
static int gm_alloc(sem_ctx* c, int m) {
  if (m < 1 || m >= sem::kGmMax) {
    sem::set_error("restart must be in [1, 31]");
    return SEM_EINVAL;
  }
  const size_t n = (size_t)c->hp.n_local;
  if (!c->d_gs) {
    SEM_TRY(dalloc(&c->d_gs, 1));
    SEM_TRY(dalloc(&c->d_ktick, 4));
    CUDA_TRY(cudaMemsetAsync(c->d_ktick, 0, 4 * sizeof(unsigned), c->stream));
    SEM_TRY(dalloc(&c->d_kpart, (size_t)4 * c->num_sms * sem::kGmMax));
    SEM_TRY(dalloc(&c->d_gt, n));
    sem::GmresState init{};
    init.one = 1.0;
    CUDA_TRY(cudaMemcpyAsync(c->d_gs, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  if (m + 1 > c->gm_cap) {
    if (c->d_V) cudaFree(c->d_V);
    c->d_V = nullptr;
    SEM_TRY(dalloc(&c->d_V, (m + 1) * (size_t)c->ldv));
    // finite contents: unused basis vectors are multiplied by zero coefficients
    CUDA_TRY(cudaMemsetAsync(c->d_V, 0, (m + 1) * (size_t)c->ldv * sizeof(double), c->stream));
    c->gm_cap = m + 1;
  }
  return SEM_OK;
}


// One rank, flat gather-scatter schedules: a GMRES restart cycle (restart
// residual, m Arnoldi steps with their preconditioner applications, the
// least-squares update) has fixed kernel arguments, so it is captured once
// (keyed by x, b, m and the preconditioner's configuration) and replayed per
// cycle (SEM_OPT_GMRES_GRAPH); the steps after convergence are the same no-ops
// as in stream mode.  nullptr: stream launches.
template <class F>
static cudaGraphExec_t gmres_cycle_graph(sem_ctx* c, double* x, const double* b, int m, bool schw,
                                         F& cycle) {
  if (!c->gm_graph || c->hp.nranks > 1 || c->timing || !sem::gs_flat(c->dp, c->gs_mode))
    return nullptr;
  if (schw && (!c->c0 || c->c0->hp.nranks > 1 || !sem::gs_flat(c->c0->dp, c->c0->gs_mode)))
    return nullptr;
  const double key[10] = {(double)(uintptr_t)x, (double)(uintptr_t)b, (double)m, schw ? 1.0 : 0.0,
                          (double)(uintptr_t)c->d_V, (double)(uintptr_t)c->d_Zs,
                          (double)(uintptr_t)c->c0, (double)c->coarse_iters,
                          (c->fdm_tc ? 1.0 : 0.0) + ((c->casm_ok && c->coarse_asm != 0) ? 2.0 : 0.0) +
                              (c->helm ? 4.0 : 0.0),
                          c->helm ? c->h1 * 1e3 + c->h2 : 0.0};
  if (c->gm_exec && std::memcmp(key, c->gm_key, sizeof(key)) == 0) return c->gm_exec;
  if (c->gm_exec) cudaGraphExecDestroy(c->gm_exec);
  c->gm_exec = nullptr;
  if (!c->cap_stream && cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  cudaStream_t s_save = c->stream, s0_save = c->c0 ? c->c0->stream : nullptr;
  c->stream = c->cap_stream;
  if (c->c0) c->c0->stream = c->cap_stream;
  c->sw_capturing = true;
  const int64_t l_c = c->launches, l_c0 = c->c0 ? c->c0->launches : 0;
  cudaGraph_t graph = nullptr;
  int st = SEM_OK;
  if (cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    st = cycle(false);
    if (cudaStreamEndCapture(c->cap_stream, &graph) != cudaSuccess) st = SEM_ECUDA;
  } else {
    st = SEM_ECUDA;
  }
  c->sw_capturing = false;
  c->stream = s_save;
  if (c->c0) c->c0->stream = s0_save;
  c->gm_launches = (c->launches - l_c) + (c->c0 ? c->c0->launches - l_c0 : 0);
  c->launches = l_c;
  if (c->c0) c->c0->launches = l_c0;
  cudaGraphExec_t ge = nullptr;
  if (st == SEM_OK && graph && cudaGraphInstantiate(&ge, graph, 0) != cudaSuccess) ge = nullptr;
  if (graph) cudaGraphDestroy(graph);
  cudaGetLastError();
  if (!ge) {
    c->gm_graph = false;   // not capturable here: stream launches from now on
    return nullptr;
  }
  c->gm_exec = ge;
  std::memcpy(c->gm_key, key, sizeof(key));
  return ge;
}

static int gmres_run(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit, int m,
                     sem_pcg_result* res) {
  if (maxit < 0 || !(tol >= 0.0)) { sem::set_error("bad tol/maxit"); return SEM_EINVAL; }
  SEM_TRY(gm_alloc(c, m));
  SEM_TRY(ensure_hist(c, maxit));
  // flexible GMRES with the Schwarz preconditioner (NEXT-1): z_j = M v_j stored
  const bool schw = c->precond == SEM_PRECOND_SCHWARZ && !c->helm;
  const int64_t ld = c->ldv;
  if (schw) {
    SEM_TRY(schwarz_setup(c));
    SEM_TRY(coarse_state(c));
    if (m > c->zs_cap) {
      if (c->d_Zs) cudaFree(c->d_Zs);
      c->d_Zs = nullptr;
      SEM_TRY(dalloc(&c->d_Zs, (size_t)m * c->ldv));
      CUDA_TRY(cudaMemsetAsync(c->d_Zs, 0, (size_t)m * c->ldv * sizeof(double), c->stream));
      c->zs_cap = m;
    }
  }
  cudaStream_t s = c->stream;
  const int64_t n = c->hp.n_local;
  const int sms = c->num_sms;
  sem::PcgState* st = c->d_st;
  sem::GmresState* gs = c->d_gs;
  double* part = c->d_kpart;
  unsigned* tk = c->d_ktick;
  double* w = c->d_wv;
  const double* dinv = c->d_dinv;
  const uint8_t* mult = c->d_mult;
  const bool dist = c->hp.nranks > 1;
  sem::PcgState init{};
  init.tol = tol;
  init.maxit = maxit;
  std::memcpy(c->h_st, &init, sizeof(init));
  CUDA_TRY(cudaMemcpyAsync(st, c->h_st, sizeof(init), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  const int* done = &st->done;
  const int* cyc = &gs->cycle_done;
  int status_done = 0;
  // one restart cycle; poll: stop enqueuing once the cycle has finished (stream
  // launches only; the captured cycle runs all m steps, finished ones no-ops)
  auto cycle = [&](bool poll) -> int {
    cudaStream_t s = c->stream;   // (the capture stream while a cycle is captured)
    // restart: V0 = (b - A x) / ||b - A x||_c, t = dinv V0
    {
      GateScope g(c, done);
      SEM_TRY(apply_op(c, x, w, sem::AX_APPLY));
    }
    CUDA_TRY(sem::launch_resid(n, b, w, c->d_V, mult, part, tk, &gs->norm2[0], done, sms, s));
    if (dist) SEM_TRY(allreduce(c, &gs->norm2[0], 1));
    CUDA_TRY(sem::launch_gm_start(gs, st, c->d_hist, s));
    CUDA_TRY(sem::launch_vnorm(n, c->d_V, c->d_V, schw ? nullptr : c->d_gt, dinv, gs, cyc, sms, s));
    c->launches += 4;
    if (schw) SEM_TRY(schwarz_apply(c, c->d_V, c->d_Zs, 3, cyc, nullptr));
    for (int j = 0; j < m; j++) {
      double* Vn = c->d_V + (size_t)(j + 1) * ld;
      {
        GateScope g(c, cyc);
        SEM_TRY(apply_op(c, schw ? c->d_Zs + (size_t)j * ld : c->d_gt, w,
                         sem::AX_APPLY));   // w = A M^-1 v_j
      }
      // two classical Gram-Schmidt passes against v_0..v_j, then ||w||_c
      CUDA_TRY(sem::launch_mdot(n, mult, w, c->d_V, ld, j + 1, part, tk, gs->h1, cyc, sms, s));
      if (dist) SEM_TRY(allreduce(c, gs->h1, j + 1));
      // second pass fused with the first pass's update: w -= V h1, h2 = V^T w
      CUDA_TRY(sem::launch_maxpy_mdot(n, w, c->d_V, ld, j + 1, gs->h1, mult, part, tk, gs->h2, cyc,
                                      sms, s));
      if (dist) SEM_TRY(allreduce(c, gs->h2, j + 1));
      CUDA_TRY(sem::launch_maxpy(n, w, c->d_V, ld, j + 1, gs->h2, -1.0, nullptr, mult, part, tk,
                                 &gs->norm2[0], cyc, sms, s));
      if (dist) SEM_TRY(allreduce(c, &gs->norm2[0], 1));
      CUDA_TRY(sem::launch_gm_arnoldi(gs, st, c->d_hist, m, s));
      CUDA_TRY(sem::launch_vnorm(n, w, Vn, schw ? nullptr : c->d_gt, dinv, gs, cyc, sms, s));
      c->launches += 6;
      if (schw && j + 1 < m) SEM_TRY(schwarz_apply(c, Vn, c->d_Zs + (size_t)(j + 1) * ld, 3, cyc, nullptr));
      if (poll && (j + 1) % kBatch == 0 && j + 1 < m) {   // stop enqueuing a finished cycle
        int cd = 0;
        CUDA_TRY(cudaMemcpyAsync(&c->h_st->done, &gs->cycle_done, sizeof(int),
                                 cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        cd = c->h_st->done;
        if (cd) break;
      }
    }
    // y = H^-1 g; x += M^-1 V y; converged / maxit -> done
    CUDA_TRY(sem::launch_gm_solve(gs, st, m, s));
    if (schw)   // x += Z y
      CUDA_TRY(sem::launch_maxpy(n, x, c->d_Zs, ld, m, gs->y, 1.0, nullptr, mult, part, tk, nullptr,
                                 done, sms, s));
    else        // x += M^-1 V y
      CUDA_TRY(sem::launch_maxpy(n, x, c->d_V, ld, m, gs->y, 1.0, dinv, mult, part, tk, nullptr,
                                 done, sms, s));
    CUDA_TRY(sem::launch_gm_end_cycle(gs, st, s));
    c->launches += 3;
    return SEM_OK;
  };
  while (!status_done) {
    cudaGraphExec_t ge = gmres_cycle_graph(c, x, b, m, schw, cycle);
    if (ge) {
      CUDA_TRY(cudaGraphLaunch(ge, s));
      c->launches += c->gm_launches;
    } else {
      SEM_TRY(cycle(true));
    }
    CUDA_TRY(cudaMemcpyAsync(&c->h_st->done, &st->done, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    status_done = c->h_st->done;
  }
  // true residual once at the end (reading Q17)
  SEM_TRY(apply_op(c, x, w, sem::AX_APPLY));
  CUDA_TRY(sem::launch_resid(n, b, w, c->d_gt, mult, part, tk, &gs->norm2[1], nullptr, sms, s));
  if (dist) SEM_TRY(allreduce(c, &gs->norm2[1], 1));
  c->launches++;
  sem::GmresState hg;
  CUDA_TRY(cudaMemcpyAsync(&hg, gs, sizeof(hg), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(c->h_st, st, sizeof(sem::PcgState), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  SEM_TRY(p2p_check(c));
  const sem::PcgState& hs = *c->h_st;
  c->last_hist = hs.iters;
  if (res) {
    res->iters = hs.iters;
    res->res_final = hg.res;
    res->res_true = std::sqrt(hg.norm2[1]);
  }
  int status = hs.done == 1 ? SEM_OK : SEM_NOT_CONVERGED;
  if (res) res->status = status;
  return status;
}

extern "C" int sem_gmres_solve(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                               int32_t restart, sem_pcg_result* r) {
  if (!c || !b || !x || !aligned16(b) || !aligned16(x) || b == x) {
    sem::set_error("sem_gmres_solve: bad arguments");
    return SEM_EINVAL;
  }
  return gmres_run(c, b, x, tol, maxit, restart, r);
}

// ---- solution projection (Fischer 1998): Z, AZ [m][n], A-orthonormal
static int proj_alloc(sem_ctx* c, int m) {
  if (m < 1 || m > sem::kGmMax) {
    sem::set_error("projection dimension must be in [1, 32]");
    return SEM_EINVAL;
  }
  SEM_TRY(gm_alloc(c, 1));
  if (m == c->proj_m) return SEM_OK;
  const size_t n = (size_t)c->hp.n_local;
  double* bufs[4] = {c->d_Z, c->d_AZ, c->d_pdelta, c->d_pbd};
  for (double* p : bufs)
    if (p) cudaFree(p);
  c->d_Z = c->d_AZ = c->d_pdelta = c->d_pbd = nullptr;
  SEM_TRY(dalloc(&c->d_Z, m * (size_t)c->ldv));
  SEM_TRY(dalloc(&c->d_AZ, m * (size_t)c->ldv));
  SEM_TRY(dalloc(&c->d_pdelta, n));
  SEM_TRY(dalloc(&c->d_pbd, n));
  c->proj_m = m;
  c->proj_k = 0;
  return SEM_OK;
}

// append x to the space (two CGS passes in the A inner product); returns 1 if skipped
static int proj_update(sem_ctx* c, const double* x, int* skipped) {
  cudaStream_t s = c->stream;
  const int64_t n = c->hp.n_local;
  const int sms = c->num_sms;
  const bool dist = c->hp.nranks > 1;
  sem::GmresState* gs = c->d_gs;
  if (c->proj_k == c->proj_m) c->proj_k = 0;   // full: reset, keep the latest
  const int k = c->proj_k;
  double* z = c->d_Z + (size_t)k * c->ldv;
  double* az = c->d_AZ + (size_t)k * c->ldv;
  CUDA_TRY(cudaMemcpyAsync(z, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  SEM_TRY(apply_op(c, z, az, sem::AX_APPLY));
  CUDA_TRY(sem::launch_mdot(n, c->d_mult, z, az, n, 1, c->d_kpart, c->d_ktick, &gs->norm2[0],
                            nullptr, sms, s));
  if (dist) SEM_TRY(allreduce(c, &gs->norm2[0], 1));
  for (int pass = 0; pass < 2 && k > 0; pass++) {
    double* coef = pass == 0 ? gs->h1 : gs->h2;
    CUDA_TRY(sem::launch_mdot(n, c->d_mult, az, c->d_Z, c->ldv, k, c->d_kpart, c->d_ktick, coef,
                              nullptr, sms, s));
    if (dist) SEM_TRY(allreduce(c, coef, k));
    CUDA_TRY(sem::launch_maxpy(n, z, c->d_Z, c->ldv, k, coef, -1.0, nullptr, c->d_mult, c->d_kpart,
                               c->d_ktick, nullptr, nullptr, sms, s));
    CUDA_TRY(sem::launch_maxpy(n, az, c->d_AZ, c->ldv, k, coef, -1.0, nullptr, c->d_mult, c->d_kpart,
                               c->d_ktick, nullptr, nullptr, sms, s));
    c->launches += 3;
  }
  CUDA_TRY(sem::launch_mdot(n, c->d_mult, z, az, n, 1, c->d_kpart, c->d_ktick, &gs->norm2[1],
                            nullptr, sms, s));
  if (dist) SEM_TRY(allreduce(c, &gs->norm2[1], 1));
  double nrm[2];
  CUDA_TRY(cudaMemcpyAsync(nrm, &gs->norm2[0], sizeof(nrm), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  c->launches += 2;
  const double nx = std::sqrt(std::fabs(nrm[0])), nz = std::sqrt(std::fabs(nrm[1]));
  if (!(nz > 1e-12 * nx)) {
    *skipped = 1;
    return SEM_OK;
  }
  // z, az /= ||z||_A  (scale: y += (1/nz - 1) y via maxpy on itself would alias; use vnorm)
  sem::GmresState* g = c->d_gs;
  const double inv = 1.0 / nz;
  CUDA_TRY(cudaMemcpyAsync(&g->inv_norm, &inv, sizeof(double), cudaMemcpyHostToDevice, s));
  CUDA_TRY(sem::launch_vnorm(n, z, z, nullptr, nullptr, g, nullptr, sms, s));
  CUDA_TRY(sem::launch_vnorm(n, az, az, nullptr, nullptr, g, nullptr, sms, s));
  c->launches += 2;
  c->proj_k = k + 1;
  *skipped = 0;
  return SEM_OK;
}

extern "C" int sem_proj_solve(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                              int32_t restart, int32_t m, sem_pcg_result* r) {
  if (!c || !b || !x || !aligned16(b) || !aligned16(x) || b == x) {
    sem::set_error("sem_proj_solve: bad arguments");
    return SEM_EINVAL;
  }
  SEM_TRY(proj_alloc(c, m));
  cudaStream_t s = c->stream;
  const int64_t n = c->hp.n_local;
  const int sms = c->num_sms;
  sem::GmresState* gs = c->d_gs;
  const int k = c->proj_k;
  // x_bar = sum <z_i, b>_c z_i ; b_defl = b - sum <z_i, b>_c A z_i
  CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  CUDA_TRY(cudaMemcpyAsync(c->d_pbd, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  if (k > 0) {
    CUDA_TRY(sem::launch_mdot(n, c->d_mult, b, c->d_Z, c->ldv, k, c->d_kpart, c->d_ktick, gs->y,
                              nullptr, sms, s));
    if (c->hp.nranks > 1) SEM_TRY(allreduce(c, gs->y, k));
    CUDA_TRY(sem::launch_maxpy(n, x, c->d_Z, c->ldv, k, gs->y, 1.0, nullptr, c->d_mult, c->d_kpart,
                               c->d_ktick, nullptr, nullptr, sms, s));
    CUDA_TRY(sem::launch_maxpy(n, c->d_pbd, c->d_AZ, c->ldv, k, gs->y, -1.0, nullptr, c->d_mult,
                               c->d_kpart, c->d_ktick, nullptr, nullptr, sms, s));
    c->launches += 3;
  }
  // delta: GMRES on the deflated right-hand side from 0; x = x_bar + delta
  const int st = gmres_run(c, c->d_pbd, c->d_pdelta, tol, maxit, restart, r);
  if (st < 0) return st;
  CUDA_TRY(sem::launch_maxpy(n, x, c->d_pdelta, n, 1, &gs->one, 1.0, nullptr, c->d_mult,
                             c->d_kpart, c->d_ktick, nullptr, nullptr, sms, s));
  c->launches++;
  int skipped = 0;
  SEM_TRY(proj_update(c, x, &skipped));
  return st;
}

extern "C" int sem_proj_reset(sem_ctx* c) {
  if (!c) return SEM_EINVAL;
  c->proj_k = 0;
  return SEM_OK;
}

extern "C" int sem_proj_size(const sem_ctx* c, int32_t* k) {
  if (!c || !k) return SEM_EINVAL;
  *k = c->proj_k;
  return SEM_OK;
}

extern "C" int sem_pcg_solve_host(sem_ctx* c, const double* b_host, double* x_host, double tol,
                                  int32_t maxit, sem_pcg_result* res) {
  if (!c || !b_host || !x_host) { sem::set_error("sem_pcg_solve_host: NULL argument"); return SEM_EINVAL; }
  const size_t bytes = (size_t)c->hp.n_local * sizeof(double);
  if (!c->d_tmp) SEM_TRY(dalloc(&c->d_tmp, 2 * (size_t)c->ldv));
  double* db = c->d_tmp;
  double* dx = c->d_tmp + c->ldv;   // 16-byte aligned
  CUDA_TRY(cudaMemcpyAsync(db, b_host, bytes, cudaMemcpyHostToDevice, c->stream));
  int st = pcg_dispatch(c, db, dx, tol, maxit, res);
  if (st < 0) return st;
  CUDA_TRY(cudaMemcpyAsync(x_host, dx, bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return st;
}

extern "C" int sem_pcg_history(const sem_ctx* c, double* host_dst, int32_t max_entries, int32_t* n) {
  if (!c || !host_dst) return SEM_EINVAL;
  int cnt = std::min(max_entries, c->last_hist + 1);
  if (cnt > 0)
    CUDA_TRY(cudaMemcpy(host_dst, c->d_hist, (size_t)cnt * sizeof(double), cudaMemcpyDeviceToHost));
  if (n) *n = cnt;
  return SEM_OK;
}

extern "C" int sem_export_field(const sem_ctx* c, int which, double* host_dst) {
  if (!c || !host_dst) return SEM_EINVAL;
  const sem::HostPlan& h = c->hp;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  switch (which) {
    case 0: std::memcpy(host_dst, h.xi.data(), h.xi.size() * sizeof(double)); return SEM_OK;
    case 1: std::memcpy(host_dst, h.w.data(), h.w.size() * sizeof(double)); return SEM_OK;
    case 2: std::memcpy(host_dst, h.D.data(), h.D.size() * sizeof(double)); return SEM_OK;
    case 3: {  // export in the factor-major [E][6][n^3] order
      std::vector<double> tmp(6 * (size_t)h.n_local);
      CUDA_TRY(cudaMemcpy(tmp.data(), c->d_G, tmp.size() * 8, cudaMemcpyDeviceToHost));
      const int n = h.n;
      const int64_t n3 = h.n3;
      for (int64_t el = 0; el < h.nloc; el++)
        for (int f = 0; f < 6; f++)
          for (int64_t p = 0; p < n3; p++)
            host_dst[el * 6 * n3 + f * n3 + p] = tmp[sem::g_index_host(el, f, (int)p, n)];
      return SEM_OK;
    }
    case 4: CUDA_TRY(cudaMemcpy(host_dst, c->d_B, (size_t)h.n_local * 8, cudaMemcpyDeviceToHost)); return SEM_OK;
    case 5: CUDA_TRY(cudaMemcpy(host_dst, c->d_dinv, (size_t)h.n_local * 8, cudaMemcpyDeviceToHost)); return SEM_OK;
  }
  sem::set_error("sem_export_field: unknown field");
  return SEM_EINVAL;
}

extern "C" int sem_export_int(const sem_ctx* c, int which, int64_t* host_dst) {
  if (!c || !host_dst) return SEM_EINVAL;
  const size_t nl = (size_t)c->hp.n_local;
  std::vector<uint8_t> tmp(nl);
  if (which == 0) {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaMemcpy(tmp.data(), c->d_mult, nl, cudaMemcpyDeviceToHost));
  } else if (which == 1) {
    uint8_t* d = nullptr;
    SEM_TRY(dalloc(&d, nl));
    CUDA_TRY(sem::launch_export_mask(c->dp, d, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaMemcpy(tmp.data(), d, nl, cudaMemcpyDeviceToHost));
    cudaFree(d);
  } else {
    sem::set_error("sem_export_int: unknown field");
    return SEM_EINVAL;
  }
  for (size_t l = 0; l < nl; l++) host_dst[l] = tmp[l];
  return SEM_OK;
}

// live plan export: the gather-scatter records the kernels use, read back from
// the device into a planner handle (its pairs / segments / shared lists are
// expanded from these records; multiplicity and mask from the device arrays)
extern "C" int sem_export_plan(const sem_ctx* c, sem_plan** out) {
  if (!c || !out) { sem::set_error("sem_export_plan: NULL argument"); return SEM_EINVAL; }
  *out = nullptr;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  sem::HostPlan p = c->hp;
  auto get = [](auto& v, const auto* d) -> cudaError_t {
    if (v.empty()) return cudaSuccess;
    return cudaMemcpy(v.data(), d, v.size() * sizeof(v[0]), cudaMemcpyDeviceToHost);
  };
  // overwrite every record with the device copy (sizes from the host plan)
  std::fill(p.f_base.begin(), p.f_base.end(), -7);
  std::fill(p.e_base.begin(), p.e_base.end(), -7);
  std::fill(p.v_base.begin(), p.v_base.end(), -7);
  std::fill(p.s_slot.begin(), p.s_slot.end(), -7);
  CUDA_TRY(get(p.f_base, c->d_fb));
  CUDA_TRY(get(p.f_axis, c->d_fax));
  CUDA_TRY(get(p.e_base, c->d_eb));
  CUDA_TRY(get(p.e_axis, c->d_eax));
  CUDA_TRY(get(p.e_nin, c->d_enin));
  CUDA_TRY(get(p.e_mask, c->d_emask));
  CUDA_TRY(get(p.v_base, c->d_vb));
  CUDA_TRY(get(p.v_nin, c->d_vnin));
  CUDA_TRY(get(p.v_mask, c->d_vmask));
  CUDA_TRY(get(p.s_slot, c->d_sslot));
  CUDA_TRY(get(p.s_off, c->d_soff));
  CUDA_TRY(get(p.s_nloc, c->d_snloc));
  CUDA_TRY(get(p.s_nr, c->d_snr));
  CUDA_TRY(get(p.s_mult, c->d_smult));
  const size_t nl = (size_t)p.n_local;
  std::vector<uint8_t> mult(nl), mask(nl);
  CUDA_TRY(cudaMemcpy(mult.data(), c->d_mult, nl, cudaMemcpyDeviceToHost));
  uint8_t* d = nullptr;
  SEM_TRY(dalloc(&d, nl));
  CUDA_TRY(sem::launch_export_mask(c->dp, d, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaMemcpy(mask.data(), d, nl, cudaMemcpyDeviceToHost));
  cudaFree(d);
  p.x_mult.assign(mult.begin(), mult.end());
  p.x_mask.assign(mask.begin(), mask.end());
  *out = sem::plan_wrap(p);
  return *out ? SEM_OK : SEM_ENOMEM;
}

extern "C" int sem_nccl_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  NCCL_TRY(ncclGetUniqueId(&u));
  std::memcpy(id, &u, 128);
  return SEM_OK;
}

extern "C" int sem_nccl_comm_init(const uint8_t id[128], int rank, int nranks, void** comm) {
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t cm;
  NCCL_TRY(ncclCommInitRank(&cm, nranks, u, rank));
  *comm = cm;
  return SEM_OK;
}

extern "C" int sem_nccl_comm_destroy(void* comm) {
  if (comm) NCCL_TRY(ncclCommDestroy(static_cast<ncclComm_t>(comm)));
  return SEM_OK;
}

extern "C" int sem_timing(sem_ctx* c, int enable) {
  if (!c) return SEM_EINVAL;
  timer_collect(c);
  c->timing = enable != 0;
  for (int q = 0; q < kTimerClasses; q++) { c->t_ms[q] = 0.0; c->t_cnt[q] = 0; }
  return SEM_OK;
}

extern "C" int sem_timing_read(sem_ctx* c, int which, double* total_ms, int64_t* count) {
  if (!c || which < 0 || which >= kTimerClasses) return SEM_EINVAL;
  timer_collect(c);
  if (total_ms) *total_ms = c->t_ms[which];
  if (count) *count = c->t_cnt[which];
  return SEM_OK;
}

extern "C" int sem_set_option(sem_ctx* c, int option, int value) {
  if (!c) return SEM_EINVAL;
  if (option == 1 || option == 5 || option == 10) {
    // SEM_OPT_FUSED_GS (1), SEM_OPT_PDL (5), SEM_OPT_GS_UPDATE (10): variants
    // measured slower than the default path in round 1 and removed
    sem::set_error("sem_set_option: option removed (measured slower variant)");
    return SEM_EINVAL;
  }
  if (option == SEM_OPT_OVERLAP) {   // collective
    cudaStreamSynchronize(c->stream);
    c->overlap = value != 0;
    return SEM_OK;
  }
  if (option == SEM_OPT_GS_MODE) {
    if (value < 0 || value > 2) {
      sem::set_error("sem_set_option: SEM_OPT_GS_MODE must be 0, 1 or 2");
      return SEM_EINVAL;
    }
    c->gs_mode = value;
    return SEM_OK;
  }
  if (option == SEM_OPT_P2P) {   // collective: every rank must set the same value
    cudaStreamSynchronize(c->stream);
    c->use_p2p = value != 0;
    return SEM_OK;
  }
  if (option == SEM_OPT_PRECOND) {   // collective for nranks > 1 (builds Schwarz)
    if (value != SEM_PRECOND_JACOBI && value != SEM_PRECOND_SCHWARZ) {
      sem::set_error("sem_set_option: SEM_OPT_PRECOND must be 0 (Jacobi) or 1 (Schwarz)");
      return SEM_EINVAL;
    }
    cudaStreamSynchronize(c->stream);
    if (value == SEM_PRECOND_SCHWARZ) SEM_TRY(schwarz_setup(c));
    c->precond = value;
    return SEM_OK;
  }
  if (option == SEM_OPT_PCG_FUSE) {
    cudaStreamSynchronize(c->stream);
    c->pcg_fuse = value != 0;
    if (c->pg_exec) cudaGraphExecDestroy(c->pg_exec);
    c->pg_exec = nullptr;
    return SEM_OK;
  }
  if (option == SEM_OPT_GMRES_GRAPH) {
    cudaStreamSynchronize(c->stream);
    c->gm_graph = value != 0;
    if (c->gm_exec) cudaGraphExecDestroy(c->gm_exec);
    c->gm_exec = nullptr;
    return SEM_OK;
  }
  if (option == SEM_OPT_SCHWARZ_GRAPH) {
    cudaStreamSynchronize(c->stream);
    c->sw_graph = value != 0;
    if (c->sw_exec) cudaGraphExecDestroy(c->sw_exec);
    c->sw_exec = nullptr;
    return SEM_OK;
  }
  if (option == SEM_OPT_PCG_GSU) {
    cudaStreamSynchronize(c->stream);
    if (value < -1 || value > 1) {
      sem::set_error("sem_set_option: SEM_OPT_PCG_GSU must be -1 (auto), 0 or 1");
      return SEM_EINVAL;
    }
    c->pcg_gsu = value;
    if (c->pg_exec) cudaGraphExecDestroy(c->pg_exec);
    c->pg_exec = nullptr;
    return SEM_OK;
  }
  if (option == SEM_OPT_PCG_GRAPH) {
    cudaStreamSynchronize(c->stream);
    c->pcg_graph = value != 0;
    if (c->pg_exec) cudaGraphExecDestroy(c->pg_exec);
    c->pg_exec = nullptr;
    return SEM_OK;
  }
  if (option == SEM_OPT_AX_PDL) {
    cudaStreamSynchronize(c->stream);
    c->ax_pdl = value != 0;
    return SEM_OK;
  }
  if (option == SEM_OPT_PCG_VARIANT) {   // collective for nranks > 1
    if (value != 0 && value != 1) {
      sem::set_error("sem_set_option: SEM_OPT_PCG_VARIANT must be 0 or 1");
      return SEM_EINVAL;
    }
    cudaStreamSynchronize(c->stream);
    c->pcg_variant = value;
    return SEM_OK;
  }
  if (option == SEM_OPT_FDM_TC) {
    cudaStreamSynchronize(c->stream);
    c->fdm_tc = value != 0;
    return SEM_OK;
  }
  if (option == SEM_OPT_COARSE_REPLICATE) {   // collective: same value on every rank
    if (value < -1 || value > 1) {
      sem::set_error("sem_set_option: SEM_OPT_COARSE_REPLICATE must be -1, 0 or 1");
      return SEM_EINVAL;
    }
    cudaStreamSynchronize(c->stream);
    c->coarse_replicate = value;
    if (c->c0 && c->c0_repl != coarse_replicated(c)) {
      schwarz_drop_coarse(c);
      SEM_TRY(schwarz_setup(c));
    }
    return SEM_OK;
  }
  if (option == SEM_OPT_COARSE_ASM) {
    if (value < -1 || value > 2) {
      sem::set_error("sem_set_option: SEM_OPT_COARSE_ASM must be -1, 0, 1 or 2");
      return SEM_EINVAL;
    }
    cudaStreamSynchronize(c->stream);
    c->coarse_asm = value;
    if (c->g0exec) cudaGraphExecDestroy(c->g0exec);
    c->g0exec = nullptr;
    c->g0_iters = -1;
    SEM_TRY(coarse_assemble(c));
    return SEM_OK;
  }
  if (option == SEM_OPT_COARSE_GRAPH) {
    cudaStreamSynchronize(c->stream);
    c->coarse_graph = value != 0;
    return SEM_OK;
  }
  if (option == SEM_OPT_COARSE_ITERS) {
    if (value < 0 || value > 10000) {
      sem::set_error("sem_set_option: SEM_OPT_COARSE_ITERS must be in [0, 10000]");
      return SEM_EINVAL;
    }
    cudaStreamSynchronize(c->stream);
    c->coarse_iters = value;
    return SEM_OK;
  }
  sem::set_error("sem_set_option: unknown option");
  return SEM_EINVAL;
}

extern "C" int sem_p2p_pingpong(sem_ctx* c, int peer, int iters, int64_t* rtt_ns) {
  if (!c || !rtt_ns || iters < 1) return SEM_EINVAL;
  if (!c->p2p_ok || peer < 0 || peer >= c->hp.nranks || peer == c->hp.rank) {
    sem::set_error("sem_p2p_pingpong: needs peer-memory mailboxes and a peer rank != self");
    return SEM_EINVAL;
  }
  long long* d = nullptr;
  SEM_TRY(dalloc(&d, (size_t)iters));
  cudaError_t e = sem::launch_p2p_pingpong(c->p2p, peer, iters, c->ep_ping[peer], d, c->stream);
  c->ep_ping[peer] += (uint64_t)iters;
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && c->hp.rank < peer)
    e = cudaMemcpy(rtt_ns, d, sizeof(long long) * iters, cudaMemcpyDeviceToHost);
  cudaFree(d);
  CUDA_TRY(e);
  return p2p_check(c);
}

extern "C" int sem_p2p_write_bw(sem_ctx* c, int peer, int64_t bytes, int reps, double* gbps) {
  if (!c || !gbps || bytes < 16 || reps < 1) return SEM_EINVAL;
  if (!c->p2p_ok || peer < 0 || peer >= c->hp.nranks) {
    sem::set_error("sem_p2p_write_bw: needs peer-memory mailboxes");
    return SEM_EINVAL;
  }
  const int64_t n = bytes / 16 * 2;   // doubles (even)
  double* src = nullptr;
  SEM_TRY(dalloc(&src, (size_t)n));
  // zeros: the receive entries stay in their initial (flag 0) state
  CUDA_TRY(cudaMemsetAsync(src, 0, sizeof(double) * n, c->stream));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CUDA_TRY(sem::launch_p2p_write(c->p2p, peer, src, n, sem::P2P::kMinRecv * 4, 1, c->stream));
  cudaEventRecord(e0, c->stream);
  cudaError_t e = sem::launch_p2p_write(c->p2p, peer, src, n, sem::P2P::kMinRecv * 4, reps, c->stream);
  cudaEventRecord(e1, c->stream);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(src);
  CUDA_TRY(e);
  *gbps = (double)n * 8.0 * reps / (ms * 1e-3) / 1e9;
  return SEM_OK;
}

extern "C" int sem_debug_read(sem_ctx* c, int which, int64_t* out, int n) {
  if (!c || !out) return SEM_EINVAL;
  if (which == 0) {   // per-block phase timestamps of the fused exchange kernel [5][2048]
    cudaStreamSynchronize(c->stream);
    std::vector<unsigned long long> t(5 * 2048, 0);
    if (sem::p2p_debug_read_blocks(t.data(), 5 * 2048) != 0) return SEM_ECUDA;
    for (int q = 0; q < n && q < 5 * 2048; q++) out[q] = (int64_t)t[q];
    return SEM_OK;
  }
  return SEM_EINVAL;
}

extern "C" int sem_launch_count(const sem_ctx* c, int64_t* n) {
  if (!c || !n) return SEM_EINVAL;
  *n = c->launches;
  return SEM_OK;
}
