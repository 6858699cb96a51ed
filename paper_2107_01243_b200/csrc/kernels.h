// Launchers for the libsem CUDA kernels (called from api.cu).
#pragma once
#include <utility>
#include <cstdint>
#include <vector>
#include <atomic>
#include <cuda_runtime.h>

namespace sem {

// kernel modes of the element operator
enum AxMode { AX_ONLY = 0, AX_APPLY = 1, AX_PCG = 2 };

// device view of the gather-scatter plan
// PCG loop launches with programmatic dependent launch (thread-local switch set
// by pcg_run; kernels call pdl_wait / pdl_trigger, see dev_common.cuh)
void set_pdl(bool on);
bool pdl_on();
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// Launch geometry and function attributes belong to a device: the launchers
// cache them per device index (kMaxDev) in atomics (loopback ranks launch from
// several host threads).
constexpr int kMaxDev = 16;
inline int device_index() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDev) ? d : 0;
}

struct DevPlan {
  int N = 0, n = 0, nloc = 0;
  int64_t n_local = 0;
  int nF = 0, nEd = 0, nV = 0, nS = 0;
  int64_t nbuf = 0;                 // receive / send buffer entries (P > 1)
  const double* D = nullptr;        // [n*n]
  const uint8_t* bmask = nullptr;   // [nloc]
  const int32_t* f_base = nullptr;  // [nF][2]
  const uint8_t* f_axis = nullptr;
  const int32_t* e_base = nullptr;  // [nEd][4]
  const uint8_t* e_axis = nullptr;
  const uint8_t* e_nin = nullptr;
  const uint8_t* e_mask = nullptr;
  const int32_t* v_base = nullptr;  // [nV][8]
  const uint8_t* v_nin = nullptr;
  const uint8_t* v_mask = nullptr;
  const int32_t* f_start = nullptr; // [nloc+1] entities created by each element (gs_dev.cuh)
  const int32_t* e_start = nullptr;
  const int32_t* v_start = nullptr;
  unsigned long long* gs_ctr = nullptr;   // [2] chunk counters (gs_local, exchange), never reset
  // shared points (P > 1)
  const int32_t* s_slot = nullptr;  // [8][nS]
  const int32_t* s_off = nullptr;   // [8][nS]
  const uint8_t* s_nloc = nullptr;
  const uint8_t* s_nr = nullptr;
  const uint8_t* s_mask = nullptr;
  const uint8_t* s_mult = nullptr;
  const int8_t* s_rank = nullptr;   // [8][nS] involved ranks (ascending)
};

// PCG scalars, resident on the device (no per-iteration host sync)
struct PcgState {
  double sigma;          // <p, A p>
  double rho_old;        // <r, z>_c of the previous iteration
  double rho_new;        // <r, z>_c   (rho_new, gamma adjacent: one allreduce)
  double gamma;          // <r, r>_c
  double tol;
  double res_true;
  double sigma_part[2];  // per Ax launch when the operator is split (Alg. 1 overlap)
  double loc[4];         // P > 1: this rank's rho_new, gamma, sigma, res_true partial sums;
                         // the allreduce is out-of-place loc -> global, hence idempotent
  double alpha, beta;    // flexible PCG (Schwarz) scalars
  double dz[2];          // flexible PCG: <z', r'>_c, <z', w>_c
  double loc_dz[2];      // P > 1: this rank's partials of dz
  double cg3[3];         // single-reduction PCG: gamma = <r,u>_c, eps = <r,r>_c, delta = <w,u>_c
  double cg3_loc[3];     // P > 1: this rank's partials of cg3 (one allreduce per iteration)
  uint64_t ep0[3];       // device-side epochs (graph-replayed PCG at P > 1): iteration k
                         // uses ep0[site] + k for the gs exchange, sigma and (rho', gamma)
  int it;                // completed iterations
  int done;              // 0 running, 1 converged, 2 breakdown, 3 NaN, 4 maxit
  int iters;
  int maxit;
  unsigned tickets[8];   // last-block tickets
};

// restarted GMRES state (krylov.cu), device-resident; restart <= kGmMax - 1
constexpr int kGmMax = 32;
struct GmresState {
  double H[(kGmMax + 1) * kGmMax];   // Hessenberg, row stride kGmMax (rotated in place)
  double cs[kGmMax], sn[kGmMax];     // Givens rotations
  double g[kGmMax + 1], y[kGmMax];   // rotated residual vector, solution coefficients
  double h1[kGmMax], h2[kGmMax];     // the two CGS passes' projections
  double norm2[2];                   // c-weighted squared norms (reduction outputs)
  double inv_norm, res, one;         // 1/||.|| for the next basis vector; |g_{j+1}|; 1.0
  int j, jy, cycle_done, converged;  // Arnoldi step, back-substituted size, gates
};

struct AxLaunch {
  const double* u;
  double* w;
  const double* G;
  int r0lo, r0hi, r1lo, r1hi;     // element ranges (local indices)
  double* red_partial;            // PCG: per-block partials
  unsigned* red_ticket;
  double* red_out;                // PCG: reduced sigma (last block), or nullptr: partials only
  const int* done;
  double Dm[144];                 // D (row-major n x n), read from the constant bank
  int* red_count;                 // PCG partials only: number of partials (written by block 0)
  // Helmholtz variant (NEXT-2): w = h1 A_L u + h2 B_L u before gs and mask
  const double* B;
  double h1, h2;
  int gate;                       // 1: any mode returns early when *done (GMRES cycle gate)
  int pdl_pref;                   // 1: launched with PDL; prefetch the first G planes before
                                  //    waiting for the preceding grid
  // PF (one-rank Jacobi-PCG, p update fused): u = p_old (in place), rr = r,
  // dinv, pout = p (= u), beta = the CG state's beta (0 on the first iteration)
  const double* rr;
  const double* dinv;
  double* pout;
  const double* beta;
};

// NVLink peer-memory collectives (p2p.cu): mailbox layout and device view
struct P2P {
  static constexpr int kMaxP = 64;
  static constexpr int kSites = 4;   // allreduce call sites
  static constexpr size_t kSlotOff = 0;
  static constexpr size_t kArFlagOff = kSlotOff + (size_t)kSites * 2 * kMaxP * 4 * 8;
  // gather-scatter receive entries: 16 B "LL" records {lo32, flag, hi32, flag},
  // two epoch parities interleaved per entry (see p2p.cu)
  static constexpr size_t kPingOff = kArFlagOff + (size_t)kSites * kMaxP * 8;   // [kMaxP] ping-pong flags
  static constexpr size_t kRecvOff = kPingOff + (size_t)kMaxP * 8;
  static constexpr int64_t kMinRecv = 1 << 18;   // receive entries allocated at least (probes)
  int P = 1, me = 0, nnbr = 0;
  char* local = nullptr;            // this rank's mailbox
  char* const* peers = nullptr;     // [P] mailbox of every rank (peers[me] == local)
  const int64_t* rdelta = nullptr;  // [P] neighbour recv offset - own send offset
  const int32_t* nbrs = nullptr;    // [nnbr] neighbour ranks
  int* err = nullptr;               // raised on a wait timeout
  uint64_t* xflag = nullptr;        // [kXflags] per packer block: epoch of its finished pack
  static constexpr int kXflags = 8192;
};
enum ArSite { AR_SIG = 0, AR_RG = 1, AR_RES = 2, AR_MISC = 3 };
// peer-memory allreduce fused into a CG kernel (c.P <= 1: unused): the kernel
// waits for the global sums of epoch e_wait and/or publishes its partials as e_pub
struct PeerSync {
  P2P c;
  uint64_t e_wait = 0, e_pub = 0;
  const PcgState* dev = nullptr;   // non-null: the epochs come from dev->ep0 and dev->it
};

cudaError_t launch_gs_pack_p2p(const DevPlan& P, const double* u, double* part, const P2P& c,
                               uint64_t epoch, cudaStream_t s);
int p2p_debug_read_blocks(unsigned long long* out, int n);   // [5][2048] exchange phases
// pack + rank-local gs + unpack in one co-resident kernel (two-kernel operator, nranks > 1)
// sig_part/sig_count (PCG): the Ax kernel's per-CTA sigma partials, or nullptr
cudaError_t launch_gs_exchange_p2p(const DevPlan& P, double* u, double* part, const P2P& c,
                                   uint64_t epoch, int apply_mask, PcgState* st, int nparts,
                                   uint64_t e_sig, const double* sig_part, const int* sig_count,
                                   uint64_t* base, int mode, cudaStream_t s);
// st != nullptr (PCG): also combines the sigma parts and publishes them (epoch e_sig)
cudaError_t launch_gs_unpack_p2p(const DevPlan& P, double* u, const double* part, const P2P& c,
                                 uint64_t epoch, int apply_mask, PcgState* st, int nparts,
                                 uint64_t e_sig, cudaStream_t s);
// Krylov BLAS-1 (krylov.cu); every kernel is skipped when *done (nullptr: never)
cudaError_t launch_mdot(int64_t n, const uint8_t* mult, const double* a, const double* V,
                        int64_t ldv, int K, double* part, unsigned* ticket, double* out,
                        const int* done, int num_sms, cudaStream_t s);
cudaError_t launch_maxpy(int64_t n, double* y, const double* V, int64_t ldv, int K,
                         const double* coef, double alpha, const double* dinv, const uint8_t* mult,
                         double* part, unsigned* ticket, double* out_norm, const int* done,
                         int num_sms, cudaStream_t s);
// y -= sum_i coef[i] V_i, then out[i] = <y, V_i>_c in the same pass (K <= 32)
cudaError_t launch_maxpy_mdot(int64_t n, double* y, const double* V, int64_t ldv, int K,
                              const double* coef, const uint8_t* mult, double* part,
                              unsigned* ticket, double* out, const int* done, int num_sms,
                              cudaStream_t s);
// single-reduction (Chronopoulos-Gear) Jacobi PCG (krylov.cu, reading Q34)
cudaError_t launch_cgcg_init(int64_t n, const double* b, const double* dinv, const uint8_t* mult,
                             double* x, double* r, double* u, double* p, double* s, double* part,
                             unsigned* ticket, double* out2, int num_sms, cudaStream_t st);
cudaError_t launch_cgcg_update(int64_t n, const double* dinv, const uint8_t* mult, double* u,
                               const double* w, double* p, double* s, double* x, double* r,
                               double* part, unsigned* ticket, double* out2, const PcgState* ps,
                               int num_sms, cudaStream_t st);
cudaError_t launch_cgcg_scalar(int stage, PcgState* ps, double* hist, cudaStream_t st);
cudaError_t launch_resid(int64_t n, const double* b, const double* w, double* v,
                         const uint8_t* mult, double* part, unsigned* ticket, double* out,
                         const int* done, int num_sms, cudaStream_t s);
cudaError_t launch_vnorm(int64_t n, const double* w, double* v, double* t, const double* dinv,
                         const GmresState* gs, const int* done, int num_sms, cudaStream_t s);
cudaError_t launch_gm_start(GmresState* gs, PcgState* st, double* hist, cudaStream_t s);
cudaError_t launch_gm_arnoldi(GmresState* gs, PcgState* st, double* hist, int m, cudaStream_t s);
cudaError_t launch_gm_solve(GmresState* gs, PcgState* st, int m, cudaStream_t s);
cudaError_t launch_gm_end_cycle(GmresState* gs, PcgState* st, cudaStream_t s);

// NEXT-1 two-level Schwarz (schwarz.cu)
cudaError_t launch_fdm_setup(int n, int nloc, int64_t e_lo, int ex, int ey, int ez,
                             const double* box, int deform, double amp, const int* per,
                             const double* xi, const double* wq, const double* D, double* S,
                             double* lam, cudaStream_t s);
cudaError_t launch_fdm(int n, int nloc, const double* r, const uint8_t* mult, const double* S,
                       const double* lam, const double* xi, double* y, double* b0,
                       const int* gate, int num_sms, bool tensor_cores, cudaStream_t s);
cudaError_t launch_schwarz_combine(int n, int nloc, const double* y, const double* x0,
                                   const uint8_t* mult, const double* xi, double* z,
                                   const double* r, const double* w, double* partial,
                                   unsigned* ticket, double* dots, const int* gate, int num_sms,
                                   cudaStream_t s);
cudaError_t launch_fcg_scalar(int stage, PcgState* st, double* hist, cudaStream_t s);
cudaError_t launch_xpay(int64_t n, double* p, const double* z, const PcgState* st, int num_sms,
                        cudaStream_t s);
cudaError_t launch_gate_state(PcgState* st, const int* gate, cudaStream_t s);
cudaError_t launch_rel_tol(PcgState* st, double rtol, cudaStream_t s);
cudaError_t launch_copy_gate(int* dst, const int* gate, cudaStream_t s);

// assembled coarse operator (coarse.cu): CG state and operands on the nu unique
// unmasked N = 1 vertices
struct CoarseCg {
  double gamma, sigma, alpha, beta, tol, mean, red;
  int it, done, maxit;     // done: 0 running, 1 converged, 2 breakdown, 3 NaN, 4 maxit, 5 gated
  unsigned ticket[4];
};
struct CoarseAsm {
  int nu = 0, K = 0;       // unknowns, ELL width
  int64_t n0 = 0;          // coarse E-vector slots
  int periodic = 0;        // fully periodic: remove the mean of the right-hand side
  const int32_t* col = nullptr;      // [K][nu] ELL, ascending per row, padded (row, 0.0)
  const double* val = nullptr;
  const int32_t* u2s_ptr = nullptr;  // [nu + 1] unique -> slots (ascending)
  const int32_t* u2s = nullptr;
  const int32_t* uidx = nullptr;     // [n0] slot -> unique, -1 masked
  double *b = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr;   // [nu]
  double* partial = nullptr;         // [grid]
  CoarseCg* st = nullptr;
};
int coarse_asm_grid(int nu, int num_sms);
// small coarse problems (nu <= kCoarseClusterMax): the whole solve on one 8-CTA cluster
constexpr int kCoarseClusterMax = 1 << 14;   // C2 (8192): 0.232 -> 0.189 ms; C3 (32768): 0.315 -> 0.373, slower
bool coarse_asm_cluster_ok(int nu);
cudaError_t launch_coarse_asm_cluster(const CoarseAsm& A, const double* b0, double* x0,
                                      const int* gate, int maxit, double rtol, cudaStream_t s,
                                      int64_t* launches);
// x0 = A0^-1 b0 by <= maxit CG steps on the assembled operator (b0, x0: E-vectors)
cudaError_t launch_coarse_asm_solve(const CoarseAsm& A, const double* b0, double* x0,
                                    const int* gate, int maxit, double rtol, int grid,
                                    cudaStream_t s, int64_t* launches);

// interconnect probes for the performance model: one-thread ping-pong
// with `peer` (round-trip ns per sample), and one-sided peer writes (bandwidth)
cudaError_t launch_p2p_pingpong(const P2P& c, int peer, int iters, uint64_t e0, long long* out,
                                cudaStream_t s);
cudaError_t launch_p2p_write(const P2P& c, int peer, const double* src, int64_t n, int64_t cap,
                             int reps, cudaStream_t s);
cudaError_t launch_ar_publish(const P2P& c, int site, uint64_t epoch, const double* v, int K,
                              cudaStream_t s);
cudaError_t launch_ar_finish(const P2P& c, int site, uint64_t epoch, double* out, int K,
                             cudaStream_t s);

// returns max resident CTAs/SM for the Ax kernel of this N and mode
int ax_occupancy(int N, int mode);
// helm: the Helmholtz variant (a.B, a.h1, a.h2), AX_APPLY / AX_PCG
// pf: AX_PCG with the p update fused in (p = dinv r + beta p, see AxLaunch)
cudaError_t launch_ax(const DevPlan& P, const AxLaunch& a, int mode, int grid, cudaStream_t s,
                      bool helm = false, bool pf = false);
int ax_groups(int N, int nelem);   // element groups processed per launch

// setup
cudaError_t launch_geom(const DevPlan& P, const double* xi, const double* wq, int64_t e_lo,
                        int ex, int ey, int ez, const double* box, int deform, double amp,
                        double* G, double* B, int* bad, cudaStream_t s);
cudaError_t launch_coords(const DevPlan& P, const double* xi, int64_t e_lo, int ex, int ey, int ez,
                          const double* box, int deform, double amp, double* X, double* Y,
                          double* Z, cudaStream_t s);
cudaError_t launch_diag(const DevPlan& P, const double* G, double* d, cudaStream_t s);
cudaError_t launch_mult(const DevPlan& P, uint8_t* mult, cudaStream_t s);
cudaError_t launch_invert_mask(const DevPlan& P, double* d, cudaStream_t s);
cudaError_t launch_scale(const double* B, const double* f, double* b, int64_t n, cudaStream_t s);
cudaError_t launch_scale_mask(const DevPlan& P, const double* B, const double* f, double* b,
                              cudaStream_t s);
cudaError_t launch_helm_diag(double* d, const double* B, double h1, double h2, int64_t n,
                             cudaStream_t s);
cudaError_t launch_mask(const DevPlan& P, double* u, cudaStream_t s);
cudaError_t launch_export_mask(const DevPlan& P, uint8_t* m, cudaStream_t s);

// gather-scatter (standalone)
// *base: host copy of the chunk counter (advanced by the tickets the launch takes)
// mode: 0 auto (flat while w fits in L2, else element-ordered chunks), 1 flat, 2 chunks
// sig (one-rank PCG, SEM_GS_SIGMA): the gs kernel's last block also sums the Ax
// kernel's sigma partials into st->sigma (the CG update's order and block size)
struct GsSigma {
  const double* part = nullptr;
  const int* count = nullptr;
  PcgState* st = nullptr;
};
cudaError_t launch_gs_local(const DevPlan& P, double* u, int apply_mask, uint64_t* base,
                            int mode, cudaStream_t s, const GsSigma* sig = nullptr);
cudaError_t launch_gs_pack(const DevPlan& P, const double* u, double* part, double* sendbuf,
                           cudaStream_t s);
cudaError_t launch_gs_unpack(const DevPlan& P, double* u, const double* part,
                             const double* recvbuf, int apply_mask, PcgState* st, int nparts,
                             cudaStream_t s);

// reductions / CG vector kernels
int cg_grid(int num_sms);
cudaError_t launch_dot_c(const DevPlan& P, const uint8_t* mult, const double* a, const double* b,
                         double* partial, unsigned* ticket, double* out, int grid, cudaStream_t s);
cudaError_t launch_sum_c(const DevPlan& P, const uint8_t* mult, const double* a, double* partial,
                         unsigned* ticket, double* out2, int grid, cudaStream_t s);
cudaError_t launch_sub_scalar(double* a, const double* scal, int64_t n, cudaStream_t s);
cudaError_t launch_cg_init(const DevPlan& P, const uint8_t* mult, const double* dinv,
                           const double* b, double* x, double* r, double* p, double* partial,
                           PcgState* st, double* out2, const PeerSync& ps, int grid,
                           cudaStream_t s, int pzero = 0);
cudaError_t launch_cg_start(PcgState* st, double* hist, const PeerSync& ps, cudaStream_t s);
// sig_part/sig_count: the Ax kernel's per-CTA sigma partials (P = 1; every block
// re-sums them in a fixed order) or nullptr (P > 1: sigma is already allreduced).
// x != nullptr (one rank, p update fused into the Ax kernel): also x += alpha p,
// and the last block ends the iteration (convergence, beta, history)
cudaError_t launch_cg_update(const DevPlan& P, const uint8_t* mult, const double* dinv, double* r,
                             const double* w, double* partial, PcgState* st, double* out2,
                             const double* sig_part, const int* sig_count, const PeerSync& ps,
                             int grid, cudaStream_t s, double* x = nullptr,
                             const double* p = nullptr, double* hist = nullptr, int end_here = 1,
                             const int32_t* gu = nullptr);
// PF over NCCL / loopback: end of the iteration after the host-side allreduce
cudaError_t launch_cg_end_iter(PcgState* st, double* hist, cudaStream_t s);
bool gs_flat(const DevPlan& P, int mode);   // the gs schedule `mode` resolves to the flat sweep
// x += alpha p, then (unless the solve ended) p = dinv r + beta p
cudaError_t launch_cg_p(const DevPlan& P, const double* dinv, const double* r, double* p, double* x,
                        PcgState* st, double* hist, const PeerSync& ps, int grid, cudaStream_t s);
cudaError_t launch_cg_residual(const DevPlan& P, const uint8_t* mult, const double* b,
                               const double* w, double* partial, PcgState* st, double* out1,
                               const PeerSync& ps, int grid, cudaStream_t s);

// loopback multi-rank transport (loopback.cu; tests): P rank contexts on one
// device, collectives by device copies with rank-ordered sums
struct LoopComm;
LoopComm* loop_lookup(const void* handle);   // nullptr unless a live loopback handle
int loop_rank(const LoopComm* c);
int loop_size(const LoopComm* c);
// Alg. 1 exchange: send + off[k] (cnt[k] doubles) to nbr[k], receive into recv + off[k]
int loop_sendrecv(LoopComm* c, const double* send, double* recv, const std::vector<int32_t>& nbr,
                  const std::vector<int64_t>& off, const std::vector<int64_t>& cnt, cudaStream_t s);
int loop_allreduce(LoopComm* c, const double* in, double* out, size_t count, cudaStream_t s);
int loop_allgather(LoopComm* c, const void* in, void* out, size_t bytes, cudaStream_t s);

}  // namespace sem
