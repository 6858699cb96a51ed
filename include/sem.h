/*
 * sem.h -- C ABI of the B200-native matrix-free SEM pressure-Poisson hot path
 * (Neko, arxiv 2107.01243).  Implemented by paper_2107_01243_b200/libsem.so
 * (hand-written CUDA for sm_100a + NCCL).  No torch types cross this boundary:
 * plain pointers and sizes only.
 *
 * Citations "P:L<n>" are lines of the paper text;
 * readings Q1..Q22 where the paper is silent or garbled are in DESIGN.md.
 *
 * Data layout (reading Q3, the paper leaves it free):
 *   element e = ex + Ex*(ey + Ey*ez); rank r owns the contiguous element range
 *   [r*E/P, (r+1)*E/P) (lexicographic partition); its local element index is
 *   e - r*E/P.  A field is an E-vector u_L: n_local = E_local*(N+1)^3
 *   fp64 values, slot l = e_local*n^3 + i + n*j + n^2*k with n = N+1 and i
 *   running along x fastest.  Field pointers passed to hot calls are DEVICE
 *   pointers, 16-byte aligned (a torch.cuda tensor satisfies this), caller
 *   owned, at least n_local doubles.
 *
 * Status codes: every function returns one of the values below.  On an error
 * sem_last_error() returns a thread-local message.  No exception crosses the ABI.
 * All device work is ordered on sem_mesh.stream; sem_ax/sem_gs/sem_apply/
 * sem_rhs are asynchronous with respect to the host, sem_setup and the PCG
 * solves block.  Calls marked "collective" must be made by every rank in
 * the same order.  One context per stream / host thread.
 */
#ifndef SEM_H
#define SEM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEM_OK 0
#define SEM_NOT_CONVERGED 1    /* PCG hit maxit; result filled */
#define SEM_EINVAL (-1)        /* bad argument: counts, extents, N outside 1..11,
                                  periodic axis with < 2 elements, P > E, NULL or
                                  misaligned pointer */
#define SEM_EGEOM (-2)         /* Jacobian <= 0 at some GLL point */
#define SEM_ECUDA (-3)         /* CUDA runtime error (or no device) */
#define SEM_ENCCL (-4)         /* NCCL error */
#define SEM_ENOMEM (-5)        /* allocation failed */
#define SEM_EBREAKDOWN (-6)    /* CG breakdown: p^T A p <= 0 or NaN */

typedef struct sem_ctx sem_ctx; /* opaque; owns D, G, B, plan, dinv, work vectors */

/* Hexahedral box mesh ("E non-overlapping hexahedral elements").
   Non-periodic faces carry homogeneous Dirichlet conditions (Eq. 5). */
typedef struct {
  int32_t ex, ey, ez;                 /* elements per axis (>= 1; >= 2 if periodic) */
  double x0, x1, y0, y1, z0, z1;      /* box extents, x1 > x0 etc. */
  int32_t periodic[3];                /* 1 = periodic axis */
  int32_t deform;                     /* 0 Cartesian; 1 x_m += a sin X sin Y sin Z on the
                                         box rescaled to (0,2pi)^3 (reading Q4) */
  double deform_amp;                  /* a */
  int32_t rank, nranks;               /* this process and the element partition size */
  void* nccl_comm;                    /* nranks > 1: ncclComm_t (sem_nccl_*) or a loopback
                                         handle (sem_loopback_comm); else NULL */
  void* stream;                       /* cudaStream_t all work is ordered on (NULL = legacy) */
} sem_mesh;

/* ---- setup (GLL space, D, geometric factors G^e, numbering) ----
   Builds the GLL rule and derivative matrix (Eq. 7), the node
   coordinates and the six geometric factors G = J w_i w_j w_k (dr/dx)(dr/dx)^T
   and mass B = J w_i w_j w_k (reading Q5) on the device, the gather-scatter plan
   (element-local entities summed on this GPU, entities shared with
   other ranks exchanged through the multi-rank transport -- NVLink peer memory
   by default, NCCL, or the single-device loopback of sem_loopback_*), the
   Dirichlet mask and the Jacobi inverse diagonal (reading Q14).  Collective,
   blocking.  N in 1..11.  For nranks > 1, nccl_comm is an ncclComm_t
   (sem_nccl_comm_init) or a loopback handle (sem_loopback_comm). */
int sem_setup(const sem_mesh* m, int N, sem_ctx** out);
int sem_destroy(sem_ctx* c);
/* n_local = local slots, e_local = local elements, n_glob = unique global DOF */
int sem_sizes(const sem_ctx* c, int64_t* n_local, int64_t* e_local, int64_t* n_glob);

/* ---- hot path ----
   sem_ax:    w_L = A_L u_L, A^e = D^T G^e D per element (Eq. 9); no gs, no mask.
   sem_gs:    u_L <- Q Q^T u_L in place (Eq. 10), sum over all slots
              sharing a global number, in ascending slot order within a rank and
              ascending rank order across ranks (reading Q10).  Collective.
   sem_apply: w = mask(Q Q^T A_L u) -- the CG operator: the Ax kernel
              (mask in its epilogue), then the gather-scatter kernel; at
              nranks > 1 the shared partials travel through the transport
              (one peer-memory exchange kernel, or Alg. 1's overlapped
              pack / send-recv / unpack).  Collective.
   u and w must not alias. */
int sem_ax(sem_ctx* c, const double* u, double* w);
int sem_gs(sem_ctx* c, double* u);
int sem_apply(sem_ctx* c, const double* u, double* w);

/* b = mask(Q Q^T (B .* f)) with f the nodal values of the forcing (Eq. 6 RHS,
   collocated quadrature, reading Q12); on a fully periodic box the unique-DOF
   mean is removed (reading Q13).  Collective. */
int sem_rhs(sem_ctx* c, const double* f, double* b);
/* device node coordinates (x, y, z per slot), for evaluating forcing terms */
int sem_coords(sem_ctx* c, double* X, double* Y, double* Z);

/* ---- Jacobi-preconditioned CG (readings Q14-Q17) ----
   x0 = 0; stops when sqrt(<r,r>_c) <= tol (absolute, c = 1/multiplicity) or
   after maxit iterations (iterations = applications of A).  res_final is the
   recursive residual, res_true = sqrt(<b - A x, b - A x>_c) computed once at the
   end.  Returns SEM_OK, SEM_NOT_CONVERGED or an error.  Collective, blocking.
   sem_pcg_solve takes device b, x; sem_pcg_solve_host takes HOST b, x and does
   the host<->device copies itself (end-to-end entry point); both run the
   preconditioner selected by SEM_OPT_PRECOND (Jacobi, or flexible PCG with
   the two-level Schwarz preconditioner). */
typedef struct {
  int32_t iters;      /* applications of A in the loop (reading Q16) */
  double res_final;   /* recursive residual sqrt(<r,r>_c) at exit */
  double res_true;    /* sqrt(<b - A x, b - A x>_c), one extra A at the end (Q17) */
  int32_t status;     /* SEM_OK, SEM_NOT_CONVERGED or an error code */
} sem_pcg_result;
int sem_pcg_solve(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                  sem_pcg_result* res);
/* NEXT-2: the Helmholtz operator of the velocity solves, h1 A + h2 B (P:L257
   "followed by a Helmholtz equation for each velocity component").
   sem_helm_apply: w = mask(QQ^T (h1 A_L u + h2 B_L u)) for any local u (B_L the
   diagonal GLL mass); asynchronous, like sem_apply.  sem_rhs_mass: b =
   mask(QQ^T (B .* f)) WITHOUT the periodic mean projection of sem_rhs (the
   Helmholtz system is nonsingular for h2 > 0).  sem_helm_pcg_solve: Jacobi-PCG
   on h1 A + h2 B (h1, h2 >= 0, not both 0) with the exact assembled diagonal
   QQ^T(h1 diag(A_L) + h2 B_L) (cached per (h1, h2)); same contract, status
   codes and result as sem_pcg_solve.  Always the two-kernel operator. */
int sem_helm_apply(sem_ctx* c, double h1, double h2, const double* u, double* w);
int sem_rhs_mass(sem_ctx* c, const double* f, double* b);
int sem_helm_pcg_solve(sem_ctx* c, double h1, double h2, const double* b, double* x,
                       double tol, int32_t maxit, sem_pcg_result* r);
/* NEXT-3 (Table 2 "GMRES ... Projections 20"): the pressure
   solver pipeline.  sem_gmres_solve: restarted GMRES(restart), restart in
   [1, 31], right Jacobi preconditioning, x0 = 0, same tolerance / iteration /
   result conventions as sem_pcg_solve (an iteration = one operator application
   in the Arnoldi process; res_final = the Arnoldi residual estimate, res_true =
   ||b - A x||_c).  sem_proj_solve: Fischer's solution projection with a space
   of m <= 32 A-orthonormal previous solutions kept in the context: x_bar =
   sum <z_i, b>_c z_i, GMRES on b - A x_bar, x = x_bar + delta, then x is
   A-orthonormalised into the space (reset to the latest solution when full;
   skipped if negligible).  Changing m resets the space; sem_proj_reset empties
   it.  Collective for nranks > 1; blocking. */
int sem_gmres_solve(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                    int32_t restart, sem_pcg_result* r);
int sem_proj_solve(sem_ctx* c, const double* b, double* x, double tol, int32_t maxit,
                   int32_t restart, int32_t m, sem_pcg_result* r);
int sem_proj_reset(sem_ctx* c);
int sem_proj_size(const sem_ctx* c, int32_t* k);
/* NEXT-1 ("two-level additive overlapping Schwarz method ...
   M0^-1 = R0^T A0^-1 R0 + sum_k R_k^T A~_k^-1 R_k"; the coarse grid on linear
   elements solved by "few (~10) CG iterations"; readings Q28-Q32 in DESIGN.md).
   sem_schwarz_apply: z = M r for an assembled residual r (device, n_local,
   slot order; r and z must not alias):
     z = mask( c^1/2 QQ^T (A~^-1 (c^1/2 r))_L + R0^T A0^-1 R0 r )
   A~_e = the separable operator of element e with one node of overlap
   (applied by fast diagonalisation), A0 = the N = 1 operator on the same mesh
   (an internal second context), A0^-1 = at most SEM_OPT_COARSE_ITERS plain CG
   steps from 0 (stopped at ||r0||_c <= 1e-12 ||b0||_c).  which: 1 = local
   part, 2 = coarse part, 3 = both.  The first call builds the preconditioner
   (collective for nranks > 1, blocking); later calls are asynchronous on the
   stream.  With SEM_OPT_PRECOND = SEM_PRECOND_SCHWARZ, sem_pcg_solve runs
   flexible PCG (beta = -alpha <z', w>_c / rho) and sem_gmres_solve /
   sem_proj_solve run flexible GMRES (the preconditioned basis is stored) with
   M; sem_helm_pcg_solve keeps Jacobi (the paper's velocity solver). */
int sem_schwarz_apply(sem_ctx* c, const double* r, double* z, int32_t which);
int sem_pcg_solve_host(sem_ctx* c, const double* b_host, double* x_host, double tol,
                       int32_t maxit, sem_pcg_result* res);
/* recursive residual history of the last solve: hist[k] after k iterations */
int sem_pcg_history(const sem_ctx* c, double* host_dst, int32_t max_entries, int32_t* n);

/* ---- exports for parity tests (host buffers, caller allocated) ----
   which: 0 xi[n], 1 w[n], 2 D[n*n], 3 G[E_local*6*n^3], 4 B[n_local], 5 dinv[n_local] */
int sem_export_field(const sem_ctx* c, int which, double* host_dst);
/* which: 0 multiplicity[n_local], 1 mask[n_local] (1 = Dirichlet slot) */
int sem_export_int(const sem_ctx* c, int which, int64_t* host_dst);

typedef struct sem_plan sem_plan;
/* Live plan export (P:L107 global numbering, P:L231 pairs / segments, Alg. 1
   shared lists): a planner handle (query it with the sem_plan_* accessors
   below, free it with sem_plan_destroy) built from the gather-scatter
   records the context's kernels use, copied back from the device: the face /
   edge / vertex incidence records and the shared-point lists expand into the
   pairs, segments and per-neighbour lists; multiplicity and mask are the
   device arrays; global numbers come from the lattice formula (reading Q6,
   never stored on the device).  Blocking. */
int sem_export_plan(const sem_ctx* c, sem_plan** out);

/* ---- host-only planner (no device needed; used by CPU tests) ----
   Exposes the gather-scatter plan a rank would build for this mesh: lattice
   global numbering (reading Q6), multiplicity, mask, the injective pairs
   (l_a < l_b) sorted by l_a and the non-injective segments sorted by first
   slot, the neighbour ranks and, per neighbour, the shared global
   numbers in ascending order (Alg. 1 buffers). */
int sem_plan_create(const sem_mesh* m, int N, sem_plan** out);
int sem_plan_destroy(sem_plan* p);
int sem_plan_sizes(const sem_plan* p, int64_t* n_local, int64_t* npairs, int64_t* nseg,
                   int64_t* nsegslots, int32_t* n_nbr);
int sem_plan_slots(const sem_plan* p, int64_t* gid, int64_t* mult, int64_t* mask);
int sem_plan_pairs(const sem_plan* p, int64_t* pairs, int64_t* seg_off, int64_t* seg_slot);
int sem_plan_neighbors(const sem_plan* p, int32_t* ranks, int64_t* counts);
int sem_plan_shared(const sem_plan* p, int32_t q, int64_t* gids);
/* GLL nodes xi[n], weights w[n] and D[n*n] (row-major, D[i*n+j] = l_j'(xi_i)) */
int sem_plan_space(const sem_plan* p, double* xi, double* w, double* D);

/* ---- NCCL bootstrap (one process per GPU; the 128-byte unique id is
   broadcast by the caller, e.g. with torch.distributed) ---- */
int sem_nccl_unique_id(uint8_t id[128]);
int sem_nccl_comm_init(const uint8_t id[128], int rank, int nranks, void** comm);
int sem_nccl_comm_destroy(void* comm);

/* ---- loopback multi-rank transport (tests on ONE device) ----
   P rank contexts in one process on one GPU, each driven by its own host
   thread with its own stream.  sem_loopback_create makes a world of nranks
   ranks; sem_loopback_comm returns rank r's handle, passed as
   sem_mesh.nccl_comm with rank = r, nranks = P.  Every collective runs the
   NCCL transport's path (pack, neighbour exchange, unpack with ascending-rank
   sums; allreduces summed in ascending rank order) with device copies and
   host barriers instead of NCCL; the peer-memory transport is not used.
   flags & 1: process neighbours in reverse order and delay each rank's
   arrival randomly (completion order changes, results must not).  A rank
   that does not reach a collective within flags >> 8 seconds (0: 120 s)
   makes it fail with SEM_ENCCL on the ranks that did.  Destroy the world after every context using it. */
int sem_loopback_create(int nranks, int flags, void** world);
int sem_loopback_comm(void* world, int rank, void** comm);
int sem_loopback_destroy(void* world);

/* ---- instrumentation ----
   sem_timing(c, 1) records CUDA events on the context stream around every
   launch of kernel class `which` (0 = Ax kernel of apply/PCG, 1 = CG
   update, 2 = p update, 3 = Ax only, 4 = gather-scatter kernel of apply/PCG,
   5 = peer-memory pack, 6 = peer-memory unpack, 7 = Schwarz local-solve kernel,
   8 = Schwarz combine kernel, 9 = Ax kernel with the fused p update of the
   one-rank PCG iteration); sem_timing_read returns the summed
   device time in ms and the number of timed launches since the last reset.
   sem_launch_count returns the number of kernels this context has launched. */
int sem_timing(sem_ctx* c, int enable);
int sem_timing_read(sem_ctx* c, int which, double* total_ms, int64_t* count);
int sem_launch_count(const sem_ctx* c, int64_t* n);
/* instrumentation: which = 0 -> per-block phase timestamps (ns, %globaltimer)
   of the last peer-memory exchange kernel, [5][2048] (phases: start, packed,
   local gs done, unpack done, end; 0 for absent blocks) */
int sem_debug_read(sem_ctx* c, int which, int64_t* out, int n);
/* Interconnect probes for the performance model (nranks > 1 with
   peer-memory mailboxes).  sem_p2p_pingpong: collective between this rank and
   `peer` (both call it with the same iters); the lower rank writes `iters`
   round-trip times (ns, one flag each way through the mailboxes) into host
   rtt_ns.  sem_p2p_write_bw: one-sided, writes `bytes` of zeros into the peer's
   receive area `reps` times with 16-B stores and returns GB/s; do not call
   while an exchange with that peer is in flight.  Both block. */
int sem_p2p_pingpong(sem_ctx* c, int peer, int iters, int64_t* rtt_ns);
int sem_p2p_write_bw(sem_ctx* c, int peer, int64_t bytes, int reps, double* gbps);
/* Option numbers 1 (fused Ax+gs kernel), 5 (programmatic dependent launch of
   every PCG kernel) and 10 (gs fused with the CG update) are retired: those
   variants were measured slower than the default path and
   removed; setting them returns SEM_EINVAL. */
/* Multi-GPU transport of the hot path (nranks > 1): 1 (default) = NVLink peer
   memory (CUDA-IPC mailboxes, see p2p.cu), 0 = NCCL send/recv + allreduce.
   Falls back to NCCL automatically if peer memory cannot be mapped. */
#define SEM_OPT_P2P 2
/* nranks > 1: 1 = Alg. 1 overlap (Ax on the boundary elements, send,
   Ax on the interior elements while the partials travel); 0 = one Ax launch. */
#define SEM_OPT_OVERLAP 3
/* Rank-local gather-scatter schedule (results bit-identical in every mode):
   0 (default) auto, 1 = flat (each entity class swept over the whole grid;
   best while w is L2-resident), 2 = element-ordered chunks pulled dynamically
   by the blocks (each element's w streamed from HBM about once).  Auto picks
   2 when w exceeds 256 MB. */
#define SEM_OPT_GS_MODE 4
/* Preconditioner of sem_pcg_solve / sem_gmres_solve / sem_proj_solve:
   SEM_PRECOND_JACOBI (default) or SEM_PRECOND_SCHWARZ (NEXT-1; setting it
   builds the Schwarz preconditioner: collective, blocking). */
#define SEM_OPT_PRECOND 6
#define SEM_PRECOND_JACOBI 0
#define SEM_PRECOND_SCHWARZ 1
/* maximum CG iterations of the Schwarz coarse solve (default 10) */
#define SEM_OPT_COARSE_ITERS 7
/* 1 (default) = on one rank the Schwarz coarse solve is captured once and
   replayed as a CUDA graph (identical results); 0 = stream launches */
#define SEM_OPT_COARSE_GRAPH 8
/* 1 (default) = at N = 7 the Schwarz local solves run their six 8x8
   contractions on the fp64 tensor cores (DMMA m8n8k4); 0 = CUDA-core kernel */
#define SEM_OPT_FDM_TC 9
/* Schwarz coarse level at nranks > 1: 0 = distributed over the ranks (each
   coarse CG step exchanges and allreduces), 1 = replicated (one all-gather of
   the restricted right-hand side, then every rank solves the whole N = 1
   problem; needs an even element partition), -1 (default) = auto (replicated
   when the coarse problem has <= 2^26 slots, the bound of the assembled
   coarse operator).  Collective. */
#define SEM_OPT_COARSE_REPLICATE 11
/* Jacobi-PCG recurrences of sem_pcg_solve / sem_helm_pcg_solve /
   sem_pcg_solve_host: 0 (default) = standard (two reductions per iteration),
   1 = single-reduction Chronopoulos-Gear form: the dots
   <r,u>, <r,r> of the update pass and <w,u> of the operator application are
   reduced together, one allreduce per iteration at nranks > 1 (one extra
   vector pass per iteration).  Same iterates in exact arithmetic (DESIGN.md
   reading Q34).  Collective. */
#define SEM_OPT_PCG_VARIANT 12
/* 1 (default) = in PCG iterations the Ax kernel alone is launched with
   programmatic dependent launch and its producer warp streams the first
   geometric-factor planes before waiting for the preceding kernel; 0 = plain
   order.  Identical results. */
#define SEM_OPT_AX_PDL 13
/* 1 (default) = on one rank with the flat gather-scatter schedule, the
   kernels of each batch of 8 Jacobi-PCG iterations are captured once into a
   CUDA graph (cached per x / Jacobi operand) and replayed; 0 = stream
   launches.  Identical results. */
#define SEM_OPT_PCG_GRAPH 14
/* 1 (default) = Jacobi-PCG fuses the p update p = dinv r + beta p into the
   next iteration's Ax kernel (which streams p, r, dinv and writes p) and
   x += alpha p into the r update: three kernels per iteration (Ax, gs or the
   exchange kernel, update; at nranks > 1 over NCCL / loopback a one-thread
   kernel ends the iteration after the allreduce) instead of four; 0 =
   separate p kernel.  Same arithmetic (each
   value is computed by the same expression), iterates equal up to the
   sigma partial-sum order. */
#define SEM_OPT_PCG_FUSE 15
/* 1 = on one rank with SEM_OPT_PCG_FUSE, the PCG iteration launches no
   gather-scatter kernel: the r update sums the unassembled w = A_L p over each
   shared point's incidences on read (ascending slots, the gs kernel's sum)
   through a per-element incidence table (496 B per element, built on the
   first solve); 0 = separate gs kernel; -1 (default) = auto, 1 when the
   vector exceeds 64 MiB (below, the separate gs kernel on an L2-resident w is
   faster) and one z-layer of elements holds at most 8 MiB of it (beyond, the
   +z face partners fall out of the L2 before reuse).  Identical results. */
#define SEM_OPT_PCG_GSU 16
/* Schwarz coarse solve when the coarse level is single-rank (one rank, or
   the replicated level): -1 (default) / 1 = CG on the ASSEMBLED N = 1 operator
   over the unique unmasked vertices (ELL, built once at Schwarz setup from the
   element matrices; up to 2^14 unknowns the whole solve runs on one 8-CTA
   thread-block cluster), 2 = the assembled operator always with the
   multi-kernel solve, 0 = CG on the element operator + gather-scatter over the
   E-vector slots (also beyond 2^26 coarse slots).  Same iterates in exact
   arithmetic (reading Q35). */
#define SEM_OPT_COARSE_ASM 17
/* 1 (default) = on one rank with the flat gather-scatter schedule, the kernels
   of each batch of 8 flexible-PCG (Schwarz) iterations, the coarse solve
   included, are captured once into a CUDA graph and replayed; 0 = stream
   launches.  Identical results. */
#define SEM_OPT_SCHWARZ_GRAPH 18
/* 1 (default) = on one rank with the flat gather-scatter schedule, each GMRES
   restart cycle (restart residual, the m Arnoldi steps with their
   preconditioner applications, the least-squares update) is captured once
   into a CUDA graph and replayed; 0 = stream launches (polling every 8
   steps).  Identical results. */
#define SEM_OPT_GMRES_GRAPH 19
int sem_set_option(sem_ctx* c, int option, int value);

const char* sem_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SEM_H */
