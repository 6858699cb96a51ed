// Internal declarations of libsem (B200-native SEM Poisson hot path).
// Host planner (plan.cpp), device kernels (*.cu) and the C ABI (api.cu).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/sem.h"

namespace sem {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);

// ---------------------------------------------------------------- entities
// The gather-scatter plan is entity based: every
// element face, edge and vertex shared by >= 2 elements is one entity; its
// points are the face/edge interior nodes (or the vertex).  All incidences
// of an entity see the same point parametrisation (conforming, aligned hex
// box mesh), so a point's slot in incidence t is base[t] + offset(kind, p).
enum EntClass { CLS_FACE = 0, CLS_EDGE = 1, CLS_VERT = 2 };
constexpr int kRefsPerElem = 26;   // 6 faces + 12 edges + 8 vertices
// Per-element incidence table of the gather-on-read CG update (SEM_OPT_PCG_GSU,
// kern.cu gu_gather): for each of the element's sub-entities the slot bases of
// ALL incidences of its local entity, ascending, -1 padded (all -1: not a
// local entity).  Faces 2a+b (normal axis a, side b) x 2 bases at [0, 12);
// edges 4a + s_lo + 2 s_hi (direction a, sides of the two other axes in
// ascending order) x 4 at [12, 60); vertices s_x + 2 s_y + 4 s_z x 8 at
// [60, 124).  A point's slot in incidence t is base[t] + its offset along the
// entity (the spanning coordinates), as in the gs kernel.
constexpr int kGuEdge = 12, kGuVert = 60, kGuInts = 124;

struct HostPlan {
  sem_mesh m{};
  int N = 0, n = 0;
  int64_t n3 = 0;
  int64_t E = 0, e_lo = 0, e_hi = 0, nloc = 0, n_local = 0, nglob = 0;
  int rank = 0, nranks = 1;
  bool fully_periodic = false;
  std::vector<double> xi, w, D;           // GLL rule, D[i*n+j] = l_j'(xi_i)
  std::vector<uint8_t> bmask;             // [nloc] bit (2a+b): face (axis a, side b) Dirichlet
  // local entities (all incidences on this rank), SoA
  int64_t nF = 0, nEd = 0, nV = 0;
  std::vector<int32_t> f_base;            // [2][nF]
  std::vector<uint8_t> f_axis;            // [nF] face normal axis
  std::vector<int32_t> e_base;            // [4][nEd]
  std::vector<uint8_t> e_axis, e_nin, e_mask;
  std::vector<int32_t> v_base;            // [8][nV]
  std::vector<uint8_t> v_nin, v_mask;
  // entities are created by their smallest local element, in element order:
  // element el created faces [f_start[el], f_start[el+1]) (likewise edges, vertices)
  std::vector<int32_t> f_start, e_start, v_start;   // [nloc + 1]
  // shared points (some incidence on another rank), ascending gid
  int64_t nS = 0;
  std::vector<int64_t> s_gid;
  std::vector<int32_t> s_slot;            // [8][nS] local slots ascending (-1 pad)
  std::vector<uint8_t> s_nloc, s_mult, s_mask, s_nr;
  std::vector<int32_t> s_off;             // [8][nS] per involved rank (ascending): -1 self, else buffer index
  std::vector<int8_t> s_rank;             // [8][nS] the involved ranks (ascending), -1 pad
  std::vector<int32_t> nbr_rank;
  std::vector<int64_t> nbr_off, nbr_cnt;
  int64_t nbuf = 0;
  // Alg. 1 overlap: boundary elements [b0lo,b0hi) U [b1lo,b1hi), interior [ilo,ihi)
  int64_t b0lo = 0, b0hi = 0, b1lo = 0, b1hi = 0, ilo = 0, ihi = 0;
  // live-context export (sem_export_plan): multiplicity and mask read back from
  // the device (empty for a host-only plan, which derives them itself)
  std::vector<int64_t> x_mult, x_mask;
};
// a planner handle around a copy of p (sem_export_plan; destroyed by sem_plan_destroy)
sem_plan* plan_wrap(const HostPlan& p);

int build_plan(const sem_mesh* m, int N, HostPlan* p);   // returns SEM_* status
// the kGuInts-per-element incidence table of the local entities
void build_gu_table(const HostPlan& p, std::vector<int32_t>* tab);
// device G layout (see dev_common.cuh g_index): G[e][k][f][i + n j]
inline int64_t g_index_host(int64_t el, int f, int p, int n) {
  const int n2 = n * n, k = p / n2, ij = p - k * n2;
  return el * 6 * n2 * n + (int64_t)(k * 6 + f) * n2 + ij;
}
void gll_rule(int N, std::vector<double>* xi, std::vector<double>* w);
void deriv_matrix(int N, const std::vector<double>& xi, std::vector<double>* D);
int64_t lattice_gid(const HostPlan& p, int64_t e_global, int i, int j, int k);
bool slot_masked(const HostPlan& p, int64_t e_global, int i, int j, int k);

}  // namespace sem
