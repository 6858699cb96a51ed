// Host planner: GLL space (Eq. 7), derivative matrix and
// the entity-based gather-scatter plan (P:L107 global numbering, P:L202
// local/shared classification, P:L231 injective/non-injective split) for a
// conforming hexahedral box mesh partitioned into contiguous element ranges.
//
// Runs once per sem_setup; nothing here is on the timed path.  The plan is
// per entity (face/edge/vertex of the element lattice), not per slot: the
// device kernels derive each point's slots from the entity's incidence bases,
// so no per-slot index array is streamed from HBM.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "sem_internal.h"

namespace sem {

// -------------------------------------------------------------- GLL rule
// Legendre L_k and the GLL polynomial q(x) = L_{N+1}(x) - L_{N-1}(x), whose
// roots are exactly the N+1 GLL points (q = -(2N+1)/(N(N+1)) (1-x^2) L_N'),
// with q'(x) = (2N+1) L_N(x).  Newton in long double, seeded at the
// Chebyshev-Gauss-Lobatto points.
static void legendre3(int N, long double x, long double* Lnm1, long double* Ln,
                      long double* Lnp1) {
  long double a = 1.0L, b = x;  // L_0, L_1
  if (N == 0) { *Lnm1 = 0; *Ln = a; *Lnp1 = b; return; }
  for (int k = 1; k < N; k++) {
    long double c = ((2 * k + 1) * x * b - k * a) / (k + 1);
    a = b; b = c;
  }
  // a = L_{N-1}, b = L_N
  long double c = ((2 * N + 1) * x * b - N * a) / (N + 1);
  *Lnm1 = a; *Ln = b; *Lnp1 = c;
}

void gll_rule(int N, std::vector<double>* xi, std::vector<double>* w) {
  const int n = N + 1;
  std::vector<long double> x(n);
  x[0] = -1.0L;
  x[N] = 1.0L;
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int i = 1; i < N; i++) {
    long double t = -cosl(pi * i / N);
    for (int it = 0; it < 100; it++) {
      long double lm, l, lp;
      legendre3(N, t, &lm, &l, &lp);
      long double dt = (lp - lm) / ((2 * N + 1) * l);
      t -= dt;
      if (fabsl(dt) < 1e-19L) break;
    }
    x[i] = t;
  }
  for (int i = 0; i < n / 2; i++) {   // exact antisymmetry xi_{N-i} = -xi_i
    long double s = 0.5L * (x[N - i] - x[i]);
    x[i] = -s;
    x[N - i] = s;
  }
  if (N % 2 == 0) x[N / 2] = 0.0L;
  xi->resize(n);
  w->resize(n);
  for (int i = 0; i < n; i++) {
    long double lm, l, lp;
    legendre3(N, x[i], &lm, &l, &lp);
    (*xi)[i] = (double)x[i];
    (*w)[i] = (double)(2.0L / ((long double)N * (N + 1) * l * l));
  }
}

// D_ij = l_j'(xi_i) = L_N(xi_i) / (L_N(xi_j)(xi_i - xi_j)), i != j;
// D_ii = -sum_{j != i} D_ij (reading Q2), evaluated in long double.
void deriv_matrix(int N, const std::vector<double>& xi, std::vector<double>* D) {
  const int n = N + 1;
  std::vector<long double> L(n);
  for (int i = 0; i < n; i++) {
    long double lm, l, lp;
    legendre3(N, (long double)xi[i], &lm, &l, &lp);
    L[i] = l;
  }
  D->assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; i++) {
    long double s = 0.0L;
    for (int j = 0; j < n; j++) {
      if (i == j) continue;
      long double d = L[i] / (L[j] * ((long double)xi[i] - (long double)xi[j]));
      (*D)[(size_t)i * n + j] = (double)d;
      s += d;
    }
    (*D)[(size_t)i * n + i] = (double)(-s);
  }
}

// -------------------------------------------------------------- lattice
static inline void ecoords(const sem_mesh& m, int64_t e, int64_t c[3]) {
  c[0] = e % m.ex;
  c[1] = (e / m.ex) % m.ey;
  c[2] = e / ((int64_t)m.ex * m.ey);
}

// insertion sort of the <= 8 incidences / ranks of one entity (std::sort's
// 16-element insertion threshold trips -Warray-bounds on the fixed arrays)
template <typename T, typename Less>
static void small_sort(T* a, int n, Less less) {
  for (int x = 1; x < n; x++) {
    T v = a[x];
    int y = x - 1;
    while (y >= 0 && less(v, a[y])) {
      a[y + 1] = a[y];
      y--;
    }
    a[y + 1] = v;
  }
}

int64_t lattice_gid(const HostPlan& p, int64_t e, int i, int j, int k) {
  int64_t c[3];
  ecoords(p.m, e, c);
  const int64_t Ea[3] = {p.m.ex, p.m.ey, p.m.ez};
  const int loc[3] = {i, j, k};
  int64_t L[3], Nl[3];
  for (int a = 0; a < 3; a++) {
    int64_t len = Ea[a] * p.N;
    L[a] = c[a] * p.N + loc[a];
    if (p.m.periodic[a]) L[a] %= len;
    Nl[a] = len + (p.m.periodic[a] ? 0 : 1);
  }
  return L[0] + Nl[0] * (L[1] + Nl[1] * L[2]);
}

bool slot_masked(const HostPlan& p, int64_t e, int i, int j, int k) {
  int64_t c[3];
  ecoords(p.m, e, c);
  const int64_t Ea[3] = {p.m.ex, p.m.ey, p.m.ez};
  const int loc[3] = {i, j, k};
  for (int a = 0; a < 3; a++) {
    if (p.m.periodic[a]) continue;
    int64_t L = c[a] * p.N + loc[a];
    if (L == 0 || L == Ea[a] * p.N) return true;
  }
  return false;
}

// per-element incidence table of the local entities (sem_internal.h kGu*): each
// incidence's element and sub-entity follow from its base (element block +
// the fixed coordinates; the spanning ones are 0 in a base)
void build_gu_table(const HostPlan& p, std::vector<int32_t>* tab) {
  const int n = p.n, N = p.N;
  const int64_t n3 = p.n3;
  tab->assign((size_t)p.nloc * kGuInts, -1);
  int32_t* T = tab->data();
  auto split = [&](int32_t b, int64_t* el, int c[3]) {
    *el = b / n3;
    const int64_t r = b - *el * n3;
    c[0] = (int)(r % n);
    c[1] = (int)((r / n) % n);
    c[2] = (int)(r / ((int64_t)n * n));
  };
  int c[3];
  int64_t el;
  for (int64_t f = 0; f < p.nF; f++) {
    const int a = p.f_axis[f];
    for (int t = 0; t < 2; t++) {
      split(p.f_base[2 * f + t], &el, c);
      int32_t* r = T + el * kGuInts + 2 * (2 * a + (c[a] == N));
      r[0] = p.f_base[2 * f];
      r[1] = p.f_base[2 * f + 1];
    }
  }
  for (int64_t e = 0; e < p.nEd; e++) {
    const int a = p.e_axis[e];
    const int lo = a == 0 ? 1 : 0, hi = a == 2 ? 1 : 2;
    for (int t = 0; t < p.e_nin[e]; t++) {
      split(p.e_base[4 * e + t], &el, c);
      int32_t* r = T + el * kGuInts + kGuEdge + 4 * (4 * a + (c[lo] == N) + 2 * (c[hi] == N));
      for (int x = 0; x < 4; x++) r[x] = p.e_base[4 * e + x];
    }
  }
  for (int64_t v = 0; v < p.nV; v++) {
    for (int t = 0; t < p.v_nin[v]; t++) {
      split(p.v_base[8 * v + t], &el, c);
      int32_t* r = T + el * kGuInts + kGuVert + 8 * ((c[0] == N) + 2 * (c[1] == N) + 4 * (c[2] == N));
      for (int x = 0; x < 8; x++) r[x] = p.v_base[8 * v + x];
    }
  }
}

// local entity id (0..25) <-> kind / sides
//   faces 0..5: 2a + side_a ; edges 6..17: 6 + 4a + s_f1 + 2 s_f2 (f1<f2 the
//   fixed axes) ; vertices 18..25: 18 + sx + 2 sy + 4 sz
struct LocalEnt {
  int cls;        // CLS_FACE/EDGE/VERT
  int axis;       // face normal axis / edge axis / -1
  bool fixed[3];  // axes on which the entity sits at a vertex plane
  int side[3];    // 0 / 1 on fixed axes
};

static LocalEnt decode(int lid) {
  LocalEnt L{};
  if (lid < 6) {
    L.cls = CLS_FACE;
    L.axis = lid / 2;
    for (int a = 0; a < 3; a++) L.fixed[a] = (a == L.axis);
    L.side[L.axis] = lid % 2;
  } else if (lid < 18) {
    int q = lid - 6;
    L.cls = CLS_EDGE;
    L.axis = q / 4;
    int f1 = L.axis == 0 ? 1 : 0, f2 = L.axis == 2 ? 1 : 2;
    for (int a = 0; a < 3; a++) L.fixed[a] = (a != L.axis);
    L.side[f1] = q % 2;
    L.side[f2] = (q / 2) % 2;
  } else {
    int q = lid - 18;
    L.cls = CLS_VERT;
    L.axis = -1;
    for (int a = 0; a < 3; a++) { L.fixed[a] = true; L.side[a] = (q >> a) & 1; }
  }
  return L;
}

static int encode(const LocalEnt& L) {
  if (L.cls == CLS_FACE) return 2 * L.axis + L.side[L.axis];
  if (L.cls == CLS_EDGE) {
    int f1 = L.axis == 0 ? 1 : 0, f2 = L.axis == 2 ? 1 : 2;
    return 6 + 4 * L.axis + L.side[f1] + 2 * L.side[f2];
  }
  return 18 + L.side[0] + 2 * L.side[1] + 4 * L.side[2];
}

struct Inc {
  int64_t e;   // global element
  int lid;     // local entity id in that element
  int side[3];
};

// all elements incident to the entity (element c, local entity L)
static int incidences(const sem_mesh& m, const int64_t c[3], const LocalEnt& L, Inc out[8],
                      bool* masked) {
  const int64_t Ea[3] = {m.ex, m.ey, m.ez};
  int64_t cand[3][2];
  int cside[3][2];
  int ncand[3];
  *masked = false;
  for (int a = 0; a < 3; a++) {
    if (!L.fixed[a]) {
      cand[a][0] = c[a]; cside[a][0] = 0; ncand[a] = 1;
      continue;
    }
    int64_t v = c[a] + L.side[a];  // vertex-lattice coordinate
    ncand[a] = 0;
    if (m.periodic[a]) {
      v %= Ea[a];
      cand[a][ncand[a]] = (v - 1 + Ea[a]) % Ea[a]; cside[a][ncand[a]++] = 1;
      cand[a][ncand[a]] = v;                       cside[a][ncand[a]++] = 0;
    } else {
      if (v == 0 || v == Ea[a]) *masked = true;
      if (v - 1 >= 0) { cand[a][ncand[a]] = v - 1; cside[a][ncand[a]++] = 1; }
      if (v < Ea[a]) { cand[a][ncand[a]] = v; cside[a][ncand[a]++] = 0; }
    }
  }
  int cnt = 0;
  for (int x = 0; x < ncand[0]; x++)
    for (int y = 0; y < ncand[1]; y++)
      for (int z = 0; z < ncand[2]; z++) {
        Inc& I = out[cnt++];
        I.e = cand[0][x] + Ea[0] * (cand[1][y] + Ea[1] * cand[2][z]);
        LocalEnt K = L;
        K.side[0] = L.fixed[0] ? cside[0][x] : 0;
        K.side[1] = L.fixed[1] ? cside[1][y] : 0;
        K.side[2] = L.fixed[2] ? cside[2][z] : 0;
        for (int a = 0; a < 3; a++) I.side[a] = K.side[a];
        I.lid = encode(K);
      }
  small_sort(out, cnt, [](const Inc& a, const Inc& b) { return a.e < b.e; });
  return cnt;
}

static inline int64_t rank_lo(int64_t E, int P, int r) { return (int64_t)r * E / P; }

static int rank_of(int64_t E, int P, int64_t e) {
  int r = (int)((e * P) / E);
  if (r >= P) r = P - 1;
  while (r + 1 < P && rank_lo(E, P, r + 1) <= e) r++;
  while (r > 0 && rank_lo(E, P, r) > e) r--;
  return r;
}

// slot offset (within the element block) of point p of an entity incidence
static inline int64_t point_offset(const LocalEnt& L, int N, int n, int p, int loc[3]) {
  const int64_t stride[3] = {1, n, (int64_t)n * n};
  int64_t off = 0;
  int s1 = -1, s2 = -1;
  for (int a = 0; a < 3; a++) {
    if (L.fixed[a]) {
      loc[a] = L.side[a] * N;
    } else if (s1 < 0) {
      s1 = a;
    } else {
      s2 = a;
    }
  }
  if (L.cls == CLS_FACE) {
    loc[s1] = 1 + p % (N - 1);
    loc[s2] = 1 + p / (N - 1);
  } else if (L.cls == CLS_EDGE) {
    loc[s1] = 1 + p;
  }
  for (int a = 0; a < 3; a++) off += loc[a] * stride[a];
  return off;
}

int build_plan(const sem_mesh* mp, int N, HostPlan* P) {
  const sem_mesh& m = *mp;
  if (N < 1 || N > 11) { set_error("N must be in 1..11"); return SEM_EINVAL; }
  if (m.ex < 1 || m.ey < 1 || m.ez < 1) { set_error("element counts must be >= 1"); return SEM_EINVAL; }
  const int32_t Ea[3] = {m.ex, m.ey, m.ez};
  for (int a = 0; a < 3; a++)
    if (m.periodic[a] && Ea[a] < 2) {
      set_error("a periodic axis needs >= 2 elements (reading Q7)");
      return SEM_EINVAL;
    }
  if (!(m.x1 > m.x0) || !(m.y1 > m.y0) || !(m.z1 > m.z0)) {
    set_error("degenerate box extents");
    return SEM_EINVAL;
  }
  const int64_t E = (int64_t)m.ex * m.ey * m.ez;
  if (m.nranks < 1 || m.rank < 0 || m.rank >= m.nranks || m.nranks > E) {
    set_error("bad rank/nranks (need 0 <= rank < nranks <= E)");
    return SEM_EINVAL;
  }
  HostPlan& p = *P;
  p.m = m;
  p.N = N;
  p.n = N + 1;
  p.n3 = (int64_t)p.n * p.n * p.n;
  p.E = E;
  p.rank = m.rank;
  p.nranks = m.nranks;
  p.e_lo = rank_lo(E, m.nranks, m.rank);
  p.e_hi = rank_lo(E, m.nranks, m.rank + 1);
  p.nloc = p.e_hi - p.e_lo;
  p.n_local = p.nloc * p.n3;
  if (p.n_local > INT32_MAX) { set_error("more than 2^31 slots on one rank"); return SEM_EINVAL; }
  p.fully_periodic = m.periodic[0] && m.periodic[1] && m.periodic[2];
  {
    int64_t g = 1;
    for (int a = 0; a < 3; a++) g *= (int64_t)Ea[a] * N + (m.periodic[a] ? 0 : 1);
    p.nglob = g;
  }
  gll_rule(N, &p.xi, &p.w);
  deriv_matrix(N, p.xi, &p.D);

  const int n = p.n;
  const int64_t n3 = p.n3;
  const int nf_pts = (N - 1) * (N - 1), ne_pts = N - 1;
  p.bmask.assign(p.nloc, 0);
  std::vector<uint8_t> boundary(p.nloc, 0);

  struct SP {
    int64_t gid;
    int nloc;
    int32_t slot[8];
    int mult;
    int mask;
    int nr;
    int ranks[8];
  };
  std::vector<SP> sps;

  p.f_start.assign(p.nloc + 1, 0);
  p.e_start.assign(p.nloc + 1, 0);
  p.v_start.assign(p.nloc + 1, 0);
  for (int64_t el = 0; el < p.nloc; el++) {
    const int64_t e = p.e_lo + el;
    p.f_start[el] = (int32_t)p.nF;
    p.e_start[el] = (int32_t)p.nEd;
    p.v_start[el] = (int32_t)p.nV;
    int64_t c[3];
    ecoords(m, e, c);
    uint8_t bm = 0;
    for (int a = 0; a < 3; a++) {
      if (m.periodic[a]) continue;
      if (c[a] == 0) bm |= (uint8_t)(1u << (2 * a));
      if (c[a] == Ea[a] - 1) bm |= (uint8_t)(1u << (2 * a + 1));
    }
    p.bmask[el] = bm;
    for (int lid = 0; lid < kRefsPerElem; lid++) {
      LocalEnt L = decode(lid);
      if (L.cls == CLS_FACE && N < 2) continue;   // no face interior points at N=1
      if (L.cls == CLS_EDGE && N < 2) continue;
      Inc inc[8];
      bool masked;
      int nin = incidences(m, c, L, inc, &masked);
      if (nin < 2) continue;
      // creator: the smallest LOCAL incident element
      int64_t creator = -1;
      int nloc_inc = 0;
      for (int t = 0; t < nin; t++)
        if (inc[t].e >= p.e_lo && inc[t].e < p.e_hi) {
          if (creator < 0) creator = inc[t].e;
          nloc_inc++;
        }
      if (creator != e) continue;
      if (nloc_inc == nin) {
        // local entity
        int32_t base[8];
        for (int t = 0; t < nin; t++) {
          LocalEnt K = decode(inc[t].lid);
          int loc[3];
          int64_t off0 = point_offset(K, N, n, 0, loc);
          // base = element block + fixed-axis offset; point_offset(p) - point_offset(0)
          // is identical across incidences, so store base = block + offset(p=0) minus
          // the spanning part of p=0
          int64_t span0 = 0;
          const int64_t stride[3] = {1, n, (int64_t)n * n};
          for (int a = 0; a < 3; a++)
            if (!K.fixed[a]) span0 += stride[a];   // spanning coords start at 1
          base[t] = (int32_t)((inc[t].e - p.e_lo) * n3 + off0 - span0);
        }
        if (L.cls == CLS_FACE) {
          p.nF++;
          p.f_base.push_back(base[0]);
          p.f_base.push_back(base[1]);
          p.f_axis.push_back((uint8_t)L.axis);
        } else if (L.cls == CLS_EDGE) {
          p.nEd++;
          for (int t = 0; t < 4; t++) p.e_base.push_back(t < nin ? base[t] : -1);
          p.e_axis.push_back((uint8_t)L.axis);
          p.e_nin.push_back((uint8_t)nin);
          p.e_mask.push_back(masked ? 1 : 0);
        } else {
          p.nV++;
          for (int t = 0; t < 8; t++) p.v_base.push_back(t < nin ? base[t] : -1);
          p.v_nin.push_back((uint8_t)nin);
          p.v_mask.push_back(masked ? 1 : 0);
        }
      } else {
        // shared with other ranks: one record per point
        int npts = L.cls == CLS_FACE ? nf_pts : (L.cls == CLS_EDGE ? ne_pts : 1);
        int ranks[8], nr = 0;
        for (int t = 0; t < nin; t++) {
          int r = rank_of(E, m.nranks, inc[t].e);
          bool seen = false;
          for (int q = 0; q < nr; q++) seen |= (ranks[q] == r);
          if (!seen) ranks[nr++] = r;
          if (inc[t].e >= p.e_lo && inc[t].e < p.e_hi) boundary[inc[t].e - p.e_lo] = 1;
        }
        small_sort(ranks, nr, [](int a, int b) { return a < b; });
        for (int pt = 0; pt < npts; pt++) {
          SP s{};
          s.nloc = 0;
          s.mult = nin;
          s.mask = masked ? 1 : 0;
          s.nr = nr;
          for (int q = 0; q < nr; q++) s.ranks[q] = ranks[q];
          for (int t = 0; t < 8; t++) s.slot[t] = -1;
          for (int t = 0; t < nin; t++) {
            LocalEnt K = decode(inc[t].lid);
            int loc[3];
            int64_t off = point_offset(K, N, n, pt, loc);
            if (t == 0) s.gid = lattice_gid(p, inc[t].e, loc[0], loc[1], loc[2]);
            if (inc[t].e >= p.e_lo && inc[t].e < p.e_hi)
              s.slot[s.nloc++] = (int32_t)((inc[t].e - p.e_lo) * n3 + off);
          }
          sps.push_back(s);
        }
      }
    }
  }

  p.f_start[p.nloc] = (int32_t)p.nF;
  p.e_start[p.nloc] = (int32_t)p.nEd;
  p.v_start[p.nloc] = (int32_t)p.nV;

  // shared points: ascending gid; per neighbour buffers in that order
  std::sort(sps.begin(), sps.end(), [](const SP& a, const SP& b) { return a.gid < b.gid; });
  p.nS = (int64_t)sps.size();
  std::vector<int64_t> cnt(m.nranks, 0);
  for (const SP& s : sps)
    for (int q = 0; q < s.nr; q++)
      if (s.ranks[q] != m.rank) cnt[s.ranks[q]]++;
  std::vector<int64_t> off(m.nranks, 0);
  p.nbuf = 0;
  for (int q = 0; q < m.nranks; q++)
    if (cnt[q] > 0) {
      p.nbr_rank.push_back(q);
      p.nbr_off.push_back(p.nbuf);
      p.nbr_cnt.push_back(cnt[q]);
      off[q] = p.nbuf;
      p.nbuf += cnt[q];
    }
  p.s_gid.resize(p.nS);
  p.s_slot.assign(8 * p.nS, -1);
  p.s_off.assign(8 * p.nS, 0);
  p.s_nloc.resize(p.nS);
  p.s_mult.resize(p.nS);
  p.s_mask.resize(p.nS);
  p.s_nr.resize(p.nS);
  p.s_rank.assign(8 * p.nS, -1);
  std::vector<int64_t> pos(m.nranks, 0);
  for (int64_t i = 0; i < p.nS; i++) {
    const SP& s = sps[i];
    p.s_gid[i] = s.gid;
    p.s_nloc[i] = (uint8_t)s.nloc;
    p.s_mult[i] = (uint8_t)s.mult;
    p.s_mask[i] = (uint8_t)s.mask;
    p.s_nr[i] = (uint8_t)s.nr;
    for (int t = 0; t < 8; t++) p.s_slot[t * p.nS + i] = s.slot[t];
    for (int q = 0; q < s.nr; q++) {
      int r = s.ranks[q];
      p.s_rank[q * p.nS + i] = (int8_t)r;
      p.s_off[q * p.nS + i] = (r == m.rank) ? -1 : (int32_t)(off[r] + pos[r]++);
    }
  }

  // Alg. 1 overlap ranges: boundary elements first, interior in between
  if (m.nranks == 1 || p.nS == 0) {
    p.ilo = 0; p.ihi = p.nloc;
  } else {
    int64_t a = 0;
    while (a < p.nloc && boundary[a]) a++;
    int64_t b = p.nloc;
    while (b > a && boundary[b - 1]) b--;
    bool ok = a < b;
    for (int64_t el = a; ok && el < b; el++)
      if (boundary[el]) ok = false;
    if (ok) {
      p.b0lo = 0; p.b0hi = a; p.b1lo = b; p.b1hi = p.nloc; p.ilo = a; p.ihi = b;
    } else {
      p.b0lo = 0; p.b0hi = p.nloc; p.ilo = p.ihi = 0;
    }
  }
  return SEM_OK;
}

}  // namespace sem

// ------------------------------------------------------------------ C ABI:
// host-only planner (CPU tests)
struct sem_plan {
  sem::HostPlan p;
};

extern "C" int sem_plan_create(const sem_mesh* m, int N, sem_plan** out) {
  if (!m || !out) { sem::set_error("NULL argument"); return SEM_EINVAL; }
  *out = nullptr;
  sem_plan* h = new (std::nothrow) sem_plan();
  if (!h) return SEM_ENOMEM;
  int st = sem::build_plan(m, N, &h->p);
  if (st != SEM_OK) { delete h; return st; }
  *out = h;
  return SEM_OK;
}

sem_plan* sem::plan_wrap(const sem::HostPlan& p) {
  sem_plan* h = new (std::nothrow) sem_plan();
  if (h) h->p = p;
  return h;
}

extern "C" int sem_plan_destroy(sem_plan* h) {
  delete h;
  return SEM_OK;
}

// expand entities into (pairs, segments); slot lists are ascending
static void expand(const sem::HostPlan& p, std::vector<std::vector<int64_t>>* groups) {
  const int N = p.N, n = p.n;
  const int64_t stride[3] = {1, n, (int64_t)n * n};
  auto span_axes = [&](int cls, int axis, int* s1, int* s2) {
    *s1 = *s2 = -1;
    for (int a = 0; a < 3; a++) {
      bool fixed = cls == sem::CLS_VERT || (cls == sem::CLS_FACE ? a == axis : a != axis);
      if (!fixed) { if (*s1 < 0) *s1 = a; else *s2 = a; }
    }
  };
  for (int64_t f = 0; f < p.nF; f++) {
    int s1, s2;
    span_axes(sem::CLS_FACE, p.f_axis[f], &s1, &s2);
    for (int pt = 0; pt < (N - 1) * (N - 1); pt++) {
      int64_t o = (1 + pt % (N - 1)) * stride[s1] + (1 + pt / (N - 1)) * stride[s2];
      groups->push_back({p.f_base[2 * f] + o, p.f_base[2 * f + 1] + o});
    }
  }
  for (int64_t e = 0; e < p.nEd; e++) {
    int s1, s2;
    span_axes(sem::CLS_EDGE, p.e_axis[e], &s1, &s2);
    for (int pt = 0; pt < N - 1; pt++) {
      std::vector<int64_t> g;
      for (int t = 0; t < p.e_nin[e]; t++) g.push_back(p.e_base[4 * e + t] + (1 + pt) * stride[s1]);
      groups->push_back(g);
    }
  }
  for (int64_t v = 0; v < p.nV; v++) {
    std::vector<int64_t> g;
    for (int t = 0; t < p.v_nin[v]; t++) g.push_back(p.v_base[8 * v + t]);
    groups->push_back(g);
  }
  for (int64_t s = 0; s < p.nS; s++) {
    if (p.s_nloc[s] < 2) continue;
    std::vector<int64_t> g;
    for (int t = 0; t < p.s_nloc[s]; t++) g.push_back(p.s_slot[t * p.nS + s]);
    groups->push_back(g);
  }
}

extern "C" int sem_plan_sizes(const sem_plan* h, int64_t* n_local, int64_t* npairs,
                              int64_t* nseg, int64_t* nsegslots, int32_t* n_nbr) {
  if (!h) return SEM_EINVAL;
  const sem::HostPlan& p = h->p;
  std::vector<std::vector<int64_t>> g;
  expand(p, &g);
  int64_t np = 0, ns = 0, nss = 0;
  for (auto& v : g) {
    if (v.size() == 2) np++;
    else { ns++; nss += (int64_t)v.size(); }
  }
  if (n_local) *n_local = p.n_local;
  if (npairs) *npairs = np;
  if (nseg) *nseg = ns;
  if (nsegslots) *nsegslots = nss;
  if (n_nbr) *n_nbr = (int32_t)p.nbr_rank.size();
  return SEM_OK;
}

extern "C" int sem_plan_slots(const sem_plan* h, int64_t* gid, int64_t* mult, int64_t* mask) {
  if (!h) return SEM_EINVAL;
  const sem::HostPlan& p = h->p;
  const int n = p.n;
  for (int64_t el = 0; el < p.nloc; el++)
    for (int k = 0; k < n; k++)
      for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++) {
          int64_t l = el * p.n3 + i + n * j + (int64_t)n * n * k;
          if (gid) gid[l] = sem::lattice_gid(p, p.e_lo + el, i, j, k);
          if (mask) mask[l] = sem::slot_masked(p, p.e_lo + el, i, j, k) ? 1 : 0;
          if (mult) mult[l] = 1;
        }
  if (!p.x_mult.empty()) {   // live export: the device's multiplicity and mask
    for (int64_t l = 0; l < p.n_local; l++) {
      if (mult) mult[l] = p.x_mult[l];
      if (mask) mask[l] = p.x_mask[l];
    }
    return SEM_OK;
  }
  if (mult) {
    std::vector<std::vector<int64_t>> g;
    expand(p, &g);
    for (auto& v : g)
      for (int64_t s : v) mult[s] = (int64_t)v.size();
    for (int64_t s = 0; s < p.nS; s++)
      for (int t = 0; t < p.s_nloc[s]; t++) mult[p.s_slot[t * p.nS + s]] = p.s_mult[s];
  }
  return SEM_OK;
}

extern "C" int sem_plan_pairs(const sem_plan* h, int64_t* pairs, int64_t* seg_off,
                              int64_t* seg_slot) {
  if (!h) return SEM_EINVAL;
  std::vector<std::vector<int64_t>> g;
  expand(h->p, &g);
  std::vector<std::pair<int64_t, int64_t>> pr;
  std::vector<const std::vector<int64_t>*> sg;
  for (auto& v : g) {
    if (v.size() == 2) pr.push_back({std::min(v[0], v[1]), std::max(v[0], v[1])});
    else sg.push_back(&v);
  }
  std::sort(pr.begin(), pr.end());
  std::sort(sg.begin(), sg.end(), [](const std::vector<int64_t>* a,
                                     const std::vector<int64_t>* b) { return (*a)[0] < (*b)[0]; });
  for (size_t i = 0; i < pr.size(); i++) {
    pairs[2 * i] = pr[i].first;
    pairs[2 * i + 1] = pr[i].second;
  }
  seg_off[0] = 0;
  for (size_t s = 0; s < sg.size(); s++) {
    for (size_t t = 0; t < sg[s]->size(); t++) seg_slot[seg_off[s] + t] = (*sg[s])[t];
    seg_off[s + 1] = seg_off[s] + (int64_t)sg[s]->size();
  }
  return SEM_OK;
}

extern "C" int sem_plan_neighbors(const sem_plan* h, int32_t* ranks, int64_t* counts) {
  if (!h) return SEM_EINVAL;
  for (size_t q = 0; q < h->p.nbr_rank.size(); q++) {
    ranks[q] = h->p.nbr_rank[q];
    counts[q] = h->p.nbr_cnt[q];
  }
  return SEM_OK;
}

extern "C" int sem_plan_shared(const sem_plan* h, int32_t q, int64_t* gids) {
  if (!h) return SEM_EINVAL;
  const sem::HostPlan& p = h->p;
  int64_t c = 0;
  for (int64_t s = 0; s < p.nS; s++)
    for (int t = 0; t < p.s_nr[s]; t++)
      if (p.s_off[t * p.nS + s] >= 0) {
        // the t-th involved rank: recover it from the neighbour buffer index
        int64_t o = p.s_off[t * p.nS + s];
        for (size_t k = 0; k < p.nbr_rank.size(); k++)
          if (p.nbr_rank[k] == q && o >= p.nbr_off[k] && o < p.nbr_off[k] + p.nbr_cnt[k])
            gids[c++] = p.s_gid[s];
      }
  return SEM_OK;
}

extern "C" int sem_plan_space(const sem_plan* h, double* xi, double* w, double* D) {
  if (!h || !xi || !w || !D) return SEM_EINVAL;
  std::memcpy(xi, h->p.xi.data(), h->p.xi.size() * sizeof(double));
  std::memcpy(w, h->p.w.data(), h->p.w.size() * sizeof(double));
  std::memcpy(D, h->p.D.data(), h->p.D.size() * sizeof(double));
  return SEM_OK;
}
