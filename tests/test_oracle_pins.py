"""Pins for the CPU oracle against what the paper and the mathematics fix.

Nothing here compares the oracle with itself: every expected value is a
closed form, an mpmath computation, a dense/explicit-matrix construction in
numpy/scipy, a brute-force enumeration, or a SPEC.md/paper worked example
(tests/golden/*.json, each with its citation).  A plausible mistake (dropped
term, wrong sign or index, transposed operand) fails at least one of them.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from sem_inputs import (CONFIGS, MeshSpec, f_sin, f_tgv, p_tgv, random_field, tgv_box,
                        u_sin, unit_box)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- helpers
def kron_ops(D):
    """Reference-element derivative matrices for slot p = i + n j + n^2 k."""
    n = D.shape[0]
    I = np.eye(n)
    Dr = np.kron(I, np.kron(I, D))
    Ds = np.kron(I, np.kron(D, I))
    Dt = np.kron(D, np.kron(I, I))
    return Dr, Ds, Dt


def dense_element_matrix(D, Ge):
    """A^e = D^T G^e D (Eq. 9), built as explicit matrices."""
    n3 = D.shape[0] ** 3
    Dr, Ds, Dt = kron_ops(D)
    g = [np.diag(Ge[f * n3:(f + 1) * n3]) for f in range(6)]  # rr ss tt rs rt st
    Ops = [Dr, Ds, Dt]
    Gm = [[g[0], g[3], g[4]], [g[3], g[1], g[5]], [g[4], g[5], g[2]]]
    A = np.zeros((n3, n3))
    for a in range(3):
        for b in range(3):
            A += Ops[a].T @ Gm[a][b] @ Ops[b]
    return A


def explicit_Q(gid, nglob):
    n = len(gid)
    return sp.csr_matrix((np.ones(n), (np.arange(n), gid)), shape=(n, nglob))


def mp_gll_nodes(N, dps=50):
    """Roots of (1 - x^2) L_N'(x) at 50 digits, independent of the oracle."""
    mpmath.mp.dps = dps
    coeffs = mpmath.taylor(lambda x: mpmath.legendre(N, x), 0, N)
    dcoef = [k * coeffs[k] for k in range(1, N + 1)]  # ascending coefficients of L_N'
    if N == 1:
        inner = []
    else:
        inner = sorted(mpmath.polyroots(dcoef[::-1], maxsteps=200, extraprec=200))
    return [mpmath.mpf(-1)] + [mpmath.re(r) for r in inner] + [mpmath.mpf(1)]


# ---------------------------------------------------------------- c1 GLL
def test_gll_closed_forms():
    g = _gold("gll_closed_forms.json")["rules"]
    env = {"sqrt": math.sqrt}
    for Ns, rule in g.items():
        N = int(Ns)
        xi, w = O.gll(N)
        xe = [eval(s, env) for s in rule["nodes"]]
        we = [eval(s.replace("/", "*1.0/"), env) for s in rule["weights"]]
        np.testing.assert_allclose(xi, xe, rtol=0, atol=2e-16)
        np.testing.assert_allclose(w, we, rtol=2e-15, atol=0)


@pytest.mark.parametrize("N", [5, 7, 9, 11])
def test_gll_vs_mpmath(N):
    xi, w = O.gll(N)
    ref = mp_gll_nodes(N)
    np.testing.assert_allclose(xi, [float(r) for r in ref], rtol=0, atol=2e-15)
    wref = [2 / (N * (N + 1) * mpmath.legendre(N, r) ** 2) for r in ref]
    np.testing.assert_allclose(w, [float(v) for v in wref], rtol=3e-15)
    assert abs(w.sum() - 2.0) < 1e-14


@pytest.mark.parametrize("N", list(range(1, 12)))
def test_gll_quadrature_exactness(N):
    xi, w = O.gll(N)
    for k in range(0, 2 * N):
        exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
        assert abs(np.dot(w, xi ** k) - exact) < 1e-14, (N, k)
    # degree 2N is NOT integrated exactly by an (N+1)-point Lobatto rule
    assert abs(np.dot(w, xi ** (2 * N)) - 2.0 / (2 * N + 1)) > 1e-9


def test_appendix_a_n7():
    # SURVEY Appendix A (mpmath 50 digits); 1/28 end weight is exact: 2/(N(N+1)).
    xi, w = O.gll(7)
    assert w[0] == pytest.approx(1.0 / 28.0, rel=1e-15)
    assert xi[1] == pytest.approx(-0.87174014850960662, abs=2e-16)
    assert w[3] == pytest.approx(0.41245879465870388, rel=2e-15)


# ---------------------------------------------------------------- c2 D
def test_deriv_n1_golden():
    g = _gold("spec_examples.json")["deriv_N1"]["D"]
    np.testing.assert_array_equal(O.deriv(1), np.array(g))


@pytest.mark.parametrize("N", list(range(1, 12)))
def test_deriv_polynomial_exactness(N):
    xi, _ = O.gll(N)
    D = O.deriv(N, xi)
    assert np.abs(D @ np.ones(N + 1)).max() < 1e-13 * N * N
    for k in range(1, N + 1):
        np.testing.assert_allclose(D @ xi ** k, k * xi ** (k - 1), rtol=0, atol=5e-13 * N * N)
    # closed-form corner entries and centro-antisymmetry D_ij = -D_{N-i,N-j}
    assert D[0, 0] == pytest.approx(-N * (N + 1) / 4.0, rel=1e-13)
    assert D[N, N] == pytest.approx(N * (N + 1) / 4.0, rel=1e-13)
    np.testing.assert_allclose(D, -D[::-1, ::-1], atol=1e-12 * N * N)


@pytest.mark.parametrize("N", [3, 7])
def test_deriv_vs_mpmath_lagrange(N):
    """l_j'(xi_i) by differentiating the Lagrange product formula at 50 digits."""
    nodes = mp_gll_nodes(N)
    n = N + 1
    ref = np.zeros((n, n))
    for j in range(n):
        def lj(x, j=j):
            p = mpmath.mpf(1)
            for m in range(n):
                if m != j:
                    p *= (x - nodes[m]) / (nodes[j] - nodes[m])
            return p
        for i in range(n):
            ref[i, j] = float(mpmath.diff(lj, nodes[i]))
    np.testing.assert_allclose(O.deriv(N), ref, rtol=0, atol=5e-14 * n * n)


# ---------------------------------------------------------------- c9 Ax kernel
@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_ax_raw_matches_dense_kronecker(N):
    """Random D, random G, random u: sum-factorised Eq. 9 == explicit D^T G D."""
    rng = np.random.default_rng(100 + N)
    n = N + 1
    E = 3
    D = rng.standard_normal((n, n))
    G = rng.standard_normal(E * 6 * n ** 3)
    u = rng.standard_normal(E * n ** 3)
    w = O.ax_raw(E, N, D, G, u)
    for e in range(E):
        A = dense_element_matrix(D, G[e * 6 * n ** 3:(e + 1) * 6 * n ** 3])
        np.testing.assert_allclose(w[e * n ** 3:(e + 1) * n ** 3], A @ u[e * n ** 3:(e + 1) * n ** 3],
                                   rtol=0, atol=1e-12 * np.abs(A).sum(1).max())


@pytest.mark.parametrize("N", [1, 2, 4])
def test_diag_raw_matches_dense(N):
    rng = np.random.default_rng(200 + N)
    n = N + 1
    D = rng.standard_normal((n, n))
    G = rng.standard_normal(2 * 6 * n ** 3)
    d = O.diag_raw(2, N, D, G)
    for e in range(2):
        A = dense_element_matrix(D, G[e * 6 * n ** 3:(e + 1) * 6 * n ** 3])
        np.testing.assert_allclose(d[e * n ** 3:(e + 1) * n ** 3], np.diag(A), rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- c4-c5 geometry
def test_cartesian_geometry_closed_form():
    spec = MeshSpec(3, 2, 2, 0.0, 1.5, -1.0, 1.0, 0.0, 0.5, periodic=(0, 1, 0))
    N = 4
    o = O.Oracle(spec, N)
    n = N + 1
    xi, w = O.gll(N)
    hx, hy, hz = 1.5 / 3, 2.0 / 2, 0.5 / 2
    W = np.einsum("k,j,i->kji", w, w, w).ravel()
    G = o.get("G").reshape(o.E, 6, n ** 3)
    B = o.get("B").reshape(o.E, n ** 3)
    for e in range(o.E):
        np.testing.assert_allclose(G[e, 0], W * hy * hz / (2 * hx), rtol=1e-13)
        np.testing.assert_allclose(G[e, 1], W * hx * hz / (2 * hy), rtol=1e-13)
        np.testing.assert_allclose(G[e, 2], W * hx * hy / (2 * hz), rtol=1e-13)
        assert np.abs(G[e, 3:]).max() < 1e-13 * G[e, 0].max()
        np.testing.assert_allclose(B[e], W * hx * hy * hz / 8, rtol=1e-13)
    assert B.sum() == pytest.approx(1.5 * 2.0 * 0.5, rel=1e-14)


def test_unit_cube_mass_spec():
    # unit cube single element, B = w_i w_j w_k / 8
    o = O.Oracle(unit_box(1, 1, 1), 2)
    _, w = O.gll(2)
    np.testing.assert_allclose(o.get("B"), np.einsum("k,j,i->kji", w, w, w).ravel() / 8, rtol=1e-14)


def test_deformed_geometry_invariants():
    spec = tgv_box(4, 4, 4, deform=1)
    N = 7
    o = O.Oracle(spec, N)
    n3 = (N + 1) ** 3
    B = o.get("B")
    assert B.sum() == pytest.approx((2 * math.pi) ** 3, rel=1e-6)
    G = o.get("G").reshape(o.E, 6, n3)
    # per point G symmetric positive definite
    M = np.stack([G[:, 0], G[:, 3], G[:, 4], G[:, 3], G[:, 1], G[:, 5], G[:, 4], G[:, 5], G[:, 2]],
                 -1).reshape(-1, 3, 3)
    assert np.linalg.eigvalsh(M).min() > 0
    assert np.abs(G[:, 3:]).max() > 1e-3  # genuinely curvilinear
    # conformity: slots with the same gid coincide (modulo the period)
    gid = o.get_int("gid")
    for name in "XYZ":
        x = o.get(name)
        first = np.full(o.nglob, np.nan)
        first[gid[::-1]] = x[::-1]
        d = np.abs(np.mod(x - first[gid] + math.pi, 2 * math.pi) - math.pi)
        assert d.max() < 1e-13


def test_nonpositive_jacobian_rejected():
    spec = tgv_box(4, 4, 4, deform=1, amp=2.0)
    with pytest.raises(O.OracleError):
        O.Oracle(spec, 5)


# ---------------------------------------------------------------- c6-c8 numbering
def test_numbering_golden():
    g = _gold("spec_examples.json")["numbering"]["cases"]
    for case in g:
        o = O.Oracle(unit_box(*case["mesh"], periodic=case["periodic"]), case["N"])
        assert o.nglob == case["nglob"]
        assert len(np.unique(o.get_int("gid"))) == case["nglob"]


@pytest.mark.parametrize("mesh,per,N", [((2, 3, 2), (0, 0, 0), 3), ((3, 2, 2), (1, 0, 1), 2),
                                        ((2, 2, 2), (1, 1, 1), 4), ((4, 2, 3), (0, 1, 0), 1)])
def test_numbering_equals_coordinate_coincidence(mesh, per, N):
    """Brute force: equivalence classes of slots by coordinate coincidence."""
    spec = unit_box(*mesh, periodic=per)
    o = O.Oracle(spec, N)
    gid = o.get_int("gid")
    keys = []
    for name, p in zip("XYZ", per):
        x = o.get(name)
        if p:
            x = np.mod(x, 1.0)
            x[np.abs(x - 1.0) < 1e-12] = 0.0
        keys.append(np.round(x * 1e9).astype(np.int64))
    keys = np.stack(keys, 1)
    _, cls = np.unique(keys, axis=0, return_inverse=True)
    cls = cls.ravel()
    assert len(np.unique(cls)) == o.nglob
    # same partition: gid -> cls is a bijection
    pairs = np.unique(np.stack([gid, cls], 1), axis=0)
    assert len(pairs) == o.nglob
    expect = 1
    for a in range(3):
        expect *= mesh[a] * N + (0 if per[a] else 1)
    assert o.nglob == expect


def test_multiplicity_periodic_counts():
    g = _gold("spec_examples.json")["mult_periodic_N7"]["counts"]
    o = O.Oracle(tgv_box(2, 2, 2), 7)
    mult = o.get_int("mult")[: 8 ** 3]
    for m, cnt in g.items():
        assert int((mult == int(m)).sum()) == cnt
    assert np.sum(1.0 / o.get_int("mult")) == pytest.approx(o.nglob, rel=1e-14)


def test_c1_mask_golden():
    g = _gold("spec_examples.json")["c1_mask"]
    spec, N = CONFIGS["C1"]
    o = O.Oracle(spec, N)
    gid, mask = o.get_int("gid"), o.get_int("mask")
    assert o.nglob == g["nglob"]
    assert len(np.unique(gid[mask == 0])) == g["unmasked"]
    # mask is a property of the gid (consistent on all its slots)
    mg = np.zeros(o.nglob, dtype=np.int64)
    mg[gid] = mask
    assert np.array_equal(mg[gid], mask)


def test_partition_golden():
    g = _gold("spec_examples.json")["partition"]
    o = O.Oracle(unit_box(2, 2, 2), 1, nranks=g["P"])
    rank = o.get_int("rank").reshape(g["E"], -1)[:, 0]
    assert rank.tolist() == g["ranks"]


# ---------------------------------------------------------------- c10 gs
@pytest.mark.parametrize("spec,N", [(unit_box(3, 2, 2), 3), (tgv_box(3, 2, 4), 2),
                                    (tgv_box(2, 2, 2, deform=1), 4)])
def test_gs_equals_explicit_QQT(spec, N):
    o = O.Oracle(spec, N)
    Q = explicit_Q(o.get_int("gid"), o.nglob)
    u = random_field(o.nslots, seed=3)
    np.testing.assert_allclose(o.gs(u), Q @ (Q.T @ u), rtol=0, atol=1e-14)
    np.testing.assert_array_equal(o.gs(np.ones(o.nslots)), o.get_int("mult").astype(float))


def test_gs_partition_invariance():
    spec = tgv_box(4, 4, 4)
    u = random_field(tgv_box(4, 4, 4).n_slots(7), seed=5)
    ref = O.Oracle(spec, 7, 1).gs(u)
    for P in (2, 4, 8, 5):
        v = O.Oracle(spec, 7, P).gs(u)
        assert np.abs(v - ref).max() <= 1e-12 * np.abs(ref).max()


def test_gs_continuous_field_gives_mult_times_field():
    o = O.Oracle(tgv_box(3, 3, 2), 3)
    gid = o.get_int("gid")
    y = random_field(o.nglob, seed=9)
    u = y[gid]
    np.testing.assert_allclose(o.gs(u), o.get_int("mult") * u, rtol=1e-15)


def test_plan_structure():
    o = O.Oracle(tgv_box(2, 3, 2), 3)
    pairs, off, slots = o.plan()
    gid, mult = o.get_int("gid"), o.get_int("mult")
    assert np.all(pairs[:, 0] < pairs[:, 1])
    assert np.all(np.diff(pairs[:, 0]) > 0)
    assert np.all(gid[pairs[:, 0]] == gid[pairs[:, 1]])
    assert np.all(mult[pairs[:, 0]] == 2)
    firsts = slots[off[:-1]]
    assert np.all(np.diff(firsts) > 0)
    covered = np.concatenate([pairs.ravel(), slots])
    assert np.array_equal(np.sort(covered), np.flatnonzero(mult > 1))


def test_shared_lists():
    o = O.Oracle(tgv_box(2, 2, 4), 2, nranks=4)
    gid, rank = o.get_int("gid"), o.get_int("rank")
    for r in range(4):
        for q in range(4):
            if r == q:
                continue
            ref = np.intersect1d(gid[rank == r], gid[rank == q])
            assert np.array_equal(o.shared(r, q), ref)


# ---------------------------------------------------------------- c9-c11 operator
def test_ax_constant_is_zero_and_symmetric():
    o = O.Oracle(tgv_box(3, 2, 2, deform=1), 5)
    w = o.ax(np.full(o.nslots, 3.0))
    assert np.abs(w).max() < 1e-11
    gid = o.get_int("gid")
    u = random_field(o.nglob, 1)[gid]
    v = random_field(o.nglob, 2)[gid]
    a, b = o.dot_c(v, o.apply(u)), o.dot_c(u, o.apply(v))
    assert abs(a - b) < 1e-12 * abs(a)
    assert o.dot_c(u, o.apply(u)) > 0


@pytest.mark.parametrize("N", [3, 4, 7])
def test_exact_laplacian_identity_cartesian(N):
    """(A u)_g = B_g (-lap u)(x_g) at interior gids for degree <= N-1 polynomials."""
    spec = MeshSpec(2, 3, 2, 0.0, 1.0, 0.0, 1.5, -0.5, 0.5)
    o = O.Oracle(spec, N)
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    d = N - 1
    u = X ** d * Y ** max(d - 1, 0) + Z ** d + X * Y * Z ** max(d - 2, 0)
    lap = (d * (d - 1) * X ** max(d - 2, 0) * Y ** max(d - 1, 0)
           + (max(d - 1, 0) * max(d - 2, 0) * X ** d * Y ** max(d - 3, 0) if d >= 3 else 0)
           + d * (d - 1) * Z ** max(d - 2, 0)
           + (X * Y * max(d - 2, 0) * max(d - 3, 0) * Z ** max(d - 4, 0) if d >= 4 else 0))
    Au = o.gs(o.ax(u))
    Bg = o.gs(o.get("B"))
    interior = o.get_int("mask") == 0
    np.testing.assert_allclose(Au[interior], (-Bg * lap)[interior], rtol=0,
                               atol=1e-11 * np.abs(Bg * lap).max() + 1e-13)


def test_energy_identity_deformed():
    """u = x (isoparametric): u^T A_L u = integral |grad x|^2 = sum B exactly."""
    spec = MeshSpec(3, 2, 2, 0.0, 2 * math.pi, 0.0, 2 * math.pi, 0.0, 2 * math.pi, deform=1)
    o = O.Oracle(spec, 6)
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    vol = o.get("B").sum()
    for U in (X, Y, Z):
        assert np.dot(U, o.ax(U)) == pytest.approx(vol, rel=1e-12)
    # grad x . grad y = 0 exactly: pins the cross factors G_rs, G_rt, G_st
    for U, V in ((X, Y), (X, Z), (Y, Z)):
        assert abs(np.dot(U, o.ax(V))) < 1e-11 * vol


def _dense_assembled(o):
    n3 = o.n ** 3
    D, G = o.get("D"), o.get("G")
    Q = explicit_Q(o.get_int("gid"), o.nglob).toarray()
    AL = np.zeros((o.nslots, o.nslots))
    for e in range(o.E):
        AL[e * n3:(e + 1) * n3, e * n3:(e + 1) * n3] = dense_element_matrix(D, G[e * 6 * n3:(e + 1) * 6 * n3])
    return Q, Q.T @ AL @ Q


def test_operator_and_jacobi_vs_dense_assembly():
    spec, N = CONFIGS["C1"]
    o = O.Oracle(spec, N)
    Q, A = _dense_assembled(o)
    gid, mask = o.get_int("gid"), o.get_int("mask")
    mg = np.zeros(o.nglob, dtype=bool)
    mg[gid] = mask.astype(bool)
    keep = ~mg
    y = random_field(o.nglob, 4)
    y[mg] = 0
    ref = Q @ (np.where(keep, A @ y, 0.0))
    np.testing.assert_allclose(o.apply(Q @ y), ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    dinv = o.get("dinv")
    expect = np.where(keep, 1.0 / np.diag(A), 0.0)[gid]
    np.testing.assert_allclose(dinv, expect, rtol=1e-13)


def test_pcg_c1_matches_dense_solve():
    spec, N = CONFIGS["C1"]
    o = O.Oracle(spec, N)
    Q, A = _dense_assembled(o)
    gid, mask = o.get_int("gid"), o.get_int("mask")
    mg = np.zeros(o.nglob, dtype=bool)
    mg[gid] = mask.astype(bool)
    keep = ~mg
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    b = o.rhs(f_sin(X, Y, Z))
    bg = b[np.unique(gid, return_index=True)[1]]
    xk = np.linalg.solve(A[np.ix_(keep, keep)], bg[keep])
    xg = np.zeros(o.nglob)
    xg[keep] = xk
    r = o.pcg(b, 1e-13, 1000)
    assert r["status"] == 0
    assert r["iters"] <= int(keep.sum())
    np.testing.assert_allclose(r["x"], xg[gid], rtol=0, atol=1e-12 * np.abs(xg).max())
    assert r["res_true"] < 1e-12
    # A-norm error is monotone non-increasing (CG optimality)
    errs = []
    for k in range(1, r["iters"] + 1):
        xkk = o.pcg(b, 0.0, k)["x"]
        e = (xkk[np.unique(gid, return_index=True)[1]] - xg)[keep]
        errs.append(e @ A[np.ix_(keep, keep)] @ e)
    assert all(errs[i + 1] <= errs[i] * (1 + 1e-10) + 1e-30 for i in range(len(errs) - 1))


def test_spectral_convergence_dirichlet():
    """e_inf ratio > 10 per dN=2, < 1e-8 at N=8 (2^3 elements)."""
    spec, _ = CONFIGS["C1"]
    errs = []
    for N in (2, 4, 6, 8):
        o = O.Oracle(spec, N)
        X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
        r = o.pcg(o.rhs(f_sin(X, Y, Z)), 1e-14, 5000)
        errs.append(np.abs(r["x"] - u_sin(X, Y, Z)).max())
    assert all(errs[i] / errs[i + 1] > 10 for i in range(3)), errs
    assert errs[-1] < 1e-8


def test_tgv_pressure_periodic_convergence():
    spec = tgv_box(4, 4, 4)
    errs = []
    for N in (3, 5, 7):
        o = O.Oracle(spec, N)
        X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
        b = o.rhs(f_tgv(X, Y, Z))
        assert abs(o.dot_c(np.ones(o.nslots), b)) < 1e-13
        x = o.pcg(b, 1e-12, 5000)["x"]
        B = o.get("B")
        x = x - np.dot(B, x) / B.sum()          # reading Q18: mean removal
        errs.append(np.abs(x - p_tgv(X, Y, Z)).max())
    assert errs[0] / errs[1] > 10 and errs[1] / errs[2] > 10, errs
    assert errs[-1] < 1e-5


def _analytic_metric(spec, N, xi, w):
    """Closed-form G and B of the sinusoidal map (reading Q4) at the GLL nodes.

    x_a(r) = X_a + (L_a / 2 pi) amp sin(Xh) sin(Yh) sin(Zh), X_a linear in r_a
    with dX_a/dr_a = h_a / 2.  The exact Jacobian M_ab = dx_a/dr_b is written out
    from that formula (no derivative matrix, no interpolation), then
    G_ab = J w w w sum_m (M^-1)_am (M^-1)_bm and B = J w w w.
    """
    ex, ey, ez = spec.ex, spec.ey, spec.ez
    lo = np.array([spec.x0, spec.y0, spec.z0])
    L = np.array([spec.x1 - spec.x0, spec.y1 - spec.y0, spec.z1 - spec.z0])
    h = L / np.array([ex, ey, ez])
    amp = spec.deform_amp
    n = N + 1
    Gs, Bs = [], []
    for e in range(ex * ey * ez):
        eidx = np.array([e % ex, (e // ex) % ey, e // (ex * ey)])
        for k in range(n):
            for j in range(n):
                for i in range(n):
                    X = lo + h * (eidx + 0.5 * (np.array([xi[i], xi[j], xi[k]]) + 1.0))
                    th = 2 * math.pi * (X - lo) / L
                    s, c = np.sin(th), np.cos(th)
                    grad = amp * np.array([c[0] * s[1] * s[2], s[0] * c[1] * s[2],
                                           s[0] * s[1] * c[2]])   # d dlt / d theta_b
                    # dx_a/dX_b = delta_ab + (L_a/2pi) grad_b (2pi/L_b); dX_b/dr_b = h_b/2
                    M = (np.eye(3) + np.outer(L, grad / L)) * (h / 2)[None, :]
                    J = np.linalg.det(M)
                    R = np.linalg.inv(M)        # R[b][a] = dr_b/dx_a
                    wq = w[i] * w[j] * w[k]
                    g = J * wq * (R @ R.T)
                    Gs.append([g[0, 0], g[1, 1], g[2, 2], g[0, 1], g[0, 2], g[1, 2]])
                    Bs.append(J * wq)
    G = np.array(Gs).reshape(-1, n ** 3, 6).transpose(0, 2, 1)
    return G, np.array(Bs)


def test_deformed_metric_converges_to_closed_form():
    """Isoparametric G/B (D applied to the node coordinates) converge spectrally
    to the exact metric of the sinusoidal map.  Pins every deformed-mesh G
    entry, cross factors included: a transposed inverse, a dropped term of the
    cofactor expansion or a swapped factor pair leaves an O(1) error that does
    not decay with N."""
    spec = tgv_box(2, 2, 2, deform=1)
    errs = []
    for N in (3, 5, 7, 9, 11):
        o = O.Oracle(spec, N)
        xi, w = O.gll(N)
        Ga, Ba = _analytic_metric(spec, N, xi, w)
        G = o.get("G").reshape(o.E, 6, (N + 1) ** 3)
        B = o.get("B")
        # scale-free: error relative to the largest entry at this N
        eg = np.abs(G - Ga).max() / np.abs(Ga).max()
        eb = np.abs(B - Ba).max() / np.abs(Ba).max()
        errs.append(max(eg, eb))
    assert all(b < a / 5 for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-8, errs
