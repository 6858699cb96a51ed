"""Pins of the oracle's restarted GMRES and solution projection (SURVEY 8(f)
NEXT-3; Table 2 "GMRES ... Projections 20") against
quantities built independently of the oracle's routines: the dense assembled
operator (explicit Kronecker element matrices + explicit Q), numpy least
squares over an explicitly built Krylov space, and the algebraic properties
SPEC lists for the projection space."""
import numpy as np
import pytest

import oracle as O
from sem_inputs import CONFIGS, f_sin, random_field, tgv_box, unit_box, u_sin
from test_oracle_pins import _dense_assembled


def _reduced(o):
    """Dense assembled A on the unmasked unique DOFs, the unique->slot map."""
    Q, A = _dense_assembled(o)
    gid, mask = o.get_int("gid"), o.get_int("mask")
    mg = np.zeros(o.nglob, dtype=bool)
    mg[gid] = mask.astype(bool)
    keep = ~mg
    first = np.unique(gid, return_index=True)[1]   # one slot per unique DOF
    return Q, A[np.ix_(keep, keep)], keep, gid, first


def _to_slots(o, keep, gid, yk):
    yg = np.zeros(o.nglob)
    yg[keep] = yk
    return yg[gid]


@pytest.mark.parametrize("spec,N", [(CONFIGS["C1"][0], 3), (unit_box(2, 2, 3, periodic=(1, 0, 0)), 3)])
def test_gmres_dense_solve(spec, N):
    o = O.Oracle(spec, N)
    Q, A, keep, gid, first = _reduced(o)
    b = o.rhs(f_sin(o.get("X"), o.get("Y"), o.get("Z")))
    xk = np.linalg.solve(A, b[first][keep])
    for restart in (30, 5):
        r = o.gmres(b, 1e-12, 2000, restart)
        assert r["status"] == 0
        np.testing.assert_allclose(r["x"], _to_slots(o, keep, gid, xk), rtol=0,
                                   atol=1e-10 * np.abs(xk).max())
        assert r["res_true"] < 1e-11


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8])
def test_gmres_iterate_is_the_krylov_minimiser(k):
    """After k iterations (no restart), x_k = M^-1 K_k y with K_k = span{b, (A M^-1) b,
    ...} minimising ||b - A x||_2 over the unique DOFs (c-weighted norm of slot
    vectors = Euclidean norm on unique DOFs) -- numpy least squares."""
    o = O.Oracle(tgv_box(2, 2, 2, deform=1), 3)
    Q, A, keep, gid, first = _reduced(o)
    Minv = 1.0 / np.diag(A)
    bk = random_field(o.nglob, seed=5)[keep]
    b = _to_slots(o, keep, gid, bk)
    # explicit Krylov basis, orthonormalised with numpy QR for conditioning
    K = np.zeros((len(bk), k))
    v = bk.copy()
    for i in range(k):
        K[:, i] = v
        v = A @ (Minv * v)
    K, _ = np.linalg.qr(K)
    y = np.linalg.lstsq(A @ (Minv[:, None] * K), bk, rcond=None)[0]
    xk = Minv * (K @ y)
    r = o.gmres(b, 0.0, k, k + 3)
    assert r["iters"] == k
    np.testing.assert_allclose(r["x"], _to_slots(o, keep, gid, xk), rtol=0,
                               atol=1e-9 * np.abs(xk).max())
    # the Arnoldi residual estimate equals the true least-squares residual
    assert abs(r["hist"][k] - np.linalg.norm(bk - A @ xk)) <= 1e-9 * np.linalg.norm(bk)


def test_gmres_residual_monotone_within_cycles():
    o = O.Oracle(tgv_box(3, 3, 3, deform=1), 4)
    b = o.rhs(random_field(o.nslots, seed=9))
    restart = 6
    r = o.gmres(b, 1e-12, 60, restart)
    h = r["hist"]
    for c0 in range(0, len(h) - 1, restart):
        seg = h[c0:c0 + restart + 1]
        assert all(seg[i + 1] <= seg[i] * (1 + 1e-13) for i in range(len(seg) - 1))


def test_projection_empty_and_exact_deflation():
    o = O.Oracle(CONFIGS["C1"][0], 3)
    Q, A, keep, gid, first = _reduced(o)
    p = o.proj(20)
    b = o.rhs(f_sin(o.get("X"), o.get("Y"), o.get("Z")))
    xb, bd = p.project(b)
    assert np.all(xb == 0) and np.array_equal(bd, b)
    # store z1 (any continuous field), then b = A z1 is deflated exactly
    z1k = random_field(o.nglob, seed=3)[keep]
    assert p.update(_to_slots(o, keep, gid, z1k))
    b1 = _to_slots(o, keep, gid, A @ z1k)
    xb, bd = p.project(b1)
    assert np.abs(bd).max() <= 1e-10 * np.abs(b1).max()
    np.testing.assert_allclose(xb, _to_slots(o, keep, gid, z1k), rtol=0, atol=1e-10 * np.abs(z1k).max())


def test_projection_gram_identity_and_reset():
    o = O.Oracle(tgv_box(2, 2, 3, deform=1), 3)
    Q, A, keep, gid, first = _reduced(o)
    m = 6
    p = o.proj(m)
    for i in range(m):
        assert p.update(_to_slots(o, keep, gid, random_field(o.nglob, seed=20 + i)[keep]))
        G = p.gram()
        assert G.shape == (i + 1, i + 1)
        np.testing.assert_allclose(G, np.eye(i + 1), rtol=0, atol=1e-8)
    # independent check of A-orthonormality with the dense operator
    assert p.size == m
    # m+1-th update: reset, keep the latest only
    p.update(_to_slots(o, keep, gid, random_field(o.nglob, seed=99)[keep]))
    assert p.size == 1
    # a direction already in the space is skipped
    p2 = o.proj(4)
    x = _to_slots(o, keep, gid, random_field(o.nglob, seed=7)[keep])
    assert p2.update(x) and not p2.update(2.0 * x) and p2.size == 1


def test_projection_pipeline_repeated_and_sequence():
    """Repeated identical solves need 0 or 1 Krylov iterations; on a slowly
    varying sequence of right-hand sides the projection cuts the iterations."""
    o = O.Oracle(CONFIGS["C1"][0], 4)
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    p = o.proj(20)
    b = o.rhs(f_sin(X, Y, Z))
    r1 = p.solve(b, 1e-10, 500)
    r2 = p.solve(b, 1e-10, 500)
    assert r1["status"] == 0 and r2["iters"] <= 1
    Q, A, keep, gid, first = _reduced(o)
    np.testing.assert_allclose(r2["x"], _to_slots(o, keep, gid, np.linalg.solve(A, b[first][keep])),
                               rtol=0, atol=1e-9)
    pp = o.proj(20)
    it_proj, it_plain = [], []
    for t in range(6):
        f = u_sin(X, Y, Z) * (1.0 + 0.05 * t) + 0.02 * t * np.sin(2 * np.pi * X) * np.sin(np.pi * Y) * np.sin(np.pi * Z)
        bt = o.rhs(f)
        it_proj.append(pp.solve(bt, 1e-10, 500)["iters"])
        it_plain.append(o.gmres(bt, 1e-10, 500)["iters"])
    assert sum(it_proj[1:]) < sum(it_plain[1:]), (it_proj, it_plain)


def test_arnoldi_basis_orthonormal_where_single_pass_mgs_is_not():
    """Reading Q25 pin: the oracle's Arnoldi step (modified Gram-Schmidt applied
    twice) keeps V^T C V = I to ~1e-13 on a case where the same Arnoldi process
    with ONE MGS pass -- written out here in numpy on the dense assembled
    operator -- loses orthogonality by orders of magnitude more (the Krylov
    space nearly captures an invariant subspace, kappa(K) ~ 1/eps^(1/2)).  Also
    A M^-1 V_m = V_{m+1} H (the Arnoldi relation) to rounding."""
    o = O.Oracle(tgv_box(2, 2, 2, deform=1), 3)
    Q, A, keep, gid, first = _reduced(o)
    Minv = 1.0 / np.diag(A)
    bk = random_field(o.nglob, seed=11)[keep]
    m = 40
    V, H = o.arnoldi(_to_slots(o, keep, gid, bk), m)
    c = 1.0 / o.get_int("mult")
    gram = (V * c) @ V.T
    loss2 = np.abs(gram - np.eye(m + 1)).max()
    # single-pass MGS on the unique DOFs (Euclidean = the c-weighted slot norm)
    W = np.zeros((len(bk), m + 1))
    W[:, 0] = bk / np.linalg.norm(bk)
    for j in range(m):
        w = A @ (Minv * W[:, j])
        for i in range(j + 1):
            w -= (w @ W[:, i]) * W[:, i]
        W[:, j + 1] = w / np.linalg.norm(w)
    loss1 = np.abs(W.T @ W - np.eye(m + 1)).max()
    assert loss2 <= 1e-12, loss2
    assert loss1 >= 1e3 * loss2, (loss1, loss2)
    # Arnoldi relation on the unique DOFs: A M^-1 V_m = V_{m+1} H
    Vk = np.stack([v[first][keep] for v in V], axis=1)
    R = A @ (Minv[:, None] * Vk[:, :m]) - Vk @ H
    assert np.abs(R).max() <= 1e-11 * np.abs(A).max()
