"""Pins of the oracle's two-level additive overlapping Schwarz preconditioner
("M0^-1 = R0^T A0^-1 R0 + sum_k R_k^T A~_k^-1 R_k",
"the coarse grid (on linear elements) is solved for using ... few (~10) CG
iterations"; readings Q28-Q32 in DESIGN.md) against quantities built without
the oracle's Schwarz routines:

* the dense assembled operator (explicit Kronecker element matrices + explicit
  Q, `_dense_assembled`): on Cartesian meshes the separable local operator must
  be exactly its principal submatrix on the element's unmasked nodes;
* hat functions on the element-vertex lattice evaluated at the physical node
  coordinates (the prolongation R0^T) and the dense N = 1 operator (A0);
* numpy dense solves and pseudo-inverses for the complete two-level operator;
* textbook properties: one-element exactness, symmetry, positivity, and
  convergence to the dense solution.
"""
import numpy as np
import pytest

import oracle as O
from sem_inputs import MeshSpec, f_sin, f_tgv, random_field, tgv_box, unit_box
from test_oracle_pins import _dense_assembled


def _unique_maps(o):
    gid, mask = o.get_int("gid"), o.get_int("mask")
    mg = np.zeros(o.nglob, dtype=bool)
    mg[gid] = mask.astype(bool)
    first = np.unique(gid, return_index=True)[1]
    return gid, mg, first


CART = [
    (MeshSpec(3, 3, 4, periodic=(1, 1, 1)), 3),
    (unit_box(2, 2, 2), 3),
    (MeshSpec(3, 2, 3, x1=2.0, y1=0.5, z1=1.5, periodic=(1, 0, 1)), 2),
    (MeshSpec(2, 3, 2, x1=0.7, z1=1.3), 4),
]


@pytest.mark.parametrize("spec,N", CART)
def test_local_operator_is_principal_submatrix(spec, N):
    """Q28: on Cartesian meshes A~_e = A[element nodes, element nodes] (unmasked)."""
    o = O.Oracle(spec, N)
    s = o.schwarz(10)
    _, A = _dense_assembled(o)
    gid, mg, _ = _unique_maps(o)
    n3 = o.n ** 3
    scale = np.abs(A).max()
    for e in range(o.E):
        g = gid[e * n3:(e + 1) * n3]
        keep = ~mg[g]
        At = s.local_matrix(e)
        ref = A[np.ix_(g, g)]
        np.testing.assert_allclose(At[np.ix_(keep, keep)], ref[np.ix_(keep, keep)], rtol=0,
                                   atol=1e-13 * scale)
        assert np.all(At[~keep, :] == 0.0) and np.all(At[:, ~keep] == 0.0)


def _hat_prolongation(o, o0):
    """R0^T as a dense (nglob x nglob0) matrix: trilinear hat functions of the
    coarse vertices (element-vertex lattice), evaluated at the fine nodes'
    physical coordinates; periodic axes use the wrapped distance."""
    spec = o.spec
    ext = np.array([spec.x1 - spec.x0, spec.y1 - spec.y0, spec.z1 - spec.z0])
    h = ext / np.array([spec.ex, spec.ey, spec.ez])
    gid, _, first = _unique_maps(o)
    gid0, _, first0 = _unique_maps(o0)
    Xf = np.stack([o.get(a)[first] for a in "XYZ"], 1)
    Xc = np.stack([o0.get(a)[first0] for a in "XYZ"], 1)
    d = np.abs(Xf[:, None, :] - Xc[None, :, :])
    for a in range(3):
        if spec.periodic[a]:
            d[:, :, a] = np.minimum(d[:, :, a], ext[a] - d[:, :, a])
    return np.prod(np.clip(1.0 - d / h, 0.0, None), axis=2)


@pytest.mark.parametrize("spec,N", CART[:3])
def test_two_level_operator_vs_dense(spec, N):
    """z = W^1/2 sum_e R_e^T A_e^-1 R_e W^1/2 r + P A0^+ P^T r with every piece
    built densely (A_e principal submatrices, P hat functions, A0 dense N=1)."""
    o = O.Oracle(spec, N)
    o0 = O.Oracle(spec, 1)
    s = o.schwarz(coarse_iters=2000)    # coarse CG run to convergence
    Q, A = _dense_assembled(o)
    _, A0 = _dense_assembled(o0)
    gid, mg, first = _unique_maps(o)
    _, mg0, _ = _unique_maps(o0)
    n3 = o.n ** 3
    mult = np.bincount(gid, minlength=o.nglob).astype(float)
    w = np.sqrt(1.0 / mult)
    r = o.mask_apply(o.gs(random_field(o.nslots, 11)))     # an assembled residual
    if all(spec.periodic):
        r = r - o.dot_c(r, np.ones_like(r)) / o.dot_c(np.ones_like(r), np.ones_like(r))
    rg = r[first]
    zl = np.zeros(o.nglob)
    for e in range(o.E):
        g = gid[e * n3:(e + 1) * n3]
        k = g[~mg[g]]
        zl[k] += np.linalg.solve(A[np.ix_(k, k)], (w * rg)[k])
    zl *= w
    P = _hat_prolongation(o, o0)
    P[:, mg0] = 0.0
    A0r = A0[np.ix_(~mg0, ~mg0)]
    y0 = np.zeros(o0.nglob)
    y0[~mg0] = np.linalg.pinv(A0r) @ (P.T @ rg)[~mg0]
    zc = P @ y0
    zc[mg] = 0.0
    for which, ref in ((1, zl), (2, zc), (3, zl + zc)):
        z = s.apply(r, which)
        np.testing.assert_allclose(z, ref[gid], rtol=0, atol=1e-10 * np.abs(ref).max())


def test_single_element_is_exact():
    """one Dirichlet element, the local solve is A^-1 and the coarse
    space is empty: PCG and GMRES converge in one iteration."""
    o = O.Oracle(unit_box(1, 1, 1), 5)
    s = o.schwarz(10)
    b = o.rhs(f_sin(o.get("X"), o.get("Y"), o.get("Z")))
    for r in (s.pcg(b, 1e-11, 10), s.gmres(b, 1e-11, 10)):
        assert r["status"] == 0 and r["iters"] == 1, r["iters"]


def _rand_range(o, seed):
    v = o.mask_apply(o.gs(random_field(o.nslots, seed) * o.get("c")))
    if all(o.spec.periodic):
        one = np.ones_like(v)
        v = v - o.dot_c(v, one) / o.dot_c(one, one)
    return v


@pytest.mark.parametrize("spec,N", [(tgv_box(3, 3, 3, deform=1), 4), (unit_box(3, 2, 2), 5)])
def test_symmetric_positive(spec, N):
    """v^T M v > 0; with an exact coarse solve M is symmetric."""
    o = O.Oracle(spec, N)
    s = o.schwarz(coarse_iters=2000)
    for q in range(4):
        u, v = _rand_range(o, 2 * q), _rand_range(o, 2 * q + 1)
        Mu, Mv = s.apply(u), s.apply(v)
        a, b = o.dot_c(Mu, v), o.dot_c(u, Mv)
        assert abs(a - b) <= 1e-11 * (abs(a) + abs(b) + 1e-300) + 1e-14
        assert o.dot_c(Mu, u) > 0.0


def test_pcg_gmres_match_dense_solve():
    spec, N = unit_box(2, 3, 2), 3
    o = O.Oracle(spec, N)
    s = o.schwarz(10)
    _, A = _dense_assembled(o)
    gid, mg, first = _unique_maps(o)
    b = o.rhs(f_sin(o.get("X"), o.get("Y"), o.get("Z")))
    x = np.zeros(o.nglob)
    x[~mg] = np.linalg.solve(A[np.ix_(~mg, ~mg)], b[first][~mg])
    for r in (s.pcg(b, 1e-12, 500), s.gmres(b, 1e-12, 500, 30), s.gmres(b, 1e-12, 500, 4)):
        assert r["status"] == 0
        np.testing.assert_allclose(r["x"], x[gid], rtol=0, atol=1e-10 * np.abs(x).max())
        assert r["res_true"] <= 1e-11


@pytest.mark.parametrize("spec,N", [(tgv_box(4, 4, 4), 7), (tgv_box(3, 3, 3, deform=1), 5)])
def test_fewer_iterations_than_jacobi(spec, N):
    """S:L441 / S:L754: on the periodic pressure Poisson the two-level Schwarz
    needs fewer iterations than Jacobi (PCG and GMRES), same solution."""
    o = O.Oracle(spec, N)
    s = o.schwarz(10)
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    b = o.rhs(f_tgv(X, Y, Z))
    rj = o.pcg(b, 1e-10, 2000)
    gj = o.gmres(b, 1e-10, 2000, 30)
    rs = s.pcg(b, 1e-10, 500)
    gs = s.gmres(b, 1e-10, 500, 30)
    assert rs["status"] == 0 and gs["status"] == 0
    assert rs["iters"] < rj["iters"] and gs["iters"] < gj["iters"], (rs["iters"], rj["iters"],
                                                                     gs["iters"], gj["iters"])
    Bm = o.get("B")

    def dm(v):
        return v - (Bm * v).sum() / Bm.sum()
    np.testing.assert_allclose(dm(rs["x"]), dm(rj["x"]), rtol=0, atol=1e-8)
    np.testing.assert_allclose(dm(gs["x"]), dm(rj["x"]), rtol=0, atol=1e-8)


def test_projection_pipeline_with_schwarz():
    """P:L257 pressure pipeline (projection + GMRES + Schwarz): each solution
    solves its system; cumulative iterations over slowly varying right-hand
    sides do not exceed those without projection."""
    spec, N = tgv_box(3, 3, 3), 4
    o = O.Oracle(spec, N)
    s = o.schwarz(10)
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    b0 = o.rhs(f_tgv(X, Y, Z))
    db = o.rhs(np.sin(X) * np.cos(2 * Y))
    pr = o.proj(20)
    pr.set_schwarz(s)
    it_p = it_0 = 0
    for k in range(6):
        b = b0 + 0.01 * k * db + 1e-4 * o.rhs(random_field(o.nslots, 40 + k))
        r = pr.solve(b, 1e-10, 500)
        assert r["status"] == 0
        res = b - o.apply(r["x"])
        assert np.sqrt(o.dot_c(res, res)) <= 1e-9
        it_p += r["iters"]
        it_0 += s.gmres(b, 1e-10, 500)["iters"]
    assert it_p <= it_0, (it_p, it_0)
