"""Pins of the oracle's Helmholtz operator h1 A + h2 B (
P:L257 "a Helmholtz equation for each velocity component") against
things other than itself: explicit dense assembly (Kronecker element matrices,
explicit Q, diagonal mass), quadrature of 1 (domain volume), SPD-ness at the
paper's velocity-solve coefficients, a dense solve, and spectral convergence to
a manufactured solution of (-h1 lap + h2) u = f."""
import math

import numpy as np
import pytest

import oracle as O
from sem_inputs import CONFIGS, f_sin, random_field, tgv_box, u_sin, unit_box
from test_oracle_pins import dense_element_matrix, explicit_Q


def _dense_helm(o, h1, h2):
    """Q^T (h1 A_L + h2 diag(B_L)) Q, and the element-level matrix H_L."""
    n3 = o.n ** 3
    D, G, B = o.get("D"), o.get("G"), o.get("B")
    Q = explicit_Q(o.get_int("gid"), o.nglob).toarray()
    HL = np.zeros((o.nslots, o.nslots))
    for e in range(o.E):
        s = slice(e * n3, (e + 1) * n3)
        HL[s, s] = h1 * dense_element_matrix(D, G[e * 6 * n3:(e + 1) * 6 * n3])
    HL += h2 * np.diag(B)
    return Q, HL, Q.T @ HL @ Q


@pytest.mark.parametrize("spec,N", [(CONFIGS["C1"][0], 3), (tgv_box(2, 2, 2, deform=1), 3),
                                    (unit_box(2, 2, 3, periodic=(1, 0, 0)), 2)])
@pytest.mark.parametrize("h1,h2", [(1.0, 0.0), (0.7, 3.0), (0.0, 1.0)])
def test_helm_apply_and_jacobi_vs_dense(spec, N, h1, h2):
    o = O.Oracle(spec, N)
    Q, HL, H = _dense_helm(o, h1, h2)
    mask = o.get_int("mask").astype(bool)
    u = random_field(o.nslots, 17)                      # discontinuous local vector
    ref = Q @ (Q.T @ (HL @ u))
    ref[mask] = 0.0
    got = o.helm_apply(h1, h2, u)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    gid = o.get_int("gid")
    mg = np.zeros(o.nglob, dtype=bool)
    mg[gid] = mask
    dg = np.diag(H)
    expect = np.where(mg, 0.0, 1.0 / np.where(mg, 1.0, dg))[gid]
    np.testing.assert_allclose(o.helm_dinv(h1, h2), expect, rtol=1e-13)


def test_helm_mass_quadrature_of_one():
    """h1=0, h2=1 on the constant field -> assembled mass weights whose
    unique-DOF sum is the domain volume ((2 pi)^3; the deformed map is a bijection)."""
    o = O.Oracle(tgv_box(3, 2, 3, deform=1), 5)
    w = o.helm_apply(0.0, 1.0, np.ones(o.nslots))
    assert abs(o.dot_c(np.ones(o.nslots), w) - (2 * math.pi) ** 3) < 1e-10


def test_helm_spd_velocity_coefficients():
    """h1 = 1/Re, h2 = b0/dt with Re=1600, dt=5e-4 (b0 = 1): u^T H u > 0
    for 100 random continuous u on a 2^3 mesh."""
    o = O.Oracle(tgv_box(2, 2, 2, deform=1), 4)
    gid = o.get_int("gid")
    h1, h2 = 1.0 / 1600.0, 1.0 / 5e-4
    rng = np.random.default_rng(3)
    for _ in range(100):
        u = rng.uniform(-1, 1, o.nglob)[gid]
        assert o.dot_c(u, o.helm_apply(h1, h2, u)) > 0.0


def test_helm_pcg_matches_dense_solve():
    spec, N = CONFIGS["C1"]
    o = O.Oracle(spec, N)
    h1, h2 = 1.0, 10.0
    Q, _, H = _dense_helm(o, h1, h2)
    gid, mask = o.get_int("gid"), o.get_int("mask")
    mg = np.zeros(o.nglob, dtype=bool)
    mg[gid] = mask.astype(bool)
    keep = ~mg
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    b = o.rhs_mass(f_sin(X, Y, Z))
    bg = b[np.unique(gid, return_index=True)[1]]
    xg = np.zeros(o.nglob)
    xg[keep] = np.linalg.solve(H[np.ix_(keep, keep)], bg[keep])
    r = o.helm_pcg(h1, h2, b, 1e-13, 1000)
    assert r["status"] == 0 and r["iters"] <= int(keep.sum())
    np.testing.assert_allclose(r["x"], xg[gid], rtol=0, atol=1e-12 * np.abs(xg).max())
    assert r["res_true"] < 1e-12


def test_helm_periodic_is_nonsingular():
    """h2 > 0 removes the constant null space: the fully periodic system with a
    nonzero-mean right-hand side converges (the Poisson one would not)."""
    o = O.Oracle(tgv_box(3, 3, 3), 4)
    b = o.rhs_mass(np.ones(o.nslots))
    r = o.helm_pcg(1.0, 2.0, b, 1e-12, 2000)
    assert r["status"] == 0
    np.testing.assert_allclose(r["x"], 0.5, rtol=0, atol=1e-10)   # H 1 = h2 B 1  ->  x = 1/h2


def test_helm_spectral_convergence():
    """(-h1 lap + h2) u* = f with u* = sin(pi x) sin(pi y) sin(pi z) on the Dirichlet
    unit box: f = (3 pi^2 h1 + h2) u*; error ratio > 10 per dN = 2, < 1e-8 at N = 8."""
    spec, _ = CONFIGS["C1"]
    h1, h2 = 0.5, 4.0
    errs = []
    for N in (2, 4, 6, 8):
        o = O.Oracle(spec, N)
        X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
        f = (3 * math.pi ** 2 * h1 + h2) * u_sin(X, Y, Z)
        r = o.helm_pcg(h1, h2, o.rhs_mass(f), 1e-14, 5000)
        errs.append(np.abs(r["x"] - u_sin(X, Y, Z)).max())
    assert all(errs[i] / errs[i + 1] > 10 for i in range(3)), errs
    assert errs[-1] < 1e-8
