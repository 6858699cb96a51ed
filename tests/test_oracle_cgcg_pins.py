"""Pins of the oracle's single-reduction (Chronopoulos-Gear) Jacobi PCG
(the lower-ranked variant after NEXT-1..4; "pipelined
Krylov solvers"; reading Q34): the dense solve of the assembled system, and
the exact-arithmetic identity with the standard PCG recurrences (a different
algorithm in the oracle: two reductions per iteration), iterate by iterate."""
import numpy as np
import pytest

import oracle as O
from sem_inputs import CONFIGS, f_sin, f_tgv, tgv_box, unit_box
from test_oracle_pins import _dense_assembled


def _rhs(o):
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    return o.rhs((f_tgv if all(o.spec.periodic) else f_sin)(X, Y, Z))


def test_cgcg_dense_solve():
    spec, N = CONFIGS["C1"]
    o = O.Oracle(spec, N)
    _, A = _dense_assembled(o)
    gid, mask = o.get_int("gid"), o.get_int("mask")
    mg = np.zeros(o.nglob, dtype=bool)
    mg[gid] = mask.astype(bool)
    first = np.unique(gid, return_index=True)[1]
    b = _rhs(o)
    xg = np.zeros(o.nglob)
    xg[~mg] = np.linalg.solve(A[np.ix_(~mg, ~mg)], b[first][~mg])
    r = o.cgcg(b, 1e-12, 500)
    assert r["status"] == 0
    np.testing.assert_allclose(r["x"], xg[gid], rtol=0, atol=1e-12 * np.abs(xg).max())
    assert r["res_true"] <= 1e-11


@pytest.mark.parametrize("spec,N", [(CONFIGS["C1"][0], 3), (tgv_box(4, 4, 4), 7),
                                    (tgv_box(3, 3, 3, deform=1), 5),
                                    (unit_box(3, 2, 4, periodic=(1, 0, 0)), 4)])
def test_cgcg_equals_pcg(spec, N):
    """Same Krylov iterates as the two-reduction PCG: iteration count within 1,
    residual history and solution equal up to rounding."""
    o = O.Oracle(spec, N)
    b = _rhs(o)
    a = o.pcg(b, 1e-10, 3000)
    g = o.cgcg(b, 1e-10, 3000)
    assert g["status"] == 0 and abs(a["iters"] - g["iters"]) <= 1
    k = min(len(a["hist"]), len(g["hist"]), 20)
    np.testing.assert_allclose(g["hist"][:k], a["hist"][:k], rtol=1e-8, atol=1e-12 * a["hist"][0])
    assert np.abs(g["x"] - a["x"]).max() <= 1e-9


def test_cgcg_edge_cases():
    spec, N = CONFIGS["C1"]
    o = O.Oracle(spec, N)
    b = np.zeros(o.nslots)
    r = o.cgcg(b, 1e-10, 10)
    assert r["status"] == 0 and r["iters"] == 0 and np.all(r["x"] == 0.0)
    r = o.cgcg(_rhs(o), 1e-10, 0)
    assert r["status"] == 1 and r["iters"] == 0
