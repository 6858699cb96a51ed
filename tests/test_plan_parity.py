"""Integer / index parity of the product's host planner with the oracle:
global numbering, multiplicity, mask, injective pairs, non-injective segments
and per-neighbour shared lists must match BIT-EXACTLY.  Also the product's own
GLL rule and derivative matrix against the oracle's (independent code)."""
import numpy as np
import pytest

import oracle as O
import paper_2107_01243_b200 as sem
from sem_inputs import CONFIGS, tgv_box, unit_box

MESHES = [
    (unit_box(2, 2, 2), 3),
    (unit_box(3, 2, 4, periodic=(1, 0, 0)), 2),
    (unit_box(2, 3, 2, periodic=(0, 1, 1)), 4),
    (tgv_box(2, 2, 2), 1),
    (tgv_box(3, 4, 2), 5),
    (tgv_box(4, 4, 4, deform=1), 7),
    (unit_box(5, 3, 2), 6),
]


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2107_01243_b200 import build
    build.build()


@pytest.mark.parametrize("spec,N", MESHES)
def test_numbering_mult_mask_bit_exact(spec, N):
    o = O.Oracle(spec, N)
    p = sem.Plan(spec, N)
    gid, mult, mask = p.slots()
    assert np.array_equal(gid, o.get_int("gid"))
    assert np.array_equal(mult, o.get_int("mult"))
    assert np.array_equal(mask, o.get_int("mask"))


@pytest.mark.parametrize("spec,N", MESHES)
def test_gs_maps_bit_exact(spec, N):
    o = O.Oracle(spec, N)
    p = sem.Plan(spec, N)
    op, ooff, oslots = o.plan()
    pp, poff, pslots = p.pairs()
    assert np.array_equal(pp, op)
    assert np.array_equal(poff, ooff)
    assert np.array_equal(pslots, oslots)


@pytest.mark.parametrize("N", list(range(1, 12)))
def test_space_matches_oracle(N):
    p = sem.Plan(unit_box(2, 2, 2), N)
    xi, w, D = p.space()
    oxi, ow = O.gll(N)
    np.testing.assert_allclose(xi, oxi, rtol=0, atol=1e-15)
    np.testing.assert_allclose(w, ow, rtol=2e-15, atol=0)
    np.testing.assert_allclose(D, O.deriv(N, oxi), rtol=0, atol=4e-15 * N * N)


@pytest.mark.parametrize("spec,N,P", [(tgv_box(2, 2, 4), 3, 2), (tgv_box(2, 2, 4), 2, 4),
                                      (unit_box(3, 2, 5), 3, 3), (tgv_box(3, 3, 2), 2, 5),
                                      (tgv_box(4, 2, 2), 4, 8)])
def test_partition_neighbours_and_shared_lists(spec, N, P):
    o = O.Oracle(spec, N, nranks=P)
    ogid, orank = o.get_int("gid"), o.get_int("rank")
    for r in range(P):
        p = sem.Plan(spec, N, rank=r, nranks=P)
        gid, mult, mask = p.slots()
        sel = orank == r
        assert np.array_equal(gid, ogid[sel])
        assert np.array_equal(mult, o.get_int("mult")[sel])   # global multiplicity
        assert np.array_equal(mask, o.get_int("mask")[sel])
        ranks, counts = p.neighbors()
        expect = [q for q in range(P) if q != r and len(o.shared(r, q))]
        assert ranks.tolist() == expect
        for q, cnt in zip(ranks, counts):
            g = p.shared(int(q))
            assert len(g) == cnt
            assert np.array_equal(g, o.shared(r, int(q)))


def test_c3_plan_counts():
    """32^3 periodic N=7: per element 3 faces, 3 edges, 1 vertex; 3.54M pairs."""
    spec, N = CONFIGS["C3"]
    p = sem.Plan(spec, N)
    assert p.npairs == 32 ** 3 * 3 * (N - 1) ** 2
    assert p.nseg == 32 ** 3 * (3 * (N - 1) + 1)
