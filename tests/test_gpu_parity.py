"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs.

Tolerances (BASELINE.json north_star):
  * integer / index work (multiplicity, mask): bit-exact;
  * gather-scatter: bit-exact (both sides add the same operands in ascending
    slot order, rank-ordered partials);
  * Ax, apply, rhs, geometry: normwise relative ||y_gpu - y_ref||_inf /
    ||y_ref||_inf <= 1e-12 (reading Q22);
  * PCG: iteration count +-1, final residuals and solution within 1e-10 (abs).
"""
import numpy as np
import pytest

import oracle as O
from sem_inputs import (CONFIGS, MeshSpec, f_sin, f_tgv, random_field, tgv_box, unit_box,
                        weak_scaled)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2107_01243_b200 import build
    build.build()
    torch.cuda.set_device(0)


def sem():
    import paper_2107_01243_b200 as s
    return s


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def nrel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


MESHES = [
    (CONFIGS["C1"][0], 3),                       # Dirichlet, 8 elements
    (unit_box(3, 2, 5, periodic=(1, 0, 0)), 7),  # mixed BC, 30 elements
    (tgv_box(4, 3, 5, deform=1), 7),             # curvilinear, all 6 G
    (tgv_box(2, 2, 2), 1),                       # N=1: vertices only
    (unit_box(5, 2, 1), 2),                      # ragged tail for NE=8 (n=3)
    (tgv_box(3, 3, 3, deform=1), 4),
    (unit_box(2, 3, 2, periodic=(0, 1, 1)), 5),
    (tgv_box(2, 2, 3, deform=1), 11),            # maximum N
    (unit_box(3, 3, 2), 9),
    (tgv_box(3, 2, 3, deform=1), 6),             # odd n: u blocks 8 mod 16 every other element
    (unit_box(3, 2, 3, periodic=(0, 0, 1)), 8),
    (tgv_box(2, 3, 2, deform=1), 10),
]
IDS = [f"{s.ex}x{s.ey}x{s.ez}-p{''.join(map(str, s.periodic))}-d{s.deform}-N{N}" for s, N in MESHES]


@pytest.mark.parametrize("spec,N", MESHES, ids=IDS)
def test_setup_exports(spec, N):
    o = O.Oracle(spec, N)
    with sem().sem_setup(spec, N) as c:
        assert c.n_local == o.nslots and c.n_glob == o.nglob
        assert np.array_equal(c.export_int("mult"), o.get_int("mult"))
        assert np.array_equal(c.export_int("mask"), o.get_int("mask"))
        assert nrel(c.export_field("G"), o.get("G")) < 1e-12
        assert nrel(c.export_field("B"), o.get("B")) < 1e-12
        assert nrel(c.export_field("dinv"), o.get("dinv")) < 1e-12
        X, Y, Z = c.coords()
        for t, name in zip((X, Y, Z), "XYZ"):
            assert np.abs(host(t) - o.get(name)).max() < 1e-13


@pytest.mark.parametrize("spec,N", MESHES, ids=IDS)
def test_ax_gs_apply_parity(spec, N):
    o = O.Oracle(spec, N)
    u = random_field(o.nslots, seed=11)
    with sem().sem_setup(spec, N) as c:
        du, dw = dev(u), c.zeros()
        c.ax(du, dw)
        w_ax = host(dw)
        assert nrel(w_ax, o.ax(u)) <= 1e-12
        # gather-scatter: bit-exact (same operands, same ascending order)
        dv = dev(u)
        c.gs(dv)
        assert np.array_equal(host(dv), o.gs(u))
        # the operator: Ax (+ mask) then gs
        dw.zero_()
        c.apply(du, dw)
        w_ap, ref = host(dw), o.apply(u)
        assert nrel(w_ap, ref) <= 1e-12
        assert np.all(w_ap[o.get_int("mask") == 1] == 0.0)
        # continuity: every slot of a gid holds the same value, exactly
        gid = o.get_int("gid")
        first = np.zeros(o.nglob)
        first[gid] = w_ap
        assert np.array_equal(first[gid], w_ap)


def test_apply_is_deterministic_and_schedules_agree_bitwise():
    spec, N = tgv_box(6, 5, 4, deform=1), 7
    u = random_field(spec.n_slots(N), seed=5)
    with sem().sem_setup(spec, N) as c:
        du = dev(u)
        outs = []
        for mode in (0, 1, 2, 0):
            c.set_gs_mode(mode)
            w = c.zeros()
            c.apply(du, w)
            outs.append(host(w))
        for o in outs[1:]:
            assert np.array_equal(outs[0], o)


@pytest.mark.parametrize("N", [1, 3, 7])
@pytest.mark.parametrize("mode", [1, 2], ids=["flat", "chunks"])
def test_gs_schedules_bit_exact(N, mode):
    """Both rank-local gs schedules (SEM_OPT_GS_MODE) give the oracle's sums
    bit for bit; the chunk counter carries across calls without a reset."""
    spec = tgv_box(9, 7, 6, deform=1)
    o = O.Oracle(spec, N)
    u = random_field(o.nslots, seed=11)
    ref_gs, ref_ap = o.gs(u), o.apply(u)
    with sem().sem_setup(spec, N) as c:
        c.set_gs_mode(mode)
        w = c.zeros()
        for _ in range(3):
            g = dev(u)
            c.gs(g)
            assert np.array_equal(host(g), ref_gs)
            c.apply(dev(u), w)
            assert nrel(host(w), ref_ap) <= 1e-12


@pytest.mark.parametrize("N", [2, 4, 6, 8, 10])
def test_odd_n_ring_wrap(N):
    """More elements than resident CTAs, so every CTA cycles through both u
    slots and all G slots (odd n: u blocks alternate between 0 and 8 mod 16)."""
    spec = tgv_box(12, 10, 10, deform=1)
    o = O.Oracle(spec, N)
    u = random_field(o.nslots, seed=7)
    with sem().sem_setup(spec, N) as c:
        du = dev(u)
        w = c.zeros()
        c.ax(du, w)
        assert nrel(host(w), o.ax(u)) <= 1e-12
        c.apply(du, w)
        assert nrel(host(w), o.apply(u)) <= 1e-12


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_full_size_apply(cfg):
    """BASELINE configs[1] (the bench workload) and configs[2] at full size."""
    spec, N = CONFIGS[cfg]
    o = O.Oracle(spec, N)
    u = random_field(o.nslots, seed=0)
    with sem().sem_setup(spec, N) as c:
        du, dw = dev(u), c.zeros()
        c.ax(du, dw)
        assert nrel(host(dw), o.ax(u)) <= 1e-12
        ref = o.apply(u)
        for mode in (1, 2):
            c.set_gs_mode(mode)
            dw.zero_()
            c.apply(du, dw)
            assert nrel(host(dw), ref) <= 1e-12


def test_full_size_c4():
    """BASELINE configs[3] at full size on one GPU (64^3 deformed elements, N=7,
    134M slots, all six factors nonzero): every slot of Ax and of the operator
    within 1e-12 and gs bit-exact, in both gs schedules (the chunk schedule is
    the one auto picks at this size).  The oracle needs ~20 GB of host RAM."""
    import os
    if os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") < 48e9:
        pytest.skip("host RAM < 48 GB for the full-size oracle")
    spec, N = CONFIGS["C4"]
    o = O.Oracle(spec, N)
    u = random_field(o.nslots, seed=21)
    with sem().sem_setup(spec, N) as c:
        du, dw = dev(u), c.zeros()
        c.ax(du, dw)
        assert nrel(host(dw), o.ax(u)) <= 1e-12
        ref_ap, ref_gs = o.apply(u), o.gs(u)
        for mode in (0, 1):
            c.set_gs_mode(mode)
            c.apply(du, dw)
            assert nrel(host(dw), ref_ap) <= 1e-12
            g = dev(u)
            c.gs(g)
            assert np.array_equal(host(g), ref_gs)
            del g


@pytest.mark.parametrize("spec,N,fun", [(CONFIGS["C1"][0], 3, f_sin), (tgv_box(4, 4, 3), 5, f_tgv),
                                        (tgv_box(3, 4, 3, deform=1), 6, f_tgv),
                                        (unit_box(2, 3, 2, periodic=(0, 1, 1)), 5, f_sin),
                                        (CONFIGS["C1"][0], 3, None),
                                        (unit_box(3, 2, 2, periodic=(0, 1, 0)), 4, None)])
def test_rhs_parity(spec, N, fun):
    """fun None: a random f, nonzero on the Dirichlet boundary (every masked slot,
    including the ones no gather-scatter entity touches, must come out 0)."""
    o = O.Oracle(spec, N)
    f = fun(o.get("X"), o.get("Y"), o.get("Z")) if fun else random_field(o.nslots, seed=41)
    with sem().sem_setup(spec, N) as c:
        b = c.zeros()
        c.rhs(dev(f), b)
        assert nrel(host(b), o.rhs(f)) <= 1e-12


PCG_CASES = [
    (CONFIGS["C1"][0], 3, f_sin, 1e-10),
    (tgv_box(8, 8, 8), 7, f_tgv, 1e-10),           # reduced C3
    (tgv_box(6, 6, 6, deform=1), 5, f_tgv, 1e-10),  # reduced C4 (curvilinear)
    (unit_box(3, 2, 4, periodic=(1, 0, 0)), 6, f_sin, 1e-10),
]


@pytest.mark.parametrize("spec,N,fun,tol", PCG_CASES)
def test_pcg_parity(spec, N, fun, tol):
    o = O.Oracle(spec, N)
    f = fun(o.get("X"), o.get("Y"), o.get("Z"))
    b = o.rhs(f)
    ref = o.pcg(b, tol, 5000)
    with sem().sem_setup(spec, N) as c:
        x = c.zeros()
        r = c.pcg_solve(dev(b), x, tol, 5000)
        xs = host(x)
        assert r["status"] == 0 and ref["status"] == 0
        assert abs(r["iters"] - ref["iters"]) <= 1
        assert abs(r["res_final"] - ref["res_final"]) <= 1e-10
        assert abs(r["res_true"] - ref["res_true"]) <= 1e-10
        assert r["res_final"] <= tol
        assert np.abs(xs - ref["x"]).max() <= 1e-10
        # residual history: identical start; later CG amplifies rounding-order
        # differences (sigma is p^T A_L p on the GPU, <p,w>_c in the oracle)
        h = c.pcg_history()
        k = min(len(h), len(ref["hist"]), 8)
        np.testing.assert_allclose(h[:k], ref["hist"][:k], rtol=1e-8)
        k = min(len(h), len(ref["hist"]))
        np.testing.assert_allclose(h[:k], ref["hist"][:k], rtol=0.2, atol=1e-9)
        # end-to-end host entry point gives the same answer
        xh = np.zeros(c.n_local)
        r2 = c.pcg_solve_host(np.ascontiguousarray(b), xh, tol, 5000)
        assert r2["iters"] == r["iters"]
        assert np.array_equal(xh, xs)


def test_pcg_c3_fixed_20_iterations():
    """Full-size C3 (32^3, N=7, TGV pressure): the oracle's 20 iterations."""
    spec, N = CONFIGS["C3"]
    o = O.Oracle(spec, N)
    b = o.rhs(f_tgv(o.get("X"), o.get("Y"), o.get("Z")))
    ref = o.pcg(b, 0.0, 20)
    with sem().sem_setup(spec, N) as c:
        x = c.zeros()
        r = c.pcg_solve(dev(b), x, 0.0, 20)
        assert r["iters"] == 20 and r["status"] == 1
        assert abs(r["res_final"] - ref["res_final"]) <= 1e-10
        assert np.abs(host(x) - ref["x"]).max() <= 1e-10
        np.testing.assert_allclose(c.pcg_history(), ref["hist"], rtol=1e-9)


def test_pcg_edge_cases():
    spec, N = CONFIGS["C1"]
    with sem().sem_setup(spec, N) as c:
        x = c.zeros()
        # zero right-hand side: converged before the first iteration
        r = c.pcg_solve(c.zeros(), x, 1e-10, 100)
        assert r["iters"] == 0 and r["status"] == 0
        assert float(x.abs().max()) == 0.0
        # maxit = 0
        o = O.Oracle(spec, N)
        b = dev(o.rhs(f_sin(o.get("X"), o.get("Y"), o.get("Z"))))
        r = c.pcg_solve(b, x, 1e-10, 0)
        assert r["iters"] == 0 and r["status"] == 1
        # bad arguments are rejected loudly
        with pytest.raises(sem().SemError):
            c.pcg_solve(b, b, 1e-10, 10)
        with pytest.raises(sem().SemError):
            c.apply(b, b)


def test_launch_counts_and_native_library_loaded():
    import os
    spec, N = CONFIGS["C1"]
    with sem().sem_setup(spec, N) as c:
        u = c.zeros()
        w = c.zeros()
        n0 = c.launch_count()
        c.apply(u, w)
        assert c.launch_count() == n0 + 2   # Ax, gs at P=1
        for opt in (1, 5, 10):   # retired slower variants are rejected
            with pytest.raises(sem().SemError):
                c._set_option(opt, 1)
    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert os.path.basename(sem().lib_path()) in maps   # libsem.so (or a SEM_LIB build)


# ---------------------------------------------------------------- NEXT-2: Helmholtz h1 A + h2 B
HELM_MESHES = [(CONFIGS["C1"][0], 3), (tgv_box(4, 3, 5, deform=1), 7), (unit_box(3, 2, 3), 4),
               (tgv_box(3, 3, 2, deform=1), 11), (tgv_box(12, 10, 10, deform=1), 6)]


@pytest.mark.parametrize("spec,N", HELM_MESHES,
                         ids=[f"{s.ex}x{s.ey}x{s.ez}-d{s.deform}-N{N}" for s, N in HELM_MESHES])
@pytest.mark.parametrize("h1,h2", [(1.0, 0.0), (0.3, 2.5), (1.0 / 1600.0, 2000.0)])
def test_helm_apply_parity(spec, N, h1, h2):
    o = O.Oracle(spec, N)
    u = random_field(o.nslots, seed=31)          # discontinuous: exercises the element-level B term
    with sem().sem_setup(spec, N) as c:
        w = c.zeros()
        c.helm_apply(h1, h2, dev(u), w)
        assert nrel(host(w), o.helm_apply(h1, h2, u)) <= 1e-12
        f = random_field(o.nslots, seed=32)
        b = c.zeros()
        c.rhs_mass(dev(f), b)
        assert nrel(host(b), o.rhs_mass(f)) <= 1e-12


@pytest.mark.parametrize("spec,N,h1,h2", [(CONFIGS["C1"][0], 3, 1.0, 10.0),
                                          (tgv_box(6, 6, 6, deform=1), 5, 0.5, 3.0),
                                          (tgv_box(8, 8, 8), 7, 1.0 / 1600.0, 2000.0)])
def test_helm_pcg_parity(spec, N, h1, h2):
    """Helmholtz Jacobi-PCG: iterations +-1 and x within 1e-10 of the oracle's
    (fully periodic boxes included: h2 > 0 makes the system nonsingular)."""
    o = O.Oracle(spec, N)
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    fun = f_sin if not all(spec.periodic) else f_tgv
    b = o.rhs_mass(fun(X, Y, Z))
    ref = o.helm_pcg(h1, h2, b, 1e-10, 3000)
    with sem().sem_setup(spec, N) as c:
        x = c.zeros()
        r = c.helm_pcg_solve(h1, h2, dev(b), x, 1e-10, 3000)
        assert r["status"] == 0 and abs(r["iters"] - ref["iters"]) <= 1
        assert np.abs(host(x) - ref["x"]).max() <= 1e-10
        assert abs(r["res_final"] - ref["res_final"]) <= 1e-10
        assert abs(r["res_true"] - ref["res_true"]) <= 1e-10
        # the Poisson solve on the same context is unaffected afterwards
        c.apply(dev(b), x)
        assert nrel(host(x), o.apply(b)) <= 1e-12


def test_ring_release_stress():
    """Regression for the G-ring write-after-read hazard: a CTA released a G
    slot right after issuing its shared-memory reads, so the producer's TMA
    could overwrite factors still being read (showed as ~6 % wrong Helmholtz
    applications at n=7 with NE=2, PPC=1).  Repeated applies must all match."""
    spec, N = tgv_box(12, 10, 10, deform=1), 6
    o = O.Oracle(spec, N)
    u = random_field(o.nslots, seed=31)
    ref_h, ref_p = o.helm_apply(0.3, 2.5, u), o.apply(u)
    with sem().sem_setup(spec, N) as c:
        w = c.zeros()
        du = dev(u)
        for _ in range(60):
            c.helm_apply(0.3, 2.5, du, w)
            assert nrel(host(w), ref_h) <= 1e-12
            c.apply(du, w)
            assert nrel(host(w), ref_p) <= 1e-12


# ---------------------------------------------------------------- NEXT-3: GMRES and projection
@pytest.mark.parametrize("spec,N,restart", [(CONFIGS["C1"][0], 3, 30), (tgv_box(6, 6, 6, deform=1), 5, 30),
                                            (tgv_box(6, 6, 6, deform=1), 5, 7),
                                            (unit_box(3, 2, 4, periodic=(1, 0, 0)), 6, 12),
                                            (unit_box(3, 1, 3), 4, 30)])   # odd n_local
def test_gmres_parity(spec, N, restart):
    o = O.Oracle(spec, N)
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    fun = f_tgv if all(spec.periodic) else f_sin
    b = o.rhs(fun(X, Y, Z))
    ref = o.gmres(b, 1e-10, 3000, restart)
    with sem().sem_setup(spec, N) as c:
        x = c.zeros()
        r = c.gmres_solve(dev(b), x, 1e-10, 3000, restart)
        assert r["status"] == 0 and abs(r["iters"] - ref["iters"]) <= 1, (r, ref["iters"])
        assert np.abs(host(x) - ref["x"]).max() <= 1e-10
        assert abs(r["res_true"] - ref["res_true"]) <= 1e-10
        assert r["res_final"] <= 1e-10


def test_projection_pipeline_parity():
    """A slowly varying sequence of pressure right-hand sides through the
    projection + GMRES pipeline: per-solve iterations and x close (Q27), the
    same space size as the oracle's, and fewer iterations as the space fills.
    Each right-hand side carries a small seeded random part, so the deflated
    right-hand sides stay well above rounding (a purely low-dimensional family
    is spanned after a few solves and GMRES then converges on rounding noise,
    where iteration counts are not reproducible by any two implementations)."""
    spec, N = tgv_box(6, 5, 6, deform=1), 5
    o = O.Oracle(spec, N)
    X, Y, Z = o.get("X"), o.get("Y"), o.get("Z")
    op = o.proj(20)
    its = []
    with sem().sem_setup(spec, N) as c:
        for t in range(6):
            f = (f_tgv(X, Y, Z) * (1.0 + 0.05 * t) + 0.3 * t * np.cos(X) * np.cos(2 * Z)
                 + 1e-4 * random_field(o.nslots, seed=100 + t))
            b = o.rhs(f)
            ref = op.solve(b, 1e-10, 3000, 30)
            x = c.zeros()
            r = c.proj_solve(dev(b), x, 1e-10, 3000, 30, 20)
            assert r["status"] == 0, (t, r)
            assert abs(r["iters"] - ref["iters"]) <= max(1, 0.05 * ref["iters"]), (t, r, ref["iters"])
            assert np.abs(host(x) - ref["x"]).max() <= 1e-9
            assert c.proj_size() == op.size
            its.append(r["iters"])
        # the same right-hand side again: as many iterations as the oracle (a few:
        # the stored solution's residual sits just under tol; S:L414's "0 or 1"
        # holds on easy cases, see tests/test_oracle_gmres_pins.py)
        ref = op.solve(b, 1e-10, 3000, 30)
        x = c.zeros()
        r = c.proj_solve(dev(b), x, 1e-10, 3000, 30, 20)
        assert abs(r["iters"] - ref["iters"]) <= 1 and r["iters"] < its[-1] // 4, (r, ref["iters"])
    assert its[-1] < its[0], its


@pytest.mark.parametrize("spec,N", [(CONFIGS["C1"][0], 3), (tgv_box(4, 3, 5, deform=1), 7),
                                    (unit_box(3, 2, 5, periodic=(1, 0, 0)), 5), (tgv_box(2, 2, 2), 1),
                                    (unit_box(3, 1, 3), 4)])
def test_pcg_single_reduction_parity(spec, N):
    """SEM_OPT_PCG_VARIANT = 1 (Chronopoulos-Gear, reading Q34) against the
    oracle's single-reduction PCG: iterations +-1, x and residuals within 1e-10;
    also the Helmholtz operator through the same recurrences."""
    o = O.Oracle(spec, N)
    fun = f_tgv if all(spec.periodic) else f_sin
    b = o.rhs(fun(o.get("X"), o.get("Y"), o.get("Z")))
    ref = o.cgcg(b, 1e-10, 3000)
    with sem().sem_setup(spec, N) as c:
        c.set_pcg_variant("single_reduction")
        x = c.zeros()
        r = c.pcg_solve(dev(b), x, 1e-10, 3000)
        assert r["status"] == 0 and abs(r["iters"] - ref["iters"]) <= 1, (r, ref["iters"])
        assert np.abs(host(x) - ref["x"]).max() <= 1e-10
        assert abs(r["res_true"] - ref["res_true"]) <= 1e-10
        h = c.pcg_history()
        k = min(len(h), len(ref["hist"]), 6)
        np.testing.assert_allclose(h[:k], ref["hist"][:k], rtol=1e-8, atol=1e-12 * ref["hist"][0])
        h1, h2 = 1.0 / 1600.0, 2000.0
        bh = o.rhs_mass(fun(o.get("X"), o.get("Y"), o.get("Z")))
        refh = o.helm_pcg(h1, h2, bh, 1e-10, 2000)
        xh = c.zeros()
        rh = c.helm_pcg_solve(h1, h2, dev(bh), xh, 1e-10, 2000)
        assert rh["status"] == 0 and abs(rh["iters"] - refh["iters"]) <= 1, (rh, refh["iters"])
        assert np.abs(host(xh) - refh["x"]).max() <= 1e-10


@pytest.mark.parametrize("spec,N", [(CONFIGS["C2"][0], 7), (tgv_box(4, 3, 5, deform=1), 7),
                                    (unit_box(3, 2, 5, periodic=(1, 0, 0)), 5)])
def test_ax_pdl_identical(spec, N):
    """SEM_OPT_AX_PDL (PDL launch of the PCG Ax kernel, G prefetched before the
    grid wait) gives bit-identical PCG iterates."""
    o = O.Oracle(spec, N) if spec.E <= 64 else None
    n = spec.E * (N + 1) ** 3
    b = random_field(n, seed=21)
    with sem().sem_setup(spec, N) as c:
        bd = c.zeros()
        c.apply(dev(b), bd)          # an assembled, masked right-hand side
        out = []
        for on in (False, True, False, True):
            c.set_ax_pdl(on)
            x = c.zeros()
            r = c.pcg_solve(bd, x, 0.0, 25)
            out.append((host(x), r["res_final"]))
        assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]
        assert np.array_equal(out[1][0], out[3][0])
        if o is not None:
            ref = o.pcg(host(bd), 0.0, 25)
            assert np.abs(out[1][0] - ref["x"]).max() <= 1e-10 * max(1.0, np.abs(ref["x"]).max())


# ---------------------------------------------------------------- live plan export
LIVE_PLAN = [(unit_box(2, 2, 2), 3, 1), (tgv_box(3, 4, 2), 5, 1), (tgv_box(4, 4, 4, deform=1), 7, 1),
             (unit_box(3, 2, 4, periodic=(1, 0, 0)), 2, 1), (tgv_box(2, 2, 4), 3, 2),
             (unit_box(3, 2, 5), 3, 3), (tgv_box(4, 2, 2), 4, 4)]


@pytest.mark.parametrize("spec,N,P", LIVE_PLAN, ids=[f"{s.ex}x{s.ey}x{s.ez}-N{N}-P{P}" for s, N, P in LIVE_PLAN])
def test_live_plan_export_bit_exact(spec, N, P):
    """sem_export_plan: the gather-scatter records the device kernels use, read
    back from a live context (P > 1: each rank of a loopback world), expand to
    the oracle's numbering, multiplicity, mask, pairs, segments and shared
    lists bit-exactly (Alg. 1)."""
    import threading
    import torch
    o = O.Oracle(spec, N, nranks=P)
    plans = [None] * P
    if P == 1:
        with sem().sem_setup(spec, N) as c:
            plans[0] = c.export_plan()
    else:
        world = sem().loopback_create(P)
        errs = []

        def rank(r):
            try:
                st = torch.cuda.Stream()
                with sem().sem_setup(spec, N, rank=r, nranks=P, nccl_comm=sem().loopback_comm(world, r),
                                     stream=st.cuda_stream) as c:
                    plans[r] = c.export_plan()
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
        th = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        sem().loopback_destroy(world)
        assert not errs, errs
    orank = o.get_int("rank")
    for r, p in enumerate(plans):
        sel = orank == r
        gid, mult, mask = p.slots()
        assert np.array_equal(gid, o.get_int("gid")[sel])
        assert np.array_equal(mult, o.get_int("mult")[sel])
        assert np.array_equal(mask, o.get_int("mask")[sel])
        ranks, counts = p.neighbors()
        assert ranks.tolist() == [q for q in range(P) if q != r and len(o.shared(r, q))]
        for q in ranks:
            assert np.array_equal(p.shared(int(q)), o.shared(r, int(q)))
    if P == 1:
        op, ooff, oslots = o.plan()
        pp, poff, pslots = plans[0].pairs()
        assert np.array_equal(pp, op) and np.array_equal(poff, ooff) and np.array_equal(pslots, oslots)


@pytest.mark.parametrize("spec,N", [(tgv_box(8, 8, 8), 7), (CONFIGS["C1"][0], 3), (tgv_box(4, 3, 5, deform=1), 5)])
def test_pcg_graph_identical(spec, N):
    """SEM_OPT_PCG_GRAPH: 8-iteration batches replayed as a CUDA graph give the
    stream-launched iterates bit for bit (and the graph is reused by a second
    solve with the same operands)."""
    o = O.Oracle(spec, N)
    fun = f_tgv if all(spec.periodic) else f_sin
    b = dev(o.rhs(fun(o.get("X"), o.get("Y"), o.get("Z"))))
    ref = o.pcg(host(b), 1e-10, 3000)
    with sem().sem_setup(spec, N) as c:
        outs = []
        for g in (False, True, True):
            c.set_pcg_graph(g)
            x = c.zeros()
            r = c.pcg_solve(b, x, 1e-10, 3000)
            outs.append((host(x), r["iters"], c.pcg_history()))
        for x_, it, h in outs[1:]:
            assert it == outs[0][1] and np.array_equal(x_, outs[0][0]) and np.array_equal(h, outs[0][2])
        assert abs(outs[0][1] - ref["iters"]) <= 1 and np.abs(outs[0][0] - ref["x"]).max() <= 1e-10


PF_CASES = [(CONFIGS["C1"][0], 3), (tgv_box(8, 8, 8), 7), (tgv_box(4, 3, 5, deform=1), 6),
            (unit_box(3, 2, 5, periodic=(1, 0, 0)), 5), (tgv_box(3, 3, 2, deform=1), 8),
            (unit_box(2, 3, 2), 10), (tgv_box(2, 2, 2), 1), (tgv_box(3, 2, 2), 11)]


@pytest.mark.parametrize("spec,N", PF_CASES, ids=[f"{s.ex}x{s.ey}x{s.ez}-N{N}" for s, N in PF_CASES])
def test_pcg_fused_p_update(spec, N):
    """SEM_OPT_PCG_FUSE: the p update fused into the Ax kernel (p = dinv r +
    beta p in the kernel's prologue, x += alpha p in the r update) reaches the
    oracle's iterate like the four-kernel iteration (every n incl. odd ones,
    Dirichlet and periodic, Helmholtz); same iteration count."""
    o = O.Oracle(spec, N)
    fun = f_tgv if all(spec.periodic) else f_sin
    b = o.rhs(fun(o.get("X"), o.get("Y"), o.get("Z")))
    ref = o.pcg(b, 1e-10, 3000)
    with sem().sem_setup(spec, N) as c:
        res = {}
        for fuse in (True, False):
            c.set_pcg_fuse(fuse)
            x = c.zeros()
            r = c.pcg_solve(dev(b), x, 1e-10, 3000)
            res[fuse] = (host(x), r)
            assert r["status"] == 0 and abs(r["iters"] - ref["iters"]) <= 1, (fuse, r, ref["iters"])
            assert np.abs(host(x) - ref["x"]).max() <= 1e-10
            assert abs(r["res_true"] - ref["res_true"]) <= 1e-10
        assert abs(res[True][1]["iters"] - res[False][1]["iters"]) <= 1
        # Helmholtz PCG through the same fused kernel
        bh = c.zeros()
        c.rhs_mass(dev(fun(o.get("X"), o.get("Y"), o.get("Z"))), bh)
        refh = o.helm_pcg(0.5, 3.0, host(bh), 1e-10, 2000)
        xs = []
        for fuse in (True, False):
            c.set_pcg_fuse(fuse)
            xh = c.zeros()
            rh = c.helm_pcg_solve(0.5, 3.0, bh, xh, 1e-10, 2000)
            assert rh["status"] == 0 and abs(rh["iters"] - refh["iters"]) <= 1
            assert np.abs(host(xh) - refh["x"]).max() <= 1e-10
            xs.append((host(xh), rh["iters"]))
        assert abs(xs[0][1] - xs[1][1]) <= 1 and np.abs(xs[0][0] - xs[1][0]).max() <= 1e-10


@pytest.mark.parametrize("spec,N", PF_CASES, ids=[f"{s.ex}x{s.ey}x{s.ez}-N{N}" for s, N in PF_CASES])
def test_pcg_gather_on_read_identical(spec, N):
    """SEM_OPT_PCG_GSU: the r update sums the unassembled w over each shared
    point's incidences (ascending slots) instead of a separate gs kernel -- the
    same sums in the same order, so the PCG iterates (x, iteration count, final
    residual) are bitwise those of the gs-kernel iteration, for Poisson and
    Helmholtz, with and without graph replay."""
    o = O.Oracle(spec, N)
    fun = f_tgv if all(spec.periodic) else f_sin
    f = fun(o.get("X"), o.get("Y"), o.get("Z"))
    b = o.rhs(f)
    with sem().sem_setup(spec, N) as c:
        bh = c.zeros()
        c.rhs_mass(dev(f), bh)
        for graph in (True, False):
            c.set_pcg_graph(graph)
            out = {}
            for gsu in (True, False):
                c.set_pcg_gsu(gsu)
                x = c.zeros()
                r = c.pcg_solve(dev(b), x, 1e-10, 3000)
                xh = c.zeros()
                rh = c.helm_pcg_solve(0.5, 3.0, bh, xh, 1e-10, 2000)
                out[gsu] = (host(x), r, host(xh), rh)
            (x1, r1, xh1, rh1), (x0, r0, xh0, rh0) = out[True], out[False]
            assert r1["status"] == 0 and r1["iters"] == r0["iters"], (graph, r1, r0)
            assert r1["res_final"] == r0["res_final"] and np.array_equal(x1, x0), graph
            assert rh1["iters"] == rh0["iters"] and np.array_equal(xh1, xh0), graph
        c.set_pcg_graph(True)
        c.set_pcg_gsu(-1)
