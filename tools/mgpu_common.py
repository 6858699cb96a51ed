"""Multi-rank parity cases shared by the NCCL worker (tools/mgpu_worker.py, one
process per GPU) and the single-GPU loopback test (tests/test_loopback.py, one
host thread per rank on cuda:0).

Every rank builds its z-slab (lexicographic element range) of the mesh
through the C ABI; the local E-vectors are gathered and compared with the
oracle run with the SAME number of ranks, so the gather-scatter summation
order -- ascending slots within a rank, ascending ranks across (P:L204-229
Alg. 1, reading Q10) -- is identical:
  * gs: bit-exact;  apply / rhs: normwise 1e-12 (reading Q22);
  * PCG and single-reduction PCG: iterations +-1, x within 1e-10;
  * GMRES(20): reading Q27's bars;  two-level Schwarz (both coarse modes):
    M r within 1e-11, flexible PCG iterations +-1 and x within 1e-10.
"""
import numpy as np

from sem_inputs import f_sin, f_tgv, random_field, tgv_box, unit_box

CASES = [
    (tgv_box(4, 4, 8), 5, f_tgv),                    # z-slabs, periodic: 2 planes shared
    (unit_box(3, 2, 5), 4, f_sin),                   # Dirichlet, slabs cut mid-layer
    (tgv_box(4, 4, 8, deform=1), 7, f_tgv),          # curvilinear, overlap path
    (unit_box(4, 3, 8, periodic=(1, 0, 0)), 3, f_sin),
]


def case_field(ci, spec, N):
    return random_field(spec.E * (N + 1) ** 3, seed=100 + ci)


def rank_slice(spec, N, rank, P):
    n3 = (N + 1) ** 3
    lo, hi = rank * spec.E // P, (rank + 1) * spec.E // P
    return lo * n3, hi * n3


def rank_run(c, u_local, fun, schwarz=True):
    """One rank's share of the case on context c (inputs: this rank's slice of
    the random field).  Returns host arrays and solver results."""
    import torch
    du = torch.from_numpy(np.ascontiguousarray(u_local)).cuda()
    w = c.zeros()
    c.apply(du, w)
    g = du.clone()
    c.gs(g)
    X, Y, Z = c.coords()
    fv = fun(X, Y, Z, xp=torch)
    b = c.zeros()
    c.rhs(fv, b)
    x = c.zeros()
    r = c.pcg_solve(b, x, 1e-10, 3000)
    # the same solve with stream launches instead of the replayed CUDA graph
    # (P > 1 over peer memory: device-side epochs in the graph)
    xs_ = c.zeros()
    c.set_pcg_graph(False)
    rs_ = c.pcg_solve(b, xs_, 1e-10, 3000)
    c.set_pcg_graph(True)
    xc = c.zeros()
    c.set_pcg_variant("single_reduction")   # one allreduce per iteration
    rc = c.pcg_solve(b, xc, 1e-10, 3000)
    c.set_pcg_variant("standard")
    xg = c.zeros()
    rg = c.gmres_solve(b, xg, 1e-10, 3000, 20)
    out = {"w": w, "g": g, "b": b, "x": x, "r": r, "xc": xc, "rc": rc, "xg": xg, "rg": rg,
           "x_nograph": xs_, "r_nograph": rs_}
    if schwarz:
        # NEXT-1: the fine gs and the N = 1 coarse CG run through the same transport
        c.set_precond("schwarz")
        for mode, tag in ((0, "dist"), (1, "repl")):
            c.set_coarse_replicate(mode)
            zs, xs = c.zeros(), c.zeros()
            c.schwarz_apply(b, zs)
            out["rs_" + tag] = c.pcg_solve(b, xs, 1e-10, 3000)
            out["zs_" + tag], out["xs_" + tag] = zs, xs
        c.set_coarse_replicate(-1)
        c.set_precond("jacobi")
    torch.cuda.current_stream().synchronize()
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}


class OracleRefs:
    """Oracle results of one case at P ranks (computed once, reused across
    transports and gs schedules)."""

    def __init__(self, spec, N, fun, u, P):
        import oracle as O
        o = O.Oracle(spec, N, nranks=P)
        self.w = o.apply(u)
        self.g = o.gs(u)
        self.b = o.rhs(fun(o.get("X"), o.get("Y"), o.get("Z")))
        self.pcg = o.pcg(self.b, 1e-10, 3000)
        self.cgcg = o.cgcg(self.b, 1e-10, 3000)
        self.gmres = o.gmres(self.b, 1e-10, 3000, 20)
        self._o = o
        self._schw = None

    def schwarz(self, B):
        if self._schw is None:
            s = self._o.schwarz(10)
            self._schw = (s.apply(B), s.pcg(B, 1e-10, 3000))
        return self._schw


def check(parts, ref, tag, schwarz=True):
    """parts: rank_run outputs in rank order; returns a list of failure strings."""
    fails = []
    cat = lambda k: np.concatenate([p[k] for p in parts])  # noqa: E731
    W, Gs, B, X = cat("w"), cat("g"), cat("b"), cat("x")
    e = np.abs(W - ref.w).max() / np.abs(ref.w).max()
    if not e <= 1e-12:
        fails.append(f"{tag}: apply rel err {e:.2e}")
    if not np.array_equal(Gs, ref.g):
        fails.append(f"{tag}: gs not bit-exact (max diff {np.abs(Gs - ref.g).max():.2e})")
    e = np.abs(B - ref.b).max() / np.abs(ref.b).max()
    if not e <= 1e-12:
        fails.append(f"{tag}: rhs rel err {e:.2e}")
    r = parts[0]["r"]
    for p in parts[1:]:
        if p["r"]["iters"] != r["iters"]:
            fails.append(f"{tag}: ranks disagree on the iteration count")
    if abs(r["iters"] - ref.pcg["iters"]) > 1 or r["status"] != 0:
        fails.append(f"{tag}: pcg iters {r['iters']} vs {ref.pcg['iters']} st {r['status']}")
    dx = np.abs(X - ref.pcg["x"]).max()
    if not dx <= 1e-10:
        fails.append(f"{tag}: pcg x diff {dx:.2e}")
    if not abs(r["res_final"] - ref.pcg["res_final"]) <= 1e-10:
        fails.append(f"{tag}: pcg res {r['res_final']:.3e} vs {ref.pcg['res_final']:.3e}")
    if parts[0]["r_nograph"]["iters"] != r["iters"] or not np.array_equal(cat("x_nograph"), X):
        fails.append(f"{tag}: graph-replayed and stream-launched PCG differ")
    rc = parts[0]["rc"]
    if abs(rc["iters"] - ref.cgcg["iters"]) > 1 or rc["status"] != 0:
        fails.append(f"{tag}: single-reduction pcg iters {rc['iters']} vs {ref.cgcg['iters']}")
    if not np.abs(cat("xc") - ref.cgcg["x"]).max() <= 1e-10:
        fails.append(f"{tag}: single-reduction pcg x diff {np.abs(cat('xc') - ref.cgcg['x']).max():.2e}")
    rg = parts[0]["rg"]
    # restarted GMRES amplifies the rounding of rank-partitioned dots across
    # restarts (reading Q27): iterations within max(1, 5 %), x within 1e-9
    if abs(rg["iters"] - ref.gmres["iters"]) > max(1, 0.05 * ref.gmres["iters"]) or rg["status"] != 0:
        fails.append(f"{tag}: gmres iters {rg['iters']} vs {ref.gmres['iters']}")
    if not np.abs(cat("xg") - ref.gmres["x"]).max() <= 1e-9:
        fails.append(f"{tag}: gmres x diff {np.abs(cat('xg') - ref.gmres['x']).max():.2e}")
    if schwarz:
        ref_z, refs = ref.schwarz(B)
        for mode in ("dist", "repl"):
            Z = cat("zs_" + mode)
            e = np.abs(Z - ref_z).max() / np.abs(ref_z).max()
            if not e <= 1e-11:
                fails.append(f"{tag}: schwarz ({mode}) apply rel err {e:.2e}")
            rs = parts[0]["rs_" + mode]
            if abs(rs["iters"] - refs["iters"]) > 1 or rs["status"] != 0:
                fails.append(f"{tag}: schwarz ({mode}) pcg iters {rs['iters']} vs {refs['iters']}")
            dxs = np.abs(cat("xs_" + mode) - refs["x"]).max()
            if not dxs <= 1e-10:
                fails.append(f"{tag}: schwarz ({mode}) pcg x diff {dxs:.2e}")
    return fails
