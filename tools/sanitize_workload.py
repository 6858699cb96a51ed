"""Small workload for compute-sanitizer (memcheck / initcheck / synccheck /
racecheck): C1 PCG, a 4^3-element N=7 slice of C2 (apply, Ax,
gs in every schedule, PCG, single-reduction PCG, GMRES, projection,
Helmholtz), two-level Schwarz (local + coarse, graph and stream launches),
and a 2-rank loopback run (Alg. 1 exchange + rank-ordered allreduces).
Each stage checks its result against the oracle, so a sanitizer run that
exits 0 also computed the right numbers."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import CONFIGS, f_sin, f_tgv, random_field, tgv_box, unit_box  # noqa: E402

stages = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "schwarz", "loopback"]
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731


def check(tag, ok):
    print(f"{tag}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        sys.exit(3)


if "c1" in stages:
    spec, N = CONFIGS["C1"]
    o = O.Oracle(spec, N)
    b = o.rhs(f_sin(o.get("X"), o.get("Y"), o.get("Z")))
    ref = o.pcg(b, 1e-10, 1000)
    with sem.sem_setup(spec, N) as c:
        x = c.zeros()
        r = c.pcg_solve(dev(b), x, 1e-10, 1000)
        check("c1 pcg", abs(r["iters"] - ref["iters"]) <= 1 and
              np.abs(x.cpu().numpy() - ref["x"]).max() <= 1e-10)

if "c2" in stages:
    spec, N = unit_box(4, 4, 4, periodic=(1, 1, 1)), 7
    o = O.Oracle(spec, N)
    u = random_field(o.nslots, seed=3)
    with sem.sem_setup(spec, N) as c:
        du, w = dev(u), c.zeros()
        c.ax(du, w)
        check("c2 ax", np.abs(w.cpu().numpy() - o.ax(u)).max() <= 1e-12 * np.abs(o.ax(u)).max())
        for mode in (1, 2):
            c.set_gs_mode(mode)
            g = du.clone()
            c.gs(g)
            check(f"c2 gs mode {mode}", np.array_equal(g.cpu().numpy(), o.gs(u)))
            c.apply(du, w)
            ra = o.apply(u)
            check(f"c2 apply mode {mode}", np.abs(w.cpu().numpy() - ra).max() <= 1e-12 * np.abs(ra).max())
        c.set_gs_mode(0)
        s = 2 * np.pi
        b = o.rhs(f_tgv(s * o.get("X"), s * o.get("Y"), s * o.get("Z")))
        ref = o.pcg(b, 1e-10, 2000)
        for variant in ("standard", "single_reduction"):
            c.set_pcg_variant(variant)
            x = c.zeros()
            r = c.pcg_solve(dev(b), x, 1e-10, 2000)
            check(f"c2 pcg {variant}", abs(r["iters"] - ref["iters"]) <= 1 and
                  np.abs(x.cpu().numpy() - ref["x"]).max() <= 1e-10)
        c.set_pcg_variant("standard")
        xg = c.zeros()
        rg = c.gmres_solve(dev(b), xg, 1e-10, 2000, 10)
        check("c2 gmres", rg["status"] == 0)
        for q in range(3):
            xp = c.zeros()
            rp = c.proj_solve(dev(b * (1.0 + 0.1 * q)), xp, 1e-10, 2000, 10, 4)
            check(f"c2 projection {q}", rp["status"] == 0)
        xh = c.zeros()
        bh = c.zeros()
        c.rhs_mass(dev(np.ones(o.nslots)), bh)
        rh = c.helm_pcg_solve(0.5, 10.0, bh, xh, 1e-10, 500)
        check("c2 helmholtz", rh["status"] == 0)

if "schwarz" in stages:
    spec, N = tgv_box(4, 4, 4, deform=1), 7
    o = O.Oracle(spec, N)
    b = o.rhs(f_tgv(o.get("X"), o.get("Y"), o.get("Z")))
    with sem.sem_setup(spec, N) as c:
        c.set_precond("schwarz")
        for graph in (True, False):
            c.set_coarse_graph(graph)
            x = c.zeros()
            r = c.pcg_solve(dev(b), x, 1e-10, 500)
            check(f"schwarz pcg graph={graph}", r["status"] == 0)
        c.set_fdm_tc(False)
        z = c.zeros()
        c.schwarz_apply(dev(b), z)
        xg = c.zeros()
        rg = c.gmres_solve(dev(b), xg, 1e-10, 500, 20)
        check("schwarz gmres", rg["status"] == 0)

if "loopback" in stages:
    spec, N = tgv_box(2, 2, 4), 5
    o = O.Oracle(spec, N, nranks=2)
    u = random_field(o.nslots, seed=4)
    b = o.rhs(f_tgv(o.get("X"), o.get("Y"), o.get("Z")))
    ref = o.pcg(b, 1e-10, 1000)
    world = sem.loopback_create(2)
    outs = [None, None]

    def rank(q):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            h = o.nslots // 2
            sl = slice(q * h, (q + 1) * h)
            with sem.sem_setup(spec, N, rank=q, nranks=2, nccl_comm=sem.loopback_comm(world, q),
                               stream=st.cuda_stream) as c:
                g = dev(u[sl])
                c.gs(g)
                x = c.zeros()
                r = c.pcg_solve(dev(b[sl]), x, 1e-10, 1000)
                c.set_precond("schwarz")
                xs = c.zeros()
                rs = c.pcg_solve(dev(b[sl]), xs, 1e-10, 1000)
                outs[q] = (g.cpu().numpy(), x.cpu().numpy(), r, rs)
    th = [threading.Thread(target=rank, args=(q,)) for q in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    sem.loopback_destroy(world)
    check("loopback gs", np.array_equal(np.concatenate([outs[0][0], outs[1][0]]), o.gs(u)))
    check("loopback pcg", abs(outs[0][2]["iters"] - ref["iters"]) <= 1 and
          np.abs(np.concatenate([outs[0][1], outs[1][1]]) - ref["x"]).max() <= 1e-10)
    check("loopback schwarz pcg", outs[0][3]["status"] == 0)
torch.cuda.synchronize()
print("sanitize workload done", flush=True)
