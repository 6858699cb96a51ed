"""SURVEY 8(d)/(e) measurements that bench.py (C2 PCG step) does not cover.

  python tools/measure.py single            # one GPU: triad, C3, C4, N-sweep
  torchrun --nproc-per-node P tools/measure.py strong   # C3/C4 strong scaling
  torchrun --nproc-per-node P tools/measure.py c5_strong|c5_weak [N,...]   # C5 at ~1e9 DOF

Each result is one JSON line on stdout (rank 0).  All timings are CUDA events
on the context stream after warm-up, max over ranks for P > 1.  Denominators:
nominal 8 TB/s, the measured copy peak (MEASURED_PEAKS.json) and an fp64
STREAM triad measured in the same run (paper's convention).
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import CONFIGS, f_tgv, p_tgv, tgv_box  # noqa: E402

NOMINAL = 8000.0


def peak_copy():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def bytes_model(N):
    fb = 1.0 - ((N - 1) / (N + 1)) ** 3
    return fb, 64.0, 64.0 + 20.0 * fb


def out(d):
    print(json.dumps(d), flush=True)


def timed(fn, st, reps, warm=3, sync=None):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    if sync:
        sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps   # ms


def triad(st):
    """a = b + s c over 2^27 fp64 (1 GiB per vector): 24 B per element."""
    n = 1 << 27
    b = torch.rand(n, dtype=torch.float64, device="cuda")
    c = torch.rand(n, dtype=torch.float64, device="cuda")
    a = torch.empty_like(b)
    ms = timed(lambda: torch.add(b, c, alpha=3.0, out=a), st, 20)
    return 24.0 * n / (ms * 1e-3) / 1e9


def op_rates(c, N, st, reps, tri):
    n = c.n_local
    u = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    w = c.zeros()
    fb, bax, baxgs = bytes_model(N)
    res = {}

    cases = [("ax", lambda: c.ax(u, w), bax, 0), ("ax_gs", lambda: c.apply(u, w), baxgs, 0),
             ("ax_gs_flat", lambda: c.apply(u, w), baxgs, 1),
             ("ax_gs_chunks", lambda: c.apply(u, w), baxgs, 2)]
    for name, fn, bpp, mode in cases:
        c.set_gs_mode(mode)
        ms = timed(fn, st, reps)
        gbs = bpp * n / (ms * 1e-3) / 1e9
        res[name] = {"ms": round(ms, 4), "gdofs": round(n / (ms * 1e-3) / 1e9, 2),
                     "useful_GBps": round(gbs, 0), "frac_nominal": round(gbs / NOMINAL, 3),
                     "frac_copy": round(gbs / peak_copy(), 3),
                     "frac_triad": round(gbs / tri, 3) if tri else None}
    c.set_gs_mode(0)
    del u, w
    return res


def helm(cfg="C3", h1=1.0 / 1600.0, h2=2000.0):
    """NEXT-2 Helmholtz on a BASELINE config: h1 A + h2 B apply rate (72 + 20 f_b
    B/pt: the Ax kernel also streams B) and Jacobi-PCG to 1e-10 at the velocity-
    solve coefficients of S:L302 (Re = 1600, dt = 5e-4)."""
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    spec, N = CONFIGS[cfg]
    fb = bytes_model(N)[0]
    with sem.sem_setup(spec, N, stream=st.cuda_stream) as c:
        n = c.n_local
        u = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        w = c.zeros()
        ms = timed(lambda: c.helm_apply(h1, h2, u, w), st, 50)
        bpp = 72.0 + 20.0 * fb
        gbs = bpp * n / (ms * 1e-3) / 1e9
        X, Y, Z = c.coords()
        f = h1 * f_tgv(X, Y, Z, xp=torch) + h2 * p_tgv(X, Y, Z, xp=torch)   # (-h1 lap + h2) p*
        b = c.zeros()
        c.rhs_mass(f, b)
        x = c.zeros()
        c.helm_pcg_solve(h1, h2, b, x, 1e-10, 2000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        r = c.helm_pcg_solve(h1, h2, b, x, 1e-10, 2000)
        e1.record(st)
        torch.cuda.synchronize()
        pms = e0.elapsed_time(e1)
        einf = float((x - p_tgv(X, Y, Z, xp=torch)).abs().max())
        out({"what": f"{cfg}_helm", "h1": h1, "h2": h2, "apply_ms": round(ms, 4),
             "apply_gdofs": round(n / (ms * 1e-3) / 1e9, 2), "apply_B_per_pt": round(bpp, 1),
             "apply_frac_nominal": round(gbs / NOMINAL, 3), "apply_frac_copy": round(gbs / peak_copy(), 3),
             "pcg_iters": r["iters"], "pcg_status": r["status"], "pcg_ms": round(pms, 3),
             "pcg_iter_per_s": round(r["iters"] / (pms * 1e-3), 1),
             "pcg_gdofs": round(n * r["iters"] / (pms * 1e-3) / 1e9, 2), "e_inf_vs_p*": einf})


def schwarz(cfgs=("C3", "C4")):
    """NEXT-1: the two-level Schwarz preconditioner on BASELINE
    configs: time of one application (local FDM part, coarse part, both), the
    FDM kernel against HBM (8 r + 1 mult + 8 y B/pt + 24 (n^2 + n) B of
    factors per element), and time-to-solution to 1e-10 on the TGV pressure
    right-hand side: Jacobi-PCG, Schwarz flexible PCG, Jacobi GMRES(30),
    Schwarz flexible GMRES(30)."""
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    for cfg in cfgs:
        spec, N = CONFIGS[cfg]
        n1 = N + 1
        with sem.sem_setup(spec, N, stream=st.cuda_stream) as c:
            n = c.n_local
            if os.environ.get("COARSE_ASM") == "0":   # A/B: element-operator coarse CG
                c.set_coarse_asm(False)
            if os.environ.get("SCHWARZ_GRAPH") == "0":   # A/B: stream-launched Schwarz batches
                c.set_schwarz_graph(False)
            if os.environ.get("GMRES_GRAPH") == "0":     # A/B: stream-launched GMRES cycles
                c.set_gmres_graph(False)
            X, Y, Z = c.coords()
            b = c.zeros()
            c.rhs(f_tgv(X, Y, Z, xp=torch), b)
            del X, Y, Z
            z = c.zeros()
            c.schwarz_apply(b, z, 3)
            res = {"what": f"{cfg}_schwarz", "n_local": n,
                   "coarse": "element" if os.environ.get("COARSE_ASM") == "0" else "assembled"}
            for which, name in ((1, "local"), (2, "coarse"), (3, "both")):
                ms = timed(lambda: c.schwarz_apply(b, z, which), st, 20)   # graph on
                c.timing(True)
                timed(lambda: c.schwarz_apply(b, z, which), st, 5)
                t_fdm, k_fdm = c.timing_read(7)
                t_cmb, k_cmb = c.timing_read(8)
                c.timing(False)
                res[f"apply_{name}_ms"] = round(ms, 4)
                if which == 1 and k_fdm:
                    fdm_ms = t_fdm / k_fdm
                    bpp = 17.0 + 24.0 * (n1 * n1 + n1) / n1 ** 3
                    res["fdm_kernel_ms"] = round(fdm_ms, 4)
                    res["fdm_B_per_pt"] = round(bpp, 2)
                    res["fdm_GBps"] = round(bpp * n / (fdm_ms * 1e-3) / 1e9, 0)
                    res["fdm_frac_copy"] = round(bpp * n / (fdm_ms * 1e-3) / 1e9 / peak_copy(), 3)
                    res["combine_kernel_ms"] = round(t_cmb / max(k_cmb, 1), 4)
                    if n1 == 8:   # the CUDA-core kernel for comparison
                        c.set_fdm_tc(False)
                        c.timing(True)
                        timed(lambda: c.schwarz_apply(b, z, 1), st, 5)
                        t2, k2 = c.timing_read(7)
                        c.timing(False)
                        c.set_fdm_tc(True)
                        res["fdm_cuda_core_kernel_ms"] = round(t2 / max(k2, 1), 4)
            for pc in ("jacobi", "schwarz"):
                c.set_precond(pc)
                for solver in ("pcg", "gmres"):
                    x = c.zeros()
                    # Jacobi GMRES needs thousands of iterations on C3/C4: capped at
                    # 300 (ms_per_iter is the comparable number there)
                    mi = 300 if (solver == "gmres" and pc == "jacobi") else 3000
                    fn = (lambda: c.pcg_solve(b, x, 1e-10, mi)) if solver == "pcg" else \
                        (lambda: c.gmres_solve(b, x, 1e-10, mi, 30))
                    fn()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    r = fn()
                    e1.record(st)
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                    res[f"{solver}_{pc}"] = {"iters": r["iters"], "status": r["status"],
                                             "ms": round(ms, 3), "res_true": r["res_true"],
                                             "ms_per_iter": round(ms / max(r["iters"], 1), 4)}
            c.set_precond("jacobi")
            out(res)


def pcg_rate(c, st, iters):
    """fixed-iteration PCG (tol 0) on the TGV right-hand side: iter/s, GDOF/s"""
    X, Y, Z = c.coords()
    b = c.zeros()
    c.rhs(f_tgv(X, Y, Z, xp=torch), b)
    del X, Y, Z
    x = c.zeros()
    c.pcg_solve(b, x, 0.0, 5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    r = c.pcg_solve(b, x, 0.0, iters)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return {"iters": r["iters"], "ms": round(ms, 3), "iter_per_s": round(r["iters"] / (ms * 1e-3), 1),
            "gdofs": round(c.n_local * r["iters"] / (ms * 1e-3) / 1e9, 2)}


def single():
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    tri = triad(st)
    out({"what": "triad", "GBps": round(tri, 0), "copy_peak_GBps": peak_copy(),
         "gpu": torch.cuda.get_device_name(0)})
    # C3: Ax / Ax+gs rates (where the >=60% target is evaluated) and the PCG solve to tol
    spec, N = CONFIGS["C3"]
    with sem.sem_setup(spec, N, stream=st.cuda_stream) as c:
        out({"what": "C3_ops", "n_p": c.n_local, **op_rates(c, N, st, 50, tri)})
        X, Y, Z = c.coords()
        b = c.zeros()
        c.rhs(f_tgv(X, Y, Z, xp=torch), b)
        x = c.zeros()
        c.pcg_solve(b, x, 1e-10, 5000)   # warm
        x.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        r = c.pcg_solve(b, x, 1e-10, 5000)
        e1.record(st)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms = e0.elapsed_time(e1)
        B = torch.from_numpy(c.export_field("B")).cuda()
        xm = x - (B * x).sum() / B.sum()                       # reading Q18
        einf = float((xm - p_tgv(X, Y, Z, xp=torch)).abs().max())
        out({"what": "C3_pcg_to_tol", "tol": 1e-10, "iters": r["iters"], "status": r["status"],
             "res_final": r["res_final"], "res_true": r["res_true"], "ms": round(ms, 2),
             "wall_s": round(wall, 4), "iter_per_s": round(r["iters"] / (ms * 1e-3), 1),
             "gdofs": round(c.n_local * r["iters"] / (ms * 1e-3) / 1e9, 2), "e_inf_vs_p*": einf})
        del X, Y, Z, b, x, B, xm
    torch.cuda.empty_cache()
    # C4 at P = 1: deformed 64^3, all 6 factors nonzero
    spec, N = CONFIGS["C4"]
    with sem.sem_setup(spec, N, stream=st.cuda_stream) as c:
        out({"what": "C4_ops_P1", "n_p": c.n_local, **op_rates(c, N, st, 10, tri)})
        out({"what": "C4_pcg_P1", **pcg_rate(c, st, 50)})
    torch.cuda.empty_cache()
    sweep(range(1, 12), st, tri)


def sweep(Ns, st=None, tri=None):
    """N sweep at fixed n_p ~ 1.25e8 (SURVEY C5 per-GPU size: E_axis = 500/(N+1))"""
    if st is None:
        torch.cuda.set_device(0)
        st = torch.cuda.current_stream()
        tri = triad(st)
    for N in Ns:
        ea = int(round(500.0 / (N + 1)))
        ez = max(8, int(round(ea / 8.0)) * 8)
        spec = tgv_box(ea, ea, ez)
        t0 = time.perf_counter()
        with sem.sem_setup(spec, N, stream=st.cuda_stream) as c:
            setup_s = time.perf_counter() - t0
            fb, _, baxgs = bytes_model(N)
            out({"what": "sweep", "N": N, "mesh": [ea, ea, ez], "E": spec.E, "n_p": c.n_local,
                 "f_b": round(fb, 3), "ax_gs_B_per_pt": round(baxgs, 1), "setup_s": round(setup_s, 1),
                 **op_rates(c, N, st, 10, tri)})
        torch.cuda.empty_cache()


def c5(Ns):
    """BASELINE configs[4] at its stated size: per N, E_axis = round(1000/(N+1)) in x, y and z
    rounded to a multiple of 8 (sem_inputs.c5_mesh), n_p ~ 1e9 local points on ONE GPU:
    Ax, Ax+gs (both gs schedules) and a 20-iteration Jacobi-PCG (b = A u, tol 0)."""
    from sem_inputs import c5_mesh
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    tri = triad(st)
    for N in Ns:
        spec = c5_mesh(N)
        t0 = time.perf_counter()
        with sem.sem_setup(spec, N, stream=st.cuda_stream) as c:
            setup_s = time.perf_counter() - t0
            fb, _, baxgs = bytes_model(N)
            res = {"what": "c5", "N": N, "mesh": [spec.ex, spec.ey, spec.ez], "E": spec.E,
                   "n_p": c.n_local, "f_b": round(fb, 3), "ax_gs_B_per_pt": round(baxgs, 1),
                   "setup_s": round(setup_s, 1), "triad_GBps": round(tri, 0),
                   **op_rates(c, N, st, 5, tri)}
            u = torch.empty(c.n_local, dtype=torch.float64, device="cuda").uniform_(-1, 1)
            b = c.zeros()
            c.apply(u, b)
            del u
            x = c.zeros()
            c.pcg_solve(b, x, 0.0, 4)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            r = c.pcg_solve(b, x, 0.0, 20)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            res["pcg"] = {"iters": r["iters"], "ms": round(ms, 2),
                          "iter_per_s": round(r["iters"] / (ms * 1e-3), 2),
                          "gdofs": round(c.n_local * r["iters"] / (ms * 1e-3) / 1e9, 2)}
            del b, x
            out(res)
        torch.cuda.empty_cache()


def strong():
    import torch.distributed as dist
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [sem.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = sem.nccl_comm_init(uid[0], rank, P)
    st = torch.cuda.current_stream()

    def mx(v):
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for cfg in ("C3", "C4"):
        spec, N = CONFIGS[cfg]
        with sem.sem_setup(spec, N, rank=rank, nranks=P, nccl_comm=comm, stream=st.cuda_stream) as c:
            n_tot = spec.E * (N + 1) ** 3
            u = torch.empty(c.n_local, dtype=torch.float64, device="cuda").uniform_(-1, 1)
            w = c.zeros()
            ms = mx(timed(lambda: c.apply(u, w), st, 20, sync=dist.barrier))
            p = pcg_rate(c, st, 100 if cfg == "C3" else 40)
            pms = mx(p["ms"])
            if rank == 0:
                out({"what": f"{cfg}_strong", "P": P, "n_p_total": n_tot,
                     "ax_gs_ms": round(ms, 4), "ax_gs_gdofs": round(n_tot / (ms * 1e-3) / 1e9, 2),
                     "pcg_iters": p["iters"], "pcg_ms": round(pms, 3),
                     "pcg_iter_per_s": round(p["iters"] / (pms * 1e-3), 1),
                     "pcg_gdofs": round(n_tot * p["iters"] / (pms * 1e-3) / 1e9, 2)})
            del u, w
        torch.cuda.empty_cache()
    sem.nccl_comm_destroy(comm)
    dist.destroy_process_group()


def c5_scale(Ns, kind):
    """BASELINE configs[4] scaling at ~1e9 DOF (torchrun, one rank per GPU):
    strong = the ~1e9-point C5 mesh of order N over P GPUs; weak = ~1e9 points per
    GPU (the C5 mesh stacked P times along z).  Per N: operator (Ax + gs with the
    exchange) and a 20-iteration Jacobi-PCG (b = A u, tol 0), max over ranks."""
    import torch.distributed as dist
    from sem_inputs import c5_mesh, weak_scaled
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [sem.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = sem.nccl_comm_init(uid[0], rank, P)
    st = torch.cuda.current_stream()

    def mx(v):
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for N in Ns:
        spec = c5_mesh(N) if kind == "strong" else weak_scaled(c5_mesh(N), P)
        t0 = time.perf_counter()
        with sem.sem_setup(spec, N, rank=rank, nranks=P, nccl_comm=comm, stream=st.cuda_stream) as c:
            setup_s = mx(time.perf_counter() - t0)
            n_tot = spec.E * (N + 1) ** 3
            u = torch.empty(c.n_local, dtype=torch.float64, device="cuda").uniform_(-1, 1)
            b = c.zeros()
            ms = mx(timed(lambda: c.apply(u, b), st, 5, sync=dist.barrier))
            del u
            x = c.zeros()
            c.pcg_solve(b, x, 0.0, 3)
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            r = c.pcg_solve(b, x, 0.0, 20)
            e1.record(st)
            torch.cuda.synchronize()
            pms = mx(e0.elapsed_time(e1))
            if rank == 0:
                out({"what": f"c5_{kind}", "P": P, "N": N, "mesh": [spec.ex, spec.ey, spec.ez],
                     "n_p_total": n_tot, "setup_s": round(setup_s, 1),
                     "ax_gs_ms": round(ms, 3), "ax_gs_gdofs": round(n_tot / (ms * 1e-3) / 1e9, 2),
                     "pcg_iters": r["iters"], "pcg_ms": round(pms, 2),
                     "pcg_gdofs": round(n_tot * r["iters"] / (pms * 1e-3) / 1e9, 2)})
            del b, x
        torch.cuda.empty_cache()
        dist.barrier()
    sem.nccl_comm_destroy(comm)
    dist.destroy_process_group()


def schwarz_strong(cfgs=("C3", "C4")):
    """NEXT-1 at P ranks: time-to-solution (tol 1e-10, TGV pressure RHS) of
    Jacobi-PCG, Schwarz flexible PCG and Schwarz flexible GMRES(30); the
    coarse N=1 solve runs distributed over the same ranks (its ten CG steps
    each carry a gather-scatter exchange and two allreduces)."""
    import torch.distributed as dist
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [sem.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = sem.nccl_comm_init(uid[0], rank, P)
    st = torch.cuda.current_stream()

    def mx(v):
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for cfg in cfgs:
        spec, N = CONFIGS[cfg]
        with sem.sem_setup(spec, N, rank=rank, nranks=P, nccl_comm=comm, stream=st.cuda_stream) as c:
            X, Y, Z = c.coords()
            b = c.zeros()
            c.rhs(f_tgv(X, Y, Z, xp=torch), b)
            del X, Y, Z
            res = {"what": f"{cfg}_schwarz_strong", "P": P}
            runs = [("jacobi", "pcg", -1), ("schwarz", "pcg", 0), ("schwarz", "gmres", 0)]
            if P > 1:   # the replicated coarse solve (one all-gather, no per-step collectives)
                runs += [("schwarz", "pcg", 1), ("schwarz", "gmres", 1)]
            for pc, solver, rep in runs:
                c.set_precond(pc)
                if pc == "schwarz":
                    c.set_coarse_replicate(rep)
                x = c.zeros()
                fn = (lambda: c.pcg_solve(b, x, 1e-10, 3000)) if solver == "pcg" else \
                    (lambda: c.gmres_solve(b, x, 1e-10, 3000, 30))
                fn()
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                r = fn()
                e1.record(st)
                torch.cuda.synchronize()
                ms = mx(e0.elapsed_time(e1))
                key = f"{solver}_{pc}" + ("_replicated" if rep == 1 else "")
                res[key] = {"iters": r["iters"], "status": r["status"], "ms": round(ms, 3)}
            c.set_precond("jacobi")
            if rank == 0:
                out(res)
        torch.cuda.empty_cache()
    sem.nccl_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "single"
    if mode == "strong":
        strong()
    elif mode == "sweep":
        sweep([int(v) for v in sys.argv[2].split(",")])
    elif mode == "c5":
        c5([int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else range(1, 12))
    elif mode in ("c5_strong", "c5_weak"):   # torchrun: C5 scaling at ~1e9 DOF
        c5_scale([int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else (3, 7, 11),
                 mode[3:])
    elif mode == "schwarz_strong":
        schwarz_strong(tuple(sys.argv[2].split(",")) if len(sys.argv) > 2 else ("C3", "C4"))
    elif mode == "schwarz":
        schwarz(tuple(sys.argv[2].split(",")) if len(sys.argv) > 2 else ("C3", "C4"))
    elif mode == "helm":
        helm(sys.argv[2] if len(sys.argv) > 2 else "C3")
    elif mode == "ops":   # Ax / Ax+gs rates (all gs schedules) on named configs
        torch.cuda.set_device(0)
        st0 = torch.cuda.current_stream()
        tri0 = triad(st0)
        for cfg in sys.argv[2].split(","):
            spec, N = CONFIGS[cfg]
            with sem.sem_setup(spec, N, stream=st0.cuda_stream) as c:
                out({"what": f"{cfg}_ops", "n_p": c.n_local, **op_rates(c, N, st0, 50, tri0)})
            torch.cuda.empty_cache()
    else:
        single()
