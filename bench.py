#!/usr/bin/env python
"""Benchmark of the B200-native SEM pressure-Poisson hot path.

A "step" is one Jacobi-PCG iteration over the whole hot path:
Ax+mask with <p,Ap> fused, the gather-scatter (with, for N > 1,
the NVLink peer-memory exchange of shared entities, Alg. 1, and the allreduce),
the r update with <r,z>_c and <r,r>_c, the convergence test and the x and p
updates.

Workload (BASELINE.json configs[1], default --config C2): the 8192-element
Cartesian box (32x16x16 elements, N=7, all 6 geometric factors stored and
streamed, BP5 convention) per GPU; with N GPUs the box is stacked N times
along z and partitioned into z-slabs (weak scaling, one slab of 8192 elements
per GPU).  --config C4 is the strong-scaling workload (BASELINE configs[3]:
the 64^3-element deformed mesh split over the N GPUs).  At N=1 the line also
carries the north-star Ax+gs number on C3 (BASELINE configs[2], working set
>> L2, rotating operands).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sem|reference]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run (one rank per GPU, rendezvous on 127.0.0.1).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 Ax+gather-scatter GDOF/s and PCG iter/s at 1-8 B200; % HBM roofline"
UNIT = "GDOF/s"
E2E_TOL, E2E_MAXIT = 1e-10, 5000   # one end-to-end step: a host solve of b -> x to tolerance


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="sem", choices=["sem", "reference"])
    ap.add_argument("--config", default="C2", choices=["C2", "C3", "C4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 Ax+gs block (N=1)")
    return ap.parse_args()


def strong(cfg):
    """C4 (BASELINE configs[3]) is the strong-scaling workload: fixed total mesh."""
    return cfg == "C4"


def workload(cfg, P):
    """(mesh of the whole job, N, mesh per GPU at N=1)."""
    from sem_inputs import CONFIGS, weak_scaled
    spec, N = CONFIGS[cfg]
    return (spec if strong(cfg) else weak_scaled(spec, P)), N, spec


def relaunch(args):
    """--gpus N > 1 without a torchrun environment: start N ranks ourselves."""
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.run(cmd, env=env).returncode


def bytes_model(N):
    """SURVEY 8(d) per-point algorithmic bytes (paper Eq. 12 Q, cold cache)."""
    fb = 1.0 - ((N - 1) / (N + 1)) ** 3           # fraction of slots on element faces
    return {"f_b": fb, "ax": 64.0, "ax_pf": 88.0, "ax_gs": 64.0 + 20.0 * fb,
            "pcg_iter_fused": 152.0 + 20.0 * fb, "flops_ax": 12 * (N + 1) + 15}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line).
    One sampler per node (local rank 0, every local GPU), started before the
    warm-up and given a second to initialise: a per-rank nvidia-smi starting
    at the timed region stalled kernel launches on all ranks (one 4-GPU C4
    run measured 3.2 instead of 1.04 ms per iteration)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, indices, settle=0.5):
        self.indices, self.proc, self.settle, self.first = indices, None, settle, []

    def __enter__(self):
        if not self.indices:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--id=" + ",".join(str(i) for i in self.indices),
                 f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            # wait until the sampler has initialised (its first rows are out), so
            # the NVML start-up cannot overlap the timed region
            import select
            if select.select([self.proc.stdout], [], [], 15.0)[0]:
                for _ in self.indices:
                    self.first.append(self.proc.stdout.readline())
            time.sleep(self.settle)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in self.first + out.splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return None
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in self.rows for q in range(4)
                          if r[5 + q].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------------------- oracle arm
def oracle_pcg_rate(spec, N, target_s=15.0, max_iters=None):
    """Time the CPU oracle (as it stands) doing PCG iterations on `spec`."""
    import oracle as O
    from sem_inputs import f_tgv
    o = O.Oracle(spec, N)
    s = 2 * math.pi
    b = o.rhs(f_tgv(s * o.get("X"), s * o.get("Y"), s * o.get("Z")))
    t0 = time.perf_counter()
    o.pcg(b, 0.0, 1)
    t1 = time.perf_counter() - t0
    it = max(1, int(target_s / max(t1, 1e-3)))
    if max_iters:
        it = min(it, max_iters)
    t0 = time.perf_counter()
    r = o.pcg(b, 0.0, it)
    dt = time.perf_counter() - t0
    return {"iters": r["iters"], "seconds": dt, "n_p": o.nslots,
            "gdofs": o.nslots * r["iters"] / dt / 1e9}


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    _, N, spec1 = workload(args.config, 1)
    if strong(args.config):   # per-GPU share of the strong-scaling mesh
        from dataclasses import replace
        ezp = max(1, spec1.ez // max(args.gpus, 1))
        spec1 = replace(spec1, ez=ezp, z1=spec1.z0 + (spec1.z1 - spec1.z0) * ezp / spec1.ez)
    from dataclasses import replace
    # bounded sample: shrink the z extent so K+W oracle iterations stay ~minutes
    probe = replace(spec1, ez=2, z1=spec1.z0 + (spec1.z1 - spec1.z0) * 2 / spec1.ez)
    rp = oracle_pcg_rate(probe, N, target_s=2.0, max_iters=3)
    per_elem_s = rp["seconds"] / rp["iters"] / probe.E
    budget = 150.0 / max(args.steps + args.warmup, 1)     # seconds per step
    ez = max(2, min(spec1.ez, int(budget / (per_elem_s * spec1.ex * spec1.ey))))
    sample = replace(spec1, ez=ez, z1=spec1.z0 + (spec1.z1 - spec1.z0) * ez / spec1.ez)
    import oracle as O
    from sem_inputs import f_tgv
    o = O.Oracle(sample, N)
    s = 2 * math.pi
    b = o.rhs(f_tgv(s * o.get("X"), s * o.get("Y"), s * o.get("Z")))
    if args.warmup:
        o.pcg(b, 0.0, args.warmup)
    t0 = time.perf_counter()
    r = o.pcg(b, 0.0, args.steps)
    dt = time.perf_counter() - t0
    value = o.nslots * args.steps / dt / 1e9
    desc = (f"oracle PCG, {args.steps} iterations (tol=0) on a {sample.ex}x{sample.ey}x{sample.ez}"
            f"-element slice of the {args.config} box, N={N}, {o.nslots} slots")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if strong(args.config) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(args.config, args.gpus),
                       "step": "one Jacobi-PCG iteration"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "iters": r["iters"]}
    print(json.dumps(line), flush=True)
    return 0


def workload_desc(cfg, P):
    from sem_inputs import CONFIGS
    spec1, N = CONFIGS[cfg]
    if strong(cfg):
        return (f"{cfg}: {spec1.ex}x{spec1.ey}x{spec1.ez} elements in total (strong scaling, "
                f"z-slabs over {P} GPU(s)), N={N}, periodic, deformed (a={spec1.deform_amp})")
    return (f"{cfg}: {spec1.ex}x{spec1.ey}x{spec1.ez} elements per GPU (box stacked x{P} along z), "
            f"N={N}, periodic, all 6 G stored")


def time_applies(ctx, sets, reps, stream, barrier, max_over_ranks):
    """sem_apply over rotating (u, w) operand sets; returns ms per apply and the
    per-kernel split (Ax+mask, gs) from the context's CUDA-event timers."""
    import torch
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for q in range(3):
        u, w = sets[q % len(sets)]
        ctx.apply(u, w)
    barrier()
    ev0.record(stream)
    for q in range(reps):
        u, w = sets[q % len(sets)]
        ctx.apply(u, w)
    ev1.record(stream)
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1)) / reps
    ctx.timing(True)
    for q in range(reps):
        u, w = sets[q % len(sets)]
        ctx.apply(u, w)
    ax_ms, ax_n = ctx.timing_read(0)
    gs_ms, gs_n = ctx.timing_read(4)
    ctx.timing(False)
    return ms, ax_ms / max(ax_n, 1), gs_ms / max(gs_n, 1)


def c3_block(sem, stream, barrier, peak, reps):
    """North-star number: fp64 Ax+gs on C3 (32^3 elements, N=7,
    u and w 134 MB each), two rotating (u, w) sets so no operand is reused
    while L2-resident (P:L355, P:L361 cold-cache Q)."""
    import torch
    from sem_inputs import CONFIGS
    spec, N = CONFIGS["C3"]
    ctx = sem.sem_setup(spec, N, stream=stream.cuda_stream)
    nl = ctx.n_local
    sets = []
    for q in range(2):
        u = torch.empty(nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        sets.append((u, ctx.zeros()))
    ms, ax_ms, gs_ms = time_applies(ctx, sets, reps, stream, barrier, lambda v: v)
    bm = bytes_model(N)
    out = {"workload": "C3: 32x32x32 elements, N=7, (0,2pi)^3 periodic; 2 rotating (u, w) sets "
                       "(536 MB of operands + 805 MB G >> 126 MB L2)",
           "n_p": nl, "gdofs": nl / (ms / 1e3) / 1e9, "ms": ms,
           "bytes_per_pt": bm["ax_gs"],
           "frac_of_8TBps": nl * bm["ax_gs"] / (ms / 1e3) / 8e12,
           "frac_of_measured": nl * bm["ax_gs"] / (ms / 1e3) / 1e9 / peak,
           "ax_ms": ax_ms, "gs_ms": gs_ms,
           "ax_frac_of_measured": nl * 64.0 / (ax_ms / 1e3) / 1e9 / peak,
           "gs_frac_of_measured": nl * 20.0 * bm["f_b"] / (gs_ms / 1e3) / 1e9 / peak}
    del sets
    ctx.close()
    return out


# --------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "sem":
        return relaunch(args)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    import paper_2107_01243_b200 as sem
    from paper_2107_01243_b200 import build as sem_build
    from sem_inputs import f_tgv

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    P = world
    if args.gpus != P and P > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {P}")
    torch.cuda.set_device(local)
    dist = None
    if P > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        sem_build.build()
    if dist:
        dist.barrier()
    sem.load()

    spec, N, spec1 = workload(args.config, P)
    comm = None
    if P > 1:
        uid = [sem.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = sem.nccl_comm_init(uid[0], rank, P)
    stream = torch.cuda.current_stream()
    ctx = sem.sem_setup(spec, N, rank=rank, nranks=P, nccl_comm=comm, stream=stream.cuda_stream)
    nl = ctx.n_local
    n_p_total = nl * P

    # synthetic right-hand side: TGV pressure forcing on the unit box (x 2 pi)
    X, Y, Z = ctx.coords()
    s = 2 * math.pi
    f = f_tgv(s * X, s * Y, s * Z, xp=torch)
    b = ctx.zeros()
    ctx.rhs(f, b)
    x = ctx.zeros()
    del X, Y, Z, f
    torch.cuda.synchronize()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # the node's clock sampler runs from before the warm-up through the timed region
    n_node = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    with Clocks(list(range(n_node)) if local == 0 else []) as clk:
        # ---- warm-up (W iterations)
        ctx.pcg_solve(b, x, 0.0, max(args.warmup, 3))
        barrier()

        # ---- timed: exactly K PCG iterations (one solve, tol=0)
        l0 = ctx.launch_count()
        barrier()
        ev0.record(stream)
        res = ctx.pcg_solve(b, x, 0.0, args.steps)
        ev1.record(stream)
        barrier()
    launches = ctx.launch_count() - l0
    t_ms = max_over_ranks(ev0.elapsed_time(ev1))
    assert res["iters"] == args.steps, res
    value = n_p_total * args.steps / (t_ms / 1e3) / 1e9

    # ---- dominant kernel (Ax + mask + sigma), CUDA events on the context stream
    ctx.timing(True)
    ctx.pcg_solve(b, x, 0.0, args.steps)
    # the Ax kernel with the fused p update is timer class 9 (the final
    # true-residual apply, class 0, is excluded); per iteration
    k_ms, k_cnt = ctx.timing_read(9)
    u_ms, u_cnt = ctx.timing_read(1)
    p_ms, p_cnt = ctx.timing_read(2)
    g_ms, g_cnt = ctx.timing_read(4)
    ctx.timing(False)
    # per operator application (the split Alg. 1 operator launches the kernel
    # twice per application at N > 1): steps iterations + 1 true-residual apply
    n_apply = args.steps
    k_avg = max_over_ranks(k_ms / n_apply)
    bm = bytes_model(N)
    peak, peak_src = peaks()
    # the Ax kernel also performs the p update (PF): p_old, r, dinv in, p out
    pf = True
    kbytes = bm["ax_pf"] if pf else bm["ax"]
    achieved = nl * kbytes / (k_avg / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fjs:
            tj = json.load(fjs)
        key = f"{args.config}_N{N}_P1"
        if key in tj:
            traffic = tj[key]["dram_bytes_per_launch"]
    except Exception:
        pass

    # ---- Ax+gs alone (sem_apply) over 4 rotating (u, w) sets (268 MB/GPU of
    # operands > L2 at C2), and Ax alone, K repetitions each
    sets = []
    for q in range(4):
        u = torch.empty(nl, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        sets.append((u, ctx.zeros()))
    apply_ms, apply_ax_ms, apply_gs_ms = time_applies(ctx, sets, args.steps, stream, barrier,
                                                      max_over_ranks)
    ev0.record(stream)
    for q in range(args.steps):
        u, w = sets[q % 4]
        ctx.ax(u, w)
    ev1.record(stream)
    barrier()
    ax_ms = max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
    del sets

    # ---- end to end through the C ABI with HOST buffers (pinned): one step is
    # the call a user makes -- H2D of b, Jacobi-PCG to the absolute tolerance
    # 1e-10 (reading Q15), D2H of x -- and the metric counts its iterations
    e2e = None
    if not args.no_e2e:
        bh = torch.empty(nl, dtype=torch.float64, pin_memory=True)
        bh.copy_(b)
        xh = torch.empty(nl, dtype=torch.float64, pin_memory=True)
        bn, xn = bh.numpy(), xh.numpy()
        barrier()
        t0 = time.perf_counter()
        r1 = ctx.pcg_solve_host(bn, xn, E2E_TOL, E2E_MAXIT)   # warm (graph capture)
        t1 = max_over_ranks(time.perf_counter() - t0)
        e2e_steps = int(max(1, min(5, 8.0 / max(t1, 1e-3))))
        barrier()
        t0 = time.perf_counter()
        its = 0
        for _ in range(e2e_steps):
            r1 = ctx.pcg_solve_host(bn, xn, E2E_TOL, E2E_MAXIT)
            its += r1["iters"]
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": n_p_total * its / e2e_s / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 8 * n_p_total, "d2h_bytes_per_step": 8 * n_p_total,
               "step": (f"sem_pcg_solve_host: H2D b, Jacobi-PCG to tol {E2E_TOL:g} "
                        f"({r1['iters']} iterations, status {r1['status']}, true residual "
                        f"{r1['res_true']:.2e}), D2H x"),
               "steps": e2e_steps, "ms_per_solve": e2e_s / e2e_steps * 1e3}

    # ---- CPU baseline: the oracle as it stands, rank 0 at N=1 only
    cpu = None
    if rank == 0 and P == 1 and not args.no_cpu_baseline:
        from dataclasses import replace
        sample = replace(spec1, ez=4, z1=spec1.z0 + (spec1.z1 - spec1.z0) * 4 / spec1.ez)
        r = oracle_pcg_rate(sample, N, target_s=12.0)
        cpu = {"value": r["gdofs"], "unit": UNIT, "cores": cores(), "kind": "oracle",
               "sample": (f"oracle PCG (plain C, OpenMP Ax, serial gs/dots) {r['iters']} "
                          f"iterations on a {sample.ex}x{sample.ey}x{sample.ez}-element slice of "
                          f"the {args.config} box, N={N} ({r['n_p']} slots), {r['seconds']:.1f} s")}

    c3 = None
    if P == 1 and not args.no_c3 and args.config == "C2":
        c3 = c3_block(sem, stream, barrier, peak, max(args.steps, 20))

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": P, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong(args.config) else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": workload_desc(args.config, P),
                "N": N, "elements": spec.E, "n_p": n_p_total, "n_glob": ctx.n_glob,
                "step": (("one Jacobi-PCG iteration, three kernels: p update + Ax + mask + <p,Ap> "
                          "kernel, gather-scatter kernel with the NVLink peer-memory exchange and "
                          "sigma allreduce, r and x update + <r,z>_c, <r,r>_c + allreduce + "
                          "convergence kernel") if P > 1 else
                         ("one Jacobi-PCG iteration, three kernels replayed as a CUDA graph: "
                          "p update + Ax + mask + <p,Ap> kernel, gather-scatter kernel, "
                          "r and x update + <r,z>_c, <r,r>_c + convergence kernel")),
                "l2": (f"no flush: per-iteration working set {nl * 104 / 1e6:.0f} MB/GPU "
                       "(G, u, w, r, p, x, dinv) > 126 MB L2"),
                "parallelism": (f"element z-slabs x{P}, NVLink peer-memory gs exchange + "
                                "allreduce (CUDA IPC)") if P > 1 else "single GPU",
            },
            "pcg_iter_per_s": args.steps / (t_ms / 1e3),
            "ax_gs": {"gdofs": n_p_total / (apply_ms / 1e3) / 1e9, "ms": apply_ms,
                      "frac_of_8TBps": nl * bm["ax_gs"] / (apply_ms / 1e3) / 8e12,
                      "frac_of_measured": nl * bm["ax_gs"] / (apply_ms / 1e3) / 1e9 / peak,
                      "ax_ms": apply_ax_ms, "gs_ms": apply_gs_ms,
                      "operands": "4 rotating (u, w) sets"},
            "ax_gs_c3": c3,
            "ax_only": {"gdofs": n_p_total / (ax_ms / 1e3) / 1e9, "ms": ax_ms,
                        "gbs_64B_per_pt": nl * 64 / (ax_ms / 1e3) / 1e9},
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": (f"ax_kernel<{N + 1},AX_PCG,PF> (p = dinv r + beta p, Ax, mask, sigma)"
                           if pf else f"ax_kernel<{N + 1},AX_PCG> (Ax+mask+sigma)"),
                "bytes_per_pt": kbytes, "hbm_mandatory_bytes_per_pt": kbytes,
                "avg_ms_per_apply": k_avg, "launches": k_cnt, "applies": n_apply,
                "peak_source": peak_src,
                "step_share": k_ms / max(k_ms + u_ms + p_ms + g_ms, 1e-9),
                "other_kernels_ms_per_step": {"gs": g_ms / max(g_cnt, 1),
                                              "cg_update": u_ms / max(u_cnt, 1),
                                              "cg_p": p_ms / max(p_cnt, 1)},
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
            "res_final": res["res_final"],
        }
        print(json.dumps(line), flush=True)

    ctx.close()
    if comm is not None:
        sem.nccl_comm_destroy(comm)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
