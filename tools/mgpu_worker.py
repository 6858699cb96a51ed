"""Multi-GPU parity worker (launched by tests/test_multigpu.py under torchrun).

One process per GPU with an NCCL communicator; every rank runs the cases of
tools/mgpu_common.py through the C ABI with both transports (NVLink peer
memory, NCCL) and both gather-scatter schedules; rank 0 gathers the local
E-vectors and compares them with the oracle run with the same number of ranks
(bars in mgpu_common).  Exits non-zero on any mismatch.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from mgpu_common import CASES, OracleRefs, case_field, check, rank_run, rank_slice  # noqa: E402
from sem_inputs import random_field  # noqa: E402


def bench_config_check(rank, P, comm):
    """The bench's own multi-GPU configuration (C2 per GPU, weak-scaled along z,
    peer-memory transport, graph-replayed PCG with device-side epochs): the
    operator on a seeded random field normwise within 1e-12 of the oracle run
    with the same number of ranks, and 3 fixed PCG iterations (tol 0) on b = A u
    within 1e-10 of the oracle's iterate."""
    from sem_inputs import CONFIGS, weak_scaled
    spec = weak_scaled(CONFIGS["C2"][0], P)
    N = CONFIGS["C2"][1]
    u = random_field(spec.E * (N + 1) ** 3, seed=2024)
    lo, hi = rank_slice(spec, N, rank, P)
    fails = []
    with sem.sem_setup(spec, N, rank=rank, nranks=P, nccl_comm=comm) as c:
        du = torch.from_numpy(u[lo:hi]).cuda()
        w = c.zeros()
        c.apply(du, w)
        x = c.zeros()
        r = c.pcg_solve(w, x, 0.0, 3)
        torch.cuda.synchronize()
        out = {"w": w.cpu().numpy(), "x": x.cpu().numpy(), "iters": r["iters"]}
    parts = [None] * P
    dist.all_gather_object(parts, out)
    if rank == 0:
        import oracle as O
        o = O.Oracle(spec, N, nranks=P)
        wr = o.apply(u)
        W = np.concatenate([p["w"] for p in parts])
        e = np.abs(W - wr).max() / np.abs(wr).max()
        if not e <= 1e-12:
            fails.append(f"bench config P={P}: apply rel err {e:.2e}")
        ref = o.pcg(wr, 0.0, 3)
        X = np.concatenate([p["x"] for p in parts])
        dx = np.abs(X - ref["x"]).max()
        if parts[0]["iters"] != 3 or not dx <= 1e-10:
            fails.append(f"bench config P={P}: 3 PCG iterations x diff {dx:.2e}")
        print(f"bench config P={P} ({spec.ex}x{spec.ey}x{spec.ez}, N={N}): apply rel err {e:.2e}, "
              f"3-iteration PCG max |dx| {dx:.2e}", flush=True)
    return fails


def failure_path(rank, P, comm):
    """A rank that enters a peer-memory collective alone gets SEM_ENCCL after
    the bounded wait (~4 s; every later wait of that rank gives up at once),
    instead of hanging the GPU.  The other ranks keep their contexts (and
    mailboxes) alive until it returns."""
    spec, N, _ = CASES[1]
    fails = []
    with sem.sem_setup(spec, N, rank=rank, nranks=P, nccl_comm=comm) as c:
        c.set_p2p(True)
        if rank == 0:
            b = torch.rand(c.n_local, dtype=torch.float64, device="cuda")
            x = c.zeros()
            t0 = time.time()
            try:
                c.pcg_solve(b, x, 1e-10, 100)
                fails.append("failure path: a lone rank's PCG returned without error")
            except sem.SemError as e:
                if e.status != sem.SEM_ENCCL:
                    fails.append(f"failure path: status {e.status}, expected SEM_ENCCL")
            dt = time.time() - t0
            print(f"failure path: lone rank 0 PCG returned after {dt:.1f} s", flush=True)
            if dt > 30:
                fails.append(f"failure path took {dt:.1f} s")
        dist.barrier()
    return fails


def main():
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [sem.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = sem.nccl_comm_init(uid[0], rank, P)
    fails = []
    for ci, (spec, N, fun) in enumerate(CASES):
        u = case_field(ci, spec, N)
        lo, hi = rank_slice(spec, N, rank, P)
        ref = OracleRefs(spec, N, fun, u, P) if rank == 0 else None
        for p2p, gsm in ((True, 0), (True, 2), (False, 2)):
            with sem.sem_setup(spec, N, rank=rank, nranks=P, nccl_comm=comm) as c:
                c.set_p2p(p2p)
                c.set_gs_mode(gsm)
                assert c.n_local == hi - lo
                out = rank_run(c, u[lo:hi], fun)
                parts = [None] * P
                dist.all_gather_object(parts, out)
                if rank == 0:
                    tag = f"case{ci} P={P} p2p={p2p} gs_mode={gsm}"
                    f = check(parts, ref, tag)
                    fails += f
                    print(f"{tag}: {'FAIL' if f else 'ok'} pcg iters {out['r']['iters']} "
                          f"(oracle {ref.pcg['iters']})", flush=True)
    fails += bench_config_check(rank, P, comm)
    fails += failure_path(rank, P, comm)
    sem.nccl_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        for f in fails:
            print("FAIL", f, flush=True)
        print("RESULT", "FAIL" if fails else "PASS", flush=True)
        sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
