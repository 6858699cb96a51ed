"""Per-phase timing of the multi-GPU hot path (torchrun, one rank per GPU).
C2 box per GPU stacked along z.  Prints, for each transport (peer memory /
NCCL): apply (Ax+gs with exchange) and PCG-iteration times, max over ranks."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import CONFIGS, f_tgv, weak_scaled  # noqa: E402


def main():
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [sem.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = sem.nccl_comm_init(uid[0], rank, P)
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    spec1, N = CONFIGS[cfg]
    spec = weak_scaled(spec1, P)
    st = torch.cuda.current_stream()
    res = {}
    with sem.sem_setup(spec, N, rank=rank, nranks=P, nccl_comm=comm, stream=st.cuda_stream) as c:
        X, Y, Z = c.coords()
        s = 2 * math.pi
        b = c.zeros()
        c.rhs(f_tgv(s * X, s * Y, s * Z, xp=torch), b)
        x, w = c.zeros(), c.zeros()
        u = torch.empty(c.n_local, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def timed(fn, reps):
            fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0.record(st)
            for _ in range(reps):
                fn()
            e1.record(st)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item()) * 1e3

        for p2p, ov in ((True, True), (True, False), (False, True)):
            c.set_p2p(p2p)
            c.set_overlap(ov)
            tag = ("p2p" if p2p else "nccl") + ("_ov" if ov else "_noov")
            res[f"{tag}_apply_us"] = timed(lambda: c.apply(u, w), 50)
            res[f"{tag}_gs_us"] = timed(lambda: c.gs(w), 50)
            res[f"{tag}_pcg_iter_us"] = timed(lambda: c.pcg_solve(b, x, 0.0, 40), 3) / 40
            c.timing(True)
            c.pcg_solve(b, x, 0.0, 40)
            for k, nm in ((0, "ax"), (1, "upd"), (2, "p"), (4, "gs"), (5, "pack"), (6, "unpack")):
                ms, cnt = c.timing_read(k)
                res[f"{tag}_k_{nm}_us"] = ms * 1e3 / 41
            c.timing(False)
        res["ax_only_us"] = timed(lambda: c.ax(u, w), 50)
        c.set_p2p(True)
        c.set_overlap(False)
        def xts():
            xt = c.debug_read(0, 5 * 2048).reshape(5, 2048)
            nb = int((xt[0] > 0).sum())
            xt = xt[:, :nb].astype(np.float64)
            rel = (xt - xt[0].min()) / 1e3
            summ = {"grid": nb}
            for name, sl in (("pack", slice(0, 64)), ("rest", slice(nb - 256, nb))):
                for ph, pn in enumerate(("start", "packed", "local", "unpacked", "end")):
                    v = rel[ph, sl]
                    summ[f"{name}_{pn}"] = [round(float(np.min(v)), 2), round(float(np.median(v)), 2),
                                             round(float(np.max(v)), 2)]
            summ["local_max"] = round(float(rel[2].max()), 2)
            summ["end_max"] = round(float(rel[4].max()), 2)
            return summ

        c.pcg_solve(b, x, 0.0, 5)
        summ = {"pcg": xts()}
        for _ in range(10):
            c.gs(w)
        summ["gs"] = xts()
        allx = [None] * P
        dist.all_gather_object(allx, summ)
        res["n_shared"] = float(c.n_local)
    if rank == 0:
        print(json.dumps({"P": P, "cfg": cfg, **{k: round(v, 2) for k, v in res.items()}}))
        for r, sm in enumerate(allx):
            for k, v in sm.items():
                print(json.dumps({"rank": r, "ctx": k, **v}))
    sem.nccl_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
