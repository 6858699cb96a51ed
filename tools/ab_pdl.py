"""A/B of programmatic dependent launch in the PCG loop (C2 per GPU, weak).
  python tools/ab_pdl.py            (or under torchrun for P > 1)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2107_01243_b200 as sem  # noqa: E402
from sem_inputs import CONFIGS, f_tgv, weak_scaled  # noqa: E402


def main():
    P = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm, dist = None, None
    if P > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [sem.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = sem.nccl_comm_init(uid[0], rank, P)
    spec, N = CONFIGS["C2"]
    st = torch.cuda.current_stream()
    res = {}
    with sem.sem_setup(weak_scaled(spec, P), N, rank=rank, nranks=P, nccl_comm=comm,
                       stream=st.cuda_stream) as c:
        X, Y, Z = c.coords()
        b = c.zeros()
        c.rhs(f_tgv(6.283185307179586 * X, 6.283185307179586 * Y, 6.283185307179586 * Z, xp=torch), b)
        x = c.zeros()
        for rep in range(3):
            for on in (False, True):
                c.set_pdl(on)
                c.pcg_solve(b, x, 0.0, 20)
                torch.cuda.synchronize()
                if dist:
                    dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                c.pcg_solve(b, x, 0.0, 200)
                e1.record(st)
                torch.cuda.synchronize()
                t = torch.tensor([e0.elapsed_time(e1) / 200 * 1e3], device="cuda", dtype=torch.float64)
                if dist:
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                res.setdefault("pdl" if on else "plain", []).append(round(float(t.item()), 2))
    if rank == 0:
        print(json.dumps({"P": P, "us_per_iter": res}))
    if comm is not None:
        sem.nccl_comm_destroy(comm)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
